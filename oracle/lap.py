"""CPU restatement of the linear-assignment solver the reference calls.

TEST INFRASTRUCTURE ONLY. Nothing in the product package imports this module;
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may use it, and only as the checker.

The reference solves its padded square problem with
``scipy.optimize.linear_sum_assignment`` (``tf/assoc.py:76``), a third-party
dependency that is not vendored under ``/root/reference`` (pinned here by the
image: scipy 1.18.1). scipy documents it as "a modified Jonker-Volgenant
algorithm with no initialization" (D.F. Crouse, "On implementing 2D
rectangular assignment algorithms", IEEE TAES 2016): one shortest augmenting
path (Dijkstra over reduced costs) per row, rows taken in ascending order,
followed by a dual update and an augmentation along the path.

Which optimum is returned when several exist depends on three published
details of that algorithm, restated here because the GPU solver must make the
same choices:

* the candidate-column list starts in *descending* column order;
* when several columns share the minimum tentative distance, a column that is
  still unassigned (a sink) wins, and among equals the later list position
  wins for sinks, the earlier one otherwise;
* a visited column is removed from the list by moving the last entry into
  its slot.

``solve_square`` returns ``col4row`` for a square matrix and the number of
Dijkstra iterations it used (a cost model for the device solver).
"""

from __future__ import annotations

import math

import numpy as np


def solve_square(cost: np.ndarray) -> tuple[np.ndarray, int]:
    """Shortest-augmenting-path LAP on an n x n finite matrix (Crouse 2016)."""
    c = np.asarray(cost, dtype=np.float64)
    n = c.shape[0]
    assert c.shape == (n, n)
    u = [0.0] * n
    v = [0.0] * n
    col4row = [-1] * n
    row4col = [-1] * n
    iterations = 0
    for cur in range(n):
        dist = [math.inf] * n
        path = [-1] * n
        visited_rows = [False] * n
        visited_cols = [False] * n
        order = list(range(n - 1, -1, -1))
        live = n
        min_val = 0.0
        row = cur
        sink = -1
        while sink < 0:
            iterations += 1
            visited_rows[row] = True
            best_pos = -1
            best = math.inf
            for pos in range(live):
                col = order[pos]
                reduced = min_val + c[row, col] - u[row] - v[col]
                if reduced < dist[col]:
                    path[col] = row
                    dist[col] = reduced
                if dist[col] < best or (dist[col] == best and row4col[col] < 0):
                    best = dist[col]
                    best_pos = pos
            min_val = best
            if min_val == math.inf:
                raise ValueError("cost matrix is infeasible")
            col = order[best_pos]
            if row4col[col] < 0:
                sink = col
            else:
                row = row4col[col]
            visited_cols[col] = True
            live -= 1
            order[best_pos] = order[live]
        u[cur] += min_val
        for r in range(n):
            if visited_rows[r] and r != cur:
                u[r] += min_val - dist[col4row[r]]
        for col in range(n):
            if visited_cols[col]:
                v[col] -= min_val - dist[col]
        col = sink
        while True:
            r = path[col]
            row4col[col] = r
            col4row[r], col = col, col4row[r]
            if r == cur:
                break
    return np.asarray(col4row, dtype=np.int64), iterations


def brute_force(cost: np.ndarray) -> tuple[int, float]:
    """(max finite cardinality, min total) by exhaustive permutation; <= 7x7.

    Independent check of the objective pinned by ``tests/oracles.py:84-101``
    in the reference suite.
    """
    import itertools

    cost = np.asarray(cost, dtype=float)
    n_rows, n_cols = cost.shape
    n = max(n_rows, n_cols, 1)
    best = (-1, math.inf)
    for perm in itertools.permutations(range(n)):
        card, total = 0, 0.0
        for r in range(n_rows):
            col = perm[r]
            if col < n_cols and math.isfinite(cost[r, col]):
                card += 1
                total += cost[r, col]
        if card > best[0] or (card == best[0] and total < best[1]):
            best = (card, total)
    return best
