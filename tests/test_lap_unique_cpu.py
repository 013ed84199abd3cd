"""The near-optimum test the device applies after each component solve
(lap_unique, csrc/tf_device.cuh), restated in Python and checked against
brute force on small rectangular problems with many ties.

A component is solved from its smaller side: nr rows, all processed by the
shortest-augmenting-path solver, nc >= nr columns, non-entry cells at the
sentinel. The device keeps that solve only if no other row-perfect matching
with a different set of finite pairs costs within eps of the optimum; the
brute force enumerates every such matching.
"""

import itertools
import math

import numpy as np
import pytest


def sap_rect(cost, n_proc):
    """Crouse's shortest augmenting path on an n_proc x n cost matrix (all rows
    processed; the oracle/lap.py order), returning col4row, u, v."""
    nr, n = cost.shape
    u, v = [0.0] * nr, [0.0] * n
    col4row, row4col = [-1] * nr, [-1] * n
    for cur in range(n_proc):
        dist, path = [math.inf] * n, [-1] * n
        vis_r, vis_c = [False] * nr, [False] * n
        order, live, min_val, row, sink = list(range(n - 1, -1, -1)), n, 0.0, cur, -1
        while sink < 0:
            vis_r[row] = True
            best_pos, best = -1, math.inf
            for pos in range(live):
                c = order[pos]
                r = min_val + cost[row, c] - u[row] - v[c]
                if r < dist[c]:
                    path[c], dist[c] = row, r
                if dist[c] < best or (dist[c] == best and row4col[c] < 0):
                    best, best_pos = dist[c], pos
            min_val = best
            c = order[best_pos]
            if row4col[c] < 0:
                sink = c
            else:
                row = row4col[c]
            vis_c[c] = True
            live -= 1
            order[best_pos] = order[live]
        u[cur] += min_val
        for r in range(nr):
            if vis_r[r] and r != cur:
                u[r] += min_val - dist[col4row[r]]
        for c in range(n):
            if vis_c[c]:
                v[c] -= min_val - dist[c]
        c = sink
        while True:
            r = path[c]
            row4col[c] = r
            col4row[r], c = c, col4row[r]
            if r == cur:
                break
    return col4row, np.array(u), np.array(v)


def _row_arcs(i, cost, finite, col4row, row4col, u, v, sentinel, eps):
    """Near-tight cells of row i other than its own: (target row or None for
    a free column, is an entry cell); sentinel cells only when u_i >= sentinel - eps."""
    nr, nc = cost.shape
    out = []
    for j in range(nc):
        if j == col4row[i]:
            continue
        if finite[i, j]:
            near = cost[i, j] - u[i] - v[j] <= eps
        else:
            near = u[i] >= sentinel - eps and v[j] >= sentinel - u[i] - eps
        if near:
            out.append((row4col[j] if row4col[j] >= 0 else None, bool(finite[i, j])))
    return out


def lap_unique(cost, finite, col4row, u, v, sentinel, eps):
    """Python statement of the device's lap_unique (same active-row graph, same rules)."""
    nr, nc = cost.shape
    row4col = [-1] * nc
    for r, c in enumerate(col4row):
        row4col[c] = r
    arcs = [_row_arcs(i, cost, finite, col4row, row4col, u, v, sentinel, eps) for i in range(nr)]
    active = [i for i in range(nr) if arcs[i]]
    idx = {r: k for k, r in enumerate(active)}
    m = len(active)
    if m == 0:
        return True
    A, FA = [0] * m, [0] * m
    to_free, ftofree, fm = [False] * m, [False] * m, [False] * m
    for k, i in enumerate(active):
        fm[k] = bool(finite[i, col4row[i]])
        for tgt, fin in arcs[i]:
            if tgt is None:
                to_free[k] = True
                ftofree[k] = ftofree[k] or fin
            elif tgt in idx:
                A[k] |= 1 << idx[tgt]
                if fin:
                    FA[k] |= 1 << idx[tgt]
    Rc = A[:]
    while True:
        nxt = [Rc[i] | _or(Rc, Rc[i]) for i in range(m)]
        if nxt == Rc:
            break
        Rc = nxt
    tf_rows = sum(1 << k for k in range(m) if to_free[k])
    free_reach = [to_free[k] or (Rc[k] & tf_rows) != 0 for k in range(m)]
    fr_rows = sum(1 << k for k, i in enumerate(active) if v[col4row[i]] >= -eps)
    RF = fr_rows | _or(Rc, fr_rows)
    for i in range(m):
        start = (RF >> i) & 1
        if fm[i] and (Rc[i] >> i) & 1:
            return False
        if fm[i] and start and free_reach[i]:
            return False
        if ftofree[i] and start:
            return False
        for k in range(m):
            if (FA[i] >> k) & 1 and ((Rc[k] >> i) & 1 or (start and free_reach[k])):
                return False
    return True


def _or(R, mask):
    out = 0
    for k in range(len(R)):
        if (mask >> k) & 1:
            out |= R[k]
    return out


def brute_unique(cost, finite, eps):
    """Max-cardinality, then min-cost finite matchings: is the best finite
    pair set unique (no other set within eps)?"""
    nr, nc = cost.shape
    best = {}
    for perm in itertools.permutations(range(nc), nr):
        pairs = frozenset((r, c) for r, c in enumerate(perm) if finite[r, c])
        best[pairs] = (len(pairs), sum(cost[r, c] for r, c in pairs))
    card = max(v[0] for v in best.values())
    opt = min(v[1] for v in best.values() if v[0] == card)
    return sum(1 for v in best.values() if v[0] == card and v[1] <= opt + eps) == 1


@pytest.mark.parametrize("seed", range(6))
def test_lap_unique_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    agree = alternatives = 0
    for _ in range(400):
        nr = int(rng.integers(1, 6))
        nc = int(rng.integers(nr, 7))
        finite = rng.random((nr, nc)) < rng.uniform(0.3, 0.9)
        # small integer costs: plenty of exact ties and equal sums (a + d == b + c)
        cost_f = rng.integers(0, 4, (nr, nc)).astype(np.float64) * 0.25
        amp = max(float(np.abs(cost_f[finite]).max()) if finite.any() else 1.0, 1.0)
        sentinel = 2.0 * nc * amp + 1.0
        cost = np.where(finite, cost_f, sentinel)
        col4row, u, v = sap_rect(cost, nr)
        eps = 1e-9 * amp
        got = lap_unique(cost, finite, col4row, u, v, sentinel, eps)
        want = brute_unique(cost_f, finite, eps)
        assert got == want, (cost_f.tolist(), finite.tolist(), col4row)
        agree += 1
        alternatives += not want
    assert alternatives > 20          # the cases exercise genuine near-optima


def test_equal_sum_distinct_costs_is_not_unique():
    """The advisor's case: four distinct costs with a + d == b + c."""
    cost_f = np.array([[0.0, 0.5], [1.0, 1.5]])
    finite = np.ones((2, 2), bool)
    sentinel = 2 * 2 * 1.5 + 1
    col4row, u, v = sap_rect(cost_f, 2)
    assert not lap_unique(cost_f, finite, col4row, u, v, sentinel, 1e-9)
    cost_f = np.array([[0.0, 0.5], [1.0, 1.25]])
    col4row, u, v = sap_rect(cost_f, 2)
    assert lap_unique(cost_f, finite, col4row, u, v, sentinel, 1e-9)
