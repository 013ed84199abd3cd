"""CPU oracle for the decode -> NMS -> association hot path.

TEST INFRASTRUCTURE ONLY. This package restates, on the CPU, the reference's
algorithm for the path the product accelerates (``trackforge`` under
``/root/reference/pkg/src``; every function cites the reference file:line it
follows). It exists to *check* the CUDA path, never to stand in for it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
  leg (``cpu_baseline`` and ``--impl reference``) may import it;
* the product package ``paper_2011_03910_b200`` never imports it and fails
  loudly when its CUDA library is missing.

Modules:

* ``oracle.heads``   - YOLO-head geometry and the numpy decode oracle (no
  reference exists for the decode; its semantics are pinned in DESIGN.md and
  SURVEY.md section 7 H1). Parity for the decode is therefore *unpinned* by any
  reference test; it is pinned by this restatement only.
* ``oracle.tracker`` - restatement of ``tf/core.py``, ``tf/postproc.py``,
  ``tf/motion.py``, ``tf/assoc.py`` and ``tf/tracker.py`` with the same numpy /
  scipy arithmetic, pinned bit-for-bit against golden vectors produced by the
  reference itself (``tests/golden/make_golden.py``).
* ``oracle.lap``     - restatement of scipy's shortest-augmenting-path LAP
  (the third-party solver behind ``tf/assoc.py:76``), pinned against scipy
  including its tie-breaking.
"""
