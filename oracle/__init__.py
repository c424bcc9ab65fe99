"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the VQ + grid-sampling hot path.

This package restates the reference's algorithm (semsplat 0.1.0, the read-only
tree at /root/reference/pkg/src/semsplat) on the CPU so the CUDA product path can
be checked against it.  It is imported only by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs, and there only as the checker or as the timed CPU baseline.
The product package ``paper_2603_09632_b200`` never imports it.

Pinning: ``oracle.vq`` and the back-projection in ``oracle.grid`` are checked
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and against the
reference's own known-answer tests (``tests/test_oracle_pins.py``).  The voxel
key / dedup / occupancy part of ``oracle.grid`` has no reference counterpart:
its definitions follow SURVEY.md §8(a) g8 and are pinned by hand-computed KATs
only ("parity unpinned" for that part).
"""
