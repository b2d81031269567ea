"""CPU oracle for the GPA bilateral-filter hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import this package, and only as the checker or as
the timed CPU baseline.  The product path (`paper_1603_08109_b200`) never
imports it and fails loudly when the CUDA library is missing.

Parity pin: `gpa_oracle.py` is checked against golden vectors produced by the
reference package itself (`tests/golden/make_golden.py`, run in the build
container where `/root/reference` is importable) in `tests/test_oracle.py`.
"""
