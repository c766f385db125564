"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 NumPy/SciPy implementation of the hot path of arXiv
2108.04167 (ADMM for the SVM dual with an HSS-approximated Gaussian kernel),
written from PAPER.md and the readings listed in DESIGN.md ("Readings").
Citations `P:n` are PAPER.md line numbers; `AMB-n` / `T*`, `R*`, `H*`, `U*`,
`S*`, `M*`, `A*` are the step labels of SURVEY.md §8(c) restated in DESIGN.md.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product path
(`paper_2108_04167_b200`) never imports it, and it never imports the product.
It shares no code with the CUDA path; the only shared module is `datagen`
(seeded inputs, no method arithmetic).

Parity status: every function is pinned by `tests/test_oracle_*.py` against
closed forms, brute force or library routines.
"""
from . import rng, kernel, tree, hss, ann, ulv, admm, svm, qp  # noqa: F401
