"""The five BASELINE.json configs as frozen knobs.

Every number here is a configuration constant, not a result: the GPU path and
the oracle both read it.  `beta` values for configs 1-4 were chosen by
`scripts/calibrate_beta.py`, which calls only `oracle/` (AMB-9 in DESIGN.md).
"""
from __future__ import annotations

import copy


def beta_schedule(n: int) -> float:
    """PAPER.md:286 (§3.3): beta = 1e2 for d in [1e4,1e5], 1e3 for [1e5,1e6], 1e4 for d >= 1e6.

    Below 1e4 the paper is silent; we extend the smallest tier downward.
    """
    if n >= 1_000_000:
        return 1e4
    if n >= 100_000:
        return 1e3
    return 1e2


# Field meanings:
#   n, n_test   train / test points;  r  feature count (paper's r)
#   h           Gaussian kernel width;  C  box bound(s) (Eq. 1)
#   beta        ADMM penalty / ULV shift
#   max_it      ADMM iterations (PAPER.md:286 fixes 10; BASELINE.json configs override)
#   leaf        leaf size m;  cap  rank cap k_max;  s = sketch columns = cap + 16
#   rel_tol, abs_tol   rank rule AMB-10;  rank_mode  'adaptive' | 'fixed'
#   seeds       data 1000+c, Omega 2000+c, tree 3000+c
_CONFIGS = {
    0: dict(name="cfg0_gmm2k", n=2000, n_test=500, r=8, h=1.0, C=[1.0], beta=1.0,
            max_it=200, leaf=64, cap=1024, s=1040, rel_tol=1e-6, abs_tol=0.0,
            rank_mode="fixed", ranks_file="tests/golden/cfg0_ranks.json", gpus=[1]),
    1: dict(name="cfg1_uniform32k", n=32768, n_test=8192, r=22, h=0.5, C=[10.0], beta=None,
            max_it=500, leaf=128, cap=128, s=144, rel_tol=1e-4, abs_tol=0.0,
            rank_mode="adaptive", gpus=[1]),
    2: dict(name="cfg2_binary131k", n=131072, n_test=32768, r=123, h=2.0, C=[1.0], beta=None,
            max_it=500, leaf=256, cap=256, s=272, rel_tol=1e-3, abs_tol=0.0,
            rank_mode="adaptive", gpus=[1, 2]),
    3: dict(name="cfg3_mixed524k", n=524288, n_test=131072, r=54, h=1.0, C=[1.0], beta=None,
            max_it=1000, leaf=256, cap=256, s=272, rel_tol=1e-3, abs_tol=0.0,
            rank_mode="adaptive", gpus=[1, 2, 4, 8]),
    4: dict(name="cfg4_grid65k", n=65536, n_test=16384, r=8, h=[0.25, 0.5, 1.0, 2.0, 4.0],
            C=[0.1, 1.0, 10.0, 100.0, 1e3, 1e4], beta=None,
            max_it=200, leaf=64, cap=64, s=80, rel_tol=1e-6, abs_tol=0.0,
            rank_mode="adaptive", gpus=[1, 2, 4, 8]),
}

# Calibrated shifts (scripts/calibrate_beta.py -> configs/beta_calibration.jsonl; AMB-9):
# beta = max(schedule(n), 10^ceil(log10(-4 lambda_min(K~)))) with lambda_min from the ORACLE's
# HSS at the full config size.  None = use beta_schedule(n).
#   cfg 1: lambda_min = -331.65  -> 1e4      cfg 2: lambda_min = -5185.1 -> 1e5 (chaos gate -> 1e6)
#   cfg 4 (per h): 0.25: -7.09 -> 1e2; 0.5: -91.5 -> 1e3; 1: -476.3 -> 1e4; 2: -627.3 -> 1e4;
#                  4: -206.7 -> 1e3
#   cfg 3: lambda_min = -62850.4 -> 1e6  (oracle at n = 524288: 8256 s of host compression + eigsh)
# AMB-9 chaos gate at MaxIt (scripts/make_fullsize_goldens.py, oracle only, full size): cfg 1
# (1e4) 6.1e-10, cfg 4 (per h) <= 5.8e-11 pass; cfg 2 at 1e5 gave 5.97e-9 > 1e-9, so cfg 2 is
# re-frozen one decade up at 1e6 (SURVEY AMB-9: "raise that beta and re-freeze it"); cfg 3 at 1e6
# gave 5.4e-6 > 1e-9 (1000 iterations), re-frozen at 1e7: 4.7e-12.
_BETA = {1: 1e4, 2: 1e6, 3: 1e7, 4: None}
_BETA_PER_H = {4: {0.25: 1e2, 0.5: 1e3, 1.0: 1e4, 2.0: 1e4, 4.0: 1e3}}
# The same rule for the HSS-ANN K~ (sampling = "ann"; scripts/calibrate_beta.py --sampling ann):
#   cfg 3: lambda_min = -4.43 -> schedule 1e3   (oracle ANN build at n = 524288: 629 s)
_BETA_ANN = {3: 1e3}

# HSS-ANN sampling knobs (readings N1-N3): neighbours per point (the paper's
# Table 4 setting "hss_approximate_neighbors 64"), random-projection trees, their leaf
# size (<= 256; leaf * r * 8 bytes must fit shared memory, hence 128 for r = 123), seed 4000+c.
_ANN = dict(ann_neighbors=64, ann_trees=4, ann_leaf=256)
_ANN_LEAF = {2: 128}

for _c, _cfg in _CONFIGS.items():
    _cfg["id"] = _c
    _cfg["seed_data"] = 1000 + _c
    _cfg["seed_omega"] = 2000 + _c
    _cfg["seed_tree"] = 3000 + _c
    _cfg.update(_ANN)
    _cfg["ann_leaf"] = _ANN_LEAF.get(_c, _ANN["ann_leaf"])
    _cfg["ann_seed"] = 4000 + _c
    if _cfg["beta"] is None:
        b = _BETA.get(_c)
        _cfg["beta"] = b if b is not None else beta_schedule(_cfg["n"])
    if _c in _BETA_PER_H:
        _cfg["beta_per_h"] = dict(_BETA_PER_H[_c])
    _cfg["beta_ann"] = _BETA_ANN.get(_c, beta_schedule(_cfg["n"]))

CONFIGS = _CONFIGS


def get_config(c: int, **overrides) -> dict:
    """A deep copy of config `c` with overrides (e.g. n=4096 for a scaled parity case)."""
    cfg = copy.deepcopy(_CONFIGS[c])
    cfg.update(overrides)
    return cfg
