"""Write tests/golden/cfg0_ranks.json: per-node ranks of config 0 from the ORACLE's
adaptive run (rel_tol 1e-6, cap 1024, s 1040), AMB-11.  Calls only oracle/ + datagen/.
Both sides then run config 0 in fixed-rank mode with these ranks."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402
from oracle import pipeline  # noqa: E402


def main():
    cfg = datagen.get_config(0)
    F, y, Ft, yt = datagen.generate(0)
    perm, ranges, Om, H = pipeline.build(F, cfg, ranks=None)
    nn = 2 ** (H.L + 1) - 1
    ranks = pipeline.ranks_array(H, nn).tolist()
    out = dict(citation="AMB-11 (DESIGN.md): config 0 ranks from the oracle's adaptive run "
               "(rel_tol 1e-6, cap 1024, s 1040, AMB-10 rule); root = -1. Written by "
               "scripts/make_cfg0_ranks.py (oracle only).",
               L=H.L, ranks=ranks, cap_hits=int(sum(H.cap_hit.values())))
    with open(os.path.join(ROOT, "tests/golden/cfg0_ranks.json"), "w") as f:
        json.dump(out, f)
    print(H.L, max(ranks), out["cap_hits"])


if __name__ == "__main__":
    main()
