"""Writes tests/golden/cfg1_brute.json using ONLY oracle/brute.py (enumeration) and tsgen.

cfg1 = BASELINE.json configs[0]: batch 1, N=5, C=3, 3^5 = 243 labelings, tsgen seed
0x200200876+1, quantum s=15.  Values are the §5.1 definitions summed over
all labelings; the tie rule is DESIGN.md reading R5.
Run: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

import tsgen  # noqa: E402
from oracle import brute  # noqa: E402

cfg = tsgen.CONFIGS[1]
pot = tsgen.config_potentials(cfg)
z, best = brute.argmax(pot[0], cfg.N)
out = {
    "cite": "BASELINE.json configs[0]; brute-force enumeration of all 243 labelings (P:149 footnote)",
    "generator": {"seed": cfg.seed, "s": cfg.quantum, "B": cfg.B, "N": cfg.N, "C": cfg.C},
    "pot_sha256": hashlib.sha256(np.ascontiguousarray(pot).tobytes()).hexdigest(),
    "logZ": brute.log_partition(pot[0], cfg.N),
    "marginals": brute.marginals(pot[0], cfg.N).tolist(),
    "viterbi_path": z.tolist(),
    "viterbi_score": best,
}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg1_brute.json"), "w") as f:
    json.dump(out, f, indent=1)
print("logZ", out["logZ"], "path", out["viterbi_path"], "score", best)
