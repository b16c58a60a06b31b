"""Rounding-sensitivity floor of R for a configuration: run the oracle (a
numpy restatement of the reference, differing only in rounding) and compare
its R-sketch with the reference's golden sketch.

    python tests/golden/oracle_floor.py 2      (~10-15 min of CPU at n=16384)
For config 2 (kappa ~1e17) this gives 2.14e-3: the reference's own R is not
reproducible to 100*tol at this conditioning, so tests/test_gpu_fullsize.py
compares the GPU R against this floor there (and against 100*tol elsewhere).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle.hqr_oracle as O  # noqa: E402
from paper_1809_10585_b200 import gen  # noqa: E402

if __name__ == "__main__":
    ci = int(sys.argv[1])
    g = dict(np.load(os.path.join(HERE, f"golden_full_cfg{ci}.npz")))
    a = gen.gen_config(ci)
    y, t, r = O.hqr(a, gen.CONFIGS[ci]["tol"])
    G = np.random.default_rng(0x5C37).standard_normal((a.n, 8))
    rg = O.happly(r, G)
    print(ci, "oracle vs reference R-sketch relative difference %.3e"
          % (np.linalg.norm(rg - g["RG"]) / np.linalg.norm(g["RG"])))
