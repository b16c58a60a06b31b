"""The reference's own rounding floor for R: run the REFERENCE package
(hodlrqr) on the full-size BASELINE inputs with its panel width n_b = 16 and
compare the R sketch R @ G with the golden sketch of its default n_b = 32
(tests/golden/make_golden_full.py).  The two runs differ only in the order of
floating-point operations inside the dense leaf QRs, so their difference is
how far the reference's R is reproducible at all; an implementation cannot be
judged more tightly than that.

Run in the build container only (needs /root/reference):
    python tests/golden/make_floor_ref.py [config ...]
writes tests/golden/golden_floor_ref.json
"""

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, REF)

import hodlrqr as ref  # noqa: E402

from paper_1809_10585_b200 import gen  # noqa: E402
from make_golden import to_ref  # noqa: E402


def main():
    which = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 4]
    path = os.path.join(HERE, "golden_floor_ref.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for ci in which:
        c = gen.CONFIGS[ci]
        g = np.load(os.path.join(HERE, f"golden_full_cfg{ci}.npz"))
        a = to_ref(gen.gen_config(ci, seed=0))
        t0 = time.time()
        f = ref.hqr(a, c["tol"], n_b=16)
        G = np.random.default_rng(0x5C37).standard_normal((a.n, 8))
        rg = ref.apply_dense(f.r, G)
        rel = float(np.linalg.norm(rg - g["RG"]) / np.linalg.norm(g["RG"]))
        out[str(ci)] = {"r_sketch_nb16_vs_nb32": rel, "n": a.n, "tol": c["tol"], "seconds": time.time() - t0}
        print(ci, out[str(ci)], flush=True)
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
