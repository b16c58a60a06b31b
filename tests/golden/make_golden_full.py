"""Golden scalars and R-sketches for the full-size BASELINE configurations,
produced by running the REFERENCE package (hodlrqr) on the same inputs.

Run in the build container only (needs /root/reference); minutes of CPU:
    python tests/golden/make_golden_full.py [config ...]
For each config: ||A||_2 estimate, e_orth / e_acc (reference's power-iteration
estimates), max ranks of Y, T, R, and the sketch R @ G for a fixed Gaussian
G (n x 8) -- the dense R itself is too large to store; relative Frobenius
error of the sketch stands in for that of R.
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, REF)

import hodlrqr as ref  # noqa: E402
from hodlrqr.bench import metrics as ref_metrics  # noqa: E402

from paper_1809_10585_b200 import gen  # noqa: E402
from make_golden import to_ref  # noqa: E402


def sketch_matrix(n):
    return np.random.default_rng(0x5C37).standard_normal((n, 8))


def main():
    which = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 3, 4]
    for ci in which:
        c = gen.CONFIGS[ci]
        t0 = time.time()
        a = gen.gen_config(ci, seed=0)
        ra = to_ref(a)
        t1 = time.time()
        f = ref.hqr(ra, c["tol"])
        t2 = time.time()
        m = ref_metrics(ra, f, eps=c["tol"], estimate=True, compute_ranks=False)
        G = sketch_matrix(a.n)
        out = dict(config=ci, n=a.n, tol=c["tol"], norm_est=ref.hodlr_spectral_norm(ra),
                   e_orth=m["e_orth"], e_acc=m["e_acc"], t_hqr=t2 - t1,
                   rank_y=ref.stats(f.y)["max_offdiag_rank"], rank_t=ref.stats(f.t)["max_offdiag_rank"],
                   rank_r=ref.stats(f.r)["max_offdiag_rank"],
                   RG=ref.apply_dense(f.r, G), r_diag_head=np.array(
                       [np.diag(leaf.dense)[:8] for leaf in _leaves(f.r)[:4]]))
        np.savez_compressed(os.path.join(HERE, f"golden_full_cfg{ci}.npz"), **out)
        print(ci, {k: v for k, v in out.items() if np.ndim(v) == 0}, f"gen {t1 - t0:.1f}s", flush=True)


def _leaves(h):
    if h.is_leaf:
        return [h]
    return _leaves(h.a11) + _leaves(h.a22)


if __name__ == "__main__":
    main()
