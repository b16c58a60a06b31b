"""Generate golden vectors by running the REFERENCE package (hodlrqr) itself.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
Outputs tests/golden/golden_*.npz.  Inputs come from paper_1809_10585_b200.gen
(deterministic, seeded) and are converted to the reference's own classes, so
the fixtures pin the reference's outputs on exactly the inputs our tests use.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, REF)

import hodlrqr as ref  # noqa: E402  (the reference package)
from hodlrqr.bench import metrics as ref_metrics  # noqa: E402

from paper_1809_10585_b200 import gen  # noqa: E402
from paper_1809_10585_b200.hodlr import HodlrMatrix, LowRankBlock, build_partition, to_dense  # noqa: E402

CASES = {
    # name: (builder, eps, dense outputs?)
    "random_n256": (lambda: gen.gen_random_hodlr(256, 32, 4, 8.0, seed=0), 1e-10, True),
    "illcond_n256": (lambda: gen.gen_illcond_hodlr(256, 32, 4, 8.0, seed=1), 1e-10, True),
    "logkernel_n256": (lambda: gen.gen_logkernel_hodlr(256, 32, 1e-10), 1e-10, True),
    "ragged_n200": (lambda: gen.gen_random_hodlr(200, 24, 3, 8.0, seed=2), 1e-12, True),
    "leaf_n48": (lambda: gen.gen_random_hodlr(48, 64, 1, 8.0, seed=3), 1e-14, True),
    "cfg0_n1024": (lambda: gen.gen_config(0), 1e-10, False),
    "cfg4_n1024": (lambda: gen.gen_random_hodlr(1024, 128, 16, 8.0, seed=5), 1e-10, False),
}


def to_ref(h: HodlrMatrix):
    if h.is_leaf:
        return ref.HodlrMatrix(dense=h.dense.copy())
    return ref.HodlrMatrix(a11=to_ref(h.a11), a22=to_ref(h.a22),
                           a12=ref.LowRankBlock(h.a12.L, h.a12.R, h.a12.left_orthogonal),
                           a21=ref.LowRankBlock(h.a21.L, h.a21.R, h.a21.left_orthogonal))


def main():
    for name, (build, eps, dense) in CASES.items():
        a = build()
        ra = to_ref(a)
        norm = ref.hodlr_spectral_norm(ra)
        f = ref.hqr(ra, eps)
        out = {"eps": eps, "norm_est": norm, "n": a.n,
               "input_dense_fro": np.linalg.norm(to_dense(a)),
               "rank_y": ref.stats(f.y)["max_offdiag_rank"],
               "rank_t": ref.stats(f.t)["max_offdiag_rank"],
               "rank_r": ref.stats(f.r)["max_offdiag_rank"],
               "mem_y": ref.stats(f.y)["memory_scalars"],
               "mem_t": ref.stats(f.t)["memory_scalars"],
               "mem_r": ref.stats(f.r)["memory_scalars"]}
        m = ref_metrics(ra, f, eps=eps, compute_ranks=False)
        out["e_orth"], out["e_acc"], out["kappa2"] = m["e_orth"], m["e_acc"], m["kappa2"]
        rd = ref.to_dense(f.r)
        out["r_diag"] = np.diag(rd)
        out["r_fro"] = np.linalg.norm(rd)
        if dense:
            out["R"], out["Y"], out["T"] = rd, ref.to_dense(f.y), ref.to_dense(f.t)
        np.savez_compressed(os.path.join(HERE, f"golden_{name}.npz"), **out)
        print(name, {k: v for k, v in out.items() if np.ndim(v) == 0})

    # structured column [A; B; C] through hqr_rec (reference test_hqr.py pattern)
    rng = np.random.default_rng(33)
    h = gen.gen_random_hodlr(64, 16, 2, 8.0, seed=7)
    bl, br = rng.standard_normal((9, 2)), rng.standard_normal((2, 64))
    c = rng.standard_normal((5, 64))
    col = ref.StructuredColumn(to_ref(h), ref.LowRankBlock(bl, br), c)
    y, t, r = ref.hqr_rec(col, 1e-14, 1e-14)
    np.savez_compressed(os.path.join(HERE, "golden_structured_col.npz"),
                        bl=bl, br=br, c=c, Y=y.to_dense(), T=ref.to_dense(t), R=ref.to_dense(r))
    # dense block_qr known answers
    a = np.random.default_rng(11).standard_normal((70, 45))
    wy, rr = ref.block_qr(a, 8)
    np.savez_compressed(os.path.join(HERE, "golden_block_qr.npz"), A=a, Y=wy.Y, T=wy.T, R=rr)
    print("done")


if __name__ == "__main__":
    main()
