"""ctypes binding of libhqb200.so (include/hodlrqr_b200.h).

numpy structured dtypes mirror the C descriptor structs byte for byte
(checked against offsetof() by tests/test_abi.py).  Loading fails loudly:
there is no CPU fallback for the factorization path.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HQ_LIB", os.path.join(HERE, "libhqb200.so"))

P = np.uint64  # device pointer
I = np.int32

GEMM_TERM = np.dtype([("a", P), ("b", P), ("lda", I), ("ldb", I), ("ta", I), ("tb", I),
                      ("k", I), ("k_ri", I), ("mask_a", I), ("mask_b", I),
                      ("alpha", np.float64)], align=True)
GEMM_PROB = np.dtype([("c", P), ("ldc", I), ("m", I), ("m_ri", I), ("n", I), ("n_ri", I),
                      ("term0", I), ("nterm", I), ("item0", I), ("beta", np.float64),
                      ("ws", P), ("cnt", P)], align=True)
PIECE = np.dtype([("p", P), ("ld", I), ("cols", I), ("cols_ri", I), ("pad_", I),
                  ("alpha", np.float64)], align=True)
CONCAT_PROB = np.dtype([("dst", P), ("dst2", P), ("ldd", I), ("ldd2", I), ("rows", I),
                        ("piece0", I), ("npiece", I), ("ktot_ri", I)], align=True)
QR_PROB = np.dtype([("w", P), ("tau", P), ("tpanel", P), ("tfull", P), ("ldw", I), ("ldt", I),
                    ("m", I), ("m_ri", I), ("k", I), ("k_ri", I)], align=True)
APPLYQ_PROB = np.dtype([("w", P), ("tau", P), ("tpanel", P), ("x", P), ("x0", P),
                        ("ldw", I), ("ldx", I), ("ldx0", I), ("m", I), ("m_ri", I),
                        ("k", I), ("k_ri", I), ("c", I), ("c_ri", I), ("r0", I), ("r0_ri", I),
                        ("trans", I)], align=True)
SVD_PROB = np.dtype([("c", P), ("u", P), ("work", P), ("ldc", I), ("ldu", I), ("m", I),
                     ("m_ri", I), ("n", I), ("n_ri", I), ("cap", I), ("rank_ri", I),
                     ("flag_ri", I), ("eps_slot", I), ("eps_scale", np.float64),
                     ("xform", I), ("pad_", I)], align=True)
QRCP_PROB = np.dtype([("c", P), ("ldc", I), ("m", I), ("m_ri", I), ("n", I), ("n_ri", I),
                      ("r_ri", I), ("eps_slot", I), ("pad_", I), ("stop_scale", np.float64)], align=True)
SLAB = np.dtype([("v", P), ("yv", P), ("ld", I), ("ldy", I), ("k_ri", I), ("pad_", I)], align=True)
LEAF_PROB = np.dtype([("leaf", P), ("panel", P), ("nl", I), ("ldp", I), ("slab0", I),
                      ("nslab", I), ("m_ri", I), ("pad_", I)], align=True)

COPY_ITEM = np.dtype([("src", P), ("dst", P), ("rows", I), ("cols", I), ("cols_ri", I),
                      ("lds", I), ("ldd", I), ("mode", I)], align=True)

ROWBLK_PROB = np.dtype([("s", P), ("w", P), ("lds", I), ("ldw", I), ("ch", I), ("rows_total", I),
                        ("k", I), ("k_ri", I), ("ncol", I), ("ncol_ri", I), ("ms_ri", I),
                        ("mode", I)], align=True)

STRUCT_SIZES = {"hq_rowblk_prob": ROWBLK_PROB, "hq_copy_item": COPY_ITEM, "hq_gemm_term": GEMM_TERM, "hq_gemm_prob": GEMM_PROB, "hq_piece": PIECE,
                "hq_concat_prob": CONCAT_PROB, "hq_qr_prob": QR_PROB,
                "hq_applyq_prob": APPLYQ_PROB, "hq_svd_prob": SVD_PROB, "hq_qrcp_prob": QRCP_PROB, "hq_slab": SLAB,
                "hq_leaf_prob": LEAF_PROB}

EXPORTS = ("hq_abi_version", "hq_device_check", "hq_gemm", "hq_gemm_tiled", "hq_gemm_skinny", "hq_concat", "hq_qr", "hq_applyq",
           "hq_svd", "hq_svd_block", "hq_qrcp", "hq_leaf_gather", "hq_leaf_scatter", "hq_zero", "hq_power_step", "hq_copy",
           "hq_pack_offsets", "hq_rowblocks")

_vp, _i, _d, _i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64
SIGNATURES = {
    "hq_abi_version": [],
    "hq_device_check": [],
    "hq_gemm": [_vp, _vp, _i, _vp, _vp, _i, _i, _vp],
    "hq_gemm_tiled": [_vp, _vp, _i, _vp, _vp, _i, _i, _i, _vp],
    "hq_gemm_skinny": [_vp, _vp, _i, _vp, _vp, _i, _i, _i, _i, _vp],
    "hq_concat": [_vp, _vp, _i, _vp, _vp, _i],
    "hq_qr": [_vp, _vp, _i, _vp, _i],
    "hq_applyq": [_vp, _vp, _i, _vp, _i, _i],
    "hq_svd": [_vp, _vp, _i, _vp, _vp, _i, _i, _i],
    "hq_svd_block": [_vp, _vp, _i, _vp, _vp, _i],
    "hq_qrcp": [_vp, _vp, _i, _vp, _vp, _i, _i, _i],
    "hq_leaf_gather": [_vp, _vp, _i, _vp, _vp, _i],
    "hq_leaf_scatter": [_vp, _vp, _i, _vp, _vp, _i],
    "hq_zero": [_vp, _vp, _i, _i64],
    "hq_copy": [_vp, _vp, _i, _vp],
    "hq_pack_offsets": [_vp, _vp, _i, _vp, _vp, _vp, _i],
    "hq_rowblocks": [_vp, _vp, _i, _vp, _i],
    "hq_power_step": [_vp, _vp, _vp, _vp, _i, _i, _vp, _d, _d, _vp, _vp, _i, _i],
}

_LIB = None
ABI_VERSION = 6   # HQ_ABI_VERSION in include/hodlrqr_b200.h


class LibraryError(RuntimeError):
    pass


def load(build_if_missing: bool = True):
    """Load (building in-tree if needed) the CUDA library; raise if impossible."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if build_if_missing:
        from . import build
        if build.stale():
            try:
                build.build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                # a stale library may have other descriptor layouts: never load it
                raise LibraryError(f"{LIB_PATH} is out of date and cannot be rebuilt: {exc}") from exc
    if not os.path.exists(LIB_PATH):
        raise LibraryError(f"{LIB_PATH} missing; run `python -m paper_1809_10585_b200.build`")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    got = lib.hq_abi_version()
    if got != ABI_VERSION:
        raise LibraryError(f"{LIB_PATH} has ABI version {got}, this binding expects {ABI_VERSION}; rebuild it")
    _LIB = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        raise LibraryError(f"{what} failed with CUDA error {rc}")
