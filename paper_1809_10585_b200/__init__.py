"""B200-native recursive Householder QR of HODLR matrices (arXiv 1809.10585).

Drop-in for the reference package ``hodlrqr``'s hot path: build a HODLR
matrix with the host containers, then ``hqr(a, eps)`` factors it on the GPU
(libhqb200.so, sm_100a) into Y, T, R with A ~= (I - Y T Y^T) R.
"""

from .hodlr import (GENERAL, UNIT_LOWER_TRIANGULAR, UPPER_TRIANGULAR, HodlrMatrix,
                    LowRankBlock, PartitionTree, TruncationControl, build_partition,
                    hodlr_identity, stats, to_dense, validate_structure)
from .hqr import (HodlrQRFactors, HQREngine, PlanIO, RankCapacityError, StructuredColumn, StructuredY,
                  clear_engines, engine_for, hqr, hqr_batched, hqr_rec)
from .construct import compress_block, from_dense
from .operators import (HodlrOperator, QROperator, apply_dense, apply_q, apply_q_transpose,
                        apply_transpose_dense, metrics)

__version__ = "0.1.0"

__all__ = ["GENERAL", "UNIT_LOWER_TRIANGULAR", "UPPER_TRIANGULAR", "HodlrMatrix", "LowRankBlock",
           "PartitionTree", "TruncationControl", "build_partition", "hodlr_identity", "stats",
           "to_dense", "validate_structure", "HodlrQRFactors", "HQREngine", "PlanIO",
           "RankCapacityError", "clear_engines", "engine_for", "hqr", "hqr_batched", "HodlrOperator",
           "QROperator", "apply_dense", "apply_q", "apply_q_transpose", "apply_transpose_dense", "metrics",
           "compress_block", "from_dense",
           "StructuredColumn", "StructuredY", "hqr_rec"]
