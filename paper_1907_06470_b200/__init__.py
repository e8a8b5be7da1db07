"""B200-native randomized-SVD hot path for the `xsvd` reference (arXiv 1907.06470).

Drop-in for the reference's hot-path entry points (same names, arguments,
return types and error classes):

    from paper_1907_06470_b200 import randomized_svd, RsvdConfig, BlockPool, matrix_from_dense
    pool = BlockPool()
    a = matrix_from_dense(pool, "A", array, precision=Precision.DOUBLE)
    res = randomized_svd(pool, a, RsvdConfig(rank=20, oversample=10, power=2, seed=1))

The arithmetic runs in the in-tree CUDA library (paper_1907_06470_b200/_lib/
libxsvdb200.so, C ABI in include/xsvd_b200.h). There is no CPU fallback.
"""

from .core import (CANONICAL_CELL, BlockPartition, DenseBlock, Density, MatrixDescriptor,
                   Precision, SparseBlock, transpose_view, wider)
from .errors import (BlockAbsentError, BlockCorruptError, BudgetError, ConfigMismatchError,
                     ConvergenceError, FormatError, ParseError, PlanNotFoundError, ShapeError,
                     XsvdError)
from .formats import (parse_matrix_market, read_block_file, read_matrix_market_info,
                      write_block_file, write_matrix_market)
from .kernels import MultiplyStats, QRResult, SmallSVDResult, block_multiply, gram, svd_small, thin_qr
from .pipeline import (STAGE_NAMES, PlanRunner, RsvdConfig, RsvdResult, StageClock, auto_select_q,
                       full_svd, gaussian_matrix, randomized_svd, resume, run_command)
from .store import BlockStore, StepRecord
from .pool import BlockPool, StoredMatrix, create_matrix, matrix_from_coo, matrix_from_dense

__all__ = [
    "BlockPartition", "BlockPool", "BudgetError", "CANONICAL_CELL", "ConvergenceError",
    "DenseBlock", "Density", "MatrixDescriptor", "MultiplyStats", "ParseError", "Precision",
    "QRResult", "parse_matrix_market", "read_matrix_market_info", "write_matrix_market",
    "RsvdConfig", "RsvdResult", "STAGE_NAMES", "ShapeError", "SmallSVDResult", "SparseBlock",
    "StageClock", "StoredMatrix", "XsvdError", "block_multiply", "create_matrix",
    "auto_select_q", "full_svd", "gaussian_matrix", "gram", "matrix_from_coo", "matrix_from_dense", "randomized_svd",
    "svd_small", "thin_qr", "transpose_view", "wider",
    "BlockAbsentError", "BlockCorruptError", "BlockStore", "ConfigMismatchError", "FormatError",
    "PlanNotFoundError", "PlanRunner", "StepRecord", "read_block_file", "resume", "run_command",
    "write_block_file",
]
