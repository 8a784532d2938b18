"""B200-native mixed-precision HODLR matrix-vector product (arXiv 2407.21637).

The hot path is ``linops.matvec`` -- the reference's Algorithm 3 HODLR_MATVEC
 -- running as hand-written sm_100a CUDA
behind the C ABI of ``include/hodlr_b200.h``.
"""

from .formats import BF16, FP16, FP32, FP64, NAMED_FORMATS, Q52, PrecisionFormat, parse_format  # noqa: F401
from .model import HodlrMatrix, LowRankFactor, PrecisionPlan, build_tree, load_hodlr, save_hodlr, storage_bits  # noqa: F401
from .linops import HodlrOperator, matvec, operator_for  # noqa: F401
from . import lu  # noqa: F401  (HODLR LU, Alg. 4)

__version__ = "0.1.0"
