"""paper_2308_03120_b200 -- a B200-native drop-in for the data-parallel hot path
of Bandicoot / devmat (arXiv 2308.03120): lazily built expressions fused into
one sm_100a kernel per tree, numpy-order-exact reductions, and tcgen05 GEMM.

    import paper_2308_03120_b200 as dm

    A = dm.Matrix.from_numpy(a)          # column-major, resident in HBM
    s = dm.accu(2 * A + B % C - dm.exp(D))   # one fused kernel, bit-exact order
    C = (A @ B.t()).eval()               # NT GEMM, no transpose pass

The public names mirror reference/pkg/src/devmat/__init__.py.
"""
from .errors import (BackendError, BoundsError, BufferError_, DevmatError, DimensionError, ElemTypeError,
                     KernelCacheWarning, NotPositiveDefiniteError, NotSymmetricError, PrecisionUnsupportedError,
                     SingularMatrixError)
from .expr import (EvalPlan, ExprNode, Relational, Shape, build_node, census, evaluate, evaluate_many, plan, plan_reduce,
                   rewrite_trans, shape_of)
from .linalg import as_scalar, gemm, gemv, norm, trace
from .matrix import Col, HostMatrix, Mat, Matrix, Row, Subview, conv_to, to_device, to_host
from .ops import (absolute, accu, acos, all, any, asin, atan, cos, diagmat, diagvec, dot, exp, eye, find,
                  join_cols, join_rows, linspace, log, log10, max, mean, min, ones, power, randn, randu,
                  reduce_max, reduce_min, repmat, reshape, resize, schur, sin, sqrt, square, stddev, sum, tan,
                  trans, var, vectorise, zeros)
from .runtime import (Counters, DeviceBuffer, DeviceDescriptor, KernelInvocation, __version__, counters, init,
                      is_initialised, set_seed, shutdown, synchronise, wall_clock)

abs = absolute  # noqa: A001 - Armadillo spelling
