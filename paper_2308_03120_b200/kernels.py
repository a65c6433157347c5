"""Kernel inventory of the device library: element types, kinds and the
fixed geometry constants of the reference (kernels.py:28-92).

No computation happens here -- every kind named below executes as CUDA in
libb200mat.so.  The kind names are the reference's, so plans and
``KernelInvocation`` objects read the same on both implementations.
"""
from __future__ import annotations

import numpy as np

ELEM_TYPES = ("f32", "f64", "i32", "u64")
NP_DTYPE = {
    "f32": np.dtype(np.float32),
    "f64": np.dtype(np.float64),
    "i32": np.dtype(np.int32),
    "u64": np.dtype(np.uint64),
}
FLOAT_TYPES = ("f32", "f64")
INT_TYPES = ("i32", "u64")


def is_float(elem_type: str) -> bool:
    return elem_type in FLOAT_TYPES


def itemsize(elem_type: str) -> int:
    return NP_DTYPE[elem_type].itemsize


EOP_UNARY = ("eop_exp", "eop_log", "eop_log10", "eop_sqrt", "eop_square", "eop_pow", "eop_abs",
             "eop_cos", "eop_sin", "eop_tan", "eop_acos", "eop_asin", "eop_atan")
EOP_SCALAR = ("eop_scalar_plus", "eop_scalar_minus_pre", "eop_scalar_minus_post",
              "eop_scalar_times", "eop_scalar_div_pre", "eop_scalar_div_post")
EGLUE = ("eglue_plus", "eglue_minus", "eglue_schur", "eglue_div")
FUSED = ("fused_chain", "fused_reduce")
REDUCE = ("reduce_accu", "reduce_min", "reduce_max", "reduce_dot")
REDUCE_DIM = ("rdim_sum", "rdim_min", "rdim_max", "rdim_mean", "rdim_var")
GENERATOR = ("gen_fill_const", "gen_eye", "gen_linspace", "gen_randu", "gen_randn", "gen_repmat")
MOVEMENT = ("mov_copy", "mov_transpose", "mov_resize", "mov_reshape_copy", "mov_extract_strided",
            "mov_insert_strided", "mov_join_rows", "mov_join_cols", "mov_diagmat_build",
            "mov_diagvec_extract")
GEMM = ("gemm",)
ELEMENTWISE = EOP_UNARY + EOP_SCALAR + EGLUE
ALL_KINDS = ELEMENTWISE + FUSED + REDUCE + REDUCE_DIM + GENERATOR + MOVEMENT + GEMM

# Fixed block geometry of the reference (kernels.py:85-92).  REDUCE_BLOCK is
# semantic here: it fixes the summation order that the device reproduces.
ELEM_BLOCK = 1 << 16
REDUCE_BLOCK = 1 << 13
GEMM_PANEL = 64
DIM_BLOCK = 64

# The reference splits element-wise chains after 8 stages (kernels.py:91-92).
# Splitting never changes bits (every stage rounds), so the B200 planner fuses
# much deeper trees into one kernel; REFERENCE_CHAIN_MAX reproduces the
# reference's plan shape on request (plan(..., chain_max=8)).
REFERENCE_CHAIN_MAX = 8
FUSED_CHAIN_MAX = 48
# a fused kernel reads at most this many distinct inputs (include/b200mat.h)
FUSED_INPUTS_MAX = 16
