"""Process-wide runtime: the firewall between the expression layer and the
B200 device library.

Public surface and semantics follow the reference's runtime module
(reference/pkg/src/devmat/runtime.py:366-703): memory acquisition and
(stream-ordered) release, a FIFO queue of kernel invocations, scalar
reductions that return one value to the host, synchronous bulk transfers,
instrumentation counters, a process singleton with automatic selection.
What lives *under* the surface is different: the queue is a CUDA stream,
buffers come from the stream-ordered CUDA memory pool, and every invocation
is translated into a ``bm_invocation`` C struct and handed to
libb200mat.so (include/b200mat.h).  Nothing is computed in Python.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import pathlib
import threading
import time
from dataclasses import dataclass, field, fields, replace

import numpy as np

from . import _clib
from . import kernels
from .errors import BackendError, BufferError_, ElemTypeError

__version__ = "0.1.0"

# "b200" is the device; the reference's backend names are accepted as aliases
# so `dm.init("parallel")` in existing code lands on the GPU unchanged.
BACKENDS = ("b200", "reference", "parallel")
CACHE_DIR_ENV = "KERNEL_CACHE_DIR"
BACKEND_ENV = "DEFAULT_BACKEND"
SEED_ENV = "RNG_SEED"


# ---------------------------------------------------------------------------
# domain types (runtime.py:59-144)

@dataclass(frozen=True)
class DeviceDescriptor:
    backend_name: str
    device_id: int
    worker_count: int
    supports_f64: bool
    gpu_name: str = ""
    sm_count: int = 0

    @property
    def descriptor_hash(self) -> str:
        text = (f"backend={self.backend_name};device={self.device_id};workers={self.worker_count};"
                f"f64={int(self.supports_f64)};gpu={self.gpu_name};sm={self.sm_count};arch=sm_100a;"
                f"version={__version__}")
        return hashlib.sha256(text.encode()).hexdigest()[:16]


@dataclass(frozen=True)
class DeviceBuffer:
    device_id: int
    buffer_id: int
    length: int
    elem_type: str
    ptr: int = 0          # device address (opaque to the expression layer)


@dataclass(frozen=True)
class FlatView:
    """1-D strided window into a buffer (elements)."""
    buf: DeviceBuffer
    offset: int = 0
    count: int = -1
    stride: int = 1


@dataclass(frozen=True)
class BlockView:
    """2-D column-major window: element (r, c) at offset + r + c * lda."""
    buf: DeviceBuffer
    offset: int
    rows: int
    cols: int
    lda: int


@dataclass(frozen=True)
class KernelInvocation:
    kind: str
    inputs: tuple = ()
    output: object = None
    scalars: tuple = ()
    params: dict = field(default_factory=dict)


@dataclass
class Counters:
    launches: int = 0
    compiles: int = 0
    cache_hits: int = 0
    transfers_h2d: int = 0
    transfers_d2h: int = 0
    bytes_h2d: int = 0
    bytes_d2h: int = 0
    buffers_acquired: int = 0
    buffers_released: int = 0

    def __sub__(self, other: "Counters") -> "Counters":
        return Counters(**{f.name: getattr(self, f.name) - getattr(other, f.name) for f in fields(Counters)})

    def copy(self) -> "Counters":
        return replace(self)


# ---------------------------------------------------------------------------
# translation of KernelInvocation -> bm_invocation

MANIFEST_NAME = "kernels.manifest"


@dataclass(frozen=True)
class KernelCacheEntry:
    """One line of the kernel-cache manifest (runtime.py:112-122 of the
    reference): device descriptor hash, kind, input and output element type,
    source hash; tab-separated, hashes are 16 lowercase hex digits."""
    descriptor_hash: str
    kind: str
    in_type: str
    out_type: str
    source_hash: str

    def line(self) -> str:
        return "\t".join((self.descriptor_hash, self.kind, self.in_type, self.out_type, self.source_hash))


def _hex16(t: str) -> bool:
    return len(t) == 16 and set(t) <= set("0123456789abcdef")


def load_manifest(cache_dir) -> dict:
    """Read the manifest in ``cache_dir``; an unreadable, truncated (no final
    newline) or malformed file warns KernelCacheWarning and reads as empty
    (a cold cache), the reference's contract (runtime.py:156-189).  The B200
    library's real cache is the NVRTC cubin directory (BM_CACHE_DIR); this
    index is kept for code that manages the reference's manifest."""
    import pathlib
    import warnings
    from .errors import KernelCacheWarning
    path = pathlib.Path(cache_dir) / MANIFEST_NAME
    if not path.exists():
        return {}
    try:
        text = path.read_text(encoding="utf-8")
    except (OSError, UnicodeDecodeError) as exc:
        warnings.warn(f"kernel cache {path} unreadable ({exc}): cold start", KernelCacheWarning)
        return {}
    if text and text[-1] != "\n":
        warnings.warn(f"kernel cache {path} truncated: cold start", KernelCacheWarning)
        return {}
    out = {}
    for no, ln in enumerate(text.split("\n")[:-1] if text else [], 1):
        if not ln:
            continue
        f = ln.split("\t")
        if not (len(f) == 5 and _hex16(f[0]) and _hex16(f[4]) and f[1] in kernels.ALL_KINDS
                and f[2] in kernels.ELEM_TYPES and f[3] in kernels.ELEM_TYPES):
            warnings.warn(f"kernel cache {path}: bad line {no}: cold start", KernelCacheWarning)
            return {}
        e = KernelCacheEntry(*f)
        out[(e.descriptor_hash, e.kind, e.in_type, e.out_type)] = e
    return out


def store_manifest(cache_dir, entries: dict) -> None:
    """Write the manifest atomically (sorted lines, temp file + rename)."""
    import pathlib
    d = pathlib.Path(cache_dir)
    d.mkdir(parents=True, exist_ok=True)
    body = "".join(sorted(e.line() + "\n" for e in entries.values()))
    tmp = d / (MANIFEST_NAME + ".tmp")
    tmp.write_text(body, encoding="utf-8")
    os.replace(tmp, d / MANIFEST_NAME)


_REDUCE_OP = {"reduce_accu": _clib.BM_R_ACCU, "reduce_min": _clib.BM_R_MIN, "reduce_max": _clib.BM_R_MAX,
              "reduce_dot": _clib.BM_R_DOT, "accu": _clib.BM_R_ACCU, "min": _clib.BM_R_MIN,
              "max": _clib.BM_R_MAX, "dot": _clib.BM_R_DOT}
_RDIM_OP = {"rdim_sum": _clib.BM_R_ACCU, "rdim_min": _clib.BM_R_MIN, "rdim_max": _clib.BM_R_MAX,
            "rdim_mean": _clib.BM_R_MEAN, "rdim_var": _clib.BM_R_VAR}
_MOVE_SUB = {"mov_extract_strided": _clib.BM_MOV_EXTRACT, "mov_insert_strided": _clib.BM_MOV_INSERT,
             "mov_resize": _clib.BM_MOV_RESIZE, "mov_reshape_copy": _clib.BM_MOV_RESHAPE,
             "mov_join_rows": _clib.BM_MOV_JOIN_ROWS, "mov_join_cols": _clib.BM_MOV_JOIN_COLS,
             "mov_diagmat_build": _clib.BM_MOV_DIAGMAT, "mov_diagvec_extract": _clib.BM_MOV_DIAGVEC,
             "gen_repmat": _clib.BM_MOV_REPMAT}
_NPSTR_TO_ELEM = {np.dtype(v).str: k for k, v in kernels.NP_DTYPE.items()}


def scalar_for(k, elem_type: str):
    """The scalar constant as the device sees it: np.float32(k) / np.float64(k)
    for floats, dtype(int(k)) for integers with numpy's overflow checks
    (kernels.py:280-283)."""
    dt = kernels.NP_DTYPE[elem_type]
    if dt.kind in "iu":
        return dt.type(int(k))
    return dt.type(k)


def _fill_view(cv: _clib.View, view) -> None:
    buf = view.buf
    cv.base = buf.ptr
    cv.dtype = _clib.DTYPE_CODE[buf.elem_type]
    if isinstance(view, FlatView):
        count = view.count if view.count >= 0 else buf.length
        cv.offset, cv.count, cv.stride = view.offset, count, view.stride
        cv.rows, cv.cols, cv.lda = 1, count, view.stride
        cv.is_block = 0
    else:
        cv.offset, cv.count, cv.stride = view.offset, view.rows * view.cols, 1
        cv.rows, cv.cols, cv.lda = view.rows, view.cols, view.lda
        cv.is_block = 1


def _view_bounds_ok(view) -> bool:
    buf = view.buf
    if isinstance(view, FlatView):
        count = view.count if view.count >= 0 else buf.length
        if count == 0:
            return True
        last = view.offset + view.stride * (count - 1)
        return view.offset >= 0 and 0 <= last < buf.length
    if view.rows == 0 or view.cols == 0:
        return True
    last = view.offset + (view.cols - 1) * view.lda + (view.rows - 1)
    return view.offset >= 0 and last < buf.length


class _ProgramBuilder:
    """Encodes a post-order stage program (expr.py:611-657) into opcode triples
    and a scalar table for one compute dtype."""

    def __init__(self, inv: _clib.Invocation, elem_type: str):
        self.inv = inv
        self.elem = elem_type
        self.n = 0
        self.ns = 0

    def _push(self, tag: int, op: int, arg: int) -> None:
        if self.n >= _clib.BM_MAX_PROG:
            raise BufferError_("fused program longer than the device limit")
        self.inv.prog[3 * self.n] = tag
        self.inv.prog[3 * self.n + 1] = op
        self.inv.prog[3 * self.n + 2] = arg
        self.n += 1

    def _scalar(self, k) -> int:
        if self.ns >= _clib.BM_MAX_SCALARS:
            raise BufferError_("fused program has too many scalars")
        v = scalar_for(k, self.elem)
        if kernels.NP_DTYPE[self.elem].kind in "iu":
            iv = int(v)
            self.inv.iscalars[self.ns] = iv - (1 << 64) if iv >= (1 << 63) else iv
            self.inv.fscalars[self.ns] = 0.0
        else:
            self.inv.fscalars[self.ns] = float(k)
            self.inv.iscalars[self.ns] = 0
        self.ns += 1
        return self.ns - 1

    def stage(self, st: tuple) -> None:
        tag = st[0]
        if tag == "load":
            self._push(_clib.BM_P_LOAD, 0, int(st[1]))
        elif tag == "unary":
            op = st[1]
            if op == "eop_pow":
                k = st[2]
                if kernels.NP_DTYPE[self.elem].kind in "iu" and int(k) < 0:
                    raise ValueError("Integers to negative integer powers are not allowed.")
                self._push(_clib.BM_P_UNARY, _clib.UNARY_CODE[op], self._scalar(k))
            else:
                self._push(_clib.BM_P_UNARY, _clib.UNARY_CODE[op], -1)
        elif tag == "scalar":
            self._push(_clib.BM_P_SCALAR, _clib.SCALAR_CODE[st[1]], self._scalar(st[2]))
        elif tag == "glue":
            self._push(_clib.BM_P_GLUE, _clib.GLUE_CODE[st[1]], 0)
        else:
            raise KeyError(tag)

    def finish(self) -> None:
        self.inv.n_prog = self.n
        self.inv.n_scalars = self.ns


def _single_stage_program(kind: str, scalars: tuple, n_in: int) -> tuple:
    if kind in kernels.EGLUE:
        return (("load", 0), ("load", 1), ("glue", kind))
    if kind in kernels.EOP_SCALAR:
        return (("load", 0), ("scalar", kind, scalars[0]))
    if kind in kernels.EOP_UNARY:
        return (("load", 0), ("unary", kind, scalars[0] if scalars else None))
    raise KeyError(kind)


_CODE_TO_ELEM = {v: k for k, v in _clib.DTYPE_CODE.items()}


def build_invocation(inv: KernelInvocation) -> _clib.Invocation:
    """KernelInvocation (runtime.py:103-109) -> bm_invocation (b200mat.h)."""
    c = _clib.Invocation()
    kind = inv.kind
    ins = list(inv.inputs)
    if len(ins) > _clib.BM_MAX_INPUTS:
        raise BufferError_("too many inputs for one device invocation")
    c.n_inputs = len(ins)
    for i, v in enumerate(ins):
        _fill_view(c.inputs[i], v)
    if inv.output is not None:
        c.has_output = 1
        _fill_view(c.output, inv.output)
    p = inv.params

    if kind in kernels.ELEMENTWISE or kind == "fused_chain" or kind == "mov_copy":
        c.kind = _clib.BM_K_EWISE
        if kind == "fused_chain":
            elem = _NPSTR_TO_ELEM[np.dtype(p["compute_dtype"]).str]
            program = p["program"]
        elif kind == "mov_copy":
            elem = ins[0].buf.elem_type
            program = (("load", 0),)
        else:
            elem = ins[0].buf.elem_type
            program = _single_stage_program(kind, inv.scalars, len(ins))
        c.compute_dtype = _clib.DTYPE_CODE[elem]
        pb = _ProgramBuilder(c, elem)
        for st in program:
            pb.stage(st)
        pb.finish()
        return c
    if kind in _REDUCE_OP or kind == "fused_reduce":
        c.kind = _clib.BM_K_REDUCE
        if kind == "fused_reduce":
            elem = _NPSTR_TO_ELEM[np.dtype(p["compute_dtype"]).str]
            program = p["program"]
            c.reduce_op = _REDUCE_OP[p["op"]]
        else:
            elem = ins[0].buf.elem_type
            c.reduce_op = _REDUCE_OP[kind]
            program = (("load", 0), ("load", 1)) if kind == "reduce_dot" else (("load", 0),)
        c.compute_dtype = _clib.DTYPE_CODE[elem]
        pb = _ProgramBuilder(c, elem)
        for st in program:
            pb.stage(st)
        pb.finish()
        return c
    if kind == "fused_rdim":
        # dim-0 sum / mean / min / max of an element-wise program (b200mat.h BM_K_RDIM_FUSED)
        c.kind = _clib.BM_K_RDIM_FUSED
        elem = _NPSTR_TO_ELEM[np.dtype(p["compute_dtype"]).str]
        c.compute_dtype = _clib.DTYPE_CODE[elem]
        c.reduce_op = _RDIM_OP[p["op"]]
        c.dim = int(p.get("dim", 0))
        c.iparams[0] = int(p["rows"])
        c.iparams[1] = int(p.get("cols", 0))
        pb = _ProgramBuilder(c, elem)
        for st in p["program"]:
            pb.stage(st)
        pb.finish()
        return c
    if kind in _RDIM_OP:
        c.kind = _clib.BM_K_RDIM
        c.reduce_op = _RDIM_OP[kind]
        c.dim = int(p["dim"])
        c.compute_dtype = _clib.DTYPE_CODE[ins[0].buf.elem_type]
        return c
    if kind == "gemm":
        c.kind = _clib.BM_K_GEMM
        c.trans_a = int(p.get("trans_a", 0))
        c.trans_b = int(p.get("trans_b", 0))
        c.compute_dtype = _clib.DTYPE_CODE[ins[0].buf.elem_type]
        return c
    if kind == "mov_transpose":
        c.kind = _clib.BM_K_TRANSPOSE
        return c
    if kind in _MOVE_SUB:
        c.kind = _clib.BM_K_STRIDED_COPY
        c.sub_kind = _MOVE_SUB[kind]
        if kind == "mov_diagvec_extract":
            c.iparams[0] = int(p["k"])
        if kind == "gen_repmat":
            c.iparams[0] = int(p["rows_out"])
        return c
    if kind == "gen_fill_const":
        c.kind = _clib.BM_K_FILL
        out_dt = kernels.NP_DTYPE[inv.output.buf.elem_type]
        gen_val = scalar_for(inv.scalars[0], p["gen_type"])
        with np.errstate(invalid="ignore", over="ignore"):
            bits = np.array([gen_val]).astype(out_dt)
        raw = bits.tobytes() + b"\0" * (8 - out_dt.itemsize)
        c.iparams[0] = int(np.frombuffer(raw, dtype=np.int64)[0])
        return c
    if kind == "gen_eye":
        c.kind = _clib.BM_K_EYE
        out_dt = kernels.NP_DTYPE[inv.output.buf.elem_type]
        one = np.array([kernels.NP_DTYPE[p["gen_type"]].type(1)]).astype(out_dt)
        raw = one.tobytes() + b"\0" * (8 - out_dt.itemsize)
        c.iparams[0] = int(np.frombuffer(raw, dtype=np.int64)[0])
        c.iparams[2] = int(p["rows"])
        return c
    if kind == "gen_linspace":
        c.kind = _clib.BM_K_LINSPACE
        c.compute_dtype = _clib.DTYPE_CODE[p["gen_type"]]
        c.fscalars[0] = float(inv.scalars[0])
        c.fscalars[1] = float(inv.scalars[1])
        c.n_scalars = 2
        c.iparams[0] = int(p["n"])
        return c
    if kind in ("gen_randu", "gen_randn"):
        c.kind = _clib.BM_K_RANDU if kind == "gen_randu" else _clib.BM_K_RANDN
        c.compute_dtype = _clib.DTYPE_CODE[p["gen_type"]]
        c.iparams[0] = rng_key(int(p["seed"]), int(p["stream"]))
        return c
    if kind == "gemm_epi":
        # GEMM epilogue fusion: inputs A, B, then the program's inputs 1..; program input 0
        # is the product (b200mat.h BM_K_GEMM_EPI)
        c.kind = _clib.BM_K_GEMM_EPI
        elem = _NPSTR_TO_ELEM[np.dtype(p["compute_dtype"]).str]
        c.compute_dtype = _clib.DTYPE_CODE[elem]
        pb = _ProgramBuilder(c, elem)
        for st in p["program"]:
            pb.stage(st)
        pb.finish()
        c.trans_a, c.trans_b = int(p["trans_a"]), int(p["trans_b"])
        return c
    if kind == "gemm_fused":
        # GEMM prologue fusion: A's program (over inputs [0, na)), then B's
        # (loads relative to B's inputs), evaluated inside the split pre-pass
        c.kind = _clib.BM_K_GEMM_FUSED
        elem = inv.output.buf.elem_type          # f32: 3xTF32 split pre-pass; f64: DMMA producer
        c.compute_dtype = _clib.DTYPE_CODE[elem]
        pb = _ProgramBuilder(c, elem)
        for st in p["a_prog"]:
            pb.stage(st)
        npa = pb.n
        for st in p["b_prog"]:
            pb.stage(st)
        pb.finish()
        c.trans_a, c.trans_b = int(p["trans_a"]), int(p["trans_b"])
        c.iparams[0], c.iparams[1] = int(p["na"]), npa
        c.iparams[2], c.iparams[3] = int(p["a_rows"]), int(p["b_rows"])
        c.iparams[4], c.iparams[5], c.iparams[6] = int(p["m"]), int(p["n"]), int(p["k"])
        return c
    if kind == "logistic_grad":
        # fused g = X^T F(X w, ...) with r = F(...) (bm_lgrad.cuh): inputs X, w, r
        # (written), then the program's inputs 1..; program input 0 is X w
        c.kind = _clib.BM_K_LOGISTIC_GRAD
        elem = _NPSTR_TO_ELEM[np.dtype(p["compute_dtype"]).str]
        c.compute_dtype = _clib.DTYPE_CODE[elem]
        pb = _ProgramBuilder(c, elem)
        for st in p["program"]:
            pb.stage(st)
        pb.finish()
        c.iparams[0] = int(p.get("accu_ptr", 0))   # f32 slot for accu(r) in the reference's order
        return c
    if kind in ("pred_count", "pred_all_any", "pred_find_build"):
        # element-vs-scalar predicates (kernels.py:643-699): the threshold is
        # cast to the element type first (_scalar), the count is u64
        c.kind = _clib.BM_K_PRED_FIND if kind == "pred_find_build" else _clib.BM_K_PRED_COUNT
        elem = ins[0].buf.elem_type
        c.iparams[0] = _clib.PRED_CODE[p["op"]]
        k = scalar_for(p["threshold"], elem)
        if kernels.NP_DTYPE[elem].kind in "iu":
            c.iscalars[0] = int(np.array([k]).view(np.int64)[0]) if elem == "u64" else int(k)
        else:
            c.fscalars[0] = float(k)
        c.n_scalars = 1
        c.compute_dtype = _clib.BM_U64
        return c
    raise NotImplementedError(f"kernel kind {kind!r} is not provided by the B200 device library")


_M64 = (1 << 64) - 1


def _mix64_int(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def rng_key(seed: int, stream: int) -> int:
    """Per-fill key of the counter RNG (kernels.py:243), as a signed int64."""
    key = _mix64_int((seed & _M64) ^ _mix64_int(stream & _M64))
    return key - (1 << 64) if key >= (1 << 63) else key


# ---------------------------------------------------------------------------
# runtime

class Runtime:
    def __init__(self, descriptor: DeviceDescriptor, print_info: bool):
        self.descriptor = descriptor
        self.counters = Counters()
        self._lock = threading.RLock()
        self._next_buffer_id = 0
        self._next_stream_id = 0
        self.seed = int(os.environ.get(SEED_ENV, "42"))
        self._section_mark = Counters()
        self._live: dict[int, int] = {}     # buffer_id -> device pointer
        self._pool: dict[int, list] = {}    # byte size -> released device pointers (acquire_memory)
        self._pool_bytes = 0
        self._sums: dict = {}               # buffer_id -> 1-element buffer holding its accu (sum cache)
        self._queued_ids: set = set()       # buffers used by work enqueued since the last synchronise
        self._pending_error = None          # raised at the next synchronise (asynchronous error contract)
        self.cache_dir = pathlib.Path(os.environ.get(CACHE_DIR_ENV, str(pathlib.Path.home() / ".devmat")))
        self._lib = _clib.lib()
        self._jit_base = self._native_counters()
        if print_info:
            d = descriptor
            print(f"b200mat runtime: backend={d.backend_name} device={d.device_id} gpu={d.gpu_name} "
                  f"sms={d.sm_count} arch=sm_100a f64=yes jit_cache={'on' if os.environ.get('BM_CACHE_DIR', '1') else 'off'}")

    # -- instrumentation -----------------------------------------------------------
    def _native_counters(self) -> _clib.Counters:
        c = _clib.Counters()
        self._lib.bm_get_counters(ctypes.byref(c))
        return c

    def kernel_inventory_size(self) -> int:
        return len(kernels.ALL_KINDS)

    def _sync_jit_counters(self) -> None:
        n = self._native_counters()
        self.counters.compiles = n.jit_compiles - self._jit_base.jit_compiles
        self.counters.cache_hits = n.jit_cache_hits - self._jit_base.jit_cache_hits

    # -- memory ------------------------------------------------------------------------
    # Buffers released in stream order (release_deferred) are kept, by byte size, for the
    # next acquisition of the same size: reusing one is as stream-ordered as the
    # cudaFreeAsync / cudaMallocAsync pair it replaces (one stream per device), and the
    # repeated steps of a loop (config 5: r, g and a sum slot per step) skip both library
    # calls.  Bounded (POOL_MAX_BYTES, buffers up to POOL_MAX_BUFFER bytes); flushed when
    # an allocation fails and at shutdown.
    POOL_MAX_BYTES = 1 << 30
    POOL_MAX_BUFFER = 64 << 20

    @staticmethod
    def _nbytes(n: int, elem_type: str) -> int:
        return max(n * kernels.itemsize(elem_type), 16)    # bm_alloc: zero-length buffers take 16 B

    def _pool_take(self, nbytes: int) -> int:
        with self._lock:
            lst = self._pool.get(nbytes)
            if lst:
                self._pool_bytes -= nbytes
                return lst.pop()
        return 0

    def flush_pool(self) -> None:
        """Return every pooled buffer to the device allocator (stream-ordered)."""
        with self._lock:
            ptrs = [p for lst in self._pool.values() for p in lst]
            self._pool.clear()
            self._pool_bytes = 0
        for p in ptrs:
            self._lib.bm_free_async(p)

    def acquire_memory(self, n: int, elem_type: str) -> DeviceBuffer:
        if n < 0:
            raise ValueError("negative buffer length")
        if elem_type not in kernels.ELEM_TYPES:
            raise TypeError(f"unknown element type {elem_type!r}")
        nbytes = self._nbytes(n, elem_type)
        p = self._pool_take(nbytes) if self._pool else 0
        if not p:
            ptr = ctypes.c_void_p()
            rc = self._lib.bm_alloc(nbytes, ctypes.byref(ptr))
            if rc != _clib.BM_OK and self._pool:
                self.flush_pool()              # pooled buffers may be what the device lacks
                rc = self._lib.bm_alloc(nbytes, ctypes.byref(ptr))
            _clib.check(rc, "acquire_memory")
            p = ptr.value or 0
        with self._lock:
            buf = DeviceBuffer(self.descriptor.device_id, self._next_buffer_id, n, elem_type, p)
            self._next_buffer_id += 1
            self._live[buf.buffer_id] = buf.ptr
            self.counters.buffers_acquired += 1
        return buf

    def _retire(self, buf: DeviceBuffer) -> int:
        if self._sums:
            self.forget_sum(buf.buffer_id)
        with self._lock:
            ptr = self._live.pop(buf.buffer_id, None)
            if ptr is None:
                raise BufferError_(f"double release of buffer #{buf.buffer_id}")
            self.counters.buffers_released += 1
        return ptr

    def release(self, buf: DeviceBuffer) -> None:
        """Release now; the handle becomes invalid (the memory returns to the
        pool once work already queued on the stream has finished).

        The reference frees at once, so a queued kernel that still uses the
        buffer fails and the error surfaces at the next synchronise
        (runtime.py:441-447, 340-353; tests/test_runtime.py:228-235).  The
        stream-ordered free makes that race harmless here, but it is still the
        caller's bug: releasing a buffer that work enqueued since the last
        synchronise uses is reported as BufferError_ at the next synchronise
        (deterministically: on the reference it depends on the dispatcher's
        timing; a B200 kernel usually finishes before the host gets here).
        release_deferred is the ordered release and never reports."""
        bid = buf.buffer_id
        with self._lock:
            if bid in self._queued_ids:
                if self._pending_error is None:
                    self._pending_error = BufferError_(
                        f"buffer #{bid} released while queued work still used it")
        _clib.check(self._lib.bm_free(self._retire(buf)), "release")

    def release_deferred(self, buf: DeviceBuffer) -> None:
        """Stream-ordered release (runtime.py:449-451): back to the size pool, or
        cudaFreeAsync."""
        ptr = self._retire(buf)
        nbytes = self._nbytes(buf.length, buf.elem_type)
        if nbytes <= self.POOL_MAX_BUFFER:
            with self._lock:
                if self._pool_bytes + nbytes <= self.POOL_MAX_BYTES:
                    self._pool.setdefault(nbytes, []).append(ptr)
                    self._pool_bytes += nbytes
                    return
        _clib.check(self._lib.bm_free_async(ptr), "release_deferred")

    # -- sum cache ----------------------------------------------------------------------------
    # A fused step may leave accu(result) -- in the reference's order, bit-identical to
    # reduce_accu -- in a 1-element device buffer beside a matrix it returns (the fused
    # logistic step's r, expr.py _logistic).  accu() of that matrix then reads 4 bytes
    # instead of running a reduction.  Any write to the buffer through the runtime
    # (enqueue output, copies, element writes, release) forgets the entry;
    # dist.torch_view() forgets it too, since it hands out writable memory.
    def remember_sum(self, buf: DeviceBuffer, slot: DeviceBuffer) -> None:
        self.forget_sum(buf.buffer_id)
        self._sums[buf.buffer_id] = slot

    def sum_slot(self, buf: DeviceBuffer):
        """The 1-element device buffer holding the cached accu of ``buf``, or None."""
        return self._sums.get(buf.buffer_id) if self._sums else None

    def cached_sum(self, buf: DeviceBuffer):
        """The cached accu of ``buf`` as a numpy scalar, or None."""
        slot = self._sums.get(buf.buffer_id) if self._sums else None
        if slot is None:
            return None
        return self.copy_d2h(slot, 0, 1)[0]

    def forget_sum(self, buffer_id: int) -> None:
        slot = self._sums.pop(buffer_id, None)
        if slot is not None:
            self.release_deferred(slot)

    def live(self, buf: DeviceBuffer) -> bool:
        return buf.buffer_id in self._live

    def next_stream_id(self) -> int:
        with self._lock:
            s = self._next_stream_id
            self._next_stream_id += 1
        return s

    # -- queue ---------------------------------------------------------------------------
    def _validate(self, inv: KernelInvocation) -> None:
        views = list(inv.inputs) + ([inv.output] if inv.output is not None else [])
        for v in views:
            if v.buf.device_id != self.descriptor.device_id:
                raise BufferError_("cross-device buffer mix")
            if v.buf.buffer_id not in self._live:
                raise BufferError_(f"use of released buffer #{v.buf.buffer_id}")
            if not _view_bounds_ok(v):
                raise BufferError_(f"view out of bounds ({v!r})")

    def enqueue(self, inv: KernelInvocation) -> None:
        self._validate(inv)
        if self._sums:
            if inv.output is not None:
                self.forget_sum(inv.output.buf.buffer_id)
            if inv.kind == "logistic_grad":          # writes r through its input view 2
                self.forget_sum(inv.inputs[2].buf.buffer_id)
        c = build_invocation(inv)
        _clib.check(self._lib.bm_enqueue(ctypes.byref(c)), inv.kind)
        with self._lock:
            self.counters.launches += 1
            # buffers unfinished work may use (release() race report); bounded
            if len(self._queued_ids) > 4096:
                self._queued_ids.clear()
            for v in inv.inputs:
                self._queued_ids.add(v.buf.buffer_id)
            if inv.output is not None:
                self._queued_ids.add(inv.output.buf.buffer_id)

    def prebuild(self, inv: KernelInvocation):
        """Validate and build ``inv`` once.  The returned prototype is re-addressed
        per call by enqueue_prebuilt / execute_reduce_prebuilt (expr.py plan
        recipes): views keep their geometry, only buffer addresses change."""
        self._validate(inv)
        return build_invocation(inv)

    def _readdress(self, proto, bufs: list, out_buf, accu_ptr: int):
        live = self._live
        c = _clib.Invocation.from_buffer_copy(proto)
        for k, b in enumerate(bufs):
            if b.buffer_id not in live:
                raise BufferError_(f"use of released buffer #{b.buffer_id}")
            c.inputs[k].base = b.ptr
        if out_buf is not None:
            c.output.base = out_buf.ptr
        if accu_ptr:
            c.iparams[0] = accu_ptr
        return c

    def enqueue_prebuilt(self, proto, kind: str, bufs: list, out_buf, accu_ptr: int = 0) -> None:
        """enqueue() of a prototype from prebuild() on this call's buffers
        (``bufs`` = the input views' buffers in order)."""
        c = self._readdress(proto, bufs, out_buf, accu_ptr)
        if self._sums:
            if out_buf is not None:
                self.forget_sum(out_buf.buffer_id)
            if kind == "logistic_grad":
                self.forget_sum(bufs[2].buffer_id)
        _clib.check(self._lib.bm_enqueue(ctypes.byref(c)), kind)
        with self._lock:
            self.counters.launches += 1
            if len(self._queued_ids) > 4096:
                self._queued_ids.clear()
            for b in bufs:
                self._queued_ids.add(b.buffer_id)
            if out_buf is not None:
                self._queued_ids.add(out_buf.buffer_id)

    def synchronise(self) -> None:
        rc = self._lib.bm_sync()
        with self._lock:
            self._queued_ids.clear()
            err, self._pending_error = self._pending_error, None
        _clib.check(rc, "synchronise")
        if err is not None:
            raise err

    def execute_reduce(self, inv: KernelInvocation):
        """Enqueue a reducing invocation, wait, and return its scalar as a
        numpy scalar of the element type (one device-to-host transfer)."""
        return self.execute_reduce_prebuilt(self.prebuild(inv), inv.kind, [v.buf for v in inv.inputs])

    def execute_reduce_prebuilt(self, proto, kind: str, bufs: list):
        """execute_reduce() of a prototype from prebuild() on this call's buffers."""
        c = self._readdress(proto, bufs, None, 0)
        elem = _CODE_TO_ELEM[c.compute_dtype]
        dt = kernels.NP_DTYPE[elem]
        raw = (ctypes.c_char * 8)()
        rc = self._lib.bm_execute_reduce(ctypes.byref(c), raw)
        with self._lock:
            self.counters.launches += 1
        _clib.check(rc, kind)
        with self._lock:
            self._queued_ids.clear()          # the call drained the stream
        value = np.frombuffer(bytes(raw)[: dt.itemsize], dtype=dt)[0]
        nbytes = kernels.itemsize(bufs[0].elem_type) if bufs else 8
        with self._lock:
            self.counters.transfers_d2h += 1
            self.counters.bytes_d2h += nbytes
        return value

    # -- transfers --------------------------------------------------------------------------
    def copy_h2d(self, host: np.ndarray, buf: DeviceBuffer, offset: int = 0) -> None:
        if buf.buffer_id not in self._live:
            raise BufferError_(f"use of released buffer #{buf.buffer_id}")
        arr = np.ascontiguousarray(np.asarray(host).reshape(-1).astype(kernels.NP_DTYPE[buf.elem_type], copy=False))
        if offset < 0 or offset + arr.shape[0] > buf.length:
            raise BufferError_("host copy out of bounds")
        isz = arr.itemsize
        if self._sums:
            self.forget_sum(buf.buffer_id)
        _clib.check(self._lib.bm_h2d(buf.ptr + offset * isz, arr.ctypes.data, arr.nbytes), "copy_h2d")
        with self._lock:
            self.counters.transfers_h2d += 1
            self.counters.bytes_h2d += arr.nbytes

    def copy_d2h(self, buf: DeviceBuffer, offset: int = 0, count: int = -1) -> np.ndarray:
        if buf.buffer_id not in self._live:
            raise BufferError_(f"use of released buffer #{buf.buffer_id}")
        dt = kernels.NP_DTYPE[buf.elem_type]
        n = buf.length - offset if count < 0 else count
        if offset < 0 or n < 0 or offset + n > buf.length:
            raise BufferError_("device copy out of bounds")
        out = np.empty(n, dtype=dt)
        if n:
            _clib.check(self._lib.bm_d2h(out.ctypes.data, buf.ptr + offset * dt.itemsize, out.nbytes), "copy_d2h")
            with self._lock:
                self._queued_ids.clear()      # the copy drained the stream
        else:
            self.synchronise()
        with self._lock:
            self.counters.transfers_d2h += 1
            self.counters.bytes_d2h += out.nbytes
        return out

    def copy_d2d(self, src: DeviceBuffer, dst: DeviceBuffer, count: int = -1) -> None:
        """Device-side memcpy on the stream; neither a launch nor a host transfer."""
        for b in (src, dst):
            if b.buffer_id not in self._live:
                raise BufferError_(f"use of released buffer #{b.buffer_id}")
        n = src.length if count < 0 else count
        if n > src.length or n > dst.length:
            raise BufferError_("d2d copy out of bounds")
        nbytes = n * kernels.itemsize(src.elem_type)
        if self._sums:
            self.forget_sum(dst.buffer_id)
        _clib.check(self._lib.bm_d2d(dst.ptr, src.ptr, nbytes), "copy_d2d")

    def read_scalar(self, buf: DeviceBuffer, index: int):
        return self.read_elems(buf, [index])[0]

    def read_elems(self, buf: DeviceBuffer, indices) -> np.ndarray:
        if buf.buffer_id not in self._live:
            raise BufferError_(f"use of released buffer #{buf.buffer_id}")
        idx = np.ascontiguousarray(np.asarray(indices, dtype=np.int64).reshape(-1))
        if idx.size and (idx.min() < 0 or idx.max() >= buf.length):
            raise BufferError_("element index out of bounds")
        dt = kernels.NP_DTYPE[buf.elem_type]
        out = np.empty(idx.shape[0], dtype=dt)
        _clib.check(self._lib.bm_read_elems(buf.ptr, _clib.DTYPE_CODE[buf.elem_type],
                                            idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), idx.shape[0],
                                            out.ctypes.data), "read_elems")
        with self._lock:
            self.counters.transfers_d2h += 1
            self.counters.bytes_d2h += out.nbytes
        return out

    def write_scalar(self, buf: DeviceBuffer, index: int, value) -> None:
        if buf.buffer_id not in self._live:
            raise BufferError_(f"use of released buffer #{buf.buffer_id}")
        if not 0 <= index < buf.length:
            raise BufferError_("element index out of bounds")
        dt = kernels.NP_DTYPE[buf.elem_type]
        arr = np.array([value]).astype(dt)
        if self._sums:
            self.forget_sum(buf.buffer_id)
        _clib.check(self._lib.bm_write_elem(buf.ptr, _clib.DTYPE_CODE[buf.elem_type], index, arr.ctypes.data),
                    "write_scalar")
        with self._lock:
            self.counters.transfers_h2d += 1
            self.counters.bytes_h2d += dt.itemsize

    # -- counters ---------------------------------------------------------------------------
    def counters_snapshot(self) -> Counters:
        with self._lock:
            self._sync_jit_counters()
            return self.counters.copy()

    def counters_reset_section(self) -> Counters:
        with self._lock:
            self._sync_jit_counters()
            delta = self.counters - self._section_mark
            self._section_mark = self.counters.copy()
        return delta

    def stop(self) -> None:
        _clib.check(self._lib.bm_sync(), "shutdown")


# ---------------------------------------------------------------------------
# singleton management (runtime.py:563-690)

_runtime: Runtime | None = None
_runtime_lock = threading.Lock()
_generation = 0


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = _clib.lib().bm_device_count(ctypes.byref(n))
    return n.value if rc == 0 else 0


def _make_descriptor(backend: str, device_id: int, worker_count: int | None) -> DeviceDescriptor:
    if backend not in BACKENDS:
        raise BackendError(f"unknown backend {backend!r}; valid backends: {', '.join(BACKENDS)}")
    if backend == "reference" and device_id != 0:
        raise BackendError("reference backend exposes a single device id 0")
    if worker_count is not None and worker_count < 1:
        raise BackendError("worker_count must be >= 1")
    n = device_count()
    if n == 0:
        raise BackendError(f"no CUDA device available: {_clib.last_error()} (there is no CPU fallback)")
    if not 0 <= device_id < n:
        raise BackendError(f"device id {device_id} out of range: {n} CUDA device(s) visible")
    return DeviceDescriptor(backend, device_id, worker_count or 1, True)


def init(backend: str | None = None, print_info: bool = False, device_id: int = 0,
         worker_count: int | None = None) -> None:
    """Select and start the device; at most once before shutdown()."""
    global _runtime, _generation
    with _runtime_lock:
        if _runtime is not None:
            raise BackendError("runtime already initialised; call shutdown() first")
        if backend is None:
            backend = os.environ.get(BACKEND_ENV) or "b200"
        desc = _make_descriptor(backend, device_id, worker_count)
        lib = _clib.lib()
        _clib.check(lib.bm_init(desc.device_id), "bm_init")
        name = ctypes.create_string_buffer(128)
        sms = ctypes.c_int()
        lib.bm_device_info(name, 128, ctypes.byref(sms), None, None, None)
        desc = replace(desc, gpu_name=name.value.decode(), sm_count=sms.value)
        _runtime = Runtime(desc, print_info)
        _generation += 1


_shutdown_hooks: list = []   # callables run before the library shuts down (dist: forget peer exchanges)


def shutdown() -> None:
    """Drain the stream, free every live buffer, clear the singleton."""
    global _runtime, _generation
    with _runtime_lock:
        if _runtime is None:
            return
        rt = _runtime
        _generation += 1
        try:
            for hook in list(_shutdown_hooks):
                try:
                    hook()
                except Exception:  # noqa: BLE001 - shutdown must finish
                    pass
            rt.stop()
        finally:
            with rt._lock:
                for bid, ptr in list(rt._live.items()):
                    rt._lib.bm_free_async(ptr)
                    rt.counters.buffers_released += 1
                rt._live.clear()
            rt.flush_pool()
            _clib.lib().bm_shutdown()
            _runtime = None


def get_runtime() -> Runtime:
    rt = _runtime
    if rt is None:
        try:
            init()
        except BackendError:
            if _runtime is None:
                raise
        rt = _runtime
    return rt


def is_initialised() -> bool:
    return _runtime is not None


def generation() -> int:
    return _generation


def release_if_current(gen: int, buf: DeviceBuffer) -> None:
    """GC finalizer hook: stream-ordered release iff the owning runtime lives."""
    rt = _runtime
    if rt is None or gen != _generation:
        return
    try:
        rt.release_deferred(buf)
    except Exception:
        pass


def set_seed(seed: int) -> None:
    rt = get_runtime()
    with rt._lock:
        rt.seed = int(seed)
        rt._next_stream_id = 0


def counters() -> Counters:
    return get_runtime().counters_snapshot()


def synchronise() -> None:
    if _runtime is not None:
        _runtime.synchronise()


class wall_clock:
    """tic/toc timer (runtime.py:693-703)."""

    def __init__(self):
        self._t0 = time.perf_counter()

    def tic(self) -> None:
        self._t0 = time.perf_counter()

    def toc(self) -> float:
        return time.perf_counter() - self._t0


class _PinnedBlock:
    def __init__(self, nbytes: int):
        ptr = ctypes.c_void_p()
        _clib.check(_clib.lib().bm_host_alloc_pinned(max(nbytes, 1), ctypes.byref(ptr)), "pinned alloc")
        self.ptr = ptr.value
        self.nbytes = nbytes

    def __del__(self):
        try:
            _clib.lib().bm_host_free_pinned(self.ptr)
        except Exception:
            pass


def pinned_array(shape, dtype, order: str = "F") -> np.ndarray:
    """A numpy array in page-locked host memory (fast, asynchronous-capable
    host<->device copies).  Column-major by default, the layout
    Matrix.from_numpy uploads without a host-side copy.  The memory lives as
    long as the array."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    block = _PinnedBlock(n)
    buf = (ctypes.c_char * max(n, 1)).from_address(block.ptr)
    arr = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape, order=order)
    arr.setflags(write=True)
    _pinned_owners[id(arr)] = block
    import weakref
    weakref.finalize(arr, _pinned_owners.pop, id(arr), None)
    return arr


_pinned_owners: dict = {}


def check_elem_type(elem_type: str) -> None:
    if elem_type not in kernels.ELEM_TYPES:
        raise ElemTypeError(f"unknown element type {elem_type!r}")
