"""A B200 device for the UNMODIFIED reference package (baseline/_ref/devmat).

This is the binding a devmat maintainer would add, as code:
the reference's Runtime keeps its expression layer, planner, queue contract
and counters; only the two device classes behind its firewall change
(runtime.py:200-360):

* ``B200State`` replaces ``_DeviceState``: buffers are device memory from
  libb200mat.so; ``resolve(view)`` returns a ``DeviceSpan`` that the
  Runtime's transfer methods (runtime.py:497-540) read and write through the
  C ABI instead of numpy slicing.
* ``B200Device`` replaces ``_ReferenceDevice`` / ``_ParallelDevice``: its
  ``submit(("inv", inv))`` translates the KernelInvocation into a
  ``bm_invocation`` (paper_2308_03120_b200.runtime.build_invocation) and
  enqueues it on the CUDA stream (the FIFO queue); reductions fill the
  invocation's result slot like the reference's ``_execute_invocation``
  (runtime.py:285); ``drain`` is ``bm_sync``.

``install(devmat)`` swaps the classes in the reference's runtime module, so
``devmat.init("reference")`` then runs every kernel on the B200.  Nothing of
the reference is edited or copied.
"""
from __future__ import annotations

import ctypes

import numpy as np

from paper_2308_03120_b200 import _clib, kernels
from paper_2308_03120_b200 import runtime as _b2

_REDUCE_KINDS = ("reduce_accu", "reduce_min", "reduce_max", "reduce_dot")


class DeviceSpan:
    """A FlatView's elements in device memory, with the numpy-like surface the
    reference Runtime's transfer methods use on ``_DeviceState.resolve``:
    ``span[:] = host``, ``span[:] = other_span``, ``span.copy()``,
    ``span[idx_array]``, ``span[i] = v``, ``dtype``, ``itemsize``, ``shape``."""

    def __init__(self, lib, ptr: int, elem: str, offset: int, count: int, stride: int):
        self.lib = lib
        self.dtype = kernels.NP_DTYPE[elem]
        self.itemsize = self.dtype.itemsize
        self.elem = elem
        self.base = ptr + offset * self.itemsize
        self.count = count
        self.stride = stride
        self.shape = (count,)

    def _contig(self):
        if self.stride != 1 and self.count > 1:
            raise _b2.BufferError_("strided host transfer")

    def copy(self) -> np.ndarray:
        self._contig()
        out = np.empty(self.count, dtype=self.dtype)
        if self.count:
            _clib.check(self.lib.bm_d2h(out.ctypes.data, ctypes.c_void_p(self.base), out.nbytes), "d2h")
        return out

    def __getitem__(self, idx):
        idx = np.asarray(idx, dtype=np.int64).reshape(-1)
        out = np.empty(idx.shape[0], dtype=self.dtype)
        if idx.shape[0]:
            pos = np.ascontiguousarray(idx * self.stride)
            _clib.check(self.lib.bm_read_elems(ctypes.c_void_p(self.base), _clib.DTYPE_CODE[self.elem],
                                               pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pos.shape[0],
                                               out.ctypes.data), "read elems")
        return out

    def __setitem__(self, key, value) -> None:
        if isinstance(key, (int, np.integer)):
            v = np.array([value]).astype(self.dtype)
            _clib.check(self.lib.bm_write_elem(ctypes.c_void_p(self.base), _clib.DTYPE_CODE[self.elem],
                                               int(key) * self.stride, v.ctypes.data), "write elem")
            return
        if key != slice(None):
            raise TypeError("DeviceSpan supports span[:] and span[i] assignment")
        self._contig()
        if isinstance(value, DeviceSpan):
            value._contig()
            _clib.check(self.lib.bm_d2d(ctypes.c_void_p(self.base), ctypes.c_void_p(value.base),
                                        min(self.count, value.count) * self.itemsize), "d2d")
            return
        host = np.ascontiguousarray(np.asarray(value).reshape(-1).astype(self.dtype, copy=False))
        if host.shape[0] != self.count:
            raise ValueError("host transfer length mismatch")
        if self.count:
            _clib.check(self.lib.bm_h2d(ctypes.c_void_p(self.base), host.ctypes.data, host.nbytes), "h2d")


class B200State:
    """Replaces the reference's _DeviceState (runtime.py:203-244)."""

    def __init__(self, descriptor):
        self.descriptor = descriptor
        self.lib = _clib.lib()
        rc = self.lib.bm_init(0)
        if rc not in (_clib.BM_OK, _clib.BM_ERR_ARG):     # ARG: this process already initialised it
            _clib.check(rc, "bm_init")
        self.ptrs: dict[int, int] = {}
        self.bufs: dict[int, object] = {}

    def allocate(self, buf) -> None:
        p = ctypes.c_void_p()
        _clib.check(self.lib.bm_alloc(buf.length * kernels.itemsize(buf.elem_type), ctypes.byref(p)), "alloc")
        self.ptrs[buf.buffer_id] = p.value
        self.bufs[buf.buffer_id] = buf

    def free(self, buffer_id: int) -> None:
        self.bufs.pop(buffer_id)
        _clib.check(self.lib.bm_free_async(ctypes.c_void_p(self.ptrs.pop(buffer_id))), "free")

    def live(self, buffer_id: int) -> bool:
        return buffer_id in self.ptrs

    @property
    def _arrays(self) -> dict:
        """The reference's shutdown() walks _DeviceState._arrays for leftovers
        (runtime.py:631-634): the live buffer ids."""
        return self.ptrs

    def _ptr(self, buf) -> int:
        p = self.ptrs.get(buf.buffer_id)
        if p is None:
            raise _b2.BufferError_(f"use of released buffer #{buf.buffer_id}")
        return p

    def resolve(self, view) -> DeviceSpan:
        count = view.count if view.count >= 0 else view.buf.length
        return DeviceSpan(self.lib, self._ptr(view.buf), view.buf.elem_type, view.offset, count, view.stride)

    def b200_view(self, v):
        """The reference view as this package's view over the same device memory."""
        b = _b2.DeviceBuffer(v.buf.device_id, v.buf.buffer_id, v.buf.length, v.buf.elem_type, self._ptr(v.buf))
        if hasattr(v, "lda"):
            return _b2.BlockView(b, v.offset, v.rows, v.cols, v.lda)
        return _b2.FlatView(b, v.offset, v.count if v.count >= 0 else v.buf.length, v.stride)


class B200Device:
    """Replaces _ReferenceDevice / _ParallelDevice (runtime.py:290-360): the
    CUDA stream is the FIFO queue; errors raise at submit (like the reference
    backend) or, for asynchronous device faults, at drain."""

    def __init__(self, state: B200State):
        self.state = state
        self.lib = state.lib

    def submit(self, item) -> None:
        kind, payload = item
        if kind == "release":
            payload()                    # Runtime.release -> B200State.free: cudaFreeAsync, stream-ordered
            return
        if kind != "inv":
            return
        inv = payload
        st = self.state
        mapped = _b2.KernelInvocation(inv.kind, tuple(st.b200_view(v) for v in inv.inputs),
                                      None if inv.output is None else st.b200_view(inv.output),
                                      tuple(inv.scalars), dict(inv.params))
        c = _b2.build_invocation(mapped)
        if inv.kind in _REDUCE_KINDS:
            n = inv.inputs[0].count if inv.inputs[0].count >= 0 else inv.inputs[0].buf.length
            if n == 0 and "empty_value" in inv.params:
                inv.params["_result_slot"][0] = inv.params["empty_value"]
                return
            dt = kernels.NP_DTYPE[inv.inputs[0].buf.elem_type]
            raw = (ctypes.c_char * 8)()
            _clib.check(self.lib.bm_execute_reduce(ctypes.byref(c), raw), inv.kind)
            inv.params["_result_slot"][0] = np.frombuffer(bytes(raw)[: dt.itemsize], dtype=dt)[0]
            return
        if inv.kind in ("pred_count", "pred_all_any"):       # one u64 count (kernels.py:643-699)
            raw = (ctypes.c_char * 8)()
            _clib.check(self.lib.bm_execute_reduce(ctypes.byref(c), raw), inv.kind)
            cnt = int(np.frombuffer(bytes(raw), dtype=np.uint64)[0])
            if inv.kind == "pred_count":
                inv.params["_result_slot"][0] = np.uint64(cnt)
            else:
                n = inv.inputs[0].count if inv.inputs[0].count >= 0 else inv.inputs[0].buf.length
                inv.params["_result_slot"][0] = (cnt == n) if inv.params.get("want_all") else (cnt > 0)
            return
        _clib.check(self.lib.bm_enqueue(ctypes.byref(c)), inv.kind)

    def drain(self) -> None:
        _clib.check(self.lib.bm_sync(), "synchronise")

    def stop(self) -> None:
        # the reference frees its leftover buffers after stop(); the library stays
        # initialised for them (and for a later init in this process)
        self.drain()


def install(devmat) -> None:
    """Put the B200 device behind the unmodified reference's firewall: every
    backend name of ``devmat.init`` then runs on the B200."""
    rt = devmat.runtime
    rt._DeviceState = B200State
    rt._ReferenceDevice = B200Device
    rt._ParallelDevice = B200Device
