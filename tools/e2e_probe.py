"""Break down the e2e step of bench.py (GPU box): host->device copies of the
four 64 MiB pinned inputs (sync per copy, async with one sync, through
Matrix.from_numpy) and the config-1 accu."""
import ctypes
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import _clib
    from paper_2308_03120_b200.runtime import pinned_array
    dm.init("b200")
    lib = _clib.lib()
    rng = np.random.default_rng(0)
    pinned = []
    for _ in range(4):
        p = pinned_array((4096, 4096), np.float32, order="F")
        p[...] = rng.random((4096, 4096), dtype=np.float32)
        pinned.append(p)
    dev = [dm.Matrix(4096, 4096) for _ in range(4)]
    dm.accu(2 * dev[0] + dev[1] % dev[2] - dm.exp(dev[3]))
    for rep in range(5):
        t0 = time.perf_counter()
        for p, d in zip(pinned, dev):
            lib.bm_h2d(ctypes.c_void_p(d.mem.ptr), ctypes.c_void_p(p.ctypes.data), p.nbytes)
        t1 = time.perf_counter()
        for p, d in zip(pinned, dev):
            lib.bm_h2d_async(ctypes.c_void_p(d.mem.ptr), ctypes.c_void_p(p.ctypes.data), p.nbytes)
        dm.synchronise()
        t2 = time.perf_counter()
        mats = [dm.Matrix.from_numpy(p) for p in pinned]
        t3 = time.perf_counter()
        v = dm.accu(2 * mats[0] + mats[1] % mats[2] - dm.exp(mats[3]))
        t4 = time.perf_counter()
        del mats
        import gc
        live = len(dm.runtime.get_runtime()._live) if hasattr(dm, "runtime") else -1
        t5 = time.perf_counter()
        ncol = gc.collect()
        t6 = time.perf_counter()
        live2 = len(dm.runtime.get_runtime()._live) if hasattr(dm, "runtime") else -1
        print(f"live buffers before/after gc {live}/{live2} (gc {ncol} objs, {1e3*(t6-t5):.2f} ms)")
        print(f"h2d sync x4 {1e3*(t1-t0):.2f} ms  h2d async x4 {1e3*(t2-t1):.2f} ms  "
              f"from_numpy x4 {1e3*(t3-t2):.2f} ms  accu {1e3*(t4-t3):.3f} ms  v={v}")
    dm.shutdown()


if __name__ == "__main__":
    main()
