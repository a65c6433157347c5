"""Dump the generated CUDA source of a fused program, compile it offline with
nvcc for sm_100a and print register use + the load/store pattern of the SASS.
Usage: python tools/jit_sass.py cfg1|dot|accu1|store"""
import ctypes
import os
import pathlib
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main(which):
    d = tempfile.mkdtemp()
    os.environ["BM_JIT_DUMP"] = d
    os.environ["BM_CACHE_DIR"] = ""
    from test_planner import FakeMatrix, _flat
    from paper_2308_03120_b200 import _clib
    from paper_2308_03120_b200.runtime import KernelInvocation, build_invocation
    m = [FakeMatrix(4096, 4096) for _ in range(4)]
    cfg1 = (("load", 0), ("scalar", "eop_scalar_times", 2), ("load", 1), ("load", 2), ("glue", "eglue_schur"),
            ("glue", "eglue_plus"), ("load", 3), ("unary", "eop_exp", None), ("glue", "eglue_minus"))
    if which == "cfg1":
        kinv = KernelInvocation("fused_reduce", tuple(_flat(x) for x in m), None, (),
                                {"program": cfg1, "compute_dtype": "<f4", "op": "accu"})
    elif which == "dot":
        kinv = KernelInvocation("fused_reduce", (_flat(m[0]), _flat(m[1])), None, (),
                                {"program": (("load", 0), ("load", 1)), "compute_dtype": "<f4", "op": "dot"})
    elif which == "accu1":
        kinv = KernelInvocation("fused_reduce", (_flat(m[0]),), None, (),
                                {"program": (("load", 0),), "compute_dtype": "<f4", "op": "accu"})
    else:
        kinv = KernelInvocation("fused_chain", tuple(_flat(x) for x in m), _flat(m[0]), (),
                                {"program": cfg1, "compute_dtype": "<f4"})
    inv = build_invocation(kinv)
    rc = _clib.lib().bm_jit_compile_only(ctypes.byref(inv))
    assert rc == 0, _clib.last_error()
    src = next(pathlib.Path(d).glob("fused_*.cu"))
    for h in ("bm_common.cuh", "bm_reduce.cuh"):
        (pathlib.Path(d) / h).write_text((ROOT / "paper_2308_03120_b200" / "csrc" / h).read_text())
    cub = pathlib.Path(d) / "k.cubin"
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-std=c++17",
                        "-Xptxas", "-v", "-cubin", "-o", str(cub), str(src)], capture_output=True, text=True)
    print("\n".join(l for l in r.stderr.splitlines() if "registers" in l or "stack" in l))
    sass = subprocess.run(["cuobjdump", "-sass", str(cub)], capture_output=True, text=True).stdout
    lines = [l for l in sass.splitlines() if any(k in l for k in ("LDG", "STS", "LDS", "BAR", "BRA", "SHFL", "STG"))]
    print("\n".join(l.split(";")[0].strip() for l in lines[: int(os.environ.get("N", "80"))]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg1")
