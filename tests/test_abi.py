"""The C ABI library loads without a GPU and exports exactly what
include/b200mat.h declares; ctypes structs match the C layout."""
import ctypes
import pathlib
import re
import subprocess

import pytest

from paper_2308_03120_b200 import _clib

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "b200mat.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void\*|const char\*)\s+(bm_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _clib.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _clib.SIGNATURES, f"{s} has no ctypes signature"
    assert set(_clib.SIGNATURES) == set(syms)
    assert lib.bm_abi_version() == 1


def test_no_device_is_reported_not_crashed():
    lib = _clib.lib()
    n = ctypes.c_int(-1)
    rc = lib.bm_device_count(ctypes.byref(n))
    if rc != 0:
        assert n.value == 0
        assert _clib.last_error()
    # queue calls before bm_init fail cleanly
    assert lib.bm_sync() == _clib.BM_ERR_NODEVICE


def test_struct_layout_matches_c(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(bm_view), sizeof(bm_invocation),
         offsetof(bm_invocation, output), offsetof(bm_invocation, fscalars),
         offsetof(bm_invocation, prog), offsetof(bm_invocation, compute_dtype),
         offsetof(bm_invocation, iparams), sizeof(bm_counters));
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    inv = _clib.Invocation
    want = [ctypes.sizeof(_clib.View), ctypes.sizeof(inv), inv.output.offset, inv.fscalars.offset,
            inv.prog.offset, inv.compute_dtype.offset, inv.iparams.offset, ctypes.sizeof(_clib.Counters)]
    assert got == want


def test_header_constants_match_binding():
    text = HEADER.read_text()
    defs = dict(re.findall(r"#define\s+(BM_\w+)\s+(-?\d+)", text))
    for name, value in defs.items():
        if hasattr(_clib, name):
            assert getattr(_clib, name) == int(value), name
    for op, code in _clib.UNARY_CODE.items():
        assert int(defs["BM_U_" + op[4:].upper()]) == code
    scal = {"eop_scalar_plus": "PLUS", "eop_scalar_minus_pre": "MINUS_PRE", "eop_scalar_minus_post": "MINUS_POST",
            "eop_scalar_times": "TIMES", "eop_scalar_div_pre": "DIV_PRE", "eop_scalar_div_post": "DIV_POST"}
    for op, code in _clib.SCALAR_CODE.items():
        assert int(defs["BM_S_" + scal[op]]) == code


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_clib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


# ---- the C example (examples/c_abi_example.c): the ABI from C, no Python -------------------------

def _build_c_example(tmp_path):
    import subprocess
    root = pathlib.Path(__file__).resolve().parents[1]
    exe = tmp_path / "c_abi_example"
    lib_dir = root / "paper_2308_03120_b200"
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", str(root / "include"),
           str(root / "examples" / "c_abi_example.c"), "-L", str(lib_dir), "-lb200mat",
           f"-Wl,-rpath,{lib_dir}", "-lm", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    assert _build_c_example(tmp_path).exists()


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import subprocess
    exe = _build_c_example(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_abi_example: ok" in r.stdout
