"""SASS census of the product's kernels (runs here, no GPU): the instructions that
prove the Blackwell paths (B200_PROFILING.md, "What proves a Blackwell-native
kernel") counted per kernel, for the ahead-of-time kernels in libb200mat.so and
for the NVRTC kernels, whose generated sources are dumped by the CPU compile
tests (BM_JIT_DUMP) and compiled here with nvcc for sm_100a with the same
options.  Usage: python tools/sass_census.py > profiles/r02_sass_census.md"""
import collections
import os
import pathlib
import re
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2308_03120_b200" / "csrc"
COLS = [("UTC*MMA", re.compile(r"\bUTC\w*MMA\b")), ("UTMALDG", re.compile(r"\bUTMALDG\b")),
        ("UTMASTG", re.compile(r"\bUTMASTG\b")), ("UBLKCP", re.compile(r"\bUBLKCP\b")),
        ("LDTM", re.compile(r"\bLDTM\b")), ("STTM", re.compile(r"\bSTTM\b")), ("DMMA", re.compile(r"\bDMMA\b")),
        ("HMMA", re.compile(r"\bHMMA\b")), ("LDGSTS", re.compile(r"\bLDGSTS\b")), ("SYNCS", re.compile(r"\bSYNCS\b")),
        ("LDG", re.compile(r"\bLDG\b")), ("STG", re.compile(r"\bSTG\b")), ("LDL", re.compile(r"\bLDL\b")),
        ("STL", re.compile(r"\bSTL\b"))]
HOT = re.compile(r"gemm|split|reduce|rdim|lgrad|fold|exch|dot|accu|bm_store|bm_")


def census(sass: str) -> dict:
    out = {}
    name, counts = None, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name, counts = m.group(1), collections.Counter()
            out[name] = counts
            continue
        if counts is None or "/*" not in line:
            continue
        ins = line.split("*/", 1)[-1]
        for col, rx in COLS:
            if rx.search(ins):
                counts[col] += 1
    return out


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else list(names)


def table(rows, title):
    print(f"## {title}\n")
    print("| kernel | " + " | ".join(c for c, _ in COLS) + " |")
    print("|---|" + "---|" * len(COLS))
    for name, c in rows:
        print(f"| `{name}` | " + " | ".join(str(c.get(col, 0)) for col, _ in COLS) + " |")
    print()


def aot():
    so = ROOT / "paper_2308_03120_b200" / "libb200mat.so"
    sass = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True, check=True).stdout
    res = census(sass)
    names = list(res)
    short = demangle(names)
    rows = []
    for mangled, dem in zip(names, short):
        if not HOT.search(dem):
            continue
        dem = re.sub(r"\(.*\)$", "", dem).replace("bm::", "")
        rows.append((dem[:90], res[mangled]))
    rows.sort(key=lambda r: r[0])
    table(rows, f"ahead-of-time kernels (`cuobjdump -sass {so.relative_to(ROOT)}`)")


def jit():
    d = pathlib.Path(tempfile.mkdtemp())
    env = dict(os.environ, BM_JIT_DUMP=str(d), BM_CACHE_DIR="", BM_F64_PROLOGUE="1")
    sel = ("compiles or fuses_the_consuming or f64_operand or fused_dim_kernels or "
           "split_kernel_compiles or (programs_compile_for_every_type and f32)")
    subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", str(ROOT / "tests" / "test_planner.py"),
                    "-k", sel], env=env, capture_output=True, text=True, cwd=ROOT)
    rows = []
    for src in sorted(d.glob("fused_*.cu")):
        text = src.read_text()
        m = re.search(r'extern "C" __global__ void [^(]*?(\w+)\(', text)
        kname = m.group(1) if m else src.stem
        opts = []
        first = text.splitlines()[0] if text else ""
        if first.startswith("// nvrtc:"):
            opts.append(first.split(":", 1)[1].strip())
        cub = src.with_suffix(".cubin")
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-std=c++17",
                            "-cubin", "-I", str(CSRC), "-o", str(cub), str(src)] +
                           [o for o in opts if o.startswith("-") and not o.startswith("--gpu")],
                           capture_output=True, text=True)
        if r.returncode != 0:
            rows.append((f"{kname} ({src.name}: nvcc failed)", collections.Counter()))
            continue
        sass = subprocess.run(["cuobjdump", "-sass", str(cub)], capture_output=True, text=True).stdout
        for fn, c in census(sass).items():
            tag = re.search(r"(gemm_pair_body|gemm_dmma_body|lgrad|rdim1|reduce_flat|ewise_store|split)", text)
            rows.append((f"{fn} [{tag.group(1) if tag else 'program'}]", c))
    # one row per kernel and count vector, with the number of generated sources that share it
    grouped = collections.Counter((n, tuple(sorted(c.items()))) for n, c in rows)
    rows = [(f"{n} x{k}", collections.Counter(dict(c))) for (n, c), k in sorted(grouped.items())]
    table(rows, "NVRTC kernels (sources dumped by the CPU compile tests, compiled here with nvcc; "
                "xN = generated programs with these counts)")


if __name__ == "__main__":
    print("# SASS census (round 2)\n")
    print("Instruction counts per kernel, static (in the SASS, not executed).  `UTC*MMA` = tcgen05.mma, "
          "`UTMALDG` = TMA tile load, `LDTM`/`STTM` = tcgen05.ld/st, `DMMA` = f64 tensor-core MMA, "
          "`LDGSTS` = cp.async, `SYNCS` = mbarrier ops, `LDL`/`STL` = local memory (spills or stack).  "
          "Made by `python tools/sass_census.py`.  The `LDL`/`STL` in the reduction kernels are the explicit "
          "depth-first stack of `pw_generic` (numpy's pairwise split tree for a length that is not a power-of-two "
          "number of 128-element leaves: at most 48 frames, a few per 8192 elements), not spills of the data loop; "
          "ncu counts 0 executed local loads for config 1's `bm_reduce` and `rdim0_cta_kernel` "
          "(`r02_ncu_full.md`).\n")
    aot()
    jit()
