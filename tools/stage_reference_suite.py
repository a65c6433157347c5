"""Stage the reference's own test suite for the drop-in run.

    python tools/stage_reference_suite.py

Copies /root/reference/pkg/tests/*.py (unmodified) to baseline/_ref_tests/.
Like baseline/_ref (the installed reference package), that directory is
git-ignored -- reference sources never enter this repository's history -- but
not gpurun-ignored, so it travels to the GPU box, where
tests/test_reference_suite_dropin.py runs it with ``devmat`` aliased to this
package (tests/dropin/devmat).
"""
import pathlib
import shutil

SRC = pathlib.Path("/root/reference/pkg/tests")
DST = pathlib.Path(__file__).resolve().parents[1] / "baseline" / "_ref_tests"


def main() -> None:
    DST.mkdir(parents=True, exist_ok=True)
    n = 0
    for f in sorted(SRC.glob("*.py")):
        shutil.copy2(f, DST / f.name)
        n += 1
    print(f"staged {n} reference test files in {DST}")


if __name__ == "__main__":
    main()
