"""The reference's own test suite, unmodified, against this package.

tools/stage_reference_suite.py copies /root/reference/pkg/tests to
baseline/_ref_tests (git-ignored, travels to the GPU box).  Here it runs in a
subprocess with tests/dropin first on sys.path, so every ``import devmat`` in
it is this package (tests/dropin/devmat).  Every test outcome is compared with
tests/dropin/expected.py, which classifies each reference test that cannot
pass on the B200 path and why (out of scope per SURVEY.md section 2, or a
documented divergence).  A test that fails without a
classification, or a classified one that now passes, fails this test: the
classification is exact, not a tolerance.
"""
import json
import os
import pathlib
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
SUITE = ROOT / "baseline" / "_ref_tests"
OUT = ROOT / "gpurun_out"


def run_suite(junit: pathlib.Path) -> dict:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "dropin"), str(ROOT), env.get("PYTHONPATH", "")])
    env.pop("DEFAULT_BACKEND", None)
    cmd = [sys.executable, "-m", "pytest", str(SUITE), "-q", "-p", "no:cacheprovider", "--confcutdir", str(SUITE),
           "--rootdir", str(SUITE), "--continue-on-collection-errors", f"--junitxml={junit}", "-o", "junit_family=xunit1", "--timeout", "300"]
    subprocess.run(cmd, cwd=str(SUITE), env=env, capture_output=True, text=True, timeout=3000)
    results = {}
    for case in ET.parse(junit).getroot().iter("testcase"):
        cls = case.get("classname", "")
        nodeid = cls.split(".")[-1] if "." in cls else cls
        module = cls.split(".")[0]
        name = f"{module}::{nodeid}::{case.get('name')}" if nodeid != module else f"{module}::{case.get('name')}"
        status = "passed"
        msg = ""
        for tag in ("failure", "error", "skipped"):
            el = case.find(tag)
            if el is not None:
                status = {"failure": "failed", "error": "error", "skipped": "skipped"}[tag]
                msg = (el.get("message") or "")[:300]
                break
        results[name] = (status, msg)
    return results


@pytest.mark.gpu
@pytest.mark.slow
def test_reference_suite_runs_on_b200():
    if not SUITE.exists():
        pytest.skip("baseline/_ref_tests not staged (python tools/stage_reference_suite.py)")
    sys.path.insert(0, str(ROOT / "tests" / "dropin"))
    from expected import EXPECTED_FAILURES  # noqa: E402
    OUT.mkdir(exist_ok=True)
    res = run_suite(OUT / "reference_suite_junit.xml")
    passed = sorted(k for k, (s, _) in res.items() if s == "passed")
    failed = {k: m for k, (s, m) in res.items() if s in ("failed", "error")}
    summary = {"total": len(res), "passed": len(passed), "failed": len(failed),
               "skipped": sum(1 for s, _ in res.values() if s == "skipped"),
               "failures": {k: {"message": m, "class": EXPECTED_FAILURES.get(k, "UNCLASSIFIED")}
                            for k, m in sorted(failed.items())}}
    (OUT / "reference_suite_summary.json").write_text(json.dumps(summary, indent=1))
    unexpected = sorted(set(failed) - set(EXPECTED_FAILURES))
    fixed = sorted(k for k in EXPECTED_FAILURES if res.get(k, ("missing",))[0] == "passed")
    assert not unexpected, f"unclassified failures: {unexpected[:20]}"
    assert not fixed, f"classified as failing but passes now: {fixed}"
    assert len(res) >= 299
