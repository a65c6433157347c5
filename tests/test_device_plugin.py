"""The drop-in from the other side: the unmodified reference package with the
B200 device behind its Runtime firewall (tests/dropin/b200_device.py, the
binding INTEGRATION.md describes), against the golden outputs of the
reference's own CPU backend.  Runs in a subprocess so ``import devmat`` is
the reference (baseline/_ref), not this package's alias."""
import json
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_unmodified_reference_runs_on_the_b200_device():
    if not (ROOT / "baseline" / "_ref" / "devmat").exists():
        pytest.skip("reference not installed in baseline/_ref")
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "dropin" / "run_reference_on_b200.py")],
                       capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert not res["failures"], res["failures"]
    assert res["checks"] >= 250
    assert res["cfg1_value"] == -7857368.0
    assert res["cfg1_reference_launches"] == 2        # the reference's plan: fused_chain + reduce_accu
