"""The reference's own, unchanged test suite (197 tests, /root/reference/pkg/tests,
staged into baseline/_ref_tests) run against this package as a drop-in:
rdist.linalg / rdist.resolvent / rdist.navigation are this repository's
modules (CUDA kernels), everything else is the stock reference package in
baseline/_ref (tests/reference_suite/dropin.py)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def test_reference_suite_passes_on_the_cuda_path(cuda, tmp_path):
    if not (ROOT / "baseline" / "_ref" / "rdist").exists() or not (
        (ROOT / "baseline" / "_ref_tests").exists() or Path("/root/reference/pkg/tests").exists()
    ):
        pytest.skip("reference package / tests not staged (tests/reference_suite/run.py --stage)")
    out = tmp_path / "suite.json"
    proc = subprocess.run([sys.executable, str(ROOT / "tests" / "reference_suite" / "run.py"), "--out", str(out)],
                          capture_output=True, text=True, timeout=900)
    summary = json.loads(out.read_text())
    assert summary["counts"]["failed"] == 0 and summary["counts"]["error"] == 0, summary["not_passing"][:5]
    assert summary["counts"]["passed"] == 197, proc.stdout[-2000:]
