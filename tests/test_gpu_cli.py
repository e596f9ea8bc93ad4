"""The command line (``python -m paper_2308_07403_b200 distances|navigate``)
against golden outputs of the reference's own CLI (tests/golden/make_golden_cli.py):
same exit codes, stdout, stderr and distance CSV text, byte for byte."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "tests" / "golden" / "cli"
CASES = json.loads((CLI / "cases.json").read_text())
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(CASES))
def test_cli_matches_reference(cuda, tmp_path, name):
    case = CASES[name]
    args = case["args"]
    inp = tmp_path / f"{name}.txt"
    inp.write_text((CLI / f"{name}.txt").read_text())
    cmd = [sys.executable, "-m", "paper_2308_07403_b200", args[0], "--input", str(inp)] + args[1:]
    if args[0] == "distances":
        cmd += ["--out", str(tmp_path / f"{name}.csv")]
    proc = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert proc.returncode == case["rc"], proc.stderr[-2000:]
    assert proc.stdout.replace(str(tmp_path) + "/", "") == (CLI / f"{name}.out").read_text()
    assert proc.stderr == (CLI / f"{name}.err").read_text()
    if args[0] == "distances":
        assert (tmp_path / f"{name}.csv").read_text() == (CLI / f"{name}.csv").read_text()
