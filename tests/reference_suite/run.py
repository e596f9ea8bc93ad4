"""Run the reference's unchanged test suite against this package (drop-in check).

    python tests/reference_suite/run.py --stage      # build container: copy the
        # reference's tests next to its installed package (baseline/_ref_tests,
        # git-ignored, travels to the GPU box with gpurun like baseline/_ref)
    python tests/reference_suite/run.py --out gpurun_out/reference_suite.json   # on the B200

The tests run from a temporary copy with a root conftest that installs the
drop-in (dropin.py) before collection; the reference's own conftest.py is
kept. Writes a JSON summary: counts and every non-passing test with its reason.
"""

from __future__ import annotations

import argparse
import json
import shutil
import subprocess
import sys
import tempfile
import xml.etree.ElementTree as ET
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_DIR = REPO / "baseline" / "_ref"
STAGED = REPO / "baseline" / "_ref_tests"
SOURCE = Path("/root/reference/pkg/tests")


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--pytest-args", default="-q")
    a = ap.parse_args()
    if a.stage:
        if STAGED.exists():
            shutil.rmtree(STAGED)
        shutil.copytree(SOURCE, STAGED, ignore=shutil.ignore_patterns("__pycache__"))
        print(f"staged {len(list(STAGED.glob('test_*.py')))} test files into {STAGED}")
        return 0
    tests = SOURCE if SOURCE.exists() else STAGED
    if not (REF_DIR / "rdist").exists() or not tests.exists():
        print("reference package or tests missing (run --stage and the baseline/_ref install)", file=sys.stderr)
        return 2
    with tempfile.TemporaryDirectory() as tmp:
        root = Path(tmp)
        shutil.copytree(tests, root / "tests", ignore=shutil.ignore_patterns("__pycache__"))
        (root / "conftest.py").write_text(
            "import sys\n"
            f"sys.path.insert(0, {str(HERE)!r})\n"
            "import dropin\n"
            f"dropin.install({str(REF_DIR)!r})\n")
        xml = root / "junit.xml"
        cmd = [sys.executable, "-m", "pytest", str(root / "tests"), "--rootdir", str(root), "-p", "no:cacheprovider",
               f"--junitxml={xml}", *a.pytest_args.split()]
        proc = subprocess.run(cmd, cwd=root, capture_output=True, text=True)
        print(proc.stdout[-3000:])
        print(proc.stderr[-2000:], file=sys.stderr)
        summary = {"command": "pytest <reference tests> with rdist.{linalg,resolvent,navigation} -> paper_2308_07403_b200",
                   "returncode": proc.returncode, "tests_source": str(tests)}
        if xml.exists():
            suite = ET.parse(xml).getroot()
            cases = suite.iter("testcase")
            failing = []
            counts = {"passed": 0, "failed": 0, "error": 0, "skipped": 0}
            for c in cases:
                tid = f"{c.get('classname')}::{c.get('name')}"
                kids = {k.tag: k for k in c}
                if "failure" in kids or "error" in kids:
                    tag = "failure" if "failure" in kids else "error"
                    counts["failed" if tag == "failure" else "error"] += 1
                    failing.append({"test": tid, "kind": tag, "message": (kids[tag].get("message") or "")[:300]})
                elif "skipped" in kids:
                    counts["skipped"] += 1
                else:
                    counts["passed"] += 1
            summary.update(counts=counts, total=sum(counts.values()), not_passing=failing)
        if a.out:
            Path(a.out).write_text(json.dumps(summary, indent=1) + "\n")
        print(json.dumps({k: summary.get(k) for k in ("counts", "total", "returncode")}))
        return 0 if proc.returncode == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
