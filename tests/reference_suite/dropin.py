"""Drop-in harness for the reference's own test suite (TEST INFRASTRUCTURE).

``install(ref_dir)`` makes ``import rdist`` resolve to the unmodified
reference package (installed into baseline/_ref by
``pip install --no-deps --target baseline/_ref /root/reference/pkg``) with its
hot-path modules — ``rdist.linalg``, ``rdist.resolvent``, ``rdist.navigation``
 — replaced by this repository's, exactly as a user switching
to the B200 path would: the reference's graph constructors, oracles, analog
network and experiment harness then call this package's CUDA kernels through
the reference's own import statements (rdist/__init__.py,
rdist/experiments.py:23-43, rdist/analog.py:18-19).
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[2]
HOT_PATH = ("linalg", "resolvent", "navigation")


def install(ref_dir: str | Path) -> None:
    sys.path.insert(0, str(REPO))
    if "rdist" in sys.modules:
        raise RuntimeError("rdist imported before the drop-in was installed")
    for name in HOT_PATH:
        sys.modules[f"rdist.{name}"] = importlib.import_module(f"paper_2308_07403_b200.{name}")
    sys.path.insert(0, str(ref_dir))
    rdist = importlib.import_module("rdist")
    mine = importlib.import_module("paper_2308_07403_b200.resolvent")
    assert rdist.resolvent is mine.resolvent and rdist.lu_invert.__module__ == "paper_2308_07403_b200.linalg"
    assert Path(rdist.__file__).resolve().is_relative_to(Path(ref_dir).resolve())
