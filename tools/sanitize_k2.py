"""Small K2 workloads for compute-sanitizer (racecheck / synccheck / memcheck):

  1. a 16-graph config-2 batch (8 ER + 8 lattices) through the bench pipeline
     (rdb_apsp_bits_batched_d8: K1, block-sparse plan, banded path, two
     sub-batch streams forced with RDB_GJ_SPLIT_MIN=8, ticketed update tiles);
  2. one N = 2048 matrix through the single-matrix look-ahead path;
  3. one N = 2048 matrix through the wide 256-step path (RDB_GJ_WIDE_MIN=2048);
each checked against the normal (unsanitised) expectations: D equal to the
int32 run, inverses within 1e-12 of each other.

usage: compute-sanitizer --tool racecheck python tools/sanitize_k2.py
"""

import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("RDB_GJ_SPLIT_MIN", "8")
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import single as S  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def main():
    L.load_library()
    dev = torch.device("cuda", 0)
    seeds = wl.cfg2_seeds(256)
    pick = seeds[:8] + seeds[128:136]
    bits = np.stack([wl.pack_bits(wl.cfg2_present(k, s)) for k, s in pick])
    gam = np.array([wl.cfg2_gamma(k) for k, _ in pick])
    outs = {}
    for dt in ("uint8", "int32"):
        buf = B.BatchBuffers.allocate(1024, len(pick), dev, d_dtype=dt)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gam))
        buf.counters.zero_()
        B.run_chunk(buf, len(pick))
        torch.cuda.synchronize()
        B.check_infos(L.read_pivot_info(buf.info), gam)
        outs[dt] = buf.d.cpu().numpy()
    assert np.array_equal(B.decode_d8(outs["uint8"]), outs["int32"])
    print("batch ok", flush=True)
    n = 2048
    b2 = torch.from_numpy(wl.er_bits_chunked(n, 0.01, 3).view(np.int32)).to(dev)
    m = S.build_m_bits(b2, n, 1e-3)
    S.invert_in_place(m, 1e-3)
    os.environ["RDB_GJ_WIDE_MIN"] = "2048"
    m2 = S.build_m_bits(b2, n, 1e-3)
    S.invert_in_place(m2, 1e-3)
    torch.cuda.synchronize()
    rel = ((m2 - m).abs() / m.abs().clamp_min(1e-300)).max().item()
    assert rel < 1e-12, rel
    print("single ok", rel, flush=True)


if __name__ == "__main__":
    main()
