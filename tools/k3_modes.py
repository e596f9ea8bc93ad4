"""A/B timing of K3 on the config-2 batch (256 inverses already in HBM), uint8
and int32 D, for the default library and variant libraries (--libs); outputs
must be identical. Used to measure a TMA-streamed K3 (warp-private rings of row
buffers filled by cp.async.bulk; profiles/r02_k3_stream_variants.json): no
variant beat the register-pipelined lean kernel, which is issue-bound
(45 instructions per element at 72% issue utilisation, ncu), so it was not kept.

usage: python tools/k3_modes.py [--out gpurun_out/k3_modes.json]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--libs", default="", help="comma-separated variant libraries (stream mode only)")
    a = ap.parse_args()
    L.load_library()
    variants = [x for x in a.libs.split(",") if x]
    dev = torch.device("cuda", 0)
    bits, gammas, _ = wl.cfg2_batch(256)
    peak = float(json.loads(Path("MEASURED_PEAKS.json").read_text())["hbm_gbs"]) if Path("MEASURED_PEAKS.json").exists() else 6548.8
    out = []
    for dt in ("uint8", "int32"):
        buf = B.BatchBuffers.allocate(1024, 256, dev, d_dtype=dt)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gammas))
        sh = torch.cuda.current_stream().cuda_stream
        B.run_chunk(buf, 256, sh)
        torch.cuda.synchronize()
        ref = None
        for mode in ["default"] + variants:
            if mode != "default":
                L._lib = L.load_library(mode)
            buf.counters.zero_()
            buf.stage_log_ceil(256, sh)
            torch.cuda.synchronize()
            d = buf.d.clone()
            cnt = buf.counters.clone()
            if ref is None:
                ref = (d, cnt)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(a.reps):
                buf.stage_log_ceil(256, sh)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1]) / a.reps
            nbytes = 256 * (8 * 1024 * 1024 + (1 if dt == "uint8" else 4) * 1024 * 1024)
            rec = {"d_dtype": dt, "lib": mode, "ms": ms, "GBps": nbytes / ms / 1e6,
                   "frac_of_hbm": nbytes / ms / 1e6 / peak, "d_identical": bool(torch.equal(d, ref[0])),
                   "counters_identical": bool(torch.equal(cnt, ref[1]))}
            print(json.dumps(rec), flush=True)
            out.append(rec)
        if variants:
            L._lib = L.load_library()
        del buf
        torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
