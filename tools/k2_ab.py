"""A/B of two builds of the library on the config-2 batch: K2 and step time,
SHA-256 of the inverse batch Y and of D (bitwise comparison across builds).

usage: python tools/k2_ab.py libA.so [libB.so ...] [--reps 9]
Each library runs in its own subprocess (one library per process).
"""

import argparse
import hashlib
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child(lib, reps):
    import numpy as np
    import torch

    sys.path.insert(0, str(ROOT))
    from paper_2308_07403_b200 import _lib as L
    from paper_2308_07403_b200 import batch as B
    from paper_2308_07403_b200 import workloads as wl

    L._lib = L.load_library(lib)
    dev = torch.device("cuda", 0)
    bits, gammas, _ = wl.cfg2_batch(256)
    buf = B.BatchBuffers.allocate(1024, 256, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas))
    sh = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        B.run_chunk(buf, 256, sh)
    torch.cuda.synchronize()
    hd = hashlib.sha256(buf.d.cpu().numpy().tobytes()).hexdigest()[:16]
    hyp = hashlib.sha256(buf.m.cpu().numpy().tobytes()).hexdigest()[:16]  # Y of the pipeline call (M from bits)
    buf.stage_build(256, sh)
    buf.stage_invert(256, sh)
    torch.cuda.synchronize()
    hy = hashlib.sha256(buf.m.cpu().numpy().tobytes()).hexdigest()[:16]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ts, tstep = [], []
    for _ in range(reps):
        buf.stage_build(256, sh)
        ev[0].record()
        buf.stage_invert(256, sh)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
        ev[2].record()
        B.run_chunk(buf, 256, sh)
        ev[3].record()
        torch.cuda.synchronize()
        tstep.append(ev[2].elapsed_time(ev[3]))
    print(json.dumps({"lib": lib, "k2_ms_median": float(np.median(ts)), "k2_ms_min": float(np.min(ts)),
                      "step_ms_median": float(np.median(tstep)), "sha_y": hy, "sha_y_pipeline": hyp, "sha_d": hd}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.libs[0], a.reps)
        return
    for lib in a.libs:
        subprocess.run([sys.executable, __file__, lib, "--reps", str(a.reps), "--child"], check=False)


if __name__ == "__main__":
    main()
