"""Where the e2e engine's step time goes: device time of every pipeline call on
the compute stream (CUDA events) and the gaps between consecutive calls, beside
the wall-clock step.  usage: python tools/e2e_probe.py [steps] [chunk]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 48
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 256
bits, gammas, _ = wl.cfg2_batch(256)
eng = B.APSPBatchEngine(1024, 256, chunk=chunk, d_dtype="uint8")
bp, gp = eng.pin(bits, gammas)
marks = []
orig = eng._pipeline


def timed(*a):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.cs)
    orig(*a)
    e1.record(eng.cs)
    marks.append((e0, e1))


def stream(k):
    for s in range(k):
        if s >= 2:
            eng.wait(s % 2, gp, check=False)
        eng.submit(bp, gp, s % 2)
    for s in range(max(0, k - 2), k):
        eng.wait(s % 2, gp, check=False)


stream(8)
eng._pipeline = timed
torch.cuda.synchronize()
t0 = time.perf_counter()
stream(steps)
dt = (time.perf_counter() - t0) / steps
torch.cuda.synchronize()
dur = [a.elapsed_time(b) for a, b in marks]
gap = [marks[i][1].elapsed_time(marks[i + 1][0]) for i in range(len(marks) - 1)]
span = marks[0][0].elapsed_time(marks[-1][1])
print(json.dumps({"steps": steps, "chunk": chunk, "wall_ms_per_step": dt * 1e3, "calls": len(marks),
                  "call_ms_median": float(np.median(dur)), "call_ms_min": min(dur), "call_ms_max": max(dur),
                  "gap_ms_median": float(np.median(gap)), "gap_ms_max": max(gap),
                  "compute_span_ms_per_step": span / steps}))
