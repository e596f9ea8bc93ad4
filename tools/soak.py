"""Soak of the config-2 step: N replays of the captured pipeline (and every 7th
one eager), D hashed on the device after each; any differing hash or a stall
past the deadline ends the run.  usage: python tools/soak.py [replays]"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

n_rep = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device("cuda", 0)
buf = B.BatchBuffers.allocate(1024, 256, dev, d_dtype="uint8")
buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
buf.gammas.copy_(torch.from_numpy(gammas))
sh = torch.cuda.current_stream().cuda_stream
B.run_chunk(buf, 256, sh)
torch.cuda.synchronize()
w = torch.arange(1, 1 + buf.d.numel() // 8, device=dev, dtype=torch.int64)


def digest():
    return int((buf.d.view(-1).view(torch.int64) * w).sum().item())


ref = digest()
pipe = B.CapturedPipeline(buf, 256)
t0 = time.time()
bad = 0
for it in range(n_rep):
    buf.d.fill_(0)
    if it % 7 == 6:
        B.run_chunk(buf, 256, sh)
    else:
        pipe.replay()
    ev = torch.cuda.Event()
    ev.record()
    t1 = time.monotonic()
    while not ev.query():
        if time.monotonic() - t1 > 60:
            print(json.dumps({"stalled_at": it}), flush=True)
            os._exit(3)
        time.sleep(0.0005)
    if digest() != ref:
        bad += 1
        print(json.dumps({"differs_at": it}), flush=True)
print(json.dumps({"replays": n_rep, "differing": bad, "seconds": time.time() - t0}))
