"""Does a concurrent device->host / host->device DMA stream slow the config-2
pipeline?  The captured step is replayed alone, beside a D2H copy loop of an
unrelated 268 MB buffer (the e2e engine's uint8 D per step), beside an H2D loop
of 33 MB (its bits), and beside both.  usage: python tools/dma_contention.py"""
import json
import sys
import threading
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device("cuda", 0)
buf = B.BatchBuffers.allocate(1024, 256, dev, d_dtype="uint8")
buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
buf.gammas.copy_(torch.from_numpy(gammas))
pipe = B.CapturedPipeline(buf, 256)
d_src = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
d_host = torch.empty(256 * 1024 * 1024, dtype=torch.uint8).pin_memory()
h_src = torch.empty(33 * 1024 * 1024, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(33 * 1024 * 1024, dtype=torch.uint8, device=dev)
s_d2h, s_h2d = torch.cuda.Stream(), torch.cuda.Stream()


def run(d2h, h2d, steps=40):
    stop = threading.Event()

    def pump():
        while not stop.is_set():
            if d2h:
                with torch.cuda.stream(s_d2h):
                    d_host.copy_(d_src, non_blocking=True)
            if h2d:
                with torch.cuda.stream(s_h2d):
                    h_dst.copy_(h_src, non_blocking=True)
            s_d2h.synchronize()
            s_h2d.synchronize()

    th = threading.Thread(target=pump)
    if d2h or h2d:
        th.start()
    for _ in range(5):
        pipe.replay()
    torch.cuda.current_stream().synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pipe.replay()
    e1.record()
    e1.synchronize()
    stop.set()
    if d2h or h2d:
        th.join()
    return e0.elapsed_time(e1) / steps


out = {}
for name, a, b in (("alone", 0, 0), ("with_d2h", 1, 0), ("with_h2d", 0, 1), ("with_both", 1, 1), ("alone_again", 0, 0)):
    out[name] = run(a, b)
print(json.dumps(out))
