"""Experiment: config-2 batch as two half-batches on two streams (their kernels
fill each other's tails) vs one 256-graph call."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2308_07403_b200 as rb  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

rb.load_library()
bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device("cuda", 0)


def make(lo, hi):
    buf = B.BatchBuffers.allocate(1024, hi - lo, dev, d_dtype="uint8")
    buf.bits.copy_(torch.from_numpy(bits[lo:hi].view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas[lo:hi]))
    return buf


full = make(0, 256)
halves = [make(0, 128), make(128, 256)]
quarters = [make(64 * i, 64 * (i + 1)) for i in range(4)]
streams = [torch.cuda.Stream() for _ in range(4)]


def one():
    B.run_chunk(full, 256, torch.cuda.current_stream().cuda_stream)


def split(bufs, k):
    cur = torch.cuda.current_stream()
    for i, b in enumerate(bufs):
        streams[i].wait_stream(cur)
        B.run_chunk(b, b.chunk, streams[i].cuda_stream)
    for i in range(len(bufs)):
        cur.wait_stream(streams[i])


for name, fn in (("one 256", one), ("2 x 128 on 2 streams", lambda: split(halves, 2)),
                 ("4 x 64 on 4 streams", lambda: split(quarters, 4)), ("one 256 again", one)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(5):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    t = e[0].elapsed_time(e[1]) / 5
    print(f"{name}: {t:.3f} ms per 256 graphs, {256 / t * 1e3:.0f} graphs/s", flush=True)
