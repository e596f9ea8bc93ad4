"""Would two config-2 steps in flight at once (two buffer sets, two caller
streams; the library's internal streams are shared) beat back-to-back steps on
one stream?  Eager launches and captured graphs.  usage: python tools/two_pipelines.py"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device("cuda", 0)
bufs = []
for _ in range(2):
    buf = B.BatchBuffers.allocate(1024, 256, dev, d_dtype="uint8")
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas))
    B.run_chunk(buf, 256)
    bufs.append(buf)
torch.cuda.synchronize()
ref = bufs[0].d.clone()
streams = [torch.cuda.Stream() for _ in range(2)]
pipes = []
for st, buf in zip(streams, bufs):
    with torch.cuda.stream(st):
        pipes.append(B.CapturedPipeline(buf, 256))
torch.cuda.synchronize()
steps = 40
out = {}


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def one_stream_graph():
    with torch.cuda.stream(streams[0]):
        for _ in range(steps):
            pipes[0].replay()


def two_streams_graph():
    for s in range(steps):
        with torch.cuda.stream(streams[s % 2]):
            pipes[s % 2].replay()


def two_streams_eager():
    for s in range(steps):
        with torch.cuda.stream(streams[s % 2]):
            B.run_chunk(bufs[s % 2], 256, streams[s % 2].cuda_stream)


for st in streams:
    st.wait_stream(torch.cuda.current_stream())
out["one_stream_graph_ms"] = timed(one_stream_graph)
out["two_streams_graph_ms"] = timed(two_streams_graph)
out["two_streams_eager_ms"] = timed(two_streams_eager)
out["one_stream_graph_again_ms"] = timed(one_stream_graph)
out["d_identical"] = bool(torch.equal(bufs[0].d, ref) and torch.equal(bufs[1].d, ref))
print(json.dumps(out))
