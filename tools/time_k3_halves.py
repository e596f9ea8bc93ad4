"""K3 (uint8 / int32 D) on the ER half and on the lattice half of the config-2
batch separately (the lattices hold exact zeros — unreachable pairs — that
take the kernel's rare path).  usage: python tools/time_k3_halves.py [lib.so]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

if len(sys.argv) > 1:
    L._lib = L.load_library(sys.argv[1])
bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device("cuda", 0)
sh = torch.cuda.current_stream().cuda_stream
for dt in ("uint8", "int32"):
    out = {"d_dtype": dt}
    for name, sl in (("er", slice(0, 128)), ("lattice", slice(128, 256))):
        buf = B.BatchBuffers.allocate(1024, 128, dev, d_dtype=dt)
        buf.bits.copy_(torch.from_numpy(bits[sl].view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gammas[sl]))
        B.run_chunk(buf, 128, sh)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(20):
            buf.stage_log_ceil(128, sh)
        ev[1].record()
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) / 20
        byt = 128 * 1024 * 1024 * (8 + buf.d.element_size())
        y = buf.m
        out[name] = {"ms": t, "GBps": byt / t / 1e6, "zeros_frac": float((y[:, :1024, :1024] == 0).double().mean())}
        del buf
    print(json.dumps(out), flush=True)
