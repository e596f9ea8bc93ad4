"""A/B timing of K3 (cfg2 batch, uint8 and int32 D) for library variants.
usage: python tools/time_k3.py lib_a.so [lib_b.so ...]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device("cuda", 0)
first = {}
for path in sys.argv[1:]:
    L._lib = L.load_library(path)
    res = {"lib": path}
    for dt in ("uint8", "int32"):
        buf = B.BatchBuffers.allocate(1024, 256, dev, d_dtype=dt)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gammas))
        sh = torch.cuda.current_stream().cuda_stream
        B.run_chunk(buf, 256, sh)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(10):
            buf.stage_log_ceil(256, sh)
        ev[1].record()
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) / 10
        byt = 256 * 1024 * 1024 * (8 + buf.d.element_size())
        d = buf.d.cpu()
        first.setdefault(dt, d)
        res[dt] = {"ms": t, "GBps": byt / t / 1e6, "same_d_as_first_lib": bool(torch.equal(d, first[dt]))}
        del buf
    print(json.dumps(res), flush=True)
