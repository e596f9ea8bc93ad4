"""APSP pipeline calls (rdb_apsp_bits_batched_d8) on a cfg2 slice, for ncu
launch lists: python tools/pipe_prof.py [lattice|er|mixed] [reps]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "lattice"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
bits, gammas, _ = wl.cfg2_batch(256)
sl = {"lattice": slice(128, 256), "er": slice(0, 128), "mixed": slice(0, 256)}[which]
bits, gammas = bits[sl], gammas[sl]
cnt = bits.shape[0]
buf = B.BatchBuffers.allocate(1024, cnt, torch.device("cuda"), d_dtype="uint8")
buf.bits.copy_(torch.from_numpy(np.ascontiguousarray(bits).view(np.int32)))
buf.gammas.copy_(torch.from_numpy(gammas))
sh = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for r in range(reps):
    buf.counters.zero_()
    ev[0].record()
    B.run_chunk(buf, cnt, sh)
    ev[1].record()
    torch.cuda.synchronize()
    print(which, "pipeline ms", ev[0].elapsed_time(ev[1]))
