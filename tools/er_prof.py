"""One K2 call on the 128 ER graphs of config 2, for ncu captures:
python tools/er_prof.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

bits, gammas, _ = wl.cfg2_batch(256)
bits, gammas = bits[:128], gammas[:128]
buf = B.BatchBuffers.allocate(1024, 128, torch.device("cuda"))
buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
buf.gammas.copy_(torch.from_numpy(gammas))
sh = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    buf.stage_build(128, sh)
    buf.stage_invert(128, sh)
torch.cuda.synchronize()
