"""Config 5 across GPUs: the N = 32768 inversion on a P_r x P_c grid of ranks.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
      --master-port 29511 tools/dist_invert.py --grid 2x4

Each rank builds the config-5 matrix M = I - gamma*A (the reference's
gen_random_dense(32768, 0.01, 0) pattern, bit-packed) on its GPU, keeps only
its block-cyclic tiles, runs the distributed Gauss-Jordan
(paper_2308_07403_b200.distributed over NCCL), and reports the FP64 TFLOP/s
(2 n^3 / max-over-ranks device time) as one JSON line on rank 0. With
--check, D on 256 sampled source columns is compared with BFS.
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import distributed as D  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default=None, help="PrxPc (default: 1xWORLD)")
    ap.add_argument("--n", type=int, default=wl.CFG5["n"])
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    pr, pc = (1, world) if a.grid is None else (int(x) for x in a.grid.lower().split("x"))
    lay = D.Layout(a.n, pr, pc)
    n, gamma = a.n, wl.CFG5["gamma"]
    bits = torch.from_numpy(wl.er_bits_chunked(n, wl.CFG5["p"], 0, chunk_rows=2048).view(np.int32)).to(dev)
    full = torch.empty((n, n), dtype=torch.float64, device=dev)
    L.load_library()
    L.check(L.lib().rdb_build_m_bits(bits.data_ptr(), n, n, 1, None, gamma, full.data_ptr(), n, n * n,
                                     L.stream_handle()), "build")
    grid = D.TorchGrid(lay)
    base = D.scatter(full, lay, *grid.me)
    del full
    torch.cuda.empty_cache()
    times = []
    for _ in range(a.reps):
        loc = base.clone()
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        minp, flags = D.invert_block_cyclic({grid.me: loc}, grid, D.CudaEngine())
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
    if rank == 0:
        ms = min(times)
        tf = 2.0 * n**3 / (ms * 1e-3) / 1e12
        print(json.dumps({"config": "cfg5", "n": n, "grid": f"{pr}x{pc}", "n_gpus": world, "ms": ms,
                          "inversion_tflops": tf, "per_gpu_tflops": tf / world, "min_pivot": minp,
                          "pivot_flags": flags}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
