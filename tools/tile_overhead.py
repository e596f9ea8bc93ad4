"""Per-tile overhead of the persistent DMMA engine: time rdb_gemm_local
(C += -A B, reduce-add epilogue, and C = A B, store epilogue) at fixed M = N
for several K, and fit t = tiles/SMs * (a + b * K/16).

usage: python tools/tile_overhead.py [lib.so ...]
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    libs = sys.argv[1:] or [None]
    m = n = 148 * 128 // 4 * 4  # 4736: 37 x 37 tiles ~ 9.25 rounds
    m = n = 128 * 74  # 74 x 74 = 5476 tiles = 37 rounds of 148
    ks = [64, 128, 256, 512, 1024]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for path in libs:
        if path:
            L._lib = L.load_library(path)
        else:
            L.load_library()
        sh = torch.cuda.current_stream().cuda_stream
        res = {}
        for acc in (1, 0):
            rows = []
            for k in ks:
                a = torch.randn((m, k), dtype=torch.float64, device=dev)
                b = torch.randn((k, n), dtype=torch.float64, device=dev)
                c = torch.zeros((m, n), dtype=torch.float64, device=dev)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ts = []
                for _ in range(4):
                    ev[0].record()
                    L.check(L.lib().rdb_gemm_local(a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, m, n, k, -1, -1,
                                                   -1, acc, 1, sh), "gemm")
                    ev[1].record()
                    torch.cuda.synchronize()
                    ts.append(ev[0].elapsed_time(ev[1]))
                t = float(np.median(ts[1:]))
                rounds = (m // 128) * (n // 128) / sms
                rows.append({"k": k, "ms": t, "us_per_tile_round": t * 1e3 / rounds,
                             "tflops": 2 * m * n * k / t / 1e9})
            kk = np.array([r["k"] / 16 for r in rows])
            yy = np.array([r["us_per_tile_round"] for r in rows])
            slope, icpt = np.polyfit(kk, yy, 1)
            res["reduce" if acc else "store"] = {"rows": rows, "us_per_chunk": slope, "us_overhead_per_tile": icpt,
                                                 "ideal_us_per_chunk": 2 * 128 * 128 * 16 / (37.0e12 / sms) * 1e6}
        print(json.dumps({"lib": path, **res}), flush=True)


if __name__ == "__main__":
    main()
