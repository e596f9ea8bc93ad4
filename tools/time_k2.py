"""A/B timing of K2 (batched cfg2 inversion + one large inversion) for engine
variants built with `make BUILD=build_x LIB=tools/_var/lib_x.so EXTRA=-D...`.

usage: python tools/time_k2.py tools/_var/lib_a.so [tools/_var/lib_b.so ...]
Prints one JSON line per library (ms per cfg2 K2 call, TFLOP/s, single-N ms).
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    bits, gammas, _ = wl.cfg2_batch(256)
    single_n = int(dict(a.split("=") for a in sys.argv[1:] if "=" in a).get("single", 16384))
    for path in [a for a in sys.argv[1:] if "=" not in a]:
        L._lib = L.load_library(path)
        buf = B.BatchBuffers.allocate(1024, 256, dev)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gammas))
        sh = torch.cuda.current_stream().cuda_stream
        B.run_chunk(buf, 256, sh)
        torch.cuda.synchronize()
        ref_d = buf.d.clone()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for _ in range(5):
            buf.stage_build(256, sh)
            ev[0].record()
            buf.stage_invert(256, sh)
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        t = float(np.median(ts))
        B.run_chunk(buf, 256, sh)
        torch.cuda.synchronize()
        same = bool(torch.equal(ref_d, buf.d))
        n = single_n
        gen = torch.Generator(device=dev).manual_seed(7)
        m0 = (torch.rand((n, n), generator=gen, device=dev) < 0.01).to(torch.float64).mul_(-1e-4)
        m0.diagonal().fill_(1.0)
        m1 = m0.clone()
        work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=dev)
        info = L.pivot_info_tensor(1, dev)
        st = []
        for _ in range(2):
            m1.copy_(m0)
            ev[0].record()
            L.check(L.lib().rdb_invert(m1.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), sh), "invert")
            ev[1].record()
            torch.cuda.synchronize()
            st.append(ev[0].elapsed_time(ev[1]))
        print(json.dumps({"lib": path, "k2_ms": t, "k2_all": ts, "k2_tflops": 2 * 1024**3 * 256 / t / 1e9,
                          "d_same_as_first_run": same, "single_n": n, "single_ms": min(st),
                          "single_tflops": 2 * n**3 / min(st) / 1e9}), flush=True)
        del buf, m0, m1, work
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
