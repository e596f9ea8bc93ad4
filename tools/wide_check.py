"""Wide (NB=256) vs narrow (NB=128) single-matrix inversion: agreement and speed.
usage: python tools/wide_check.py [n ...]"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

L.load_library()
dev = torch.device("cuda", 0)
for n in [int(x) for x in sys.argv[1:]] or [4096, 8192]:
    bits = torch.from_numpy(wl.er_bits_chunked(n, 0.01, 0, chunk_rows=2048).view(np.int32)).to(dev)
    m0 = torch.empty((n, n), dtype=torch.float64, device=dev)
    L.check(L.lib().rdb_build_m_bits(bits.data_ptr(), n, n, 1, None, 1e-4, m0.data_ptr(), n, n * n,
                                     L.stream_handle()), "build")
    out = {}
    for mode, env in (("narrow", "0"), ("wide", "1024")):
        os.environ["RDB_GJ_WIDE_MIN"] = env
        work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=dev)
        info = L.pivot_info_tensor(1, dev)
        m = m0.clone()
        ts = []
        for rep in range(3):
            m.copy_(m0)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            L.check(L.lib().rdb_invert(m.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), L.stream_handle()),
                    "invert")
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        rec = L.read_pivot_info(info)[0]
        out[mode] = (m.clone(), min(ts), rec)
        del work
    a, b = out["narrow"][0], out["wide"][0]
    rel = float(((a - b).abs() / a.abs().clamp_min(1e-300)).max())
    res = {"n": n, "narrow_ms": out["narrow"][1], "wide_ms": out["wide"][1],
           "narrow_tflops": 2 * n**3 / out["narrow"][1] / 1e9, "wide_tflops": 2 * n**3 / out["wide"][1] / 1e9,
           "max_rel_diff": rel, "min_pivot": [out["narrow"][2].min_pivot, out["wide"][2].min_pivot],
           "flags": [out["narrow"][2].flags, out["wide"][2].flags],
           "min_index": [out["narrow"][2].min_index, out["wide"][2].min_index]}
    print(json.dumps(res), flush=True)
