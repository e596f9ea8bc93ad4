import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2308_07403_b200 import _lib as L, workloads as wl
L.load_library(); dev = torch.device('cuda', 0)
for n in (1024, 1536, 2048, 3072, 4096):
    bits = torch.from_numpy(wl.er_bits_chunked(n, 0.01, 0, chunk_rows=2048).view(np.int32)).to(dev)
    m0 = torch.empty((n, n), dtype=torch.float64, device=dev)
    L.check(L.lib().rdb_build_m_bits(bits.data_ptr(), n, n, 1, None, 1e-4, m0.data_ptr(), n, n * n, L.stream_handle()), 'b')
    res = {}
    for mode, env, la in (("narrow", "0", "1"), ("wide", "256", "1"), ("wide_nola", "256", "0")):
        os.environ["RDB_GJ_WIDE_MIN"] = env; os.environ["RDB_GJ_WIDE_LA"] = la
        work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=dev)
        info = L.pivot_info_tensor(1, dev)
        m = m0.clone()
        L.check(L.lib().rdb_invert(m.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), L.stream_handle()), 'i')
        torch.cuda.synchronize(); res[mode] = m
    a = res["narrow"]
    print(n, {k: float(((v - a).abs() / a.abs().clamp_min(1e-300)).max()) for k, v in res.items() if k != "narrow"}, flush=True)
