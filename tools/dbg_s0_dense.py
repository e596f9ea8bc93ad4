import os, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L, batch as B, workloads as wl
if len(sys.argv) > 1 and sys.argv[1] != "-":
    L._lib = L.load_library(sys.argv[1])
n, p, count = 1024, 0.02, 12
rng = np.random.default_rng(n)
presents = []
for k in range(count):
    q = rng.random((n, n)) < p
    if k == 5:
        q[n - 7, :200] = True
    np.fill_diagonal(q, False)
    presents.append(q)
bits = np.stack([wl.pack_bits(q) for q in presents])
gam = np.full(count, 1e-2)
dev = torch.device("cuda")
sh = torch.cuda.current_stream().cuda_stream
res = {}
for mode in ("default", "dense"):
    os.environ.pop("RDB_GJ_DW_S0", None)
    if mode == "dense":
        os.environ["RDB_GJ_DW_S0"] = "0"
    buf = B.BatchBuffers.allocate(n, count, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gam))
    buf.stage_build(count, sh)
    buf.stage_invert(count, sh)
    torch.cuda.synchronize()
    y = buf.m.clone()
    for poison in (None, float("nan"), 0.0):
        if poison is not None:
            buf.m.fill_(poison)
        B.run_chunk(buf, count, sh)
        torch.cuda.synchronize()
        yp, d = buf.m.clone(), buf.d.clone()
        buf.stage_log_ceil(count, sh)
        torch.cuda.synchronize()
        print("   K3 alone on the final Y == pipeline D:", bool(torch.equal(buf.d, d)), "| env", os.environ.get("RDB_GJ_DW_S0"))
        bad = [b for b in range(count) if not torch.equal(y[b], yp[b])]
        rel = ((y - yp).abs() / y.abs().clamp_min(1e-300)).max().item()
        print(mode, "poison", poison, "graphs whose pipeline Y != generic Y (bitwise):", bad, "max rel", rel)
        res[(mode, poison)] = d
    del buf
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import rdist_oracle as orc
ref0 = orc.d_to_int32(orc.run_rdist(wl.weights_from_present(presents[0]), 1e-2))
for k, v in res.items():
    print(k, "graph 0 D == oracle:", bool(np.array_equal(v[0].cpu().numpy(), ref0)))
ks = list(res)
for k in ks[1:]:
    eq = bool(torch.equal(res[k], res[ks[0]]))
    print(k, "D equal to first:", eq)
    if not eq:
        dd = res[k] != res[ks[0]]
        idx = dd.nonzero()
        print("   differing:", int(dd.sum()), "graphs", sorted(set(idx[:, 0].tolist())), "rows", int(idx[:, 1].min()), int(idx[:, 1].max()),
              "cols", int(idx[:, 2].min()), int(idx[:, 2].max()), "values", res[k][dd][:8].tolist(), "vs", res[ks[0]][dd][:8].tolist())
