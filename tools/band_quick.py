import os, sys, json, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
from paper_2308_07403_b200 import batch as B, workloads as wl, _lib as L
bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device('cuda')
res = {}
for mode in ('0', '1'):
    os.environ['RDB_GJ_BAND'] = mode
    buf = B.BatchBuffers.allocate(1024, 256, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32))); buf.gammas.copy_(torch.from_numpy(gammas))
    sh = torch.cuda.current_stream().cuda_stream
    buf.stage_build(256, sh); buf.stage_invert(256, sh); torch.cuda.synchronize()
    res[mode] = buf.m.cpu().numpy()
    info = L.read_pivot_info(buf.info)
    print(mode, [ (i.min_pivot, i.min_index, i.flags) for i in info[126:130]])
    del buf
a, b = res['0'], res['1']
for g in (0, 127, 128, 129, 255):
    nz = a[g] != 0
    print(g, np.array_equal(a[g] == 0, b[g] == 0), np.max(np.abs(b[g][nz] - a[g][nz]) / np.abs(a[g][nz])), np.isnan(b[g]).sum())
