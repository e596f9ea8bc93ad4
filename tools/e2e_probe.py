import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2308_07403_b200 as rb
from paper_2308_07403_b200 import batch as B, workloads as wl
rb.load_library()
bits, gammas, _ = wl.cfg2_batch(256)
dev = torch.device('cuda', 0)
for chunk in (128, 256):
    # device-only: same chunking, no copies
    buf = B.BatchBuffers.allocate(1024, chunk, dev, d_dtype='uint8')
    buf.bits.copy_(torch.from_numpy(bits[:chunk].view(np.int32))); buf.gammas.copy_(torch.from_numpy(gammas[:chunk]))
    sh = torch.cuda.current_stream().cuda_stream
    for _ in range(3): B.run_chunk(buf, chunk, sh)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(5 * (256 // chunk)): B.run_chunk(buf, chunk, sh)
    e[1].record(); torch.cuda.synchronize()
    dev_ms = e[0].elapsed_time(e[1]) / 5
    del buf; torch.cuda.empty_cache()
    eng = B.APSPBatchEngine(1024, 256, chunk=chunk, d_dtype='uint8')
    bp, gp = eng.pin(bits, gammas)
    for _ in range(3): eng.run(bp, gp)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    steps = 6
    for s in range(steps):
        if s >= 2: eng.wait(s % 2, gp, check=False)
        eng.submit(bp, gp, s % 2)
    for s in range(steps - 2, steps): eng.wait(s % 2, gp, check=False)
    e2e_ms = (time.perf_counter() - t0) / steps * 1e3
    # host submit cost
    t0 = time.perf_counter(); eng.submit(bp, gp, 0); t_sub = (time.perf_counter() - t0) * 1e3; eng.wait(0, gp, check=False)
    print(f"chunk {chunk}: device-only {dev_ms:.2f} ms/256, e2e {e2e_ms:.2f} ms/256, host submit {t_sub:.2f} ms")
    del eng; torch.cuda.empty_cache()
