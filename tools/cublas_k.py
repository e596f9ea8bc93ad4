"""cuBLAS DGEMM (C -= A B through torch.addmm, fp64) at K = 128 .. 1024 on the engine's problem shape: the comparator
behind profiles/r01_engine_vs_cublas.json."""
import torch, json
torch.backends.cuda.matmul.allow_tf32 = False
dev = 'cuda'
out = {}
for k in (128, 256, 512, 1024):
    m = n = 9472
    a = torch.randn(m, k, dtype=torch.float64, device=dev); b = torch.randn(k, n, dtype=torch.float64, device=dev)
    c = torch.randn(m, n, dtype=torch.float64, device=dev)
    for _ in range(2): torch.addmm(c, a, b, beta=1.0, alpha=-1.0, out=c)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(5): torch.addmm(c, a, b, beta=1.0, alpha=-1.0, out=c)
    e[1].record(); torch.cuda.synchronize()
    t = e[0].elapsed_time(e[1]) / 5
    out[k] = round(2 * m * n * k / t / 1e9, 2)
print(json.dumps({"cublas_dgemm_addmm_tflops_by_k (M=N=9472)": out}))
