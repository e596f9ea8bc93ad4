"""cuBLAS DGEMM throughput probe (torch.matmul fp64) — a sanity comparator for the FP64 peak."""
import json, torch
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res[f"dgemm_{n}_tflops"] = 2 * n**3 / (ms * 1e-3) / 1e12
x = torch.tensor([0.3 * 0.3, 0.3, 0.1], dtype=torch.float64, device="cuda")
res["torch_log_ratio_0p09"] = float((torch.log(x[0:1]) / torch.log(x[1:2])).item())
res["gpu"] = torch.cuda.get_device_name()
print(json.dumps(res))
