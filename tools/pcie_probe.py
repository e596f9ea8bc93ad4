import torch, time
x = torch.empty(1<<28, dtype=torch.int32, device="cuda"); h = torch.empty(1<<28, dtype=torch.int32).pin_memory()
for _ in range(3): h.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): h.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print("D2H GB/s", 4*(1<<28)/dt/1e9)
b = torch.empty(1<<28, dtype=torch.int32).pin_memory()
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): x.copy_(b, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print("H2D GB/s", 4*(1<<28)/dt/1e9)
