import time, torch, numpy as np
x = torch.empty(570_000_000 // 8, dtype=torch.float64).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); t1=time.perf_counter()-t
    t=time.perf_counter(); x.copy_(y, non_blocking=True); torch.cuda.synchronize(); t2=time.perf_counter()-t
    print(f"H2D {t1*1e3:.1f} ms ({570/t1/1e3:.1f} GB/s)  D2H {t2*1e3:.1f} ms ({570/t2/1e3:.1f} GB/s)")
