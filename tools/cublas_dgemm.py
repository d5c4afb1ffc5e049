"""cuBLAS DGEMM reference throughput on this GPU (torch float64 matmul) for the solver's shapes."""
import torch
import time
torch.backends.cuda.matmul.allow_tf32 = False
for (m, n, k) in ((2000, 2000, 2000), (1000, 2000, 2000), (2000, 1000, 2000), (4096, 4096, 4096), (8192, 8192, 8192)):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM {m}x{n}x{k}: {ms:.3f} ms  {2*m*n*k/ms/1e9:.2f} TF/s")
