"""Developer tool: cuBLAS ZGEMM on the config-2 shapes (for comparison / ncu)."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False
shapes = [(128, 294912, 64), (64, 294912, 128), (4096, 72, 4096), (72, 72, 262144)]
for (m, n, k) in shapes:
    a = torch.randn(m, k, dtype=torch.complex128, device="cuda")
    b = torch.randn(k, n, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"M={m} N={n} K={k}: {ms:.3f} ms  {8*m*n*k/ms/1e9:.1f} TF", flush=True)
