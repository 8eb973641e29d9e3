"""cuBLAS GEMM throughput through torch (context: TF32 / BF16 / FP32 / FP64)."""
import torch
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
for name, dt, tf32 in (("bf16", torch.bfloat16, False), ("tf32", torch.float32, True), ("fp32", torch.float32, False),
                       ("fp64", torch.float64, False)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(2): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if dt != torch.float64 else 3
    e0.record()
    for _ in range(reps): a @ b
    e1.record(); torch.cuda.synchronize()
    print(f"{name} GEMM {n}^3: {2 * n**3 * reps / (e0.elapsed_time(e1) * 1e9):8.1f} TFLOP/s")
