"""cuBLAS DGEMM (torch float64 matmul) peak on the box, for the FP64 roofline denominator."""
import json, torch, time
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{n}_tflops_burst"] = 2 * n**3 / best / 1e9
    e0.record(); t = time.time(); k = 0
    while time.time() - t < 3:
        for _ in range(5):
            a @ b
        k += 5
        torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    res[f"dgemm_{n}_tflops_sustained"] = 2 * n**3 * k / e0.elapsed_time(e1) / 1e9
print(json.dumps(res))
