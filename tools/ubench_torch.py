"""Library ceilings on this B200: cuBLAS DGEMM/ZGEMM/SGEMM/CGEMM and int8 GEMM."""
import time, torch
torch.backends.cuda.matmul.allow_tf32 = False
def bench(fn, flops, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return flops / best / 1e9, best
for n in (2048, 4096, 8192):
    for dt, mult in ((torch.float64, 2), (torch.complex128, 8), (torch.float32, 2), (torch.complex64, 8)):
        a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
        tf, ms = bench(lambda: a @ b, mult * n**3)
        print(f"n={n} {dt}: {tf:.2f} TFLOP/s ({ms:.2f} ms)", flush=True)
    a = torch.randint(-127, 127, (n, n), device="cuda", dtype=torch.int8)
    b = torch.randint(-127, 127, (n, n), device="cuda", dtype=torch.int8).t().contiguous().t()
    try:
        tf, ms = bench(lambda: torch._int_mm(a, b), 2 * n**3)
        print(f"n={n} int8 _int_mm: {tf:.1f} TOP/s ({ms:.2f} ms)", flush=True)
    except Exception as ex:
        print("int8 failed", ex)
    a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16); b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    tf, ms = bench(lambda: a @ b, 2 * n**3)
    print(f"n={n} bf16: {tf:.1f} TFLOP/s", flush=True)
# sustained DGEMM 4 s
n = 8192
a = torch.randn(n, n, device="cuda", dtype=torch.float64); b = torch.randn(n, n, device="cuda", dtype=torch.float64)
torch.cuda.synchronize(); t0 = time.time(); cnt = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"sustained DGEMM 8192: {2*n**3*cnt/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s over {cnt} runs")
