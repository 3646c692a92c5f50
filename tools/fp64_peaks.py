"""Measure FP64 peaks on the B200 (cuBLAS DGEMM via torch, burst + sustained) and HBM copy.

Run on the GPU box; writes one JSON line. Used to fill the FP64 denominator that
MEASURED_PEAKS.json lacks.
"""
import json, time, torch

def dgemm(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    burst = 2 * n**3 / best / 1e12
    # sustained: back to back for ~4 s
    t0 = time.time(); cnt = 0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(4):
            torch.matmul(a, b); cnt += 1
        torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sus = 2 * n**3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return burst, sus

def hbm(n=1 << 30):
    a = torch.empty(n // 8, dtype=torch.float64, device="cuda").fill_(1)
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); b.copy_(a); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return 2 * n / best / 1e9

if __name__ == "__main__":
    burst, sus = dgemm()
    print(json.dumps({"fp64_dgemm_tflops": round(burst, 2), "fp64_dgemm_tflops_sustained": round(sus, 2),
                      "hbm_copy_gbs": round(hbm(), 1), "gpu": torch.cuda.get_device_name()}))
