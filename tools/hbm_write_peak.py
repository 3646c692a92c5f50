"""Write-only and copy HBM bandwidth on this GPU (K1 is a write stream: its roofline is the
write bandwidth, reported beside the copy figure of MEASURED_PEAKS.json).

  python tools/hbm_write_peak.py [--gib 4] [--json out.json]
"""
import argparse
import json

import torch


def best_ms(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=4.0)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    n = int(a.gib * 2**30) // 8
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    out = {"bytes": 8 * n, "device": torch.cuda.get_device_name(0)}
    out["write_fill_GBps"] = 8 * n / best_ms(lambda: x.fill_(1.0)) / 1e6
    out["write_zero_GBps"] = 8 * n / best_ms(lambda: x.zero_()) / 1e6
    out["copy_rw_GBps"] = 16 * n / best_ms(lambda: y.copy_(x)) / 1e6
    print(json.dumps(out))
    if a.json:
        json.dump(out, open(a.json, "w"))
