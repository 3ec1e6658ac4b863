"""Measure this box's B200 rates and write them as a HardwareProfile JSON in
the reference's load_profile format (proj/core/src/perf_model.cpp:31-50:
{"name","flops","bw_gpu","bw_h2d","bw_d2h","fast_capacity","notes"}), so the
reference's own cost model (decode_transfer_check, project_run, the CLI's
--profile) can project B200 runs.

    python tools/b200_profile.py [--out profiles/b200_profile.json]
"""
import argparse
import json
import os

import torch


def best_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "profiles", "b200_profile.json"))
    args = ap.parse_args()
    n = 256 << 20
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2d = n / (best_ms(lambda: dev.copy_(host, non_blocking=True)) * 1e-3)
    d2h = n / (best_ms(lambda: host.copy_(dev, non_blocking=True)) * 1e-3)
    del host, dev
    m = 1 << 30
    x = torch.empty(m, dtype=torch.bfloat16, device="cuda")
    y = torch.empty_like(x)
    bw = 2 * m * 2 / (best_ms(lambda: y.copy_(x)) * 1e-3)  # read + write bytes
    del x, y
    k = 8192
    a = torch.randn(k, k, dtype=torch.bfloat16, device="cuda")
    b = torch.randn(k, k, dtype=torch.bfloat16, device="cuda")
    flops = 2 * k ** 3 / (best_ms(lambda: torch.matmul(a, b)) * 1e-3)
    cap = torch.cuda.get_device_properties(0).total_memory
    prof = {"name": "b200-measured", "flops": flops, "bw_gpu": bw, "bw_h2d": h2d, "bw_d2h": d2h,
            "fast_capacity": float(cap),
            "notes": "measured on %s by tools/b200_profile.py: dense bf16 matmul 8192^3 (best of 10), "
                     "device copy of 1 Gi bf16 (read+write bytes), pinned 256 MiB cudaMemcpyAsync each way; "
                     "the zero-copy V recall reaches 35-48 GB/s of the bw_h2d figure (DESIGN.md 5)"
                     % torch.cuda.get_device_name(0)}
    with open(args.out, "w") as f:
        json.dump(prof, f, indent=1)
    print(json.dumps(prof))


if __name__ == "__main__":
    main()
