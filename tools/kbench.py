"""Kernel-level timing probe (development tool, not the bench contract).

Builds a C2-shaped cache with --layers layers and prints per-launch device
times of the scoring / selection / recall kernels, pipelined and serial.
    python tools/kbench.py --layers 8 --steps 3 [--tune key=val ...]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2404_18057_b200 import kcache as kc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv", type=int, default=32)
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--topn", type=int, default=128)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tune", action="append", default=[])
    args = ap.parse_args()
    L, b, n, n_kv, h, s, N = args.layers, args.batch, args.heads, args.kv, 128, args.s, args.topn
    d = n * h
    cfg = kc.ModelConfig(L, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s, n_kv)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, L, 2, "f16"))
    kb = torch.empty(s * b, n_kv * h, dtype=torch.float16, device="cuda")
    vb = torch.empty_like(kb)
    for l in range(L):
        kc.fill_uniform(kb, 2 + 100 * l)
        kc.fill_uniform(vb, 3 + 100 * l)
        cache.append_kv_device(l, kb, vb)
    torch.cuda.synchronize()
    del kb, vb
    for l in range(L):
        cache.offload_prefill_v(l)
    cache.begin_decode()
    qs = []
    for l in range(L):
        q = torch.empty(b, d, dtype=torch.float16, device="cuda")
        kc.fill_uniform(q, 1 + 100 * l)
        qs.append(q.float())
    nc = min(N, s)
    outs = [{"out": torch.empty(b, d, device="cuda"), "indices": torch.empty(b * n, nc, dtype=torch.int32, device="cuda"),
             "weights": torch.empty(b * n, nc, device="cuda"), "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")}
            for _ in range(L)]
    for kv in args.tune:
        k, v = kv.split("=")
        cache.set_tuning(k, int(v))
    res = {}
    for pipe in (1, 0):
        cache.set_tuning("pipeline", pipe)
        for _ in range(2):
            cache.decode_topn_layers_device(list(range(L)), qs, N, outs)
        torch.cuda.synchronize()
        cache.profile(True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            cache.decode_topn_layers_device(list(range(L)), qs, N, outs)
        e1.record()
        torch.cuda.synchronize()
        step = e0.elapsed_time(e1) / args.steps
        r = {"step_ms": step, "per_layer_ms": step / L}
        for kind in ("score", "select", "recall"):
            t = cache.profile_launches(kind)
            r[kind] = {"mean_us": 1e3 * statistics.mean(t), "min_us": 1e3 * min(t), "max_us": 1e3 * max(t),
                       "first_layers_us": [round(1e3 * x, 1) for x in t[:L]]}
        cache.profile(False)
        res["pipelined" if pipe else "serial"] = r
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
