"""Config 4 (BASELINE.json configs[3]): the paper's batch-size / throughput
claim. At a fixed per-GPU HBM budget for the KV cache, full-KV attention holds
K and V in HBM, KCache holds only K (V in pinned host memory), so KCache fits
~2x the batch. This sweeps the batch for both and times one decode-attention
step over all layers (CUDA events, inputs resident):

    python tools/c4_batch_sweep.py [--budget-gib 96] [--s 32768] [--out profiles/c4_batch_sweep.json]

Shape: LLaMA2-13B (40 layers, 40 heads x 128, MHA), fp16 K/V, N = 128.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2404_18057_b200 import kcache as kc  # noqa: E402


def build(L, b, n, h, s, resident):
    d = n * h
    cfg = kc.ModelConfig(L, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s, n)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(L if resident else 0, L, 2, "f16"))
    kb = torch.empty(s * b, d, dtype=torch.float16, device="cuda")
    vb = torch.empty_like(kb)
    for layer in range(L):
        kc.fill_uniform(kb, 2 + 100 * layer)
        kc.fill_uniform(vb, 3 + 100 * layer)
        cache.append_kv_device(layer, kb, vb)
    torch.cuda.synchronize()
    del kb, vb
    torch.cuda.empty_cache()
    for layer in range(L):
        cache.offload_prefill_v(layer)
    cache.begin_decode()
    qs = []
    for layer in range(L):
        q = torch.empty(b, d, dtype=torch.float16, device="cuda")
        kc.fill_uniform(q, 1 + 100 * layer)
        qs.append(q.float())
    return cache, qs


def time_steps(fn, stream, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--topn", type=int, default=128)
    ap.add_argument("--budget-gib", type=float, default=96.0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    L, n, h, s, N = args.layers, args.heads, 128, args.s, args.topn
    budget = int(args.budget_gib * (1 << 30))
    k_per_seq = 2 * L * n * h * s          # fp16 K bytes of one sequence
    b_full = budget // (2 * k_per_seq)
    b_kc = budget // k_per_seq
    stream = torch.cuda.Stream()
    rows = []

    def sweep(batches, mode):
        for b in batches:
            t0 = time.time()
            cache, qs = build(L, b, n, h, s, resident=(mode == "full"))
            setup = time.time() - t0
            outs = [torch.empty(b, n * h, dtype=torch.float32, device="cuda") for _ in range(L)]
            if mode == "full":
                def fn():
                    for layer in range(L):
                        cache.decode_full_device(layer, qs[layer], outs[layer], stream=stream)
            else:
                nc = min(N, s)
                douts = [{"out": outs[layer]} for layer in range(L)]

                def fn():
                    cache.decode_topn_layers_device(list(range(L)), qs, N, douts, stream=stream,
                                                    want_selection=False)
            ms = time_steps(fn, stream, args.steps, args.warmup)
            hbm = cache.fast_bytes_used()
            kv_bytes = (2 if mode == "full" else 1) * b * k_per_seq
            rec = {"mode": mode, "batch": b, "ms_per_step": ms, "tokens_per_s": b / (ms * 1e-3),
                   "kv_hbm_bytes": hbm, "hbm_stream_gbs": kv_bytes / (ms * 1e-3) / 1e9, "setup_s": setup}
            print(json.dumps(rec), flush=True)
            rows.append(rec)
            cache.close()
            del qs, outs
            torch.cuda.empty_cache()

    steps_full = sorted({max(1, b_full // 4), max(1, b_full // 2), b_full})
    steps_kc = sorted({max(1, b_full // 4), max(1, b_full // 2), b_full, b_kc})
    sweep(steps_full, "full")
    sweep(steps_kc, "kcache")
    best_full = max(r["tokens_per_s"] for r in rows if r["mode"] == "full")
    best_kc = max(r["tokens_per_s"] for r in rows if r["mode"] == "kcache")
    summary = {"config": "C4: LLaMA2-13B shape (40 layers, 40 x 128 MHA), fp16, s=%d, N=%d" % (s, N),
               "kv_hbm_budget_bytes": budget, "max_batch_full_kv": b_full, "max_batch_kcache": b_kc,
               "best_tokens_per_s_full_kv": best_full, "best_tokens_per_s_kcache": best_kc,
               "kcache_over_full": best_kc / best_full, "rows": rows,
               "gpu": torch.cuda.get_device_name(0)}
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
