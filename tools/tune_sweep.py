"""Tuning sweep on one resident cache (development tool, not the bench).

Builds a C2-shaped cache with --layers layers once, then for every tuning
combination measures the unprofiled pipelined step time (CUDA events on a
dedicated stream, no per-kernel events) and prints one line per combination.
    python tools/tune_sweep.py --layers 8 --grid recall_ctas=8,16,32,64 --grid score_chunk=0,2048
"""
import argparse
import itertools
import json
import os
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--grid", action="append", default=[], help="key=v1,v2,...")
    ap.add_argument("--resident", type=int, default=0, help="V-resident layers (0 = all offloaded)")
    ap.add_argument("--run-layers", default="", help="comma list: decode only these layers (default all)")
    ap.add_argument("--profile", action="store_true", help="also print per-kernel event times (perturbs overlap)")
    ap.add_argument("--per-step", action="store_true", help="print every step's time")
    ap.add_argument("--graph", action="store_true", help="capture every step into the cache's step graph")
    ap.add_argument("--engine", action="store_true",
                    help="one single-layer call per layer (layer l+1 ordered after layer l: the engine's dependency)")
    args = ap.parse_args()
    L, b, n, n_kv, h, s, N = args.layers, args.batch, args.heads, args.kv, 128, args.s, args.topn
    d = n * h
    cfg = kc.ModelConfig(L, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s, n_kv)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(args.resident, L, 2, "f16"))
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
    stream = torch.cuda.Stream()
    keys = [g.split("=")[0] for g in args.grid]
    vals = [[int(x) for x in g.split("=")[1].split(",")] for g in args.grid]
    run = [int(x) for x in args.run_layers.split(",")] if args.run_layers else list(range(L))
    qs = [qs[l] for l in run]
    outs = outs[:len(run)]
    k_bytes = 2 * b * n_kv * s * h * len(run)
    for combo in itertools.product(*vals) if vals else [()]:
        for k, v in zip(keys, combo):
            cache.set_tuning(k, v)
        def step():
            if args.graph:
                cache.step_graph_begin(N, stream)
            if args.engine:
                for i, l in enumerate(run):
                    cache.decode_topn_layers_device([l], [qs[i]], N, [outs[i]], stream=stream)
            else:
                cache.decode_topn_layers_device(run, qs, N, outs, stream=stream)
            if args.graph:
                cache.step_graph_launch(stream)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        ms = evs[0].elapsed_time(evs[-1]) / args.steps
        per_step = [round(evs[i].elapsed_time(evs[i + 1]), 2) for i in range(args.steps)]
        rec = {"tune": dict(zip(keys, combo)), "engine": args.engine, "step_ms": round(ms, 4), "per_layer_us": round(1e3 * ms / len(run), 1),
               "k_only_gbs": round(k_bytes / (ms * 1e-3) / 1e9, 1)}
        if args.per_step:
            rec["per_step_ms"] = per_step
        if args.profile:
            cache.profile(True)
            for _ in range(2):
                cache.decode_topn_layers_device(run, qs, N, outs, stream=stream)
            torch.cuda.synchronize()
            for kind in ("score", "select", "recall"):
                t = cache.profile_launches(kind)
                rec[kind + "_us"] = round(1e3 * sum(t) / len(t), 1) if t else None
            cache.profile(False)
        print(json.dumps(rec), flush=True)
    cache.close()


if __name__ == "__main__":
    main()
