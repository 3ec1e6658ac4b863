"""Config 5 (BASELINE.json configs[4]): top-N x context sweep locating the
crossover from HBM-bound scoring to host-link-bound V recall.

For every context s and top-N, one KCache decode step over --layers layers
(LLaMA2-7B attention shape, batch 8, fp16, V in pinned host memory) is timed
pipelined (CUDA events) and, in a separate serial pass, per kernel:

    python tools/c5_crossover.py [--layers 4] [--out profiles/c5_crossover.json]

K time per layer is 2*b*n*s*h bytes at HBM rate, V time 2*b*n*N*h bytes at the
recall rate, so the recall dominates when s/N drops below
BW_HBM / BW_recall (same form as perf_model.cpp:165-174).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2404_18057_b200 import kcache as kc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--contexts", default="4096,8192,16384,32768,65536,131072")
    ap.add_argument("--topns", default="32,64,128,256,512")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    L, b, n, h = args.layers, args.batch, args.heads, 128
    d = n * h
    stream = torch.cuda.Stream()
    rows = []
    for s in [int(x) for x in args.contexts.split(",")]:
        cfg = kc.ModelConfig(L, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s, n)
        cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, L, 2, "f16"))
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
        outs = [{"out": torch.empty(b, d, dtype=torch.float32, device="cuda")} for _ in range(L)]
        for N in [int(x) for x in args.topns.split(",")]:
            def step():
                cache.decode_topn_layers_device(list(range(L)), qs, N, outs, stream=stream, want_selection=False)
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            # serial pass: each kernel alone (the stream-ordered kernels: the
            # dataflow consumer merges selection and recall into one launch)
            cache.set_tuning("pipeline", 0)
            cache.set_tuning("consume", 0)
            cache.profile(True)
            step()
            torch.cuda.synchronize()
            per = {}
            for kind in ("score", "select", "recall"):
                t = cache.profile_launches(kind)
                per[kind + "_us"] = 1e3 * sum(t) / max(len(t), 1)
            cache.profile(False)
            cache.set_tuning("pipeline", 1)
            cache.set_tuning("consume", 1)
            nc = min(N, s)
            k_bytes = 2 * b * n * s * h
            v_bytes = 2 * b * n * nc * h
            flow = s >= 16384 and min(N, s) <= 256  # the store's auto policy (kc_capi.cu decode_topn_impl)
            rec = {"s": s, "top_n": N, "path": ("dataflow consumer" if flow else "stream-ordered") +
                   " (default policy); per-kernel *_us from the stream-ordered kernels run serially", "s_over_n": s / nc, "ms_per_step": ms, "tokens_per_s": b / (ms * 1e-3),
                   "per_layer_us": 1e3 * ms / L, "k_bytes_per_layer": k_bytes, "vsel_bytes_per_layer": v_bytes,
                   "score_gbs": k_bytes / (per["score_us"] * 1e-6) / 1e9,
                   "recall_gbs": v_bytes / (per["recall_us"] * 1e-6) / 1e9,
                   "bound": "recall" if per["recall_us"] > per["score_us"] + per["select_us"] else "scoring", **per}
            print(json.dumps(rec), flush=True)
            rows.append(rec)
        cache.close()
        del qs, outs
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"config": "C5: LLaMA2-7B attention shape, batch %d, %d layers, fp16" % (b, L),
                       "gpu": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
