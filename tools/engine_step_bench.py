"""Engine-style decode step latency (development / evidence tool).

A real decode step cannot pipeline layers (layer l+1's q needs layer l's
output), so each layer is one kc_decode_step call: append this token's K/V,
score, select, recall + P.V -- in order, layer after layer. This times such
steps on a C2-shaped cache (b=8, 32 layers, 32k context) for several row-group
counts (score_groups: intra-layer overlap of recall(group g) with
scoring(group g+1)).

    python tools/engine_step_bench.py [--layers 32] [--groups 1,2,4,8]
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
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--topn", type=int, default=128)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--groups", default="1,2,4,8")
    ap.add_argument("--out", default="")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--tune", action="append", default=[], help="key=value cache tuning knob (repeatable)")
    ap.add_argument("--graph", default="0", help="comma list of 0/1: eager launches / one CUDA Graph per step")
    args = ap.parse_args()
    L, b, n, h, s, N = args.layers, args.batch, args.heads, 128, args.s, args.topn
    d = n * h
    groups = [int(x) for x in args.groups.split(",")]
    total_steps = (args.steps + 4) * len(groups) * len(args.graph.split(","))
    cfg = kc.ModelConfig(L, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s + total_steps, n)
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
    for kv in args.tune:
        k, v = kv.split("=")
        cache.set_tuning(k, int(v))
    # this step's q/k/v rows, as one QKV projection would write them
    qkv = torch.empty(3, b, d, dtype=torch.float16, device="cuda")
    q, knew, vnew = qkv[0], qkv[1], qkv[2]
    out = torch.empty(b, d, dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()
    rows = []

    use_graph = [False]

    def step(seed):
        if use_graph[0]:
            cache.step_graph_begin(N, stream)
        for layer in range(L):
            kc.fill_uniform(qkv, 7 + seed * 1000 + layer, stream=stream)
            cache.decode_step_device(layer, q, knew, vnew, out, N, stream=stream)
        if use_graph[0]:
            cache.step_graph_launch(stream)

    seed = 0
    for g, gr in [(g, gr) for gr in args.graph.split(",") for g in groups]:
        use_graph[0] = gr == "1"
        cache.set_tuning("score_groups", g)
        for _ in range(2):
            step(seed)
            seed += 1
        torch.cuda.synchronize()
        cache.step_stats(reset=True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(seed)
            seed += 1
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        st = cache.step_stats(reset=True)
        import time as _t
        c0 = _t.perf_counter()
        step(seed)
        seed += 1
        enqueue_ms = (_t.perf_counter() - c0) * 1e3
        torch.cuda.synchronize()
        cache.step_stats(reset=True)
        if args.profile and not use_graph[0]:
            cache.profile(True)
            step(seed)
            seed += 1
            torch.cuda.synchronize()
            sp = {k: cache.profile_spans(k) for k in ("score", "select", "recall")}
            sp = {k: v for k, v in sp.items() if v}  # no select spans when the scoring kernel selects
            cache.profile(False)
            t0 = sp["score"][0][0]
            for layer in range(min(3 * max(1, g), len(sp["score"]))):
                print("  layer", layer, "  ".join(f"{k} {(sp[k][layer][0] - t0) * 1e3:.0f}-{(sp[k][layer][1] - t0) * 1e3:.0f}"
                                                  for k in sp))
            print("  mean us:", {k: round(1e3 * sum(e - a for a, e in v) / len(v), 1) for k, v in sp.items()})
        rec = {"score_groups": g, "graph": use_graph[0], "tune": args.tune, "ms_per_step": ms, "host_enqueue_ms_per_step": enqueue_ms, "tokens_per_s": b / (ms * 1e-3), "per_layer_us": 1e3 * ms / L,
               "len": cache.current_len(), "mean_dropped_mass": st["mean_dropped_mass"],
               "h2d_bytes_per_step": st["h2d_bytes"] // args.steps, "d2h_bytes_per_step": st["d2h_bytes"] // args.steps}
        print(json.dumps(rec), flush=True)
        rows.append(rec)
    cache.close()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"config": "engine-style decode step (append + TopN per layer, no cross-layer pipelining), "
                                 "LLaMA2-7B attention shape b=%d, %d layers, %dk context, N=%d" % (b, L, s // 1024, N),
                       "gpu": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
