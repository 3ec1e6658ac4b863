"""Per-launch timeline of one pipelined decode step (development tool).

    python tools/timeline.py --layers 8 [--tune key=val ...]
Prints, for each layer, start/end (us) of scoring, selection and recall on
their streams, relative to the step start.
"""
import argparse
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
    ap.add_argument("--tune", action="append", default=[])
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--verbose", action="store_true")
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
    for _ in range(3):
        cache.decode_topn_layers_device(list(range(L)), qs, N, outs)
    torch.cuda.synchronize()
    ap_steps = args.steps
    for step in range(ap_steps):
        cache.profile(True)
        cache.decode_topn_layers_device(list(range(L)), qs, N, outs)
        torch.cuda.synchronize()
        sp = {k: cache.profile_spans(k) for k in ("score", "select", "recall")}
        cache.profile(False)
        t0 = sp["score"][0][0]
        end = max(e for k in sp for _, e in sp[k])
        if args.verbose or step == 0:
            print("layer   score(start-end)      select(start-end)     recall(start-end)   [us]")
            for l in range(L):
                row = [f"{(a - t0) * 1e3:8.1f}-{(e - t0) * 1e3:8.1f}" for a, e in (sp[k][l] for k in ("score", "select", "recall"))]
                print(f"{l:5d}  " + "   ".join(row))
        dur = {k: sum(e - a for a, e in sp[k]) / L * 1e3 for k in sp}
        print(f"step {step}: span {(end - t0) * 1e3:.1f} us, per layer {(end - t0) * 1e3 / L:.1f} us; mean durations "
              + ", ".join(f"{k} {v:.1f}" for k, v in dur.items()), flush=True)


if __name__ == "__main__":
    main()
