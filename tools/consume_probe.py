"""Development probe: per-row phase durations of the dataflow consumer
(tuning consume_dbg) on a C2/C3-shaped cache, pipelined or engine-style."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_18057_b200 import kcache as kc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv", type=int, default=32)
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--topn", type=int, default=128)
    ap.add_argument("--tune", action="append", default=[])
    ap.add_argument("--engine", action="store_true")
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
    for t in args.tune:
        k, v = t.split("=")
        cache.set_tuning(k, int(v))
    cache.set_tuning("consume_dbg", 1)
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
    names = ["ready", "stats", "bound", "cands", "selected", "finished", "recalled", "wait0"]
    for rep in range(3):
        if args.engine:
            for l in range(L):
                cache.decode_topn_layers_device([l], [qs[l]], N, [outs[l]], stream=stream)
        else:
            cache.decode_topn_layers_device(list(range(L)), qs, N, outs, stream=stream)
        torch.cuda.synchronize()
    st = cache.consume_stamps().astype(np.int64)  # last layer of the last call
    t0 = st[:, 7].min()
    rel = (st - t0) / 1e3
    ph = {}
    ph["wait_us"] = float(np.mean(st[:, 0] - st[:, 7]) / 1e3)
    for a, bb, nm in [(0, 1, "stats_us"), (1, 2, "pass1_us"), (2, 3, "pass2_us"), (3, 4, "select_us"),
                      (4, 5, "finish_us"), (5, 6, "recall_us"), (0, 6, "row_total_us")]:
        dd = st[:, bb] - st[:, a]
        ok = (st[:, bb] > 0) & (st[:, a] > 0)
        ph[nm] = float(np.mean(dd[ok]) / 1e3) if ok.any() else None
    ph["first_ready_us"] = float(rel[:, 0].min())
    ph["last_ready_us"] = float(rel[:, 0].max())
    ph["last_done_us"] = float(rel[:, 6].max())
    print(json.dumps({"cfg": vars(args), "phases": {k: (round(v, 2) if v is not None else None) for k, v in ph.items()}}))
    cache.close()


if __name__ == "__main__":
    main()
