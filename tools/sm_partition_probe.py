"""Development probe (not the bench): scoring bandwidth vs the number of SMs
it may use. tools/libsm_blocker.so parks one spinning 1024-thread CTA with
200 KB of shared memory on each of k SMs; the pipelined C2-shaped decode then
runs on the other 148 - k. Prints, per k, the step time and the per-kernel
event times (cache.profile). Feeds the SM-partitioning plan.
    python tools/sm_partition_probe.py --layers 8 --blocked 0,12,20,28,36
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2404_18057_b200 import kcache as kc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--kv", type=int, default=32)
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--blocked", default="0,12,20,28,36")
    args = ap.parse_args()
    lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsm_blocker.so"))
    lib.sm_blocker_launch.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    L, b, n, n_kv, h, s, N = args.layers, args.batch, 32, args.kv, 128, args.s, 128
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
    outs = [{"out": torch.empty(b, d, device="cuda"),
             "indices": torch.empty(b * n, nc, dtype=torch.int32, device="cuda"),
             "weights": torch.empty(b * n, nc, device="cuda"),
             "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")} for _ in range(L)]
    run = list(range(L))
    stream, bstream, rstream = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    k_bytes_layer = 2 * b * n_kv * s * h
    for _ in range(3):
        cache.decode_topn_layers_device(run, qs, N, outs, stream=stream)
    torch.cuda.synchronize()
    for k in [int(x) for x in args.blocked.split(",")]:
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        if k:
            assert lib.sm_blocker_launch(k, flag.data_ptr(), bstream.cuda_stream) == 0
            time.sleep(0.05)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        evs[0].record(stream)
        for _ in range(args.steps):
            cache.decode_topn_layers_device(run, qs, N, outs, stream=stream)
        evs[1].record(stream)
        evs[1].synchronize()
        ms = evs[0].elapsed_time(evs[1]) / args.steps
        cache.profile(True)
        for _ in range(2):
            cache.decode_topn_layers_device(run, qs, N, outs, stream=stream)
        stream.synchronize()
        rec = {"blocked_sms": k, "free_sms": 148 - k, "step_ms": round(ms, 4), "per_layer_us": round(1e3 * ms / L, 1)}
        for kind in ("score", "select", "recall"):
            t = cache.profile_launches(kind)
            rec[kind + "_us"] = round(1e3 * sum(t) / len(t), 1) if t else None
        cache.profile(False)
        if rec["score_us"]:
            rec["score_tbs"] = round(k_bytes_layer / (rec["score_us"] * 1e-6) / 1e12, 2)
        with torch.cuda.stream(rstream):
            flag.fill_(1)
        torch.cuda.synchronize()
        print(json.dumps(rec), flush=True)
    cache.close()


if __name__ == "__main__":
    main()
