"""Prefill V offload rate (development / evidence tool).

During prefill the append kernel writes an offloaded layer's V straight into
the host arena (mapped stores over PCIe) while K goes to HBM; a V-resident
layer keeps both in HBM. This times the prefill append of one C2-shaped layer
(b=8, 32 heads x 128, 32k positions, fp16; chunks of `--chunk` positions) for
a resident and an offloaded layer and reports the offload rate, which
tests/test_perf_model_cpu.py feeds to the reference's prefill_overlap_check
(the paper's Eq. 1-2, perf_model.cpp:147-162).

    python tools/prefill_offload_bench.py [--out profiles/r01_prefill_offload.json]
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
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--chunk", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    b, n, h, s, chunk = args.batch, args.heads, 128, args.s, args.chunk
    d = n * h
    stream = torch.cuda.Stream()
    kb = torch.empty(chunk * b, d, dtype=torch.float16, device="cuda")
    vb = torch.empty_like(kb)
    kc.fill_uniform(kb, 2)
    kc.fill_uniform(vb, 3)
    torch.cuda.synchronize()
    res = {}
    for kind, resident in (("resident", 1), ("offloaded", 0)):
        times = []
        for _ in range(args.reps):
            cfg = kc.ModelConfig(1, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s, n)
            cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(resident, 1, 2, "f16"))
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _c in range(s // chunk):
                cache.append_kv_device(0, kb, vb, stream=stream)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            arena = cache.v_arena_kind()
            cache.close()
        res[kind] = {"ms_per_layer": min(times), "v_arena": arena if kind == "offloaded" else "hbm"}
    kv_bytes = 2 * b * s * d  # per tensor, fp16
    off = res["offloaded"]["ms_per_layer"]
    resd = res["resident"]["ms_per_layer"]
    rec = {"config": f"C2 layer prefill append: batch {b}, {n}x{h}, {s} positions, fp16, chunks of {chunk}",
           "gpu": torch.cuda.get_device_name(0), "v_bytes_per_layer": kv_bytes,
           "resident_ms_per_layer": resd, "offloaded_ms_per_layer": off,
           "offload_extra_ms_per_layer": off - resd,
           "offload_gbs": kv_bytes / ((off - resd) * 1e-3) / 1e9 if off > resd else None,
           "offloaded_layer_v_gbs": kv_bytes / (off * 1e-3) / 1e9,
           "v_arena": res["offloaded"]["v_arena"],
           "note": "offload_gbs = V bytes / (offloaded - resident append time): the host-write rate the "
                   "prefill pays; the V append is a separate launch after the K append"}
    print(json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
