"""Prefill V offload (development / evidence tool).

Two paths for the prefill V of an offloaded layer (kc_set_tuning
"prefill_stage"):
* 1 (default): the append kernel writes V into an HBM stage; offload_prefill_v
  sends the stage to the host arena on the cache's offload stream -- an SM
  copy kernel for the (managed) arena, the copy engine for pinned layers -- so
  the transfer runs behind the next layer's work: the paper's overlapped
  offload (Eq. 1-2, perf_model.cpp:147-162);
* 0: the append kernel writes V straight into the host arena (SM-issued PCIe
  stores, the r01 path): the transfer sits inside the append.

Measures, on a C2-shaped layer (b=8, 32 heads x 128, 32k positions, fp16,
appended in chunks of --chunk positions):
  1. the D2H rate of one staged offload (offload_prefill_v + kc_sync);
  2. a prefill timeline of --layers layers, each = append its K/V chunks +
     --compute-ms of stand-in layer compute (fp16 GEMMs on the same stream,
     the projections / FFN the engine runs between appends), then
     offload_prefill_v -- total time per mode, vs no offload at all (V kept in
     HBM: resident layers).

    python tools/prefill_offload_bench.py [--layers 4] [--compute-ms 30] [--out profiles/r02_prefill_offload.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2404_18057_b200 import kcache as kc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--chunk", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--compute-ms", type=float, default=30.0)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    b, n, h, s, chunk, L = args.batch, args.heads, 128, args.s, args.chunk, args.layers
    d = n * h
    stream = torch.cuda.Stream()
    kb = torch.empty(chunk * b, d, dtype=torch.float16, device="cuda")
    vb = torch.empty_like(kb)
    kc.fill_uniform(kb, 2)
    kc.fill_uniform(vb, 3)
    # stand-in layer compute: square fp16 GEMMs, calibrated to --compute-ms
    ga = torch.randn(8192, 8192, dtype=torch.float16, device="cuda")
    gb = torch.randn(8192, 8192, dtype=torch.float16, device="cuda")
    with torch.cuda.stream(stream):
        for _ in range(3):
            torch.mm(ga, gb)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(10):
            torch.mm(ga, gb)
    e1.record(stream)
    e1.synchronize()
    gemm_ms = e0.elapsed_time(e1) / 10
    n_gemm = max(1, round(args.compute_ms / gemm_ms))
    torch.cuda.synchronize()

    def make(resident, stage):
        cfg = kc.ModelConfig(L, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s, n)
        cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(L if resident else 0, L, 2, "f16"))
        cache.set_tuning("prefill_stage", stage)
        return cache

    def append_layer(cache, layer):
        for _c in range(s // chunk):
            cache.append_kv_device(layer, kb, vb, stream=stream)

    rec = {"config": f"C2 layer prefill: batch {b}, {n}x{h}, {s} positions, fp16, chunks of {chunk}",
           "gpu": torch.cuda.get_device_name(0), "v_bytes_per_layer": 2 * b * s * d}
    # 1. D2H rate of one staged offload (SM copy kernel into the managed arena,
    # by grid size)
    rec["staged_offload_gbs"] = {}
    for ctas in (8, 16, 32, 64):
        cache = make(False, 1)
        cache.set_tuning("stage_copy_ctas", ctas)
        append_layer(cache, 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cache.offload_prefill_v(0)
        cache.sync()
        dt = time.perf_counter() - t0
        rec["staged_offload_gbs"][ctas] = 2 * b * s * d / dt / 1e9
        rec["v_arena"] = cache.v_arena_kind()
        cache.close()
    # 2. timelines
    rows = {}
    for mode, resident, stage in (("v_in_hbm", True, 1), ("mapped_stores", False, 0), ("staged", False, 1)):
        cache = make(resident, stage)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        per_layer = []
        for layer in range(L):
            a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            append_layer(cache, layer)
            c.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(n_gemm):
                    torch.mm(ga, gb)
            stream.synchronize()  # the engine's layer boundary (host reads the layer's output)
            cache.offload_prefill_v(layer)
            per_layer.append(a.elapsed_time(c))
        cache.begin_decode()  # waits for the last layer's D2H
        torch.cuda.synchronize()
        total = (time.perf_counter() - t0) * 1e3
        rows[mode] = {"total_ms": total, "append_ms_per_layer": per_layer}
        cache.close()
    rec["layers"] = L
    rec["compute_ms_per_layer"] = n_gemm * gemm_ms
    rec["timelines"] = rows
    base = rows["v_in_hbm"]["total_ms"]
    rec["offload_cost_ms"] = {k: v["total_ms"] - base for k, v in rows.items() if k != "v_in_hbm"}
    rec["note"] = ("total = L x (append + stand-in compute) + what the offload adds; staged: the D2H of layer l "
                   "overlaps layer l+1, only the last layer's copy shows (begin_decode waits for it)")
    print(json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
