#!/usr/bin/env python
"""KCache decode-attention benchmark (BASELINE.json metric).

Metric: "KCache decode-attn tokens/s/GPU, LLaMA2-7B shape 32k ctx; % of
HBM+H2D roofline". One step = decode_attention_topn for every layer of one
decode token of the whole batch: q.K^T scoring over the HBM-resident K cache,
top-N selection, recall of the selected V rows from pinned host memory, P.V
(SURVEY.md section 8(d)). tokens/s = batch / step time.

Default workload (N=1): configs[1] -- LLaMA2-7B shape, 32 layers, batch 8,
32k context, N=128, fp16 K in HBM (64 GiB) and fp16 V in pinned host memory
(64 GiB), synthetic SeededRng inputs. Inputs (64 GiB of K) dwarf the 126 MB
L2, so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c1]
    python bench.py --impl reference ...   # the reference CPU path, all host cores

Multi-GPU (torchrun): one process per GPU, each with its own batch of
sequences and its own K/V shards (partition by request batch, no collective on
the data path): weak scaling, value = all ranks' tokens / max-over-ranks time.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(workload="LLaMA2-7B-shape KCache decode attention: 32 layers, batch 8, 32k context, N=128, "
                        "fp16 K in HBM / fp16 V in host memory (read zero-copy over PCIe)",
               n_layers=32, batch=8, n_heads=32, n_kv=32, h=128, s=32768, top_n=128),
    "c3": dict(workload="LLaMA3-8B-shape GQA (32 q / 8 kv heads) KCache decode attention: 32 layers, batch 32, "
                        "16k context, N=128",
               n_layers=32, batch=32, n_heads=32, n_kv=8, h=128, s=16384, top_n=128),
    "c1": dict(workload="LLaMA2-7B-shape single attention layer, batch 1, 4k context, N=128",
               n_layers=1, batch=1, n_heads=32, n_kv=32, h=128, s=4096, top_n=128),
}
METRIC = "KCache decode-attn tokens/s/GPU, LLaMA2-7B shape 32k ctx; % of HBM+H2D roofline"
UNIT = "tokens/s"
SEED_Q, SEED_K, SEED_V = 1, 2, 3


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        load = [x for x in sm if x > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": smax, "reasons": reasons, "samples": len(rows)}


def h2d_bandwidth(torch):
    """Pinned cudaMemcpyAsync of 256 MiB, best of 10 (SURVEY 8(d) BW_H2D)."""
    n = 256 << 20
    src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    del src, dst
    return n / (best * 1e-3) / 1e9


def cpu_reference_sample(cfg, threads, passes, warm=1):
    """The reference decode_attention_topn (oracle/_ref) on host threads: one
    pass = a whole decode step (every layer's q against the layer cache, all
    batch rows, all heads); returns (seconds per step list, kind, sample)."""
    from oracle.oracle import Reference, ReferenceBench
    if cfg["n_kv"] != cfg["n_heads"] or not Reference.available():
        return None
    hps = 16 if cfg["n_heads"] % 16 == 0 else cfg["n_heads"]
    rb = ReferenceBench(cfg["s"], cfg["batch"], cfg["n_heads"], cfg["h"], hps, cfg["top_n"], threads,
                        seeds=(SEED_Q, SEED_K, SEED_V), n_layers=cfg["n_layers"])
    try:
        for _ in range(warm):
            rb.run()
        times = [rb.run()[0] for _ in range(passes)]
    finally:
        rb.close()
    sample = (f"reference decode_attention_topn (oracle/_ref, -O3 -ffp-contract=off), a whole step: "
              f"{cfg['n_layers']} layers' q (seeds of the GPU arm) x {cfg['batch']} rows x {cfg['n_heads']} heads "
              f"at s={cfg['s']}, N={cfg['top_n']}, against one fp32 layer cache (the fp32 cache of all "
              f"{cfg['n_layers']} layers would need {4 * 2 * cfg['n_layers'] * cfg['batch'] * cfg['s'] * cfg['n_heads'] * cfg['h'] / 2**30:.0f} GiB "
              f"of host RAM; the per-layer work is identical), {threads} threads over "
              f"{cfg['n_layers'] * cfg['batch'] * cfg['n_heads'] // hps} (layer, row, 16-head) items")
    return times, "reference", sample


def resolve_shard(args, cfg, world):
    """How N > 1 ranks split the work: "batch" = every rank
    serves its own batch of cfg["batch"] sequences (weak scaling), "units" =
    the (batch row, kv head) units of ONE global batch are partitioned
    (strong scaling). auto: units for config 3 (a fixed global batch of 32,
    BASELINE.json configs[2]) and whenever the weak-scaling V shards would not
    fit in host memory; batch otherwise."""
    if world == 1:
        return "batch"
    if args.shard != "auto":
        return args.shard
    if args.config == "c3":
        return "units"
    from paper_2404_18057_b200.sharding import host_mem_available
    v_all = world * 2 * cfg["n_layers"] * cfg["batch"] * cfg["n_kv"] * cfg["s"] * cfg["h"]
    avail = host_mem_available()
    return "units" if avail and v_all > 0.85 * avail else "batch"


def config_block(cfg, args, world, shard):
    """The workload keys both arms report (same dict, so the driver can match
    the reference arm's config to this arm's)."""
    b, n_kv, L = cfg["batch"], cfg["n_kv"], cfg["n_layers"]
    units = b * n_kv
    if shard == "units":
        per = (units + world - 1) // world
        par = f"(batch row, kv head) units of one global batch: {per} of {units} per rank, no data-path collective"
        gb = b
        k_gpu = 2 * L * per * cfg["s"] * cfg["h"]
    else:
        par = f"partition by request batch x{world}, no data-path collective"
        gb = b * world
        k_gpu = 2 * L * units * cfg["s"] * cfg["h"]
    return {"workload": cfg["workload"], "config": args.config, "layers": L, "global_batch": gb,
            "n_heads": cfg["n_heads"], "n_kv_heads": n_kv, "head_dim": cfg["h"], "s": cfg["s"],
            "top_n": cfg["top_n"], "shard": shard, "parallelism": par, "data_dist": args.dist,
            "l2": "inputs larger than L2 (%.1f GiB K per GPU)" % (k_gpu / 2**30)}


def run_reference_arm(args, cfg):
    rank, _, world = dist_env()
    if rank != 0:
        return
    shard = resolve_shard(args, cfg, world)
    threads = os.cpu_count() or 1
    res = cpu_reference_sample(cfg, threads, passes=args.steps, warm=args.warmup)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built or config is GQA (reference is MHA-only)"}))
        return
    times, kind, sample = res
    t_step = statistics.mean(times)
    # whole job: the reference serves the same global batch on the host cores
    value = (cfg["batch"] * (world if shard == "batch" else 1)) / t_step
    if shard == "batch" and world > 1:
        t_step = t_step * world  # the host runs every rank's batch in turn
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak" if shard == "batch" else "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (SeededRng, fp16-rounded, fed as fp32)",
        "config": config_block(cfg, args, world, shard),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class RankWorkload:
    """This rank's share of the workload, resident: the TieredKVCache (K in
    HBM, V in host memory or -- resident=True -- in HBM), the layers' q and
    the output buffers. shard "batch": the rank's own batch of cfg["batch"]
    sequences (data seeded per rank); "units": the rank's (batch, kv head)
    units of the global batch (sharding.UnitShard; the global data, sliced)."""

    def __init__(self, kc, torch, cfg, dev, rank, world, shard, resident=False, tune=(), extra_seq=0,
                 dist="uniform"):
        from paper_2404_18057_b200.sharding import UnitShard, gpu_numa_node
        L, B, n, n_kv, h, s = (cfg[k] for k in ("n_layers", "batch", "n_heads", "n_kv", "h", "s"))
        G = n // n_kv
        self.numa = gpu_numa_node(dev.index)
        if shard == "units":
            self.shard = UnitShard(B, n_kv, G, h, world, rank)
            mcfg = self.shard.model_config(kc, L, s + extra_seq)
            self.b, self.rows = 1, self.shard.n_units
            seed_off = 0
        else:
            self.shard = None
            d = n * h
            mcfg = kc.ModelConfig(L, d, n, h, kc.ModelConfig.default_ffn_hidden(d), 32000, s + extra_seq, n_kv)
            self.b, self.rows = B, B * n_kv
            seed_off = 1_000_003 * rank
        self.d = mcfg.d_model
        self.slots = self.b * mcfg.n_heads
        self.cache = kc.TieredKVCache(mcfg, self.b, kc.TierPlacement.kcache(L if resident else 0, L, 2, "f16"),
                                      device=dev.index, numa_node=-1 if resident else self.numa)
        for kv in tune:
            key, val = kv.split("=")
            self.cache.set_tuning(key, int(val))
        kbuf = torch.empty(s * B, n_kv * h, dtype=torch.float16, device=dev)
        vbuf = torch.empty_like(kbuf)
        for layer in range(L):
            if dist == "peaked":
                # SURVEY 8(d)'s realistic locality (verify.cpp:417-431): keys
                # nearly orthogonal to q except 24 planted hot positions per
                # (batch, kv head), each a constant row in [6, 8]
                import numpy as np
                kc.fill_uniform(kbuf, SEED_K + 100 * layer + seed_off, lo=-0.05, hi=0.05)
                rng = np.random.default_rng(SEED_K + 100 * layer + seed_off)
                hot = torch.as_tensor(np.concatenate([rng.choice(s, 24, replace=False) for _ in range(B * n_kv)]),
                                      device=dev)
                unit = torch.arange(B * n_kv, device=dev).repeat_interleave(24)
                vals = torch.as_tensor(rng.uniform(6.0, 8.0, B * n_kv * 24), dtype=torch.float16, device=dev)
                kbuf.view(s, B * n_kv, h)[hot, unit, :] = vals[:, None]
            else:
                kc.fill_uniform(kbuf, SEED_K + 100 * layer + seed_off)
            kc.fill_uniform(vbuf, SEED_V + 100 * layer + seed_off)
            if self.shard is None:
                self.cache.append_kv_device(layer, kbuf, vbuf)
            else:
                self.cache.append_kv_device(layer, self.shard.kv_rows(kbuf).contiguous(),
                                            self.shard.kv_rows(vbuf).contiguous())
        torch.cuda.synchronize()
        del kbuf, vbuf
        torch.cuda.empty_cache()
        for layer in range(L):
            self.cache.offload_prefill_v(layer)
        self.cache.begin_decode()
        self.qs = []
        for layer in range(L):
            q16 = torch.empty(B, n * h, dtype=torch.float16, device=dev)
            if dist == "peaked":
                kc.fill_uniform(q16, SEED_Q + 100 * layer + seed_off, lo=0.5, hi=1.0)
            else:
                kc.fill_uniform(q16, SEED_Q + 100 * layer + seed_off)
            q = q16.float()
            self.qs.append(q if self.shard is None else self.shard.q_rows(q).contiguous())

    def close(self):
        self.cache.close()
        self.qs = []


ENGINE_STEPS = 8


def engine_step(kc, torch, wl, cfg, dev, args, barrier):
    """The engine-realistic decode step (Engine::forward_decode,
    engine.cpp:124-165): layer l+1's q needs layer l's output, so every layer
    is its own library call -- kc_decode_step: append this token's K/V row
    (the new V row to the host arena), score, select, recall + P.V -- with
    only the intra-layer overlap of row groups (recall of group g under the
    scoring of group g+1). Run after the headline legs: it grows the cache by
    warm-up + timed steps positions."""
    L, N = cfg["n_layers"], cfg["top_n"]
    cache = wl.cache
    b, d, kvw = wl.b, wl.d, cache.kv_width
    q16 = [torch.empty(b, d, dtype=torch.float16, device=dev) for _ in range(L)]
    kv16 = [torch.empty(2, b, kvw, dtype=torch.float16, device=dev) for _ in range(L)]
    for layer in range(L):
        kc.fill_uniform(q16[layer], 900 + layer)
        kc.fill_uniform(kv16[layer], 950 + layer)
    out = torch.empty(b, d, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def step():
        for layer in range(L):
            cache.decode_step_device(layer, q16[layer], kv16[layer][0], kv16[layer][1], out, N, stream=stream)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ENGINE_STEPS):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    cache.step_stats(reset=True)
    return e0.elapsed_time(e1) / ENGINE_STEPS


def full_kv_step(kc, torch, cfg, dev, rank, world, shard, args, barrier):
    """decode_attention_full over every layer with K and V resident in HBM
    (C2: 128 GiB), timed like the KCache step. Returns the per-step numbers."""
    L, n_kv, h, s = (cfg[k] for k in ("n_layers", "n_kv", "h", "s"))
    wl = RankWorkload(kc, torch, cfg, dev, rank, world, shard, resident=True)
    outs = [torch.empty(wl.b, wl.d, dtype=torch.float32, device=dev) for _ in range(L)]
    stream = torch.cuda.Stream(device=dev)

    def step():
        for layer in range(L):
            wl.cache.decode_full_device(layer, wl.qs[layer], outs[layer], stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps = min(args.steps, 10)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / steps
    kv_bytes = 2 * 2 * wl.rows * s * h * L
    wl.close()
    del outs
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "steps": steps, "kv_bytes_per_step": kv_bytes,
            "hbm_gbs": kv_bytes / (ms * 1e-3) / 1e9, "hbm_bytes": kv_bytes}


def run_ours(args, cfg):
    import numpy as np
    import torch

    from paper_2404_18057_b200 import kcache as kc

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    L, B, n, n_kv, h, s, N = (cfg[k] for k in ("n_layers", "batch", "n_heads", "n_kv", "h", "s", "top_n"))
    G = n // n_kv
    nc = min(N, s)
    shard = resolve_shard(args, cfg, world)
    # every rank keeps its V shard in host memory (C2 weak scaling: 64 GiB per
    # rank): refuse cleanly rather than drive the host out of memory
    from paper_2404_18057_b200.sharding import host_mem_available, partition_units
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    rows_rank = len(partition_units(B, n_kv, world, rank)) if shard == "units" else B * n_kv
    v_bytes_rank = 2 * L * rows_rank * s * h
    avail = host_mem_available()
    if avail and local_world * v_bytes_rank > 0.92 * avail:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "error": "host memory: %d ranks x %.1f GiB V shards exceed "
                              "MemAvailable %.1f GiB" % (local_world, v_bytes_rank / 2**30, avail / 2**30)}))
        sys.exit(3)
    t0 = time.time()
    wl = RankWorkload(kc, torch, cfg, dev, rank, world, shard, tune=args.tune,
                      extra_seq=0 if args.no_engine else ENGINE_STEPS + 2, dist=args.dist)
    cache, qs, b, d, slots = wl.cache, wl.qs, wl.b, wl.d, wl.slots
    numa = wl.numa
    v_arena = cache.v_arena_kind()
    setup_s = time.time() - t0
    outs = [{"out": torch.empty(b, d, dtype=torch.float32, device=dev),
             "indices": torch.empty(slots, nc, dtype=torch.int32, device=dev),
             "weights": torch.empty(slots, nc, dtype=torch.float32, device=dev),
             "dropped": torch.empty(slots, dtype=torch.float64, device=dev)} for _ in range(L)]
    layers = list(range(L))
    stream = torch.cuda.Stream(device=dev)  # a dedicated (non-legacy) stream for the device path

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def step():
        return cache.decode_topn_layers_device(layers, qs, N, outs, stream=stream)

    def timed_steps(n):
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(n):
            inf = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return ev0.elapsed_time(ev1) / n, inf

    sampler = ClockSampler(local_rank)
    sampler.start()
    for _ in range(args.warmup):
        step()
    # the timed region: no per-kernel events inside
    ms_local, info = timed_steps(args.steps)
    # separate profiled passes: events around the scoring launches only (the
    # roofline kernel; its step time shows the perturbation), then around every
    # launch for the breakdown
    prof_steps = min(args.steps, 10)
    cache.profile(True, kinds=("score",))
    score_prof_ms, _ = timed_steps(prof_steps)
    score_ms, score_n = cache.profile_read("score")
    cache.profile(True)
    prof_ms, _ = timed_steps(prof_steps)
    select_ms, select_n = cache.profile_read("select")
    recall_ms, recall_n = cache.profile_read("recall")
    all_score_ms, _ = cache.profile_read("score")
    # each kernel alone (serial schedule): what the pipelined overlap costs it
    cache.set_tuning("pipeline", 0)
    cache.profile(True)
    serial_ms, _ = timed_steps(min(prof_steps, 3))
    iso = {k: cache.profile_read(k) for k in ("score", "select", "recall")}
    cache.profile(False)
    cache.set_tuning("pipeline", 1)
    h2d_per_layer = info[0][1]

    # ---- end to end: host (pinned) q in, every output back to the host ----
    qh = [torch.empty(b, d, dtype=torch.float32, pin_memory=True) for _ in range(L)]
    for i in range(L):
        qh[i].copy_(qs[i])
    qh_np = [t.numpy() for t in qh]
    outs_h = [{"out": torch.empty(b, d, dtype=torch.float32, pin_memory=True).numpy(),
               "indices": torch.empty(slots, nc, dtype=torch.int32, pin_memory=True).numpy(),
               "weights": torch.empty(slots, nc, dtype=torch.float32, pin_memory=True).numpy(),
               "dropped": torch.empty(slots, dtype=torch.float64, pin_memory=True).numpy()} for _ in range(L)]
    e2e_steps = 0 if args.no_e2e else args.steps
    # the decode loop's host buffers are fixed: bind them once (ctypes
    # argument arrays), every step is one kc_decode_topn_layers call
    e2e_call = cache.prepare_topn_layers_host(layers, qh_np, N, outs_h)
    for _ in range(args.warmup if e2e_steps else 0):
        e2e_call()
    barrier()
    te0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    te1 = time.perf_counter()
    barrier()
    e2e_ms_local = (te1 - te0) * 1e3 / max(e2e_steps, 1)
    clocks = sampler.stop()
    # BW_H2D of the roofline: every rank copies at once (ranks may share a
    # PCIe switch uplink), the slowest rank's rate counts
    barrier()
    h2d_local = h2d_bandwidth(torch)
    e2e_check = float(np.abs(outs_h[0]["out"]).sum())
    del e2e_call, outs_h, qh, qh_np
    # unit shards: gather layer 0's outputs of every rank into the global
    # [batch, d] (outside the timed region; verification / checksum only)
    gathered = None
    if shard == "units":
        from paper_2404_18057_b200.sharding import gather_units
        full_out = gather_units(outs[0]["out"], wl.shard)
        gathered = {"shape": list(full_out.shape), "abs_sum": float(full_out.abs().sum())}

    # ---- the engine-realistic step (no cross-layer pipelining), labelled apart ----
    engine_ms_local = 0.0 if args.no_engine else engine_step(kc, torch, wl, cfg, dev, args, barrier)

    from paper_2404_18057_b200.sharding import max_over_ranks
    ms, e2e_ms, neg_h2d, engine_ms = max_over_ranks([ms_local, e2e_ms_local, -h2d_local, engine_ms_local],
                                                    device=dev)
    h2d_bw = -neg_h2d
    wl.close()
    del qs, outs, cache
    torch.cuda.empty_cache()

    # ---- the comparator: full-KV-in-HBM decode attention on the same workload ----
    full = None
    if not args.no_full_kv:
        full = full_kv_step(kc, torch, cfg, dev, rank, world, shard, args, barrier)
        if world > 1:
            from paper_2404_18057_b200.sharding import max_over_ranks
            full["ms_per_step"] = max_over_ranks([full["ms_per_step"]], device=dev)[0]
            full["hbm_gbs"] = full["kv_bytes_per_step"] / (full["ms_per_step"] * 1e-3) / 1e9

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    hbm_peak, peak_kind = measured_peaks()
    k_bytes_layer = 2 * wl.rows * s * h  # this rank's K per layer (one scoring launch's bytes)
    v_bytes_layer = 2 * wl.rows * nc * h
    score_avg_ms = score_ms / max(score_n, 1)
    achieved = k_bytes_layer / (score_avg_ms * 1e-3) / 1e9
    traffic = None
    # the committed ncu capture is of the N=1 launch (same bytes per launch as
    # a batch shard; a unit shard's launch is smaller)
    for name in (("ncu_score_summary_%s.json" % args.config, "ncu_score_summary.json")
                 if shard == "batch" else ()):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                prof = json.load(f)
        except (OSError, ValueError):
            continue
        if prof.get("config") == args.config:
            traffic = prof.get("dram_bytes_per_launch")
            break
    t_k = L * k_bytes_layer / (hbm_peak * 1e9)
    t_v = L * v_bytes_layer / (h2d_bw * 1e9)
    global_batch = B * world if shard == "batch" else B
    value = global_batch / (ms * 1e-3)
    e2e_value = global_batch / (e2e_ms * 1e-3)
    # MHA: the dataflow path (scoring, the select-only consumer of each row as
    # the scoring completes it, the recall + P.V kernel under the next layer);
    # GQA: scoring, selection, recall (+ the kv-head -> q-head index expansion
    # of the outputs)
    flow = n_kv == n
    launches_per_layer = 3 + (1 if G > 1 else 0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if shard == "batch" else "strong",
        "vs_baseline": None, "dtype": "f16 storage / f32 accumulate",
        "data": ("synthetic (SeededRng SplitMix64 U[-1,1], fp16-rounded)" if args.dist == "uniform" else
                 "synthetic, peaked: K U[-0.05,0.05] with 24 hot rows in [6,8] per (batch, kv head), q U[0.5,1], "
                 "V U[-1,1], fp16-rounded"),
        "config": config_block(cfg, args, world, shard),
        "placement": {"pipeline": ("dataflow: a persistent consumer grid selects each (batch, kv head) row while "
                                   "the scoring streams the later rows (kc_consume.cu); the layer's recall + P.V runs "
                                   "on a side stream under the next layer's scoring" if flow else
                                   "stream-ordered: scoring(l) -> selection(l) on the main stream, recall(l) + P.V on "
                                   "a side stream under scoring(l+1)"),
                      "v_arena_numa_node": numa,
                      "v_arena": v_arena + " (UVM managed, host-resident: large GPU pages, no per-row page walks; "
                                 "pinned beyond the driver's managed-memory cap; KCACHE_V_ARENA=pinned forces pinned)"},
        "per_gpu_tokens_per_s": value / world,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": ("score_fast_kernel (q.K^T, TMA bulk-staged K)" if n_kv == n else
                                "score_mma_kernel (GQA q.K^T on the tensor cores, TMA bulk-staged K)"),
                     "peak_note": "a read-only K stream against the measured read+write copy rate: frac can "
                                  "exceed 1 (ncu: 86 % of the HW DRAM peak, profiles/)",
                     "algorithmic_bytes_per_launch": k_bytes_layer, "avg_launch_ms": score_avg_ms},
        "step_roofline": {"k_bytes_per_step": L * k_bytes_layer, "vsel_bytes_per_step": L * v_bytes_layer,
                          "hbm_gbs": hbm_peak, "h2d_gbs_measured": h2d_bw,
                          "h2d_note": "pinned 256 MiB cudaMemcpyAsync, best of 10, all %d rank(s) at once, "
                                      "slowest rank" % world,
                          "t_roof_sum_ms": (t_k + t_v) * 1e3, "t_roof_max_ms": max(t_k, t_v) * 1e3,
                          "frac_of_sum_roofline": (t_k + t_v) * 1e3 / ms,
                          "frac_of_max_roofline": max(t_k, t_v) * 1e3 / ms},
        "kernel_ms_per_step": {"score": all_score_ms / prof_steps,
                               ("consume (the selection, spans the scoring)" if flow else "select"):
                                   select_ms / prof_steps,
                               "recall_pv": recall_ms / prof_steps, "profiled_step_ms": prof_ms,
                               "score_only_profiled_step_ms": score_prof_ms,
                               "note": "separate profiled passes (CUDA events around launches perturb the "
                                       "pipelined overlap; ms_per_step is the unprofiled timed region)"},
        "h2d_ledger_bytes_per_layer": h2d_per_layer,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": L * b * d * 4,
                "d2h_bytes_per_step": L * (b * d * 4 + slots * nc * 8 + slots * 8), "ms_per_step": e2e_ms,
                "path": "kc_decode_topn_layers with pinned host q / outputs (TieredKVCache.prepare_topn_layers_host: buffers bound once, one C-ABI call per step)"},
        "kernel_isolated_ms_per_launch": {("consume" if flow and k == "select" else k): iso[k][0] / max(iso[k][1], 1)
                                          for k in iso},
        "serial_step_ms": serial_ms,
        "gpu_launches": launches_per_layer * L * args.steps,
        "clocks": clocks,
        "setup_s": setup_s,
        "e2e_checksum": e2e_check,
    }
    if gathered is not None:
        line["gathered_layer0_out"] = gathered
    if not args.no_engine:
        line["engine_ms_per_step"] = engine_ms
        line["engine"] = {
            "value": global_batch / (engine_ms * 1e-3), "unit": UNIT, "ms_per_step": engine_ms,
            "steps": ENGINE_STEPS, "frac_of_max_roofline": max(t_k, t_v) * 1e3 / engine_ms,
            "note": "engine-realistic decode step: one kc_decode_step per layer (append + TopN, engine.cpp:124-165), "
                    "layer l+1 waits for layer l (no cross-layer overlap); inside a layer the dataflow consumer "
                    "(MHA) or two row groups (GQA) overlap selection / recall with the scoring; NOT the headline (which pipelines the recall of layer l under the scoring of "
                    "layer l+1, the attention-only bench of SURVEY.md section 7)"}
    line["roofline"]["achieved_isolated"] = k_bytes_layer / (iso["score"][0] / max(iso["score"][1], 1) * 1e-3) / 1e9
    if full is not None:
        full_ms = full["ms_per_step"]
        line["full_kv"] = dict(full, value=global_batch / (full_ms * 1e-3), unit=UNIT,
                               kcache_over_full=full_ms / ms,
                               note="same workload with K and V in HBM, fused flash-decode kernel "
                                    "(decode_attention_full, attention.cpp:91-114): the paper's comparator")
    if world == 1 and not args.no_cpu_baseline:
        res = cpu_reference_sample(cfg, os.cpu_count() or 1, passes=1, warm=0)
        if res is not None:
            times, kind, sample = res
            cpu_val = b / statistics.mean(times)
            line["cpu_baseline"] = {"value": cpu_val, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": kind,
                                    "sample": sample}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--topn", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-kv", action="store_true", help="skip the full-KV-in-HBM comparator")
    ap.add_argument("--no-engine", action="store_true", help="skip the engine-realistic (per-layer) step")
    ap.add_argument("--tune", action="append", default=[], help="kc_set_tuning key=value")
    ap.add_argument("--dist", default="uniform", choices=["uniform", "peaked"],
                    help="synthetic K/q: U[-1,1], or near-orthogonal keys with 24 planted hot positions per row")
    ap.add_argument("--shard", default="auto", choices=["auto", "batch", "units"],
                    help="N>1: own batch per rank (weak) or (batch, kv head) units of one batch (strong)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.topn:
        cfg["top_n"] = args.topn
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
