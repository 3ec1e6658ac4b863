"""Development probe: what the end-to-end leg (host q in, host outputs back)
adds per output on a C3-shaped cache, 8-layer calls.
    python tools/e2e_probe.py"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2404_18057_b200 import kcache as kc
b, n, h, s, N, L, n_kv = 32, 32, 128, 16384, 128, 8, 8
cfg = kc.small_config(L, n * h, n, s, kv_heads=n_kv)
cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, L, 2, "f16"))
kb = torch.empty(s * b, n_kv * h, dtype=torch.float16, device="cuda"); vb = torch.empty_like(kb)
for l in range(L):
    kc.fill_uniform(kb, 2 + 100 * l); kc.fill_uniform(vb, 3 + 100 * l); cache.append_kv_device(l, kb, vb)
torch.cuda.synchronize(); del kb, vb
for l in range(L): cache.offload_prefill_v(l)
cache.begin_decode()
qs = []
for l in range(L):
    q = torch.empty(b, n * h, dtype=torch.float16, device="cuda"); kc.fill_uniform(q, 1 + 100 * l); qs.append(q.float())
slots = b * n
qh = [torch.empty(b, n * h, dtype=torch.float32, pin_memory=True) for _ in range(L)]
for i in range(L): qh[i].copy_(qs[i])
qh_np = [t.numpy() for t in qh]
def mk(keys):
    d = []
    for _ in range(L):
        o = {}
        if "out" in keys: o["out"] = torch.empty(b, n * h, dtype=torch.float32, pin_memory=True).numpy()
        if "indices" in keys: o["indices"] = torch.empty(slots, N, dtype=torch.int32, pin_memory=True).numpy()
        if "weights" in keys: o["weights"] = torch.empty(slots, N, dtype=torch.float32, pin_memory=True).numpy()
        if "dropped" in keys: o["dropped"] = torch.empty(slots, dtype=torch.float64, pin_memory=True).numpy()
        d.append(o)
    return d
stream = torch.cuda.Stream()
outs_d = [{"out": torch.empty(b, n * h, device="cuda")} for _ in range(L)]
def dev():
    cache.decode_topn_layers_device(list(range(L)), qs, N, outs_d, stream=stream, want_selection=False); torch.cuda.synchronize()
def timeit(fn, reps=10):
    for _ in range(3): fn()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    return (time.perf_counter() - t0) * 1e6 / reps / L
print("device (sync each call)", round(timeit(dev), 1))
for keys in (("out",), ("out", "dropped"), ("out", "weights"), ("out", "indices"), ("out", "indices", "weights", "dropped")):
    call = cache.prepare_topn_layers_host(list(range(L)), qh_np, N, mk(keys))
    print(keys, round(timeit(call), 1), flush=True)
cache.close()
