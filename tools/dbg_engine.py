"""Development probe: the engine step (kc_decode_step per layer) vs single-layer
decode calls, dataflow (consume 2) vs stream-ordered, on a C3-shaped cache:
the dispatch-order sensitivity of the GQA dataflow.
    EXTRA=200 python tools/dbg_engine.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_18057_b200 import kcache as kc

b, n, h, s, N, L, n_kv = int(os.environ.get('B', 32)), 32, 128, int(os.environ.get('S', 16384)), 128, 8, int(os.environ.get('KV', 8))
cfg = kc.small_config(L, n * h, n, s + int(os.environ.get('EXTRA', '64')), kv_heads=n_kv)
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
q16 = [torch.empty(b, n * h, dtype=torch.float16, device="cuda") for _ in range(L)]
kv16 = [torch.empty(2, b, n_kv * h, dtype=torch.float16, device="cuda") for _ in range(L)]
for l in range(L):
    kc.fill_uniform(q16[l], 900 + l)
    kc.fill_uniform(kv16[l], 950 + l)
out = torch.empty(b, n * h, dtype=torch.float32, device="cuda")
nc = N
o1 = {"out": out}
stream = torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps): fn()
    e1.record(stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / L * 1e3
def step():
    for l in range(L):
        cache.decode_step_device(l, q16[l], kv16[l][0], kv16[l][1], out, N, stream=stream)
def topn():
    for l in range(L):
        cache.decode_topn_layers_device([l], [q16[l]], N, [o1], stream=stream, want_selection=False)
q32 = [x.float() for x in q16]
def topn32():
    for l in range(L):
        cache.decode_topn_layers_device([l], [q32[l]], N, [o1], stream=stream, want_selection=False)
outs = [{"out": torch.empty(b, n * h, device="cuda"), "indices": torch.empty(b * n, nc, dtype=torch.int32, device="cuda"),
         "weights": torch.empty(b * n, nc, device="cuda"), "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")} for _ in range(L)]
def topn_sel():
    for l in range(L):
        cache.decode_topn_layers_device([l], [q32[l]], N, [outs[l]], stream=stream)
def topn_sep():
    for l in range(L):
        cache.decode_topn_layers_device([l], [q32[l]], N, [{"out": outs[l]["out"]}], stream=stream, want_selection=False)
def topn_drop():
    for l in range(L):
        cache.decode_topn_layers_device([l], [q32[l]], N, [{"out": outs[l]["out"], "dropped": outs[l]["dropped"]}], stream=stream)
def gaps(fn):
    fn(); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * L)]
    import time
    h = []
    for l in range(L):
        ev[2 * l].record(stream)
        t0 = time.perf_counter()
        cache.decode_topn_layers_device([l], [q32[l]], N, [{"out": outs[l]["out"]}], stream=stream, want_selection=False)
        h.append((time.perf_counter() - t0) * 1e6)
        ev[2 * l + 1].record(stream)
    torch.cuda.synchronize()
    inside = [ev[2 * l].elapsed_time(ev[2 * l + 1]) * 1e3 for l in range(L)]
    between = [ev[2 * l + 1].elapsed_time(ev[2 * l + 2]) * 1e3 for l in range(L - 1)]
    return [round(x, 1) for x in inside], [round(x, 1) for x in between], [round(x, 1) for x in h]
def app():
    for l in range(L):
        cache.append_kv_device(l, kv16[l][0], kv16[l][1], stream=stream)
def app_topn():
    for l in range(L):
        cache.append_kv_device(l, kv16[l][0], kv16[l][1], stream=stream)
        cache.decode_topn_layers_device([l], [q32[l]], N, [{"out": outs[l]["out"]}], stream=stream, want_selection=False)
def app_topn16():
    for l in range(L):
        cache.append_kv_device(l, kv16[l][0], kv16[l][1], stream=stream)
        cache.decode_topn_layers_device([l], [q16[l]], N, [{"out": outs[l]["out"]}], stream=stream, want_selection=False)
def step32():
    for l in range(L):
        cache.decode_step_device(l, q32[l], kv16[l][0].float(), kv16[l][1].float(), out, N, stream=stream)
cache.set_tuning("consume", 0)
r = [round(t(f, reps=2), 1) for f in (app_topn, app_topn16, step)]
print("stream-ordered", r, flush=True)
cache.set_tuning("consume", 2)
for ctas in [int(x) for x in os.environ.get('CTAS', '0').split(',')]:
    cache.set_tuning("consume_ctas", ctas)
    r = [round(t(f, reps=2), 1) for f in (app_topn, app_topn16, step)]
    print("consume 2 ctas", ctas, "append+topn(q32) / append+topn(q16) / decode_step, us per layer", r, flush=True)
cache.close()
