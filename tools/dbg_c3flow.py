"""Development probe (race detector): repeated C3-shaped multi-layer calls
must leave bit-identical logits (keep_logits 1, kc_debug_read "logits0").
Found the score_mma_kernel ring-stage race fixed in r02."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_18057_b200 import kcache as kc

b, n, h, s, N, L, n_kv = 32, 32, 128, 16384, 128, 3, 8
cfg = kc.small_config(L, n * h, n, s, kv_heads=n_kv)
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
    q = torch.empty(b, n * h, dtype=torch.float16, device="cuda")
    kc.fill_uniform(q, 1 + 100 * l)
    qs.append(q.float())
nc = N
def outs():
    return [{"out": torch.full((b, n * h), float("nan"), device="cuda"),
             "indices": torch.empty(b * n, nc, dtype=torch.int32, device="cuda"),
             "weights": torch.empty(b * n, nc, device="cuda"),
             "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")} for _ in range(L)]
stream = torch.cuda.Stream()
def single(consume, sync_each=False):
    o = outs()
    cache.set_tuning("consume", consume)
    for l in range(L):
        cache.decode_topn_layers_device([l], [qs[l]], N, [o[l]], stream=stream)
        if sync_each: torch.cuda.synchronize()
    torch.cuda.synchronize()
    cache.set_tuning("consume", 1)
    return o
def multi():
    o = outs()
    cache.decode_topn_layers_device(list(range(L)), qs, N, o, stream=stream)
    torch.cuda.synchronize()
    return o
def cmp(tag, a, bb):
    for l in range(L):
        d = {k: int((a[l][k] != bb[l][k]).reshape(a[l][k].shape[0], -1).any(1).sum()) for k in ("out", "indices", "weights", "dropped")}
        print(tag, "layer", l, d, flush=True)
import numpy as np
cache.set_tuning("keep_logits", 1)
LB = b * n * 16384 * 4
def snap():
    lg = cache.debug_buffer("logits0", LB).view(np.float32)
    return lg.copy()
def trial(tag, tune, reps=8):
    for k, v in tune.items(): cache.set_tuning(k, v)
    multi(); base = snap()
    res = []
    for t in range(reps):
        multi(); cur = snap()
        res.append(int((cur != base).sum()))
    for k in tune: cache.set_tuning(k, DEF[k])
    print(tag, tune, res, flush=True)
DEF = {"pipeline": 1, "recall_dbg": 0, "score_mma": 1}
trial("default", {})
trial("serial", {"pipeline": 0})
trial("recall without loads", {"recall_dbg": 1})
trial("tcgen05", {"score_mma": 3})
cache.close()
