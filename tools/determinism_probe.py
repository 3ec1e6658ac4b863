"""Development probe (race detector): repeated full-size decode calls on one
cache must return bit-identical outputs, in every orchestration.
    python tools/determinism_probe.py [c2|c3] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_18057_b200 import kcache as kc  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
b, n, h, s, N, L, n_kv = (8, 32, 128, 32768, 128, 3, 32) if shape == "c2" else (32, 32, 128, 16384, 128, 3, 8)
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
stream = torch.cuda.Stream()


def outs():
    return [{"out": torch.full((b, n * h), float("nan"), device="cuda"),
             "indices": torch.empty(b * n, N, dtype=torch.int32, device="cuda"),
             "weights": torch.empty(b * n, N, device="cuda"),
             "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")} for _ in range(L)]


def multi():
    o = outs()
    cache.decode_topn_layers_device(list(range(L)), qs, N, o, stream=stream)
    torch.cuda.synchronize()
    return o


def single():
    o = outs()
    for l in range(L):
        cache.decode_topn_layers_device([l], [qs[l]], N, [o[l]], stream=stream)
    torch.cuda.synchronize()
    return o


ref = None
MODES = (("multi", {}, multi), ("single", {}, single), ("multi ordered", {"consume": 0}, multi),
         ("single ordered", {"consume": 0}, single), ("multi dataflow", {"consume": 2}, multi),
         ("single dataflow", {"consume": 2}, single), ("multi tma recall", {"recall_tma": 1}, multi),
         ("single tma recall ordered", {"recall_tma": 1, "consume": 0}, single))
if os.environ.get("TC"):  # tcgen05 scoring rounds differently: its own reference
    MODES = (("multi tcgen05", {"score_mma": 3}, multi), ("single tcgen05", {"score_mma": 3}, single),
             ("multi tcgen05 persistent", {"score_mma": 3, "tc_grid": 2}, multi))
DEFAULT = {"consume": 1, "recall_tma": 0, "score_mma": 1, "tc_grid": 0}
for mode, tune, fn in MODES:
    for k, v in tune.items():
        cache.set_tuning(k, v)
    bad = []
    for _ in range(reps):
        o = fn()
        if ref is None:
            ref = o
        bad.append(sum(int((o[l][key] != ref[l][key]).reshape(o[l][key].shape[0], -1).any(1).sum())
                       for l in range(L) for key in ("out", "indices", "weights", "dropped")))
    for k in tune:
        cache.set_tuning(k, DEFAULT[k])
    print(shape, mode, bad, flush=True)
cache.close()
