import sys, numpy as np
sys.path.insert(0, ".")
from oracle.oracle import synth_matrix
from paper_2404_18057_b200 import kcache as kc
b, n, n_kv, h, dtype = 1, 4, 4, 128, "bf16"
s_, N_ = 20000, 300
cfg = kc.small_config(1, n * h, n, s_, kv_heads=n_kv)
cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, 1, 2, dtype))
k = synth_matrix(2, s_ * b, n_kv * h, dtype=dtype); v = synth_matrix(3, s_ * b, n_kv * h, dtype=dtype)
cache.append_kv(0, k, v); cache.offload_prefill_v(0); cache.begin_decode()
q = synth_matrix(1, b, n * h, dtype=dtype)
cache.set_tuning("consume", 0)
ref = kc.decode_attention_topn(q, cache, 0, N_, False)
cache.set_tuning("consume", 1); cache.set_tuning("keep_logits", 1)
r = kc.decode_attention_topn(q, cache, 0, N_, False)  # ls = 0
lstride = (s_ + 31) // 32 * 32
lg = cache.debug_buffer("logits0", n * lstride * 4).view(np.float32).reshape(n, lstride)
gm = cache.debug_buffer("gmax0", n * lstride // 8 * 4).view(np.float32).reshape(n, lstride // 8)
for row in range(n):
    a = set(ref.selection.indices[row].tolist()); c = set(r.selection.indices[row].tolist())
    true_gm = np.full(lstride // 8, -np.inf, np.float32)
    t = lg[row, :s_]
    ng = (s_ + 7) // 8
    tg = np.array([t[i*8:(i+1)*8].max() for i in range(ng)], np.float32)
    bad = np.nonzero(tg != gm[row, :ng])[0]
    print("row", row, "diff", sorted(a ^ c)[:6], "gmax mismatches", len(bad), bad[:10], gm[row, bad[:5]], tg[bad[:5]])
cache.close()
