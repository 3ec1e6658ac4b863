import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle.oracle import synth_matrix
from paper_2404_18057_b200 import kcache as kc
from tests.test_gpu_parity import build_cache
fails = 0
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    b, n, n_kv, h, s, N, L = 2, 8, 4, 128, 600, 32, 3
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", n_layers=L)
    qs = [torch.from_numpy(synth_matrix(20 + l, b, n * h)).pin_memory().numpy() for l in range(L)]
    singles = [kc.decode_attention_topn(qs[l], cache, l, N, False) for l in range(L)]
    nc = min(N, s)
    def pinned(shape, dt):
        return torch.zeros(shape, dtype=dt).pin_memory().numpy()
    outs = [{"out": pinned((b, n * h), torch.float32), "indices": pinned((b * n, nc), torch.int32).view(np.uint32),
             "weights": np.zeros((b * n, nc), np.float32), "dropped": pinned(b * n, torch.float64)} for _ in range(L)]
    call = cache.prepare_topn_layers_host(list(range(L)), qs, N, outs)
    for rep in range(3):
        for o in outs:
            for a in o.values():
                a.fill(0)
        call()
        for l in range(L):
            for key, ref in (("out", singles[l].out), ("indices", singles[l].selection.indices),
                             ("weights", singles[l].selection.weights), ("dropped", singles[l].selection.dropped_mass)):
                got = outs[l][key]
                if not np.array_equal(got, ref):
                    fails += 1
                    bad = np.argwhere(got.reshape(got.shape[0], -1) != np.asarray(ref).reshape(got.shape[0], -1))
                    print("trial", trial, "rep", rep, "layer", l, key, "n_bad", len(bad), "first", bad[:3].tolist(),
                          "got", got.reshape(-1)[:4], "ref", np.asarray(ref).reshape(-1)[:4], flush=True)
    cache.close()
print("fails", fails)
