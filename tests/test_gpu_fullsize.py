"""Full-size parity: EVERY (batch, kv head) slot of one layer of each
BASELINE.json config shape against the CPU oracle (oracle/kcache_oracle.c,
pinned to the reference by tests/test_oracle_golden.py), under the rules of
tests/parity.py.

K and V are generated on the GPU with kc_fill_uniform (bit-identical to the
SeededRng stream: test_gpu_parity.py::test_fill_uniform_matches_seeded_rng),
copied back once, and sliced per slot for the oracle. Shapes:
* C2: LLaMA2-7B, b=8, 32 x 128, s=32k, N=128 -- uniform and "peaked" keys
  (U[-0.05, 0.05] with planted hot positions, verify.cpp:417-431);
* C3: LLaMA3-8B GQA 32/8, b=32, s=16k, N=128 (reports the epsilon-window
  swap count of the GQA selection key);
* C4: LLaMA2-13B, 40 x 128 (d=5120), b=7, s=32k, N=128;
* C5 corners: 128k x N in {32, 128, 512} (MHA: the dataflow consumer's
  streamed selection; GQA at 128k: the global-key selection kernel), and
  4k x N=512.
"""
import numpy as np
import pytest

from oracle.oracle import synth_matrix
from tests.parity import check_group

pytestmark = pytest.mark.gpu


def _layer(kc, b, n, n_kv, h, s, N, dtype="f16", dist="uniform", renorm=False, seeds=(2, 3, 1)):
    import torch
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16}[dtype]
    cfg = kc.small_config(1, n * h, n, s, kv_heads=n_kv)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, 1, 2, dtype))
    k = torch.empty(s * b, n_kv * h, dtype=tdt, device="cuda")
    v = torch.empty_like(k)
    kc.fill_uniform(v, seeds[1])
    if dist == "peaked":
        # keys nearly orthogonal to q except a few planted hot positions per
        # (batch, kv head), each a constant row in [6, 8] (verify.cpp:417-431)
        kc.fill_uniform(k, seeds[0], lo=-0.05, hi=0.05)
        rng = np.random.default_rng(seeds[0])
        kv3 = k.view(s, b, n_kv, h)
        for bb in range(b):
            for kvh in range(n_kv):
                hot = rng.choice(s, size=24, replace=False)
                vals = torch.tensor(rng.uniform(6.0, 8.0, size=24), dtype=tdt, device="cuda")
                kv3[torch.as_tensor(hot, device="cuda"), bb, kvh, :] = vals[:, None]
        q = synth_matrix(seeds[2], b, n * h, lo=0.5, hi=1.0, dtype=dtype)
    else:
        kc.fill_uniform(k, seeds[0])
        q = synth_matrix(seeds[2], b, n * h, dtype=dtype)
    cache.append_kv_device(0, k, v)
    torch.cuda.synchronize()
    k_host = k.float().cpu().numpy()  # exact widening of the stored 16-bit values
    v_host = v.float().cpu().numpy()
    del k, v
    cache.offload_prefill_v(0)
    cache.begin_decode()
    res = kc.decode_attention_topn(q, cache, 0, N, renorm)
    cache.close()
    return res, q, k_host, v_host


def _check_all(oracle, res, q, k_host, v_host, b, n, n_kv, h, s, N, renorm):
    """Every (batch, kv head) group; returns (epsilon-window swaps, groups)."""
    G = n // n_kv
    nc = min(N, s)
    assert res.h2d_bytes == 2 * b * n_kv * nc * h
    swaps = 0
    for bb in range(b):
        for kvh in range(n_kv):
            ks = k_host[bb::b, kvh * h:(kvh + 1) * h]
            vs = v_host[bb::b, kvh * h:(kvh + 1) * h]
            heads = [kvh * G + g for g in range(G)]
            qg = q[bb].reshape(n, h)[heads]
            o_out, o_idx, o_w, o_dr = oracle.decode_topn_group(qg, ks, vs, N, renorm)
            probs = np.stack([oracle.head_weights(qg[g], ks) for g in range(G)])
            # logit magnitude of the group (tests/parity.py: fp32 rounding of
            # large logits in another summation order)
            mag = float((np.abs(ks) @ np.abs(qg).T).max()) / np.sqrt(h)
            slots = [bb * n + hd for hd in heads]
            for sl in slots[1:]:
                np.testing.assert_array_equal(res.selection.indices[sl], res.selection.indices[slots[0]])
            swaps += check_group(res.selection.indices[slots[0]], res.selection.weights[slots],
                                 res.selection.dropped_mass[slots], res.out[bb].reshape(n, h)[heads], probs, vs,
                                 N, renorm, ora_idx=o_idx, ora_out=o_out, logit_mag=mag)
    return swaps, b * n_kv


CASES = {
    # name: (b, n, n_kv, s, N, dtype, dist, renorm)
    "c2": (8, 32, 32, 32768, 128, "f16", "uniform", False),
    "c2-peaked": (8, 32, 32, 32768, 128, "f16", "peaked", False),
    "c2-renorm-bf16": (8, 32, 32, 32768, 128, "bf16", "uniform", True),
    "c3": (32, 32, 8, 16384, 128, "f16", "uniform", False),
    "c3-peaked": (32, 32, 8, 16384, 128, "f16", "peaked", False),
    "c4-13b": (7, 40, 40, 32768, 128, "f16", "uniform", False),
    "c5-128k-N32": (1, 32, 32, 131072, 32, "f16", "uniform", False),
    "c5-128k-N128": (1, 32, 32, 131072, 128, "f16", "uniform", False),
    "c5-128k-N512": (1, 32, 32, 131072, 512, "f16", "uniform", False),
    "c5-128k-N128-peaked": (1, 32, 32, 131072, 128, "f16", "peaked", False),
    "c5-128k-gqa-N128": (1, 32, 8, 131072, 128, "f16", "uniform", False),
    "c5-4k-N512": (8, 32, 32, 4096, 512, "f16", "uniform", False),
}


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name", list(CASES))
def test_full_layer_every_slot(kc, oracle, name):
    b, n, n_kv, s, N, dtype, dist, renorm = CASES[name]
    h = 128
    res, q, k_host, v_host = _layer(kc, b, n, n_kv, h, s, N, dtype, dist, renorm)
    swaps, groups = _check_all(oracle, res, q, k_host, v_host, b, n, n_kv, h, s, N, renorm)
    print(f"\n[{name}] groups={groups} epsilon-window index swaps={swaps} "
          f"mean dropped={float(np.mean(res.selection.dropped_mass)):.6f}")
    # a swap is legal only inside the epsilon window (check_group asserts
    # that); they must stay rare
    assert swaps <= max(2, groups // 8)


def test_score_observer_rows(kc, oracle):
    """ScoreObserver (attention.hpp:34-35, called per slot at
    attention.cpp:137-139): the full softmax row of every (batch, head), in
    slot order, equals the oracle's head_weights within the parity tolerance
    and does not change the TopN result."""
    b, n, n_kv, h, s, N = 2, 8, 4, 128, 3000, 64
    G = n // n_kv
    cfg = kc.small_config(1, n * h, n, s, kv_heads=n_kv)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, 1, 2, "f16"))
    k = synth_matrix(2, s * b, n_kv * h)
    v = synth_matrix(3, s * b, n_kv * h)
    q = synth_matrix(1, b, n * h)
    cache.append_kv(0, k, v)
    cache.offload_prefill_v(0)
    cache.begin_decode()
    seen = []

    def observer(bi, head, w):
        seen.append((bi, head, np.array(w, copy=True)))

    with_obs = kc.decode_attention_topn(q, cache, 0, N, False, observer=observer)
    plain = kc.decode_attention_topn(q, cache, 0, N, False)
    assert [(x[0], x[1]) for x in seen] == [(bi, hd) for bi in range(b) for hd in range(n)]
    for bi, hd, w in seen:
        ks = k[bi::b, (hd // G) * h:(hd // G + 1) * h]
        want = oracle.head_weights(q[bi, hd * h:(hd + 1) * h], ks)
        assert w.shape == (s,)
        np.testing.assert_allclose(w, want, rtol=1e-4, atol=1e-12)
        assert abs(float(w.astype(np.float64).sum()) - 1.0) < 1e-4
        # the observer's row and the selection agree: weights are the row at the indices
        sl = bi * n + hd
        np.testing.assert_array_equal(with_obs.selection.weights[sl], w[with_obs.selection.indices[sl]])
    np.testing.assert_array_equal(with_obs.out, plain.out)
    np.testing.assert_array_equal(with_obs.selection.indices, plain.selection.indices)
    full_seen = []
    kc.decode_attention_full(q, cache, 0, observer=lambda bi, hd, w: full_seen.append((bi, hd)))
    assert full_seen == [(bi, hd) for bi in range(b) for hd in range(n)]
    cache.close()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("n_kv", [32, 8], ids=["c2", "c3"])
def test_full_size_pipelined_layers_equal_single_calls(kc, n_kv):
    """The bench's multi-layer call at full size -- MHA: the select-only
    consumer + the recall kernel under the next layer's scoring; GQA: the
    stream-ordered path with the cached row selection -- equals single-layer
    calls (the recalling consumer; MHA checked against the oracle above) and
    stream-ordered single-layer calls bit for bit, over 3 layers (both scoring
    slots, the selection ring). Repeated multi-layer calls stay bit-identical:
    the scoring beside a running recall once read an overwritten ring stage
    (score_mma_kernel released stages before its shared-memory loads
    returned: an 8-position tile of wrong logits every few C3 layers)."""
    import torch
    b, n, h, s, N, L = (8, 32, 128, 32768, 128, 3) if n_kv == 32 else (32, 32, 128, 16384, 128, 3)
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
    nc = min(N, s)

    def outs():
        return [{"out": torch.full((b, n * h), float("nan"), device="cuda"),
                 "indices": torch.empty(b * n, nc, dtype=torch.int32, device="cuda"),
                 "weights": torch.empty(b * n, nc, device="cuda"),
                 "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")} for _ in range(L)]
    stream = torch.cuda.Stream()
    multi, single = outs(), outs()
    cache.decode_topn_layers_device(list(range(L)), qs, N, multi, stream=stream)
    for l in range(L):
        cache.decode_topn_layers_device([l], [qs[l]], N, [single[l]], stream=stream)
    cache.set_tuning("consume", 0)
    ordered = outs()
    for l in range(L):
        cache.decode_topn_layers_device([l], [qs[l]], N, [ordered[l]], stream=stream)
    cache.set_tuning("consume", 1)
    torch.cuda.synchronize()
    for l in range(L):
        for key in ("out", "indices", "weights", "dropped"):
            assert torch.equal(multi[l][key], single[l][key]), (l, key)
            assert torch.equal(multi[l][key], ordered[l][key]), (l, key)
    for rep in range(6):
        again = outs()
        cache.decode_topn_layers_device(list(range(L)), qs, N, again, stream=stream)
        torch.cuda.synchronize()
        for l in range(L):
            for key in ("out", "indices", "weights", "dropped"):
                assert torch.equal(multi[l][key], again[l][key]), (rep, l, key)
    # the dataflow consumer forced on every shape (GQA included), multi- and
    # single-layer calls
    cache.set_tuning("consume", 2)
    forced_multi, forced_single = outs(), outs()
    cache.decode_topn_layers_device(list(range(L)), qs, N, forced_multi, stream=stream)
    for l in range(L):
        cache.decode_topn_layers_device([l], [qs[l]], N, [forced_single[l]], stream=stream)
    cache.set_tuning("consume", 1)
    torch.cuda.synchronize()
    for l in range(L):
        for key in ("out", "indices", "weights", "dropped"):
            assert torch.equal(multi[l][key], forced_multi[l][key]), ("forced multi", l, key)
            assert torch.equal(multi[l][key], forced_single[l][key]), ("forced single", l, key)
    cache.close()
