"""Parity of the CUDA decode path against the CPU oracle (and the reference).

Inputs are SeededRng streams (proj/core/include/kcache/rng.hpp:13-26) rounded
to the storage dtype, fed identically to both sides. Rules: tests/parity.py.
"""
import numpy as np
import pytest

from oracle.oracle import Reference, synth, synth_matrix, synth_slot_rows
from tests.parity import check_group

pytestmark = pytest.mark.gpu


def build_cache(kc, b, n, n_kv, h, s, dtype, resident=0, max_seq=None, n_layers=1, seeds=(2, 3)):
    cfg = kc.small_config(n_layers, n * h, n, max_seq or max(s, 1), kv_heads=n_kv)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(resident, n_layers, 2, dtype))
    ks, vs = [], []
    for layer in range(n_layers):
        k = synth_matrix(seeds[0] + 100 * layer, s * b, n_kv * h, dtype=dtype)
        v = synth_matrix(seeds[1] + 100 * layer, s * b, n_kv * h, dtype=dtype)
        cache.append_kv(layer, k, v)
        cache.offload_prefill_v(layer)
        ks.append(k)
        vs.append(v)
    cache.begin_decode()
    return cache, ks, vs


def slot_rows(m, b, batch, kvh, h):
    """[s][h] rows of (batch row b, kv head kvh) from a position-major matrix."""
    return m[b::batch, kvh * h:(kvh + 1) * h]


def compare_all(oracle, res, q, k, v, b_, n, n_kv, h, s, top_n, renorm, ordered=True):
    G = n // n_kv
    o_out, o_idx, o_w, o_dr = oracle.decode_topn(q, k, v, b_, n, n_kv, h, s, top_n, renorm, ordered)
    swaps = 0
    for b in range(b_):
        for kvh in range(n_kv):
            ks = slot_rows(k, b, b_, kvh, h)
            vs = slot_rows(v, b, b_, kvh, h)
            heads = [kvh * G + g for g in range(G)]
            probs = np.stack([oracle.head_weights(q[b, hd * h:(hd + 1) * h], ks) for hd in heads])
            slots = [b * n + hd for hd in heads]
            for sl in slots[1:]:
                np.testing.assert_array_equal(res.selection.indices[sl], res.selection.indices[slots[0]])
            swaps += check_group(res.selection.indices[slots[0]], res.selection.weights[slots],
                                 res.selection.dropped_mass[slots],
                                 res.out[b].reshape(n, h)[heads], probs, vs, top_n, renorm,
                                 ora_idx=o_idx[slots[0]], ora_out=o_out[b].reshape(n, h)[heads])
    return swaps


CASES = [
    # b, n, n_kv, h, s, N, dtype
    (1, 4, 4, 16, 50, 8, "f32"),       # generic scoring path
    (2, 4, 4, 128, 300, 32, "f16"),    # TMA path, MHA
    (2, 8, 4, 128, 257, 16, "f16"),    # GQA G=2, ragged tail stage
    (1, 8, 2, 128, 1000, 64, "bf16"),  # GQA G=4, bf16
    (2, 16, 2, 128, 700, 128, "f16"),  # GQA G=8
    (3, 2, 2, 8, 33, 40, "f32"),       # N > s clamps
    (1, 1, 1, 1, 4, 2, "f32"),         # h = 1
    (1, 4, 4, 128, 1, 4, "f16"),       # single position
    (2, 4, 4, 64, 129, 1, "bf16"),     # N = 1, generic h
    (1, 4, 4, 128, 5000, 2000, "f16"),  # N > 1024: the full radix pass, 2000 survivors
    (1, 4, 2, 128, 3000, 3000, "bf16"),  # N = s (GQA): everything selected
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
@pytest.mark.parametrize("renorm", [False, True])
@pytest.mark.parametrize("select_global", [0, 1])
def test_random_cases_vs_oracle(kc, oracle, case, renorm, select_global):
    b, n, n_kv, h, s, N, dtype = case
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, dtype)
    cache.set_tuning("select_global", select_global)
    q = synth_matrix(1, b, n * h, dtype=dtype)
    res = kc.decode_attention_topn(q, cache, 0, N, renorm)
    compare_all(oracle, res, q, ks[0], vs[0], b, n, n_kv, h, s, N, renorm)
    nc = min(N, s)
    assert res.h2d_bytes == 2 * b * n_kv * nc * h
    assert cache.h2d_bytes_total() == res.h2d_bytes


def test_reverse_accumulation_fault_hook(kc, oracle):
    b, n, h, s, N = 2, 4, 128, 200, 64
    cache, ks, vs = build_cache(kc, b, n, n, h, s, "f16")
    q = synth_matrix(1, b, n * h)
    fwd = kc.decode_attention_topn(q, cache, 0, N, False)
    rev = kc.decode_attention_topn(q, cache, 0, N, False, ordered_accumulation=False)
    np.testing.assert_array_equal(fwd.selection.indices, rev.selection.indices)
    compare_all(oracle, rev, q, ks[0], vs[0], b, n, n, h, s, N, False, ordered=False)
    # the hook changes the summation order only
    assert not np.array_equal(fwd.out, rev.out)
    np.testing.assert_allclose(fwd.out, rev.out, rtol=1e-4, atol=1e-6)


def test_c1_against_the_reference(kc, oracle):
    """Config 1: LLaMA2-7B single layer, b=1, 32x128, 4k, N=128 -- GPU vs the
    unmodified reference (oracle/_ref) and the restatement on identical inputs."""
    b, n, h, s, N = 1, 32, 128, 4096, 128
    cache, ks, vs = build_cache(kc, b, n, n, h, s, "f16")
    q = synth_matrix(1, b, n * h)
    res = kc.decode_attention_topn(q, cache, 0, N, False)
    swaps = compare_all(oracle, res, q, ks[0], vs[0], b, n, n, h, s, N, False)
    assert swaps <= 2
    if Reference.available():
        r_out, r_idx, r_w, r_dr, r_h2d = Reference().decode_topn(q, ks[0], vs[0], b, n, h, s, N)
        assert r_h2d == res.h2d_bytes == 2 * b * n * N * h
        same = sum(np.array_equal(r_idx[i], res.selection.indices[i]) for i in range(n))
        assert same >= n - 2
        np.testing.assert_allclose(res.selection.dropped_mass, r_dr, atol=1e-6)


def test_pipelined_layers_equal_single_calls(kc):
    b, n, n_kv, h, s, N, L = 2, 8, 4, 128, 600, 32, 4
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", n_layers=L)
    qs = [synth_matrix(10 + l, b, n * h) for l in range(L)]
    singles = [kc.decode_attention_topn(qs[l], cache, l, N, False) for l in range(L)]
    nc = min(N, s)
    outs = [{"out": np.zeros((b, n * h), np.float32), "indices": np.zeros((b * n, nc), np.uint32),
             "weights": np.zeros((b * n, nc), np.float32), "dropped": np.zeros(b * n, np.float64)}
            for _ in range(L)]
    info = cache.decode_topn_layers_host(list(range(L)), qs, N, outs)
    for l in range(L):
        np.testing.assert_array_equal(outs[l]["out"], singles[l].out)
        np.testing.assert_array_equal(outs[l]["indices"], singles[l].selection.indices)
        np.testing.assert_array_equal(outs[l]["weights"], singles[l].selection.weights)
        np.testing.assert_array_equal(outs[l]["dropped"], singles[l].selection.dropped_mass)
        assert info[l] == (nc, 2 * b * n_kv * nc * h)


def test_prepared_host_call_pinned_and_pageable(kc):
    """The bench's end-to-end call: buffers bound once (prepare_topn_layers_host),
    called repeatedly; pinned outputs take the direct D2H, a pageable one the
    staging copy -- bit-identical to single-layer calls every time."""
    import torch
    b, n, n_kv, h, s, N, L = 2, 8, 4, 128, 600, 32, 3
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", n_layers=L)
    qs = [torch.from_numpy(synth_matrix(20 + l, b, n * h)).pin_memory().numpy() for l in range(L)]
    singles = [kc.decode_attention_topn(qs[l], cache, l, N, False) for l in range(L)]
    nc = min(N, s)

    def pinned(shape, dt):
        return torch.zeros(shape, dtype=dt).pin_memory().numpy()
    outs = [{"out": pinned((b, n * h), torch.float32), "indices": pinned((b * n, nc), torch.int32).view(np.uint32),
             "weights": np.zeros((b * n, nc), np.float32), "dropped": pinned(b * n, torch.float64)}
            for _ in range(L)]
    call = cache.prepare_topn_layers_host(list(range(L)), qs, N, outs)
    for _ in range(3):
        for o in outs:
            for a in o.values():
                a.fill(0)
        info = call()
        for l in range(L):
            np.testing.assert_array_equal(outs[l]["out"], singles[l].out)
            np.testing.assert_array_equal(outs[l]["indices"], singles[l].selection.indices)
            np.testing.assert_array_equal(outs[l]["weights"], singles[l].selection.weights)
            np.testing.assert_array_equal(outs[l]["dropped"], singles[l].selection.dropped_mass)
            assert info[l] == (nc, 2 * b * n_kv * nc * h)


def test_repeated_decode_and_decode_appends(kc, oracle):
    """Decode is idempotent across calls, and K/V appended in the
    decode phase (engine.cpp:143: append before attention) are scored and
    recalled; the appended V goes to the host arena with a D2H ledger event."""
    b, n, n_kv, h, s, N = 2, 8, 4, 128, 700, 64
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", max_seq=s + 8)
    q = synth_matrix(1, b, n * h)
    first = kc.decode_attention_topn(q, cache, 0, N, False)
    for _ in range(4):
        again = kc.decode_attention_topn(q, cache, 0, N, False)
        np.testing.assert_array_equal(again.out, first.out)
        np.testing.assert_array_equal(again.selection.indices, first.selection.indices)
    k, v = ks[0], vs[0]
    d2h0 = cache.d2h_bytes_total()
    for step in range(3):
        knew = synth_matrix(50 + step, b, n_kv * h)
        vnew = synth_matrix(60 + step, b, n_kv * h)
        knew[:, :h] = 4.0 * np.float32(np.float16(0.25))  # make the new position attractive for kv head 0
        cache.append_kv(0, knew, vnew)
        k = np.concatenate([k, knew])
        v = np.concatenate([v, vnew])
        assert cache.d2h_bytes_total() - d2h0 == 2 * b * n_kv * h * (step + 1)
        res = kc.decode_attention_topn(q, cache, 0, N, False)
        compare_all(oracle, res, q, k, v, b, n, n_kv, h, s + step + 1, N, False)
        res2 = kc.decode_attention_topn(q, cache, 0, N, False)
        np.testing.assert_array_equal(res2.out, res.out)


def test_resident_layer_reads_hbm_v(kc, oracle):
    b, n, h, s, N = 2, 4, 128, 300, 16
    cache, ks, vs = build_cache(kc, b, n, n, h, s, "f16", resident=1, n_layers=2)
    q = synth_matrix(1, b, n * h)
    res0 = kc.decode_attention_topn(q, cache, 0, N, True)
    res1 = kc.decode_attention_topn(q, cache, 1, N, True)
    assert res0.h2d_bytes == 0 and res1.h2d_bytes == 2 * b * n * N * h
    compare_all(oracle, res0, q, ks[0], vs[0], b, n, n, h, s, N, True)
    compare_all(oracle, res1, q, ks[1], vs[1], b, n, n, h, s, N, True)


@pytest.mark.parametrize("case", [(2, 4, 4, 128, 500, "f16"), (1, 8, 2, 128, 333, "bf16"), (2, 4, 4, 16, 77, "f32")])
def test_decode_full_vs_oracle(kc, oracle, case):
    b, n, n_kv, h, s, dtype = case
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, dtype, resident=1)
    q = synth_matrix(1, b, n * h, dtype=dtype)
    got = kc.decode_attention_full(q, cache, 0)
    want = oracle.decode_full(q, ks[0], vs[0], b, n, n_kv, h, s)
    np.testing.assert_allclose(got, want, rtol=1e-3, atol=1e-6)
    # TopN with N >= s equals full attention (attention.hpp:56-62), within tolerance on the GPU
    topn = kc.decode_attention_topn(q, cache, 0, s + 7, False)
    np.testing.assert_allclose(topn.out, got, rtol=1e-3, atol=1e-6)
    assert np.all(np.abs(topn.selection.dropped_mass) <= 1e-6)
    np.testing.assert_array_equal(topn.selection.indices, np.tile(np.arange(s, dtype=np.uint32), (b * n, 1)))


def _full_size(kc, oracle, b, n, n_kv, s, N, samples, seed_q=1, seeds=(2, 3)):
    import torch
    h = 128
    cfg = kc.small_config(1, n * h, n, s, kv_heads=n_kv)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, 1, 2, "f16"))
    rows = s * b
    k = torch.empty(rows, n_kv * h, dtype=torch.float16, device="cuda")
    kc.fill_uniform(k, seeds[0])
    v = torch.empty_like(k)
    kc.fill_uniform(v, seeds[1])
    cache.append_kv_device(0, k, v)
    torch.cuda.synchronize()
    del k, v
    cache.offload_prefill_v(0)
    cache.begin_decode()
    q = synth_matrix(seed_q, b, n * h)
    res = kc.decode_attention_topn(q, cache, 0, N, False)
    assert res.h2d_bytes == 2 * b * n_kv * N * h
    G = n // n_kv
    rng = np.random.default_rng(0)
    swaps = 0
    for _ in range(samples):
        bb = int(rng.integers(b))
        kvh = int(rng.integers(n_kv))
        ks = synth_slot_rows(seeds[0], s, b, n_kv * h, bb, kvh * h, h)
        vs = synth_slot_rows(seeds[1], s, b, n_kv * h, bb, kvh * h, h)
        heads = [kvh * G + g for g in range(G)]
        qg = q[bb].reshape(n, h)[heads]
        o_out, o_idx, o_w, o_dr = oracle.decode_topn_group(qg, ks, vs, N)
        probs = np.stack([oracle.head_weights(qg[g], ks) for g in range(G)])
        slots = [bb * n + hd for hd in heads]
        swaps += check_group(res.selection.indices[slots[0]], res.selection.weights[slots],
                             res.selection.dropped_mass[slots], res.out[bb].reshape(n, h)[heads], probs, vs,
                             N, False, ora_idx=o_idx, ora_out=o_out)
    cache.close()
    return swaps


def test_c2_layer_full_size_sampled(kc, oracle):
    """Config 2 shape (LLaMA2-7B, b=8, 32k, N=128), one layer at full size;
    sampled slots against the oracle."""
    _full_size(kc, oracle, b=8, n=32, n_kv=32, s=32768, N=128, samples=6)


def test_c3_layer_full_size_sampled(kc, oracle):
    """Config 3 shape (LLaMA3-8B GQA 32/8, b=32, 16k), one layer, sampled."""
    _full_size(kc, oracle, b=32, n=32, n_kv=8, s=16384, N=128, samples=4)


def test_fill_uniform_matches_seeded_rng(kc):
    import torch
    for dt, name in [(torch.float32, "f32"), (torch.float16, "f16"), (torch.bfloat16, "bf16")]:
        t = torch.empty(10007, dtype=dt, device="cuda")
        kc.fill_uniform(t, 12345, offset=77, lo=-0.05, hi=0.05)
        want = synth(12345, np.arange(77, 77 + 10007, dtype=np.uint64), -0.05, 0.05, name)
        np.testing.assert_array_equal(t.float().cpu().numpy(), want)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_gqa_tensor_core_scoring_precision(kc, oracle, dtype, G):
    """The GQA scoring runs on the tensor cores with q split into fp16 hi+lo
    (scaled so the head's max |q| sits at 2^14) or three bf16 parts; with q
    elements spread over three decades the result must still meet the parity
    rules against the fp32 oracle and match the CUDA-core path."""
    b, n_kv, h, s, N = 2, 2, 128, 1500, 48
    n = n_kv * G
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, dtype)
    rng = np.random.default_rng(G)
    q = (rng.uniform(-1, 1, (b, n * h)) * 10.0 ** rng.uniform(-3, 0, (b, n * h))).astype(np.float32)
    res = kc.decode_attention_topn(q, cache, 0, N, False)
    compare_all(oracle, res, q, ks[0], vs[0], b, n, n_kv, h, s, N, False)
    cache.set_tuning("score_mma", 0)
    ref = kc.decode_attention_topn(q, cache, 0, N, False)
    cache.set_tuning("score_mma", 1)
    same = np.mean([np.array_equal(a, c) for a, c in zip(res.selection.indices, ref.selection.indices)])
    assert same >= 0.9
    np.testing.assert_allclose(res.out, ref.out, rtol=1e-3, atol=1e-6)
    cache.close()


@pytest.mark.parametrize("case", [(1, 8, 2, 40000, 64, "f16"), (1, 4, 4, 36000, 300, "bf16")],
                         ids=["gqa-40k", "mha-36k-N300"])
def test_long_rows_global_key_selection(kc, oracle, case):
    """Rows longer than the register-resident selection (32 k positions) that
    candidate mode does not cover (GQA, N > 256) go through select_kernel:
    keys in a global scratch row, bound from the thread maxima, exact
    selection of the candidates in shared memory."""
    b, n, n_kv, s, N, dtype = case
    h = 128
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, dtype)
    q = synth_matrix(1, b, n * h, dtype=dtype)
    res = kc.decode_attention_topn(q, cache, 0, N, False)
    compare_all(oracle, res, q, ks[0], vs[0], b, n, n_kv, h, s, N, False)
    cache.close()


@pytest.mark.parametrize("order", ["engine", "all-appends-first"])
def test_prefill_staged_offload_equals_mapped_stores(kc, order):
    """Prefill V of offloaded layers through the HBM stages + copy-engine D2H
    (prefill_stage 1) vs straight mapped stores (prefill_stage 0): rows read
    back before and after offload_prefill_v, the ledger, and the decode
    results are identical. "all-appends-first" appends every layer before the
    first offload, so layers beyond the two stages take the direct path."""
    b, n, n_kv, h, s, N, L = 2, 8, 4, 128, 900, 64, 4
    ks = [synth_matrix(2 + 100 * l, s * b, n_kv * h) for l in range(L)]
    vs = [synth_matrix(3 + 100 * l, s * b, n_kv * h) for l in range(L)]
    q = synth_matrix(1, b, n * h)
    results = []
    for stage in (0, 1):
        cfg = kc.small_config(L, n * h, n, s, kv_heads=n_kv)
        cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(1, L, 2, "f16"))
        cache.set_tuning("prefill_stage", stage)

        def append(l):
            for c0 in range(0, s, 300):
                cache.append_kv(l, ks[l][c0 * b:(c0 + 300) * b], vs[l][c0 * b:(c0 + 300) * b])
            np.testing.assert_array_equal(cache.v_row(l, s - 1, 1), vs[l][(s - 1) * b + 1])

        if order == "engine":
            for l in range(L):
                append(l)
                cache.offload_prefill_v(l)
                np.testing.assert_array_equal(cache.v_row(l, 7, 0), vs[l][7 * b])
        else:
            for l in range(L):
                append(l)
            for l in range(L):
                cache.offload_prefill_v(l)
        cache.begin_decode()
        got = [kc.decode_attention_topn(q, cache, l, N, False) for l in range(L)]
        sel = [[0, 5, s - 1]] * (b * n)
        gv = cache.gather_v(L - 1, sel)
        for slot in range(b * n):
            bb, hd = divmod(slot, n)
            kvh = hd // (n // n_kv)
            want = vs[L - 1][np.array(sel[slot]) * b + bb][:, kvh * h:(kvh + 1) * h]
            np.testing.assert_array_equal(np.asarray(gv.blocks[slot]).reshape(3, h), want)
        results.append((got, cache.ledger_jsonl()))
        cache.close()
    (a, la), (c, lc) = results
    assert la == lc
    for x, y in zip(a, c):
        np.testing.assert_array_equal(x.out, y.out)
        np.testing.assert_array_equal(x.selection.indices, y.selection.indices)
        np.testing.assert_array_equal(x.selection.dropped_mass, y.selection.dropped_mass)
