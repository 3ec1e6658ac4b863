"""The reference's own unit tests for the hot path, restated against the GPU
implementation through the Python mirror of the operator API.

proj/tests/test_attention.cpp, proj/tests/test_kv_cache.cpp and the arg_topk
cases of proj/tests/test_matrix.cpp. Where the reference asserts bitwise
equality between two CPU evaluation orders, the GPU assertion is the stated
tolerance; index sets, ledger bytes and error types stay
exact. Storage is fp32 here so the reference's random_matrix data is stored
unrounded.
"""
import math

import numpy as np
import pytest

from oracle.oracle import synth_matrix

pytestmark = pytest.mark.gpu

_off = [0]


def rnd(kc, rows, cols, lo=-1.0, hi=1.0, seed=11):
    """random_matrix (proj/tests/oracles.hpp:24-31) from a running stream."""
    m = synth_matrix(seed, rows, cols, lo, hi, "f32", offset=_off[0])
    _off[0] += rows * cols
    return m


def make_cache(kc, c, batch, resident, k, v, storage="f32"):
    """proj/tests/test_attention.cpp:27-36"""
    cache = kc.TieredKVCache(c, batch, kc.TierPlacement.kcache(resident, c.n_layers, 2, storage))
    for layer in range(c.n_layers):
        cache.append_kv(layer, k, v)
        cache.offload_prefill_v(layer)
    cache.begin_decode()
    return cache


# ---------------- test_attention.cpp ----------------
def test_score_scale(kc):
    for h in (16, 64, 128, 256):
        assert kc.attention_score_scale(h) == float(np.float32(1.0) / np.sqrt(np.float32(h)))


def test_decode_full_all_equal_scores_average_v(kc):
    c = kc.small_config(2, 32, 4)
    s = 8
    k = np.ones((s, c.d_model), np.float32)
    v = rnd(kc, s, c.d_model)
    cache = make_cache(kc, c, 1, 0, k, v)
    q = rnd(kc, 1, c.d_model)
    out = kc.decode_attention_full(q, cache, 0)
    np.testing.assert_allclose(out[0], v.astype(np.float64).mean(axis=0), rtol=1e-5, atol=1e-6)


def test_decode_full_empty_cache_is_state_error(kc):
    c = kc.small_config(2, 32, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(0, c.n_layers))
    with pytest.raises(kc.StateError):
        kc.decode_attention_full(np.zeros((1, c.d_model), np.float32), cache, 0)
    with pytest.raises(kc.StateError):
        kc.decode_attention_topn(np.zeros((1, c.d_model), np.float32), cache, 0, 4, False)


def test_topn_equals_full_when_n_covers_the_cache(kc):
    c = kc.small_config(3, 64, 4)
    s, batch = 24, 2
    k = rnd(kc, s * batch, c.d_model)
    v = rnd(kc, s * batch, c.d_model)
    cache = make_cache(kc, c, batch, 1, k, v)  # layer 0 resident, 1..2 offloaded
    q = rnd(kc, batch, c.d_model)
    for layer in range(c.n_layers):
        full = kc.decode_attention_full(q, cache, layer)
        for n in (s, s + 10, 4096):
            r = kc.decode_attention_topn(q, cache, layer, n, False)
            np.testing.assert_allclose(r.out, full, rtol=1e-5, atol=1e-6)
            assert r.selection.indices.shape == (batch * c.n_heads, s)
            assert np.all(np.abs(r.selection.dropped_mass) <= 1e-6)
            np.testing.assert_array_equal(r.selection.indices, np.tile(np.arange(s), (batch * c.n_heads, 1)))


def test_topn_hand_checkable_case(kc):
    c = kc.small_config(1, 1, 1)
    c.ffn_hidden = 4
    k = np.array([[math.log(0.1)], [math.log(0.4)], [math.log(0.2)], [math.log(0.3)]], np.float32)
    v = np.array([[10.0], [20.0], [30.0], [40.0]], np.float32)
    cache = make_cache(kc, c, 1, 0, k, v)
    q = np.ones((1, 1), np.float32)
    r = kc.decode_attention_topn(q, cache, 0, 2, False)
    assert list(r.selection.indices[0]) == [1, 3]
    assert r.selection.weights[0][0] == pytest.approx(0.4, rel=1e-5)
    assert r.selection.weights[0][1] == pytest.approx(0.3, rel=1e-5)
    assert r.selection.dropped_mass[0] == pytest.approx(0.3, rel=1e-5)
    assert r.out[0, 0] == pytest.approx(20.0, rel=1e-4)
    renorm = kc.decode_attention_topn(q, cache, 0, 2, True)
    assert renorm.out[0, 0] == pytest.approx(20.0 / 0.7, rel=1e-4)


def test_monotone_coverage_in_n(kc):
    c = kc.small_config(1, 32, 4)
    for inst in range(10):
        s = 32
        k = rnd(kc, s, c.d_model, -2.0, 2.0)
        v = rnd(kc, s, c.d_model)
        cache = make_cache(kc, c, 1, 0, k, v)
        q = rnd(kc, 1, c.d_model, -2.0, 2.0)
        prev = None
        for n in range(1, s + 1):
            r = kc.decode_attention_topn(q, cache, 0, n, False)
            if prev is not None:
                assert np.all(r.selection.dropped_mass <= prev + 1e-12)
                for slot in range(r.selection.indices.shape[0]):  # selections are nested
                    assert set(prev_idx[slot]) <= set(r.selection.indices[slot])
            prev = r.selection.dropped_mass
            prev_idx = r.selection.indices


def test_renormalized_output_is_a_convex_combination(kc):
    c = kc.small_config(1, 32, 4)
    s = 20
    k = rnd(kc, s, c.d_model)
    v = rnd(kc, s, c.d_model)
    cache = make_cache(kc, c, 1, 0, k, v)
    q = rnd(kc, 1, c.d_model)
    r = kc.decode_attention_topn(q, cache, 0, 5, True)
    for head in range(c.n_heads):
        idx = r.selection.indices[head]
        sel = v[idx][:, head * c.head_dim:(head + 1) * c.head_dim]
        got = r.out[0, head * c.head_dim:(head + 1) * c.head_dim]
        assert np.all(got >= sel.min(axis=0) - 1e-5)
        assert np.all(got <= sel.max(axis=0) + 1e-5)


def test_h2d_byte_accounting_per_call(kc):
    c = kc.small_config(2, 64, 4)
    s = 10
    k = rnd(kc, s, c.d_model)
    v = rnd(kc, s, c.d_model)
    cache = make_cache(kc, c, 1, 1, k, v)
    q = rnd(kc, 1, c.d_model)
    off = kc.decode_attention_topn(q, cache, 1, 64, False)
    assert off.h2d_bytes == 2 * 1 * c.n_heads * s * c.head_dim  # clamped to s
    off4 = kc.decode_attention_topn(q, cache, 1, 4, False)
    assert off4.h2d_bytes == 2 * 1 * c.n_heads * 4 * c.head_dim
    assert off4.selection.indices.shape[1] == 4
    res = kc.decode_attention_topn(q, cache, 0, 4, False)
    assert res.h2d_bytes == 0
    with pytest.raises(ValueError):
        kc.decode_attention_topn(q, cache, 0, 0, False)


def test_topn_error_vs_full_is_zero_at_full_coverage(kc):
    c = kc.small_config(4, 64, 4)
    s = 256
    k = rnd(kc, s, c.d_model)
    v = rnd(kc, s, c.d_model)
    cache = make_cache(kc, c, 1, 0, k, v)
    q = rnd(kc, 1, c.d_model)
    full = kc.decode_attention_full(q, cache, 0)
    errs = {}
    for n in (16, 64, 256):
        r = kc.decode_attention_topn(q, cache, 0, n, False)
        errs[n] = float(np.abs(full.astype(np.float64) - r.out).max())
    assert errs[256] <= 1e-6  # reference: exactly 0 (same CPU order); GPU: tolerance
    assert errs[16] >= errs[64] >= errs[256]


def test_sparsity_bound_on_concentrated_rows(kc):
    c = kc.small_config(1, 32, 4)
    rng = np.random.default_rng(7)
    for inst in range(10):
        s = 40
        k = rnd(kc, s, c.d_model, -0.05, 0.05)
        hot = int(rng.integers(s))
        k[hot, :] = 6.0
        v = rnd(kc, s, c.d_model)
        cache = make_cache(kc, c, 1, 0, k, v)
        q = np.ones((1, c.d_model), np.float32)
        full = kc.decode_attention_full(q, cache, 0)
        topn = kc.decode_attention_topn(q, cache, 0, 4, False)
        dm = float(topn.selection.dropped_mass.max())
        vmax = float(np.abs(v).max())
        assert np.all(np.abs(full - topn.out) <= dm * vmax + 1e-6)
        assert all(hot in topn.selection.indices[hd] for hd in range(c.n_heads))


def test_uniform_keys_tie_to_lowest_positions(kc):
    """All-equal keys: every probability ties; the reference's stable sort
    keeps the N lowest positions (matrix.cpp:116-121)."""
    c = kc.small_config(1, 64, 4)
    s = 3000
    k = np.full((s, c.d_model), 0.5, np.float32)
    v = rnd(kc, s, c.d_model)
    cache = make_cache(kc, c, 1, 0, k, v)
    q = rnd(kc, 1, c.d_model)
    for n in (1, 7, 128, 1500):
        for sg in (0, 1):
            cache.set_tuning("select_global", sg)
            r = kc.decode_attention_topn(q, cache, 0, n, False)
            np.testing.assert_array_equal(r.selection.indices, np.tile(np.arange(n), (c.n_heads, 1)))
            np.testing.assert_allclose(r.selection.weights, 1.0 / s, rtol=1e-5)


def test_planted_tie_blocks_at_the_boundary(kc):
    """Groups of identical keys straddling the N-th place: survivors are the
    strictly larger keys plus the lowest positions of the boundary group."""
    c = kc.small_config(1, 16, 1)
    s = 5000
    k = rnd(kc, s, c.d_model, -0.1, 0.1)
    rng = np.random.default_rng(5)
    top = rng.choice(s, 40, replace=False)
    k[top[:20]] = 1.0     # 20 strictly largest
    k[top[20:]] = 0.75    # 20 tied next
    v = rnd(kc, s, c.d_model)
    cache = make_cache(kc, c, 1, 0, k, v)
    q = np.full((1, c.d_model), 0.5, np.float32)
    r = kc.decode_attention_topn(q, cache, 0, 30, False)
    want = np.sort(np.concatenate([top[:20], np.sort(top[20:])[:10]]))
    np.testing.assert_array_equal(r.selection.indices[0], want)


# ---------------- test_kv_cache.cpp ----------------
def fill_prefill(kc, cache, length):
    c = cache.config
    for layer in range(c.n_layers):
        cache.append_kv(layer, rnd(kc, length * cache.batch, c.d_model), rnd(kc, length * cache.batch, c.d_model))
        cache.offload_prefill_v(layer)
    cache.begin_decode()


def test_baseline_placement_never_records_d2h(kc):
    c = kc.small_config(4, 64, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.baseline(c.n_layers))
    fill_prefill(kc, cache, 16)
    cache.append_kv(0, rnd(kc, 1, 64), rnd(kc, 1, 64))
    assert cache.d2h_bytes_total() == 0 and cache.h2d_bytes_total() == 0 and cache.slow_bytes_used() == 0


def test_prefill_offload_accounts_bytes_per_layer(kc):
    c = kc.small_config(1, 64, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(0, c.n_layers))
    cache.append_kv(0, rnd(kc, 128, 64), rnd(kc, 128, 64))
    assert cache.d2h_bytes_total() == 0
    cache.offload_prefill_v(0)
    assert cache.d2h_bytes_total() == 16384


def test_decode_append_to_offloaded_layer_records_one_row(kc):
    c = kc.small_config(2, 64, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(1, c.n_layers))
    fill_prefill(kc, cache, 8)
    before = cache.d2h_bytes_total()
    cache.append_kv(0, rnd(kc, 1, 64), rnd(kc, 1, 64))
    cache.append_kv(1, rnd(kc, 1, 64), rnd(kc, 1, 64))
    assert cache.d2h_bytes_total() - before == 2 * 1 * 64


def test_byte_counters_after_offload(kc):
    c = kc.small_config(4, 64, 4)
    resident, s, b = 1, 32, 2
    cache = kc.TieredKVCache(c, b, kc.TierPlacement.kcache(resident, c.n_layers))
    fill_prefill(kc, cache, s)
    unit = 2 * b * s * c.d_model
    assert cache.fast_bytes_used() == unit * (c.n_layers + resident)
    assert cache.slow_bytes_used() == unit * (c.n_layers - resident)
    assert cache.current_len() == s


def test_double_offload_is_a_state_error(kc):
    c = kc.small_config(2, 32, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(1, c.n_layers))
    cache.append_kv(1, rnd(kc, 4, 32), rnd(kc, 4, 32))
    cache.offload_prefill_v(0)
    cache.offload_prefill_v(0)
    cache.offload_prefill_v(1)
    with pytest.raises(kc.StateError):
        cache.offload_prefill_v(1)


def test_begin_decode_requires_offload(kc):
    c = kc.small_config(2, 32, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(1, c.n_layers))
    cache.append_kv(1, rnd(kc, 4, 32), rnd(kc, 4, 32))
    with pytest.raises(kc.StateError):
        cache.begin_decode()


def test_append_errors(kc):
    c = kc.small_config(2, 32, 4)
    cache = kc.TieredKVCache(c, 2, kc.TierPlacement.kcache(0, c.n_layers))
    with pytest.raises(IndexError):
        cache.append_kv(7, rnd(kc, 2, 32), rnd(kc, 2, 32))
    with pytest.raises(kc.ShapeError):
        cache.append_kv(0, rnd(kc, 2, 16), rnd(kc, 2, 32))
    with pytest.raises(kc.ShapeError):
        cache.append_kv(0, rnd(kc, 3, 32), rnd(kc, 3, 32))


def test_gather_paper_shape_charge(kc):
    c = kc.small_config(1, 4096, 32)
    cache = kc.TieredKVCache(c, 2, kc.TierPlacement.kcache(0, c.n_layers))
    fill_prefill(kc, cache, 128)
    sel = [list(range(128)) for _ in range(2 * 32)]
    got = cache.gather_v(0, sel)
    assert got.h2d_bytes == 2097152
    assert cache.h2d_bytes_total() == 2097152


def test_gather_resident_bypass(kc):
    c = kc.small_config(2, 64, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(2, c.n_layers))
    fill_prefill(kc, cache, 10)
    got = cache.gather_v(1, [[0, 1, 2]] * 4)
    assert got.h2d_bytes == 0 and cache.h2d_bytes_total() == 0
    assert got.blocks[0].size == 3 * c.head_dim


@pytest.mark.parametrize("storage", ["f32", "f16", "bf16"])
def test_gather_rows_are_returned_bitwise(kc, storage):
    c = kc.small_config(1, 64, 4)
    cache = kc.TieredKVCache(c, 2, kc.TierPlacement.kcache(0, c.n_layers, 2, storage))
    k = synth_matrix(41, 40, 64, dtype=storage)
    v = synth_matrix(42, 40, 64, dtype=storage)
    cache.append_kv(0, k, v)
    cache.offload_prefill_v(0)
    cache.begin_decode()
    sel = [[1, 7, 19]] * 8
    got = cache.gather_v(0, sel)
    for b in range(2):
        for head in range(4):
            block = got.blocks[b * 4 + head]
            for r, pos in enumerate(sel[b * 4 + head]):
                np.testing.assert_array_equal(block[r], v[pos * 2 + b, head * 16:(head + 1) * 16])
    for pos in (0, 5, 19):
        np.testing.assert_array_equal(cache.k_row(0, pos, 1), k[pos * 2 + 1])
        np.testing.assert_array_equal(cache.v_row(0, pos, 0), v[pos * 2])


def test_gather_out_of_range_index_throws(kc):
    c = kc.small_config(1, 64, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(0, c.n_layers))
    fill_prefill(kc, cache, 10)
    with pytest.raises(IndexError):
        cache.gather_v(0, [[0, 10]] * 4)
    with pytest.raises(IndexError):
        cache.k_row(0, 10, 0)


def test_fast_tier_capacity_budget(kc):
    c = kc.small_config(2, 64, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(2, c.n_layers), 4096)
    cache.append_kv(0, rnd(kc, 8, 64), rnd(kc, 8, 64))
    with pytest.raises(kc.CapacityError):
        cache.append_kv(1, rnd(kc, 16, 64), rnd(kc, 16, 64))


def test_ledger_serializes_to_json_lines(kc):
    c = kc.small_config(1, 32, 4)
    cache = kc.TieredKVCache(c, 1, kc.TierPlacement.kcache(0, c.n_layers))
    cache.append_kv(0, rnd(kc, 2, 32), rnd(kc, 2, 32))
    cache.offload_prefill_v(0)
    assert cache.ledger_jsonl() == '{"phase":"prefill","layer":0,"dir":"D2H","bytes":128,"elements":64}\n'


def test_ledger_totals_equal_sum_of_events(kc):
    c = kc.small_config(3, 32, 4)
    cache = kc.TieredKVCache(c, 2, kc.TierPlacement.kcache(1, c.n_layers))
    fill_prefill(kc, cache, 12)
    sel = [[0, 3, 5]] * 8
    cache.gather_v(1, sel)
    cache.gather_v(2, sel)
    ev = cache.ledger()
    assert sum(e.bytes for e in ev if e.dir == "D2H") == cache.d2h_bytes_total()
    assert sum(e.bytes for e in ev if e.dir == "H2D") == cache.h2d_bytes_total()
    assert cache.h2d_bytes_total() == 2 * (2 * 4 * 3 * c.head_dim) * 2


def test_ledger_identities_over_a_decode_run(kc):
    """proj/tests/test_engine.cpp:143-172: per step H2D = offloaded layers x
    2*b*n*min(N, len)*h, with the current token appended before attention."""
    for N in (1, 8, 4096):
        for L in (0, 2, 4):
            c = kc.small_config(4, 32, 4)
            b, prompt = 2, 6
            cache = kc.TieredKVCache(c, b, kc.TierPlacement.kcache(L, c.n_layers))
            fill_prefill(kc, cache, prompt)
            for step in range(3):
                before = cache.h2d_bytes_total()
                q = rnd(kc, b, c.d_model)
                for layer in range(c.n_layers):
                    cache.append_kv(layer, rnd(kc, b, c.d_model), rnd(kc, b, c.d_model))
                    kc.decode_attention_topn(q, cache, layer, N, False)
                length = prompt + step + 1
                assert cache.h2d_bytes_total() - before == (4 - L) * 2 * b * c.n_heads * min(N, length) * c.head_dim


# ---------------- test_matrix.cpp (arg_topk) ----------------
def test_arg_topk_examples(kc):
    vals = [0.1, 0.4, 0.2, 0.3]
    assert list(kc.arg_topk(vals, 2)) == [1, 3]
    assert list(kc.arg_topk(vals, 9)) == [0, 1, 2, 3]
    assert list(kc.arg_topk([0.5, 0.5, 0.1], 1)) == [0]
    with pytest.raises(ValueError):
        kc.arg_topk(vals, 0)


def test_arg_topk_selection_property_and_reference_equality(kc, oracle):
    rng = np.random.default_rng(11)
    for rep in range(100):
        n = int(rng.integers(1, 3000))
        vals = rng.uniform(-1, 1, n).astype(np.float32)
        if rep % 3 == 0:
            vals = np.round(vals * 4) / 4  # many ties
        k = int(rng.integers(1, 400))
        idx = kc.arg_topk(vals, k)
        assert len(idx) == min(k, n)
        assert np.all(np.diff(idx.astype(np.int64)) > 0)
        np.testing.assert_array_equal(idx, oracle.arg_topk(vals, k))


# ---------------- prefill_attention (attention.cpp:31-62) ----------------
@pytest.mark.parametrize("s,n,h", [(1, 4, 16), (33, 4, 16), (77, 2, 64), (300, 2, 128), (130, 1, 256)])
def test_prefill_attention_matches_reference(kc, s, n, h):
    """GPU causal prefill vs the reference's own prefill_attention: same dot,
    max, ordered exp-sum and ascending P.V order, so outputs agree to float
    rounding of expf (GPU) vs std::exp (glibc); most elements are bitwise."""
    from oracle.oracle import Reference
    d = n * h
    q = synth_matrix(51, s, d, dtype="f32")
    k = synth_matrix(52, s, d, dtype="f32")
    v = synth_matrix(53, s, d, dtype="f32")
    got = kc.prefill_attention(q, k, v, n)
    if Reference.available():
        want = Reference().prefill_attention(q, k, v, n)
    else:  # restated from attention.cpp:31-62 in float64 (no _ref on this box)
        want = np.zeros((s, d), np.float64)
        scale = float(np.float32(1.0) / np.sqrt(np.float32(h)))
        for hd in range(n):
            sl = slice(hd * h, (hd + 1) * h)
            sc = (q[:, sl].astype(np.float64) @ k[:, sl].T.astype(np.float64)) * scale
            sc[np.triu_indices(s, 1)] = -np.inf
            p = np.exp(sc - sc.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            want[:, sl] = p @ v[:, sl].astype(np.float64)
    np.testing.assert_allclose(got, want, rtol=2e-5, atol=2e-6)
    # position 0 attends to itself only: out = v[0] exactly
    np.testing.assert_array_equal(got[0], v[0])


def test_prefill_attention_errors(kc):
    """attention.cpp:32-37"""
    q = np.zeros((4, 8), np.float32)
    with pytest.raises(kc.ShapeError):
        kc.prefill_attention(q, np.zeros((4, 6), np.float32), q, 2)
    with pytest.raises(kc.ShapeError):
        kc.prefill_attention(q, q, q, 3)
    with pytest.raises(kc.ShapeError):
        kc.prefill_attention(q, q, q, 0)
