"""Candidate-mode selection (MHA): the scoring kernel emits only each split's
possible top-N positions, the selection kernel ranks those, and rows whose
candidate set cannot be proven complete are redone densely from q and K
(kc_score.cu emit_candidates, kc_select.cu select_cand_kernel).

The candidate path must be an exact re-implementation of the dense path:
identical indices, weights, dropped mass and outputs, bit for bit, on random,
tie-flooded and underflowing (p == 0 ties) rows, and the forced dense redo
must reproduce the scoring kernel's scores bit for bit.
"""
import numpy as np
import pytest

from oracle.oracle import synth_matrix
from tests.test_gpu_parity import build_cache, compare_all

pytestmark = pytest.mark.gpu

DEFAULTS = {"select_cand": 0, "cand_force_fallback": 0, "score_groups": 0, "score_chunk": 0,
            "recall_pipe": -1, "score_mma": 1, "recall_ctas": 32, "tlb_ahead": -1, "consume": 1, "consume_ctas": 0,
            "recall_lean": -1, "recall_tma": 0}


def _run(kc, cache, q, N, renorm=False, **tune):
    tune.setdefault("select_cand", 1)
    for k, v in tune.items():
        cache.set_tuning(k, v)
    res = kc.decode_attention_topn(q, cache, 0, N, renorm)
    for k in tune:
        cache.set_tuning(k, DEFAULTS[k])
    return res


def _assert_same(a, b):
    np.testing.assert_array_equal(a.selection.indices, b.selection.indices)
    np.testing.assert_array_equal(a.selection.weights, b.selection.weights)
    np.testing.assert_array_equal(a.selection.dropped_mass, b.selection.dropped_mass)
    np.testing.assert_array_equal(a.out, b.out)


CASES = [
    # b, n, h, s, N, dtype
    (2, 4, 128, 300, 32, "f16"),
    (1, 8, 128, 5000, 128, "f16"),     # several splits, ragged last split
    (2, 4, 128, 4097, 1, "bf16"),      # N = 1
    (1, 4, 128, 3000, 128, "f16"),     # N = 128 (the candidate-mode maximum)
    (1, 4, 128, 3000, 256, "f16"),     # N = 256: dense path
    (1, 4, 128, 2000, 300, "f16"),     # N > 256: dense path
    (1, 2, 128, 100, 128, "bf16"),     # N >= s: everything selected
    (2, 4, 128, 40000, 128, "f16"),    # s > 32k: dense fallback is the global-keys kernel
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_candidates_equal_dense_bitwise(kc, oracle, case):
    b, n, h, s, N, dtype = case
    cache, ks, vs = build_cache(kc, b, n, n, h, s, dtype)
    q = synth_matrix(1, b, n * h, dtype=dtype)
    for renorm in (False, True):
        cand = _run(kc, cache, q, N, renorm)
        dense = _run(kc, cache, q, N, renorm, select_cand=2)
        redo = _run(kc, cache, q, N, renorm, cand_force_fallback=1)
        _assert_same(cand, dense)
        _assert_same(redo, dense)
    if s <= 5000:
        compare_all(oracle, cand, q, ks[0], vs[0], b, n, n, h, s, N, True)


def test_tie_flood_selects_lowest_positions(kc, oracle):
    """Every K row equal: every score ties, the reference's stable sort keeps
    the lowest positions (matrix.cpp:109-122); 20000 candidates per row exceed
    the candidate capacity, so this also runs the capacity fallback."""
    b, n, h, s, N = 1, 2, 128, 20000, 64
    cfg = kc.small_config(1, n * h, n, s)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, 1, 2, "f16"))
    k = np.full((s * b, n * h), 0.25, np.float32)
    v = synth_matrix(3, s * b, n * h)
    cache.append_kv(0, k, v)
    cache.offload_prefill_v(0)
    cache.begin_decode()
    q = synth_matrix(1, b, n * h)
    res = _run(kc, cache, q, N)
    np.testing.assert_array_equal(res.selection.indices, np.tile(np.arange(N, dtype=np.uint32), (b * n, 1)))
    dense = _run(kc, cache, q, N, select_cand=2)
    _assert_same(res, dense)
    cache.close()


def test_underflow_ties_take_lowest_positions(kc, oracle):
    """A few planted positions hold all the mass; every other p underflows to
    exactly 0, so the N-th p is 0 and the zero-probability positions tie: the
    reference keeps the lowest of them. The candidate bound cannot prove this
    row complete, so it takes the dense redo."""
    b, n, h, s, N = 1, 2, 128, 3000, 16
    hot = [2500, 700, 1999]
    cfg = kc.small_config(1, n * h, n, s)
    cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, 1, 2, "f16"))
    k = np.full((s * b, n * h), -2.0, np.float32)
    for j in hot:
        k[j, :] = 8.0
    v = synth_matrix(3, s * b, n * h)
    cache.append_kv(0, k, v)
    cache.offload_prefill_v(0)
    cache.begin_decode()
    q = np.ones((b, n * h), np.float32)
    res = _run(kc, cache, q, N)
    o_out, o_idx, o_w, o_dr = oracle.decode_topn(q, k, v, b, n, n, h, s, N, False, True)
    want = np.array(sorted(hot + [j for j in range(s) if j not in hot][:N - len(hot)]), np.uint32)
    for slot in range(b * n):
        np.testing.assert_array_equal(o_idx[slot], want)
        np.testing.assert_array_equal(res.selection.indices[slot], want)
    _assert_same(res, _run(kc, cache, q, N, select_cand=2))
    cache.close()


VARIANTS = {
    "groups2": dict(score_groups=2), "groups5": dict(score_groups=5), "cand": dict(select_cand=1),
    "cand-groups3": dict(select_cand=1, score_groups=3), "recall-pipe": dict(recall_pipe=1),
    "recall-pipe-per-row": dict(recall_pipe=1, recall_ctas=0), "recall-plain": dict(recall_pipe=0),
    "recall-ctas128": dict(recall_ctas=128), "recall-lean": dict(recall_pipe=1, recall_lean=1),
    "recall-not-lean": dict(recall_lean=0),
    "recall-tma": dict(recall_tma=1), "recall-tma-per-row": dict(recall_tma=1, recall_ctas=0), "no-tlb-warm": dict(tlb_ahead=0), "chunk4096": dict(score_chunk=4096),
}


@pytest.mark.parametrize("tune", list(VARIANTS.values()), ids=list(VARIANTS))
@pytest.mark.parametrize("n_kv", [8, 2], ids=["mha", "gqa4"])
def test_pipeline_variants_bitwise(kc, tune, n_kv):
    """Row groups, the recall variants and candidate selection reproduce the
    default path bit for bit; another split length changes only the rounding
    of the softmax statistics."""
    b, n, h, s, N, L = 2, 8, 128, 3000, 64, 7  # L > kRing (3): ring slots are reused
    if n_kv != n and "select_cand" in tune:
        pytest.skip("candidate selection is MHA-only")
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", n_layers=L)
    qs = [synth_matrix(10 + l, b, n * h) for l in range(L)]
    nc = min(N, s)

    def run():
        outs = [{"out": np.zeros((b, n * h), np.float32), "indices": np.zeros((b * n, nc), np.uint32),
                 "weights": np.zeros((b * n, nc), np.float32), "dropped": np.zeros(b * n, np.float64)}
                for _ in range(L)]
        cache.decode_topn_layers_host(list(range(L)), qs, N, outs)
        return outs

    base = run()
    for k, v in tune.items():
        cache.set_tuning(k, v)
    got = run()
    for k in tune:
        cache.set_tuning(k, DEFAULTS[k])
    for l in range(L):
        if "score_chunk" in tune:
            np.testing.assert_array_equal(got[l]["indices"], base[l]["indices"])
            for key in ("out", "weights"):
                np.testing.assert_allclose(got[l][key], base[l][key], rtol=1e-5, atol=5e-9)
            np.testing.assert_allclose(got[l]["dropped"], base[l]["dropped"], atol=1e-6)
            continue
        for key in ("out", "indices", "weights", "dropped"):
            np.testing.assert_array_equal(got[l][key], base[l][key])
