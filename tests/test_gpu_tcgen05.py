"""GQA scoring on the 5th-generation tensor cores (kc_score_tc.cu,
score_mma 3): tcgen05.mma from 2-D TMA (SWIZZLE_128B) K tiles and a q-parts B
operand, fp32 accumulators in TMEM. Against the CPU oracle (tests/parity.py
rules) and against the mma.sync kernel (score_mma 1): the same index sets
except epsilon-window swaps, outputs within fp32 rounding of another
summation order."""
import numpy as np
import pytest

from oracle.oracle import synth_matrix
from tests.test_gpu_parity import build_cache, compare_all

pytestmark = pytest.mark.gpu

CASES = [
    # b, n, n_kv, s, N, dtype
    (2, 8, 4, 3000, 64, "f16"),     # G = 2
    (2, 8, 2, 777, 16, "f16"),      # G = 4, s not a multiple of 128
    (1, 8, 1, 2500, 32, "bf16"),    # G = 8, bf16: 24 q-part rows (N = 32)
    (1, 16, 4, 5000, 128, "bf16"),  # G = 4, bf16 (N = 16)
    (3, 8, 2, 129, 200, "f16"),     # N > s, one position past a stage
    (2, 4, 4, 3000, 64, "f16"),     # MHA (one q head in two parts, N = 16)
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_tcgen05_scoring_parity(kc, oracle, case):
    b, n, n_kv, s, N, dtype = case
    h = 128
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, dtype)
    q = synth_matrix(1, b, n * h, dtype=dtype)
    for chunk in (0, 1024):
        cache.set_tuning("score_chunk", chunk)
        cache.set_tuning("score_mma", 1)
        ref = kc.decode_attention_topn(q, cache, 0, N, False)
        cache.set_tuning("score_mma", 3)
        got = kc.decode_attention_topn(q, cache, 0, N, False)
        compare_all(oracle, got, q, ks[0], vs[0], b, n, n_kv, h, s, N, False)
        same = np.mean([np.array_equal(a, c) for a, c in zip(ref.selection.indices, got.selection.indices)])
        assert same >= 0.9
        np.testing.assert_allclose(got.out, ref.out, rtol=1e-3, atol=1e-6 * max(np.abs(ref.out).max(), 1e-30))
    cache.set_tuning("score_mma", 1)
    cache.set_tuning("score_chunk", 0)
    cache.close()


def test_tcgen05_pipelined_layers(kc):
    """Multi-layer calls with the tcgen05 scoring (one tensor map per layer)
    equal single-layer calls bit for bit."""
    b, n, n_kv, h, s, N, L = 2, 8, 2, 128, 1500, 32, 4
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", n_layers=L)
    cache.set_tuning("score_mma", 3)
    qs = [synth_matrix(30 + l, b, n * h) for l in range(L)]
    singles = [kc.decode_attention_topn(qs[l], cache, l, N, False) for l in range(L)]
    nc = min(N, s)
    outs = [{"out": np.zeros((b, n * h), np.float32), "indices": np.zeros((b * n, nc), np.uint32),
             "weights": np.zeros((b * n, nc), np.float32), "dropped": np.zeros(b * n, np.float64)} for _ in range(L)]
    cache.decode_topn_layers_host(list(range(L)), qs, N, outs)
    for l in range(L):
        np.testing.assert_array_equal(outs[l]["out"], singles[l].out)
        np.testing.assert_array_equal(outs[l]["indices"], singles[l].selection.indices)
    cache.close()


@pytest.mark.parametrize("tc_grid", [1, 2])
def test_tcgen05_persistent_grid_bitwise(kc, tc_grid):
    """The persistent-grid launch of the tcgen05 scoring (tc_grid CTAs per SM
    walking the items) computes every item with the same instructions: the
    outputs equal the one-CTA-per-item launch bit for bit."""
    b, n, n_kv, h, s, N = 4, 16, 4, 128, 9000, 64
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16")
    q = synth_matrix(5, b, n * h)
    cache.set_tuning("score_mma", 3)
    cache.set_tuning("score_chunk", 1024)
    ref = kc.decode_attention_topn(q, cache, 0, N, False)
    cache.set_tuning("tc_grid", tc_grid)
    got = kc.decode_attention_topn(q, cache, 0, N, False)
    cache.set_tuning("tc_grid", 0)
    cache.set_tuning("score_mma", 1)
    cache.set_tuning("score_chunk", 0)
    np.testing.assert_array_equal(got.out, ref.out)
    np.testing.assert_array_equal(got.selection.indices, ref.selection.indices)
    np.testing.assert_array_equal(got.selection.weights, ref.selection.weights)
    cache.close()
