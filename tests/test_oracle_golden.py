"""CPU: pin the oracle restatement (oracle/kcache_oracle.c) to the reference.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py
over oracle/_ref); known-answer tests are the reference's own
(proj/tests/test_attention.cpp:153-178, test_matrix.cpp:42-159,
test_kv_cache.cpp:114-131). When oracle/_ref is present (this container) the
restatement is also compared against it live on fresh random cases.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle.oracle import Reference, synth, synth_matrix

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden_meta.json")))


def _inputs(c):
    d = c["n"] * c["h"]
    q = synth_matrix(c["seed0"] + 1, c["b"], d, c["lo"] if "lo" in c else -1.0, c.get("hi", 1.0), c["dtype"])
    k = synth_matrix(c["seed0"] + 2, c["s"] * c["b"], d, c.get("lo", -1.0), c.get("hi", 1.0), c["dtype"])
    v = synth_matrix(c["seed0"] + 3, c["s"] * c["b"], d, -1.0, 1.0, c["dtype"])
    return q, k, v


@pytest.mark.parametrize("ci", range(len(META["topn"])))
def test_decode_topn_matches_reference_golden(oracle, ci):
    c = META["topn"][ci]
    q, k, v = _inputs(c)
    out, idx, w, dr = oracle.decode_topn(q, k, v, c["b"], c["n"], c["n"], c["h"], c["s"], c["N"],
                                         bool(c["renorm"]), bool(c["ordered"]))
    # bitwise: same fp32 operation order as the reference (-ffp-contract=off)
    np.testing.assert_array_equal(out, GOLD[f"topn{ci}_out"])
    np.testing.assert_array_equal(idx, GOLD[f"topn{ci}_idx"])
    np.testing.assert_array_equal(w, GOLD[f"topn{ci}_w"])
    np.testing.assert_array_equal(dr, GOLD[f"topn{ci}_dropped"])
    # ledger: bytes * b * n * min(N, s) * h for an offloaded layer, 0 resident
    want = 0 if c["resident"] else 2 * c["b"] * c["n"] * min(c["N"], c["s"]) * c["h"]
    assert c["h2d"] == want


@pytest.mark.parametrize("ci", range(len(META["full"])))
def test_decode_full_matches_reference_golden(oracle, ci):
    c = META["full"][ci]
    q, k, v = _inputs(c)
    got = oracle.decode_full(q, k, v, c["b"], c["n"], c["n"], c["h"], c["s"])
    np.testing.assert_array_equal(got, GOLD[f"full{ci}_out"])


def test_arg_topk_matches_reference_golden(oracle):
    for ci, k in enumerate(META["argtopk_k"]):
        vals = GOLD[f"argtopk{ci}_vals"]
        np.testing.assert_array_equal(oracle.arg_topk(vals, k), GOLD[f"argtopk{ci}_idx"])


def test_softmax_matches_reference_golden(oracle):
    np.testing.assert_array_equal(oracle.softmax(GOLD["softmax_in"]), GOLD["softmax_out"])


def test_rng_streams_match_reference_golden(oracle):
    for seed in (1, 2, 3, 12345):
        want = GOLD[f"rng{seed}"]
        np.testing.assert_array_equal(synth(seed, np.arange(257, dtype=np.uint64), -1.0, 1.0, "f32"), want)
        assert oracle.uniform(seed, 100) == want[100]
    np.testing.assert_array_equal(synth(7, np.arange(257, dtype=np.uint64), -0.05, 0.05, "f32"), GOLD["rng7_narrow"])


# ---- the reference's own known-answer tests, restated -------------------------
def test_kat_softmax_row_01_04_02_03(oracle):
    """proj/tests/test_attention.cpp:153-178: h=1, keys ln(.1,.4,.2,.3), N=2."""
    k = np.array([[math.log(0.1)], [math.log(0.4)], [math.log(0.2)], [math.log(0.3)]], np.float32)
    v = np.array([[10.0], [20.0], [30.0], [40.0]], np.float32)
    q = np.ones((1, 1), np.float32)
    out, idx, w, dr = oracle.decode_topn(q, k, v, 1, 1, 1, 1, 4, 2, False)
    assert list(idx[0]) == [1, 3]
    assert w[0][0] == pytest.approx(0.4, rel=1e-5) and w[0][1] == pytest.approx(0.3, rel=1e-5)
    assert dr[0] == pytest.approx(0.3, rel=1e-5)
    assert out[0, 0] == pytest.approx(20.0, rel=1e-4)
    out, *_ = oracle.decode_topn(q, k, v, 1, 1, 1, 1, 4, 2, True)
    assert out[0, 0] == pytest.approx(20.0 / 0.7, rel=1e-4)


def test_kat_arg_topk_examples(oracle):
    """proj/tests/test_matrix.cpp:123-132."""
    vals = [0.1, 0.4, 0.2, 0.3]
    assert list(oracle.arg_topk(vals, 2)) == [1, 3]
    assert list(oracle.arg_topk(vals, 9)) == [0, 1, 2, 3]
    assert list(oracle.arg_topk([0.5, 0.5, 0.1], 1)) == [0]
    with pytest.raises(ValueError):
        oracle.arg_topk(vals, 0)


def test_kat_softmax_examples(oracle):
    """SPEC.md softmax examples (uniform, max-subtraction, closed form)."""
    np.testing.assert_allclose(oracle.softmax([0, 0, 0, 0]), [0.25] * 4)
    np.testing.assert_allclose(oracle.softmax([1000, 1000]), [0.5, 0.5])
    np.testing.assert_allclose(oracle.softmax([0, math.log(3)]), [0.25, 0.75], rtol=1e-6)


def test_topn_with_n_ge_s_equals_full_bitwise(oracle):
    """proj/tests/test_attention.cpp:126-151 on the restatement."""
    b, n, h, s = 2, 4, 16, 24
    q, k, v = synth_matrix(1, b, n * h, dtype="f32"), synth_matrix(2, s * b, n * h, dtype="f32"), \
        synth_matrix(3, s * b, n * h, dtype="f32")
    full = oracle.decode_full(q, k, v, b, n, n, h, s)
    for N in (s, s + 10, 4096):
        out, idx, w, dr = oracle.decode_topn(q, k, v, b, n, n, h, s, N, False)
        np.testing.assert_array_equal(out, full)
        assert np.all(np.abs(dr) <= 1e-6)
        np.testing.assert_array_equal(idx, np.tile(np.arange(s, dtype=np.uint32), (b * n, 1)))


def test_gqa_extension_reduces_to_reference_for_group_one(oracle):
    """The GQA rule (sum of the group's p) with G = 1 is the reference's rule."""
    b, n, h, s, N = 2, 4, 16, 60, 9
    q, k, v = synth_matrix(1, b, n * h), synth_matrix(2, s * b, n * h), synth_matrix(3, s * b, n * h)
    mha = oracle.decode_topn(q, k, v, b, n, n, h, s, N, False)
    for bb in range(b):
        for head in range(n):
            ks = k[bb::b, head * h:(head + 1) * h]
            vs = v[bb::b, head * h:(head + 1) * h]
            o, idx, w, dr = oracle.decode_topn_group(q[bb:bb + 1, head * h:(head + 1) * h], ks, vs, N)
            slot = bb * n + head
            np.testing.assert_array_equal(idx, mha[1][slot])
            np.testing.assert_array_equal(w[0], mha[2][slot])
            np.testing.assert_array_equal(o[0], mha[0][bb, head * h:(head + 1) * h])


def test_gqa_selection_uses_group_probability_sum(oracle):
    """GQA (G=4): indices shared by the group = top-N of sum_g p_g."""
    G, h, s, N = 4, 32, 200, 17
    qg = synth_matrix(5, G, h)
    ks = synth_matrix(6, s, h)
    vs = synth_matrix(7, s, h)
    out, idx, w, dr = oracle.decode_topn_group(qg, ks, vs, N)
    probs = np.stack([oracle.head_weights(qg[g], ks) for g in range(G)])
    key = probs[0].copy()
    for g in range(1, G):
        key = (key + probs[g]).astype(np.float32)
    np.testing.assert_array_equal(idx, oracle.arg_topk(key, N))
    for g in range(G):
        np.testing.assert_array_equal(w[g], probs[g][idx])
        assert dr[g] == pytest.approx(1.0 - probs[g][idx].astype(np.float64).sum(), abs=1e-12)


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref is built only where /root/reference exists")
def test_restatement_equals_live_reference_random(oracle):
    ref = Reference()
    rng = np.random.default_rng(3)
    for _ in range(12):
        b = int(rng.integers(1, 4))
        n = int(rng.choice([1, 2, 4, 8]))
        h = int(rng.choice([1, 8, 16, 64]))
        s = int(rng.integers(1, 200))
        N = int(rng.integers(1, 260))
        renorm = bool(rng.integers(2))
        seed = int(rng.integers(1 << 30))
        q, k, v = synth_matrix(seed, b, n * h, dtype="f32"), synth_matrix(seed + 1, s * b, n * h, dtype="f32"), \
            synth_matrix(seed + 2, s * b, n * h, dtype="f32")
        a = oracle.decode_topn(q, k, v, b, n, n, h, s, N, renorm)
        r = ref.decode_topn(q, k, v, b, n, h, s, N, renorm)
        for x, y in zip(a, r[:4]):
            np.testing.assert_array_equal(x, y)
