"""The dataflow consumer (kc_consume.cu): selection + V recall + P.V of each
(batch, kv head) row as the scoring kernel completes it, on a persistent grid
beside the scoring. It re-implements select_reg_kernel + recall_pv_kernel
(the stream-ordered path, tuning consume 0) and must match it bit for bit:
indices, weights, dropped mass, renormaliser-driven outputs -- on random rows,
rows that take its exact path (N >= s, tie floods, p-underflow ties, N > 1024
candidates), GQA groups, other head dims / storage types (generic scoring
kernel), long rows, single and pipelined multi-layer calls that reuse every
ring and scoring slot, and any consumer grid size. (consume 2 forces the
consumer for these small shapes; by default it serves MHA rows of >= 16 k
positions with N <= 256, covered at full size by test_gpu_fullsize.py.)
"""
import numpy as np
import pytest

from oracle.oracle import synth_matrix
from tests.test_gpu_parity import build_cache, compare_all

pytestmark = pytest.mark.gpu


DEFAULTS = {"consume": 1, "consume_ctas": 0, "select_cached": 1, "consume_recall": -1}


def _decode(kc, cache, q, N, renorm=False, reverse=False, **tune):
    for k, v in tune.items():
        cache.set_tuning(k, v)
    res = kc.decode_attention_topn(q, cache, 0, N, renorm, ordered_accumulation=not reverse)
    for k in tune:
        cache.set_tuning(k, DEFAULTS[k])
    return res


def _same(a, b):
    np.testing.assert_array_equal(a.selection.indices, b.selection.indices)
    np.testing.assert_array_equal(a.selection.weights, b.selection.weights)
    np.testing.assert_array_equal(a.selection.dropped_mass, b.selection.dropped_mass)
    np.testing.assert_array_equal(a.out, b.out)


CASES = [
    # b, n, n_kv, h, s, N, dtype
    (2, 8, 8, 128, 3000, 64, "f16"),     # MHA, fast path
    (2, 8, 2, 128, 3000, 64, "f16"),     # GQA G = 4
    (1, 8, 1, 128, 2500, 32, "bf16"),    # GQA G = 8
    (2, 4, 4, 128, 333, 32, "f16"),      # short rows: exact path (empty warp segments)
    (1, 4, 4, 128, 100, 128, "bf16"),    # N >= s: everything selected
    (1, 4, 4, 128, 4097, 1, "f16"),      # N = 1, ragged
    (1, 4, 4, 128, 6000, 300, "f16"),    # N > 256
    (1, 2, 2, 128, 9000, 1100, "f16"),   # N > 1024: exact path
    (1, 4, 4, 64, 2000, 40, "f16"),      # h = 64: generic scoring kernel
    (1, 4, 2, 128, 1500, 50, "f32"),     # fp32 storage: generic scoring kernel
    (1, 4, 4, 128, 40000, 128, "f16"),   # s > 32k (stream-ordered path: candidate mode)
    (1, 8, 1, 128, 3000, 300, "f16"),    # G * N > 2048: weights read back from global memory
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_consumer_equals_stream_ordered_bitwise(kc, oracle, case):
    b, n, n_kv, h, s, N, dtype = case
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, dtype)
    q = synth_matrix(1, b, n * h, dtype=dtype)
    for renorm, reverse in ((False, False), (True, False), (False, True)):
        ref = _decode(kc, cache, q, N, renorm, reverse, consume=0)
        flow = _decode(kc, cache, q, N, renorm, reverse, consume=2)
        _same(flow, ref)
    if s <= 6000:
        compare_all(oracle, flow, q, ks[0], vs[0], b, n, n_kv, h, s, N, False, ordered=False)
    cache.close()


@pytest.mark.parametrize("ctas", [1, 3, 64, 1000])
def test_consumer_grid_sizes_bitwise(kc, ctas):
    b, n, h, s, N = 4, 8, 128, 2000, 48
    cache, ks, vs = build_cache(kc, b, n, n, h, s, "f16")
    q = synth_matrix(5, b, n * h)
    ref = _decode(kc, cache, q, N, consume=0)
    _same(_decode(kc, cache, q, N, consume=2, consume_ctas=ctas), ref)
    cache.close()


@pytest.mark.parametrize("n_kv", [8, 2], ids=["mha", "gqa4"])
def test_consumer_pipelined_layers_bitwise(kc, n_kv):
    """Multi-layer calls: L > kRing (selection ring slots reused) and > 2
    (scoring slots alternate; layer i+2's scoring waits for layer i's
    consumer), repeated calls, host and device outputs."""
    import torch
    b, n, h, s, N, L = 2, 8, 128, 2500, 64, 7
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", n_layers=L)
    qs = [synth_matrix(10 + l, b, n * h) for l in range(L)]
    nc = min(N, s)

    def run_host():
        outs = [{"out": np.zeros((b, n * h), np.float32), "indices": np.zeros((b * n, nc), np.uint32),
                 "weights": np.zeros((b * n, nc), np.float32), "dropped": np.zeros(b * n, np.float64)}
                for _ in range(L)]
        cache.decode_topn_layers_host(list(range(L)), qs, N, outs)
        return outs

    cache.set_tuning("consume", 0)
    base = run_host()
    cache.set_tuning("consume", 2)
    # multi-layer calls: select-only consumer + the recall kernel (auto), and
    # the consumer recalling itself
    for own in (-1, 1, -1):
        cache.set_tuning("consume_recall", own)
        got = run_host()
        for l in range(L):
            for key in ("out", "indices", "weights", "dropped"):
                np.testing.assert_array_equal(got[l][key], base[l][key])
    cache.set_tuning("consume_recall", -1)
    # device-resident calls on a user stream, back to back without a sync
    stream = torch.cuda.Stream()
    dq = [torch.from_numpy(q).cuda() for q in qs]
    douts = [{"out": torch.empty(b, n * h, device="cuda"), "indices": torch.empty(b * n, nc, dtype=torch.int32, device="cuda"),
              "weights": torch.empty(b * n, nc, device="cuda"), "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")}
             for _ in range(L)]
    for _ in range(3):
        cache.decode_topn_layers_device(list(range(L)), dq, N, douts, stream=stream)
    torch.cuda.synchronize()
    for l in range(L):
        np.testing.assert_array_equal(douts[l]["out"].cpu().numpy(), base[l]["out"])
        np.testing.assert_array_equal(douts[l]["indices"].cpu().numpy().view(np.uint32), base[l]["indices"])
        np.testing.assert_array_equal(douts[l]["dropped"].cpu().numpy(), base[l]["dropped"])
    cache.set_tuning("consume", 1)
    cache.close()


def test_consumer_tie_flood_and_underflow(kc, oracle):
    """Rows the fast path cannot bound (every score ties; p underflows to 0
    for all but three positions) go through the consumer's exact path: the
    lowest positions win the ties, as in the reference's stable sort."""
    b, n, h, s, N = 1, 2, 128, 5000, 16
    cfg = kc.small_config(1, n * h, n, s)
    for kind in ("flood", "underflow"):
        cache = kc.TieredKVCache(cfg, b, kc.TierPlacement.kcache(0, 1, 2, "f16"))
        if kind == "flood":
            k = np.full((s * b, n * h), 0.25, np.float32)
            q = synth_matrix(1, b, n * h)
        else:
            k = np.full((s * b, n * h), -2.0, np.float32)
            for j in (4500, 700, 1999):
                k[j, :] = 8.0
            q = np.ones((b, n * h), np.float32)
        v = synth_matrix(3, s * b, n * h)
        cache.append_kv(0, k, v)
        cache.offload_prefill_v(0)
        cache.begin_decode()
        flow = _decode(kc, cache, q, N, consume=2)
        _same(flow, _decode(kc, cache, q, N, consume=0))
        o_out, o_idx, o_w, o_dr = oracle.decode_topn(q, k, v, b, n, n, h, s, N, False, True)
        for slot in range(b * n):
            np.testing.assert_array_equal(flow.selection.indices[slot], o_idx[slot])
        cache.close()


@pytest.mark.parametrize("case", [(40, 8, 4, 3000, 64, "f16"), (160, 8, 1, 1500, 32, "bf16"),
                                  (80, 8, 2, 8192, 128, "f16"), (80, 4, 2, 333, 32, "f16")],
                         ids=["G2", "G8", "G4-8k", "G2-short"])
def test_cached_gqa_selection_bitwise(kc, oracle, case):
    """The stream-ordered GQA selection with shared-memory-cached selection
    values (select_rows_cached_kernel, default) against select_reg_kernel
    (select_cached 0) and the consumer: bit for bit. The cached kernel serves
    launches of more rows than SMs (160 (batch, kv head) rows here)."""
    b, n, n_kv, s, N, dtype = case
    h = 128
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, dtype)
    q = synth_matrix(3, b, n * h, dtype=dtype)
    for renorm in (False, True):
        cached = _decode(kc, cache, q, N, renorm, consume=0)
        reg = _decode(kc, cache, q, N, renorm, consume=0, select_cached=0)
        flow = _decode(kc, cache, q, N, renorm, consume=2)
        _same(cached, reg)
        _same(flow, reg)
    if s <= 1000:
        compare_all(oracle, cached, q, ks[0], vs[0], b, n, n_kv, h, s, N, True)
    cache.close()


def test_device_calls_order_before_later_calls(kc):
    """A device-mode call enqueued on one stream, then -- without a sync -- a
    device-mode call on another stream and a host-mode call: the later calls
    order after it (the store's device-work event), so every result equals a
    synchronised single call."""
    import torch
    b, n, h, s, N, L = 2, 8, 128, 20000, 64, 3  # >= 16 k: the dataflow path
    cache, ks, vs = build_cache(kc, b, n, n, h, s, "f16", n_layers=L)
    qs = [synth_matrix(40 + l, b, n * h) for l in range(L)]
    ref = [kc.decode_attention_topn(qs[l], cache, l, N, False) for l in range(L)]
    nc = min(N, s)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    dq = [torch.from_numpy(q).cuda() for q in qs]
    torch.cuda.synchronize()

    def outs():
        return [{"out": torch.full((b, n * h), float("nan"), device="cuda"),
                 "indices": torch.empty(b * n, nc, dtype=torch.int32, device="cuda"),
                 "weights": torch.empty(b * n, nc, device="cuda"),
                 "dropped": torch.empty(b * n, dtype=torch.float64, device="cuda")} for _ in range(L)]
    oa, ob = outs(), outs()
    for _ in range(2):
        cache.decode_topn_layers_device(list(range(L)), dq, N, oa, stream=sa)
        cache.decode_topn_layers_device(list(range(L)), dq, N, ob, stream=sb)
        host = kc.decode_attention_topn(qs[1], cache, 1, N, False)  # host mode, main stream
        np.testing.assert_array_equal(host.out, ref[1].out)
    torch.cuda.synchronize()
    for l in range(L):
        for o in (oa, ob):
            np.testing.assert_array_equal(o[l]["out"].cpu().numpy(), ref[l].out)
            np.testing.assert_array_equal(o[l]["indices"].cpu().numpy().view(np.uint32), ref[l].selection.indices)
    cache.close()


@pytest.mark.parametrize("flow_join", [1, 0])
def test_device_call_without_selection_outputs(kc, flow_join):
    """Device-mode GQA dataflow calls that return only the attention output
    (the caller's stream joins the consumer through the output stream and a
    marker kernel, flow_join 1, or directly): back-to-back single-layer calls
    equal the stream-ordered results bit for bit."""
    import torch
    b, n, n_kv, h, s, N, L = 2, 8, 2, 128, 3000, 64, 3
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s, "f16", n_layers=L)
    qs = [torch.from_numpy(synth_matrix(60 + l, b, n * h)).cuda() for l in range(L)]
    stream = torch.cuda.Stream()

    def run(consume):
        cache.set_tuning("consume", consume)
        outs = [torch.full((b, n * h), float("nan"), device="cuda") for _ in range(L)]
        for l in range(L):
            cache.decode_topn_layers_device([l], [qs[l]], N, [{"out": outs[l]}], stream=stream, want_selection=False)
        torch.cuda.synchronize()
        cache.set_tuning("consume", 1)
        return outs

    cache.set_tuning("flow_join", flow_join)
    ref = run(0)
    got = run(2)
    cache.set_tuning("flow_join", 1)
    for l in range(L):
        assert torch.equal(got[l], ref[l]), l
    cache.close()



def test_consumer_waits_for_counter_reset(kc):
    """The dataflow counters of a first call are zeroed on the caller's
    stream; the consumer (another stream) must order after that reset. Test
    hook dbg_ctr_race: the new counters start as 0xffffffff (a stale
    allocation) and the reset is delayed by 20 ms -- a consumer that polled
    them early would take every row as complete and read unwritten partials
    (seen as rare full-suite failures before the fix: weights off by 1e3
    with correct indices)."""
    b, n, h, s, N = 2, 8, 128, 20000, 64  # >= 16 k: the dataflow path
    cache, ks, vs = build_cache(kc, b, n, n, h, s, "f16")
    q = synth_matrix(9, b, n * h)
    ref = _decode(kc, cache, q, N, consume=0)
    # the consumer kernel loaded already (a first launch can synchronise the
    # context while the module loads, which would hide the race)
    _same(_decode(kc, cache, q, N, consume=2), ref)
    cache.close()
    cache, ks, vs = build_cache(kc, b, n, n, h, s, "f16")
    cache.set_tuning("dbg_ctr_race", 1)
    got = _decode(kc, cache, q, N, consume=2)
    _same(got, ref)
    cache.close()
