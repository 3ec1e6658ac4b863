"""Engine decode-step attention block (proj/core/src/engine.cpp:139-160)
through kc_decode_step: per layer, append this step's K/V row of every batch
row, then TopN (offloaded layers) or full attention (resident layers), with
StepStats (engine.hpp:37-45) accumulated on the device -- checked against the
CPU oracle on the grown cache and against the engine's own stats rules."""
import numpy as np
import pytest

from oracle.oracle import synth_matrix
from tests.test_gpu_parity import build_cache

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,n_kv,dtype", [(4, 4, "f16"), (8, 4, "bf16")], ids=["mha-f16", "gqa-bf16"])
def test_decode_steps_vs_oracle_and_stats(kc, oracle, n, n_kv, dtype):
    b, h, s0, N, L, steps = 2, 128, 300, 32, 2, 3
    G = n // n_kv
    cache, ks, vs = build_cache(kc, b, n, n_kv, h, s0, dtype, resident=1, n_layers=L, max_seq=s0 + steps)
    cache.step_stats(reset=True)
    d2h0 = cache.d2h_bytes_total()
    for step in range(steps):
        s = s0 + step + 1
        want_hist = np.zeros(8, np.int64)
        want_dropped = 0.0
        for layer in range(L):
            knew = synth_matrix(500 + 10 * step + layer, b, n_kv * h, dtype=dtype)
            vnew = synth_matrix(600 + 10 * step + layer, b, n_kv * h, dtype=dtype)
            q = synth_matrix(700 + 10 * step + layer, b, n * h, dtype=dtype)
            ks[layer] = np.concatenate([ks[layer], knew])
            vs[layer] = np.concatenate([vs[layer], vnew])
            full = layer < 1  # the engine runs full attention on V-resident layers
            out = cache.decode_step(layer, q, knew, vnew, N, full=full)
            assert cache.current_len() == s
            if full:
                want = oracle.decode_full(q, ks[layer], vs[layer], b, n, n_kv, h, s)
                np.testing.assert_allclose(out, want, rtol=1e-3, atol=1e-6)
                continue
            o_out, o_idx, o_w, o_dr = oracle.decode_topn(q, ks[layer], vs[layer], b, n, n_kv, h, s, N, False, True)
            np.testing.assert_allclose(out, o_out, rtol=1e-3, atol=1e-5 * np.abs(o_out).max())
            for slot in range(b * n):
                for idx in o_idx[slot]:
                    want_hist[min(7, int(idx) * 8 // s)] += 1
                want_dropped += float(o_dr[slot])
        st = cache.step_stats(reset=True)
        nc = min(N, s)
        assert st["h2d_bytes"] == 2 * b * n_kv * nc * h  # one TopN layer, kv-head row sets
        assert st["d2h_bytes"] == 2 * b * n_kv * h        # the offloaded layer's new V row
        assert st["selections"] == b * n
        assert st["position_histogram"] == want_hist.tolist()
        assert sum(st["position_histogram"]) == b * n * nc
        assert abs(st["dropped_sum"] - want_dropped) <= 1e-6 * b * n
        assert abs(st["mean_dropped_mass"] - want_dropped / (b * n)) <= 1e-6
    assert cache.d2h_bytes_total() - d2h0 == steps * 2 * b * n_kv * h
    # every step row landed where the reference's append_kv puts it
    for layer in range(L):
        for pos in (s0, s0 + steps - 1):
            for bb in range(b):
                np.testing.assert_array_equal(cache.v_row(layer, pos, bb), vs[layer][pos * b + bb])
    cache.close()


def test_decode_step_device_equals_host(kc):
    import torch
    b, n, h, s0, N = 2, 4, 128, 200, 16
    outs = []
    for device in (False, True):
        cache, ks, vs = build_cache(kc, b, n, n, h, s0, "f16", n_layers=1, max_seq=s0 + 2)
        knew = synth_matrix(55, b, n * h)
        vnew = synth_matrix(56, b, n * h)
        q = synth_matrix(57, b, n * h)
        if device:
            out = torch.empty(b, n * h, dtype=torch.float32, device="cuda")
            cache.decode_step_device(0, torch.from_numpy(q).cuda(), torch.from_numpy(knew).cuda(),
                                     torch.from_numpy(vnew).cuda(), out, N)
            torch.cuda.synchronize()
            outs.append((out.cpu().numpy(), cache.step_stats()))
        else:
            outs.append((cache.decode_step(0, q, knew, vnew, N), cache.step_stats()))
        cache.close()
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]


def test_decode_step_errors(kc):
    b, n, h, s0 = 1, 2, 128, 10
    cache, ks, vs = build_cache(kc, b, n, n, h, s0, "f16", n_layers=1, max_seq=s0 + 1)
    q = synth_matrix(1, b, n * h)
    row = synth_matrix(2, b, n * h)
    with pytest.raises(ValueError):
        cache.decode_step(0, q, row, row, 0)  # top_n = 0 (attention.cpp:119-122)
    cache.decode_step(0, q, row, row, 4)
    with pytest.raises(kc.StateError):
        cache.decode_step(0, q, row, row, 4)  # past max_seq (kv_cache.cpp:117-119)
    with pytest.raises(kc.ShapeError):
        cache.decode_step(0, q, row[:, :h], row, 4)
    cache.close()


@pytest.mark.parametrize("n,n_kv,dtype,consume", [(4, 4, "f16", 1), (8, 2, "bf16", 1), (4, 4, "f16", 2)],
                         ids=["mha-f16", "gqa-bf16", "mha-f16-dataflow"])
def test_step_graph_equals_eager(kc, n, n_kv, dtype, consume):
    """One CUDA Graph per decode step (kc_step_graph_begin / _launch): the
    captured-then-launched step writes the same outputs, bit for bit, and the
    same StepStats, ledger bytes and cache rows as the eager calls (consume 2:
    the dataflow consumer, eagerly beside its scoring, in the graph after it)."""
    import torch
    b, h, s0, N, L, steps = 2, 128, 500, 64, 3, 3
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16}[dtype]
    runs = []
    for graph in (False, True):
        cache, ks, vs = build_cache(kc, b, n, n_kv, h, s0, dtype, resident=1, n_layers=L, max_seq=s0 + steps + 1)
        cache.set_tuning("consume", consume)
        stream = torch.cuda.Stream()
        cache.step_stats(reset=True)
        outs, stats = [], []
        for step in range(steps):
            ins = [[torch.from_numpy(synth_matrix(900 + 10 * step + l + 100 * j, b, (n if j == 0 else n_kv) * h,
                                                  dtype=dtype)).to(tdt).cuda() for j in range(3)] for l in range(L)]
            out = [torch.full((b, n * h), float("nan"), dtype=torch.float32, device="cuda") for _ in range(L)]
            torch.cuda.synchronize()
            if graph:
                cache.step_graph_begin(N, stream)
            for l in range(L):
                cache.decode_step_device(l, ins[l][0], ins[l][1], ins[l][2], out[l], N, full=l < 1, stream=stream)
            if graph:
                cache.step_graph_launch(stream)
            stream.synchronize()
            outs.append([o.cpu().numpy() for o in out])
            stats.append(cache.step_stats(reset=True))
        rows = [cache.v_row(l, s0 + steps - 1, bb) for l in range(L) for bb in range(b)]
        runs.append((outs, stats, cache.d2h_bytes_total(), cache.h2d_bytes_total(), rows))
        cache.close()
    (eo, es, ed, eh, er), (go, gs, gd, gh, gr) = runs
    for step in range(steps):
        for l in range(L):
            assert not np.isnan(go[step][l]).any()
            np.testing.assert_array_equal(go[step][l], eo[step][l])
        assert gs[step] == es[step]
    assert (gd, gh) == (ed, eh)
    for a, c in zip(gr, er):
        np.testing.assert_array_equal(a, c)


def test_step_graph_rejects_host_io(kc):
    import torch
    b, n, h, s0 = 1, 2, 128, 100
    cache, ks, vs = build_cache(kc, b, n, n, h, s0, "f16", n_layers=1, max_seq=s0 + 2)
    stream = torch.cuda.Stream()
    cache.step_graph_begin(8, stream)
    with pytest.raises(kc.StateError):
        cache.decode_step(0, synth_matrix(1, b, n * h), synth_matrix(2, b, n * h), synth_matrix(3, b, n * h), 8)
    with pytest.raises(kc.StateError):
        cache.step_graph_begin(8, stream)  # one capture at a time
    cache.step_graph_launch(stream)  # ends the (empty) capture
    stream.synchronize()
    cache.close()


def test_gqa_engine_step_dataflow_equals_stream_ordered(kc):
    """kc_decode_step on a GQA cache through the dataflow consumer (consume 2,
    16 k positions, 64 rows, its small auto grid) equals the stream-ordered
    step bit for bit, layer after layer with the append and fp16 q of an
    engine step."""
    import torch
    b, n, n_kv, h, s, N, L, steps = 8, 32, 8, 128, 16384, 128, 2, 3
    cfg = kc.small_config(L, n * h, n, s + 16, kv_heads=n_kv)
    outs = {}
    for consume in (0, 2):
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
        cache.set_tuning("consume", consume)
        stream = torch.cuda.Stream()
        # every step's inputs stay alive until the stream is done with them
        # (the calls are asynchronous on `stream`)
        ins = []
        for t in range(steps):
            for l in range(L):
                q = torch.empty(b, n * h, dtype=torch.float16, device="cuda")
                kv = torch.empty(2, b, n_kv * h, dtype=torch.float16, device="cuda")
                kc.fill_uniform(q, 500 + 10 * t + l)
                kc.fill_uniform(kv, 700 + 10 * t + l)
                ins.append((l, q, kv, torch.empty(b, n * h, device="cuda")))
        torch.cuda.synchronize()
        res = []
        for l, q, kv, out in ins:
            cache.decode_step_device(l, q, kv[0], kv[1], out, N, stream=stream)
            res.append(out)
        torch.cuda.synchronize()
        outs[consume] = [r.cpu() for r in res]
        cache.close()
    diffs = [float((a - c).abs().max()) for a, c in zip(outs[0], outs[2])]
    assert all(d == 0.0 for d in diffs), diffs
