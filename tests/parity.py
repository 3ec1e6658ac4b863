"""Parity rules between the CUDA path and the CPU oracle.

* index sets identical, except positions whose oracle selection key lies
  within EPS_KEY (relative) of the N-th retained key;
* weights within W_RTOL relative;
* dropped mass within DROP_ATOL;
* outputs |out - ref| <= atol + OUT_RTOL*|ref| with atol = 1e-6*max|V|*sum(p_sel)
  (raw) or 1e-5*max|V| (renormalised), ref recomputed in fp64 over the GPU's own
  index set with the oracle's probabilities (so a legal boundary swap does not
  count twice). When the caller passes the group's logit magnitude
  L1 = scale * max_j sum_i |q_i k_ji| (large for peaked rows: ~60 for keys of
  6-8 against q in [0.5, 1]), atol grows by LOGIT_C * 2^-24 * sqrt(h) * L1 *
  max|V| * sum(p_sel): an fp32 dot of that magnitude summed in another order
  differs by ~u*sqrt(h)*L1 in the logit, which moves every p by that relative
  amount -- visible where the output cancels to ~0;
* ledger bytes exact.
"""
import numpy as np

EPS_KEY = 1e-5
W_RTOL = 1e-4
DROP_ATOL = 1e-6
OUT_RTOL = 1e-3
LOGIT_C = 4.0


def softmax_rows(q, kslot, h):
    """fp64 softmax of one q head against one kv slot (for tolerances only)."""
    s = (kslot.astype(np.float64) @ q.astype(np.float64)) * np.float64(np.float32(1.0) / np.sqrt(np.float32(h)))
    e = np.exp(s - s.max())
    return e / e.sum()


def check_group(gpu_idx, gpu_w, gpu_dropped, gpu_out, probs, vslot, top_n, renormalize, ora_idx=None,
                ora_w=None, ora_dropped=None, ora_out=None, logit_mag=0.0):
    """One (batch, kv head) group. probs [G][s] oracle fp32 probabilities,
    vslot [s][h]. gpu_* for the G q heads: idx [nc] (shared), w [G][nc],
    dropped [G], out [G][h]."""
    G, s = probs.shape
    nc = min(top_n, s)
    key = probs.sum(axis=0, dtype=np.float32) if G > 1 else probs[0]
    assert gpu_idx.shape == (nc,)
    assert np.all(np.diff(gpu_idx.astype(np.int64)) > 0), "indices not strictly ascending"
    assert gpu_idx.max() < s
    if ora_idx is None:
        order = np.lexsort((np.arange(s), -key.astype(np.float64)))
        ora_idx = np.sort(order[:nc])
    thr = key[ora_idx].min()
    diff = np.setxor1d(gpu_idx, ora_idx)
    for j in diff:
        assert abs(float(key[j]) - float(thr)) <= EPS_KEY * float(thr) + 1e-30, (
            f"index {j} (key {key[j]}) differs outside the epsilon window of the N-th key {thr}")
    for g in range(G):
        pw = probs[g][gpu_idx].astype(np.float64)
        np.testing.assert_allclose(gpu_w[g], pw, rtol=W_RTOL, atol=1e-12)
        assert abs(float(gpu_dropped[g]) - (1.0 - pw.sum())) <= DROP_ATOL
        v = vslot[gpu_idx].astype(np.float64)
        wsel = pw / pw.sum() if renormalize and pw.sum() > 0 else pw
        ref = wsel @ v
        vmax = float(np.abs(vslot).max()) if vslot.size else 0.0
        atol = 1e-5 * vmax if renormalize else 1e-6 * vmax * pw.sum()
        atol += LOGIT_C * 2.0**-24 * np.sqrt(vslot.shape[1]) * logit_mag * vmax * (1.0 if renormalize else pw.sum())
        atol = max(atol, 1e-7)
        err = np.abs(gpu_out[g].astype(np.float64) - ref)
        bound = atol + OUT_RTOL * np.abs(ref)
        worst = int(np.argmax(err - bound))
        assert np.all(err <= bound), f"head {g}: err {err[worst]} vs bound {bound[worst]} (ref {ref[worst]})"
        if ora_out is not None and diff.size == 0:
            err2 = np.abs(gpu_out[g].astype(np.float64) - ora_out[g].astype(np.float64))
            assert np.all(err2 <= atol + OUT_RTOL * np.abs(ora_out[g])), f"head {g}: vs oracle {err2.max()}"
    return diff.size
