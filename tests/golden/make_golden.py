"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

    make -C oracle && python tests/golden/make_golden.py

Runs in the build container (needs /root/reference to have built
oracle/_ref/libkcache_ref.so). Inputs are SeededRng streams so only seeds and
shapes are stored; outputs come from the reference's own
decode_attention_topn / decode_attention_full / arg_topk / softmax_inplace and
SeededRng::next_uniform (proj/core/src/{attention,matrix}.cpp,
proj/core/include/kcache/rng.hpp). The committed golden.npz pins the oracle
restatement (tests/test_oracle_golden.py) on machines without the reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference, synth_matrix  # noqa: E402

# (batch, n_heads, head_dim, s, top_n, renormalize, ordered, resident, input dtype, lo, hi)
TOPN_CASES = [
    (2, 4, 16, 50, 8, 0, 1, 0, "f16", -1.0, 1.0),
    (2, 4, 16, 50, 8, 1, 1, 0, "f16", -1.0, 1.0),
    (2, 4, 16, 50, 8, 0, 0, 0, "f16", -1.0, 1.0),
    (1, 1, 1, 4, 2, 0, 1, 0, "f32", -1.0, 1.0),
    (3, 2, 8, 33, 40, 0, 1, 0, "f32", -1.0, 1.0),
    (3, 2, 8, 33, 40, 1, 1, 1, "f32", -1.0, 1.0),
    (1, 32, 128, 300, 128, 0, 1, 0, "f16", -1.0, 1.0),
    (1, 8, 128, 700, 64, 1, 1, 0, "bf16", -2.0, 2.0),
    (2, 4, 64, 129, 1, 0, 1, 0, "f16", -1.0, 1.0),
    (1, 4, 32, 256, 256, 0, 1, 0, "f32", -1.0, 1.0),
]
FULL_CASES = [(2, 4, 16, 50, "f16"), (1, 8, 128, 300, "f16"), (3, 2, 8, 33, "f32")]


def case_inputs(b, n, h, s, dtype, lo, hi, seed0):
    d = n * h
    q = synth_matrix(seed0 + 1, b, d, lo, hi, dtype)
    k = synth_matrix(seed0 + 2, s * b, d, lo, hi, dtype)
    v = synth_matrix(seed0 + 3, s * b, d, -1.0, 1.0, dtype)
    return q, k, v


def main():
    ref = Reference()
    out = {}
    meta = {"topn": [], "full": []}
    for ci, (b, n, h, s, N, renorm, ordered, resident, dt, lo, hi) in enumerate(TOPN_CASES):
        q, k, v = case_inputs(b, n, h, s, dt, lo, hi, 100 * ci)
        o, idx, w, dr, h2d = ref.decode_topn(q, k, v, b, n, h, s, N, bool(renorm), bool(ordered), bool(resident))
        out[f"topn{ci}_out"] = o
        out[f"topn{ci}_idx"] = idx
        out[f"topn{ci}_w"] = w
        out[f"topn{ci}_dropped"] = dr
        meta["topn"].append(dict(b=b, n=n, h=h, s=s, N=N, renorm=renorm, ordered=ordered, resident=resident,
                                 dtype=dt, lo=lo, hi=hi, seed0=100 * ci, h2d=h2d))
    for ci, (b, n, h, s, dt) in enumerate(FULL_CASES):
        q, k, v = case_inputs(b, n, h, s, dt, -1.0, 1.0, 1000 + 100 * ci)
        out[f"full{ci}_out"] = ref.decode_full(q, k, v, b, n, h, s)
        meta["full"].append(dict(b=b, n=n, h=h, s=s, dtype=dt, seed0=1000 + 100 * ci))
    # arg_topk on random rows with planted ties, and the reference's softmax
    rng = np.random.default_rng(7)
    topk = []
    for ci in range(40):
        n_ = int(rng.integers(1, 300))
        vals = rng.integers(-20, 20, n_).astype(np.float32) / 8.0  # many exact ties
        k_ = int(rng.integers(1, 320))
        out[f"argtopk{ci}_vals"] = vals
        out[f"argtopk{ci}_idx"] = ref.arg_topk(vals, k_)
        topk.append(k_)
    meta["argtopk_k"] = topk
    row = rng.standard_normal(1000).astype(np.float32) * 5
    out["softmax_in"] = row
    out["softmax_out"] = ref.softmax(row)
    for seed in (1, 2, 3, 12345):
        out[f"rng{seed}"] = ref.rng_uniform(seed, 257, -1.0, 1.0)
    out["rng7_narrow"] = ref.rng_uniform(7, 257, -0.05, 0.05)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
