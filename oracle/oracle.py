"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracle and the reference.

* ``Restatement`` wraps ``oracle/liboracle.so`` (kcache_oracle.c, the plain-C
  restatement of the reference hot path; every function cites the reference
  file:line it follows).
* ``Reference`` wraps ``oracle/_ref/libkcache_ref.so``: the unmodified
  reference core (proj/core/src/{matrix,model,kv_cache,attention}.cpp) built
  by ``oracle/Makefile`` plus a C-ABI shim (``oracle/ref_capi.cpp``).
* ``synth`` reproduces the reference's SeededRng stream
  (proj/core/include/kcache/rng.hpp:13-26) counter-indexed in numpy, rounded to
  the storage dtype, so the GPU and the oracle see identical inputs.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module; the product path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_c = ctypes
_fp = _c.POINTER(_c.c_float)
_u32p = _c.POINTER(_c.c_uint32)
_dp = _c.POINTER(_c.c_double)
_u64p = _c.POINTER(_c.c_uint64)
_sz = _c.c_size_t

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def build(ref: bool = True) -> None:
    """Compile the restatement (and the reference when its sources exist)."""
    target = "all" if ref else "restatement"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


# ---------------------------------------------------------------------------
# synthetic inputs (same stream as SeededRng; element order = append_kv rows)
def splitmix_at(seed: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def round_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)).astype(np.uint32)
    return r.view(np.float32)


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        return round_bf16(x)
    return x.astype(np.float32)


def synth(seed: int, idx: np.ndarray, lo: float = -1.0, hi: float = 1.0, dtype: str = "f16") -> np.ndarray:
    """Element(s) ``idx`` of SeededRng(seed).next_uniform(lo, hi), rounded to dtype."""
    u = (splitmix_at(seed, np.asarray(idx)) >> np.uint64(11)).astype(np.float64) * 2.0**-53
    f = u.astype(np.float32)
    x = np.float32(lo) + f * np.float32(np.float32(hi) - np.float32(lo))
    return round_to(x.astype(np.float32), dtype)


def synth_matrix(seed: int, rows: int, cols: int, lo=-1.0, hi=1.0, dtype="f16", offset=0) -> np.ndarray:
    idx = np.arange(offset, offset + rows * cols, dtype=np.uint64)
    return synth(seed, idx, lo, hi, dtype).reshape(rows, cols)


def synth_slot_rows(seed: int, s: int, batch: int, width: int, b: int, col0: int, h: int,
                    lo=-1.0, hi=1.0, dtype="f16") -> np.ndarray:
    """The s rows [pos][col0:col0+h] of batch row b of a position-major
    [s*batch][width] synthetic matrix, without generating the rest."""
    pos = np.arange(s, dtype=np.uint64)[:, None]
    col = np.arange(h, dtype=np.uint64)[None, :]
    idx = (pos * np.uint64(batch) + np.uint64(b)) * np.uint64(width) + np.uint64(col0) + col
    return synth(seed, idx, lo, hi, dtype)


# ---------------------------------------------------------------------------
def _f(a):
    return a.ctypes.data_as(_fp)


class Restatement:
    """oracle/liboracle.so (kcache_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        lib = _c.CDLL(path)
        lib.kco_uniform.restype = _c.c_float
        lib.kco_uniform.argtypes = [_c.c_uint64, _c.c_uint64, _c.c_float, _c.c_float]
        lib.kco_arg_topk.restype = _sz
        lib.kco_arg_topk.argtypes = [_fp, _sz, _sz, _u32p]
        lib.kco_softmax_inplace.argtypes = [_fp, _sz]
        lib.kco_decode_topn.restype = _c.c_int
        lib.kco_decode_topn.argtypes = [_sz] * 5 + [_fp] * 3 + [_sz, _c.c_int, _c.c_int, _fp, _u32p, _fp, _dp]
        lib.kco_decode_full.restype = _c.c_int
        lib.kco_decode_full.argtypes = [_sz] * 5 + [_fp] * 4
        lib.kco_decode_topn_group.restype = _c.c_int
        lib.kco_decode_topn_group.argtypes = [_sz] * 3 + [_fp] * 3 + [_sz, _c.c_int, _c.c_int, _fp, _u32p, _fp, _dp]
        lib.kco_head_weights.argtypes = [_sz, _sz, _fp, _fp, _fp]
        self.lib = lib

    def uniform(self, seed, i, lo=-1.0, hi=1.0):
        return self.lib.kco_uniform(seed, i, lo, hi)

    def arg_topk(self, values, k):
        v = np.ascontiguousarray(values, dtype=np.float32)
        out = np.zeros(max(len(v), 1), dtype=np.uint32)
        n = self.lib.kco_arg_topk(_f(v), len(v), k, out.ctypes.data_as(_u32p))
        if n == ctypes.c_size_t(-1).value:
            raise ValueError("arg_topk: k must be >= 1")
        return out[:n].copy()

    def softmax(self, row):
        r = np.array(row, dtype=np.float32)
        self.lib.kco_softmax_inplace(_f(r), len(r))
        return r

    def decode_topn(self, q, k, v, batch, n_heads, n_kv_heads, h, s, top_n, renormalize=False, ordered=True):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        nc = min(top_n, s)
        out = np.zeros((batch, n_heads * h), np.float32)
        idx = np.zeros((batch * n_heads, nc), np.uint32)
        w = np.zeros((batch * n_heads, nc), np.float32)
        dropped = np.zeros(batch * n_heads, np.float64)
        rc = self.lib.kco_decode_topn(batch, n_heads, n_kv_heads, h, s, _f(q), _f(k), _f(v), top_n,
                                      int(renormalize), int(ordered), _f(out),
                                      idx.ctypes.data_as(_u32p), _f(w), dropped.ctypes.data_as(_dp))
        if rc != 0:
            raise ValueError("oracle decode_topn rejected its arguments")
        return out, idx, w, dropped

    def decode_full(self, q, k, v, batch, n_heads, n_kv_heads, h, s):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros((batch, n_heads * h), np.float32)
        rc = self.lib.kco_decode_full(batch, n_heads, n_kv_heads, h, s, _f(q), _f(k), _f(v), _f(out))
        if rc != 0:
            raise ValueError("oracle decode_full rejected its arguments")
        return out

    def decode_topn_group(self, q_group, kslot, vslot, top_n, renormalize=False, ordered=True):
        q_group = np.ascontiguousarray(q_group, np.float32)
        kslot = np.ascontiguousarray(kslot, np.float32)
        vslot = np.ascontiguousarray(vslot, np.float32)
        G, h = q_group.shape
        s = kslot.shape[0]
        nc = min(top_n, s)
        out = np.zeros((G, h), np.float32)
        idx = np.zeros(nc, np.uint32)
        w = np.zeros((G, nc), np.float32)
        dropped = np.zeros(G, np.float64)
        rc = self.lib.kco_decode_topn_group(G, h, s, _f(q_group), _f(kslot), _f(vslot), top_n,
                                            int(renormalize), int(ordered), _f(out),
                                            idx.ctypes.data_as(_u32p), _f(w), dropped.ctypes.data_as(_dp))
        if rc != 0:
            raise ValueError("oracle decode_topn_group rejected its arguments")
        return out, idx, w, dropped

    def head_weights(self, qhead, kslot):
        qhead = np.ascontiguousarray(qhead, np.float32)
        kslot = np.ascontiguousarray(kslot, np.float32)
        s, h = kslot.shape
        p = np.zeros(s, np.float32)
        self.lib.kco_head_weights(h, s, _f(qhead), _f(kslot), _f(p))
        return p


REF_ERRORS = {1: "ShapeError", 2: "StateError", 3: "CapacityError", 4: "invalid_argument",
              5: "out_of_range", 9: "exception"}


class Reference:
    """oracle/_ref/libkcache_ref.so: the unmodified reference core + shim."""

    PATH = os.path.join(HERE, "_ref", "libkcache_ref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        lib = _c.CDLL(self.PATH)
        lib.kcref_last_error.restype = _c.c_char_p
        lib.kcref_decode_topn.restype = _c.c_int
        lib.kcref_decode_topn.argtypes = [_sz] * 4 + [_fp] * 3 + [_sz, _c.c_int, _c.c_int, _c.c_int,
                                                                  _fp, _u32p, _fp, _dp, _u64p, _u64p]
        lib.kcref_decode_full.restype = _c.c_int
        lib.kcref_decode_full.argtypes = [_sz] * 4 + [_fp] * 3 + [_c.c_int, _fp]
        lib.kcref_prefill.restype = _c.c_int
        lib.kcref_prefill.argtypes = [_sz] * 3 + [_fp] * 4
        lib.kcref_arg_topk.restype = _c.c_long
        lib.kcref_arg_topk.argtypes = [_fp, _sz, _sz, _u32p]
        lib.kcref_softmax.argtypes = [_fp, _sz]
        lib.kcref_rng_uniform.argtypes = [_c.c_uint64, _sz, _c.c_float, _c.c_float, _fp]
        lib.kcref_bench_create.restype = _c.c_void_p
        lib.kcref_bench_create.argtypes = [_sz] * 6 + [_c.c_int, _c.c_uint, _c.c_uint64, _c.c_uint64, _c.c_uint64,
                                                       _sz]
        lib.kcref_bench_run.restype = _c.c_double
        lib.kcref_bench_run.argtypes = [_c.c_void_p, _dp]
        lib.kcref_bench_destroy.argtypes = [_c.c_void_p]
        self.lib = lib

    def _err(self, rc):
        raise RuntimeError(f"reference {REF_ERRORS.get(rc, rc)}: {self.lib.kcref_last_error().decode()}")

    def prefill_attention(self, q, k, v, n_heads):
        q, k, v = (np.ascontiguousarray(a, np.float32) for a in (q, k, v))
        s, d = q.shape
        out = np.zeros((s, d), np.float32)
        rc = self.lib.kcref_prefill(s, n_heads, d // n_heads, _f(q), _f(k), _f(v), _f(out))
        if rc:
            self._err(rc)
        return out

    def decode_topn(self, q, k, v, batch, n_heads, h, s, top_n, renormalize=False, ordered=True, resident=False):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        nc = min(top_n, s)
        out = np.zeros((batch, n_heads * h), np.float32)
        idx = np.zeros((batch * n_heads, nc), np.uint32)
        w = np.zeros((batch * n_heads, nc), np.float32)
        dropped = np.zeros(batch * n_heads, np.float64)
        h2d = _c.c_uint64(0)
        tot = _c.c_uint64(0)
        rc = self.lib.kcref_decode_topn(batch, n_heads, h, s, _f(q), _f(k), _f(v), top_n, int(renormalize),
                                        int(ordered), int(resident), _f(out), idx.ctypes.data_as(_u32p), _f(w),
                                        dropped.ctypes.data_as(_dp), _c.byref(h2d), _c.byref(tot))
        if rc != 0:
            self._err(rc)
        return out, idx, w, dropped, h2d.value

    def decode_full(self, q, k, v, batch, n_heads, h, s, resident=False):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros((batch, n_heads * h), np.float32)
        rc = self.lib.kcref_decode_full(batch, n_heads, h, s, _f(q), _f(k), _f(v), int(resident), _f(out))
        if rc != 0:
            self._err(rc)
        return out

    def arg_topk(self, values, k):
        v = np.ascontiguousarray(values, dtype=np.float32)
        out = np.zeros(max(len(v), 1), dtype=np.uint32)
        n = self.lib.kcref_arg_topk(_f(v), len(v), k, out.ctypes.data_as(_u32p))
        if n < 0:
            self._err(-n)
        return out[:n].copy()

    def softmax(self, row):
        r = np.array(row, dtype=np.float32)
        self.lib.kcref_softmax(_f(r), len(r))
        return r

    def rng_uniform(self, seed, n, lo=-1.0, hi=1.0):
        out = np.zeros(n, np.float32)
        self.lib.kcref_rng_uniform(seed, n, lo, hi, _f(out))
        return out


class ReferenceBench:
    """The reference decode_attention_topn timed on host threads (cpu baseline)."""

    def __init__(self, s, batch, n_heads, h, heads_per_shard, top_n, threads, seeds=(1, 2, 3), renormalize=False,
                 n_layers=1):
        self.ref = Reference()
        self.handle = self.ref.lib.kcref_bench_create(s, batch, n_heads, h, heads_per_shard, top_n,
                                                      int(renormalize), threads, *seeds, n_layers)
        if not self.handle:
            raise RuntimeError(self.ref.lib.kcref_last_error().decode())

    def run(self):
        cs = _c.c_double(0)
        t = self.ref.lib.kcref_bench_run(self.handle, _c.byref(cs))
        return t, cs.value

    def close(self):
        if self.handle:
            self.ref.lib.kcref_bench_destroy(self.handle)
            self.handle = None
