"""Python mirror of the reference's KCache operator API over the C ABI.

The reference exposes its decode-step TopN attention as C++
(proj/core/include/kcache/{attention,kv_cache,matrix,model}.hpp); this module
gives the same names, argument meanings and error behaviour in Python, bound
with ctypes to ``libkcache_b200.so`` (include/kcache_c.h). All compute runs in
the library's sm_100a kernels; there is no CPU path, and importing this module
fails loudly when the library has not been built.

    cfg = ModelConfig(n_layers=1, d_model=4096, n_heads=32, head_dim=128,
                      ffn_hidden=ModelConfig.default_ffn_hidden(4096), vocab=64,
                      max_seq=4096)
    cache = TieredKVCache(cfg, batch=1, placement=TierPlacement.kcache(0, 1))
    cache.append_kv(0, k_rows, v_rows); cache.offload_prefill_v(0); cache.begin_decode()
    res = decode_attention_topn(q, cache, 0, top_n=128, renormalize=False)

Exceptions map like the C++ shim: ShapeError (ValueError), StateError,
CapacityError (RuntimeError), ``invalid_argument`` -> ValueError,
``out_of_range`` -> IndexError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkcache_b200.so")

KC_OK, KC_ESHAPE, KC_ESTATE, KC_ECAPACITY, KC_EARG, KC_ERANGE, KC_ECUDA, KC_EOVERFLOW = range(8)
KC_F32, KC_F16, KC_BF16 = 0, 1, 2
KC_RENORMALIZE, KC_REVERSE_ACCUM, KC_IO_DEVICE, KC_FULL = 1, 2, 4, 8
DTYPES = {"f32": KC_F32, "f16": KC_F16, "bf16": KC_BF16}


class ShapeError(ValueError):
    """kcache::ShapeError (errors.hpp:10-14)."""


class StateError(RuntimeError):
    """kcache::StateError (errors.hpp:16-21)."""


class CapacityError(RuntimeError):
    """kcache::CapacityError (errors.hpp:34-38)."""


class CudaError(RuntimeError):
    pass


class _Config(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "max_seq")]


class _TopnOut(C.Structure):
    _fields_ = [("out", C.c_void_p), ("indices", C.c_void_p), ("weights", C.c_void_p),
                ("dropped_mass", C.c_void_p), ("nc", C.c_uint64), ("h2d_bytes", C.c_uint64)]


class _StepStats(C.Structure):
    _fields_ = [("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("selections", C.c_uint64),
                ("dropped_sum", C.c_double), ("position_histogram", C.c_uint64 * 8)]


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libkcache_b200.so (raises ImportError if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    u64, vp, i32, u32 = C.c_uint64, C.c_void_p, C.c_int, C.c_uint32
    p64 = C.POINTER(C.c_uint64)
    sig = {
        "kc_last_error": (C.c_char_p, []),
        "kc_version": (C.c_char_p, []),
        "kc_cache_create": (i32, [C.POINTER(_Config), u64, u64, u64, i32, i32, u64, i32, i32, C.POINTER(vp)]),
        "kc_cache_destroy": (i32, [vp]),
        "kc_append_kv": (i32, [vp, u64, vp, vp, u64]),
        "kc_append_kv_device": (i32, [vp, u64, vp, vp, i32, u64, vp]),
        "kc_offload_prefill_v": (i32, [vp, u64]),
        "kc_begin_decode": (i32, [vp]),
        "kc_decode_topn": (i32, [vp, u64, vp, i32, u64, u32, C.POINTER(_TopnOut), vp]),
        "kc_decode_topn_layers": (i32, [vp, u64, p64, C.POINTER(vp), i32, u64, u32, C.POINTER(_TopnOut), vp]),
        "kc_decode_full": (i32, [vp, u64, vp, i32, u32, vp, vp]),
        "kc_decode_step": (i32, [vp, u64, vp, vp, vp, i32, u64, u32, vp, vp]),
        "kc_step_stats_read": (i32, [vp, C.POINTER(_StepStats), i32]),
        "kc_step_graph_begin": (i32, [vp, u64, vp]),
        "kc_step_graph_launch": (i32, [vp, vp]),
        "kc_score_probs": (i32, [vp, u64, vp, i32, vp]),
        "kc_gather_v": (i32, [vp, u64, vp, vp, vp, p64]),
        "kc_read_row": (i32, [vp, u64, u64, u64, i32, vp]),
        "kc_current_len": (i32, [vp, p64]),
        "kc_phase": (i32, [vp, C.POINTER(i32)]),
        "kc_fast_bytes_used": (i32, [vp, p64]),
        "kc_slow_bytes_used": (i32, [vp, p64]),
        "kc_d2h_bytes_total": (i32, [vp, p64]),
        "kc_h2d_bytes_total": (i32, [vp, p64]),
        "kc_ledger_size": (i32, [vp, p64]),
        "kc_ledger_event": (i32, [vp, u64, C.POINTER(i32), p64, C.POINTER(i32), p64, p64]),
        "kc_layer_storage": (i32, [vp, u64, C.POINTER(vp), C.POINTER(vp), C.POINTER(i32)]),
        "kc_sync": (i32, [vp]),
        "kc_v_arena_kind": (i32, [vp, C.POINTER(i32)]),
        "kc_set_tuning": (i32, [vp, C.c_char_p, C.c_int64]),
        "kc_profile": (i32, [vp, i32]),
        "kc_profile_read": (i32, [vp, C.c_char_p, C.POINTER(C.c_double), p64]),
        "kc_profile_launch": (i32, [vp, C.c_char_p, u64, C.POINTER(C.c_double)]),
        "kc_profile_span": (i32, [vp, C.c_char_p, u64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "kc_arg_topk": (i32, [vp, u64, u64, vp, p64]),
        "kc_score_chunk_plan": (i32, [u64, u64, u64, C.POINTER(C.c_int64)]),
        "kc_debug_read": (i32, [vp, C.c_char_p, vp, u64]),
        "kc_prefill_attention": (i32, [vp, vp, vp, u64, u64, u64, vp, i32]),
        "kc_prefill_attention_device": (i32, [vp, vp, vp, u64, u64, u64, vp, vp]),
        "kc_fill_uniform": (i32, [vp, i32, u64, u64, u64, C.c_float, C.c_float, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc == KC_OK:
        return
    msg = load().kc_last_error().decode()
    if rc == KC_ESHAPE:
        raise ShapeError(msg)
    if rc == KC_ESTATE:
        raise StateError(msg)
    if rc == KC_ECAPACITY:
        raise CapacityError(msg)
    if rc == KC_EARG:
        raise ValueError(msg)
    if rc == KC_ERANGE:
        raise IndexError(msg)
    if rc == KC_EOVERFLOW:
        raise OverflowError(msg)
    raise CudaError(msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------------------
# model.hpp
@dataclasses.dataclass
class ModelConfig:
    """ModelConfig (model.hpp:18-40); n_kv_heads=0 means MHA (the reference)."""
    n_layers: int = 0
    d_model: int = 0
    n_heads: int = 0
    head_dim: int = 0
    ffn_hidden: int = 0
    vocab: int = 0
    max_seq: int = 0
    n_kv_heads: int = 0

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    def validate(self) -> None:
        if min(self.n_layers, self.d_model, self.n_heads, self.head_dim, self.max_seq) < 1:
            raise ShapeError("ModelConfig: all counts must be >= 1")
        if self.ffn_hidden < 1:
            raise ShapeError("ModelConfig: ffn_hidden must be >= 1")
        if self.vocab < 2:
            raise ShapeError("ModelConfig: vocab must be >= 2")
        if self.d_model != self.n_heads * self.head_dim:
            raise ShapeError("ModelConfig: d_model must equal n_heads * head_dim")
        if self.n_heads % self.kv_heads:
            raise ShapeError("ModelConfig: n_kv_heads must divide n_heads")

    @staticmethod
    def default_ffn_hidden(d_model: int) -> int:
        return ((8 * d_model + 2) // 3 + 15) // 16 * 16

    @staticmethod
    def toy() -> "ModelConfig":
        return ModelConfig(4, 64, 4, 16, 176, 256, 4096)

    @staticmethod
    def shape_7b() -> "ModelConfig":
        return ModelConfig(32, 4096, 32, 128, ModelConfig.default_ffn_hidden(4096), 32000, 32768)


def small_config(layers: int, d: int, heads: int, max_seq: int = 8192, kv_heads: int = 0) -> ModelConfig:
    """The reference tests' helper (proj/tests/test_attention.cpp:15-25)."""
    return ModelConfig(layers, d, heads, d // heads, ModelConfig.default_ffn_hidden(d), 64, max_seq, kv_heads)


# ---------------------------------------------------------------------------
# kv_cache.hpp
@dataclasses.dataclass
class TierPlacement:
    """TierPlacement (kv_cache.hpp:50-65) + the physical storage dtype."""
    resident_layers: int = 0
    n_layers: int = 0
    bytes_per_element: int = 2
    storage: str = "f32"

    @staticmethod
    def baseline(n_layers: int, bytes_per_element: int = 2, storage: str = "f32") -> "TierPlacement":
        return TierPlacement(n_layers, n_layers, bytes_per_element, storage)

    @staticmethod
    def kcache(resident_layers: int, n_layers: int, bytes_per_element: int = 2, storage: str = "f32") -> "TierPlacement":
        return TierPlacement(resident_layers, n_layers, bytes_per_element, storage)

    def validate(self) -> None:
        if self.resident_layers > self.n_layers:
            raise ShapeError("TierPlacement: resident_layers must be <= n_layers")
        if self.bytes_per_element == 0:
            raise ShapeError("TierPlacement: bytes_per_element must be >= 1")

    def v_resident(self, layer: int) -> bool:
        return layer < self.resident_layers


@dataclasses.dataclass
class TransferEvent:
    phase: str
    layer: int
    dir: str
    bytes: int
    elements: int


@dataclasses.dataclass
class GatheredV:
    head_dim: int
    blocks: list
    h2d_bytes: int


@dataclasses.dataclass
class TopNSelection:
    """TopNSelection (attention.hpp:20-30); arrays are [slot][nc]."""
    batch: int
    n_heads: int
    indices: np.ndarray
    weights: np.ndarray
    dropped_mass: np.ndarray

    def slot(self, batch_idx: int, head: int) -> int:
        return batch_idx * self.n_heads + head


@dataclasses.dataclass
class TopNResult:
    out: np.ndarray
    selection: TopNSelection
    h2d_bytes: int


def footprint(config: ModelConfig, batch: int, seq_len: int, mode: str, resident_layers: int,
              bytes_per_element: int) -> dict:
    """memory_footprint (kv_cache.cpp:48-66), without the weight term."""
    per_layer = bytes_per_element * batch * seq_len * config.d_model
    if mode == "baseline":
        return {"fast_bytes": 2 * per_layer * config.n_layers, "slow_bytes": 0}
    return {"fast_bytes": per_layer * (config.n_layers + resident_layers),
            "slow_bytes": per_layer * (config.n_layers - resident_layers)}


class TieredKVCache:
    """TieredKVCache (kv_cache.hpp:98-154) backed by HBM K / pinned-host V."""

    def __init__(self, config: ModelConfig, batch: int, placement: TierPlacement,
                 fast_capacity_bytes: Optional[int] = None, device: int = 0, numa_node: int = -1):
        lib = load()
        config.validate()
        placement.validate()
        if placement.n_layers != config.n_layers:
            raise ShapeError("TieredKVCache: placement layer count differs from config")
        if batch == 0:
            raise ShapeError("TieredKVCache: batch must be >= 1")
        self.config = config
        self.batch = batch
        self.placement = placement
        self._h = C.c_void_p()
        cfg = _Config(config.n_layers, config.d_model, config.n_heads, config.kv_heads, config.head_dim,
                      config.max_seq)
        _check(lib.kc_cache_create(C.byref(cfg), batch, placement.resident_layers, placement.bytes_per_element,
                                   DTYPES[placement.storage], int(fast_capacity_bytes is not None),
                                   fast_capacity_bytes or 0, device, numa_node, C.byref(self._h)))
        self._lib = lib

    def close(self) -> None:
        if self._h:
            self._lib.kc_cache_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def kv_width(self) -> int:
        return self.config.kv_heads * self.config.head_dim

    def append_kv(self, layer: int, k_rows, v_rows) -> None:
        """k_rows/v_rows: [m*batch][n_kv*h] position-major fp32 (host)."""
        if layer >= self.config.n_layers:
            raise IndexError(f"TieredKVCache: layer {layer} out of range")
        k = _f32(k_rows)
        v = _f32(v_rows)
        if k.ndim != 2 or v.ndim != 2 or k.shape[1] != self.kv_width or v.shape[1] != self.kv_width:
            raise ShapeError("append_kv: row width must equal d_model")
        if k.shape[0] != v.shape[0] or k.shape[0] == 0 or k.shape[0] % self.batch:
            raise ShapeError("append_kv: need a positive multiple of batch rows for K and V")
        _check(self._lib.kc_append_kv(self._h, layer, _ptr(k), _ptr(v), k.shape[0]))

    def append_kv_device(self, layer: int, k, v, stream=None) -> None:
        """Device (torch CUDA) rows of any storage dtype, async on `stream`."""
        import torch
        dt = {torch.float32: KC_F32, torch.float16: KC_F16, torch.bfloat16: KC_BF16}[k.dtype]
        assert k.is_contiguous() and v.is_contiguous() and k.shape == v.shape and k.dtype == v.dtype
        rows = k.numel() // self.kv_width
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(self._lib.kc_append_kv_device(self._h, layer, k.data_ptr(), v.data_ptr(), dt, rows, st))

    def offload_prefill_v(self, layer: int) -> None:
        _check(self._lib.kc_offload_prefill_v(self._h, layer))

    def begin_decode(self) -> None:
        _check(self._lib.kc_begin_decode(self._h))

    def gather_v(self, layer: int, selection: Sequence[Sequence[int]]) -> GatheredV:
        if layer >= self.config.n_layers:
            raise IndexError(f"TieredKVCache: layer {layer} out of range")
        if len(selection) != self.batch * self.config.n_heads:
            raise ShapeError("gather_v: selection must cover batch * n_heads slots")
        counts = np.array([len(s) for s in selection], dtype=np.uint64)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.uint32) for s in selection])
                                    if len(selection) else np.zeros(0, np.uint32), dtype=np.uint32)
        h = self.config.head_dim
        out = np.zeros((max(int(counts.sum()), 1), h), np.float32)
        h2d = C.c_uint64(0)
        _check(self._lib.kc_gather_v(self._h, layer, _ptr(flat) if flat.size else None, _ptr(counts), _ptr(out),
                                     C.byref(h2d)))
        blocks, off = [], 0
        for c in counts:
            blocks.append(out[off:off + int(c)].copy())
            off += int(c)
        return GatheredV(h, blocks, h2d.value)

    def _row(self, layer, pos, b, which):
        out = np.zeros(self.kv_width, np.float32)
        _check(self._lib.kc_read_row(self._h, layer, pos, b, which, _ptr(out)))
        return out

    def k_row(self, layer: int, pos: int, batch_idx: int) -> np.ndarray:
        return self._row(layer, pos, batch_idx, 0)

    def v_row(self, layer: int, pos: int, batch_idx: int) -> np.ndarray:
        return self._row(layer, pos, batch_idx, 1)

    def _u64(self, fn) -> int:
        x = C.c_uint64(0)
        _check(fn(self._h, C.byref(x)))
        return x.value

    def current_len(self) -> int:
        return self._u64(self._lib.kc_current_len)

    def phase(self) -> str:
        x = C.c_int(0)
        _check(self._lib.kc_phase(self._h, C.byref(x)))
        return "prefill" if x.value == 0 else "decode"

    def fast_bytes_used(self) -> int:
        return self._u64(self._lib.kc_fast_bytes_used)

    def slow_bytes_used(self) -> int:
        return self._u64(self._lib.kc_slow_bytes_used)

    def d2h_bytes_total(self) -> int:
        return self._u64(self._lib.kc_d2h_bytes_total)

    def h2d_bytes_total(self) -> int:
        return self._u64(self._lib.kc_h2d_bytes_total)

    def ledger(self) -> list:
        n = self._u64(self._lib.kc_ledger_size)
        ev = []
        for i in range(n):
            ph, d = C.c_int(), C.c_int()
            layer, b, e = C.c_uint64(), C.c_uint64(), C.c_uint64()
            _check(self._lib.kc_ledger_event(self._h, i, C.byref(ph), C.byref(layer), C.byref(d), C.byref(b),
                                             C.byref(e)))
            ev.append(TransferEvent("prefill" if ph.value == 0 else "decode", layer.value,
                                    "D2H" if d.value == 0 else "H2D", b.value, e.value))
        return ev

    def ledger_jsonl(self) -> str:
        """TransferLedger::write_jsonl (kv_cache.cpp:31-37) byte format."""
        return "".join('{"phase":"%s","layer":%d,"dir":"%s","bytes":%d,"elements":%d}\n'
                       % (e.phase, e.layer, e.dir, e.bytes, e.elements) for e in self.ledger())

    def layer_storage(self, layer: int):
        k, v, on_host = C.c_void_p(), C.c_void_p(), C.c_int()
        _check(self._lib.kc_layer_storage(self._h, layer, C.byref(k), C.byref(v), C.byref(on_host)))
        return k.value, v.value, bool(on_host.value)

    def v_arena_kind(self) -> str:
        """'managed' (host-resident UVM, default), 'pinned', 'device' or 'mixed'."""
        k = C.c_int()
        _check(self._lib.kc_v_arena_kind(self._h, C.byref(k)))
        return ("managed", "pinned", "device", "mixed")[k.value]

    def set_tuning(self, key: str, value: int) -> None:
        _check(self._lib.kc_set_tuning(self._h, key.encode(), int(value)))

    def sync(self) -> None:
        _check(self._lib.kc_sync(self._h))

    def profile(self, enable: bool, kinds=("score", "select", "recall")) -> None:
        """Per-launch CUDA-event timing of the given kernel kinds."""
        mask = sum(1 << i for i, k in enumerate(("score", "select", "recall")) if k in kinds)
        _check(self._lib.kc_profile(self._h, (mask << 1) if enable else 0))

    def profile_read(self, kernel: str):
        """(summed device ms, launches) of 'score' / 'select' / 'recall'."""
        ms, n = C.c_double(0), C.c_uint64(0)
        _check(self._lib.kc_profile_read(self._h, kernel.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def profile_launches(self, kernel: str) -> list:
        """Per-launch device ms of 'score' / 'select' / 'recall'."""
        _, n = self.profile_read(kernel)
        out = []
        for i in range(n):
            ms = C.c_double(0)
            _check(self._lib.kc_profile_launch(self._h, kernel.encode(), i, C.byref(ms)))
            out.append(ms.value)
        return out

    def profile_spans(self, kernel: str) -> list:
        """[(start_ms, end_ms)] of every profiled launch since profile(True)."""
        _, n = self.profile_read(kernel)
        out = []
        for i in range(n):
            a, b = C.c_double(0), C.c_double(0)
            _check(self._lib.kc_profile_span(self._h, kernel.encode(), i, C.byref(a), C.byref(b)))
            out.append((a.value, b.value))
        return out

    def consume_stamps(self):
        """Development probe (tuning consume_dbg 1): the dataflow consumer's
        per-row phase timestamps of the last decode call, ns, [rows][8]:
        0 row ready, 1 stats, 2 bound, 3 candidates, 4 selected, 5 finished,
        6 recalled, 7 wait start."""
        import numpy as np
        out = np.zeros((self.batch * self.config.kv_heads, 8), dtype=np.uint64)
        _check(self._lib.kc_debug_read(self._h, b"consume", out.ctypes.data, out.nbytes))
        return out

    def debug_buffer(self, what: str, nbytes: int):
        """Development probe: raw bytes of an internal device buffer."""
        import numpy as np
        out = np.zeros(nbytes, dtype=np.uint8)
        _check(self._lib.kc_debug_read(self._h, what.encode(), out.ctypes.data, nbytes))
        return out

    # ---- device-resident decode (bench / engine path) ----
    def decode_topn_layers_device(self, layers: Sequence[int], qs, top_n: int, outs, renormalize=False,
                                  stream=None, want_selection=True) -> list:
        """Pipelined decode_attention_topn over several layers with device q
        (torch fp32/fp16/bf16 [batch, n_heads*h]) and device outputs.
        outs: list of dicts with torch tensors 'out' [batch, d] fp32 and
        optionally 'indices' (int32 [slots, nc]), 'weights', 'dropped'."""
        import torch
        n = len(layers)
        dt = {torch.float32: KC_F32, torch.float16: KC_F16, torch.bfloat16: KC_BF16}[qs[0].dtype]
        arr_l = (C.c_uint64 * n)(*layers)
        arr_q = (C.c_void_p * n)(*[q.data_ptr() for q in qs])
        arr_o = (_TopnOut * n)()
        for i, o in enumerate(outs):
            arr_o[i].out = o["out"].data_ptr()
            if want_selection:
                arr_o[i].indices = o["indices"].data_ptr() if "indices" in o else None
                arr_o[i].weights = o["weights"].data_ptr() if "weights" in o else None
                arr_o[i].dropped_mass = o["dropped"].data_ptr() if "dropped" in o else None
        flags = KC_IO_DEVICE | (KC_RENORMALIZE if renormalize else 0)
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(self._lib.kc_decode_topn_layers(self._h, n, arr_l, arr_q, dt, top_n, flags, arr_o, st))
        return [(arr_o[i].nc, arr_o[i].h2d_bytes) for i in range(n)]

    def decode_full_device(self, layer: int, q, out, stream=None) -> None:
        """decode_attention_full with device q (torch fp32/fp16/bf16 [batch,
        n_heads*h]) and device out (torch fp32 [batch, d]); asynchronous on
        `stream` (default: torch's current stream)."""
        import torch
        dt = {torch.float32: KC_F32, torch.float16: KC_F16, torch.bfloat16: KC_BF16}[q.dtype]
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(self._lib.kc_decode_full(self._h, layer, q.data_ptr(), dt, KC_IO_DEVICE, out.data_ptr(), st))

    # ---- engine decode-step attention block (engine.cpp:139-160) ----
    def decode_step(self, layer: int, q, k_new, v_new, top_n: int, renormalize: bool = False,
                    full: bool = False) -> np.ndarray:
        """Append this step's K/V rows ([batch, kv_width] host fp32) to `layer`
        and run its attention (TopN, or full with full=True) for host q;
        returns out [batch, d_model]. TopN calls accumulate step_stats()."""
        q, k_new, v_new = _f32(q), _f32(k_new), _f32(v_new)
        if k_new.shape != (self.batch, self.kv_width) or v_new.shape != k_new.shape:
            raise ShapeError("append_kv: row width must equal d_model")
        out = np.zeros((self.batch, self.config.d_model), np.float32)
        flags = (KC_RENORMALIZE if renormalize else 0) | (KC_FULL if full else 0)
        _check(self._lib.kc_decode_step(self._h, layer, _ptr(q), _ptr(k_new), _ptr(v_new), KC_F32, top_n,
                                        flags, _ptr(out), None))
        return out

    def decode_step_device(self, layer: int, q, k_new, v_new, out, top_n: int, renormalize: bool = False,
                           full: bool = False, stream=None) -> None:
        """Same with device torch tensors (one dtype for q / k_new / v_new), asynchronous."""
        import torch
        dt = {torch.float32: KC_F32, torch.float16: KC_F16, torch.bfloat16: KC_BF16}[q.dtype]
        flags = KC_IO_DEVICE | (KC_RENORMALIZE if renormalize else 0) | (KC_FULL if full else 0)
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(self._lib.kc_decode_step(self._h, layer, q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), dt,
                                        top_n, flags, out.data_ptr(), st))

    def step_graph_begin(self, top_n: int, stream) -> None:
        """Start capturing one decode step on `stream` (a torch.cuda.Stream):
        the decode_step_device / decode_full_device calls that follow are
        recorded, and step_graph_launch replays them as one CUDA Graph."""
        _check(self._lib.kc_step_graph_begin(self._h, top_n, stream.cuda_stream))

    def step_graph_launch(self, stream) -> None:
        """End the capture and launch the step's graph on `stream`."""
        _check(self._lib.kc_step_graph_launch(self._h, stream.cuda_stream))

    def step_stats(self, reset: bool = True) -> dict:
        """StepStats (engine.hpp:37-45) accumulated by decode_step since the last reset."""
        st = _StepStats()
        _check(self._lib.kc_step_stats_read(self._h, C.byref(st), 1 if reset else 0))
        return {"h2d_bytes": st.h2d_bytes, "d2h_bytes": st.d2h_bytes, "selections": st.selections,
                "dropped_sum": st.dropped_sum,
                "mean_dropped_mass": st.dropped_sum / st.selections if st.selections else 0.0,
                "position_histogram": list(st.position_histogram)}

    def decode_topn_layers_host(self, layers: Sequence[int], qs: Sequence[np.ndarray], top_n: int,
                                outs: Sequence[dict], renormalize=False) -> list:
        """Same with host numpy buffers (H2D of q and D2H of every output inside
        the call, which returns finished): the end-to-end path."""
        return self.prepare_topn_layers_host(layers, qs, top_n, outs, renormalize)()

    def prepare_topn_layers_host(self, layers: Sequence[int], qs: Sequence[np.ndarray], top_n: int,
                                 outs: Sequence[dict], renormalize=False) -> "TopnLayersHostCall":
        """decode_topn_layers_host bound to fixed host buffers: the argument
        arrays are built once, every call() is one kc_decode_topn_layers
        (a decode loop that refills the same pinned q / output buffers each
        step pays no per-step marshalling)."""
        return TopnLayersHostCall(self, layers, qs, top_n, outs, renormalize)


class TopnLayersHostCall:
    """One kc_decode_topn_layers call over fixed host buffers (the ctypes
    argument arrays are built here once); keeps the buffers alive."""

    def __init__(self, cache: "TieredKVCache", layers, qs, top_n: int, outs, renormalize=False):
        n = len(layers)
        self._cache, self._qs, self._outs = cache, list(qs), list(outs)
        self._n = n
        self._arr_l = (C.c_uint64 * n)(*layers)
        self._arr_q = (C.c_void_p * n)(*[q.ctypes.data for q in qs])
        self._arr_o = (_TopnOut * n)()
        for i, o in enumerate(outs):
            self._arr_o[i].out = o["out"].ctypes.data
            self._arr_o[i].indices = o["indices"].ctypes.data if "indices" in o else None
            self._arr_o[i].weights = o["weights"].ctypes.data if "weights" in o else None
            self._arr_o[i].dropped_mass = o["dropped"].ctypes.data if "dropped" in o else None
        self._dt = {np.dtype(np.float32): KC_F32, np.dtype(np.float16): KC_F16}[qs[0].dtype]
        self._top_n = top_n
        self._flags = KC_RENORMALIZE if renormalize else 0

    def __call__(self) -> list:
        c = self._cache
        _check(c._lib.kc_decode_topn_layers(c._h, self._n, self._arr_l, self._arr_q, self._dt, self._top_n,
                                            self._flags, self._arr_o, None))
        return [(self._arr_o[i].nc, self._arr_o[i].h2d_bytes) for i in range(self._n)]


# ---------------------------------------------------------------------------
# attention.hpp
def attention_score_scale(head_dim: int) -> float:
    return float(np.float32(1.0) / np.sqrt(np.float32(head_dim)))


def _check_decode_inputs(q: np.ndarray, cache: TieredKVCache) -> None:
    if q.ndim != 2 or q.shape[0] != cache.batch or q.shape[1] != cache.config.d_model:
        raise ShapeError("decode attention: q must be batch x d_model")
    if cache.current_len() == 0:
        raise StateError("decode attention: cache is empty")


def decode_attention_topn(q, cache: TieredKVCache, layer: int, top_n: int, renormalize: bool,
                          ordered_accumulation: bool = True, observer=None) -> TopNResult:
    """decode_attention_topn (attention.hpp:64-67) on the GPU."""
    if top_n == 0:
        raise ValueError("decode_attention_topn: top_n must be >= 1")
    q = _f32(q)
    _check_decode_inputs(q, cache)
    if observer is not None:
        _observe(q, cache, layer, observer)
    n = cache.config.n_heads
    slots = cache.batch * n
    nc = min(top_n, cache.current_len())
    out = np.zeros((cache.batch, cache.config.d_model), np.float32)
    idx = np.zeros((slots, nc), np.uint32)
    w = np.zeros((slots, nc), np.float32)
    dropped = np.zeros(slots, np.float64)
    o = _TopnOut(_ptr(out), _ptr(idx), _ptr(w), _ptr(dropped), 0, 0)
    flags = (KC_RENORMALIZE if renormalize else 0) | (0 if ordered_accumulation else KC_REVERSE_ACCUM)
    _check(cache._lib.kc_decode_topn(cache.handle, layer, _ptr(q), KC_F32, top_n, flags, C.byref(o), None))
    return TopNResult(out, TopNSelection(cache.batch, n, idx, w, dropped), o.h2d_bytes)


def decode_attention_full(q, cache: TieredKVCache, layer: int, observer=None) -> np.ndarray:
    """decode_attention_full (attention.hpp:45-46) on the GPU."""
    q = _f32(q)
    _check_decode_inputs(q, cache)
    if observer is not None:
        _observe(q, cache, layer, observer)
    out = np.zeros((cache.batch, cache.config.d_model), np.float32)
    _check(cache._lib.kc_decode_full(cache.handle, layer, _ptr(q), KC_F32, 0, _ptr(out), None))
    return out


def score_probs(q, cache: TieredKVCache, layer: int) -> np.ndarray:
    q = _f32(q)
    _check_decode_inputs(q, cache)
    s = cache.current_len()
    probs = np.zeros((cache.batch * cache.config.n_heads, s), np.float32)
    _check(cache._lib.kc_score_probs(cache.handle, layer, _ptr(q), KC_F32, _ptr(probs)))
    return probs


def _observe(q, cache, layer, observer) -> None:
    probs = score_probs(q, cache, layer)
    n = cache.config.n_heads
    for slot in range(probs.shape[0]):
        observer(slot // n, slot % n, probs[slot])


def score_chunk_plan(s: int, rows: int, group: int) -> int:
    """The split length the store picks for s positions over `rows` (batch x
    kv head) rows of GQA group `group` (set it as "score_chunk" on a shard to
    reproduce the unsharded cache bit for bit)."""
    c = C.c_int64(0)
    _check(load().kc_score_chunk_plan(s, rows, group, C.byref(c)))
    return c.value


def prefill_attention(q, k, v, n_heads: int, device: int = -1) -> np.ndarray:
    """prefill_attention (attention.hpp:40, attention.cpp:31-62): causal
    attention of one sequence on the GPU; q, k, v: s x d fp32."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    if q.shape != k.shape or q.shape != v.shape:
        raise ShapeError("prefill_attention: Q/K/V shapes differ")
    if n_heads == 0 or q.shape[1] % n_heads != 0:
        raise ShapeError("prefill_attention: cols must divide into heads")
    out = np.zeros_like(q)
    if q.shape[0]:
        _check(load().kc_prefill_attention(_ptr(q), _ptr(k), _ptr(v), q.shape[0], n_heads, q.shape[1] // n_heads,
                                           _ptr(out), device))
    return out


# ---------------------------------------------------------------------------
# matrix.hpp / test-data helpers
def arg_topk(values, k: int) -> np.ndarray:
    """arg_topk (matrix.hpp:49-52) via the GPU radix select."""
    lib = load()
    v = _f32(values).ravel()
    if k == 0:
        raise ValueError("arg_topk: k must be >= 1")
    out = np.zeros(max(min(k, v.size), 1), np.uint32)
    cnt = C.c_uint64(0)
    _check(lib.kc_arg_topk(_ptr(v) if v.size else None, v.size, k, _ptr(out), C.byref(cnt)))
    return out[:cnt.value].copy()


def fill_uniform(tensor, seed: int, offset: int = 0, lo: float = -1.0, hi: float = 1.0, stream=None) -> None:
    """Fill a CUDA tensor with SeededRng(seed) elements [offset, offset+n)
    (rng.hpp:13-26), rounded to the tensor's dtype -- synthetic inputs."""
    import torch
    dt = {torch.float32: KC_F32, torch.float16: KC_F16, torch.bfloat16: KC_BF16}[tensor.dtype]
    assert tensor.is_cuda and tensor.is_contiguous()
    st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(load().kc_fill_uniform(tensor.data_ptr(), dt, tensor.numel(), seed, offset, lo, hi, st))


def version() -> str:
    return load().kc_version().decode()
