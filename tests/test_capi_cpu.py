"""CPU: the drop-in boundary builds, loads and exports what its headers declare.

No compute calls (no GPU here): the library is loaded with ctypes, every
function declared in include/kcache_c.h must resolve, the C++ operator API
(include/kcache/*.hpp) must be defined in the same library, and the
kernels must be sm_100a SASS with the TMA bulk copy in the scoring kernel.
"""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2404_18057_b200", "libkcache_b200.so")
HDR = os.path.join(ROOT, "include", "kcache_c.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import ctypes
    assert os.path.exists(LIB), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    return ctypes.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_signatures_cover_the_header():
    from paper_2404_18057_b200 import kcache
    lib = kcache.load()
    for n in declared_functions():
        fn = getattr(lib, n)
        assert fn.restype is not None or n in (), n
    assert kcache.version().startswith("kcache-b200")


def test_cpp_operator_api_is_in_the_library():
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    syms = subprocess.run([nm, "-D", "-C", LIB], capture_output=True, text=True).stdout
    for s in ["kcache::decode_attention_topn(", "kcache::decode_attention_full(", "kcache::arg_topk(",
              "kcache::TieredKVCache::TieredKVCache(", "kcache::TieredKVCache::append_kv(",
              "kcache::TieredKVCache::gather_v(", "kcache::TieredKVCache::offload_prefill_v(",
              "kcache::TieredKVCache::begin_decode(", "kcache::memory_footprint(", "kcache::TransferLedger::write_jsonl("]:
        assert s in syms, s


def test_kernels_are_sm100a_with_tma_bulk_copies():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-lelf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", LIB], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass            # cp.async.bulk (TMA) K staging
    assert "SYNCS" in sass             # mbarrier pipeline
    assert "score_fast_kernel" in sass and "select_reg_kernel" in sass and "recall_pv_kernel" in sass
    assert "consume_kernel" in sass    # the dataflow consumer
    # tcgen05 GQA scoring (kc_score_tc.cu): 2-D TMA loads, tensor-core MMA into
    # TMEM, TMEM loads
    assert "UTMALDG" in sass and "UTCHMMA" in sass and "LDTM" in sass


def test_status_codes_match_the_python_mapping():
    from paper_2404_18057_b200 import kcache
    src = open(HDR).read()
    codes = dict(re.findall(r"#define (KC_E[A-Z]+|KC_OK) (\d+)", src))
    assert int(codes["KC_OK"]) == kcache.KC_OK
    assert int(codes["KC_ESHAPE"]) == kcache.KC_ESHAPE
    assert int(codes["KC_ESTATE"]) == kcache.KC_ESTATE
    assert int(codes["KC_ECAPACITY"]) == kcache.KC_ECAPACITY
    assert int(codes["KC_EARG"]) == kcache.KC_EARG
    assert int(codes["KC_ERANGE"]) == kcache.KC_ERANGE


def test_host_side_validation_matches_reference_errors():
    """ModelConfig / TierPlacement checks run before any device work
    (model.cpp:13-27, kv_cache.cpp:39-46); the footprint formula pins the
    reference's test_kv_cache.cpp:183-211 numbers."""
    from paper_2404_18057_b200 import kcache as kc
    with pytest.raises(kc.ShapeError):
        kc.ModelConfig(1, 30, 4, 8, 16, 64, 10).validate()
    with pytest.raises(kc.ShapeError):
        kc.ModelConfig(1, 32, 4, 8, 16, 1, 10).validate()
    with pytest.raises(kc.ShapeError):
        kc.ModelConfig(0, 32, 4, 8, 16, 64, 10).validate()
    with pytest.raises(kc.ShapeError):
        kc.ModelConfig(1, 32, 4, 8, 16, 64, 10, n_kv_heads=3).validate()
    with pytest.raises(kc.ShapeError):
        kc.TierPlacement(3, 2).validate()
    with pytest.raises(kc.ShapeError):
        kc.TierPlacement(0, 2, 0).validate()
    c7 = kc.ModelConfig.shape_7b()
    assert kc.footprint(c7, 8, 32768, "baseline", 0, 2)["fast_bytes"] == 137438953472
    fp = kc.footprint(c7, 8, 32768, "kcache", 2, 2)
    assert fp["fast_bytes"] == 73014444032
    assert fp["fast_bytes"] + fp["slow_bytes"] == 137438953472
    assert kc.attention_score_scale(128) == float(np.float32(1) / np.sqrt(np.float32(128)))
    assert kc.ModelConfig.default_ffn_hidden(4096) == 10928  # ceil(8d/3) to a multiple of 16


def test_split_plan_is_balanced():
    """kc_score_chunk_plan (host-side, no GPU): splits are 64-position
    multiples of bounded length that cover the row, and a row a few positions
    past a multiple of the target (the decode phase after a 16 k prefill)
    gets no extra split of a handful of positions (C3 at 16 k + 7: 17 splits
    before r02's plan; the 64-position rounding may merge one instead)."""
    from paper_2404_18057_b200 import kcache as kc
    for rows, g, hi in ((256, 1, 2048), (256, 4, 8192), (64, 4, 8192), (8, 1, 2048), (512, 4, 8192)):
        for s in (100, 1000, 4096, 4100, 16384, 16391, 16448, 32768, 32775, 65536, 131072, 131100):
            c = kc.score_chunk_plan(s, rows, g)
            n = (s + c - 1) // c
            assert c % 64 == 0 and 64 <= c <= max(hi, 64 * ((s + 63) // 64)), (s, rows, g, c)
            assert (n - 1) * c < s <= n * c
        for base in (4096, 16384, 32768, 131072):
            c0 = kc.score_chunk_plan(base, rows, g)
            if c0 >= hi:  # splits at the length cap: one more position needs one more split
                continue
            for extra in (1, 7, 40):
                c1 = kc.score_chunk_plan(base + extra, rows, g)
                assert (base + extra + c1 - 1) // c1 <= (base + c0 - 1) // c0, (base, extra, rows, g, c0, c1)
    assert kc.score_chunk_plan(16384, 256, 4) == 1024  # C3: ~28 GQA items per SM
    assert kc.score_chunk_plan(32768, 256, 1) == 1216  # C2
