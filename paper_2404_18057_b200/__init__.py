"""B200-native KCache decode-step attention (arXiv 2404.18057).

``kcache`` mirrors the reference's operator API (TieredKVCache,
decode_attention_topn, decode_attention_full, arg_topk) over the C ABI of
``libkcache_b200.so`` (include/kcache_c.h), whose sm_100a kernels do all the
work. See DESIGN.md.
"""
from . import kcache  # noqa: F401
