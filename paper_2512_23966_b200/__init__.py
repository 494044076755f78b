"""LoZA streaming sparse attention (arXiv 2512.23966) hot path for B200 (sm_100a).

The product is libloza.so (C ABI in include/loza.h, CUDA sources in csrc/);
``loza`` is its thin ctypes binding.
"""
from . import loza  # noqa: F401
from .loza import (PAPER_PATTERN, full_attn_ref, kernel_launches, loza_blend, ssa_decode, ssa_prefill,  # noqa: F401
                   ssa_select_blocks, ssa_seqpar_prefill)
