"""Seeded synthetic inputs shared by the oracle side and the CUDA side (no method arithmetic)."""
from .gen import (Spec, TID_DO, TID_K, TID_O_FULL, TID_O_SPARSE, TID_Q, TID_V, bf16_bits_to_f32,
                  bf16_rne_bits, gen_f32, gen_rows_bits, gen_rows_f32, gen_rows_f32_at, gen_torch, raw_normal)

__all__ = ["Spec", "TID_Q", "TID_K", "TID_V", "TID_DO", "TID_O_FULL", "TID_O_SPARSE", "gen_f32",
           "gen_rows_f32", "gen_rows_f32_at", "gen_rows_bits", "gen_torch", "raw_normal", "bf16_rne_bits", "bf16_bits_to_f32"]
