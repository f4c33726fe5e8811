"""Byte / FLOP accounting for the roofline.

kv_bytes follows SPEC S:317-325 (roofline.kv_bytes): batch x seq x 2 (K and V)
x layers x kv_heads x head_dim x dtype_bytes.  t_roof is PAPER.md 4.3.1
(P:431-435): T_roof = max(FLOPs / (P 1e12), Bytes / (BW 1e9)).
"""
from __future__ import annotations


def kv_bytes(n_layers: int, n_kv_heads: int, head_dim: int, dtype_bytes: int, batch: int, seq: int) -> int:
    return batch * seq * 2 * n_layers * n_kv_heads * head_dim * dtype_bytes


def t_roof(flops: float, nbytes: float, peak_tflops: float, bw_gbs: float) -> float:
    return max(flops / (peak_tflops * 1e12), nbytes / (bw_gbs * 1e9))


def attn_flops(n_q_heads: int, head_dim: int, logical_tokens: int) -> int:
    """4 d Hq len per beam-layer (QK^T and PV; SURVEY 8(d) 'Algorithmic work per unit')."""
    return 4 * head_dim * n_q_heads * logical_tokens
