"""fp64 decode attention over a beam's own materialised K/V (oracle; test only).

The paper describes no attention math; SURVEY ledger C10/C11 fix the textbook
definition used by decode in paged serving ("paged attention"):
for query head h with kv head h // G (consecutive q heads share one kv head),
    s_i = (q_h . K_i) * scale,  scale = 1/sqrt(d),
    o_h = sum_i softmax(s)_i V_i      over every token i < len of the beam
(the new token is appended first and attends to itself).  No mask, ALiBi,
soft-cap or window.  Computed in float64 from bf16 inputs.

``partial_state`` / ``merge_states`` state the split-KV identity the cascade
kernel relies on: for any partition of the keys into parts
with m_i = max s, l_i = sum exp(s - m_i), o_i = sum exp(s - m_i) V / l_i,
    m = max m_i,  l = sum l_i e^{m_i - m},  o = sum l_i e^{m_i - m} o_i / l.
"""
from __future__ import annotations

import numpy as np


def attention_fp64(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float) -> np.ndarray:
    """q [Hq, d], K/V [n, Hkv, d] -> o [Hq, d] (float64)."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    Hq, d = q.shape
    Hkv = K.shape[1]
    G = Hq // Hkv
    out = np.empty((Hq, d), dtype=np.float64)
    for h in range(Hq):
        kv = h // G
        s = (K[:, kv, :] @ q[h]) * scale
        w = np.exp(s - s.max())
        out[h] = (w / w.sum()) @ V[:, kv, :]
    return out


def partial_state(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float):
    """(m [Hq], l [Hq], o [Hq, d]) of one key subset (o normalised)."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    Hq, d = q.shape
    G = Hq // K.shape[1]
    m = np.empty(Hq)
    l = np.empty(Hq)
    o = np.empty((Hq, d))
    for h in range(Hq):
        s = (K[:, h // G, :] @ q[h]) * scale
        m[h] = s.max()
        w = np.exp(s - m[h])
        l[h] = w.sum()
        o[h] = (w @ V[:, h // G, :]) / l[h]
    return m, l, o


def merge_states(states):
    ms = np.stack([s[0] for s in states])          # [parts, Hq]
    ls = np.stack([s[1] for s in states])
    os_ = np.stack([s[2] for s in states])         # [parts, Hq, d]
    m = ms.max(axis=0)
    w = ls * np.exp(ms - m)
    l = w.sum(axis=0)
    o = (w[:, :, None] * os_).sum(axis=0) / l[:, None]
    return m, l, o
