"""Synthetic DASH workload: prompts and rewards keyed by
derive_seed (rng.hpp:29-35), so every rank/GPU count sees the same global round.

  prompt m   : BOS, then len-1 ids uniform over the non-special ids, from
               derive_seed(seed, "prompt", m, 0) + splitmix64 counters
  reward m,g : Bernoulli(p_m), p_m = u01(derive_seed(seed, "reward_p", m, 0)),
               draw u01(derive_seed(seed, "reward", m, g)); E[uniform group] = 2/(G+1)

Vectorised numpy restatement of oracle/dash_oracle.c dor_synthetic_* (the tests
check they agree element for element).
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + GOLD
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def fnv1a(tag: str) -> np.uint64:
    h = 0xCBF29CE484222325
    for c in tag.encode():
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return np.uint64(h)


def derive_seed(base: int, tag: str, a, b=0):
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(base) ^ fnv1a(tag))
        h = splitmix64(h ^ (np.asarray(a, dtype=np.uint64) + GOLD))
        return splitmix64(h ^ (np.asarray(b, dtype=np.uint64) + np.uint64(0x7F4A7C159E3779B9)))


def u01(x):
    return (np.asarray(x, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def synthetic_prompts(seed: int, m_lo: int, m_hi: int, length: int, vocab: int, bos: int, eos: int) -> np.ndarray:
    """[m_hi - m_lo, length] int32 prompts for global prompt ids m_lo..m_hi-1."""
    m = np.arange(m_lo, m_hi, dtype=np.uint64)
    key = derive_seed(seed, "prompt", m, 0)[:, None]
    j = np.arange(length, dtype=np.uint64)[None, :]
    nspecial = (1 if bos >= 0 else 0) + 1
    with np.errstate(over="ignore"):
        ids = (splitmix64(key + GOLD * j) % np.uint64(vocab - nspecial)).astype(np.int64)
    lo, hi = min(bos, eos), max(bos, eos)
    if lo >= 0:
        ids = ids + (ids >= lo)
    ids = ids + (ids >= hi)
    out = ids.astype(np.int32)
    if bos >= 0 and length > 0:
        out[:, 0] = bos
    return out


def synthetic_rewards(seed: int, m_lo: int, m_hi: int, G: int) -> np.ndarray:
    """[(m_hi - m_lo) * G] binary rewards, sequence s = m * G + g."""
    m = np.arange(m_lo, m_hi, dtype=np.uint64)
    pm = u01(derive_seed(seed, "reward_p", m, 0))[:, None]
    g = np.arange(G, dtype=np.uint64)[None, :]
    draw = u01(derive_seed(seed, "reward", m[:, None], g))
    return (draw < pm).astype(np.float64).reshape(-1)


# Model shapes (SURVEY App.C): reference math at Qwen2.5 dims + GQA geometry.
QWEN = {
    "0.5b": dict(vocab_size=151936, embed_dim=896, ffn_hidden=4864, n_layers=24, n_heads=14, n_kv_heads=2,
                 head_dim=64),
    "1.5b": dict(vocab_size=151936, embed_dim=1536, ffn_hidden=8960, n_layers=28, n_heads=12, n_kv_heads=2,
                 head_dim=128),
    "3b": dict(vocab_size=151936, embed_dim=2048, ffn_hidden=11008, n_layers=36, n_heads=16, n_kv_heads=2,
               head_dim=128),
}


def qwen_arch(size: str, context_len: int) -> dict:
    a = dict(QWEN[size])
    a.update(context_len=context_len, bos_id=0, eos_id=1)
    return a
