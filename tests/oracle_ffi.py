"""ctypes bindings of the TEST-ONLY oracles (oracle/lib/libdash_oracle.so, the C
restatement, and oracle/_ref/libdash_ref.so, the unmodified reference compiled in
place). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "lib", "libdash_oracle.so")
REF_LIB = os.path.join(ORACLE_DIR, "_ref", "libdash_ref.so")

_lock = threading.Lock()
_oracle = None
_ref = None

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)


class DorArch(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "vocab_size", "embed_dim", "context_len", "ffn_hidden", "n_layers", "bos_id", "eos_id",
        "n_heads", "n_kv_heads", "head_dim")]


def arch_struct(arch: dict) -> DorArch:
    return DorArch(arch["vocab_size"], arch["embed_dim"], arch["context_len"], arch["ffn_hidden"],
                   arch["n_layers"], arch["bos_id"], arch["eos_id"], arch.get("n_heads", 0),
                   arch.get("n_kv_heads", 0), arch.get("head_dim", 0))


def arch_ref_vec(arch: dict):
    return (C.c_int32 * 7)(arch["vocab_size"], arch["embed_dim"], arch["context_len"],
                           arch["ffn_hidden"], arch["n_layers"], arch["bos_id"], arch["eos_id"])


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True, stdout=subprocess.DEVNULL)


def oracle():
    global _oracle
    with _lock:
        if _oracle is None:
            if not os.path.exists(ORACLE_LIB):
                _build()
            L = C.CDLL(ORACLE_LIB)
            L.dor_splitmix64.restype = C.c_uint64
            L.dor_splitmix64.argtypes = [C.c_uint64]
            L.dor_fnv1a.restype = C.c_uint64
            L.dor_fnv1a.argtypes = [C.c_char_p]
            L.dor_derive_seed.restype = C.c_uint64
            L.dor_derive_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64, C.c_uint64]
            L.dor_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_int, u64p]
            L.dor_num_params.restype = C.c_int64
            L.dor_num_params.argtypes = [C.POINTER(DorArch)]
            L.dor_init_params.argtypes = [C.POINTER(DorArch), C.c_double, C.c_uint64, f64p]
            L.dor_init_params_ctr.argtypes = [C.POINTER(DorArch), C.c_double, C.c_uint64, f64p]
            L.dor_log_prob.restype = C.c_double
            L.dor_log_prob.argtypes = [C.POINTER(DorArch), f64p, i32p, C.c_int, i32p, C.c_int, f64p]
            L.dor_next_logits.argtypes = [C.POINTER(DorArch), f64p, i32p, C.c_int, f64p]
            L.dor_kl_term_acc.argtypes = [C.POINTER(DorArch), f64p, f64p, i32p, C.c_int, i32p, C.c_int, C.c_double,
                                          f64p]
            L.dor_kl_term_acc.restype = C.c_double
            L.dor_grad_log_prob_acc.argtypes = [C.POINTER(DorArch), f64p, i32p, C.c_int, i32p, C.c_int,
                                                C.c_double, f64p]
            L.dor_soft_logf.restype = C.c_float
            L.dor_soft_logf.argtypes = [C.c_float]
            L.dor_row_key.restype = C.c_uint32
            L.dor_row_key.argtypes = [C.c_uint64, C.c_int32]
            L.dor_gumbel.restype = C.c_float
            L.dor_gumbel.argtypes = [C.c_uint32, C.c_int32]
            L.dor_sample_rule.restype = C.c_int32
            L.dor_sample_rule.argtypes = [f32p, C.c_int, C.c_int, C.c_float, C.c_uint64, C.c_int32]
            L.dor_sample.restype = C.c_int
            L.dor_sample.argtypes = [C.POINTER(DorArch), f64p, i32p, C.c_int, C.c_int, C.c_double,
                                     C.c_uint64, i32p, f64p]
            L.dor_advantage_filter.restype = C.c_int
            L.dor_advantage_filter.argtypes = [f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                               C.c_double, f64p, u8p, i32p, i32p]
            L.dor_pg_accumulate.argtypes = [C.POINTER(DorArch), f64p, C.c_int, i32p, i64p, i32p, i64p,
                                            f64p, f64p]
            L.dor_adam_step.argtypes = [f64p, f64p, f64p, f64p, C.c_int64, C.c_int64, C.c_double,
                                        C.c_double, C.c_double, C.c_double]
            L.dor_sgd_step.argtypes = [f64p, f64p, C.c_int64, C.c_double]
            L.dor_synthetic_reward.restype = C.c_double
            L.dor_synthetic_reward.argtypes = [C.c_uint64, C.c_int64, C.c_int32]
            L.dor_synthetic_prompt.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                               i32p]
            _oracle = L
        return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


class RefStepStats(C.Structure):
    _fields_ = [("sample_s", C.c_double), ("reward_adv_s", C.c_double), ("grad_s", C.c_double),
                ("update_s", C.c_double), ("total_s", C.c_double), ("tokens_sampled", C.c_int64),
                ("kept", C.c_int32), ("n_seq", C.c_int32), ("mean_reward", C.c_double)]


def ref():
    global _ref
    with _lock:
        if _ref is None:
            if not os.path.exists(REF_LIB):
                raise FileNotFoundError(REF_LIB)
            L = C.CDLL(REF_LIB)
            L.ref_last_error.restype = C.c_char_p
            L.ref_num_params.argtypes = [i32p, i64p]
            L.ref_init_params.argtypes = [i32p, C.c_double, C.c_uint64, f64p]
            L.ref_content_hash.argtypes = [i32p, f64p, u64p]
            L.ref_sample.argtypes = [i32p, f64p, i32p, C.c_int, C.c_int, C.c_double, C.c_uint64, i32p,
                                     f64p, i32p]
            L.ref_log_prob.argtypes = [i32p, f64p, i32p, C.c_int, i32p, C.c_int, f64p, f64p]
            L.ref_grad_log_prob.argtypes = [i32p, f64p, i32p, C.c_int, i32p, C.c_int, f64p]
            L.ref_kl_term.argtypes = [i32p, f64p, f64p, i32p, C.c_int, i32p, C.c_int, f64p, f64p]
            L.ref_next_token_probs.argtypes = [i32p, f64p, i32p, C.c_int, f64p]
            L.ref_greedy_decode.argtypes = [i32p, f64p, i32p, C.c_int, C.c_int, i32p, i32p]
            L.ref_advantage.argtypes = [f64p, C.c_int, C.c_int, C.c_int, f64p]
            L.ref_normalize_std.argtypes = [f64p, f64p, C.c_int, C.c_int, C.c_double, f64p]
            L.ref_filter_by_threshold.argtypes = [f64p, C.c_int, C.c_double, u8p, i32p, f64p, f64p]
            L.ref_splitmix64.restype = C.c_uint64
            L.ref_splitmix64.argtypes = [C.c_uint64]
            L.ref_fnv1a.restype = C.c_uint64
            L.ref_fnv1a.argtypes = [C.c_char_p]
            L.ref_derive_seed.restype = C.c_uint64
            L.ref_derive_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64, C.c_uint64]
            L.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_int, u64p]
            L.ref_add_instance.argtypes = [C.c_int, C.c_uint64, i32p, i32p, C.c_char_p, C.c_int]
            L.ref_add_reward.argtypes = [C.c_int, C.c_uint64, i32p, C.c_int, f64p]
            L.ref_dash_step.argtypes = [i32p, f64p, i32p, i64p, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_uint64, C.c_int64, C.c_int, C.c_uint64, u64p, C.c_double,
                                        C.c_int, C.c_double, f64p, f64p, i64p, C.c_int,
                                        C.POINTER(RefStepStats)]
            _ref = L
        return _ref


# ----------------------------------------------------------------- helpers

def num_params(arch: dict) -> int:
    a = arch_struct(arch)
    return int(oracle().dor_num_params(C.byref(a)))


def init_params(arch: dict, scale: float, seed: int) -> np.ndarray:
    a = arch_struct(arch)
    out = np.zeros(num_params(arch), dtype=np.float64)
    oracle().dor_init_params(C.byref(a), scale, seed, ptr(out, f64p))
    return out


def init_params_ctr(arch: dict, scale: float, seed: int) -> np.ndarray:
    a = arch_struct(arch)
    out = np.zeros(num_params(arch), dtype=np.float64)
    oracle().dor_init_params_ctr(C.byref(a), scale, seed, ptr(out, f64p))
    return out


def i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def log_prob(arch, params, prompt, completion):
    a = arch_struct(arch)
    p, c = i32(prompt), i32(completion)
    per = np.zeros(max(len(c), 1), dtype=np.float64)
    tot = oracle().dor_log_prob(C.byref(a), ptr(params, f64p), ptr(p, i32p), len(p), ptr(c, i32p), len(c),
                                ptr(per, f64p))
    return tot, per[:len(c)]


def next_logits(arch, params, ctx):
    a = arch_struct(arch)
    c = i32(ctx)
    out = np.zeros(arch["vocab_size"], dtype=np.float64)
    oracle().dor_next_logits(C.byref(a), ptr(params, f64p), ptr(c, i32p), len(c), ptr(out, f64p))
    return out


def grad_log_prob(arch, params, prompt, completion, scale=1.0, grad=None):
    a = arch_struct(arch)
    p, c = i32(prompt), i32(completion)
    if grad is None:
        grad = np.zeros(num_params(arch), dtype=np.float64)
    oracle().dor_grad_log_prob_acc(C.byref(a), ptr(params, f64p), ptr(p, i32p), len(p), ptr(c, i32p),
                                   len(c), scale, ptr(grad, f64p))
    return grad


def kl_term(arch, params, base, prompt, completion, scale=1.0, grad=None):
    """kl_term (policy.cpp:487-522) restated with GQA geometry: (value, grad += scale * dKL/dP)."""
    a = arch_struct(arch)
    p, c = i32(prompt), i32(completion)
    if grad is None:
        grad = np.zeros(num_params(arch), dtype=np.float64)
    v = oracle().dor_kl_term_acc(C.byref(a), ptr(params, f64p), ptr(base, f64p), ptr(p, i32p), len(p), ptr(c, i32p),
                                 len(c), scale, ptr(grad, f64p))
    return v, grad


def sample_rule(logits_f32: np.ndarray, bos: int, inv_t: float, seq_key: int, step: int) -> int:
    lf = np.ascontiguousarray(logits_f32, dtype=np.float32)
    return int(oracle().dor_sample_rule(ptr(lf, f32p), lf.shape[0], bos, inv_t, seq_key, step))


def sample(arch, params, prompt, max_len, temperature, seq_key):
    a = arch_struct(arch)
    p = i32(prompt)
    comp = np.zeros(max(max_len, 1), dtype=np.int32)
    lp = np.zeros(max(max_len, 1), dtype=np.float64)
    n = oracle().dor_sample(C.byref(a), ptr(params, f64p), ptr(p, i32p), len(p), max_len, temperature,
                            seq_key, ptr(comp, i32p), ptr(lp, f64p))
    return comp[:n].copy(), lp[:n].copy()


def advantage_filter(rewards, group_size, kind=1, normalize=False, eps=0.0, tau=0.0):
    tau = float("-inf") if tau is None else tau   # no filter (DASHCU_FILTER_OFF)
    r = np.ascontiguousarray(rewards, dtype=np.float64)
    n = r.shape[0]
    adv = np.zeros(max(n, 1))
    kept = np.zeros(max(n, 1), dtype=np.uint8)
    idx = np.zeros(max(n, 1), dtype=np.int32)
    nk = C.c_int32(0)
    rc = oracle().dor_advantage_filter(ptr(r, f64p), n, group_size, kind, int(normalize), eps, tau,
                                       ptr(adv, f64p), ptr(kept, u8p), ptr(idx, i32p), C.byref(nk))
    if rc != 0:
        raise ValueError("InputError")
    return adv[:n], kept[:n].astype(bool), idx[:nk.value].copy()


def derive_seed(base, tag: str, a=0, b=0) -> int:
    return int(oracle().dor_derive_seed(base, tag.encode(), a, b))


def synthetic_reward(seed, m, g) -> float:
    return float(oracle().dor_synthetic_reward(seed, m, g))


def synthetic_prompt(seed, m, length, vocab, bos, eos) -> np.ndarray:
    out = np.zeros(length, dtype=np.int32)
    oracle().dor_synthetic_prompt(seed, m, length, vocab, bos, eos, ptr(out, i32p))
    return out
