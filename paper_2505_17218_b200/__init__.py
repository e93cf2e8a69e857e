"""B200-native DASH training step (arXiv 2505.17218) — Python binding of libdashcu.

The product is the C ABI in include/dashcu.h (libdashcu.so, CUDA sm_100a). This
module is a thin ctypes mirror of it for Python callers (tests, bench.py). It
has no compute of its own and no CPU fallback: if the shared library is missing
or no B200 is visible, every compute call raises.

Names follow the reference's domain (SPEC.md / proj/include/dash): policies,
rollouts, groups, advantages, kept sets.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DASHCU_LIB_PATH") or os.path.join(PKG, "lib", "libdashcu.so")

OK, E_INPUT, E_CAPACITY, E_ON_POLICY, E_DEVICE = 0, 1, 2, 3, 4
F32, BF16 = 0, 1
ADV_SINGLE_PATH, ADV_GROUP, ADV_LEAVE_ONE_OUT = 0, 1, 2
FILTER_OFF = float("-inf")  # DASHCU_FILTER_OFF: no filter_by_threshold, every sequence kept
OPT_SGD, OPT_ADAM = 0, 1
SCHED_DASH, SCHED_MULTI, SCHED_MINI = 0, 1, 2
TASK_ADD, TASK_MOD, TASK_REVERSE, TASK_PARITY, TASK_MICRO = 0, 1, 2, 3, 4
VOCAB_TASK, VOCAB_BYTE = 0, 1


def shard_span(total: int, world: int, rank: int):
    """(offset, length) of rank's slice in the sharded optimizer step (dashcu_shard_span)."""
    off, n = C.c_int64(0), C.c_int64(0)
    _check(lib().dashcu_shard_span(total, world, rank, C.byref(off), C.byref(n)))
    return off.value, n.value


class DashError(RuntimeError):
    code = E_DEVICE


class InputError(DashError, ValueError):          # errors.hpp:12-14
    code = E_INPUT


class CapacityError(DashError):                    # errors.hpp:17-19
    code = E_CAPACITY


class OnPolicyViolation(DashError):                # errors.hpp:21-23
    code = E_ON_POLICY


class DeviceError(DashError):
    code = E_DEVICE


_ERR = {E_INPUT: InputError, E_CAPACITY: CapacityError, E_ON_POLICY: OnPolicyViolation, E_DEVICE: DeviceError}


class Arch(C.Structure):
    """ArchConfig (tensors.hpp:13-24) + GQA geometry; zeros mean the reference (1, 1, d)."""
    _fields_ = [(n, C.c_int32) for n in ("vocab_size", "embed_dim", "context_len", "ffn_hidden", "n_layers",
                                         "bos_id", "eos_id", "n_heads", "n_kv_heads", "head_dim")]

    @classmethod
    def of(cls, d: dict) -> "Arch":
        return cls(*(int(d.get(f, 0)) for f, _ in cls._fields_))


class Plan(C.Structure):
    """SamplingPlan."""
    _fields_ = [("n_prompts", C.c_int32), ("group_size", C.c_int32), ("max_len", C.c_int32),
                ("temperature", C.c_double), ("round_seed", C.c_uint64), ("prompt_index_base", C.c_int64)]


class Opt(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double)]


class Schedule(C.Structure):
    """UpdateConfig of run_schedule."""
    _fields_ = [("kind", C.c_int32), ("K", C.c_int32), ("clip_eps", C.c_double), ("beta", C.c_double),
                ("weight_scale", C.c_double), ("micro_batch", C.c_int32), ("sharded", C.c_int32)]


class StepLog(C.Structure):
    _fields_ = [("surrogate", C.c_double), ("kl", C.c_double), ("clip_fraction", C.c_double),
                ("mean_abs_adv", C.c_double), ("filtered_fraction", C.c_double), ("n_items", C.c_int32),
                ("ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Stats(C.Structure):
    _fields_ = [("sample_ms", C.c_double), ("advantage_ms", C.c_double), ("accumulate_ms", C.c_double),
                ("allreduce_ms", C.c_double), ("optimizer_ms", C.c_double), ("tokens_sampled", C.c_int64),
                ("n_seq", C.c_int32), ("n_kept", C.c_int32), ("loss_tokens", C.c_int64),
                ("mean_reward", C.c_double), ("filtered_fraction", C.c_double), ("mean_abs_kept", C.c_double),
                ("kernel_launches", C.c_int64), ("decode_row_steps", C.c_int64), ("kv_pages_peak", C.c_int64),
                ("slice_recompute_mismatches", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p


def lib():
    """Load libdashcu.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.dashcu_last_error.restype = C.c_char_p
        L.dashcu_kernel_launches.restype = C.c_int64
        sig = {
            "dashcu_ctx_create": [C.c_int, C.POINTER(vp)],
            "dashcu_ctx_destroy": [vp],
            "dashcu_ctx_sync": [vp],
            "dashcu_comm_unique_id": [C.c_char_p],
            "dashcu_ctx_init_comm": [vp, C.c_int, C.c_int, C.c_char_p],
            "dashcu_arch_num_params": [C.POINTER(Arch), i64p],
            "dashcu_policy_create": [vp, C.POINTER(Arch), C.c_int, C.POINTER(vp)],
            "dashcu_policy_destroy": [vp],
            "dashcu_policy_upload": [vp, f64p, C.c_int64],
            "dashcu_policy_download": [vp, f64p, C.c_int64],
            "dashcu_policy_init_normal": [vp, C.c_double, C.c_uint64],
            "dashcu_policy_version": [vp, C.POINTER(C.c_uint64)],
            "dashcu_sample": [vp, C.POINTER(Plan), i32p, i64p, i32p, i32p, f32p],
            "dashcu_set_logits_dump": [vp, C.c_int],
            "dashcu_set_kv_pages": [vp, C.c_int64],
            "dashcu_get_logits_dump": [vp, f32p, C.c_int64],
            "dashcu_rollout_load": [vp, i32p, i64p, C.c_int32, C.c_int32, i32p, i64p],
            "dashcu_rollout_log_prob": [vp, f32p, C.c_int64],
            "dashcu_advantage_filter": [vp, f64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                        f64p, u8p, i32p, i32p],
            "dashcu_rollout_set_rewards": [vp, f64p, C.c_int32],
            "dashcu_rollout_advantage": [vp, C.c_int32, C.c_int32, C.c_double, C.c_double, f64p, u8p, i32p],
            "dashcu_grad_zero": [vp],
            "dashcu_accumulate": [vp, C.c_double, C.c_int32],
            "dashcu_accumulate_weighted": [vp, f64p, C.c_int32, C.c_int32],
            "dashcu_grad_download": [vp, f64p, C.c_int64],
            "dashcu_grad_upload": [vp, f64p, C.c_int64],
            "dashcu_allreduce_grads": [vp],
            "dashcu_optimizer_step": [vp, C.POINTER(Opt)],
            "dashcu_sharded_step": [vp, C.POINTER(Opt)],
            "dashcu_fused_step": [vp, C.POINTER(Opt)],
            "dashcu_selftest_fused_step": [vp, C.c_int32, C.c_int64, C.c_int32, C.c_double, C.c_int32, f32p, f32p,
                                           f32p, C.POINTER(C.c_uint16)],
            "dashcu_shard_span": [C.c_int64, C.c_int32, C.c_int32, i64p, i64p],
            "dashcu_get_stats": [vp, C.POINTER(Stats)],
            "dashcu_rollout_snapshot": [vp],
            "dashcu_rebalance": [vp, i32p, i32p],
            "dashcu_rebalance_plan": [C.c_int32, i32p, i64p, i32p],
            "dashcu_policy_save": [vp, C.c_char_p, C.c_int32],
            "dashcu_policy_load": [vp, C.c_char_p, C.c_int32],
            "dashcu_checkpoint_arch": [C.c_char_p, C.POINTER(Arch)],
            "dashcu_rollout_snapshot_logp": [vp, f64p, C.c_int32],
            "dashcu_accumulate_ppo": [vp, C.c_double, C.c_double, C.c_int32, i32p, C.c_int32, f64p, i32p],
            "dashcu_accumulate_kl": [vp, vp, C.c_double, C.c_int32, i32p, C.c_int32, f64p],
            "dashcu_run_schedule": [vp, C.POINTER(Schedule), C.POINTER(Opt), vp, C.POINTER(StepLog), C.c_int32,
                                    i32p],
            "dashcu_task_vocab_size": [C.c_int32, C.c_int32, i32p],
            "dashcu_task_instances": [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint64), C.c_int32, i32p,
                                      C.c_int64, i64p, C.c_char_p, C.c_int32],
            "dashcu_task_rewards": [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint64), C.c_int32, C.c_int32,
                                    i32p, C.c_int32, i32p, f64p],
            "dashcu_rollout_task_rewards": [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint64)],
            "dashcu_selftest_gemm": [vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint16), C.c_int64, C.c_int,
                                     C.POINTER(C.c_uint16), C.c_int64, C.c_int, f32p, C.c_int, C.c_int, f32p],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.dashcu_profile_enable.argtypes = [C.c_uint]
        L.dashcu_profile_enable.restype = C.c_int
        L.dashcu_profile_read.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.dashcu_profile_read.restype = C.c_int
        L.dashcu_profile_sampling.argtypes = [C.c_int]
        L.dashcu_profile_sampling.restype = C.c_int
        L.dashcu_profile_keys.argtypes = [C.c_char_p, C.c_int64]
        L.dashcu_profile_keys.restype = C.c_int64
        L.dashcu_set_knob.argtypes = [C.c_char_p, C.c_int]
        L.dashcu_set_knob.restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        msg = lib().dashcu_last_error().decode(errors="replace")
        raise _ERR.get(rc, DeviceError)(msg)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t) if a is not None else None


KNOB_DEFAULT = -(2 ** 31)


def set_knob(name: str, value) -> int:
    """Kernel-variant knob (dashcu_set_knob); value None restores the default. Returns the old value."""
    v = KNOB_DEFAULT if value is None else int({"mma": 1, "tc5": 2}.get(value, value))
    old = lib().dashcu_set_knob(name.encode(), v)
    if old == KNOB_DEFAULT:
        raise InputError(f"unknown knob {name}")
    return old


def kernel_launches() -> int:
    return int(lib().dashcu_kernel_launches())


class KProf(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


PROF_CLASSES = ("gemm_tc", "gemm_simt", "attn_decode", "attn_fwd", "attn_bwd", "sample", "lm_rows", "optimizer")


def profile_enable(classes=PROF_CLASSES, keys=False):
    """Bracket every launch of the given kernel classes with CUDA events (algorithmic flops/bytes).
    keys=True also aggregates per kernel variant + shape (profile_keys)."""
    mask = 0
    for c in classes:
        mask |= 1 << PROF_CLASSES.index(c)
    if keys:
        mask |= 1 << 31
    lib().dashcu_profile_enable(C.c_uint(mask))


def profile_sampling(period: int = 1):
    """Event-bracket one launch in `period` per class; profile_read scales to class totals."""
    lib().dashcu_profile_sampling(int(period))


def profile_keys() -> list:
    """Per-key aggregates [(key, launches, ms, flops, bytes)], largest time first."""
    n = lib().dashcu_profile_keys(None, 0)
    if n < 0:
        raise DeviceError("profile read failed")
    buf = C.create_string_buffer(n + 1)
    lib().dashcu_profile_keys(buf, n + 1)
    out = []
    for line in buf.value.decode().splitlines():
        k, l, ms, f, b = line.split("\t")
        out.append((k, int(l), float(ms), float(f), float(b)))
    return sorted(out, key=lambda r: -r[2])


def profile_read(reset=True) -> dict:
    arr = (KProf * 16)()
    n = lib().dashcu_profile_read(arr, 16, int(reset))
    if n < 0:
        raise DeviceError("profile read failed")
    return {arr[i].name.decode(): dict(launches=arr[i].launches, ms=arr[i].ms, flops=arr[i].flops,
                                       bytes=arr[i].bytes) for i in range(n)}


def _seeds(seeds):
    return np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))


def task_vocab_size(kind: int, vocab: int = VOCAB_TASK) -> int:
    n = C.c_int32(0)
    _check(lib().dashcu_task_vocab_size(kind, vocab, C.byref(n)))
    return int(n.value)


def task_instances(kind: int, difficulty: int, seeds, vocab: int = VOCAB_TASK):
    """generate_instance (tasks.cpp:105-153) per seed: (prompt_tokens, prompt_offsets, answers)."""
    sd = _seeds(seeds)
    n = sd.shape[0]
    off = np.zeros(n + 1, dtype=np.int64)
    u64 = C.POINTER(C.c_uint64)
    _check(lib().dashcu_task_instances(kind, difficulty, vocab, sd.ctypes.data_as(u64), n, None, 0, _p(off, i64p),
                                       None, 0))
    toks = np.zeros(max(int(off[-1]), 1), dtype=np.int32)
    stride = 64
    ans = C.create_string_buffer(max(n, 1) * stride)
    _check(lib().dashcu_task_instances(kind, difficulty, vocab, sd.ctypes.data_as(u64), n, _p(toks, i32p),
                                       toks.shape[0], _p(off, i64p), ans, stride))
    answers = [ans.raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode() for i in range(n)]
    return toks[:int(off[-1])], off, answers


def task_rewards(kind: int, difficulty: int, seeds, group_size: int, completions, lengths,
                 vocab: int = VOCAB_TASK) -> np.ndarray:
    """reward (tasks.cpp:155-175) of completions [n_prompts * G, stride] against seeds[m]."""
    sd = _seeds(seeds)
    comp = np.ascontiguousarray(completions, dtype=np.int32)
    lens = np.ascontiguousarray(lengths, dtype=np.int32)
    out = np.zeros(max(lens.shape[0], 1))
    _check(lib().dashcu_task_rewards(kind, difficulty, vocab, sd.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     sd.shape[0], group_size, _p(comp, i32p), comp.shape[1], _p(lens, i32p),
                                     _p(out, f64p)))
    return out[:lens.shape[0]]


def rebalance_plan(costs_per_rank):
    """Post-filter work plan (dashcu_rebalance_plan, no device work): for every rank's list of
    item costs, the rank that accumulates each item."""
    n = np.ascontiguousarray([len(c) for c in costs_per_rank], dtype=np.int32)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.int64) for c in costs_per_rank] +
                                               [np.zeros(0, dtype=np.int64)]), dtype=np.int64)
    dest = np.zeros(max(flat.shape[0], 1), dtype=np.int32)
    _check(lib().dashcu_rebalance_plan(len(costs_per_rank), _p(n, i32p), _p(flat if flat.size else
                                       np.zeros(1, np.int64), i64p), _p(dest, i32p)))
    out, off = [], 0
    for c in costs_per_rank:
        out.append(dest[off:off + len(c)].copy())
        off += len(c)
    return out


def checkpoint_arch(path: str) -> dict:
    """The architecture descriptor in a DASHCKPT file's header (no device work)."""
    a = Arch()
    _check(lib().dashcu_checkpoint_arch(os.fsencode(path), C.byref(a)))
    return {f: getattr(a, f) for f, _ in Arch._fields_}


def num_params(arch: dict) -> int:
    n = C.c_int64(0)
    a = Arch.of(arch)
    _check(lib().dashcu_arch_num_params(C.byref(a), C.byref(n)))
    return int(n.value)


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().dashcu_comm_unique_id(buf))
    return buf.raw


class Context:
    """One per GPU (dashcu_ctx): device, stream and the gradient communicator."""

    def __init__(self, device: int = 0):
        self.h = vp()
        _check(lib().dashcu_ctx_create(device, C.byref(self.h)))

    def init_comm(self, world: int, rank: int, uid: bytes):
        _check(lib().dashcu_ctx_init_comm(self.h, world, rank, uid))

    def sync(self):
        _check(lib().dashcu_ctx_sync(self.h))

    def advantage_filter(self, rewards, group_size, kind=ADV_GROUP, normalize=False, eps=0.0, tau=0.0):
        """group_advantage / normalize_std / filter_by_threshold (advantage.cpp:80-140) on the device."""
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        tau = FILTER_OFF if tau is None else tau
        n = int(r.shape[0])
        adv = np.zeros(max(n, 1))
        kept = np.zeros(max(n, 1), dtype=np.uint8)
        idx = np.zeros(max(n, 1), dtype=np.int32)
        nk = C.c_int32(0)
        _check(lib().dashcu_advantage_filter(self.h, _p(r, f64p), n, group_size, kind, int(normalize), eps, tau,
                                             _p(adv, f64p), _p(kept, u8p), _p(idx, i32p), C.byref(nk)))
        return adv[:n], kept[:n].astype(bool), idx[:nk.value].copy()

    def selftest_gemm(self, A_bits, a_kmajor, B_bits, b_kmajor, M, N, K, bias=None, epi=0, force_simt=False,
                      C_init=None):
        """Diagnostics: C = A(m,k).B(n,k) on bf16 bit patterns (uint16) via the production dispatcher."""
        A = np.ascontiguousarray(A_bits, dtype=np.uint16)
        B = np.ascontiguousarray(B_bits, dtype=np.uint16)
        out = np.zeros((M, N), dtype=np.float32) if C_init is None else np.ascontiguousarray(C_init, np.float32).copy()
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
        u16p = C.POINTER(C.c_uint16)
        _check(lib().dashcu_selftest_gemm(self.h, M, N, K, A.ctypes.data_as(u16p), A.shape[1], int(a_kmajor),
                                          B.ctypes.data_as(u16p), B.shape[1], int(b_kmajor),
                                          None if b is None else _p(b, f32p), epi, int(force_simt), _p(out, f32p)))
        return out

    def selftest_fused_step(self, g_all, w0, kind=OPT_ADAM, lr=1e-3, steps=1):
        """Virtual ranks (rows of g_all) running the fused step concurrently; (w [world x n], wT bits)."""
        g = np.ascontiguousarray(g_all, dtype=np.float32)
        w = np.ascontiguousarray(w0, dtype=np.float32)
        world, n = g.shape
        wo = np.zeros((world, n), dtype=np.float32)
        to = np.zeros((world, n), dtype=np.uint16)
        _check(lib().dashcu_selftest_fused_step(self.h, world, n, kind, lr, steps, _p(g, f32p), _p(w, f32p),
                                                _p(wo, f32p), to.ctypes.data_as(C.POINTER(C.c_uint16))))
        return wo, to

    def close(self):
        if self.h:
            lib().dashcu_ctx_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Rollout:
    completions: np.ndarray  # [n_seq, max_len], -1 padded
    lengths: np.ndarray      # [n_seq]
    logp: np.ndarray         # [n_seq, max_len] (T = 1)

    def completion(self, s: int) -> np.ndarray:
        return self.completions[s, :self.lengths[s]]


def pack_prompts(prompts):
    toks = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.int32) for p in prompts]), dtype=np.int32)
    off = np.zeros(len(prompts) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(p) for p in prompts])
    return toks, off


class Policy:
    """Device-resident policy (dashcu_policy): fp32 master weights + gradient + Adam state,
    a bf16 (or fp32) working copy, and the current rollout."""

    def __init__(self, ctx: Context, arch: dict, dtype: int = BF16):
        self.ctx = ctx
        self.arch = dict(arch)
        self.dtype = dtype
        self.h = vp()
        a = Arch.of(arch)
        _check(lib().dashcu_policy_create(ctx.h, C.byref(a), dtype, C.byref(self.h)))
        self.n_params = num_params(arch)

    # ---- parameters
    def upload(self, params: np.ndarray):
        p = np.ascontiguousarray(params, dtype=np.float64)
        _check(lib().dashcu_policy_upload(self.h, _p(p, f64p), p.shape[0]))

    def download(self) -> np.ndarray:
        out = np.zeros(self.n_params)
        _check(lib().dashcu_policy_download(self.h, _p(out, f64p), self.n_params))
        return out

    def save(self, path: str, with_optimizer: bool = True):
        """Checkpoint container (dashcu_policy_save)."""
        _check(lib().dashcu_policy_save(self.h, os.fsencode(path), int(with_optimizer)))

    def load(self, path: str, with_optimizer: bool = True):
        _check(lib().dashcu_policy_load(self.h, os.fsencode(path), int(with_optimizer)))

    def init_normal(self, scale: float, seed: int):
        _check(lib().dashcu_policy_init_normal(self.h, scale, seed))

    def version(self) -> int:
        v = C.c_uint64(0)
        _check(lib().dashcu_policy_version(self.h, C.byref(v)))
        return int(v.value)

    # ---- sampling
    def set_logits_dump(self, enable: bool):
        _check(lib().dashcu_set_logits_dump(self.h, int(enable)))

    def set_kv_pages(self, n_pages: int):
        """Cap the decode KV page pool (dashcu_set_kv_pages; 0 = worst case)."""
        _check(lib().dashcu_set_kv_pages(self.h, int(n_pages)))

    def logits_dump(self, n_seq: int, max_len: int) -> np.ndarray:
        V = self.arch["vocab_size"]
        out = np.zeros(n_seq * max(max_len, 1) * V, dtype=np.float32)
        _check(lib().dashcu_get_logits_dump(self.h, _p(out, f32p), out.shape[0]))
        return out.reshape(n_seq, max(max_len, 1), V)

    def sample(self, prompts, group_size, max_len, temperature=1.0, round_seed=0, prompt_index_base=0,
               prompt_tokens=None, prompt_offsets=None, outputs=None) -> Rollout:
        """preemptive_sample. outputs=(comp, lens, logp) reuses caller buffers."""
        if prompt_tokens is None:
            prompt_tokens, prompt_offsets = pack_prompts(prompts)
        n_prompts = len(prompt_offsets) - 1
        S = n_prompts * group_size
        if outputs is None:
            comp = np.zeros((S, max(max_len, 1)), dtype=np.int32)
            lens = np.zeros(S, dtype=np.int32)
            logp = np.zeros((S, max(max_len, 1)), dtype=np.float32)
        else:
            comp, lens, logp = outputs
        plan = Plan(n_prompts, group_size, max_len, float(temperature), int(round_seed) & (2**64 - 1),
                    int(prompt_index_base))
        _check(lib().dashcu_sample(self.h, C.byref(plan), _p(prompt_tokens, i32p), _p(prompt_offsets, i64p),
                                   _p(comp, i32p), _p(lens, i32p), _p(logp, f32p)))
        return Rollout(comp, lens, logp)

    def load_rollout(self, prompts, group_size, completions):
        pt, po = pack_prompts(prompts)
        ct = np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.int32) for c in completions] +
                                                 [np.zeros(0, dtype=np.int32)]), dtype=np.int32)
        co = np.zeros(len(completions) + 1, dtype=np.int64)
        co[1:] = np.cumsum([len(c) for c in completions])
        if ct.shape[0] == 0:
            ct = np.zeros(1, dtype=np.int32)
        _check(lib().dashcu_rollout_load(self.h, _p(pt, i32p), _p(po, i64p), len(prompts), group_size, _p(ct, i32p),
                                         _p(co, i64p)))

    def rollout_log_prob(self, n_tokens: int) -> np.ndarray:
        out = np.zeros(max(n_tokens, 1), dtype=np.float32)
        _check(lib().dashcu_rollout_log_prob(self.h, _p(out, f32p), n_tokens))
        return out[:n_tokens]

    # ---- advantage / filter
    def task_rewards(self, kind: int, difficulty: int, seeds, vocab: int = VOCAB_TASK):
        """Rewards of the current rollout from the task (dashcu_rollout_task_rewards)."""
        sd = _seeds(seeds)
        _check(lib().dashcu_rollout_task_rewards(self.h, kind, difficulty, vocab,
                                                 sd.ctypes.data_as(C.POINTER(C.c_uint64))))

    def set_rewards(self, rewards):
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        _check(lib().dashcu_rollout_set_rewards(self.h, _p(r, f64p), r.shape[0]))

    def advantage(self, kind=ADV_GROUP, normalize=False, eps=0.0, tau=0.1):
        n = self.stats()["n_seq"]
        tau = FILTER_OFF if tau is None else tau   # None: no filter (GRPO-style), every sequence kept
        adv = np.zeros(max(n, 1))
        kept = np.zeros(max(n, 1), dtype=np.uint8)
        nk = C.c_int32(0)
        _check(lib().dashcu_rollout_advantage(self.h, kind, int(normalize), eps, tau, _p(adv, f64p), _p(kept, u8p),
                                              C.byref(nk)))
        return adv[:n], kept[:n].astype(bool), int(nk.value)

    # ---- gradient / update
    def grad_zero(self):
        _check(lib().dashcu_grad_zero(self.h))

    def accumulate(self, weight_scale: float, micro_batch: int = 32):
        _check(lib().dashcu_accumulate(self.h, weight_scale, micro_batch))

    def accumulate_weighted(self, weights, micro_batch: int = 32):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        _check(lib().dashcu_accumulate_weighted(self.h, _p(w, f64p), w.shape[0], micro_batch))

    def rebalance(self):
        """Move kept sequences between ranks to even out the accumulate work (collective)."""
        o, i = C.c_int32(0), C.c_int32(0)
        _check(lib().dashcu_rebalance(self.h, C.byref(o), C.byref(i)))
        return o.value, i.value

    # ---- PPO / KL / schedules
    def snapshot(self):
        """theta_old of the current rollout (dashcu_rollout_snapshot)."""
        _check(lib().dashcu_rollout_snapshot(self.h))

    def snapshot_logp(self) -> np.ndarray:
        n = self.stats()["n_seq"]
        out = np.zeros(max(n, 1))
        _check(lib().dashcu_rollout_snapshot_logp(self.h, _p(out, f64p), n))
        return out[:n]

    def accumulate_ppo(self, weight_scale: float, clip_eps: float = 0.2, micro_batch: int = 32, subset=None):
        """Clipped-surrogate gradient over the kept (x subset) sequences; returns (surrogate, n_clipped)."""
        sub = None if subset is None else np.ascontiguousarray(subset, dtype=np.int32)
        sur, nc = C.c_double(0), C.c_int32(0)
        _check(lib().dashcu_accumulate_ppo(self.h, weight_scale, clip_eps, micro_batch, _p(sub, i32p),
                                           0 if sub is None else sub.shape[0], C.byref(sur), C.byref(nc)))
        return sur.value, nc.value

    def accumulate_kl(self, base: "Policy", coef: float, micro_batch: int = 32, subset=None) -> np.ndarray:
        """grad += coef * grad KL(base || current) over the subset (all sequences); per-sequence KL values."""
        n = self.stats()["n_seq"]
        sub = None if subset is None else np.ascontiguousarray(subset, dtype=np.int32)
        out = np.zeros(max(n if sub is None else sub.shape[0], 1))
        _check(lib().dashcu_accumulate_kl(self.h, base.h, coef, micro_batch, _p(sub, i32p),
                                          0 if sub is None else sub.shape[0], _p(out, f64p)))
        return out[:(n if sub is None else sub.shape[0])]

    def run_schedule(self, kind=SCHED_DASH, K=1, weight_scale=1.0, clip_eps=0.2, beta=0.0, micro_batch=32,
                     sharded=False, base: "Policy" = None, opt_kind=OPT_ADAM, lr=1e-3, beta1=0.9, beta2=0.999,
                     eps=1e-8):
        sc = Schedule(kind, K, clip_eps, beta, weight_scale, micro_batch, int(sharded))
        o = Opt(opt_kind, lr, beta1, beta2, eps)
        logs = (StepLog * max(K, 1))()
        n = C.c_int32(0)
        _check(lib().dashcu_run_schedule(self.h, C.byref(sc), C.byref(o), base.h if base else None, logs, max(K, 1),
                                         C.byref(n)))
        return [logs[i].as_dict() for i in range(min(n.value, max(K, 1)))]

    def grad(self) -> np.ndarray:
        out = np.zeros(self.n_params)
        _check(lib().dashcu_grad_download(self.h, _p(out, f64p), self.n_params))
        return out

    def grad_upload(self, grad):
        g = np.ascontiguousarray(grad, dtype=np.float64)
        _check(lib().dashcu_grad_upload(self.h, _p(g, f64p), g.shape[0]))

    def allreduce_grads(self):
        _check(lib().dashcu_allreduce_grads(self.h))

    def optimizer_step(self, kind=OPT_ADAM, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        o = Opt(kind, lr, beta1, beta2, eps)
        _check(lib().dashcu_optimizer_step(self.h, C.byref(o)))

    def sharded_step(self, kind=OPT_ADAM, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        """reduce-scatter + update of this rank's slice + all-gather (dashcu_sharded_step)."""
        o = Opt(kind, lr, beta1, beta2, eps)
        _check(lib().dashcu_sharded_step(self.h, C.byref(o)))

    def fused_step(self, kind=OPT_ADAM, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        """reduce-scatter + update + all-gather as one kernel over peer memory (dashcu_fused_step)."""
        o = Opt(kind, lr, beta1, beta2, eps)
        _check(lib().dashcu_fused_step(self.h, C.byref(o)))

    def stats(self) -> dict:
        s = Stats()
        _check(lib().dashcu_get_stats(self.h, C.byref(s)))
        return s.as_dict()

    def close(self):
        if self.h:
            lib().dashcu_policy_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
