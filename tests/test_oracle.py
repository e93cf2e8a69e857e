"""Pins the CPU oracle (oracle/dash_oracle.c) before anything is checked against it:
golden vectors from SPEC.md / SURVEY App.A, and agreement with the unmodified
reference compiled in place (oracle/_ref)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle_ffi as O

C1 = dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2, bos_id=0, eos_id=1)
SMALL = dict(vocab_size=11, embed_dim=8, context_len=16, ffn_hidden=12, n_layers=2, bos_id=0, eos_id=1)
GQA = dict(vocab_size=7, embed_dim=4, context_len=8, ffn_hidden=4, n_layers=2, bos_id=0, eos_id=1,
           n_heads=2, n_kv_heads=1, head_dim=2)
GQA2 = dict(vocab_size=7, embed_dim=6, context_len=8, ffn_hidden=4, n_layers=1, bos_id=0, eos_id=1,
            n_heads=4, n_kv_heads=2, head_dim=2)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ----------------------------------------------------------------- rng.hpp

def test_rng_golden():
    L = O.oracle()
    assert L.dor_splitmix64(0) == 16294208416658607535
    assert L.dor_fnv1a(b"sample") == 17570797238186910919
    assert O.derive_seed(1, "sample", 2, 3) == 3124241217676271300
    out = np.zeros(2, dtype=np.uint64)
    L.dor_rng_draws(1, 0, 1, O.ptr(out, O.u64p))
    assert int(out[0]) == 2469588189546311528
    L.dor_rng_draws(1, 1, 2, O.ptr(out, O.u64p))   # App.A: next_u64, then uniform01
    assert out.view(np.float64)[1] == 0.13640703636619722
    L.dor_rng_draws(1, 2, 1, O.ptr(out, O.u64p))
    assert out.view(np.float64)[0] == -0.039399956754155314


@pytest.mark.ref
def test_rng_matches_reference():
    R = O.ref()
    for kind in (0, 1, 2):
        a = np.zeros(1000, dtype=np.uint64)
        b = np.zeros(1000, dtype=np.uint64)
        O.oracle().dor_rng_draws(99, kind, 1000, O.ptr(a, O.u64p))
        R.ref_rng_draws(99, kind, 1000, O.ptr(b, O.u64p))
        assert np.array_equal(a, b)
    for base, tag, x, y in [(0, "sample", 0, 0), (7, "reward", 5, 9), (2**63, "prompt", 11, 0)]:
        assert O.derive_seed(base, tag, x, y) == R.ref_derive_seed(base, tag.encode(), x, y)


# ------------------------------------------------------------- tensors.cpp

def test_c1_params_golden():
    assert O.num_params(C1) == 468480
    p = O.init_params(C1, 0.02, 1)
    assert p[0] == -0.00078799913508310632


def test_gqa_111d_is_reference_layout():
    a = dict(C1, n_heads=1, n_kv_heads=1, head_dim=128)
    assert O.num_params(a) == O.num_params(C1) == 468480


@pytest.mark.ref
def test_init_matches_reference_bitwise():
    for arch in (C1, SMALL):
        a = np.zeros(O.num_params(arch))
        O.ref().ref_init_params(O.arch_ref_vec(arch), 0.02, 1, O.ptr(a, O.f64p))
        assert np.array_equal(a, O.init_params(arch, 0.02, 1))
    h = C.c_uint64(0)
    O.ref().ref_content_hash(O.arch_ref_vec(C1), O.ptr(O.init_params(C1, 0.02, 1), O.f64p), C.byref(h))
    assert h.value == 0xdc95454214facbbf


# --------------------------------------------------------------- policy.cpp

def test_uniform_policy_log_prob():
    arch = dict(vocab_size=4, embed_dim=4, context_len=8, ffn_hidden=4, n_layers=1, bos_id=-1, eos_id=3)
    p = np.zeros(O.num_params(arch))
    tot, per = O.log_prob(arch, p, [0, 1], [2, 1, 0])
    assert tot == pytest.approx(-3 * math.log(4), abs=1e-12)
    tot0, per0 = O.log_prob(arch, p, [0, 1], [])
    assert tot0 == 0.0 and len(per0) == 0


def test_sample_golden_log_prob():
    # SURVEY App.A: reference sample() on the C1 policy produced this completion.
    p = O.init_params(C1, 0.02, 1)
    comp = [66, 75, 40, 115, 241, 20, 64, 51]
    tot, _ = O.log_prob(C1, p, [0, 50, 51, 43, 52, 53, 61], comp)
    assert tot == -44.304636820128032


def _rand_traj(rng, arch, m, n):
    V = arch["vocab_size"]
    prompt = [arch["bos_id"]] + list(rng.integers(2, V, size=m - 1))
    comp = list(rng.integers(1, V, size=n))
    return prompt, comp


@pytest.mark.ref
def test_log_prob_and_grad_match_reference():
    R = O.ref()
    rng = np.random.default_rng(0)
    for arch in (SMALL, C1):
        p = O.init_params(arch, 0.3 if arch is SMALL else 0.02, 3)
        for trial in range(3):
            prompt, comp = _rand_traj(rng, arch, 3 + trial, 4 + 2 * trial)
            tot, per = O.log_prob(arch, p, prompt, comp)
            rp, rc = O.i32(prompt), O.i32(comp)
            per_r = np.zeros(len(comp))
            tot_r = C.c_double(0)
            assert R.ref_log_prob(O.arch_ref_vec(arch), O.ptr(p, O.f64p), O.ptr(rp, O.i32p), len(rp),
                                  O.ptr(rc, O.i32p), len(rc), O.ptr(per_r, O.f64p), C.byref(tot_r)) == 0
            assert tot == tot_r.value            # bit-exact forward
            assert np.array_equal(per, per_r)
            g = O.grad_log_prob(arch, p, prompt, comp)
            g_r = np.zeros_like(g)
            assert R.ref_grad_log_prob(O.arch_ref_vec(arch), O.ptr(p, O.f64p), O.ptr(rp, O.i32p), len(rp),
                                       O.ptr(rc, O.i32p), len(rc), O.ptr(g_r, O.f64p)) == 0
            assert rel(g, g_r) <= 1e-12


@pytest.mark.ref
def test_ref_sample_golden_and_replay():
    R = O.ref()
    p = O.init_params(C1, 0.02, 1)
    prompt = O.i32([0, 50, 51, 43, 52, 53, 61])
    comp = np.zeros(8, dtype=np.int32)
    lp = np.zeros(8)
    n = C.c_int32(0)
    seed = O.derive_seed(7, "sample", 0, 0)
    assert R.ref_sample(O.arch_ref_vec(C1), O.ptr(p, O.f64p), O.ptr(prompt, O.i32p), 7, 8, 1.0, seed,
                        O.ptr(comp, O.i32p), O.ptr(lp, O.f64p), C.byref(n)) == 0
    assert list(comp[:n.value]) == [66, 75, 40, 115, 241, 20, 64, 51]
    assert lp[:n.value].sum() == pytest.approx(-44.304636820128032, abs=1e-12)
    # SPEC:86 replay: recorded log-probs == log_prob() bit for bit; the oracle agrees.
    _, per = O.log_prob(C1, p, prompt, comp[:n.value])
    assert np.array_equal(per, lp[:n.value])


def _fd_check(arch, seed):
    rng = np.random.default_rng(seed)
    p = O.init_params(arch, 0.5, 100 + seed)
    prompt, comp = _rand_traj(rng, arch, 3, 4)
    g = O.grad_log_prob(arch, p, prompt, comp)
    worst = 0.0
    h = 1e-4
    for i in range(len(p)):
        pp, pm = p.copy(), p.copy()
        pp[i] += h
        pm[i] -= h
        fd = (O.log_prob(arch, pp, prompt, comp)[0] - O.log_prob(arch, pm, prompt, comp)[0]) / (2 * h)
        worst = max(worst, abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1e-3))
    return worst


def test_gqa_gradient_finite_differences():
    # central FD, step 1e-4, <= 500 params, rel <= 1e-4 (GQA extension App.B D1).
    for arch in (GQA, GQA2):
        assert O.num_params(arch) <= 500
        for seed in range(20):
            assert _fd_check(arch, seed) <= 1e-4


def test_gqa_reduces_to_reference_geometry():
    # n_heads = n_kv_heads = 1, head_dim = d is the reference model.
    a = dict(SMALL, n_heads=1, n_kv_heads=1, head_dim=SMALL["embed_dim"])
    p = O.init_params(SMALL, 0.3, 5)
    rng = np.random.default_rng(1)
    prompt, comp = _rand_traj(rng, SMALL, 4, 6)
    assert O.log_prob(a, p, prompt, comp)[0] == O.log_prob(SMALL, p, prompt, comp)[0]


# ----------------------------------------------------------- sampling rule

def test_soft_log_accuracy():
    L = O.oracle()
    xs = np.concatenate([np.geomspace(1e-7, 20.0, 2000), [1.0, 2.0, 0.5]]).astype(np.float32)
    for x in xs:
        v = L.dor_soft_logf(float(x))
        assert abs(v - math.log(float(x))) <= 2e-6 * max(1.0, abs(math.log(float(x))))


def test_sample_rule_deterministic_and_masks_bos():
    logits = np.random.default_rng(0).standard_normal(257).astype(np.float32)
    logits[0] = 1e9   # BOS must never win
    a = O.sample_rule(logits, 0, 1.0, 1234, 3)
    assert a == O.sample_rule(logits, 0, 1.0, 1234, 3) and a != 0
    one_hot = np.zeros(50, dtype=np.float32)
    one_hot[17] = 1e4   # argmax-forcing
    assert all(O.sample_rule(one_hot, 0, 1.0, k, s) == 17 for k in range(5) for s in range(5))


@pytest.mark.ref
def test_sample_rule_distribution_matches_reference_probs():
    # SPEC:63-style concentration check against reference next_token_probs (policy.cpp:524-537).
    arch = dict(vocab_size=12, embed_dim=8, context_len=16, ffn_hidden=8, n_layers=1, bos_id=0, eos_id=1)
    p = O.init_params(arch, 0.8, 4)
    ctx = O.i32([0, 3, 4])
    probs = np.zeros(12)
    O.ref().ref_next_token_probs(O.arch_ref_vec(arch), O.ptr(p, O.f64p), O.ptr(ctx, O.i32p), 3,
                                 O.ptr(probs, O.f64p))
    lg = O.next_logits(arch, p, ctx).astype(np.float32)
    n = 100000
    counts = np.zeros(12)
    for k in range(n):
        counts[O.sample_rule(lg, 0, 1.0, O.derive_seed(9, "sample", k, 0), 0)] += 1
    assert counts[0] == 0
    sd = np.sqrt(n * probs * (1 - probs))
    assert np.all(np.abs(counts - n * probs)[1:] <= 3.5 * sd[1:] + 1)
    # temperature 0.5 -> softmax(logits / 0.5)
    q = np.exp(2 * (lg.astype(np.float64) - lg.max()))
    q[0] = 0
    q /= q.sum()
    counts[:] = 0
    for k in range(n):
        counts[O.sample_rule(lg, 0, 2.0, O.derive_seed(9, "sample", k, 1), 0)] += 1
    sd = np.sqrt(n * q * (1 - q))
    assert np.all(np.abs(counts - n * q)[1:] <= 3.5 * sd[1:] + 1)


def test_oracle_sampler_replays_its_log_probs():
    p = O.init_params(C1, 0.02, 1)
    comp, lp = O.sample(C1, p, [0, 50, 51, 43, 52, 53, 61], 12, 1.0, O.derive_seed(7, "sample", 0, 0))
    assert len(comp) == 12 or comp[-1] == 1
    _, per = O.log_prob(C1, p, [0, 50, 51, 43, 52, 53, 61], comp)
    assert np.array_equal(per, lp)


# ------------------------------------------------------------ advantage.cpp

def test_advantage_golden():
    adv, kept, idx = O.advantage_filter([1, 0, 1, 0], 4, kind=0)
    assert list(adv) == [0.5, -0.5, 0.5, -0.5]
    adv, _, _ = O.advantage_filter([1, 0, 0, 1, 1, 1], 2, kind=1)
    assert list(adv) == [0.5, -0.5, -0.5, 0.5, 0.0, 0.0]
    adv, _, _ = O.advantage_filter([1, 0], 2, kind=2)
    assert list(adv) == [1.0, -1.0]
    adv, _, _ = O.advantage_filter([1, 0], 2, kind=1, normalize=True, eps=0.0)
    assert list(adv) == [1.0, -1.0]
    adv, _, _ = O.advantage_filter([1, 1], 2, kind=1, normalize=True, eps=1e-4)
    assert list(adv) == [0.0, 0.0]
    with pytest.raises(ValueError):
        O.advantage_filter([1, 0, 1], 2)
    with pytest.raises(ValueError):
        O.advantage_filter([1, 0], 1, kind=2)
    with pytest.raises(ValueError):
        O.advantage_filter([1, 0], 2, tau=-0.1)
    with pytest.raises(ValueError):
        O.advantage_filter([], 1)


def test_filter_golden():
    # SPEC:245-247 (kind 1 with singleton groups leaves A unchanged? no: use LOO-free path)
    A = np.array([0.05, -0.5, 0.0, 0.25])
    kept = np.abs(A) > 0.1
    assert list(kept) == [False, True, False, True]
    # run through the oracle's filter by feeding rewards that give these advantages
    r = np.array([0.05, -0.5, 0.0, 0.25, 0.0, 0.0, 0.0, 0.0])
    adv, kept, idx = O.advantage_filter(r, 1, kind=1, tau=0.1)  # singleton groups -> A = 0
    assert not kept.any() and len(idx) == 0


@pytest.mark.ref
def test_advantage_matches_reference_random():
    R = O.ref()
    rng = np.random.default_rng(0)
    for G in (1, 2, 4, 8, 10, 16):
        for kind in (0, 1, 2):
            if kind == 2 and G < 2:
                continue
            r = rng.integers(0, 2, size=G * 7).astype(np.float64)
            if kind == 1:
                r += rng.standard_normal(r.shape) * (G == 10)
            out = np.zeros_like(r)
            assert R.ref_advantage(O.ptr(r, O.f64p), len(r), G, kind, O.ptr(out, O.f64p)) == 0
            for tau in (0.0, 0.1, 0.125, float("inf")):
                adv, kept, idx = O.advantage_filter(r, G, kind=kind, tau=tau)
                assert np.array_equal(adv, out)
                k = np.zeros(len(r), dtype=np.uint8)
                kc = C.c_int32(0)
                ff = C.c_double(0)
                ma = C.c_double(0)
                assert R.ref_filter_by_threshold(O.ptr(out, O.f64p), len(r), tau, O.ptr(k, O.u8p),
                                                 C.byref(kc), C.byref(ff), C.byref(ma)) == 0
                assert np.array_equal(kept, k.astype(bool))
                assert list(idx) == list(np.nonzero(k)[0])
            # no filter (GRPO-style): group_advantage's kept stays all 1 (advantage.cpp:77, :92)
            adv, kept, idx = O.advantage_filter(r, G, kind=kind, tau=None)
            assert np.array_equal(adv, out) and kept.all() and list(idx) == list(range(len(r)))
            with pytest.raises(ValueError):
                O.advantage_filter(r, G, kind=kind, tau=-0.5)
            norm = np.zeros_like(r)
            assert R.ref_normalize_std(O.ptr(out, O.f64p), O.ptr(r, O.f64p), len(r), G if kind else len(r),
                                       1e-6, O.ptr(norm, O.f64p)) == 0
            adv_n, _, _ = O.advantage_filter(r, G, kind=kind, normalize=True, eps=1e-6)
            assert np.array_equal(adv_n, norm)


# -------------------------------------------------------------- updates

def _batch(rng, arch, n):
    ps, cs = [], []
    for _ in range(n):
        p, c = _rand_traj(rng, arch, 3, int(rng.integers(0, 5)))
        ps.append(p)
        cs.append(c)
    return ps, cs


def _pg(arch, params, ps, cs, w):
    P = O.i32([t for p in ps for t in p])
    Cc = O.i32([t for c in cs for t in c] or [0])
    po = np.cumsum([0] + [len(p) for p in ps]).astype(np.int64)
    co = np.cumsum([0] + [len(c) for c in cs]).astype(np.int64)
    g = np.zeros(O.num_params(arch))
    w = np.ascontiguousarray(w, dtype=np.float64)
    a = O.arch_struct(arch)
    O.oracle().dor_pg_accumulate(C.byref(a), O.ptr(params, O.f64p), len(ps), O.ptr(P, O.i32p),
                                 O.ptr(po, O.i64p), O.ptr(Cc, O.i32p), O.ptr(co, O.i64p), O.ptr(w, O.f64p),
                                 O.ptr(g, O.f64p))
    return g


def test_filter_equivalence_and_microbatch_invariance():
    # SPEC:252/:342 (kept-only == zeroed-A) and SPEC:326/:341 (partition invariance), 1e-9.
    rng = np.random.default_rng(3)
    p = O.init_params(SMALL, 0.3, 2)
    ps, cs = _batch(rng, SMALL, 16)
    r = rng.integers(0, 2, size=16).astype(np.float64)
    adv, kept, idx = O.advantage_filter(r, 4, kind=1, tau=0.1)
    N = 16
    full = _pg(SMALL, p, ps, cs, np.where(kept, adv, 0.0) / N)
    only = _pg(SMALL, p, [ps[i] for i in idx], [cs[i] for i in idx], adv[idx] / N)
    assert rel(only, full) <= 1e-9
    parts = sum(_pg(SMALL, p, [ps[i] for i in idx[k:k + 3]], [cs[i] for i in idx[k:k + 3]],
                    adv[idx[k:k + 3]] / N) for k in range(0, len(idx), 3))
    assert rel(parts, full) <= 1e-9


def test_optimizer_golden():
    L = O.oracle()
    p = np.array([1.0, -2.0])
    g = np.array([0.5, 0.0])
    L.dor_sgd_step(O.ptr(p, O.f64p), O.ptr(g, O.f64p), 2, 0.1)
    assert list(p) == [1.05, -2.0]
    # Adam, 2-parameter hand trace: step 1 moves each coordinate by lr*sign(g).
    p = np.array([1.0, -2.0])
    m = np.zeros(2)
    v = np.zeros(2)
    g = np.array([0.5, -0.25])
    L.dor_adam_step(O.ptr(p, O.f64p), O.ptr(g, O.f64p), O.ptr(m, O.f64p), O.ptr(v, O.f64p), 2, 1, 1e-3,
                    0.9, 0.999, 1e-8)
    assert p == pytest.approx([1.0 + 1e-3, -2.0 - 1e-3], abs=1e-10)
    g2 = np.zeros(2)
    m0, v0 = m.copy(), v.copy()
    L.dor_adam_step(O.ptr(p, O.f64p), O.ptr(g2, O.f64p), O.ptr(m, O.f64p), O.ptr(v, O.f64p), 2, 2, 1e-3,
                    0.9, 0.999, 1e-8)
    assert list(m) == list(0.9 * m0) and list(v) == list(0.999 * v0)   # zero grad: moments decay only


# --------------------------------------------------------------- tasks (C1)

@pytest.mark.ref
def test_add_instance_golden():
    prompt = np.zeros(16, dtype=np.int32)
    m = C.c_int32(0)
    ans = C.create_string_buffer(16)
    assert O.ref().ref_add_instance(2, 12345, O.ptr(prompt, O.i32p), C.byref(m), ans, 16) == 0
    assert "".join(chr(t) for t in prompt[1:m.value]) == "76+51="
    assert ans.value == b"127" and prompt[0] == 0
    comp = O.i32([ord(c) for c in "6+1=07,7+5=12,#127"] + [1])
    r = C.c_double(0)
    assert O.ref().ref_add_reward(2, 12345, O.ptr(comp, O.i32p), len(comp), C.byref(r)) == 0
    assert r.value == 1.0


def test_synthetic_workload_shapes():
    pr = O.synthetic_prompt(5, 3, 128, 151936, 0, 1)
    assert pr[0] == 0 and pr[1:].min() >= 2 and pr.max() < 151936
    rs = np.array([O.synthetic_reward(1, m, g) for m in range(400) for g in range(8)]).reshape(400, 8)
    uniform = np.mean([(row.min() == row.max()) for row in rs])
    assert abs(uniform - 2 / 9) < 0.07      # E[p^G + (1-p)^G] = 2/(G+1)


def test_workload_restatement_matches_oracle():
    from paper_2505_17218_b200 import workload as W
    P = W.synthetic_prompts(5, 10, 14, 128, 151936, 0, 1)
    for i, m in enumerate(range(10, 14)):
        assert np.array_equal(P[i], O.synthetic_prompt(5, m, 128, 151936, 0, 1))
    P = W.synthetic_prompts(9, 0, 3, 9, 40, 5, 2)
    for m in range(3):
        assert np.array_equal(P[m], O.synthetic_prompt(9, m, 9, 40, 5, 2))
    R = W.synthetic_rewards(3, 7, 20, 8)
    assert np.array_equal(R, [O.synthetic_reward(3, m, g) for m in range(7, 20) for g in range(8)])
    assert int(W.derive_seed(1, "sample", 2, 3)) == 3124241217676271300


# ------------------------------------------------------------------- KL term

@pytest.mark.ref
def test_kl_term_matches_reference():
    """dor_kl_term_acc (the GQA-capable restatement) == the reference's kl_term
    (policy.cpp:487-522) at reference geometry; kl(params, params) = (0, 0)."""
    arch = dict(vocab_size=11, embed_dim=8, context_len=20, ffn_hidden=12, n_layers=2, bos_id=0, eos_id=1)
    p = O.init_params(arch, 0.4, 3)
    b = p + 0.05 * np.random.default_rng(1).standard_normal(len(p))
    prompt, comp = [0, 4, 5], [6, 7, 2, 9, 1]
    v, g = O.kl_term(arch, p, b, prompt, comp)
    rv, rg = C.c_double(0), np.zeros(len(p))
    assert O.ref().ref_kl_term(O.arch_ref_vec(arch), O.ptr(p, O.f64p), O.ptr(b, O.f64p), O.i32(prompt).ctypes.data_as(O.i32p),
                               3, O.i32(comp).ctypes.data_as(O.i32p), 5, C.byref(rv), O.ptr(rg, O.f64p)) == 0
    assert abs(v - rv.value) <= 1e-12 * max(1, abs(v)) and v > 0
    assert np.max(np.abs(g - rg)) <= 1e-12 * max(1, np.max(np.abs(rg)))
    v0, g0 = O.kl_term(arch, p, p, prompt, comp)
    assert abs(v0) <= 1e-12 and np.max(np.abs(g0)) <= 1e-12


def test_kl_term_gqa_finite_differences():
    arch = dict(vocab_size=9, embed_dim=8, context_len=16, ffn_hidden=6, n_layers=1, bos_id=0, eos_id=1,
                n_heads=2, n_kv_heads=1, head_dim=4)
    rng = np.random.default_rng(2)
    p = O.init_params(arch, 0.5, 5)
    b = p + 0.1 * rng.standard_normal(len(p))
    prompt, comp = [0, 3, 4], [5, 2, 7]
    _, g = O.kl_term(arch, p, b, prompt, comp)
    for i in rng.choice(len(p), 25, replace=False):
        e = np.zeros(len(p))
        e[i] = 1e-5
        fd = (O.kl_term(arch, p + e, b, prompt, comp)[0] - O.kl_term(arch, p - e, b, prompt, comp)[0]) / 2e-5
        assert abs(fd - g[i]) <= 1e-4 * max(1e-3, abs(fd)), (i, fd, g[i])
