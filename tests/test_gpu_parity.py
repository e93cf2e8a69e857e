"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle on
identical inputs and seeds.

Standards (BASELINE.json north_star):
  * integer / index work bit-exact: sampled token ids under a shared logits dump,
    advantages, filter masks and compacted kept indices;
  * floating point within tolerance: log-probs and gradients <= 1e-3 relative in
    fp32 (DASHCU_F32) and <= 2e-2 in bf16 (DASHCU_BF16), relative error measured
    norm-wise per parameter tensor (SURVEY App.B D9).
Weights are rounded to fp32 before both sides see them, so the oracle and the
device start from identical parameters.
"""
import numpy as np
import pytest

import oracle_ffi as O
import paper_2505_17218_b200 as D

pytestmark = pytest.mark.gpu

C1 = dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2, bos_id=0, eos_id=1)
SMALL = dict(vocab_size=37, embed_dim=32, context_len=40, ffn_hidden=48, n_layers=2, bos_id=0, eos_id=1)
GQA = dict(vocab_size=64, embed_dim=64, context_len=48, ffn_hidden=128, n_layers=2, bos_id=0, eos_id=1,
           n_heads=4, n_kv_heads=2, head_dim=16)
# geometries that exercise the tensor-core attention kernels (head_dim 64 / 128)
QWENLIKE = dict(vocab_size=300, embed_dim=256, context_len=48, ffn_hidden=256, n_layers=2, bos_id=0, eos_id=1,
                n_heads=14, n_kv_heads=2, head_dim=64)
GQA128 = dict(vocab_size=64, embed_dim=128, context_len=48, ffn_hidden=128, n_layers=2, bos_id=0, eos_id=1,
              n_heads=4, n_kv_heads=2, head_dim=128)
LONG = dict(vocab_size=64, embed_dim=128, context_len=200, ffn_hidden=128, n_layers=1, bos_id=0, eos_id=1,
            n_heads=2, n_kv_heads=1, head_dim=64)
# vocab spanning many fused-sampling tiles (ragged last tile)
VBIG = dict(vocab_size=5003, embed_dim=64, context_len=32, ffn_hidden=64, n_layers=1, bos_id=0, eos_id=1,
            n_heads=1, n_kv_heads=1, head_dim=64)
# several 128-key / 128-query tiles per sequence (tcgen05 attention backward, GQA group 2)
LONGGQA = dict(vocab_size=64, embed_dim=256, context_len=320, ffn_hidden=128, n_layers=1, bos_id=0, eos_id=1,
               n_heads=4, n_kv_heads=2, head_dim=64)
# head_dim 128 (the 1.5B / 3B geometry) over several 128-key tiles
LONGGQA128 = dict(vocab_size=64, embed_dim=256, context_len=320, ffn_hidden=128, n_layers=1, bos_id=0, eos_id=1,
                  n_heads=4, n_kv_heads=2, head_dim=128)
# ffn_hidden 4096: the decode's W2 GEMM has K = 4096 over one output tile per row block
WIDEFFN = dict(vocab_size=64, embed_dim=128, context_len=48, ffn_hidden=4096, n_layers=2, bos_id=0, eos_id=1,
               n_heads=2, n_kv_heads=1, head_dim=64)
TOL = {D.F32: 1e-3, D.BF16: 2e-2}


@pytest.fixture(scope="module")
def ctx():
    return D.Context(0)


def params32(arch, scale, seed):
    """Weights rounded to fp32. `scale` is relative: N(0, (scale / sqrt(d))^2) keeps the
    residual stream O(1) so the attention softmax is not saturated (a saturated softmax
    makes fp32/bf16-vs-fp64 gradient comparisons meaningless, not wrong)."""
    sc = scale / np.sqrt(arch["embed_dim"]) if scale > 0.05 else scale
    return O.init_params(arch, sc, seed).astype(np.float32).astype(np.float64)


def tensor_slices(arch):
    """(name, slice) per parameter tensor in views() order."""
    g = dict(arch)
    nh, nkv = g.get("n_heads") or 1, g.get("n_kv_heads") or 1
    hd = g.get("head_dim") or g["embed_dim"]
    V, d, H = g["vocab_size"], g["embed_dim"], g["ffn_hidden"]
    qd, kvd = nh * hd, nkv * hd
    sizes = [("token_embed", V * d), ("pos_embed", g["context_len"] * d)]
    for l in range(g["n_layers"]):
        sizes += [(f"{l}.wq", qd * d), (f"{l}.wk", kvd * d), (f"{l}.wv", kvd * d), (f"{l}.wo", d * qd),
                  (f"{l}.w1", H * d), (f"{l}.b1", H), (f"{l}.w2", d * H), (f"{l}.b2", d)]
    sizes += [("w_out", V * d), ("b_out", V)]
    out, off = [], 0
    for n, s in sizes:
        out.append((n, slice(off, off + s)))
        off += s
    return out


def assert_grad_close(arch, got, ref, tol):
    worst = []
    for name, sl in tensor_slices(arch):
        nr = np.linalg.norm(ref[sl])
        if nr < 1e-12 * max(1.0, np.linalg.norm(ref)):
            assert np.linalg.norm(got[sl]) <= 1e-6 * max(1.0, np.linalg.norm(ref)), name
            continue
        e = np.linalg.norm(got[sl] - ref[sl]) / nr
        worst.append((e, name))
    worst.sort(reverse=True)
    assert worst[0][0] <= tol, worst[:3]


def rand_batch(rng, arch, n_prompts, G, m_range=(2, 6), len_range=(0, 9)):
    V = arch["vocab_size"]
    prompts = [[arch["bos_id"]] + list(rng.integers(2, V, size=int(rng.integers(*m_range)) - 1))
               for _ in range(n_prompts)]
    comps = []
    for p in prompts:
        for _ in range(G):
            n = int(rng.integers(*len_range))
            c = list(rng.integers(2, V, size=n))
            if n and rng.random() < 0.3:
                c[-1] = arch["eos_id"]
            comps.append(c)
    return prompts, comps


# ----------------------------------------------------------- advantage/filter

def test_advantage_filter_bit_exact(ctx):
    rng = np.random.default_rng(0)
    for G in (1, 2, 4, 8, 10, 16):
        for kind in (D.ADV_SINGLE_PATH, D.ADV_GROUP, D.ADV_LEAVE_ONE_OUT):
            if kind == D.ADV_LEAVE_ONE_OUT and G < 2:
                continue
            for binary in (True, False):
                r = rng.integers(0, 2, size=G * 33).astype(np.float64)
                if not binary:
                    r = rng.standard_normal(G * 33)
                for tau in (0.0, 0.1, 0.125, float("inf"), None):
                    for norm in (False, True):
                        a, k, i = ctx.advantage_filter(r, G, kind, norm, 1e-6, tau)
                        ra, rk, ri = O.advantage_filter(r, G, kind, norm, 1e-6, tau)
                        assert np.array_equal(a, ra) and np.array_equal(k, rk) and np.array_equal(i, ri)


def test_advantage_filter_large_and_errors(ctx):
    r = np.random.default_rng(1).integers(0, 2, size=16384).astype(np.float64)
    a, k, i = ctx.advantage_filter(r, 8, D.ADV_GROUP, False, 0, 0.1)
    ra, rk, ri = O.advantage_filter(r, 8, 1, False, 0, 0.1)
    assert np.array_equal(a, ra) and np.array_equal(k, rk) and np.array_equal(i, ri)
    with pytest.raises(D.InputError):
        ctx.advantage_filter([1.0, 0.0, 1.0], 2)
    with pytest.raises(D.InputError):
        ctx.advantage_filter([1.0, 0.0], 2, tau=-1.0)
    with pytest.raises(D.InputError):
        ctx.advantage_filter([1.0, 0.0], 2, tau=float("nan"))
    a, k, i = ctx.advantage_filter(r, 8, D.ADV_GROUP, False, 0, None)   # filter off: all kept (advantage.cpp:92)
    assert k.all() and np.array_equal(i, np.arange(len(r))) and np.array_equal(a, ra)
    with pytest.raises(D.InputError):
        ctx.advantage_filter([1.0, 0.0], 1, kind=D.ADV_LEAVE_ONE_OUT)


# ---------------------------------------------------------------- sampling

@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
@pytest.mark.parametrize("arch", [C1, GQA, QWENLIKE, GQA128, VBIG], ids=["c1", "gqa", "qwenlike", "gqa128", "vbig"])
def test_sampled_tokens_bit_exact_under_logits_dump(ctx, arch, dtype):
    pol = D.Policy(ctx, arch, dtype)
    pol.upload(params32(arch, 0.5, 3))
    rng = np.random.default_rng(2)
    prompts = [[0] + list(rng.integers(2, arch["vocab_size"], size=int(rng.integers(1, 7)))) for _ in range(5)]
    G, ML, T = 4, 12, 0.7
    pol.set_logits_dump(True)
    ro = pol.sample(prompts, G, ML, temperature=T, round_seed=11, prompt_index_base=3)
    dump = pol.logits_dump(len(prompts) * G, ML)
    inv_t = float(np.float32(1.0 / T))
    n_eos = 0
    for s in range(len(prompts) * G):
        m, g = s // G, s % G
        key = O.derive_seed(11, "sample", 3 + m, g)
        L = int(ro.lengths[s])
        cap = min(ML, arch["context_len"] - len(prompts[m]))
        assert 1 <= L <= cap
        if L < cap:
            assert ro.completions[s, L - 1] == arch["eos_id"]
            n_eos += 1
        for j in range(L):
            tok = O.sample_rule(dump[s, j], arch["bos_id"], inv_t, key, j)
            assert tok == ro.completions[s, j], (s, j)
    # the bf16 sampler walks a slice recomputed by a second GEMM; it must equal the dump
    assert pol.stats()["slice_recompute_mismatches"] == 0
    pol.close()


def test_sampling_logits_and_logp_match_oracle_f32(ctx):
    arch = SMALL
    pol = D.Policy(ctx, arch, D.F32)
    p = params32(arch, 0.5, 5)
    pol.upload(p)
    prompts = [[0, 5, 9], [0, 7], [0, 3, 4, 8, 2]]
    pol.set_logits_dump(True)
    ro = pol.sample(prompts, 3, 10, temperature=1.0, round_seed=5)
    dump = pol.logits_dump(9, 10)
    for s in range(9):
        pr = prompts[s // 3]
        comp = list(ro.completion(s))
        for j in range(len(comp)):
            ref = O.next_logits(arch, p, pr + comp[:j])
            assert np.max(np.abs(dump[s, j] - ref)) <= 1e-4 * max(1.0, np.max(np.abs(ref)))
        _, per = O.log_prob(arch, p, pr, comp)
        assert np.max(np.abs(ro.logp[s, :len(comp)] - per)) <= 1e-3 * max(1.0, np.max(np.abs(per)))
    pol.close()


def test_scheduling_independence(ctx):
    # the sampled multiset does not depend on how prompts are split
    # across workers (here: one call vs two shards with prompt_index_base).
    arch = C1
    pol = D.Policy(ctx, arch, D.F32)
    pol.upload(params32(arch, 0.3, 1))
    rng = np.random.default_rng(3)
    prompts = [[0] + list(rng.integers(2, 256, size=6)) for _ in range(8)]
    full = pol.sample(prompts, 4, 16, round_seed=9)
    a = pol.sample(prompts[:3], 4, 16, round_seed=9, prompt_index_base=0)
    b = pol.sample(prompts[3:], 4, 16, round_seed=9, prompt_index_base=3)
    assert np.array_equal(full.completions, np.concatenate([a.completions, b.completions]))
    assert np.array_equal(full.lengths, np.concatenate([a.lengths, b.lengths]))
    pol.close()


@pytest.mark.parametrize("arch", [WIDEFFN, QWENLIKE], ids=["wideffn", "qwenlike"])
def test_scheduling_independence_bf16(ctx, arch):
    """bf16 production path: one preemptive call over 160 prompts x 8 equals two shards
    (prompt_index_base) and a 2-prompt interleaved call bit-for-bit: the decode GEMMs'
    per-element fp32 summation order depends on (N, K) only, not on the batch rows."""
    pol = D.Policy(ctx, arch, D.BF16)
    pol.upload(params32(arch, 0.3, 21))
    rng = np.random.default_rng(21)
    prompts = [[0] + list(rng.integers(2, arch["vocab_size"], size=int(rng.integers(3, 9)))) for _ in range(160)]
    full = pol.sample(prompts, 8, 20, round_seed=5, temperature=0.7)
    a = pol.sample(prompts[:37], 8, 20, round_seed=5, temperature=0.7, prompt_index_base=0)
    b = pol.sample(prompts[37:], 8, 20, round_seed=5, temperature=0.7, prompt_index_base=37)
    c = pol.sample(prompts[50:52], 8, 20, round_seed=5, temperature=0.7, prompt_index_base=50)
    assert np.array_equal(full.completions, np.concatenate([a.completions, b.completions]))
    assert np.array_equal(full.lengths, np.concatenate([a.lengths, b.lengths]))
    assert np.array_equal(full.logp, np.concatenate([a.logp, b.logp]))
    assert np.array_equal(full.completions[400:416], c.completions)
    pol.close()


def test_sample_errors(ctx):
    arch = SMALL
    pol = D.Policy(ctx, arch, D.F32)
    with pytest.raises(D.InputError):
        pol.sample([[0, 2]], 2, 4, temperature=0.0)
    with pytest.raises(D.InputError):
        pol.sample([[0, 2]], 2, -1)
    with pytest.raises(D.InputError):
        pol.sample([[0, 99]], 2, 4)
    with pytest.raises(D.CapacityError):
        pol.sample([[0] + [2] * 40], 2, 4)
    ro = pol.sample([[0] + [2] * 37], 2, 10)        # cap = ctx - m = 2
    assert ro.lengths.max() <= 2
    ro = pol.sample([[0, 2]], 2, 0)                 # max_len 0 -> empty completions
    assert ro.lengths.max() == 0
    pol.close()


# --------------------------------------------------------------- log_prob

@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
@pytest.mark.parametrize("arch", [SMALL, GQA, C1, QWENLIKE, GQA128], ids=["small", "gqa", "c1", "qwenlike",
                                                                          "gqa128"])
def test_teacher_forced_log_prob(ctx, arch, dtype):
    pol = D.Policy(ctx, arch, dtype)
    p = params32(arch, 0.3, 7)
    pol.upload(p)
    prompts, comps = rand_batch(np.random.default_rng(4), arch, 4, 3)
    pol.load_rollout(prompts, 3, comps)
    n_tok = sum(len(c) for c in comps)
    lp = pol.rollout_log_prob(n_tok)
    ref = np.concatenate([O.log_prob(arch, p, prompts[s // 3], comps[s])[1] for s in range(12)] + [np.zeros(0)])
    err = np.abs(lp - ref).max() if n_tok else 0.0
    assert err <= TOL[dtype] * max(1.0, np.abs(ref).max())
    pol.close()


# ----------------------------------------------------------------- gradients

@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
@pytest.mark.parametrize("arch", [SMALL, GQA, C1, QWENLIKE, GQA128], ids=["small", "gqa", "c1", "qwenlike",
                                                                          "gqa128"])
def test_pg_gradient_parity(ctx, arch, dtype):
    pol = D.Policy(ctx, arch, dtype)
    p = params32(arch, 0.3, 8)
    pol.upload(p)
    rng = np.random.default_rng(5)
    prompts, comps = rand_batch(rng, arch, 4, 4)
    pol.load_rollout(prompts, 4, comps)
    w = rng.standard_normal(16) / 16
    w[rng.random(16) < 0.25] = 0.0
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=5)
    got = pol.grad()
    ref = np.zeros_like(got)
    for s in range(16):
        O.grad_log_prob(arch, p, prompts[s // 4], comps[s], w[s], ref)
    assert_grad_close(arch, got, ref, TOL[dtype])
    pol.close()


@pytest.mark.parametrize("kernel", ["tc5", "mma", "tc5:0", "tc5:3"])
def test_pg_gradient_parity_long_sequences(ctx, knob, kernel):
    """Ragged sequences up to 300 tokens: several key and query tiles, the causal
    diagonal tiles and ragged tile ends, through the tcgen05 and the mma.sync attention
    kernels (forward and backward); tc5:<chunk> is the backward's chunked CTA order
    (0: 2-D grid order)."""
    if kernel == "mma":
        knob("ATTN_BWD", "mma")
    if kernel.startswith("tc5:"):
        _, chunk = kernel.split(":")
        knob("ATTN_BWD_CHUNK", chunk)
        kernel = "tc5"
    knob("ATTN_FWD", kernel)  # tc5 also below its 2-tile size threshold
    arch = LONGGQA
    pol = D.Policy(ctx, arch, D.BF16)
    p = params32(arch, 0.3, 10)
    pol.upload(p)
    rng = np.random.default_rng(12)
    prompts, comps = rand_batch(rng, arch, 3, 2, m_range=(2, 20), len_range=(100, 300))
    pol.load_rollout(prompts, 2, comps)
    lp = pol.rollout_log_prob(sum(len(c) for c in comps))
    ref_lp = np.concatenate([O.log_prob(arch, p, prompts[s // 2], comps[s])[1] for s in range(6)])
    assert np.abs(lp - ref_lp).max() <= TOL[D.BF16] * max(1.0, np.abs(ref_lp).max())
    w = rng.standard_normal(6) / 6
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=6)
    got = pol.grad()
    ref = np.zeros_like(got)
    for s in range(6):
        O.grad_log_prob(arch, p, prompts[s // 2], comps[s], w[s], ref)
    assert_grad_close(arch, got, ref, TOL[D.BF16])
    pol.close()


@pytest.mark.parametrize("fwd,bwd,ctxlen", [("tc5", "tc5", 320), ("mma", "mma", 320), ("tc5", "mma", 320),
                                            ("tc5", "tc5", 600)])
def test_pg_gradient_parity_long_sequences_hd128(ctx, knob, fwd, bwd, ctxlen):
    """head_dim 128 (two swizzle atoms per tile) over ragged sequences up to 300 / 580
    tokens: the tcgen05 forward / backward (64-query tiles, transposed dQ; at 600 the key
    tiles with >= 6 query tiles split their heads over two CTAs) against the oracle, and
    the mma.sync kernels."""
    knob("ATTN_FWD", fwd)
    knob("ATTN_BWD", bwd)
    arch = dict(LONGGQA128, context_len=ctxlen)
    pol = D.Policy(ctx, arch, D.BF16)
    p = params32(arch, 0.3, 10)
    pol.upload(p)
    rng = np.random.default_rng(14)
    prompts, comps = rand_batch(rng, arch, 3, 2, m_range=(2, 20), len_range=(100, ctxlen - 20 - 1))
    pol.load_rollout(prompts, 2, comps)
    lp = pol.rollout_log_prob(sum(len(c) for c in comps))
    ref_lp = np.concatenate([O.log_prob(arch, p, prompts[s // 2], comps[s])[1] for s in range(6)])
    assert np.abs(lp - ref_lp).max() <= TOL[D.BF16] * max(1.0, np.abs(ref_lp).max())
    w = rng.standard_normal(6) / 6
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=6)
    got = pol.grad()
    ref = np.zeros_like(got)
    for s in range(6):
        O.grad_log_prob(arch, p, prompts[s // 2], comps[s], w[s], ref)
    assert_grad_close(arch, got, ref, TOL[D.BF16])
    pol.close()


def test_microbatch_invariance_and_filter_equivalence(ctx):
    arch = GQA
    pol = D.Policy(ctx, arch, D.F32)
    pol.upload(params32(arch, 0.3, 9))
    rng = np.random.default_rng(6)
    prompts, comps = rand_batch(rng, arch, 6, 4, len_range=(1, 9))
    pol.load_rollout(prompts, 4, comps)
    r = rng.integers(0, 2, size=24).astype(np.float64)
    pol.set_rewards(r)
    adv, kept, nk = pol.advantage(tau=0.1)
    ra, rk, _ = O.advantage_filter(r, 4, 1, False, 0.0, 0.1)
    assert np.array_equal(adv, ra) and np.array_equal(kept, rk)
    pol.grad_zero()
    pol.accumulate(1.0 / 24, micro_batch=1)
    g1 = pol.grad()
    pol.grad_zero()
    pol.accumulate(1.0 / 24, micro_batch=0)
    g2 = pol.grad()
    pol.grad_zero()
    pol.accumulate_weighted(np.where(kept, adv, 0.0) / 24, micro_batch=7)   # zeroed-A full batch
    g3 = pol.grad()
    assert np.linalg.norm(g1 - g2) <= 1e-5 * np.linalg.norm(g2)
    assert np.linalg.norm(g3 - g2) <= 1e-5 * np.linalg.norm(g2)
    pol.close()


def test_on_policy_violation_and_optimizer(ctx):
    arch = SMALL
    pol = D.Policy(ctx, arch, D.F32)
    p = params32(arch, 0.3, 10)
    pol.upload(p)
    prompts, comps = rand_batch(np.random.default_rng(7), arch, 2, 2, len_range=(1, 5))
    pol.load_rollout(prompts, 2, comps)
    w = np.array([0.5, -0.25, 0.125, 1.0])
    pol.grad_zero()
    pol.accumulate_weighted(w)
    g = pol.grad()
    pol.optimizer_step(D.OPT_ADAM, lr=1e-2)
    got = pol.download()
    ref = p.copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    O.oracle().dor_adam_step(O.ptr(ref, O.f64p), O.ptr(g, O.f64p), O.ptr(m, O.f64p), O.ptr(v, O.f64p), len(p), 1,
                             1e-2, 0.9, 0.999, 1e-8)
    assert np.max(np.abs(got - ref)) <= 1e-6
    with pytest.raises(D.OnPolicyViolation):
        pol.accumulate_weighted(w)
    with pytest.raises(D.InputError):
        pol.load_rollout([[0, 2]], 1, [[0]])          # BOS in completion
    with pytest.raises(D.CapacityError):
        pol.load_rollout([[0, 2]], 1, [[3] * 39])     # m + len > ctx
    pol.close()


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_sharded_step_equals_replicated_update(ctx, dtype):
    """dashcu_sharded_step (ZeRO-1 form) at world 1 == allreduce_grads +
    optimizer_step bit for bit over several Adam steps (slice-sized moments), the bf16
    working copy included (identical rollouts); the two forms cannot be mixed."""
    arch = SMALL
    p = params32(arch, 0.3, 10)
    g = np.random.default_rng(3).standard_normal(len(p)).astype(np.float32).astype(np.float64)
    a, b = D.Policy(ctx, arch, dtype), D.Policy(ctx, arch, dtype)
    for pol in (a, b):
        pol.upload(p)
    for step in range(3):
        for pol in (a, b):
            pol.grad_upload(g * (step + 1))
        a.allreduce_grads()
        a.optimizer_step(D.OPT_ADAM, lr=1e-2)
        b.sharded_step(D.OPT_ADAM, lr=1e-2)
        assert np.array_equal(a.download(), b.download())
    prompts = [[0, 5, 6], [0, 7]]
    ra, rb = a.sample(prompts, 4, 9, round_seed=5), b.sample(prompts, 4, 9, round_seed=5)
    assert np.array_equal(ra.completions, rb.completions) and np.array_equal(ra.lengths, rb.lengths)
    with pytest.raises(D.InputError):
        a.sharded_step(D.OPT_ADAM)
    with pytest.raises(D.InputError):
        b.optimizer_step(D.OPT_ADAM)
    a.close()
    b.close()


# ------------------------------------------------------------ one DASH step

@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_dash_step_c1_matches_oracle(ctx, dtype):
    """Config 1 shape: sample -> rewards -> group advantage + filter -> PG accumulate
    -> Adam, with the gradient checked against the oracle on the GPU's own rollout."""
    arch = C1
    pol = D.Policy(ctx, arch, dtype)
    p = params32(arch, 0.02, 1)
    pol.upload(p)
    M, G, ML = 16, 8, 20
    prompts = [list(O.synthetic_prompt(1, m, 7, 256, 0, 1)) for m in range(M)]
    ro = pol.sample(prompts, G, ML, round_seed=7)
    r = np.array([O.synthetic_reward(3, m, g) for m in range(M) for g in range(G)])
    pol.set_rewards(r)
    adv, kept, nk = pol.advantage(tau=0.1)
    ra, rk, ri = O.advantage_filter(r, G, 1, False, 0.0, 0.1)
    assert np.array_equal(adv, ra) and np.array_equal(kept, rk) and nk == len(ri)
    pol.grad_zero()
    pol.accumulate(1.0 / (M * G), micro_batch=32)
    got = pol.grad()
    ref = np.zeros_like(got)
    for s in ri:
        O.grad_log_prob(arch, p, prompts[s // G], list(ro.completion(s)), adv[s] / (M * G), ref)
    assert_grad_close(arch, got, ref, TOL[dtype])
    st = pol.stats()
    assert st["n_kept"] == nk and st["tokens_sampled"] == int(ro.lengths.sum())
    pol.optimizer_step(D.OPT_ADAM, lr=1e-3)
    assert pol.version() > 0
    pol.close()


@pytest.mark.ref
def test_dash_step_c1_add_task_rewards(ctx):
    """BASELINE configs[0] as specified: ADD prompts from the product's
    generate_instance (byte vocabulary, difficulty 2), 64 prompts x G=8, max_len 57,
    sampled on the GPU, rewarded by the product's task reward == the reference's
    tasks::reward on the same completions, then group advantage + filter."""
    import ctypes as C
    arch = C1
    pol = D.Policy(ctx, arch, D.BF16)
    pol.upload(params32(arch, 0.02, 1))
    M, G, ML = 64, 8, 57
    seeds = [int(O.derive_seed(1, "prompt", m, 0)) for m in range(M)]
    toks, off, answers = D.task_instances(D.TASK_ADD, 2, seeds, D.VOCAB_BYTE)
    assert np.all(np.diff(off) == 7)
    ro = pol.sample(None, G, ML, round_seed=5, prompt_tokens=toks, prompt_offsets=off)
    pol.task_rewards(D.TASK_ADD, 2, seeds, D.VOCAB_BYTE)
    adv, kept, nk = pol.advantage(tau=0.1)
    R = O.ref()
    R.ref_task_reward.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, O.i32p, C.c_int, O.f64p]
    ref_r = np.zeros(M * G)
    for s in range(M * G):
        r = C.c_double(0)
        comp = np.ascontiguousarray(ro.completions[s, :ro.lengths[s]])
        assert R.ref_task_reward(0, 2, 1, seeds[s // G], O.ptr(comp, O.i32p), int(ro.lengths[s]), C.byref(r)) == 0
        ref_r[s] = r.value
    ra, rk, ri = O.advantage_filter(ref_r, G, 1, False, 0.0, 0.1)
    assert np.array_equal(adv, ra) and np.array_equal(kept, rk) and nk == len(ri)
    assert pol.stats()["mean_reward"] == ref_r.mean()
    pol.close()


@pytest.mark.parametrize("arch", [QWENLIKE, VBIG, LONGGQA], ids=["qwenlike", "vbig", "longgqa"])
@pytest.mark.parametrize("temperature", [1.0, 0.7])
def test_backward_reuses_sampler_lse(ctx, knob, arch, temperature):
    """The bf16 backward of a sampled rollout takes each position's T = 1 log-sum-exp
    from the sampling epilogue instead of an LM-head LSE pass (same weights: on-policy).
    Gradient vs the oracle within the bf16 tolerance, and vs the recomputing path."""
    pol = D.Policy(ctx, arch, D.BF16)
    p = params32(arch, 0.5, 21)
    pol.upload(p)
    rng = np.random.default_rng(5)
    V = arch["vocab_size"]
    prompts = [[0] + list(rng.integers(2, V, size=int(rng.integers(3, 9)))) for _ in range(4)]
    G, ML = 4, min(24, arch["context_len"] - 10)
    ro = pol.sample(prompts, G, ML, temperature=temperature, round_seed=9)
    w = rng.standard_normal(len(prompts) * G) / 16
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=8)
    reuse = pol.grad()
    knob("LSE_RECOMPUTE", "1")
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=8)
    recompute = pol.grad()
    ref = np.zeros_like(reuse)
    for s in range(len(w)):
        O.grad_log_prob(arch, p, prompts[s // G], list(ro.completion(s)), w[s], ref)
    assert_grad_close(arch, reuse, ref, TOL[D.BF16])
    assert_grad_close(arch, recompute, ref, TOL[D.BF16])
    assert np.linalg.norm(reuse - recompute) <= 1e-2 * np.linalg.norm(recompute)
    pol.close()


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_long_sequences_multi_tile(ctx, dtype):
    """Sequences spanning several 64-key tiles (flash-attention tiling, causal diagonal,
    ragged tails) through log_prob, the gradient and the decode KV path."""
    arch = LONG
    pol = D.Policy(ctx, arch, dtype)
    p = params32(arch, 0.5, 12)
    pol.upload(p)
    rng = np.random.default_rng(13)
    prompts = [[0] + list(rng.integers(2, 64, size=int(rng.integers(20, 70)))) for _ in range(3)]
    comps = [list(rng.integers(2, 64, size=int(rng.integers(1, 120)))) for _ in range(6)]
    pol.load_rollout(prompts, 2, comps)
    n_tok = sum(len(c) for c in comps)
    lp = pol.rollout_log_prob(n_tok)
    ref = np.concatenate([O.log_prob(arch, p, prompts[s // 2], comps[s])[1] for s in range(6)])
    assert np.abs(lp - ref).max() <= TOL[dtype] * max(1.0, np.abs(ref).max())
    w = rng.standard_normal(6) / 6
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=4)
    got = pol.grad()
    g = np.zeros_like(got)
    for s in range(6):
        O.grad_log_prob(arch, p, prompts[s // 2], comps[s], w[s], g)
    assert_grad_close(arch, got, g, TOL[dtype])
    # decode over long contexts: sampled tokens replay bit-exactly from the logits dump
    pol.set_logits_dump(True)
    ro = pol.sample(prompts, 2, 90, round_seed=4)
    dump = pol.logits_dump(6, 90)
    for s in range(6):
        key = O.derive_seed(4, "sample", s // 2, s % 2)
        for j in range(int(ro.lengths[s])):
            assert O.sample_rule(dump[s, j], 0, 1.0, key, j) == ro.completions[s, j]
    # and the dumped logits match the oracle's forward on a few positions
    for s in (0, 5):
        comp = list(ro.completion(s))
        for j in (0, len(comp) // 2, len(comp) - 1):
            refl = O.next_logits(arch, p, prompts[s // 2] + comp[:j])
            assert np.abs(dump[s, j] - refl).max() <= (1e-3 if dtype == D.F32 else 5e-2) * max(1, np.abs(refl).max())
    pol.close()


def test_decode_wide_ffn(ctx):
    """Decode with a long-K W2 (ffn_hidden 4096, one output tile per row block): tokens
    replay bit-exactly from the logits dump, and the dumped logits match the oracle's
    forward."""
    arch = WIDEFFN
    pol = D.Policy(ctx, arch, D.BF16)
    p = params32(arch, 0.5, 21)
    pol.upload(p)
    rng = np.random.default_rng(22)
    prompts = [[0] + list(rng.integers(2, 64, size=int(rng.integers(3, 12)))) for _ in range(3)]
    pol.set_logits_dump(True)
    ro = pol.sample(prompts, 4, 30, round_seed=5)
    dump = pol.logits_dump(12, 30)
    for s in range(12):
        key = O.derive_seed(5, "sample", s // 4, s % 4)
        for j in range(int(ro.lengths[s])):
            assert O.sample_rule(dump[s, j], 0, 1.0, key, j) == ro.completions[s, j]
    for s in (0, 7, 11):
        comp = list(ro.completion(s))
        for j in (0, len(comp) // 2, max(len(comp) - 1, 0)):
            refl = O.next_logits(arch, p, prompts[s // 4] + comp[:j])
            assert np.abs(dump[s, j] - refl).max() <= 5e-2 * max(1, np.abs(refl).max())
    pol.close()


def eos_heavy_params(arch, seed, boost):
    """Weights whose b_out[eos] is raised so completions end early at random lengths."""
    p = params32(arch, 0.3, seed)
    V = arch["vocab_size"]
    p[-V + arch["eos_id"]] += boost
    return p


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_decode_retirement_and_paged_kv(ctx, knob, dtype):
    """Finished sequences leave the decode batch at every EOS check (row compaction) and
    return their KV pages: tokens, lengths and log-probs equal the run without compaction
    bit for bit, while the decode does measurably less row work (the
    reference stops each sequence at EOS, policy.cpp:425)."""
    arch = dict(QWENLIKE, context_len=200)
    pol = D.Policy(ctx, arch, dtype)
    pol.upload(eos_heavy_params(arch, 31, 1.8))   # P(EOS) ~ 2 % per step
    rng = np.random.default_rng(31)
    prompts = [[0] + list(rng.integers(2, arch["vocab_size"], size=int(rng.integers(3, 9)))) for _ in range(48)]
    G, ML = 4, 190
    a = pol.sample(prompts, G, ML, round_seed=17, temperature=0.9)
    sa = pol.stats()
    knob("DECODE_COMPACT", 0)
    b = pol.sample(prompts, G, ML, round_seed=17, temperature=0.9)
    sb = pol.stats()
    assert np.array_equal(a.completions, b.completions) and np.array_equal(a.lengths, b.lengths)
    assert np.array_equal(a.logp, b.logp)
    mean_len = a.lengths.mean()
    assert 5 < mean_len < 0.5 * ML and a.lengths.max() > 100   # EOS-heavy, but some run long
    assert sa["decode_row_steps"] < 0.75 * sb["decode_row_steps"]
    assert sa["kv_pages_peak"] < sb["kv_pages_peak"]
    # a page budget below the worst case (all 192 x 3 pages) suffices once pages recycle
    knob("DECODE_COMPACT", 1)
    pol.set_kv_pages(sa["kv_pages_peak"])
    c = pol.sample(prompts, G, ML, round_seed=17, temperature=0.9)
    assert np.array_equal(a.completions, c.completions)
    pol.set_kv_pages(sa["kv_pages_peak"] - 1)
    with pytest.raises(D.CapacityError):
        pol.sample(prompts, G, ML, round_seed=17, temperature=0.9)
    pol.set_kv_pages(0)
    pol.close()
