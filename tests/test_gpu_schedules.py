"""PPO surrogate, KL term, update schedules and interleaved sampling through the C ABI
(policy.cpp:487-522), against the
CPU oracle (oracle/dash_oracle.c, pinned to the reference's kl_term / grad_log_prob in
test_oracle.py) and against the DASH path itself where the SPEC states an identity:

  * PPO at theta == theta_old equals the PG gradient exactly;
  * items on the clipped branch contribute nothing;
  * MULTI with K = 1 equals DASH; MINI with K = 2 performs two updates on
    disjoint halves;
  * the KL gradient / value match the oracle, kl(params, params) = 0, beta = 0 is the
    No-KL update;
  * 32 interleaved micro-batch calls reproduce one preemptive call.
"""
import numpy as np
import pytest

import oracle_ffi as O
import paper_2505_17218_b200 as D
from test_gpu_parity import GQA, QWENLIKE, TOL, assert_grad_close, params32, rand_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return D.Context(0)


def rollout(pol, arch, M=6, G=4, ML=10, seed=3):
    rng = np.random.default_rng(seed)
    prompts = [[0] + list(rng.integers(2, arch["vocab_size"], size=int(rng.integers(2, 6)))) for _ in range(M)]
    ro = pol.sample(prompts, G, ML, round_seed=seed)
    r = rng.integers(0, 2, size=M * G).astype(np.float64)
    pol.set_rewards(r)
    adv, kept, nk = pol.advantage(tau=0.1)
    return prompts, ro, adv, kept


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_ppo_at_entry_equals_pg(ctx, knob, dtype):
    arch = QWENLIKE
    pol = D.Policy(ctx, arch, dtype)
    pol.upload(params32(arch, 0.3, 4))
    prompts, ro, adv, kept = rollout(pol, arch)
    N = len(adv)
    knob("LSE_RECOMPUTE", 1)   # the PG side takes the same LSE pass as PPO's pass 1
    pol.grad_zero()
    pol.accumulate(1.0 / N, micro_batch=5)
    g_pg = pol.grad()
    pol.snapshot()
    pol.grad_zero()
    sur, nclip = pol.accumulate_ppo(1.0 / N, clip_eps=0.2, micro_batch=5)   # same partition: same sums
    g_ppo = pol.grad()
    assert nclip == 0
    # rho == 1 exactly, so the row weights equal the PG ones; the gradients then differ only
    # by the attention backward's order-dependent fp32 reduce-adds (dQ / dK / dV)
    assert np.linalg.norm(g_pg - g_ppo) <= 1e-6 * np.linalg.norm(g_pg)
    assert abs(sur - adv[kept].sum() / N) <= 1e-12 * max(1.0, np.abs(adv).sum())
    pol.close()


def test_ppo_off_policy_vs_oracle(ctx):
    """After an update, rho != 1: gradient = sum_n A_n rho_n grad log pi on the unclipped
    branch and 0 on the clipped one, against the oracle's fp64 restatement (F32 path)."""
    arch = GQA
    pol = D.Policy(ctx, arch, D.F32)
    p_old = params32(arch, 0.3, 6)
    pol.upload(p_old)
    prompts, ro, adv, kept = rollout(pol, arch, M=8, G=4, ML=8, seed=5)
    N = len(adv)
    comps = [list(ro.completion(s)) for s in range(N)]
    pol.snapshot()
    old = pol.snapshot_logp()
    ref_old = np.array([O.log_prob(arch, p_old, prompts[s // 4], comps[s])[0] for s in range(N)])
    assert np.abs(old - ref_old).max() <= 1e-3 * max(1.0, np.abs(ref_old).max())
    g = np.random.default_rng(2).standard_normal(len(p_old))
    pol.grad_upload(g)
    pol.optimizer_step(D.OPT_SGD, lr=0.01)   # move theta away from theta_old
    p_new = pol.download()
    ks = np.flatnonzero(kept)
    rho = {s: np.exp(O.log_prob(arch, p_new, prompts[s // 4], comps[s])[0] - ref_old[s]) for s in ks}
    # clip range in the widest gap of |rho - 1| around its median, so that items fall on
    # both branches and none sits within rounding of the boundary
    dev = np.sort([abs(r - 1) for r in rho.values()])
    k = int(np.argmax(np.diff(dev)[len(dev) // 4:3 * len(dev) // 4])) + len(dev) // 4
    eps = 0.5 * (dev[k] + dev[k + 1])
    assert dev[k + 1] - dev[k] > 1e-4
    pol.grad_zero()
    sur, nclip = pol.accumulate_ppo(1.0 / N, clip_eps=eps, micro_batch=5)
    got = pol.grad()
    ref = np.zeros_like(got)
    n_ref_clip = 0
    for s in ks:
        a = adv[s]
        clipped = (a > 0 and rho[s] > 1 + eps) or (a < 0 and rho[s] < 1 - eps)
        n_ref_clip += clipped
        if not clipped:
            O.grad_log_prob(arch, p_new, prompts[s // 4], comps[s], a * rho[s] / N, ref)
    assert nclip == n_ref_clip and 0 < nclip < kept.sum(), (nclip, n_ref_clip, int(kept.sum()))
    assert_grad_close(arch, got, ref, TOL[D.F32])
    pol.close()


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_kl_term_vs_oracle(ctx, dtype):
    arch = QWENLIKE
    base = D.Policy(ctx, arch, dtype)
    pol = D.Policy(ctx, arch, dtype)
    pb = params32(arch, 0.3, 7)
    pc = (pb + 0.01 * np.random.default_rng(3).standard_normal(len(pb))).astype(np.float32).astype(np.float64)
    base.upload(pb)
    pol.upload(pc)
    prompts, comps = rand_batch(np.random.default_rng(8), arch, 3, 3, len_range=(1, 9))
    pol.load_rollout(prompts, 3, comps)
    pol.grad_zero()
    kl = pol.accumulate_kl(base, 0.5, micro_batch=4)
    got = pol.grad()
    ref = np.zeros_like(got)
    ref_kl = np.array([O.kl_term(arch, pc, pb, prompts[s // 3], comps[s], 0.5, ref)[0] for s in range(9)])
    assert np.abs(kl - ref_kl).max() <= TOL[dtype] * np.abs(ref_kl).max(), (kl, ref_kl)
    assert_grad_close(arch, got, ref, TOL[dtype])
    # kl(params, params) = (0, 0)
    pol.upload(pb)
    pol.load_rollout(prompts, 3, comps)
    pol.grad_zero()
    kl0 = pol.accumulate_kl(base, 1.0, micro_batch=4)
    assert np.abs(kl0).max() <= 1e-6 and np.abs(pol.grad()).max() <= 1e-6
    pol.close()
    base.close()


def test_schedules(ctx, knob):
    arch = GQA
    knob("LSE_RECOMPUTE", 1)
    p0 = params32(arch, 0.3, 9)
    pols = [D.Policy(ctx, arch, D.F32) for _ in range(3)]
    for p in pols:
        p.upload(p0)
    outs = []
    for p in pols:
        outs.append(rollout(p, arch, M=4, G=4, ML=8, seed=11))
    N = 16
    # SGD updates: Adam maps a near-zero gradient element to ~±lr whatever its size, so the
    # attention backward's order-dependent fp32 reduce-adds (~1e-7 relative) could flip it
    sgd = dict(opt_kind=D.OPT_SGD, lr=1e-2)
    # DASH vs MULTI K=1: the same update
    l_dash = pols[0].run_schedule(D.SCHED_DASH, weight_scale=1.0 / N, **sgd)
    l_multi = pols[1].run_schedule(D.SCHED_MULTI, K=1, weight_scale=1.0 / N, **sgd)
    assert len(l_dash) == 1 and len(l_multi) == 1
    # (equal up to the attention backward's order-dependent fp32 reduce-adds)
    assert np.abs(pols[0].download() - pols[1].download()).max() <= 1e-5
    # MINI K=2: two updates on disjoint halves (sequences 0-7, 8-15), each the PPO gradient of
    # its half against the entry snapshot, equal to doing it by hand
    l_mini = pols[2].run_schedule(D.SCHED_MINI, K=2, weight_scale=1.0 / N, **sgd)
    assert len(l_mini) == 2
    kept = outs[2][3]
    assert [l["n_items"] for l in l_mini] == [int(kept[:8].sum()), int(kept[8:].sum())]
    hand = D.Policy(ctx, arch, D.F32)
    hand.upload(p0)
    rollout(hand, arch, M=4, G=4, ML=8, seed=11)
    hand.snapshot()
    for k in range(2):
        hand.grad_zero()
        hand.accumulate_ppo(2.0 / N, 0.2, 32, subset=np.arange(8 * k, 8 * k + 8))
        hand.optimizer_step(D.OPT_SGD, lr=1e-2)
    assert np.abs(hand.download() - pols[2].download()).max() <= 1e-5
    with pytest.raises(D.InputError):
        pols[2].run_schedule(D.SCHED_MINI, K=3, weight_scale=1.0 / N)   # 16 % 3 != 0
    with pytest.raises(D.OnPolicyViolation):
        pols[2].run_schedule(D.SCHED_MULTI, K=2, weight_scale=1.0 / N)  # theta moved since sampling
    for p in pols + [hand]:
        p.close()


def test_schedule_with_kl(ctx, knob):
    """beta > 0 adds -beta * grad KL(base || current) over the same items; beta = 0 is DASH."""
    arch = GQA
    knob("LSE_RECOMPUTE", 1)
    p0 = params32(arch, 0.3, 12)
    base = D.Policy(ctx, arch, D.F32)
    base.upload((p0 + 0.02 * np.random.default_rng(1).standard_normal(len(p0))).astype(np.float32))
    a, b = D.Policy(ctx, arch, D.F32), D.Policy(ctx, arch, D.F32)
    for p in (a, b):
        p.upload(p0)
    ra, rb = rollout(a, arch, seed=13), rollout(b, arch, seed=13)
    N = 24
    a.run_schedule(D.SCHED_DASH, weight_scale=1.0 / N, beta=0.04, base=base, opt_kind=D.OPT_SGD, lr=1.0)
    # by hand: PG + (-0.04) * KL gradient over the kept items, then SGD with lr 1
    kept_idx = np.flatnonzero(rb[3])
    b.grad_zero()
    b.accumulate(1.0 / N, micro_batch=32)
    b.accumulate_kl(base, -0.04 / N, micro_batch=32, subset=kept_idx)
    b.optimizer_step(D.OPT_SGD, lr=1.0)
    assert np.abs(a.download() - b.download()).max() <= 1e-6
    for p in (a, b, base):
        p.close()


def test_interleaved_calls_cover_the_preemptive_round(ctx):
    """interleaved_sample: 32 calls of 2 prompts x G (prompt_index_base =
    the micro-batch's first global prompt) == one preemptive call of 64 prompts x G."""
    arch = QWENLIKE
    pol = D.Policy(ctx, arch, D.BF16)
    pol.upload(params32(arch, 0.3, 14))
    rng = np.random.default_rng(15)
    prompts = [[0] + list(rng.integers(2, arch["vocab_size"], size=5)) for _ in range(64)]
    G = 4
    full = pol.sample(prompts, G, 16, round_seed=21)
    parts = [pol.sample(prompts[2 * i:2 * i + 2], G, 16, round_seed=21, prompt_index_base=2 * i) for i in range(32)]
    assert np.array_equal(full.completions, np.concatenate([p.completions for p in parts]))
    assert np.array_equal(full.lengths, np.concatenate([p.lengths for p in parts]))
    assert sum(int(p.lengths.sum()) for p in parts) == int(full.lengths.sum())
    pol.close()


# ------------------------------------------------------------- checkpoint container

def read_ckpt(path):
    """Independent reader of the DASHCKPT layout documented in include/dashcu.h."""
    import struct
    b = open(path, "rb").read()
    assert b[:8] == b"DASHCKPT"
    ver, = struct.unpack_from("<I", b, 8)
    arch = struct.unpack_from("<10i", b, 12)
    nt, flags, t, h = struct.unpack_from("<IIqQ", b, 52)
    off = 76
    tensors = []
    for _ in range(nt):
        nl, = struct.unpack_from("<H", b, off)
        name = b[off + 2:off + 2 + nl].decode()
        off += 2 + nl
        nd = b[off]
        dims = struct.unpack_from(f"<{nd}Q", b, off + 1)
        off += 1 + 8 * nd
        cnt = int(np.prod(dims)) if nd else 1
        tensors.append((name, dims, np.frombuffer(b, dtype="<f8", count=cnt, offset=off)))
        off += 8 * cnt
    assert off == len(b)
    return ver, arch, flags, t, h, tensors


@pytest.mark.parametrize("arch", [dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2,
                                       bos_id=0, eos_id=1), GQA], ids=["c1", "gqa"])
def test_checkpoint_round_trip(ctx, tmp_path, arch):
    """save -> load reproduces sampling and the Adam continuation bit for bit;
    the file holds the views() names / shapes and the reference's content_hash."""
    import ctypes as C
    a = D.Policy(ctx, arch, D.BF16)
    a.upload(params32(arch, 0.3, 21))
    g = np.random.default_rng(4).standard_normal(a.n_params)
    a.grad_upload(g)
    a.optimizer_step(D.OPT_ADAM, lr=1e-3)
    path = str(tmp_path / "p.ckpt")
    a.save(path)
    ver, harch, flags, t, h, tensors = read_ckpt(path)
    assert ver == 1 and flags == 1 and t == 1 and D.checkpoint_arch(path)["vocab_size"] == arch["vocab_size"]
    flat = np.concatenate([x for name, _, x in tensors if not name.startswith("adam.")])
    assert np.array_equal(flat, a.download())
    assert [n for n, _, _ in tensors][:3] == ["token_embed", "pos_embed", "layers.0.wq"]
    if "n_heads" not in arch:   # reference geometry: the reference's own content_hash
        out = C.c_uint64(0)
        O.ref().ref_content_hash(O.arch_ref_vec(arch), O.ptr(np.ascontiguousarray(flat), O.f64p), C.byref(out))
        assert out.value == h
    b = D.Policy(ctx, arch, D.BF16)
    b.load(path)
    assert np.array_equal(a.download(), b.download())
    prompts = [[0, 5, 6], [0, 7, 8, 9]]
    ra, rb = a.sample(prompts, 4, 12, round_seed=3), b.sample(prompts, 4, 12, round_seed=3)
    assert np.array_equal(ra.completions, rb.completions) and np.array_equal(ra.logp, rb.logp)
    for p in (a, b):
        p.grad_upload(g * 0.5)
        p.optimizer_step(D.OPT_ADAM, lr=1e-3)
    assert np.array_equal(a.download(), b.download())
    bad = str(tmp_path / "bad.ckpt")
    raw = bytearray(open(path, "rb").read())
    raw[300] ^= 1   # inside token_embed: caught by the content hash
    open(bad, "wb").write(raw)
    with pytest.raises(D.InputError):
        b.load(bad)
    other = dict(arch, n_layers=arch["n_layers"] + 1)
    c = D.Policy(ctx, other, D.BF16)
    with pytest.raises(D.InputError):
        c.load(path)
    for p in (a, b, c):
        p.close()


# ------------------------------------------------ fused reduce-scatter / update / all-gather

def adam_fp32(w, g, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    f = np.float32
    m = f(b1) * m + f(1 - b1) * g
    v = f(b2) * v + f(1 - b2) * g * g
    c1, c2 = f(1 - b1 ** t), f(1 - b2 ** t)
    return w + f(lr) * (m / c1) / (np.sqrt(v / c2) + f(eps)), m, v


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_fused_step_virtual_ranks(ctx, world):
    """dashcu_fused_step's kernel as `world` concurrent virtual ranks on one GPU (their own
    gradient / master / bf16 / flag buffers, the same peer-pointer arrays NVLink ranks get):
    every replica ends with the same master weights = Adam over the rank-order gradient sum
    (three steps, slice-sized moments, the entry / exit barriers each step), and the bf16
    copies are their rounding."""
    n = 100003   # slices of ceil(n / world) rounded up to 64, the last one short
    rng = np.random.default_rng(world)
    g = rng.standard_normal((world, n)).astype(np.float32)
    w0 = rng.standard_normal(n).astype(np.float32)
    wo, wt = ctx.selftest_fused_step(g, w0, D.OPT_ADAM, 1e-3, steps=3)
    for r in range(1, world):
        assert np.array_equal(wo[r].view(np.uint32), wo[0].view(np.uint32))
    gs = g[0].copy()
    for r in range(1, world):
        gs = gs + g[r]
    w, m, v = w0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    for t in (1, 2, 3):   # the same gradient each step
        w, m, v = adam_fp32(w, gs, m, v, t, 1e-3)
    assert np.max(np.abs(wo[0] - w)) <= 1e-6
    from test_gpu_gemm import bf16_bits
    assert np.array_equal(wt[0], bf16_bits(wo[0]))
    wo, _ = ctx.selftest_fused_step(g, w0, D.OPT_SGD, 1e-2, steps=1)
    assert np.max(np.abs(wo[world - 1] - (w0 + np.float32(1e-2) * gs))) <= 1e-6


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_fused_step_world1_equals_sharded(ctx, dtype):
    """At world 1 dashcu_fused_step runs its kernel on the local buffers: bit-identical to
    dashcu_sharded_step over several Adam steps (same slice moments), rollouts included."""
    arch = GQA
    p = params32(arch, 0.3, 10)
    g = np.random.default_rng(3).standard_normal(len(p)).astype(np.float32).astype(np.float64)
    a, b = D.Policy(ctx, arch, dtype), D.Policy(ctx, arch, dtype)
    for pol in (a, b):
        pol.upload(p)
    for step in range(3):
        for pol in (a, b):
            pol.grad_upload(g * (step + 1))
        a.sharded_step(D.OPT_ADAM, lr=1e-2)
        b.fused_step(D.OPT_ADAM, lr=1e-2)
        assert np.array_equal(a.download(), b.download())
    ra, rb = a.sample([[0, 5, 6]], 4, 9, round_seed=5), b.sample([[0, 5, 6]], 4, 9, round_seed=5)
    assert np.array_equal(ra.completions, rb.completions)
    a.close()
    b.close()
