"""Parity at the BENCHMARKED shapes (VERDICT r1 "what's weak" 1-2).

The small-geometry tests in test_gpu_parity.py never reach the code paths the C2-C4
bench runs: a 151,936-id vocabulary (149 sampling slices per scan lane, the 16,384-row
LM-head chunks), 24-28 layers, 128 + 1,024-token sequences (9 attention key tiles), the
true Qwen2.5-0.5B width. These tests run the production bf16 path there:

  * sampled tokens bit-exact under the logits dump through the fused LM-head sampler
    (DESIGN.md §4 rule restated in oracle/dash_oracle.c dor_sample_rule);
  * the backward that REUSES the sampler's log-sum-exp (policy.cu accumulate) within the
    bf16 tolerance (2e-2 per tensor) of the fp64 oracle, and within 1e-2 of the
    recomputing path at full depth and full generation length;
  * the sampler's recorded log-probs against the teacher-forced ones (decode path vs
    forward path, SURVEY App.B D12);
  * device counter init == the oracle's restatement bit for bit, SGD == add_scaled.

Model width d / ffn H are reduced where the fp64 oracle must run over many tokens
(it is scalar CPU code); vocabulary, depth, head geometry and lengths are the bench's.
The oracle runs one thread per sequence (ctypes releases the GIL).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle_ffi as O
import paper_2505_17218_b200 as D
from test_gpu_parity import assert_grad_close, tensor_slices

pytestmark = pytest.mark.gpu

V_QWEN = 151936
# Qwen2.5-0.5B depth / heads / vocabulary at reduced width (oracle-feasible)
DEEP64 = dict(vocab_size=V_QWEN, embed_dim=128, context_len=1152, ffn_hidden=256, n_layers=24, bos_id=0,
              eos_id=1, n_heads=14, n_kv_heads=2, head_dim=64)
# Qwen2.5-1.5B depth / heads (head_dim 128)
DEEP128 = dict(vocab_size=V_QWEN, embed_dim=128, context_len=1152, ffn_hidden=256, n_layers=28, bos_id=0,
               eos_id=1, n_heads=12, n_kv_heads=2, head_dim=128)
# the true Qwen2.5-0.5B width (d 896, ffn 4864) at 2 layers
WIDE = dict(vocab_size=V_QWEN, embed_dim=896, context_len=1152, ffn_hidden=4864, n_layers=2, bos_id=0, eos_id=1,
            n_heads=14, n_kv_heads=2, head_dim=64)


@pytest.fixture(scope="module")
def ctx():
    return D.Context(0)


def make_policy(ctx, arch, scale, seed):
    """Device counter init (what the bench uses), fp32 master downloaded for the oracle."""
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(scale, seed)
    return pol, pol.download()


def prompts_for(arch, n, length, seed):
    rng = np.random.default_rng(seed)
    return [[arch["bos_id"]] + list(rng.integers(2, arch["vocab_size"], size=length - 1)) for _ in range(n)]


def check_tokens(pol, ro, prompts, G, ML, seed, inv_t, bos):
    dump = pol.logits_dump(len(prompts) * G, ML)
    checked = 0
    for s in range(len(prompts) * G):
        key = O.derive_seed(seed, "sample", s // G, s % G)
        for j in range(int(ro.lengths[s])):
            assert O.sample_rule(dump[s, j], bos, inv_t, key, j) == ro.completions[s, j], (s, j)
            checked += 1
    return dump, checked


def oracle_grad(arch, p, prompts, comps, w, G):
    def one(s):
        g = np.zeros(len(p))
        O.grad_log_prob(arch, p, prompts[s // G], comps[s], w[s], g)
        return g
    with ThreadPoolExecutor(max_workers=min(16, len(comps))) as ex:
        return sum(ex.map(one, range(len(comps))))


def test_init_normal_ctr_matches_oracle(ctx):
    """dashcu_policy_init_normal (the bench's C2-C4 init) == dor_init_params_ctr."""
    for arch in (dict(DEEP64, n_layers=2), WIDE):
        pol = D.Policy(ctx, arch, D.F32)
        pol.init_normal(0.02, 7)
        got = pol.download().astype(np.float32)
        ref = O.init_params_ctr(arch, 0.02, 7).astype(np.float32)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
        pol.close()


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_sgd_equals_add_scaled(ctx, dtype):
    """optimizer_step(SGD) == ParamTensors::add_scaled(grad, lr) (tensors.cpp:109-115)
    to fp32 rounding, at the 2-layer Qwen width."""
    arch = WIDE
    pol = D.Policy(ctx, arch, dtype)
    pol.init_normal(0.02, 3)
    p = pol.download()
    g = np.random.default_rng(4).standard_normal(len(p)).astype(np.float32).astype(np.float64)
    pol.grad_upload(g)
    pol.optimizer_step(D.OPT_SGD, lr=1e-3)
    got = pol.download()
    ref = p + 1e-3 * g
    assert np.max(np.abs(got - ref)) <= 2 * np.finfo(np.float32).eps * np.max(np.abs(ref))
    pol.close()


@pytest.mark.parametrize("arch", [DEEP64, DEEP128], ids=["24L-14/2x64", "28L-12/2x128"])
def test_sampler_full_length_qwen_vocab(ctx, arch):
    """Prompt 128 + up to 1024 sampled tokens, V = 151,936, bench depth: every token
    bit-exact under the logits dump; the sampler's T = 1 log-probs vs the teacher-forced
    ones; the LSE-reusing backward vs the recomputing one at full length."""
    pol, _ = make_policy(ctx, arch, 0.02, 11)
    prompts = prompts_for(arch, 2, 128, 3)
    G, ML, T = 2, 1024, 1.0
    pol.set_logits_dump(True)
    ro = pol.sample(prompts, G, ML, temperature=T, round_seed=13)
    _, checked = check_tokens(pol, ro, prompts, G, ML, 13, 1.0, arch["bos_id"])
    assert checked >= 2 * G * 900
    assert pol.stats()["slice_recompute_mismatches"] == 0   # recomputed slices == the GEMM's logits
    pol.set_logits_dump(False)
    # decode-path log-probs vs the teacher-forced forward on the same sequences
    ro = pol.sample(prompts, G, ML, temperature=T, round_seed=13)
    n_tok = int(ro.lengths.sum())
    tf = pol.rollout_log_prob(n_tok)
    dec = np.concatenate([ro.logp[s, :ro.lengths[s]] for s in range(len(prompts) * G)])
    gap = np.abs(tf - dec)
    assert gap.max() <= 2e-2 * max(1.0, np.abs(tf).max()), gap.max()
    # LSE reuse (sampler LSE + teacher-forced logits) vs recompute at full length / depth
    w = np.random.default_rng(5).standard_normal(len(prompts) * G) / 8
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=4)
    reuse = pol.grad()
    D.set_knob("LSE_RECOMPUTE", 1)
    try:
        pol.grad_zero()
        pol.accumulate_weighted(w, micro_batch=4)
        rec = pol.grad()
    finally:
        D.set_knob("LSE_RECOMPUTE", None)
    assert_grad_close(arch, reuse, rec, 1e-2)
    pol.close()


@pytest.mark.parametrize("arch", [DEEP64, DEEP128], ids=["24L-14/2x64", "28L-12/2x128"])
def test_lse_reuse_backward_vs_oracle_deep(ctx, arch):
    """The bench's backward (sampler LSE reused) at full depth and vocabulary against the
    fp64 oracle's grad_log_prob (policy.cpp:463-485), per tensor within 2e-2."""
    pol, p = make_policy(ctx, arch, 0.02, 17)
    prompts = prompts_for(arch, 2, 32, 4)
    G, ML = 2, 96
    ro = pol.sample(prompts, G, ML, round_seed=21)
    comps = [list(ro.completion(s)) for s in range(len(prompts) * G)]
    w = np.random.default_rng(6).standard_normal(len(comps)) / 4
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=4)
    got = pol.grad()
    ref = oracle_grad(arch, p, prompts, comps, w, G)
    # every tensor within 2e-2, the attention q / k projections of the top layers included:
    # at random init their gradient is ~1e-6 of the total and comes out of dP_ij - D_i, a
    # small difference; the forward's normaliser over the bf16-rounded P and the O residual
    # kept for D make that difference exact up to fp32 (attn_fwd_tc; 16 % -> 1.4 % at 24 layers)
    assert_grad_close(arch, got, ref, 2e-2)
    # and the teacher-forced log-probs vs the oracle
    lp = pol.rollout_log_prob(int(ro.lengths.sum()))
    ref_lp = np.concatenate([O.log_prob(arch, p, prompts[s // G], comps[s])[1] for s in range(len(comps))])
    assert np.abs(lp - ref_lp).max() <= 2e-2 * max(1.0, np.abs(ref_lp).max())
    pol.close()


def test_true_c2_width(ctx):
    """d 896 / ffn 4864 / V 151,936 / 14-2 x 64 heads (BASELINE configs[1] widths) at 2
    layers: tokens bit-exact under the dump at T = 0.7, gradient of the sampled rollout
    (sampler LSE reused) vs the fp64 oracle within 2e-2 per tensor."""
    arch = WIDE
    pol, p = make_policy(ctx, arch, 0.02, 5)
    prompts = prompts_for(arch, 2, 16, 7)
    G, ML, T = 2, 32, 0.7
    pol.set_logits_dump(True)
    ro = pol.sample(prompts, G, ML, temperature=T, round_seed=3)
    check_tokens(pol, ro, prompts, G, ML, 3, float(np.float32(1.0 / T)), arch["bos_id"])
    assert pol.stats()["slice_recompute_mismatches"] == 0
    pol.set_logits_dump(False)
    ro = pol.sample(prompts, G, ML, temperature=1.0, round_seed=3)
    comps = [list(ro.completion(s)) for s in range(len(prompts) * G)]
    w = np.random.default_rng(8).standard_normal(len(comps)) / 4
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=4)
    got = pol.grad()
    ref = oracle_grad(arch, p, prompts, comps, w, G)
    assert_grad_close(arch, got, ref, 2e-2)
    pol.close()
