"""The C restatement (oracle/dash_oracle.c) against golden vectors produced by the
UNMODIFIED reference (tests/golden/make_golden.py ran oracle/_ref, the reference compiled
in place). Runs anywhere, including machines without /root/reference."""
import os

import numpy as np
import pytest

import oracle_ffi as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")
C1 = dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2, bos_id=0, eos_id=1)
SMALL = dict(vocab_size=37, embed_dim=32, context_len=40, ffn_hidden=48, n_layers=2, bos_id=0, eos_id=1)


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def test_rng_and_seed_derivation(g):
    for kind in (0, 1, 2):
        a = np.zeros(64, dtype=np.uint64)
        O.oracle().dor_rng_draws(20250521 + kind, kind, 64, O.ptr(a, O.u64p))
        assert np.array_equal(a, g[f"rng_k{kind}"])
    for (base, a, b), tag, want in zip(g["derive_in"], g["derive_tags"], g["derive"]):
        assert O.derive_seed(int(base), str(tag), int(a), int(b)) == int(want)


def test_init_params(g):
    p = O.init_params(C1, 0.02, 1)
    assert np.array_equal(p[:256], g["init_c1_head"])


@pytest.mark.parametrize("name,arch", [("c1", C1), ("small", SMALL)])
def test_log_prob(g, name, arch):
    w = O.init_params(arch, float(g[f"lp_{name}_scale"][0]), 11)
    _, per = O.log_prob(arch, w, g[f"lp_{name}_prompt"], g[f"lp_{name}_comp"])
    assert np.array_equal(per, g[f"lp_{name}_per"])  # same operation order: bit-exact


def test_grad_log_prob(g):
    w = O.init_params(SMALL, float(g["lp_small_scale"][0]), 11)
    got = O.grad_log_prob(SMALL, w, g["lp_small_prompt"], g["lp_small_comp"])
    ref = g["grad_small"]
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_next_token_probs(g):
    w = O.init_params(SMALL, float(g["lp_small_scale"][0]), 11)
    logits = O.next_logits(SMALL, w, g["lp_small_prompt"])
    x = np.delete(logits, SMALL["bos_id"])
    p = np.exp(x - x.max())
    p /= p.sum()
    want = np.delete(g["ntp_small"], SMALL["bos_id"])
    assert np.abs(p - want).max() <= 1e-12
    assert g["ntp_small"][SMALL["bos_id"]] == 0.0


def test_advantages_and_filter(g):
    r = g["adv_rewards"]
    for kind, name in ((0, "single"), (1, "group"), (2, "loo")):
        adv, _, _ = O.advantage_filter(r, 6 if kind else 24, kind=kind)
        assert np.array_equal(adv, g[f"adv_{name}"])
    adv, _, _ = O.advantage_filter(r, 6, kind=1, normalize=True, eps=1e-6)
    assert np.array_equal(adv, g["adv_group_norm"])
    _, kept, idx = O.advantage_filter(r, 6, kind=1, tau=0.1)
    assert np.array_equal(kept, g["adv_kept_tau0.1"].astype(bool))
    assert np.array_equal(idx, np.flatnonzero(kept))
