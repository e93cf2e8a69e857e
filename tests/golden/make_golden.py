"""Generate tests/golden/reference_golden.npz from the UNMODIFIED reference compiled in
place (oracle/_ref/libdash_ref.so, built by `make -C oracle`; /root/reference exists only in
the development container). The fixtures pin the C restatement (oracle/dash_oracle.c) on any
machine, including the GPU box where the reference sources are absent:

    python tests/golden/make_golden.py        # rewrites tests/golden/reference_golden.npz

Contents (all produced by the reference's own functions):
  rng_k{0,1,2}       mt19937_64 draws: next_u64 / uniform01 bits / normal bits (rng.hpp:40-82)
  derive             derive_seed(base, tag, a, b) for a few tags (rng.hpp:29-35)
  init_c1_head       first 256 parameters of PolicyParams::init, config-1 arch (tensors.cpp:150-158)
  init_c1_hash       content hash of the full config-1 init (tensors.cpp)
  lp_*               per-token log_prob of prompt/completion pairs (policy.cpp:362-377)
  grad_small         grad_log_prob of one trajectory, small arch (policy.cpp:463-485)
  ntp                next_token_probs after a context (policy.cpp:399-424, T = 1)
  adv_*              group / leave-one-out / single-path advantages, normalize_std, and the
                     |A| > tau filter (advantage.cpp:67-140)
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_ffi as O  # noqa: E402

C1 = dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2, bos_id=0, eos_id=1)
SMALL = dict(vocab_size=37, embed_dim=32, context_len=40, ffn_hidden=48, n_layers=2, bos_id=0, eos_id=1)


def main():
    R = O.ref()
    out = {}
    for kind in (0, 1, 2):
        a = np.zeros(64, dtype=np.uint64)
        R.ref_rng_draws(20250521 + kind, kind, 64, O.ptr(a, O.u64p))
        out[f"rng_k{kind}"] = a
    der = [(0, "sample", 0, 0), (7, "reward", 5, 9), (2**63 + 5, "prompt", 11, 0), (123, "init", 3, 4)]
    out["derive_in"] = np.array([[b, a, c] for b, _, a, c in der], dtype=np.uint64)
    out["derive_tags"] = np.array([t for _, t, _, _ in der])
    out["derive"] = np.array([R.ref_derive_seed(b, t.encode(), a, c) for b, t, a, c in der], dtype=np.uint64)
    p = np.zeros(O.num_params(C1))
    R.ref_init_params(O.arch_ref_vec(C1), 0.02, 1, O.ptr(p, O.f64p))
    out["init_c1_head"] = p[:256].copy()
    h = C.c_uint64(0)
    R.ref_content_hash(O.arch_ref_vec(C1), O.ptr(p, O.f64p), C.byref(h))
    out["init_c1_hash"] = np.array([h.value], dtype=np.uint64)
    # log-probs and a gradient under larger random weights (non-trivial softmax)
    rng = np.random.default_rng(7)
    for name, arch, scale in (("c1", C1, 0.3), ("small", SMALL, 0.5)):
        w = np.zeros(O.num_params(arch))
        R.ref_init_params(O.arch_ref_vec(arch), scale, 11, O.ptr(w, O.f64p))
        V = arch["vocab_size"]
        prompt = np.array([0] + list(rng.integers(2, V, size=5)), dtype=np.int32)
        comp = np.array(list(rng.integers(2, V, size=9)) + [1], dtype=np.int32)
        per = np.zeros(len(comp))
        tot = C.c_double(0)
        R.ref_log_prob(O.arch_ref_vec(arch), O.ptr(w, O.f64p), O.ptr(prompt, O.i32p), len(prompt),
                       O.ptr(comp, O.i32p), len(comp), O.ptr(per, O.f64p), C.byref(tot))
        out[f"lp_{name}_scale"] = np.array([scale])
        out[f"lp_{name}_prompt"] = prompt
        out[f"lp_{name}_comp"] = comp
        out[f"lp_{name}_per"] = per
        if name == "small":
            g = np.zeros(O.num_params(arch))
            R.ref_grad_log_prob(O.arch_ref_vec(arch), O.ptr(w, O.f64p), O.ptr(prompt, O.i32p), len(prompt),
                                O.ptr(comp, O.i32p), len(comp), O.ptr(g, O.f64p))
            out["grad_small"] = g
            probs = np.zeros(V)
            R.ref_next_token_probs(O.arch_ref_vec(arch), O.ptr(w, O.f64p), O.ptr(prompt, O.i32p), len(prompt),
                                   O.ptr(probs, O.f64p))
            out["ntp_small"] = probs
    # advantages and the filter
    r = np.round(rng.random(24), 3) * (rng.random(24) < 0.7)
    r[:6] = 1.0  # a uniform group -> zero advantage
    out["adv_rewards"] = r
    for kind, name in ((0, "single"), (1, "group"), (2, "loo")):
        a = np.zeros(24)
        R.ref_advantage(O.ptr(r, O.f64p), 24, 6, kind, O.ptr(a, O.f64p))
        out[f"adv_{name}"] = a
    a = out["adv_group"].copy()
    na = np.zeros(24)
    R.ref_normalize_std(O.ptr(a, O.f64p), O.ptr(r, O.f64p), 24, 6, 1e-6, O.ptr(na, O.f64p))
    out["adv_group_norm"] = na
    kept = np.zeros(24, dtype=np.uint8)
    nk = C.c_int32(0)
    s1, s2 = C.c_double(0), C.c_double(0)
    R.ref_filter_by_threshold(O.ptr(out["adv_group"], O.f64p), 24, 0.1, O.ptr(kept, O.u8p), C.byref(nk),
                              C.byref(s1), C.byref(s2))
    out["adv_kept_tau0.1"] = kept
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), sorted(out))


if __name__ == "__main__":
    main()
