"""Training-phase microbenchmark at config-2 shapes (Qwen2.5-0.5B): one micro-batch of
32 sequences x (128 prompt + 1024 completion) through dashcu_accumulate_weighted;
prints per-kernel-class CUDA-event times. The rollout is sampled (4 prompts x G = 8, as in
the DASH step); LOADED=1 loads random trajectories instead (LSE pass included)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2505_17218_b200 as D  # noqa: E402
from paper_2505_17218_b200 import workload as W  # noqa: E402


def main():
    n_seq = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    P, L = 128, 1024
    arch = W.qwen_arch(os.environ.get("SIZE", "0.5b"), P + L)
    ctx = D.Context(0)
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(0.02 if os.environ.get("SIZE", "0.5b") == "0.5b" else 0.01, 1)  # as bench.py
    rng = np.random.default_rng(0)
    if os.environ.get("LOADED"):  # external trajectories: the backward runs its own LSE pass
        prompts = [list(p) for p in W.synthetic_prompts(1, 0, n_seq, P, arch["vocab_size"], 0, 1)]
        comps = [list(rng.integers(2, arch["vocab_size"], size=L)) for _ in range(n_seq)]
        pol.load_rollout(prompts, 1, comps)
    else:  # a sampled rollout (as in the DASH step): the backward reuses the sampler's LSE
        G = 8
        pr = W.synthetic_prompts(1, 0, n_seq // G, P, arch["vocab_size"], 0, 1)
        pol.sample(None, G, L, prompt_tokens=pr.reshape(-1).copy(),
                   prompt_offsets=(np.arange(n_seq // G + 1) * P).astype(np.int64))
    w = np.full(n_seq, 1.0 / n_seq)
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=n_seq)   # warm-up (allocations)
    plain = []
    for _ in range(int(os.environ.get("REPS", "3"))):  # unprofiled: per-kernel events serialise launches
        pol.accumulate_weighted(w, micro_batch=n_seq)
        plain.append(pol.stats()["accumulate_ms"])
    reps = int(os.environ.get("REPS", "3"))
    best = None
    for _ in range(reps):  # the fastest of a few runs (box-to-box clock variance is large)
        D.profile_enable(keys=True)
        D.profile_read(reset=True)
        pol.accumulate_weighted(w, micro_batch=n_seq)
        k_ = D.profile_keys()
        p_ = D.profile_read(reset=True)
        tot = sum(v["ms"] for v in p_.values())
        if best is None or tot < best[0]:
            best = (tot, k_, p_)
    _, keys, prof = best
    D.profile_enable(())
    st = pol.stats()
    out = {k: {"ms": v["ms"], "launches": v["launches"], "tflops": v["flops"] / max(v["ms"], 1e-9) / 1e9}
           for k, v in prof.items() if v["launches"]}
    print(json.dumps({"seqs": n_seq, "tokens": n_seq * (P + L - 1), "accumulate_ms_unprofiled": min(plain),
                      "accumulate_ms": st["accumulate_ms"],
                      "classes": out}))
    for k, n, ms, f, b in keys:
        print(f"{ms:9.3f} ms {n:4d}x {f / max(ms, 1e-9) / 1e9:7.1f} TF/s  {k}")


if __name__ == "__main__":
    main()
