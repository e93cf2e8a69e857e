"""Completion-length probe: samples a few prompts of a bench config and prints the length
distribution and the most frequent tokens (random-init policies should run to max_len:
P(EOS) ~ 1/V per step). Usage: python tools/len_probe.py c3 [prompts] [max_len]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B  # noqa: E402
import paper_2505_17218_b200 as D  # noqa: E402
from paper_2505_17218_b200 import workload as W  # noqa: E402

cfg = dict(B.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
M = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ML = int(sys.argv[3]) if len(sys.argv) > 3 else 256
arch = B.arch_of(cfg)
ctx = D.Context(0)
pol = D.Policy(ctx, arch, D.BF16)
pol.init_normal(float(os.environ.get("PROBE_SCALE", cfg.get("init", 0.02))), 1)
P = W.synthetic_prompts(1, 0, M, cfg["prompt_len"], arch["vocab_size"], 0, 1)
poff = (np.arange(M + 1) * cfg["prompt_len"]).astype(np.int64)
for seed in range(2):
    ro = pol.sample(None, cfg["G"], ML, 1.0, round_seed=seed, prompt_index_base=0,
                    prompt_tokens=np.ascontiguousarray(P.reshape(-1).astype(np.int32)), prompt_offsets=poff)
    L = np.asarray(ro.lengths)
    comp = np.asarray(ro.completions)
    toks = np.concatenate([comp[i, :L[i]] for i in range(len(L))])
    u, c = np.unique(toks, return_counts=True)
    top = np.argsort(-c)[:8]
    ended = (L < ML).mean()
    lp = np.asarray(ro.logp)
    print(f"seed {seed}: mean len {L.mean():.1f} min {L.min()} ended {ended:.3f} distinct {len(u)} "
          f"top {[(int(u[i]), int(c[i])) for i in top]} mean logp {np.mean([lp[i, :L[i]].mean() for i in range(len(L)) if L[i]]):.3f}",
          flush=True)
    print("  seq0", comp[0, :min(L[0], 24)].tolist())

# bench-style steps (sample, rewards, filter, accumulate, Adam lr 1e-6): lengths and
# gradient / parameter health per step
if os.environ.get("PROBE_STEPS"):
    N = M * cfg["G"]
    ptok = np.ascontiguousarray(P.reshape(-1).astype(np.int32))
    for i in range(int(os.environ["PROBE_STEPS"])):
        ro = pol.sample(None, cfg["G"], ML, 1.0, round_seed=i, prompt_index_base=0, prompt_tokens=ptok,
                        prompt_offsets=poff)
        pol.set_rewards(W.synthetic_rewards(2 + i, 0, M, cfg["G"]))
        pol.advantage(tau=cfg["tau"])
        pol.grad_zero()
        pol.accumulate(1.0 / N, cfg["micro"])
        g = pol.grad()
        pol.allreduce_grads()
        pol.optimizer_step(D.OPT_ADAM, lr=1e-6)
        p = pol.download()
        L = np.asarray(ro.lengths)
        print(f"step {i}: mean len {L.mean():.1f} ended {(L < ML).mean():.3f} grad finite {np.isfinite(g).all()} "
              f"|g| {np.linalg.norm(np.nan_to_num(g)):.3e} max|g| {np.nanmax(np.abs(g)):.3e} "
              f"params finite {np.isfinite(p).all()}", flush=True)
