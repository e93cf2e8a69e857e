"""Accumulate-phase probe: a sampled C2-shaped rollout (prompts x 8, gen 1024), then
dashcu_accumulate_weighted over all sequences in micro-batches of 32, timed by the
library's event timer and by wall clock, with the sampler-LSE reuse on and off.
Runs against whichever package is first on sys.path (A/B against ab/<old>/)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2505_17218_b200 as D  # noqa: E402
from paper_2505_17218_b200 import workload as W  # noqa: E402

prompts = int(sys.argv[1]) if len(sys.argv) > 1 else 32
arch = W.qwen_arch("0.5b", 1152)
ctx = D.Context(0)
pol = D.Policy(ctx, arch, D.BF16)
pol.init_normal(0.02, 1)
pr = W.synthetic_prompts(1, 0, prompts, 128, arch["vocab_size"], 0, 1)
pol.sample(None, 8, 1024, prompt_tokens=pr.reshape(-1).copy(), prompt_offsets=(np.arange(prompts + 1) * 128).astype(np.int64))
w = np.full(prompts * 8, 1.0 / (prompts * 8))


def setk(v):
    if hasattr(D, "set_knob"):
        D.set_knob("LSE_RECOMPUTE", v)
    else:
        os.environ["DASHCU_LSE_RECOMPUTE"] = str(v)


if os.environ.get("NCU"):  # one accumulate inside cudaProfilerStart/Stop (ncu --profile-from-start off)
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=32)
    ctx.sync()
    rt.cudaProfilerStart()
    pol.accumulate_weighted(w, micro_batch=32)
    ctx.sync()
    rt.cudaProfilerStop()
    sys.exit(0)
for rec in (0, 1):
    setk(rec)
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=32)
    ev, wall = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        pol.accumulate_weighted(w, micro_batch=32)
        ctx.sync()
        wall.append((time.perf_counter() - t0) * 1e3)
        ev.append(pol.stats()["accumulate_ms"])
    print(f"recompute={rec} seqs={prompts * 8} event_ms={min(ev):.1f} wall_ms={min(wall):.1f} per_mb={min(ev) / (prompts * 8 / 32):.2f}")
