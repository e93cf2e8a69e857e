"""Decode-phase microbenchmark at config-2 shapes (Qwen2.5-0.5B, 512 prompts x G=8):
a short sample call; prints per-kernel-class CUDA-event times per decode step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2505_17218_b200 as D  # noqa: E402
from paper_2505_17218_b200 import workload as W  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    M, G, P = int(os.environ.get("PROMPTS", "512")), 8, 128
    arch = W.qwen_arch(os.environ.get("SIZE", "0.5b"), P + 1024)
    ctx = D.Context(0)
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(0.02 if os.environ.get("SIZE", "0.5b") == "0.5b" else 0.01, 1)  # as bench.py
    prompts = W.synthetic_prompts(1, 0, M, P, arch["vocab_size"], 0, 1)
    tok, off = np.ascontiguousarray(prompts.reshape(-1)), (np.arange(M + 1) * P).astype(np.int64)
    pol.sample(None, G, steps, prompt_tokens=tok, prompt_offsets=off)     # warm-up
    pol.sample(None, G, steps, prompt_tokens=tok, prompt_offsets=off)     # unprofiled (per-kernel events
    plain_ms = pol.stats()["sample_ms"]                                   # would serialise the launches)
    D.profile_enable(keys=True)
    D.profile_read(reset=True)
    pol.sample(None, G, steps, prompt_tokens=tok, prompt_offsets=off)
    keys = D.profile_keys()
    prof = D.profile_read(reset=True)
    D.profile_enable(())
    st = pol.stats()
    out = {k: {"ms": v["ms"], "launches": v["launches"],
               "tflops": v["flops"] / max(v["ms"], 1e-9) / 1e9, "gbs": v["bytes"] / max(v["ms"], 1e-9) / 1e6}
           for k, v in prof.items() if v["launches"]}
    print(json.dumps({"decode_steps": steps, "sample_ms_unprofiled": plain_ms, "sample_ms": st["sample_ms"],
                      "classes": out}))
    for k, n, ms, f, b in keys:
        print(f"{ms:9.3f} ms {n:4d}x {f / max(ms, 1e-9) / 1e9:7.1f} TF/s  {k}")


if __name__ == "__main__":
    main()
