"""Decode retirement at C2 shapes: the sampling phase of 256 prompts x
G = 8 (Qwen2.5-0.5B shape, gen <= 1024) with b_out[eos] raised so completions end at
geometric random lengths, with finished sequences leaving the decode batch at every EOS
check (default) and with DASHCU_DECODE_COMPACT=0 (rows kept until the round ends).
Prints one JSON line per (EOS boost, compaction): mean completion length, decode row-steps
and the sampling time; tokens are identical either way (retirement only drops work)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2505_17218_b200 as D  # noqa: E402
from paper_2505_17218_b200 import workload as W  # noqa: E402


def main():
    M = int(os.environ.get("PROMPTS", "256"))
    G, P, ML = 8, 128, 1024
    arch = W.qwen_arch("0.5b", P + ML)
    V, eos = arch["vocab_size"], arch["eos_id"]
    ctx = D.Context(0)
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(0.02, 1)
    base = pol.download()
    prompts = W.synthetic_prompts(1, 0, M, P, V, 0, 1)
    tok, off = np.ascontiguousarray(prompts.reshape(-1)), (np.arange(M + 1) * P).astype(np.int64)
    # P(EOS) per step ~ e^b / V: mean length ~ V / e^b (capped at 1024)
    for target in [int(a) for a in (sys.argv[1:] or ["1024", "512", "256", "128"])]:
        p = base.copy()
        if target < ML:
            p[-V + eos] += np.log(V / target)
        pol.upload(p)
        ref = None
        for compact in (1, 0):
            D.set_knob("DECODE_COMPACT", compact)
            pol.sample(None, G, ML, prompt_tokens=tok, prompt_offsets=off, round_seed=7)  # warm-up
            ro = pol.sample(None, G, ML, prompt_tokens=tok, prompt_offsets=off, round_seed=7)
            st = pol.stats()
            if ref is None:
                ref = ro.completions.copy()
            else:
                assert np.array_equal(ref, ro.completions), "retirement changed the sampled tokens"
            print(json.dumps({"target_len": target, "compact": compact, "mean_len": float(ro.lengths.mean()),
                              "decode_row_steps": st["decode_row_steps"], "sample_ms": st["sample_ms"],
                              "kv_pages_peak": st["kv_pages_peak"]}), flush=True)
        D.set_knob("DECODE_COMPACT", None)


if __name__ == "__main__":
    main()
