"""BASELINE configs[4] on one B200: DASH vs GRPO-style step-time sweep over the
preemptive batch size (prompts sampled per step) and the gradient-filter threshold.

    python tools/sweep_c5.py [--max-len 1024] [--prompts 4,64,256,512] [--taus off,0,0.1,0.3]

Every point runs the full step of bench.py (sample -> synthetic rewards -> group
advantage + |A| filter -> micro-batched PG accumulate -> Adam) on the Qwen2.5-0.5B shape,
one warm-up step then one timed step, device-timed by the library's phase timers.
"GRPO-style" is the small sampling batch (4 prompts x G = 8 = 32 sequences, one
micro-batch) without the filter (every sequence, including the zero-advantage ones of
uniform groups, goes through the backward). Prints one JSON line per point and a table.

--interleaved M1,M2,..: the SPEC's GRPO baseline round (interleaved_sample):
the same M prompts x G served as M/4 interleaved calls of one 32-sequence micro-batch each
(sample -> rewards -> advantage, no filter -> accumulate with the round's global 1/N), then
one optimizer step -- the token multiset equals the preemptive call's (scheduling
independence), so the two round times compare like for like.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17218_b200 as D  # noqa: E402
from paper_2505_17218_b200 import workload as W  # noqa: E402


def run_point(ctx, arch, M, G, P, ML, tau, micro, seed0):
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(0.02, 1)
    prompts = W.synthetic_prompts(1, 0, M, P, arch["vocab_size"], 0, 1)
    tok = prompts.reshape(-1).copy()
    off = [i * P for i in range(M + 1)]
    import numpy as np
    off = np.array(off, dtype=np.int64)
    out = None
    for i in range(2):   # warm-up, timed
        ro = pol.sample(None, G, ML, 1.0, round_seed=seed0 + i, prompt_tokens=tok, prompt_offsets=off)
        pol.set_rewards(W.synthetic_rewards(2 + seed0 + i, 0, M, G))
        pol.advantage(tau=tau)
        pol.grad_zero()
        pol.accumulate(1.0 / (M * G), micro)
        pol.allreduce_grads()
        pol.optimizer_step(D.OPT_ADAM, lr=1e-6)
        st = pol.stats()
        dev = st["sample_ms"] + st["advantage_ms"] + st["accumulate_ms"] + st["allreduce_ms"] + st["optimizer_ms"]
        out = dict(prompts=M, seqs=M * G, tau="off" if tau is None else tau, step_ms=dev,
                   sample_ms=st["sample_ms"], accumulate_ms=st["accumulate_ms"], kept=st["n_kept"],
                   sampled_tokens=int(ro.lengths.sum()), trained_tokens=st["loss_tokens"])
    pol.close()
    out["sampled_tokens_per_s"] = out["sampled_tokens"] / (out["step_ms"] / 1e3)
    out["ms_per_sequence"] = out["step_ms"] / out["seqs"]
    return out


def run_interleaved(ctx, arch, M, G, P, ML, micro_prompts, seed0):
    import numpy as np
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(0.02, 1)
    prompts = W.synthetic_prompts(1, 0, M, P, arch["vocab_size"], 0, 1)
    N = M * G
    out = None
    for it in range(2):   # warm-up round, timed round
        samp = acc = 0.0
        toks = trained = kept = 0
        pol.grad_zero()
        for c in range(0, M, micro_prompts):
            tok = prompts[c:c + micro_prompts].reshape(-1).copy()
            off = (np.arange(micro_prompts + 1) * P).astype(np.int64)
            ro = pol.sample(None, G, ML, 1.0, round_seed=seed0 + it, prompt_index_base=c, prompt_tokens=tok,
                            prompt_offsets=off)
            pol.set_rewards(W.synthetic_rewards(2 + seed0 + it, c, c + micro_prompts, G))
            pol.advantage(tau=None)
            pol.accumulate(1.0 / N, micro_prompts * G)
            st = pol.stats()
            samp += st["sample_ms"]
            acc += st["accumulate_ms"] + st["advantage_ms"]
            toks += int(ro.lengths.sum())
            trained += st["loss_tokens"]
            kept += st["n_kept"]
        pol.allreduce_grads()
        pol.optimizer_step(D.OPT_ADAM, lr=1e-6)
        st = pol.stats()
        step = samp + acc + st["optimizer_ms"] + st["allreduce_ms"]
        out = dict(mode="interleaved", prompts=M, seqs=N, calls=M // micro_prompts, tau="off", step_ms=step,
                   sample_ms=samp, accumulate_ms=acc, kept=kept, sampled_tokens=toks, trained_tokens=trained)
    pol.close()
    out["sampled_tokens_per_s"] = out["sampled_tokens"] / (out["step_ms"] / 1e3)
    out["ms_per_sequence"] = out["step_ms"] / out["seqs"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-len", type=int, default=1024)
    ap.add_argument("--prompt-len", type=int, default=128)
    ap.add_argument("--prompts", default="4,64,256,512")
    ap.add_argument("--taus", default="off,0,0.1,0.3")
    ap.add_argument("--micro", type=int, default=32)
    ap.add_argument("--interleaved", default="", help="round sizes (prompts) for the interleaved GRPO baseline")
    args = ap.parse_args()
    G, P, ML = 8, args.prompt_len, args.max_len
    arch = W.qwen_arch("0.5b", P + ML)
    ctx = D.Context(0)
    rows = []
    for M in [int(x) for x in args.interleaved.split(",") if x]:
        r = run_interleaved(ctx, arch, M, G, P, ML, 4, 100)
        print(json.dumps(r), flush=True)
        rows.append(r)
    for M in [int(x) for x in args.prompts.split(",") if x]:
        for t in args.taus.split(","):
            tau = None if t == "off" else float(t)
            r = run_point(ctx, arch, M, G, P, ML, tau, args.micro, 100)
            print(json.dumps(r), flush=True)
            rows.append(r)
    print("\n| mode | prompts x G | tau | kept / seqs | step s | sample s | accumulate s | sampled tok/s | ms / sequence |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        mode = f"interleaved ({r['calls']} calls)" if r.get("mode") else "preemptive"
        print(f"| {mode} | {r['prompts']} x {G} | {r['tau']} | {r['kept']} / {r['seqs']} | {r['step_ms'] / 1e3:.2f} | "
              f"{r['sample_ms'] / 1e3:.2f} | {r['accumulate_ms'] / 1e3:.2f} | {r['sampled_tokens_per_s']:.0f} | "
              f"{r['ms_per_sequence']:.2f} |")


if __name__ == "__main__":
    main()
