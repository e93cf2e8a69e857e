"""Timeline of the tcgen05 attention backward for one CTA (debug build with
-DDASHCU_ATTN_TRACE, loaded via DASHCU_LIB_PATH). Runs one C2-shaped micro-batch and prints,
per iteration, the cycle offsets of the MMA issuer and of softmax warp 4 (see TR() slots)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2505_17218_b200 as D  # noqa: E402
from paper_2505_17218_b200 import workload as W  # noqa: E402

NAMES = {0: "mma:sfree", 1: "mma:S issued", 2: "mma:pready", 3: "mma:dqfree/456", 4: "sm:wait sfull", 5: "sm:sfull",
         6: "sm:h0 computed", 7: "sm:pfree", 8: "sm:dqfull", 9: "sm:dq_out done", 10: "sm:h1 computed",
         11: "sm:h1 pfree", 12: "sm:h0 loaded", 13: "sm:h1 loaded", 14: "sm:pready"}


FWD_NAMES = {0: "mma:S(t+1) issued", 1: "mma:pready", 2: "mma:PV issued", 4: "sm:wait sfull", 5: "sm:sfull",
             6: "sm:max done", 7: "sm:pair barrier", 8: "sm:exp done", 9: "sm:ofull(t-1)", 10: "sm:pready",
             11: "sm:take_o done"}


def main():
    n_seq = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    P, L = 128, 1024
    arch = W.qwen_arch("0.5b", P + L)
    ctx = D.Context(0)
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(0.02, 1)
    rng = np.random.default_rng(0)
    prompts = [list(p) for p in W.synthetic_prompts(1, 0, n_seq, P, arch["vocab_size"], 0, 1)]
    comps = [list(rng.integers(2, arch["vocab_size"], size=L)) for _ in range(n_seq)]
    pol.load_rollout(prompts, 1, comps)
    w = np.full(n_seq, 1.0 / n_seq)
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=n_seq)
    pol.accumulate_weighted(w, micro_batch=n_seq)
    global NAMES
    if os.environ.get("TRACE_FWD"):
        NAMES = FWD_NAMES
    buf = (C.c_ulonglong * (64 * 16))()
    assert D.lib().dashcu_debug_attn_trace(buf, 64 * 16) == 0
    t = np.array(buf, dtype=np.int64).reshape(64, 16)
    t0 = t[0, 4]
    prev = None
    for it in range(63):
        row = {NAMES[k]: int(t[it, k] - t0) for k in NAMES if t[it, k]}
        ordered = sorted(row.items(), key=lambda kv: kv[1])
        start = ordered[0][1] if ordered else 0
        print(f"it {it:2d} +{(start - prev) if prev is not None else 0:6d} | " +
              "  ".join(f"{k}={v - start}" for k, v in ordered))
        prev = start


if __name__ == "__main__":
    main()
