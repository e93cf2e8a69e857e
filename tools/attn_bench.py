"""Attention kernels alone at C2 micro-batch shapes (32 x 1151 tokens, 14/2 heads, hd 64):
best-of-N CUDA-event time of the forward and the backward, and TFLOP/s (causal flops).
    python tools/attn_bench.py [n_seq] [seq_len] [iters] [n_heads n_kv_heads head_dim]
Env DASHCU_ATTN_FWD / DASHCU_ATTN_BWD = mma selects the mma.sync kernels for A/B."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17218_b200 as D  # noqa: E402


def main():
    n_seq = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 1151
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    nh, nkv, hd = (int(a) for a in sys.argv[4:7]) if len(sys.argv) > 6 else (14, 2, 64)
    lib = D.lib()
    lib.dashcu_selftest_attn_timed.argtypes = [C.c_void_p] + [C.c_int] * 7 + [C.POINTER(C.c_double)]
    ctx = D.Context(0)
    pairs = n_seq * L * (L + 1) / 2
    out = {"n_seq": n_seq, "seq_len": L, "heads": [nh, nkv, hd]}
    for which, name, mult in ((0, "fwd", 4), (1, "bwd", 10)):
        ms = C.c_double(0)
        rc = lib.dashcu_selftest_attn_timed(ctx.h, n_seq, L, nh, nkv, hd, which, iters, C.byref(ms))
        assert rc == 0, lib.dashcu_last_error()
        out[name + "_ms"] = ms.value
        out[name + "_tflops"] = mult * nh * hd * pairs / (ms.value * 1e-3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
