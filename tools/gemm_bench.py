"""tcgen05 GEMM throughput on the DASH step's shapes (Qwen2.5-0.5B, config 2).
Prints one JSON line per shape: ms per launch (CUDA events) and TFLOP/s."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17218_b200 as D  # noqa: E402

SHAPES = {
    # name: (M, N, K, a_kmajor, b_kmajor, epi)
    "dec_qkv": (4096, 1152, 896, 1, 1, 0), "dec_w1": (4096, 4864, 896, 1, 1, 0),
    "dec_w2": (4096, 896, 4864, 1, 1, 0), "dec_lm": (4096, 151936, 896, 1, 1, 0),
    "fwd_w1": (36864, 4864, 896, 1, 1, 0), "fwd_w2": (36864, 896, 4864, 1, 1, 0),
    "dgrad_w1": (36864, 896, 4864, 1, 0, 0), "wgrad_w1": (4864, 896, 36864, 0, 0, 3),
    "wgrad_lm": (151936, 896, 16384, 0, 0, 3), "dgrad_lm": (16384, 896, 151936, 1, 0, 0),
    "big_sq": (8192, 8192, 8192, 1, 1, 0), "fwd_qkv": (36864, 1152, 896, 1, 1, 0),
    # W2 backward into u with the dtanh epilogue (du = (dy W2) * (1 - tanh^2))
    "dgrad_w2_dtanh": (36864, 4864, 896, 1, 0, 2),
    # residual-stream epilogue (fp32 resid in, fp32 + bf16 out)
    "dec_wo_res": (4096, 896, 896, 1, 1, 4), "dec_w2_res": (4096, 896, 4864, 1, 1, 4),
    "fwd_wo_res": (36864, 896, 896, 1, 1, 4), "dgrad_qkv_res": (36864, 896, 1152, 1, 0, 4),
    "fwd_w2_res": (36864, 896, 4864, 1, 1, 4), "dgrad_w1_res": (36864, 896, 4864, 1, 0, 4),
    # small-output weight gradients (K = tokens of a micro-batch)
    # tanh epilogue (W1 forward, decode and training)
    "dec_w1_tanh": (4096, 4864, 896, 1, 1, 1), "fwd_w1_tanh": (36864, 4864, 896, 1, 1, 1),
    "wgrad_wo": (896, 896, 36864, 0, 0, 3), "wgrad_qkv": (1152, 896, 36864, 0, 0, 3),
    # small-batch decode (the GRPO-arm micro-batch of 32 sequences, and 64)
    "s32_qkv": (32, 1152, 896, 1, 1, 0), "s32_wo_res": (32, 896, 896, 1, 1, 4),
    "s32_w1_tanh": (32, 4864, 896, 1, 1, 1), "s32_w2_res": (32, 896, 4864, 1, 1, 4),
    "s64_qkv": (64, 1152, 896, 1, 1, 0), "s64_w2_res": (64, 896, 4864, 1, 1, 4),
    "s128_w2_res": (128, 896, 4864, 1, 1, 4),
    # C4 decode (Qwen2.5-3B, 64 prompts x 8 = 512 rows) and C3 decode (1.5B, 2048 rows)
    "c4_qkv": (512, 2560, 2048, 1, 1, 0), "c4_wo_res": (512, 2048, 2048, 1, 1, 4),
    "c4_w1_tanh": (512, 11008, 2048, 1, 1, 1), "c4_w2_res": (512, 2048, 11008, 1, 1, 4),
    "c3_w2_res": (2048, 1536, 8960, 1, 1, 4),
    # the same long-K decode W2 shapes as fp32 accumulates (split-K candidates)
    "c4_w2_acc": (512, 2048, 11008, 1, 1, 3), "c3_w2_acc": (2048, 1536, 8960, 1, 1, 3),
}


def main():
    L = D.lib()
    L.dashcu_selftest_gemm_timed.argtypes = [C.c_void_p] + [C.c_int] * 7 + [C.POINTER(C.c_double)]
    ctx = D.Context(0)
    names = sys.argv[1:] or list(SHAPES)
    for n in names:
        M, N, K, ak, bk, epi = SHAPES[n]
        ms = C.c_double(0)
        rc = L.dashcu_selftest_gemm_timed(ctx.h, M, N, K, ak, bk, epi, 10, C.byref(ms))
        assert rc == 0, L.dashcu_last_error()
        print(json.dumps({"shape": n, "M": M, "N": N, "K": K, "ms": ms.value,
                          "tflops": 2.0 * M * N * K / (ms.value * 1e-3) / 1e12}), flush=True)


if __name__ == "__main__":
    main()
