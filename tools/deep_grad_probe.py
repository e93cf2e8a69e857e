"""Per-tensor gradient error of the device path vs the fp64 oracle on a deep policy
(test_gpu_scale.py geometry): which tensors lose precision in bf16, and whether the
sampler-LSE reuse contributes. Usage: python tools/deep_grad_probe.py [layers] [scale...]"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_ffi as O  # noqa: E402
import paper_2505_17218_b200 as D  # noqa: E402
from test_gpu_parity import tensor_slices  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
scales = [float(x) for x in sys.argv[2:]] or [0.02, 0.044]
arch = dict(vocab_size=151936, embed_dim=128, context_len=1152, ffn_hidden=256, n_layers=L, bos_id=0, eos_id=1,
            n_heads=14, n_kv_heads=2, head_dim=64)
ctx = D.Context(0)
rng = np.random.default_rng(4)
prompts = [[0] + list(rng.integers(2, 151936, size=31)) for _ in range(2)]
G = 2
for scale in scales:
    pb = D.Policy(ctx, arch, D.BF16)
    pb.init_normal(scale, 17)
    p = pb.download()
    ro = pb.sample(prompts, G, 96, round_seed=21)
    comps = [list(ro.completion(s)) for s in range(4)]
    w = np.random.default_rng(6).standard_normal(4) / 4

    def one(s):
        g = np.zeros(len(p))
        O.grad_log_prob(arch, p, prompts[s // G], comps[s], w[s], g)
        return g
    with ThreadPoolExecutor(4) as ex:
        ref = sum(ex.map(one, range(4)))
    res = {}
    pb.grad_zero()
    pb.accumulate_weighted(w, micro_batch=4)
    res["bf16-reuse"] = pb.grad()
    pb.load_rollout(prompts, G, comps)      # external trajectories: LSE pass recomputed
    pb.grad_zero()
    pb.accumulate_weighted(w, micro_batch=4)
    res["bf16-recompute"] = pb.grad()
    pb.close()
    pf = D.Policy(ctx, arch, D.F32)
    pf.upload(p)
    pf.load_rollout(prompts, G, comps)
    pf.grad_zero()
    pf.accumulate_weighted(w, micro_batch=4)
    res["f32"] = pf.grad()
    pf.close()
    print(f"scale {scale}: |g| {np.linalg.norm(ref):.3e}")
    for name, got in res.items():
        errs = []
        for tn, sl in tensor_slices(arch):
            nr = np.linalg.norm(ref[sl])
            errs.append((np.linalg.norm(got[sl] - ref[sl]) / max(nr, 1e-300), tn, nr))
        errs.sort(reverse=True)
        print(f"  {name:15s} worst " + ", ".join(f"{tn} {e:.2e} (|g_t| {nr:.1e})" for e, tn, nr in errs[:5]))
        qk = [e for e, tn, nr in errs if tn.endswith(".wq") or tn.endswith(".wk")]
        print(f"  {'':15s} median wq/wk {np.median(qk):.2e}, others max "
              f"{max(e for e, tn, nr in errs if not (tn.endswith('.wq') or tn.endswith('.wk'))):.2e}")
