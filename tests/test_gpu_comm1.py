"""libdashcu's NCCL calls on one GPU: with KNOB_COMM_WORLD1 the context
gets a real 1-rank NCCL communicator, so dashcu_allreduce_grads runs ncclAllReduce and
dashcu_sharded_step runs ncclReduceScatter -> slice Adam -> ncclAllGather (plus the async
error polling around them) on the round-end GPU box, which has one GPU. At world 1 every
collective is the identity: the gradient and the update must equal the communicator-free
path exactly. World 2 is tests/test_gpu_multi.py (skipped below 2 GPUs)."""
import numpy as np
import pytest

import paper_2505_17218_b200 as D
from test_gpu_multi import ARCH, G, M, batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_world1_nccl_allreduce_and_sharded_step(knob, dtype):
    prompts, comps, w = batch()
    results, g_ref = [], None
    for comm in (False, True):
        ctx = D.Context(0)
        if comm:
            knob("COMM_WORLD1", 1)
            ctx.init_comm(1, 0, D.comm_unique_id())
        pol = D.Policy(ctx, ARCH, dtype)
        pol.init_normal(0.05, 3)
        pol.load_rollout(prompts, G, comps)
        pol.grad_zero()
        pol.accumulate_weighted(w, micro_batch=4)
        g_acc = pol.grad()
        if g_ref is None:
            g_ref = g_acc
        pol.grad_upload(g_ref)                # the same gradient into both paths (the attention
        pol.allreduce_grads()                 # backward's reduce-adds are unordered, ~1e-7)
        g = pol.grad()
        pol.sharded_step(D.OPT_ADAM, lr=1e-3)
        results.append((g_acc, g, pol.download()))
        pol.close()
        ctx.close()
    (a0, g0, p0), (a1, g1, p1) = results
    assert np.linalg.norm(a0 - a1) <= 1e-6 * np.linalg.norm(a0)
    assert np.array_equal(g0, g1)          # a 1-rank NCCL all-reduce is the identity
    assert np.array_equal(p0, p1)          # reduce-scatter / all-gather of one slice: same update
