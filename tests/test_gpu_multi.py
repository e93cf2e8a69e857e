"""Multi-GPU data parallelism through libdashcu's own NCCL calls:
world 2 (one process per GPU, whole prompt groups per rank, global 1/N weights) against
world 1 on the same rollout. dashcu_allreduce_grads and dashcu_sharded_step
(reduce-scatter -> slice Adam -> all-gather) at world 2 must equal the single-GPU
gradient / update to fp32 summation order. Skipped below 2 visible GPUs (the gpurun
boxes have one; the host-side decomposition is covered on CPU by test_multirank.py)."""
import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2505_17218_b200 as D

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs 2 GPUs")]

ARCH = dict(vocab_size=300, embed_dim=256, context_len=64, ffn_hidden=256, n_layers=2, bos_id=0, eos_id=1,
            n_heads=14, n_kv_heads=2, head_dim=64)
M, G = 4, 4


def batch():
    rng = np.random.default_rng(1)
    prompts = [[0] + list(rng.integers(2, 300, size=5)) for _ in range(M)]
    comps = [list(rng.integers(2, 300, size=int(rng.integers(3, 20)))) for _ in range(M * G)]
    w = rng.standard_normal(M * G) / (M * G)
    return prompts, comps, w


def run_rank(rank, world, uid, q, dtype):
    prompts, comps, w = batch()
    ctx = D.Context(rank)
    ctx.init_comm(world, rank, uid)
    pol = D.Policy(ctx, ARCH, dtype)
    pol.init_normal(0.05, 3)
    per = M // world
    lo, hi = rank * per, (rank + 1) * per
    pol.load_rollout(prompts[lo:hi], G, comps[lo * G:hi * G])
    pol.grad_zero()
    pol.accumulate_weighted(w[lo * G:hi * G], micro_batch=4)
    pol.allreduce_grads()
    g = pol.grad()
    pol.sharded_step(D.OPT_ADAM, lr=1e-3)    # reduce-scatters the (already summed) gradient again:
    p_sh = pol.download()                     # the update uses world x grad, as below
    # the fused kernel over NVLink peer memory: same update from the same starting point
    pol2 = D.Policy(ctx, ARCH, dtype)
    pol2.init_normal(0.05, 3)
    pol2.grad_upload(g)
    pol2.fused_step(D.OPT_ADAM, lr=1e-3)
    assert np.abs(pol2.download() - p_sh).max() <= 1e-6
    pol2.close()
    q.put((rank, g, p_sh))
    pol.close()
    ctx.close()


@pytest.mark.parametrize("dtype", [D.F32, D.BF16])
def test_world2_allreduce_and_sharded_step(dtype):
    prompts, comps, w = batch()
    ctx = D.Context(0)
    pol = D.Policy(ctx, ARCH, dtype)
    pol.init_normal(0.05, 3)
    pol.load_rollout(prompts, G, comps)
    pol.grad_zero()
    pol.accumulate_weighted(w, micro_batch=4)
    g1 = pol.grad()
    pol.grad_upload(2 * g1)
    pol.optimizer_step(D.OPT_ADAM, lr=1e-3)
    p1 = pol.download()
    pol.close()
    ctx.close()
    uid = D.comm_unique_id()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=run_rank, args=(r, 2, uid, q, dtype)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (g, p)) for r, g, p in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        g, p = res[r]
        assert np.linalg.norm(g - g1) <= 1e-5 * np.linalg.norm(g1)
        assert np.max(np.abs(p - p1)) <= 1e-6
    assert np.array_equal(res[0][1], res[1][1])   # all-gathered masters identical on every rank


def run_rank_rebalance(rank, world, uid, q):
    prompts, comps, w = batch()
    rewards = np.zeros(M * G)
    rewards[:G * (M // 2)] = np.tile([1.0, 0.0, 0.0, 1.0], M // 2)   # rank 0's groups mixed, rank 1's uniform
    ctx = D.Context(rank)
    ctx.init_comm(world, rank, uid)
    pol = D.Policy(ctx, ARCH, D.F32)
    pol.init_normal(0.05, 3)
    per = M // world
    lo, hi = rank * per, (rank + 1) * per
    pol.load_rollout(prompts[lo:hi], G, comps[lo * G:hi * G])
    pol.set_rewards(rewards[lo * G:hi * G])
    pol.advantage(tau=0.1)
    before = pol.stats()["n_kept"]
    n_out, n_in = pol.rebalance()
    pol.grad_zero()
    pol.accumulate(1.0 / (M * G), micro_batch=4)
    pol.allreduce_grads()
    q.put((rank, before, n_out, n_in, pol.grad()))
    pol.close()
    ctx.close()


def test_world2_rebalance():
    """dashcu_rebalance moves kept sequences from the loaded rank to the idle one; the
    all-reduced gradient equals the single-GPU one."""
    prompts, comps, _ = batch()
    rewards = np.zeros(M * G)
    rewards[:G * (M // 2)] = np.tile([1.0, 0.0, 0.0, 1.0], M // 2)
    ctx = D.Context(0)
    pol = D.Policy(ctx, ARCH, D.F32)
    pol.init_normal(0.05, 3)
    pol.load_rollout(prompts, G, comps)
    pol.set_rewards(rewards)
    pol.advantage(tau=0.1)
    pol.grad_zero()
    pol.accumulate(1.0 / (M * G), micro_batch=4)
    g1 = pol.grad()
    pol.close()
    ctx.close()
    uid = D.comm_unique_id()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=run_rank_rebalance, args=(r, 2, uid, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == 8 and res[1][0] == 0          # kept before: all on rank 0
    assert res[0][1] == res[1][2] > 0                  # what rank 0 sent, rank 1 received
    for r in range(2):
        assert np.linalg.norm(res[r][3] - g1) <= 1e-5 * np.linalg.norm(g1)
