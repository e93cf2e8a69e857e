"""World-size-2 checks of the data-parallel DASH step on CPU (gloo), the multi-GPU
design of SURVEY §8e: prompts sharded by global index with whole groups per rank,
per-request keys independent of the split, each rank accumulating its shard's PG
gradient with the GLOBAL 1/N, one sum-allreduce, then an identical optimizer step.
The per-rank gradients come from the CPU oracle; the collective is torch.distributed.
The ZeRO-1 form (dashcu_sharded_step) is checked the same way: slices
from the library's own dashcu_shard_span (no device work), reduce-scatter, Adam on the
rank's slice with slice-sized moments, all-gather == the replicated update, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ffi as O
from paper_2505_17218_b200 import workload as W

ARCH = dict(vocab_size=13, embed_dim=8, context_len=24, ffn_hidden=12, n_layers=2, bos_id=0, eos_id=1,
            n_heads=2, n_kv_heads=1, head_dim=4)
M, G, ML, SEED = 6, 4, 6, 11


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard(rank, world):
    per = M // world
    return rank * per, (rank + 1) * per


def rank_gradient(params, lo, hi):
    """This rank's contribution: sum over its kept sequences of (A_n / N_global) grad log pi."""
    g = np.zeros_like(params)
    prompts = W.synthetic_prompts(3, lo, hi, 4, ARCH["vocab_size"], 0, 1)
    comps = []
    for i, m in enumerate(range(lo, hi)):
        for gg in range(G):
            c, _ = O.sample(ARCH, params, list(prompts[i]), ML, 1.0, O.derive_seed(SEED, "sample", m, gg))
            comps.append(list(c))
    r = W.synthetic_rewards(5, lo, hi, G)
    adv, kept, idx = O.advantage_filter(r, G, 1, False, 0.0, 0.1)   # groups never straddle ranks
    for s in idx:
        O.grad_log_prob(ARCH, params, list(prompts[s // G]), comps[s], adv[s] / (M * G), g)
    return g, comps


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = O.init_params(ARCH, 0.4, 2)
    lo, hi = shard(rank, world)
    g, comps = rank_gradient(params, lo, hi)
    g_local = g.copy()
    t = torch.from_numpy(g)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    # replicated Adam step after the allreduce: every rank ends with identical weights
    p = params.copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    gg = t.numpy().copy()
    O.oracle().dor_adam_step(O.ptr(p, O.f64p), O.ptr(gg, O.f64p), O.ptr(m, O.f64p), O.ptr(v, O.f64p), len(p), 1,
                             1e-3, 0.9, 0.999, 1e-8)
    # ZeRO-1: reduce-scatter -> Adam on this rank's slice -> all-gather
    import paper_2505_17218_b200 as D
    n = len(params)
    spans = [D.shard_span(n, world, r) for r in range(world)]
    sl = spans[0][1]
    gp = np.zeros(sl * world)
    gp[:n] = g_local
    parts = [torch.zeros(sl, dtype=torch.float64) for _ in range(world)]
    dist.reduce_scatter(parts[rank], list(torch.from_numpy(gp).split(sl)), op=dist.ReduceOp.SUM)
    off, ln = spans[rank]
    ws = np.zeros(sl)
    ws[:ln] = params[off:off + ln]
    gs = parts[rank].numpy().copy()
    ms, vs = np.zeros(sl), np.zeros(sl)
    O.oracle().dor_adam_step(O.ptr(ws, O.f64p), O.ptr(gs, O.f64p), O.ptr(ms, O.f64p), O.ptr(vs, O.f64p), ln, 1,
                             1e-3, 0.9, 0.999, 1e-8)
    out = [torch.zeros(sl, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, torch.from_numpy(ws))
    p_sharded = torch.cat(out).numpy()[:n]
    assert np.array_equal(gs[:ln], gg[off:off + ln]), ("rs", np.abs(gs[:ln] - gg[off:off + ln]).max(), np.abs(gg).max())
    assert np.array_equal(p_sharded, p), ("upd", np.abs(p_sharded - p).max())
    # bench.py reduction helpers (max of step times, sum of tokens) over the same group
    import bench
    mx = bench.allreduce([float(rank + 1)], "max")[0]
    sm = bench.allreduce([float(rank + 1)], "sum")[0]
    q.put((rank, gg, p, comps, mx, sm))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_step_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    params = O.init_params(ARCH, 0.4, 2)
    g_all, comps_all = rank_gradient(params, 0, M)
    # identical token multiset for any worker split
    assert res[0][3] + res[1][3] == comps_all
    for r in range(world):
        assert np.linalg.norm(res[r][1] - g_all) <= 1e-12 * max(1.0, np.linalg.norm(g_all))
    assert np.array_equal(res[0][2], res[1][2])            # replicated optimizer state stays in sync
    assert res[0][4] == 2.0 and res[0][5] == 3.0            # max / sum over ranks


def rebalance_worker(rank, world, port, q):
    """Post-filter rebalancing (dashcu_rebalance's plan) as every rank runs it:
    kept-item costs all-gathered, the library's planner on each rank, items accumulated where
    the plan sends them; the all-reduced gradient must not change."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2505_17218_b200 as D
    params = O.init_params(ARCH, 0.4, 2)
    per = M // world

    def items(r):   # (cost, prompt, completion, weight) of rank r's kept sequences, in index order
        lo, hi = r * per, (r + 1) * per
        prompts = W.synthetic_prompts(3, lo, hi, 4, ARCH["vocab_size"], 0, 1)
        r_ = W.synthetic_rewards(5, lo, hi, G)
        adv, kept, idx = O.advantage_filter(r_, G, 1, False, 0.0, 0.1)
        out = []
        for s in idx:
            m = lo + s // G
            c, _ = O.sample(ARCH, params, list(prompts[s // G]), ML, 1.0, O.derive_seed(SEED, "sample", m, s % G))
            out.append((4 + len(c), list(prompts[s // G]), list(c), adv[s] / (M * G)))
        return out
    mine = items(rank)
    costs = [None] * world
    dist.all_gather_object(costs, [it[0] for it in mine])
    plan = D.rebalance_plan(costs)
    before = [sum(c) for c in costs]
    after = [0] * world
    for r in range(world):
        for i, d in enumerate(plan[r]):
            after[d] += costs[r][i]
    # every rank accumulates what the plan sends it (its own kept items or imported ones)
    g = np.zeros_like(params)
    for r in range(world):
        src = mine if r == rank else items(r)
        for i, d in enumerate(plan[r]):
            if d == rank:
                _, pr, c, w = src[i]
                O.grad_log_prob(ARCH, params, pr, c, w, g)
    t = torch.from_numpy(g)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    q.put((rank, [list(p) for p in plan], before, after, t.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_rebalance_plan_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=rebalance_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    assert res[0][1] == res[1][1]                              # the same plan on every rank
    before, after = res[0][2], res[0][3]
    assert sum(before) == sum(after) and max(after) <= max(before)
    params = O.init_params(ARCH, 0.4, 2)
    g_all, _ = rank_gradient(params, 0, M)
    for r in range(world):
        assert np.linalg.norm(res[r][4] - g_all) <= 1e-12 * max(1.0, np.linalg.norm(g_all))


def test_rebalance_plan_properties():
    import paper_2505_17218_b200 as D
    rng = np.random.default_rng(0)
    for world in (2, 4, 8):
        for _ in range(20):
            costs = [list(rng.integers(10, 1200, size=int(rng.integers(0, 60)))) for _ in range(world)]
            plan = D.rebalance_plan(costs)
            load = [0] * world
            for r in range(world):
                assert len(plan[r]) == len(costs[r])
                for i, d in enumerate(plan[r]):
                    load[d] += costs[r][i]
            before = [sum(c) for c in costs]
            assert sum(load) == sum(before) and max(load) <= max(before)
            if sum(before):
                assert max(load) - sum(load) / world <= max(max(c) if c else 0 for c in costs) + 1e-9
    assert [list(x) for x in D.rebalance_plan([[100, 200, 300, 400], [50], [10, 10]])] == [[0, 0, 1, 2], [1], [0, 0]]
