#!/usr/bin/env python
"""DASH training-step benchmark (BASELINE.json metric) on 1..8 B200.

One step = the DASH hot path over one synthetic round:
  preemptive_sample (M prompts x G)  -> synthetic rewards -> group advantage + |A|
  filter -> micro-batched PG accumulate (fp32 grads) -> NCCL allreduce -> Adam.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Default workload = BASELINE configs[1] (Qwen2.5-0.5B-shaped random-init policy,
512 prompts x G=8, gen len 1024, one B200), weak-scaled: every rank samples its
own 512-prompt shard of one global round (keys derive_seed(round, "sample", m, g)),
one allreduce per optimizer step.

Reported:
  value     whole-job sampled tokens / s, device-timed (sum of the library's CUDA-
            event phase timers on its stream), max over ranks
  e2e       same metric through the C ABI with host buffers: wall clock around the
            API calls (prompts H2D, completions/logp/advantages D2H), max over ranks
  roofline  dominant kernel class: algorithmic flops (bytes) / its CUDA-event time
  cpu_baseline  the reference's own CPU DASH step (oracle/_ref) on a bounded sample
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2505_17218_b200 import workload as W  # noqa: E402

CONFIGS = {
    "c2": dict(size="0.5b", prompts=512, G=8, prompt_len=128, max_len=1024, micro=32, tau=0.1,
               workload="BASELINE configs[1]: Qwen2.5-0.5B-shaped random-init policy, 512 prompts x G=8, "
                        "gen len 1024, per B200"),
    # init std 0.01 at 1.5B / 3B: the reference math has no normalisation, and at std 0.02 the
    # 28-layer residual stream grows until the fp32 gradient of a gen-1024 rollout overflows
    # (|g| -> inf, measured with tools/len_probe.py; the update then NaNs the policy and later
    # rollouts end after ~30 tokens). At 0.01: |g| 25 (1.5B) / 237 (3B), near-uniform policy.
    "c3": dict(size="1.5b", prompts=256, G=8, prompt_len=128, max_len=1024, micro=32, tau=0.1, init=0.01,
               workload="BASELINE configs[2] shard: Qwen2.5-1.5B-shaped, 2048 prompts x G=8 over 8 B200 "
                        "(256 prompts per B200), micro-batch 32"),
    # micro-batch 16 at 3B: 32 x 2175 tokens of saved activations (~3.3 GB per layer x 36) do
    # not fit beside the weights, Adam state and the 41 GB KV cache
    "c4": dict(size="3b", prompts=64, G=8, prompt_len=128, max_len=2048, micro=16, tau=0.1, init=0.01,
               workload="BASELINE configs[3] shard: Qwen2.5-3B-shaped, gen len 2048, |A| filter 0.1, 512 prompts x G=8 "
                        "over 8 B200 (64 prompts per B200)"),
    "grpo": dict(size="0.5b", prompts=4, G=8, prompt_len=128, max_len=1024, micro=32, tau=None,
                 workload="BASELINE configs[4] GRPO-style arm: Qwen2.5-0.5B-shaped, small sampling batch (4 prompts x "
                          "G=8 per B200), no gradient filter"),
    "mini": dict(size="0.5b", prompts=64, G=8, prompt_len=128, max_len=128, micro=32, tau=0.1,
                 workload="development: Qwen2.5-0.5B-shaped, 64 prompts x G=8, gen len 128"),
    "c1": dict(size=None, prompts=64, G=8, prompt_len=7, max_len=57, micro=32, tau=0.1,
               workload="BASELINE configs[0]: SPEC tiny policy (2 layers, d=128, byte vocab), 64 prompts x G=8"),
}
C1_ARCH = dict(vocab_size=256, embed_dim=128, context_len=64, ffn_hidden=512, n_layers=2, bos_id=0, eos_id=1)
PROF_PERIOD = 17
# bounded CPU samples of the same workload: the reference arm's per-step
# sample (short, so K steps end within minutes) and the cpu_baseline sub-batch of our arm
# (8 sequences per 8 host cores x 16 generated tokens); prompt 4 tokens because the
# reference re-runs the prompt for every sample (policy.cpp:396) at ~0.5 s per token-core
REF_SAMPLE = dict(G=8, prompt_len=4, max_len=4)
CPU_BASELINE_SAMPLE = dict(G=8, prompt_len=4, max_len=16)


def prompts_of(cfg, arch, m_lo, m_hi, reference=False):
    """[m_hi - m_lo, prompt_len] prompts of global prompt ids m_lo..m_hi-1: the ADD task's
    generate_instance (difficulty 2, byte vocabulary; tasks.cpp:105-112) for configs[0],
    uniform random ids after BOS for the Qwen-shaped configs."""
    if cfg["size"] is None:
        seeds = [int(W.derive_seed(1, "prompt", m, 0)) for m in range(m_lo, m_hi)]
        if reference:   # the reference arm: the reference's own generate_instance (oracle/_ref)
            import ctypes as C
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import oracle_ffi as O
            out = np.zeros((m_hi - m_lo, 16), dtype=np.int32)
            for i, sd in enumerate(seeds):
                m, ans = C.c_int32(0), C.create_string_buffer(16)
                row = np.zeros(16, dtype=np.int32)
                if O.ref().ref_add_instance(2, C.c_uint64(sd), O.ptr(row, O.i32p), C.byref(m), ans, 16):
                    raise RuntimeError("reference generate_instance failed")
                out[i] = row
            return out[:, :cfg["prompt_len"]]
        import paper_2505_17218_b200 as D
        toks, off, _ = D.task_instances(D.TASK_ADD, 2, seeds, D.VOCAB_BYTE)
        assert np.all(np.diff(off) == cfg["prompt_len"])
        return toks.reshape(m_hi - m_lo, cfg["prompt_len"])
    return W.synthetic_prompts(1, m_lo, m_hi, cfg["prompt_len"], arch["vocab_size"], arch["bos_id"], arch["eos_id"])


def arch_of(cfg):
    if cfg["size"] is None:
        return dict(C1_ARCH)
    return W.qwen_arch(cfg["size"], cfg["prompt_len"] + cfg["max_len"])


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return dict(hbm=float(d["hbm_gbs"]), tc=float(d["bf16_tflops"]), tc_sus=float(d["bf16_tflops_sustained"]),
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, tc=1590.0, tc_sus=1400.0, src="fallback")


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.path = gpu, None, f"/tmp/dash_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # NCCL init lines: nranks, NVLink / NVLS paths
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def self_launch(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-exec as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1, exactly as the driver launches it."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # NCCL's init lines (nranks, NVLS / NVLink paths)
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def allreduce(vals, op):
    """max / sum over ranks of a small list of floats (torch.distributed plumbing)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return list(vals)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.cpu().tolist()


def barrier():
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()


def pinned(shape, dtype):
    try:
        import torch
        if torch.cuda.is_available():
            tdt = {np.int32: torch.int32, np.int64: torch.int64, np.float32: torch.float32,
                   np.float64: torch.float64}[dtype]
            return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    except Exception:
        pass
    return np.empty(shape, dtype=dtype)


# --------------------------------------------------------------- reference arm

def ref_step_runner(cfg, threads, sample_cfg=None):
    """The reference's own CPU DASH step (oracle/_ref ref_dash_step) on a bounded sample;
    run(step) -> RefStepStats (per-phase seconds, tokens)."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as O
    arch = arch_of(cfg)
    for k in ("n_heads", "n_kv_heads", "head_dim"):   # the reference is single-head (policy.cpp:93-129)
        arch.pop(k, None)
    rs = dict(sample_cfg or REF_SAMPLE, prompts=max(1, threads // 8)) if cfg["size"] else \
        dict(prompts=cfg["prompts"], G=cfg["G"], prompt_len=cfg["prompt_len"], max_len=cfg["max_len"])
    arch["context_len"] = max(arch["context_len"], rs["prompt_len"] + rs["max_len"])
    n = O.num_params(arch)
    params = (np.random.default_rng(1).standard_normal(n, dtype=np.float32) * 0.02).astype(np.float64)
    m = np.zeros(n)
    v = np.zeros(n)
    t = C.c_int64(0)
    P = prompts_of(dict(cfg, prompt_len=rs["prompt_len"]), arch, 0, rs["prompts"], reference=True)
    toks = np.ascontiguousarray(P.reshape(-1))
    off = (np.arange(rs["prompts"] + 1) * rs["prompt_len"]).astype(np.int64)
    R = O.ref()
    sample = (f"{rs['prompts']} prompt(s) x G={rs['G']}, prompt {rs['prompt_len']} tok, max_len {rs['max_len']} "
              f"of the {cfg['size'] or 'tiny'} workload (reference single-head geometry), full DASH step "
              f"(sample, reward, group adv+filter, sum A/N grad_log_prob, Adam), {threads} threads")

    def run(step):
        st = O.RefStepStats()
        rc = R.ref_dash_step(O.arch_ref_vec(arch), O.ptr(params, O.f64p), O.ptr(toks, O.i32p), O.ptr(off, O.i64p),
                             rs["prompts"], rs["G"], rs["max_len"], 1.0, 1000 + step, 0, 0, 3, None,
                             float("-inf") if cfg["tau"] is None else cfg["tau"], 1,
                             1e-6, O.ptr(m, O.f64p), O.ptr(v, O.f64p), C.byref(t), threads, C.byref(st))
        if rc != 0:
            raise RuntimeError("reference step failed")
        return st
    return run, sample


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    run, sample = ref_step_runner(cfg, threads)
    for i in range(min(args.warmup, 1)):
        run(i)
    toks, secs = 0, 0.0
    for i in range(args.steps):
        st = run(100 + i)
        toks += st.tokens_sampled
        secs += st.total_s
    val = toks / secs
    line = {"metric": "dash_step_sampled_tokens_per_s", "value": val, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": 1000 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg["workload"], "parallelism": "host threads"},
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- our arm

def run_ours(args, cfg, world, rank, local):
    import paper_2505_17218_b200 as D
    arch = arch_of(cfg)
    M, G, ML = cfg["prompts"], cfg["G"], cfg["max_len"]
    ctx = D.Context(local)
    if world > 1:
        import torch.distributed as dist
        obj = [D.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.init_comm(world, rank, obj[0])
    pol = D.Policy(ctx, arch, D.BF16)
    pol.init_normal(cfg.get("init", 0.02), 1)
    base = rank * M
    P = prompts_of(cfg, arch, base, base + M)
    ptok = pinned(P.size, np.int32)
    ptok[:] = P.reshape(-1)
    poff = pinned(M + 1, np.int64)
    poff[:] = np.arange(M + 1) * cfg["prompt_len"]
    S = M * G
    outs = (pinned((S, max(ML, 1)), np.int32), pinned(S, np.int32), pinned((S, max(ML, 1)), np.float32))
    N_global = M * G * world

    phase_prof = {"sample": {}, "accumulate": {}}

    def add_prof(ph):  # kernel-class totals of the phase that just ran (profiling on)
        for k, v in D.profile_read(reset=True).items():
            a = phase_prof[ph].setdefault(k, dict(ms=0.0, flops=0.0, bytes=0.0, launches=0))
            for f in a:
                a[f] += v[f]

    def step(i, prof=False):
        t0 = time.perf_counter()
        ro = pol.sample(None, G, ML, 1.0, round_seed=i, prompt_index_base=base, prompt_tokens=ptok,
                        prompt_offsets=poff, outputs=outs)
        if prof:
            add_prof("sample")
        r = W.synthetic_rewards(2 + i, base, base + M, G)
        pol.set_rewards(r)
        adv, kept, nk = pol.advantage(tau=cfg["tau"])
        pol.grad_zero()
        pol.accumulate(1.0 / N_global, cfg["micro"])
        if args.fused:     # ZeRO-1 form as one kernel over NVLink peer memory
            pol.fused_step(D.OPT_ADAM, lr=1e-6)
        elif args.sharded:   # ZeRO-1 form: reduce-scatter, update own slice, all-gather
            pol.sharded_step(D.OPT_ADAM, lr=1e-6)
        else:
            pol.allreduce_grads()
            pol.optimizer_step(D.OPT_ADAM, lr=1e-6)
        if prof:
            add_prof("accumulate")
        st = pol.stats()
        wall = time.perf_counter() - t0
        dev = st["sample_ms"] + st["advantage_ms"] + st["accumulate_ms"] + st["allreduce_ms"] + st["optimizer_ms"]
        return int(ro.lengths.sum()), dev, wall * 1e3, st

    for i in range(args.warmup):
        step(i)
    barrier()
    ctx.sync()
    clocks = Clocks(local)
    clocks.start()
    # per-kernel events on one launch in PROF_PERIOD of each class (a prime, so the sampled
    # launches cycle through every GEMM shape of a layer), scaled to the class totals
    D.profile_sampling(PROF_PERIOD)
    if not args.no_profile:
        D.profile_enable()
    D.profile_read(reset=True)
    l0 = D.kernel_launches()
    toks, dev_ms, wall_ms, last, phase_ms = 0, 0.0, 0.0, None, {"sample": 0.0, "accumulate": 0.0}
    for i in range(args.steps):
        a, b, c, last = step(args.warmup + i, prof=not args.no_profile)
        toks += a
        dev_ms += b
        wall_ms += c
        phase_ms["sample"] += last["sample_ms"]
        phase_ms["accumulate"] += last["accumulate_ms"] + last["allreduce_ms"] + last["optimizer_ms"]
    ctx.sync()
    barrier()
    launches = D.kernel_launches() - l0
    add_prof("accumulate")
    D.profile_enable(())
    prof = {}
    for ph in phase_prof.values():
        for k, v in ph.items():
            a = prof.setdefault(k, dict(ms=0.0, flops=0.0, bytes=0.0, launches=0))
            for f in a:
                a[f] += v[f]
    clk = clocks.stop()
    tot_toks = allreduce([toks], "sum")[0]
    dev_ms, wall_ms = allreduce([dev_ms, wall_ms], "max")
    ms_step = dev_ms / args.steps
    value = tot_toks / (dev_ms / 1e3)
    e2e = tot_toks / (wall_ms / 1e3)

    pk = peaks()
    prof = {k: v for k, v in prof.items() if v["ms"] > 0}
    if not prof:  # --no-profile
        prof = {"none": dict(ms=1.0, flops=0.0, bytes=0.0, launches=0)}
    top = max(prof.items(), key=lambda kv: kv[1]["ms"])
    name, pr = top
    hbm_bound = name in ("attn_decode", "sample", "lm_rows", "optimizer")
    per_launch_ms = pr["ms"] / max(pr["launches"], 1)
    if hbm_bound:
        achieved = pr["bytes"] / (pr["ms"] / 1e3) / 1e9
        peak, unit = pk["hbm"], "GB/s"
    else:
        achieved = pr["flops"] / (pr["ms"] / 1e3) / 1e12
        peak, unit = pk["tc_sus"], "TFLOP/s"
    traffic, traffic_note = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic_c2.json")
    if os.path.exists(tp):
        t = json.load(open(tp)).get(name)
        if t:
            traffic = t["dram_bytes"]
            traffic_note = (f"ncu --set full, {t['shape']}: DRAM {t['dram_bytes'] / 1e6:.1f} MB per launch vs "
                            f"{t['alg_bytes'] / 1e6:.1f} MB algorithmic (x{t['dram_bytes'] / t['alg_bytes']:.2f})")
    phase_roofline = phase_rooflines(phase_prof, phase_ms, pk, args.steps)

    S_all = S
    h2d = ptok.nbytes + poff.nbytes + S_all * 8       # prompts + rewards
    d2h = sum(o.nbytes for o in outs) + S_all * (8 + 1) + 4 * 8   # rollout + advantages/kept + stats
    line = {
        "metric": "dash_step_sampled_tokens_per_s", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": cfg["workload"], "model": f"Qwen2.5-{cfg['size'] or 'tiny'}-shaped (reference math,"
                   f" GQA {arch.get('n_heads', 1)}/{arch.get('n_kv_heads', 1)})", "prompts_per_gpu": M, "G": G,
                   "prompt_len": cfg["prompt_len"], "gen_len": ML, "micro_batch": cfg["micro"], "tau": cfg["tau"] if cfg["tau"] is not None else "off",
                   "optimizer": ("adam (ZeRO-1, fused peer-memory kernel)" if args.fused else
                                 "adam (sharded, ZeRO-1)" if args.sharded else "adam"), "global_batch": M * G * world, "seq_len": cfg["prompt_len"] + ML,
                   "parallelism": f"dp{world}", "init_std": cfg.get("init", 0.02),
                   "mean_completion_len": tot_toks / (args.steps * M * G * world), "l2": "inputs > L2 (KV cache + weights stream every step)"},
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm" if hbm_bound else "tensor", "kernel": name, "achieved": achieved,
                     "peak": peak, "unit": unit, "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": traffic_note,
                     "per_launch_ms": per_launch_ms, "event_sampling": f"1 in {PROF_PERIOD} launches per class",
                     "peak_source": pk["src"] + (" burst" if False else
                                                                                " sustained" if not hbm_bound else "")},
        "phases_ms": {k: last[k] for k in ("sample_ms", "advantage_ms", "accumulate_ms", "allreduce_ms",
                                           "optimizer_ms")},
        "kernel_classes": {k: {"ms_per_step": v["ms"] / args.steps, "launches": v["launches"]}
                           for k, v in prof.items() if v["launches"]},
        "phase_rooflines": phase_roofline,
        "kept": last["n_kept"], "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, arch, S, tot_toks / args.steps, last)
        except Exception as e:  # reference not built on this box
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    pol.close()
    ctx.close()


def phase_rooflines(pp, phase_ms, pk, steps):
    """Per-phase roofline fractions (north_star targets) from the phase-split kernel classes:
    decode attention (HBM-bound; K/V bytes with the group's prompt KV counted once), the
    decode projections + sampling GEMM (tensor), the decode phase against its serial floor
    (attention bytes / HBM + GEMM flops / tensor peak), and the accumulate phase (every
    tensor-core flop of the PG step over the phase time, optimizer + allreduce included)."""
    s, a = pp["sample"], pp["accumulate"]
    out = {}
    ad = s.get("attn_decode")
    if ad and ad["ms"]:
        gbs = ad["bytes"] / (ad["ms"] / 1e3) / 1e9
        out["decode_attention"] = {"achieved": gbs, "unit": "GB/s", "peak": pk["hbm"], "frac": gbs / pk["hbm"],
                                   "ms_per_step": ad["ms"] / steps}
    gf = sum(s[k]["flops"] for k in ("gemm_tc", "sample", "attn_fwd") if k in s)
    gm = sum(s[k]["ms"] for k in ("gemm_tc", "sample", "attn_fwd") if k in s)
    if gm:
        tf = gf / (gm / 1e3) / 1e12
        out["decode_gemm"] = {"achieved": tf, "unit": "TFLOP/s", "peak": pk["tc_sus"], "frac": tf / pk["tc_sus"],
                              "ms_per_step": gm / steps, "note": "prefill + decode projections + LM-head sampling"}
    if phase_ms["sample"] and ad:
        floor = ad["bytes"] / (pk["hbm"] * 1e9) * 1e3 + gf / (pk["tc_sus"] * 1e12) * 1e3
        out["decode_phase"] = {"floor_ms_per_step": floor / steps, "ms_per_step": phase_ms["sample"] / steps,
                               "frac": floor / phase_ms["sample"],
                               "note": "attention HBM floor + GEMM tensor floor, serial, over the sampling phase"}
    af = sum(a[k]["flops"] for k in ("gemm_tc", "attn_fwd", "attn_bwd", "lm_rows") if k in a)
    if phase_ms["accumulate"]:
        tf = af / (phase_ms["accumulate"] / 1e3) / 1e12
        out["accumulate_phase"] = {"achieved": tf, "unit": "TFLOP/s", "peak": pk["tc_sus"], "frac": tf / pk["tc_sus"],
                                   "ms_per_step": phase_ms["accumulate"] / steps,
                                   "kernel_ms_per_step": {k: v["ms"] / steps for k, v in a.items() if v["launches"]}}
    return out


def cpu_baseline(cfg, arch, S, toks_per_step, last):
    """The reference's own CPU DASH step (oracle/_ref, all host cores) on the BASELINE.md §3
    sub-batch, per phase, with a labelled extrapolation to this workload's step."""
    threads = os.cpu_count() or 1
    run, sample = ref_step_runner(cfg, threads, CPU_BASELINE_SAMPLE)
    st = run(0)
    grad_tokens = st.kept * (CPU_BASELINE_SAMPLE["prompt_len"] + st.tokens_sampled / max(st.n_seq, 1))
    out = {"value": st.tokens_sampled / st.total_s, "unit": "tokens/s", "cores": threads, "kind": "reference",
           "sample": sample, "sample_s": st.sample_s, "grad_s": st.grad_s, "adam_s": st.update_s,
           "sample_tok_s_per_core": st.tokens_sampled / st.sample_s / threads}
    if st.grad_s > 0 and grad_tokens:
        out["grad_tok_s_per_core"] = grad_tokens / st.grad_s / threads
    if cfg["size"] and out.get("grad_tok_s_per_core"):
        # this step's tokens on the reference (it re-runs each prompt per sample, policy.cpp:396)
        samp_tok = S * cfg["prompt_len"] + toks_per_step
        kept_tok = last["loss_tokens"] + last["n_kept"] * cfg["prompt_len"]
        box = threads
        est = samp_tok / (out["sample_tok_s_per_core"] * box) + kept_tok / (out["grad_tok_s_per_core"] * box)
        est += st.update_s
        out["extrapolated_step_s"] = est
        out["extrapolation"] = ("EXTRAPOLATION, not measured: this workload's sampled + prompt tokens at the "
                                "measured sample rate, kept tokens at the measured grad rate, plus one Adam step")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--prompts", type=int, default=None)
    ap.add_argument("--max-len", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tau", default=None, help="filter threshold override; 'off' = no filter (GRPO-style)")
    ap.add_argument("--sharded", action="store_true", help="ZeRO-1 style sharded optimizer step")
    ap.add_argument("--fused", action="store_true",
                    help="ZeRO-1 update fused into one peer-memory kernel (dashcu_fused_step)")
    ap.add_argument("--no-profile", action="store_true",
                    help="no kernel-class events in the timed region (decode steps replay as CUDA graphs; "
                         "no roofline / kernel_classes)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.prompts:
        cfg["prompts"] = args.prompts
    if args.max_len:
        cfg["max_len"] = args.max_len
    if args.tau is not None:
        cfg["tau"] = None if args.tau == "off" else float(args.tau)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    world, rank, local = dist_setup()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
    else:
        run_ours(args, cfg, world, rank, local)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
