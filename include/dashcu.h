/*
 * dashcu.h — the C ABI of the B200-native DASH training step (libdashcu.so).
 *
 * This is the drop-in boundary for the DASH hot path of arXiv 2505.17218
 * (SURVEY.md §8b). Every entry point names the reference interface it
 * replaces (paths under /root/reference/proj unless marked SPEC.md):
 *
 *   dashcu_policy_*          ParamTensors / PolicyParams      include/dash/tensors.hpp:13-82
 *   dashcu_sample            preemptive_sample
 *                            (batched dash::sample)           src/policy.cpp:379-429
 *   dashcu_rollout_log_prob  dash::log_prob                   src/policy.cpp:362-377
 *   dashcu_advantage_filter  group_advantage / normalize_std  src/advantage.cpp:80-133
 *                            filter_by_threshold              src/advantage.cpp:135-140
 *   dashcu_accumulate        pg_gradient + run_schedule(DASH) SPEC.md:284-292, :320-323
 *                            (sum of A_n * grad_log_prob      src/policy.cpp:463-485,
 *                             via add_scaled)                 src/tensors.cpp:109-115)
 *   dashcu_allreduce_grads   map-reduce over trajectories
 *   dashcu_optimizer_step    optimizer_step
 *
 * Conventions
 *  - Plain C types only; the caller owns every host buffer passed in, handles
 *    own all device memory. No device pointer escapes.
 *  - Status codes mirror include/dash/errors.hpp:10-23:
 *      0 ok, 1 InputError, 2 CapacityError, 3 OnPolicyViolation, 4 device (CUDA/NCCL).
 *    Validation happens on the host before any launch, so the error class
 *    matches the reference's throw sites (policy.cpp:183-197, :381-386;
 *    advantage.cpp:10-41, :136). dashcu_last_error() is thread-local.
 *  - Flat parameter / gradient buffers are fp64 in ParamTensors::views()
 *    order (tensors.cpp:49-71), extended with the GQA geometry below.
 *  - One dashcu_ctx per GPU, used from one host thread; calls are
 *    stream-ordered and return once their host outputs are written.
 *  - There is no CPU fallback: without an sm_100 device every entry point
 *    that computes returns 4.
 */
#ifndef DASHCU_H
#define DASHCU_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DASHCU_API __attribute__((visibility("default")))
#else
#define DASHCU_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DASHCU_OK 0
#define DASHCU_E_INPUT 1
#define DASHCU_E_CAPACITY 2
#define DASHCU_E_ON_POLICY 3
#define DASHCU_E_DEVICE 4

/* compute dtype of a policy */
#define DASHCU_F32 0  /* parity mode: fp32 weights/activations, CUDA-core GEMMs */
#define DASHCU_BF16 1 /* production: bf16 operands, tcgen05 GEMMs, fp32 master/grads */

/* advantage estimators (advantage.hpp:36-45) */
#define DASHCU_ADV_SINGLE_PATH 0 /* single_path_advantage  advantage.cpp:67-78 */
#define DASHCU_ADV_GROUP 1       /* group_advantage        advantage.cpp:80-94 */
#define DASHCU_ADV_LEAVE_ONE_OUT 2 /* leave_one_out        advantage.cpp:96-112 */
#define DASHCU_ADV_GIVEN 3         /* advantages passed in `adv` (in/out): normalize_std
                                      (advantage.cpp:114-133) and/or filter_by_threshold only */

/* tau value meaning "no filter_by_threshold" (GRPO-style baseline):
 * every sequence is kept, as group_advantage leaves AdvantageBatch::kept
 * (advantage.cpp:92). Any other tau < 0 is an InputError (advantage.cpp:136). */
#define DASHCU_FILTER_OFF (-__builtin_inf())

/* optimizers */
#define DASHCU_OPT_SGD 0
#define DASHCU_OPT_ADAM 1

typedef struct dashcu_ctx dashcu_ctx;
typedef struct dashcu_policy dashcu_policy;

/* ArchConfig (tensors.hpp:13-24) + GQA geometry extension (SURVEY App.B D1).
 * n_heads = n_kv_heads = head_dim = 0 means (1, 1, embed_dim): the reference. */
typedef struct {
  int32_t vocab_size, embed_dim, context_len, ffn_hidden, n_layers, bos_id, eos_id;
  int32_t n_heads, n_kv_heads, head_dim;
} dashcu_arch;

/* SamplingPlan. Prompt m of this call is the global prompt
 * prompt_index_base + m, so per-request keys derive_seed(round_seed, "sample",
 * m_global, g) are independent of how prompts are sharded. */
typedef struct {
  int32_t n_prompts, group_size, max_len;
  double temperature;
  uint64_t round_seed;
  int64_t prompt_index_base;
} dashcu_plan;

typedef struct {
  int32_t kind; /* DASHCU_OPT_* */
  double lr, beta1, beta2, eps;
} dashcu_opt;

typedef struct {
  double sample_ms, advantage_ms, accumulate_ms, allreduce_ms, optimizer_ms;
  int64_t tokens_sampled;   /* completion tokens of the last dashcu_sample */
  int32_t n_seq, n_kept;    /* rollout size, kept after the filter */
  int64_t loss_tokens;      /* completion tokens that entered the last accumulate */
  double mean_reward, filtered_fraction, mean_abs_kept; /* advantage.cpp:44-65 */
  int64_t kernel_launches;  /* kernels this policy launched since creation */
  int64_t decode_row_steps; /* sum over the last rollout's decode steps of the active rows */
  int64_t kv_pages_peak;    /* most completion-KV pages (per layer) in use at once */
  int64_t slice_recompute_mismatches; /* logits dump on: recomputed slice logits != the dump (0) */
} dashcu_stats;

DASHCU_API const char* dashcu_last_error(void);
DASHCU_API int dashcu_abi_version(void);

/* ---- context (one per GPU) ---- */
DASHCU_API int dashcu_ctx_create(int device, dashcu_ctx** out);
DASHCU_API int dashcu_ctx_destroy(dashcu_ctx* ctx);
DASHCU_API int dashcu_ctx_sync(dashcu_ctx* ctx);
/* NCCL communicator for the gradient allreduce (one per optimizer step). */
DASHCU_API int dashcu_comm_unique_id(uint8_t out[128]);
DASHCU_API int dashcu_ctx_init_comm(dashcu_ctx* ctx, int world, int rank, const uint8_t id[128]);

/* ---- policy parameters (tensors.hpp:50-82) ---- */
DASHCU_API int dashcu_arch_num_params(const dashcu_arch* arch, int64_t* n);
DASHCU_API int dashcu_policy_create(dashcu_ctx* ctx, const dashcu_arch* arch, int dtype, dashcu_policy** out);
DASHCU_API int dashcu_policy_destroy(dashcu_policy* pol);
/* PolicyParams <-> device, fp64 flat views() order. Upload bumps the snapshot version. */
DASHCU_API int dashcu_policy_upload(dashcu_policy* pol, const double* params, int64_t n);
DASHCU_API int dashcu_policy_download(dashcu_policy* pol, double* params, int64_t n);
/* Device counter-based N(0, scale^2) init for shapes where a
 * host PolicyParams::init is impractical; restated in oracle/. */
DASHCU_API int dashcu_policy_init_normal(dashcu_policy* pol, double scale, uint64_t seed);
DASHCU_API int dashcu_policy_version(dashcu_policy* pol, uint64_t* version);

/* ---- preemptive sampling (policy.cpp:379-429) ----
 * Samples group_size completions for each prompt (prompt_offsets[n_prompts+1]
 * into prompt_tokens). Sequence s = m*G + g. Outputs (each may be NULL):
 *   completions [n_seq*max_len] (row s: tokens, unused tail = -1)
 *   lengths     [n_seq]
 *   logp        [n_seq*max_len]  per-token log-probs at T=1 (trajectory.hpp:8-9)
 * Sampling rule: inverse CDF over fp32 logits organised in 32-id slices, one
 * counter-RNG draw per step (the reference's fp64 cumsum +
 * mt19937 stream cannot be replayed on a GPU, SURVEY App.B D2). The rollout stays resident for accumulate. */
DASHCU_API int dashcu_sample(dashcu_policy* pol, const dashcu_plan* plan, const int32_t* prompt_tokens,
                  const int64_t* prompt_offsets, int32_t* completions, int32_t* lengths, float* logp);
/* Same with explicit per-sequence keys (seq_keys[n_prompts*group_size]) instead of
 * derive_seed(round_seed, "sample", m, g): the per-trajectory form of
 * dash::sample(params, prompt, max_len, T, seed) (policy.cpp:379) with key = seed. */
DASHCU_API int dashcu_sample_keyed(dashcu_policy* pol, const dashcu_plan* plan, const int32_t* prompt_tokens,
                                   const int64_t* prompt_offsets, const uint64_t* seq_keys, int32_t* completions,
                                   int32_t* lengths, float* logp);
/* Debug: when enabled, the next dashcu_sample also records the exact fp32
 * logits its sampling rule consumed, [n_seq][max_len][vocab] (small shapes). */
DASHCU_API int dashcu_set_logits_dump(dashcu_policy* pol, int enable);
/* Cap of the decode's completion-KV page pool: n_pages pages of 64 slots per layer (each
 * page n_kv_heads x 64 x head_dim K and V values). 0 (default) = the round's worst case
 * (every sequence at max_len); a smaller pool relies on sequences finishing early (their
 * pages are recycled) and fails with CapacityError when exhausted. */
DASHCU_API int dashcu_set_kv_pages(dashcu_policy* pol, int64_t n_pages);
DASHCU_API int dashcu_get_logits_dump(dashcu_policy* pol, float* out, int64_t n);

/* Load externally produced trajectories as the rollout (n_prompts*group_size
 * sequences; completion s = completions[completion_offsets[s] .. [s+1])).
 * Validates like validate_traj (policy.cpp:191-197). */
DASHCU_API int dashcu_rollout_load(dashcu_policy* pol, const int32_t* prompt_tokens, const int64_t* prompt_offsets,
                        int32_t n_prompts, int32_t group_size, const int32_t* completions,
                        const int64_t* completion_offsets);
/* Teacher-forced per-token log-probs of the rollout (log_prob, policy.cpp:362-377),
 * concatenated over sequences in rollout order (n_tokens = sum of lengths). */
DASHCU_API int dashcu_rollout_log_prob(dashcu_policy* pol, float* per_token, int64_t n_tokens);

/* ---- advantage + gradient filter ----
 * Host-buffer form (advantage.cpp:80-140): adv[n], kept[n], kept_idx = ascending
 * compaction of kept, n_kept. kind = DASHCU_ADV_*; normalize = normalize_std. */
DASHCU_API int dashcu_advantage_filter(dashcu_ctx* ctx, const double* rewards, int32_t n, int32_t group_size,
                            int32_t kind, int32_t normalize, double eps, double tau, double* adv,
                            uint8_t* kept, int32_t* kept_idx, int32_t* n_kept);
/* Device-resident form on the current rollout: rewards in, advantages and the
 * compacted kept list stay on device for dashcu_accumulate. Outputs may be NULL. */
DASHCU_API int dashcu_rollout_set_rewards(dashcu_policy* pol, const double* rewards, int32_t n);
DASHCU_API int dashcu_rollout_advantage(dashcu_policy* pol, int32_t kind, int32_t normalize, double eps, double tau,
                             double* adv, uint8_t* kept, int32_t* n_kept);

/* ---- micro-batched policy-gradient accumulation ----
 * grad += sum over kept n of (A_n * weight_scale) * grad log pi(traj_n), in
 * micro-batches of micro_batch sequences (0 = all at once). DASH uses
 * weight_scale = 1/N with N the round's pre-filter count (App.B D4).
 * Raises OnPolicyViolation if the policy changed since the rollout was made. */
DASHCU_API int dashcu_grad_zero(dashcu_policy* pol);
DASHCU_API int dashcu_accumulate(dashcu_policy* pol, double weight_scale, int32_t micro_batch);
/* Same with explicit per-sequence weights (weights[n_seq], all sequences). */
DASHCU_API int dashcu_accumulate_weighted(dashcu_policy* pol, const double* weights, int32_t n_seq,
                               int32_t micro_batch);
/* ---- PPO surrogate, KL term, update schedules (policy.cpp:487-522) ----
 * dashcu_rollout_snapshot records theta_old for the current rollout: every sequence's
 * summed teacher-forced log-prob under the current weights (call it at schedule entry,
 * right after sampling). dashcu_accumulate_ppo then adds the gradient of the clipped
 * surrogate mean over the kept sequences (intersected with subset[n_subset], null = all):
 *   sum_n weight_scale * grad min(rho_n A_n, clip(rho_n, 1-eps, 1+eps) A_n),
 *   rho_n = exp(sum_j log pi(y_nj) - sum_j log pi_old(y_nj))   (sequence level),
 * which is weight_scale * A_n rho_n grad log pi on the unclipped branch and 0 on the clipped
 * one; the weights may differ from the snapshot (no OnPolicyViolation). At theta ==
 * theta_old rho is exactly 1 and the gradient equals dashcu_accumulate's. surrogate = the
 * sum of the scaled surrogate terms, n_clipped = items on the clipped branch (both optional). */
DASHCU_API int dashcu_rollout_snapshot(dashcu_policy* pol);
DASHCU_API int dashcu_rollout_snapshot_logp(dashcu_policy* pol, double* per_seq, int32_t n_seq);
DASHCU_API int dashcu_accumulate_ppo(dashcu_policy* pol, double weight_scale, double clip_eps, int32_t micro_batch,
                                     const int32_t* subset, int32_t n_subset, double* surrogate, int32_t* n_clipped);
/* grad += coef * sum over the listed sequences (subset, null = all) of grad_theta of the
 * reference's kl_term(params, base, traj) (exact per-token KL(base || current), policy.cpp:
 * 487-522); kl_per_seq[k] (optional) = its value. base: same context, arch and dtype. */
DASHCU_API int dashcu_accumulate_kl(dashcu_policy* pol, dashcu_policy* base, double coef, int32_t micro_batch,
                                    const int32_t* subset, int32_t n_subset, double* kl_per_seq);

#define DASHCU_SCHED_DASH 0  /* one update from the PG gradient over the whole batch */
#define DASHCU_SCHED_MULTI 1 /* K updates, each from the PPO gradient over the whole batch */
#define DASHCU_SCHED_MINI 2  /* K updates, the k-th from the PPO gradient of mini-batch k */
typedef struct {
  int32_t kind;        /* DASHCU_SCHED_* */
  int32_t K;           /* MULTI: steps per snapshot; MINI: mini-batches (n_seq % K == 0) */
  double clip_eps;     /* PPO clip range (<= 0: the SPEC default 0.2) */
  double beta;         /* KL weight (0: No-KL, the DASH preset) */
  double weight_scale; /* 1/N, N the round's pre-filter size; MINI scales it by K (mean per mini-batch) */
  int32_t micro_batch;
  int32_t sharded;     /* 1: dashcu_sharded_step instead of allreduce + optimizer_step */
} dashcu_schedule;
typedef struct {
  double surrogate;         /* PPO: sum of the scaled surrogate terms (0 for DASH) */
  double kl;                /* beta > 0: scaled sum of the KL values */
  double clip_fraction;     /* PPO: items on the clipped branch / items */
  double mean_abs_adv;      /* mean |A| over the kept items (advantage.cpp:44-65) */
  double filtered_fraction; /* 1 - kept / n */
  int32_t n_items;          /* items this update's gradient covered */
  double ms;                /* wall time of the update */
} dashcu_step_log;
/* run_schedule over the current rollout and advantage batch: DASH = one
 * accumulate + (allreduce) + optimizer step; MULTI / MINI snapshot theta_old first (the
 * policy must not have changed since sampling), then K PPO updates. beta > 0 adds
 * -beta * grad KL(base || current) over the same items (J = J_inner - beta KL). logs[k]
 * for k < max_logs; n_logs = the number of updates. */
DASHCU_API int dashcu_run_schedule(dashcu_policy* pol, const dashcu_schedule* sched, const dashcu_opt* opt,
                                   dashcu_policy* base, dashcu_step_log* logs, int32_t max_logs, int32_t* n_logs);

/* ---- post-filter rebalancing across ranks ----
 * After dashcu_rollout_advantage each rank holds a different number of kept sequences
 * (advantage.cpp:135-140). dashcu_rebalance moves kept sequences (prompt, completion,
 * advantage and the sampler's log-sum-exp rows) between ranks over NCCL so every rank's
 * accumulate covers about the same number of tokens; the next dashcu_accumulate then runs
 * over this rank's new kept set with the same global weight_scale, so the all-reduced
 * gradient is unchanged up to summation order. Collective (every rank calls it); no-op at
 * world 1. n_out / n_in: sequences sent / received. dashcu_rebalance_plan is the pure
 * planner every rank runs on the all-gathered costs: n_items[world], costs (concatenated
 * per rank, e.g. prompt + completion tokens) -> dest (the rank that accumulates each item). */
DASHCU_API int dashcu_rebalance(dashcu_policy* pol, int32_t* n_out, int32_t* n_in);
DASHCU_API int dashcu_rebalance_plan(int32_t world, const int32_t* n_items, const int64_t* costs, int32_t* dest);

DASHCU_API int dashcu_grad_download(dashcu_policy* pol, double* grad, int64_t n);
/* Replace the device gradient (fp64 views() order), e.g. a GradientVector computed elsewhere. */
DASHCU_API int dashcu_grad_upload(dashcu_policy* pol, const double* grad, int64_t n);
/* Sum gradients over the ranks of the context's communicator (no-op at world 1). */
DASHCU_API int dashcu_allreduce_grads(dashcu_policy* pol);
/* Ascent step on the fp32 master weights; refreshes the bf16 copy; bumps the version. */
DASHCU_API int dashcu_optimizer_step(dashcu_policy* pol, const dashcu_opt* opt);
/* ZeRO-1 style alternative to allreduce_grads + optimizer_step (the paper
 * trains with ZeRO): reduce-scatter the gradient, update only this rank's
 * slice [off, off+len) of the fp32 master weights with slice-sized Adam moments,
 * all-gather the master and refresh the bf16 copy. A policy uses one form or the other
 * for its whole life (InputError otherwise). After it the gradient buffer is valid only
 * on this rank's slice. */
DASHCU_API int dashcu_sharded_step(dashcu_policy* pol, const dashcu_opt* opt);
/* The same update as ONE kernel per rank over NVLink peer memory (the
 * optimizer fused into the collective): the ranks' gradient / fp32 master / bf16 buffers
 * are shared once through CUDA IPC (handles all-gathered over the communicator); the kernel
 * sums this rank's slice of every rank's gradient (rank order), updates it with the
 * slice-sized moments, and writes the new master + bf16 values into every rank's buffers,
 * between an entry and an exit barrier of system-scope flags (status 4 on a timeout).
 * Shares the moment layout of dashcu_sharded_step (the two may be mixed); world 1 runs
 * the same kernel on the local buffers. At most 8 ranks. */
DASHCU_API int dashcu_fused_step(dashcu_policy* pol, const dashcu_opt* opt);
/* The slice of a `total`-element flat vector rank `rank` of `world` owns in the sharded
 * step (no device work). */
DASHCU_API int dashcu_shard_span(int64_t total, int32_t world, int32_t rank, int64_t* off, int64_t* len);

/* ---- checkpoint container ----
 * Flat named-tensor file: "DASHCKPT", version 1, the dashcu_arch descriptor, tensor count,
 * flags (bit 0: Adam state), Adam step count, the reference's content_hash
 * (tensors.cpp:95-107), then per tensor {name, shape, row-major f64 data} in the views()
 * order and names of tensors.cpp:49-71, optionally followed by "adam.m" / "adam.v". Save
 * writes the fp32 master weights exactly (as f64); load checks the architecture, names,
 * shapes and hash (InputError otherwise), restores the master + bf16 copy (and, with
 * with_optimizer, the Adam moments and step count) and bumps the policy version. */
DASHCU_API int dashcu_policy_save(dashcu_policy* pol, const char* path, int32_t with_optimizer);
DASHCU_API int dashcu_policy_load(dashcu_policy* pol, const char* path, int32_t with_optimizer);
DASHCU_API int dashcu_checkpoint_arch(const char* path, dashcu_arch* out);

DASHCU_API int dashcu_get_stats(dashcu_policy* pol, dashcu_stats* out);

/* ---- kernel-class profiler (bench.py roofline) ----
 * Enabled classes (bit i = class i: 0 gemm_tc, 1 gemm_simt, 2 attn_decode,
 * 3 attn_fwd, 4 attn_bwd, 5 sample, 6 lm_rows, 7 optimizer) have every launch
 * bracketed by CUDA events on its stream and charged with its algorithmic
 * flops / bytes. dashcu_profile_read returns one entry per class. */
typedef struct {
  char name[32];
  int64_t launches;
  double ms, flops, bytes;
} dashcu_kprof;
DASHCU_API int dashcu_profile_enable(unsigned class_mask);
/* Bracket only one launch in `period` (>= 1, default 1) of each enabled class with events
 * (the rest are counted): profile_read then reports the sampled time / flops / bytes
 * scaled to the class totals, at a fraction of the event overhead. */
DASHCU_API int dashcu_profile_sampling(int period);
DASHCU_API int dashcu_profile_read(dashcu_kprof* out, int max, int reset);
/* With bit 31 of the class mask set, launches are also aggregated per key (kernel
 * variant + shape). Text, one line per key: "class key\tlaunches\tms\tflops\tbytes".
 * Returns the full length; copies at most cap-1 bytes + NUL. Reset with profile_read. */
DASHCU_API int64_t dashcu_profile_keys(char* buf, int64_t cap);

/* ---- synthetic verifiable tasks (host only; tasks.cpp:105-175) ----
 * generate_instance / reward of the reference's task module: the prompt feeder and the
 * trajectory reward of a DASH round. kind: DASHCU_TASK_*; vocab:
 * DASHCU_VOCAB_TASK (the task's own vocabulary, build_vocab tasks.cpp:23-53) or
 * DASHCU_VOCAB_BYTE (BASELINE configs[0]: 0 "<s>", 1 "</s>", ids 2..255 the bytes).
 * Errors: InputError for difficulty < 1 (TaskSpec::make), CapacityError for a short buffer. */
#define DASHCU_TASK_ADD 0
#define DASHCU_TASK_MOD 1
#define DASHCU_TASK_REVERSE 2
#define DASHCU_TASK_PARITY 3
#define DASHCU_TASK_MICRO 4
#define DASHCU_VOCAB_TASK 0
#define DASHCU_VOCAB_BYTE 1
DASHCU_API int dashcu_task_vocab_size(int32_t kind, int32_t vocab, int32_t* size);
/* n instances, seeds[i] = the instance seed (generate_instance(task, seed)); prompts
 * concatenated (BOS first) into prompt_tokens[prompt_cap] with prompt_offsets[n+1]
 * (prompt_tokens may be null to size the buffer); answers (optional) NUL-terminated,
 * answer_stride bytes apart. */
DASHCU_API int dashcu_task_instances(int32_t kind, int32_t difficulty, int32_t vocab, const uint64_t* seeds,
                                     int32_t n, int32_t* prompt_tokens, int64_t prompt_cap, int64_t* prompt_offsets,
                                     char* answers, int32_t answer_stride);
/* reward (tasks.cpp:155-175) of sequence s = m * group_size + g, whose completion is
 * completions[s * stride .. + lengths[s]), against instance seeds[m]. */
DASHCU_API int dashcu_task_rewards(int32_t kind, int32_t difficulty, int32_t vocab, const uint64_t* seeds,
                                   int32_t n_prompts, int32_t group_size, const int32_t* completions, int32_t stride,
                                   const int32_t* lengths, double* rewards);
/* Rewards of the policy's current rollout ("rewards on arrival") from the
 * task: same as dashcu_task_rewards + dashcu_rollout_set_rewards. */
DASHCU_API int dashcu_rollout_task_rewards(dashcu_policy* pol, int32_t kind, int32_t difficulty, int32_t vocab,
                                           const uint64_t* seeds);

/* ---- kernel-variant knobs (tests and same-box A/B tools) ----
 * Read once from DASHCU_<NAME> environment variables at library load; this call changes
 * one for the calling process (INT32_MIN restores the default). Names: GEMM_PAIR,
 * GEMM_RASTER, NO_SPLITK, NO_TMA_STORE, GEMM_RESID_DB, GEMM_RESID_DEEP, ATTN_FWD,
 * ATTN_BWD, ATTN_BWD_CHUNK, LSE_RECOMPUTE, PDL, DECODE_GRAPH, DECODE_COMPACT (csrc/common.cuh Knob).
 * Returns the previous value, INT32_MIN for an unknown name. */
DASHCU_API int dashcu_set_knob(const char* name, int value);

/* ---- diagnostics (used by the kernel tests) ----
 * dashcu_selftest_fused_step: `world` virtual ranks on this GPU, each a full replica
 * (gradient g_all[r * n ..], master w0, bf16 copy, flags, slice moments) running the fused
 * kernel on its own stream concurrently, `steps` times (Adam bias corrections per step);
 * w_out / wT_out receive every replica's master and bf16 weights [world x n]. */
DASHCU_API int dashcu_selftest_fused_step(dashcu_ctx* ctx, int32_t world, int64_t n, int32_t kind, double lr,
                                          int32_t steps, const float* g_all, const float* w0, float* w_out,
                                          uint16_t* wT_out);
/* dashcu_selftest_gemm:
 * C[M x N] (fp32, ldc = N) = A(m,k) . B(n,k) on bf16 operands given as raw
 * bit patterns, through the production GEMM dispatcher (tcgen05 when the
 * operands are TMA-legal) or, with force_simt, the CUDA-core kernel.
 * epi: 0 store, 1 tanh(acc + bias), 3 C += acc, 4 C = acc + bias + C (residual). */
DASHCU_API int dashcu_selftest_gemm(dashcu_ctx* ctx, int M, int N, int K, const uint16_t* A, int64_t lda,
                                    int a_kmajor, const uint16_t* B, int64_t ldb, int b_kmajor, const float* bias,
                                    int epi, int force_simt, float* C);
/* Timing harness: `iters` launches of the production GEMM on device-resident random
 * bf16 operands, bf16 output (epi 0) or fp32 accumulate (epi 3); mean ms per launch
 * from CUDA events on the context stream; epi 4 adds an fp32 residual input and fp32 output. */
DASHCU_API int dashcu_selftest_gemm_timed(dashcu_ctx* ctx, int M, int N, int K, int a_kmajor, int b_kmajor, int epi,
                                          int iters, double* ms);
/* Attention timing harness: packed causal attention over n_seq sequences of seq_len tokens
 * (random bf16 q/k/v, nh / nkv heads of head_dim hd), forward (which 0) or backward incl.
 * its D / zeroing prologue (which 1); best of `iters` launches in ms (CUDA events). */
DASHCU_API int dashcu_selftest_attn_timed(dashcu_ctx* ctx, int n_seq, int seq_len, int nh, int nkv, int hd, int which,
                                          int iters, double* ms);
/* Whole-library count of kernel launches (all policies, all contexts). */
DASHCU_API int64_t dashcu_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* DASHCU_H */
