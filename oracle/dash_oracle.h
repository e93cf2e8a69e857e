/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product.
 *
 * A plain-C, fp64 restatement of the reference's DASH-step algorithm
 * (/root/reference/proj, SPEC.md) plus the four contracts the reference lacks
 * (SURVEY §8c "CPU restatements required"):
 *   1. PG accumulate          sum_kept (A_n / N) * grad log pi   (App.B D4)
 *   2. Adam / SGD             SPEC:329-337 (ascent)
 *   3. Sampling               inverse-CDF counter-RNG contract of DESIGN.md §4 (App.B D2)
 *   4. GQA geometry           (n_heads, n_kv_heads, head_dim); (1, 1, d) is the reference
 * Parity pin: at GQA (1,1,d) the forward is evaluated in the reference's
 * operation order, so log-probs equal oracle/_ref bit-for-bit; gradients are
 * checked at <=1e-12 relative (tests/test_oracle.py).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may load it.
 */
#ifndef DASH_ORACLE_H
#define DASH_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ArchConfig (reference tensors.hpp:13-24) + GQA extension. */
typedef struct {
  int32_t vocab_size, embed_dim, context_len, ffn_hidden, n_layers, bos_id, eos_id;
  int32_t n_heads, n_kv_heads, head_dim; /* 0,0,0 -> 1,1,embed_dim (the reference) */
} dor_arch;

/* ---- rng.hpp:10-82 ---- */
uint64_t dor_splitmix64(uint64_t x);
uint64_t dor_fnv1a(const char* s);
uint64_t dor_derive_seed(uint64_t base, const char* tag, uint64_t a, uint64_t b);
/* mt19937_64 draws: kind 0 next_u64, 1 uniform01 bits, 2 normal bits (Marsaglia polar) */
void dor_rng_draws(uint64_t seed, int kind, int n, uint64_t* out);

/* ---- tensors.cpp ---- */
int64_t dor_num_params(const dor_arch* a);
/* byte offsets are not used; element offsets into the flat views() buffer */
typedef struct {
  int64_t token_embed, pos_embed, w_out, b_out, total;
  int64_t layer0, layer_stride; /* layer l base = layer0 + l*layer_stride */
  int64_t wq, wk, wv, wo, w1, b1, w2, b2; /* offsets relative to a layer base */
} dor_layout;
void dor_layout_of(const dor_arch* a, dor_layout* out);
/* PolicyParams::init (tensors.cpp:150-158): N(0, scale^2) in views() order */
void dor_init_params(const dor_arch* a, double scale, uint64_t seed, double* out);
/* counter-based init restated from the device kernel */
void dor_init_params_ctr(const dor_arch* a, double scale, uint64_t seed, double* out);

/* ---- policy.cpp ---- */
/* log_prob (policy.cpp:362-377); returns total, fills per_token[len] */
double dor_log_prob(const dor_arch* a, const double* params, const int32_t* prompt, int m,
                    const int32_t* completion, int len, double* per_token);
/* next-position logits after `ctx` (advance + LM head, policy.cpp:80-153) */
void dor_next_logits(const dor_arch* a, const double* params, const int32_t* ctx, int n,
                     double* logits);
/* grad += scale * grad_log_prob (policy.cpp:463-485 + backward :201-346) */
void dor_grad_log_prob_acc(const dor_arch* a, const double* params, const int32_t* prompt, int m,
                           const int32_t* completion, int len, double scale, double* grad);
/* kl_term (policy.cpp:487-522) with GQA geometry: KL(base || current) over the completion
 * positions (returned); grad += scale * d/dP of it. */
double dor_kl_term_acc(const dor_arch* a, const double* P, const double* base, const int32_t* prompt, int m,
                       const int32_t* completion, int len, double scale, double* grad);

/* ---- sampling contract (App.B D2) ---- */
float dor_soft_logf(float x);
uint32_t dor_row_key(uint64_t seq_key, int32_t step);
float dor_gumbel(uint32_t row_key, int32_t token);
/* The sampling contract: inverse CDF over exp(logit/T - max) (BOS excluded) with the
 * sums organised in 32-id slices and 32 slice blocks, software exp2 (dor_sexp2) and
 * u = (2*(row_key >> 9) + 1) * 2^-24. */
int32_t dor_sample_rule(const float* logits, int vocab, int bos, float inv_t, uint64_t seq_key,
                        int32_t step);
float dor_sexp2(float x);
/* Gumbel-max over the same counter RNG (an independent alternative rule, tests only). */
int32_t dor_sample_rule_gumbel(const float* logits, int vocab, int bos, float inv_t, uint64_t seq_key,
                               int32_t step);
/* Full-trajectory sampler: fp64 forward, logits rounded to fp32, then the rule.
 * cap = min(max_len, ctx - m); stops at EOS (policy.cpp:387, :425).
 * logp[j] = log softmax at T=1 (fp64). Returns completion length. */
int dor_sample(const dor_arch* a, const double* params, const int32_t* prompt, int m, int max_len,
               double temperature, uint64_t seq_key, int32_t* completion, double* logp);

/* ---- advantage.cpp ---- */
/* kind 0 single_path (:67-78), 1 group (:80-94), 2 leave_one_out (:96-112).
 * normalize: normalize_std (:114-133). kept = |A| > tau (:135-140).
 * kept_idx: ascending compaction of kept. Returns 0 ok, 1 input error. */
int dor_advantage_filter(const double* rewards, int n, int group_size, int kind, int normalize,
                         double eps, double tau, double* adv, uint8_t* kept, int32_t* kept_idx,
                         int32_t* n_kept);

/* ---- updates ---- */
/* grad += sum_i weight[i] * grad log pi(traj_i); trajectories packed:
 * prompts[p_off[i]..p_off[i+1]), completions[c_off[i]..c_off[i+1]) */
void dor_pg_accumulate(const dor_arch* a, const double* params, int n_traj, const int32_t* prompts,
                       const int64_t* p_off, const int32_t* completions, const int64_t* c_off,
                       const double* weight, double* grad);
/* Adam ascent: t is the 1-based step after increment */
void dor_adam_step(double* p, const double* g, double* m, double* v, int64_t n, int64_t t, double lr,
                   double b1, double b2, double eps);
void dor_sgd_step(double* p, const double* g, int64_t n, double lr);

/* ---- synthetic workload ---- */
double dor_synthetic_reward(uint64_t reward_seed, int64_t m, int32_t g);
void dor_synthetic_prompt(uint64_t seed, int64_t m, int len, int vocab, int bos, int eos,
                          int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
