// Declarations of the non-GEMM kernels (launch wrappers). Each wrapper names
// the reference computation it replaces.
#pragma once
#include "common.cuh"

namespace dashcu {

// ---- parameters / optimizer -------------------------------------------------
void init_normal_ctr(cudaStream_t s, float* w, int64_t n, double scale, uint64_t seed);
void f64_to_f32(cudaStream_t s, const double* in, float* out, int64_t n);
void f32_to_f64(cudaStream_t s, const float* in, double* out, int64_t n);
void cast_f32_bf16(cudaStream_t s, const float* in, bf16* out, int64_t n);
void fill_f32(cudaStream_t s, float* p, float v, int64_t n);
// One parameter's ascent update: SGD w + lr g, or Adam with bias
// corrections c1 = 1 - b1^t, c2 = 1 - b2^t (m, v updated in place). Shared by the replicated
// update and the fused reduce-scatter / update / all-gather kernel so both round alike.
__device__ __forceinline__ float opt_update(int kind, float wi, float gi, float* m, float* v, float lr, float b1,
                                            float b2, float eps, float c1, float c2) {
  // explicit roundings: the same bits whichever kernel inlines it
  if (kind == 0) return __fmaf_rn(lr, gi, wi);
  const float mi = __fmaf_rn(b1, *m, __fmul_rn(1.f - b1, gi));
  const float vi = __fmaf_rn(b2, *v, __fmul_rn(__fmul_rn(1.f - b2, gi), gi));
  *m = mi;
  *v = vi;
  return __fmaf_rn(lr, __fdiv_rn(__fdiv_rn(mi, c1), __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, c2)), eps)), wi);
}

// Fused reduce-scatter + update + all-gather over peer memory (dashcu_fused_step): rank
// `rank` of `world` sums its slice [off, off + len) of every rank's gradient (rank order),
// updates its master slice with its slice-sized moments and writes the new fp32 + bf16
// weights into every rank's buffers; an entry barrier (all gradients final) and an exit
// barrier (all slices written, all peer reads of this rank's gradient done) use flag words
// in every rank's memory (system-scope release / acquire, epoch-valued). Spins time out
// after ~4 s (err = 1) instead of hanging.
constexpr int kMaxFusedRanks = 8;
struct FusedStepArgs {
  int world = 1, rank = 0, kind = 1;
  int64_t off = 0, len = 0;
  float* g[kMaxFusedRanks] = {};
  float* w[kMaxFusedRanks] = {};
  bf16* wT[kMaxFusedRanks] = {};
  uint32_t* flags[kMaxFusedRanks] = {};  // rank p's flag words: [0, world) entry, [world, 2 world) exit
  float* m = nullptr;                    // this rank's slice moments
  float* v = nullptr;
  uint32_t* done = nullptr;              // this rank's block-completion counter (zero between calls)
  int* err = nullptr;
  uint32_t epoch = 0;
  float lr = 0, b1 = 0, b2 = 0, eps = 0, c1 = 1, c2 = 1;
};
void fused_step(cudaStream_t s, const FusedStepArgs& a, int grid);

// SPEC.md:329-337 (ascent). kind 0 SGD, 1 Adam. Writes the bf16 working copy if wT != null.
void optimizer_update(cudaStream_t s, int kind, float* w, const float* g, float* m, float* v, bf16* wT,
                      int64_t n, float lr, float b1, float b2, float eps, float c1, float c2);

// ---- embeddings (policy.cpp:87-92, backward :335-344) --------------------------
template <class T>
void embed_fwd(cudaStream_t s, const T* tok_emb, const T* pos_emb, const int32_t* tok, const int32_t* pos,
               int rows, int d, float* x32, T* xT);
// ---- decode rows and the paged completion KV ------------------------------
// The decode runs over its ACTIVE rows; row_seq[r] is the sequence of row r (null = identity).
// Per-sequence state (next token, prompt length, key, cap, finished flag, outputs) is indexed
// by sequence, per-row scratch (activations, logits, slice records) by row, so retiring
// finished sequences only rewrites row_seq. Completion K / V of each layer live in a pool
// of kPage-slot pages [page][kv head][kPage][hd]; page_table[seq * max_pages + i] holds
// completion slots [i kPage, (i + 1) kPage) of the sequence.
constexpr int kPage = 64;
struct DecodeRows {
  const int32_t* row_seq = nullptr;
  const int32_t* ptab = nullptr;
  int max_pages = 0;
  const int* step = nullptr;  // CUDA-graph replay: the decode step read from device memory
};
__device__ __forceinline__ int dr_seq(const DecodeRows& dr, int row) { return dr.row_seq ? dr.row_seq[row] : row; }
// element offset of completion slot `slot` of (seq, kv head) in a layer's page pool
__device__ __forceinline__ int64_t kv_slot_off(const DecodeRows& dr, int seq, int kvh, int nkv, int slot, int hd) {
  const int page = __ldg(dr.ptab + static_cast<int64_t>(seq) * dr.max_pages + slot / kPage);
  return ((static_cast<int64_t>(page) * nkv + kvh) * kPage + (slot % kPage)) * hd;
}

// decode: pos = prompt_len[seq] + step - 1, token = tok[seq], seq = row_seq[row]
template <class T>
void embed_decode(cudaStream_t s, const T* tok_emb, const T* pos_emb, const int32_t* tok,
                  const int32_t* prompt_len, int step, int rows, int d, float* x32, T* xT,
                  const int32_t* row_seq = nullptr, const int* step_dev = nullptr);
// deterministic (stable sort by id + in-order run sums); tmp: embed_bwd_tmp_bytes(rows),
// part: embed_bwd_part_floats(rows, d) floats of window partials
size_t embed_bwd_tmp_bytes(int rows);
size_t embed_bwd_part_floats(int rows, int d);
void embed_bwd(cudaStream_t s, const float* dx, const int32_t* tok, const int32_t* pos, int rows, int d, int n_tok,
               int n_pos, float* g_tok, float* g_pos, void* tmp, float* part);
// out[n] += sum_m X[m][n]  (bias gradients: db_out, db1, db2); deterministic two-pass,
// tmp holds colsum_tmp_floats<T>(M, N) floats of row-segment partials
template <class T>
size_t colsum_tmp_floats(int M, int N);
template <class T>
void colsum_acc(cudaStream_t s, const T* X, int64_t ld, int M, int N, float* out, float* tmp);
void colsum_acc_f32(cudaStream_t s, const float* X, int64_t ld, int M, int N, float* out, float* tmp);
// micro-batch packing on the device (policy.cu upload_all): one CTA per listed sequence
void pack_batch_rows(cudaStream_t s, int nseq, const int32_t* info, const float* wq, const int32_t* ptok,
                     const int32_t* comp, int max_len, int32_t* tok, int32_t* pos, int32_t* rows, int32_t* tgt,
                     int32_t* lsei, float* w);

// ---- attention (policy.cpp:105-129 forward, :292-322 backward) -------------------
// Packed variable-length causal self-attention over qkv rows [T x (qd + 2 kvd)].
template <class T>
void attn_fwd_varlen(cudaStream_t s, const T* qkv, const int32_t* seq_start, int n_seq, int max_len,
                     int nh, int nkv, int hd, T* ctx, float* lse, double alg_flops = 0);
template <class T>
void attn_bwd_varlen(cudaStream_t s, const T* qkv, const T* dctx, const float* lse, const int32_t* seq_start,
                     int n_seq, int max_len, int nh, int nkv, int hd, float* dq32, float* dkv32, double alg_flops = 0);
// Tensor-core (mma.sync) flash attention for the bf16 path; head_dim 64/128.
// Return false when the geometry is not covered (caller uses the CUDA-core kernels).
//
// Backward-consistent forward (bf16): the softmax normaliser is the sum of the bf16-ROUNDED
// probabilities the PV product consumed, and ctx_lo (optional) receives the bf16 residual
// O - bf16(O). The backward's D = dO . (ctx + ctx_lo) then equals sum_j P_ij dP_ij up to fp32
// rounding with the row's common value component cancelled exactly (in deep random-init
// policies dP_ij - D_i is a small difference, and bf16-rounded O / P would swamp it).
bool attn_fwd_tc(cudaStream_t s, const bf16* qkv, const int32_t* seq_start, int n_seq, int max_len, int rows, int nh,
                 int nkv, int hd, bf16* ctx, float* lse, double alg_flops, bf16* ctx_lo = nullptr);
// dq32 is overwritten (zeroed then accumulated), dkv32 rows are written.
bool attn_bwd_tc(cudaStream_t s, const bf16* qkv, const bf16* ctx, const bf16* dctx, const float* lse,
                 const int32_t* seq_start, int n_seq, int max_len, int rows, int nh, int nkv, int hd, float* Dbuf,
                 float* dq32, float* dkv32, double alg_flops, const bf16* ctx_lo = nullptr);
// tcgen05 forward (head_dim 64); false if not covered (DASHCU_ATTN_FWD=mma forces mma.sync)
bool attn_fwd_tc5(cudaStream_t s, const bf16* qkv, const int32_t* seq_start, int n_seq, int max_len, int rows, int nh,
                  int nkv, int hd, bf16* ctx, float* lse, bf16* ctx_lo);
// tcgen05 backward (head_dim 64): dq32 must be zero, D (Dbuf) computed; false if not covered
// (DASHCU_ATTN_BWD=mma forces the mma.sync kernel).
bool attn_bwd_tc5(cudaStream_t s, const bf16* qkv, const bf16* dctx, const float* lse, const float* Dbuf,
                  const int32_t* seq_start, int n_seq, int max_len, int rows, int nh, int nkv, int hd, float* dq32,
                  float* dkv32);
#ifdef DASHCU_ATTN_TRACE
int attn_trace_read(unsigned long long* out, int n);  // debug builds: clock64 timeline of one CTA
#endif
// qkv-gradient assembly: dqkv (T) from fp32 dq [T x qd] and dkv [T x 2 kvd]
template <class T>
void pack_dqkv(cudaStream_t s, const float* dq, const float* dkv, int rows, int qd, int kvd, T* dqkv);

// ---- decode (sampling) ------------------------------------------------------------
// Prompt KV store [L][P][nkv][Pmax][hd] (shared by the G sequences of a group) from
// prefill qkv rows; completion KV: the paged pools above (slot = completion position).
template <class T>
void kv_store_prompt(cudaStream_t s, const T* qkv, const int32_t* seq_start, int n_prompts, int pmax, int qd,
                     int kvd, int nkv, int hd, T* kstore, T* vstore);
template <class T>
void kv_append(cudaStream_t s, const T* qkv, int rows, int qd, int kvd, int nkv, int hd, int slot,
               const DecodeRows& dr, T* kpool, T* vpool);
template <class T>
void attn_decode(cudaStream_t s, const T* qkv, const T* kp, const T* vp, const T* kc, const T* vc,
                 const int32_t* prompt_len, int rows, int G, int pmax, int n_comp, int max_len, const DecodeRows& dr,
                 int nh, int nkv, int hd, T* ctx, double alg_bytes = 0);
// Tensor-core decode attention (bf16; head_dim 64/128, <= 16 query heads per KV head).
// Returns false when the geometry is not covered (caller uses attn_decode).
// append: the kernel also stores each row's new K / V (qkv) into completion slot
// n_comp - 1 (what kv_append does), so the decode step needs no separate append launch
bool attn_decode_tc_supported(int nh, int nkv, int hd);
bool attn_decode_tc(cudaStream_t s, const bf16* qkv, const bf16* kp, const bf16* vp, bf16* kc, bf16* vc,
                    const int32_t* prompt_len, int rows, int G, int pmax, int n_comp, const DecodeRows& dr, int nh,
                    int nkv, int hd, bf16* ctx, double alg_bytes, bool append);
// One sampling step over fp32 logits rows [rows x V] (policy.cpp:399-426 with the
// inverse-CDF contract of rule.cuh): per-slice partials, then sample_scan.
// part: scratch of rows * ceil(V/32) * 4 floats.
void sample_rows(cudaStream_t s, const float* logits, int rows, int V, int bos, int eos, float inv_t,
                 const uint64_t* keys, int step, const int32_t* cap, uint8_t* finished, int32_t* comp,
                 float* logp, int32_t* len, int32_t* tok_next, int max_len, float* part,
                 const int32_t* row_seq = nullptr);

// The walk's state at the chosen 32-id slice (sample_scan phase 1 -> phase 2).
struct SliceSel {
  int sb;          // chosen slice (-1: the row's sequence is not active)
  float target;    // u * total
  float sbase;     // running sum before the slice
  float ms;        // the slice's max at 1/T
  float scale;     // sexp2((m_s - M) log2e)
  float lse1;      // T = 1 log-sum-exp of the row
};
// The contract's walk over per-slice partials {m, Z, m1, Z1} (from sample_rows or the
// fused LM-head GEMM epilogue) + the token bookkeeping (EOS, cap, logp at T = 1).
// phase 0: one pass over stored fp32 logits; phase 1: down to the slice (-> sel);
// phase 2: the id walk over the slice's logits recomputed by gemm_tc_slice (logits =
// [rows x 32]); with dump != null phase 2 also counts recomputed logits that differ from
// the dumped GEMM logits (dump + row * dump_ld) into *mismatches.
void sample_scan(cudaStream_t s, const float* part, int nslices, const float* logits, int64_t logits_ld, int rows,
                 int V, int bos, int eos, float inv_t, const uint64_t* keys, int step, const int32_t* cap,
                 uint8_t* finished, int32_t* comp, float* logp, int32_t* len, int32_t* tok_next, int max_len,
                 bool compact = false,    // compact: {m, Z} records (fused epilogue at T = 1)
                 float* lse_out = nullptr,   // optional [seqs x max_len]: the row's T = 1 log-sum-exp
                 const int32_t* row_seq = nullptr,   // row -> sequence (null = identity)
                 int phase = 0, SliceSel* sel = nullptr, const float* dump = nullptr, int64_t dump_ld = 0,
                 int* mismatches = nullptr, const int* step_dev = nullptr);
// step_dev += 1 (the last node of a captured decode step)
void step_advance(cudaStream_t s, int* step_dev);
// dst[i] = src[idx[i]] (fp32 gather)
void gather_f32(cudaStream_t s, const float* src, const int32_t* idx, int n, float* dst);

// Row LSE from gemm_tc_lse partials; if logp != null also logp = logit[y] - lse.
void lse_reduce(cudaStream_t s, const float* part, int ntiles, int rows, float* lse, const bf16* Y, int d,
                const bf16* W, const float* bias, const int32_t* target, float* logp);

// ---- LM-head loss rows (policy.cpp:471-483) ------------------------------------------
// For each loss row r: lse over non-BOS logits; logp[r] = logit[y_r] - lse;
// if dz != null: dz[r][i] = w_r * (onehot(y_r) - softmax)_i, BOS column 0.
template <class T>
void lm_rows(cudaStream_t s, const float* logits, int rows, int V, int bos, const int32_t* target,
             const float* weight, float* logp, T* dz);

// PPO: per-sequence ratio from the per-row log-probs, clipped-surrogate
// gradient weight broadcast to the sequence's rows; stats [nseq x 3] {rho, clipped, term}.
void ppo_weights(cudaStream_t s, const float* logp, const int32_t* row_start, int nseq, const double* old_lp,
                 const double* adv, double eps, float* w, double* stats);

// KL term rows (kl_term, policy.cpp:487-522): value[r] = KL(base || current) at row r (fp64),
// dz[r] = w_r (softmax(lc) - softmax(lb)), BOS column 0; dz may be null.
template <class T>
void kl_rows(cudaStream_t s, const float* lc, const float* lb, int rows, int V, int bos, const float* weight,
             double* value, T* dz);

// ---- gathers ---------------------------------------------------------------------------
template <class T>
void gather_rows(cudaStream_t s, const T* src, int64_t ld_src, const int32_t* idx, int rows, int width, T* dst);
void scatter_rows_f32(cudaStream_t s, const float* src, int rows, int width, const int32_t* idx, float* dst);

// ---- advantage + filter (advantage.cpp:67-140) -------------------------------------------
void advantage_filter(cudaStream_t s, const double* r, int n, int G, int kind, int normalize, double eps,
                      double tau, double* adv, uint8_t* kept, int32_t* kept_idx, int32_t* n_kept);

}  // namespace dashcu
