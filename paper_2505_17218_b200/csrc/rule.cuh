// The sampling contract (SURVEY App.B D2), device side.
//
// Reference rule (policy.cpp:399-425): inverse CDF over an fp64 cumulative sum
// with a per-trajectory mt19937_64 — inherently sequential over the vocab and
// not replayable bit-for-bit on a GPU. The B200 rule is Gumbel-max with a
// counter RNG, so every (sequence, step, token) draw is independent and the
// argmax fuses into the LM-head epilogue:
//
//   seq_key  = derive_seed(round_seed, "sample", m_global, g)      (rng.hpp:29-35)
//   row_key  = hi32(splitmix64(seq_key + 0x9e3779b97f4a7c15 * (step + 1)))
//   h        = fmix32(fmix32(token * 0x9e3779b1 ^ row_key) + 0x7f4a7c15 + row_key)
//   u        = (2 * (h >> 9) + 1) * 2^-24                 in (0, 1), exact in fp32
//   gumbel   = -soft_log(-soft_log(u))
//   score    = fmaf(logit, 1/T, gumbel)                   BOS excluded
//   token    = argmax score, ties to the lowest id
//
// soft_log is a fixed sequence of single-rounding fp32 operations, so the CPU
// restatement (oracle/dash_oracle.c dor_sample_rule) reproduces every score
// bit-for-bit from the same fp32 logits ("bit-exact under a shared logits dump").
#pragma once
#include <stdint.h>

namespace dashcu {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ float soft_logf(float x) {
  const uint32_t bits = __float_as_uint(x);
  int e = static_cast<int>((bits >> 23) & 0xffu) - 127;
  float mant = __uint_as_float((bits & 0x7fffffu) | 0x3f800000u);
  if (mant > 1.41421356f) {
    mant = __fmul_rn(mant, 0.5f);
    e += 1;
  }
  const float f = __fsub_rn(mant, 1.0f);
  const float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
  const float z = __fmul_rn(s, s);
  float p = __fmaf_rn(z, 0.11111111f, 0.14285715f);
  p = __fmaf_rn(z, p, 0.2f);
  p = __fmaf_rn(z, p, 0.33333334f);
  p = __fmaf_rn(z, p, 1.0f);
  const float r = __fmul_rn(__fmul_rn(2.0f, s), p);
  return __fmaf_rn(static_cast<float>(e), 0.6931472f, r);
}

__host__ __device__ __forceinline__ uint32_t row_key(uint64_t seq_key, int32_t step) {
  return static_cast<uint32_t>(
      splitmix64(seq_key + 0x9e3779b97f4a7c15ull * static_cast<uint64_t>(static_cast<uint32_t>(step + 1))) >> 32);
}

__device__ __forceinline__ float gumbel(uint32_t rk, int32_t token) {
  const uint32_t h = fmix32((static_cast<uint32_t>(token) * 0x9e3779b1u) ^ rk);
  const float u = __fmul_rn(static_cast<float>((h >> 9) * 2u + 1u), 5.9604644775390625e-08f);  // 2^-24
  const float e = -soft_logf(u);
  return -soft_logf(e);
}

__device__ __forceinline__ float gumbel_score(float logit, float inv_t, uint32_t rk, int32_t token) {
  return __fmaf_rn(logit, inv_t, gumbel(rk, token));
}

// ---- exact filtering (an optimisation that never changes the argmax) -------------
// gumbel() is increasing in the 23-bit draw K = h >> 9. A token can only beat the
// running best score b if g > b - logit/T; with logit <= m (chunk max) that needs
// g > c = b - m/T, i.e. u > exp(-exp(-c)). The threshold below is evaluated with
// fast intrinsics and then loosened (1e-3 in c, 1e-4 in u), so every token that
// could win is still scored with the exact rule; the rest are provably losers.
__device__ __forceinline__ uint32_t gumbel_draw(uint32_t rk, int32_t token) {
  return fmix32((static_cast<uint32_t>(token) * 0x9e3779b1u) ^ rk) >> 9;
}
// out-of-line on purpose: the (rare) exact score is reached through a branch, so the
// common "cannot win" path costs a bit test instead of an if-converted soft-log chain
static __device__ __noinline__ float gumbel_of_draw(uint32_t k) {
  const float u = __fmul_rn(static_cast<float>(k * 2u + 1u), 5.9604644775390625e-08f);  // 2^-24
  const float e = -soft_logf(u);
  return -soft_logf(e);
}
// draws K > threshold may win (signed integer compare); -1 = everything passes
__device__ __forceinline__ int gumbel_draw_threshold(float best, float chunk_max_logit, float inv_t) {
  if (!(best > -3.0e38f)) return -1;
  const float c = best - chunk_max_logit * inv_t - 1e-3f;
  const float ustar = __expf(-__expf(-c));
  const float kf = (ustar * (1.f - 1e-4f) * 16777216.f - 1.f) * 0.5f - 1.f;
  // every K with u(K) > u* (1 - 1e-4), i.e. K > kf + 1, satisfies K > floor(kf)
  return kf < 0.f ? -1 : static_cast<int>(kf);
}

// ======================= inverse-CDF contract (current) ======================
// The reference draws u ~ U[0,1) per step and scans cum += exp(l_i/T - max) in id order,
// taking the first i with u*den < cum (policy.cpp:402-422). The B200 rule is the same
// scan, organised so it fuses into the LM-head GEMM epilogue and stays bit-reproducible
// on the CPU from the fp32 logits:
//   x_i = l_i * (1/T) (BOS excluded); slices of kSlice = 32 consecutive ids;
//   per slice s: m_s = max x_i, e_i = sexp2((x_i - m_s) * log2 e),
//                Z_s = (a0 + a1) + (a2 + a3), a_j = sum of e_i with (i - slice_start) % 4 == j,
//                accumulated in id order;
//   M = max_s m_s, S_s = Z_s * sexp2((m_s - M) * log2 e);
//   slices are grouped into 32 lane blocks of B = ceil(S / 32) consecutive slices,
//   T_j = sum of S_s over block j in order, total = sum of T_j in order;
//   target = u * total with u = (2*(hi32(row_key_64) >> 9) + 1) * 2^-24;
//   walk blocks, then slices, then ids (r = fmaf(e_i, scale_s, r)) and take the first
//   position whose running sum exceeds target (fallback: the last positive one).
// sexp2 is a fixed chain of single-rounding fp32 operations (floor, 7 fmaf, exponent
// add), so every quantity above is identical on the CPU (oracle/dash_oracle.c).
constexpr int kSlice = 32;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float sexp2(float x) {  // x <= 0 in all uses
  x = fmaxf(x, -125.f);
  const float fl = floorf(x);
  const float f = __fsub_rn(x, fl);
  float p = 1.5252734e-05f;
  p = __fmaf_rn(p, f, 1.5403530e-04f);
  p = __fmaf_rn(p, f, 1.3333558e-03f);
  p = __fmaf_rn(p, f, 9.6181291e-03f);
  p = __fmaf_rn(p, f, 5.5504109e-02f);
  p = __fmaf_rn(p, f, 2.4022651e-01f);
  p = __fmaf_rn(p, f, 6.9314718e-01f);
  p = __fmaf_rn(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + static_cast<int>(fl) * (1 << 23));  // p * 2^fl, exact
}

__device__ __forceinline__ float row_uniform(uint64_t seq_key, int32_t step) {
  const uint32_t h = row_key(seq_key, step);
  return __fmul_rn(static_cast<float>((h >> 9) * 2u + 1u), 5.9604644775390625e-08f);
}

// (score, index) argmax combine with ties to the lowest index.
__device__ __forceinline__ bool better(float s1, int i1, float s0, int i0) {
  return s1 > s0 || (s1 == s0 && i1 < i0);
}

}  // namespace dashcu
