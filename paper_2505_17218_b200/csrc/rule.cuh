// The sampling contract (SURVEY App.B D2), device side.
//
// seq_key = derive_seed(round_seed, "sample", m_global, g)      (rng.hpp:29-35)
// row_key = hi32(splitmix64(seq_key + 0x9e3779b97f4a7c15 * (step + 1)))
// and then the inverse-CDF rule documented above sexp2() below.
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

__host__ __device__ __forceinline__ uint32_t row_key(uint64_t seq_key, int32_t step) {
  return static_cast<uint32_t>(
      splitmix64(seq_key + 0x9e3779b97f4a7c15ull * static_cast<uint64_t>(static_cast<uint32_t>(step + 1))) >> 32);
}

// ======================= inverse-CDF contract ======================
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
