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

// Two sexp2 evaluations on the packed fp32x2 pipe (FADD2 / FFMA2): per lane exactly the
// single-rounding operations of sexp2 above (floor via a round-toward-minus-infinity add of
// 1.5 * 2^23, exact for |x| < 2^22), so results are bit-identical and half the instructions.
__device__ __forceinline__ void sexp2_x2(float xa, float xb, float& ra, float& rb) {
  constexpr float kMagic = 12582912.f;
  xa = fmaxf(xa, -125.f);
  xb = fmaxf(xb, -125.f);
  uint64_t x2, mg, t2, fl2, f2, p2, c;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x2) : "f"(xa), "f"(xb));
  asm("mov.b64 %0, {%1, %1};" : "=l"(mg) : "f"(kMagic));
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(t2) : "l"(x2), "l"(mg));   // floor(x) + magic
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(fl2) : "l"(t2), "l"(mg));  // floor(x)
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(f2) : "l"(x2), "l"(fl2));  // x - floor(x)
  asm("mov.b64 %0, {%1, %1};" : "=l"(p2) : "f"(1.5252734e-05f));
#define DCU_SEXP2_STEP(k)                                                  \
  asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(k));                         \
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p2) : "l"(p2), "l"(f2), "l"(c));
  DCU_SEXP2_STEP(1.5403530e-04f)
  DCU_SEXP2_STEP(1.3333558e-03f)
  DCU_SEXP2_STEP(9.6181291e-03f)
  DCU_SEXP2_STEP(5.5504109e-02f)
  DCU_SEXP2_STEP(2.4022651e-01f)
  DCU_SEXP2_STEP(6.9314718e-01f)
  DCU_SEXP2_STEP(1.0f)
#undef DCU_SEXP2_STEP
  float pa, pb, ta, tb;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(pa), "=f"(pb) : "l"(p2));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(ta), "=f"(tb) : "l"(t2));
  ra = __int_as_float(__float_as_int(pa) + (__float_as_int(ta) - 0x4b400000) * (1 << 23));
  rb = __int_as_float(__float_as_int(pb) + (__float_as_int(tb) - 0x4b400000) * (1 << 23));
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
