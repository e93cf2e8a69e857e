// tcgen05 attention backward for head_dim 64 and 128 (policy.cpp:292-322, restated for packed
// causal sequences and GQA; the mma.sync kernel in attention_tc.cu is the fallback).
//
// One CTA owns a tile of 128 keys of one (sequence, KV head) and loops over every query
// head of the KV group x every causal tile of 128 queries. Per iteration, with the key
// axis as the MMA M dimension and all accumulators in TMEM:
//   (1) S^T  = K  Q^T      M128 N128 K64   A = K  (K-major)   B = Q  (K-major)
//   (2) dP^T = V  dO^T     M128 N128 K64   A = V  (K-major)   B = dO (K-major)
//   softmax warps: P^T = exp(S^T/sqrt(d) - LSE_q), dS^T = P^T (dP^T - D_q)/sqrt(d),
//   written as bf16 into shared memory in the UMMA 128-byte-swizzle layout
//   (4) dV  += P^T dO      M128 N64 K128   A = P^T (K-major)  B = dO (MN-major)
//   (5) dK  += dS^T Q      M128 N64 K128   A = dS^T (K-major) B = Q  (MN-major)
//   (6) dQ   = dS K        M128 N64 K128   A = dS (MN-major: the dS^T bytes)  B = K (MN-major)
// dQ is read out of TMEM and reduce-added into the fp32 dQ with bulk tensor reduces
// (one 32 x 32 box per softmax warp); dK / dV stay in TMEM for the whole group (the GQA
// sum needs no atomics) and are stored once at the end.
// Warp roles: 0 TMA producer (K, V once; Q / dO double-buffered), 1 MMA issuer,
// 2 TMEM allocator, 4..11 softmax (TMEM lane quarter = warp % 4, column half = (warp-4)/4).
// The MMAs of S(i+1) are issued as soon as the softmax warps have pulled S(i) into
// registers, so they overlap the softmax of iteration i.
#include <cfloat>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "kernels.cuh"
#include "tc5.cuh"

namespace dashcu {

#if defined(DASHCU_ATTN_TRACE) && DASHCU_ATTN_TRACE != 2
// Debug builds only: clock64 timeline of CTA (0, 0), 16 slots per iteration (see TR()).
__device__ unsigned long long g_attn_trace[64 * 16];
#define TR(it, k)                                                                             \
  do {                                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && (it) < 64)           \
      g_attn_trace[(it) * 16 + (k)] = clock64();                                              \
  } while (0)
#else
#define TR(it, k) \
  do {            \
  } while (0)
#endif

namespace {

constexpr int kKeys = 128, kQ = 128, kHD = 64;
// -DDASHCU_SPLIT_EXP: half the softmax exponentials via ex2_poly (tc5.cuh). Measured
// slower for the backward (its softmax warps are issue-bound, not MUFU-bound), neutral forward.
#ifdef DASHCU_SPLIT_EXP
constexpr bool kSplitExp = true;
#else
constexpr bool kSplitExp = false;
#endif
constexpr int kTile = kKeys * kHD * 2;  // 16 KB: [128 rows x 64] bf16, 128-byte swizzle

// ST: Q / dO / (LSE, D) pipeline depth; DQR: rows of the per-warp dQ staging box (32 = one
// 4 KB bulk reduce per warp and iteration, 16 = two 2 KB reduces, freeing smem for a 3rd stage)
template <int ST, int DQR>
struct Lay {
  static constexpr int K = 0, V = kTile, Q = 2 * kTile /*ST stages*/, O = (2 + ST) * kTile /*ST stages*/;
  static constexpr int S = (2 + 2 * ST) * kTile;  // dS^T [128 keys x 128 q] x 2 buffers (P^T lives in TMEM)
  static constexpr int DQ = S + 4 * kTile;         // 8 softmax warps x DQR x 32 fp32 dQ staging
  static constexpr int LD = DQ + 8 * DQR * 128;    // per stage: sL[128], sD[128]
  static constexpr int BAR = LD + ST * 1024;
  static constexpr int BYTES = BAR + 256 + 1024;  // + alignment slack
  static_assert(BYTES <= 232448, "exceeds the 227 KB of opt-in shared memory per CTA");
};

// TMEM columns
// TMEM columns: S^T, dP^T (fp32), the dV / dK / dQ accumulators, and P^T as packed bf16
// pairs (lane = key, column c = queries 2c, 2c+1): the A operand of dV += P^T dO
constexpr uint32_t kTS = 0, kTdP = 128, kTdV = 256, kTdK = 320, kTdQ = 384, kTP = 448;

constexpr uint32_t idesc(int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// tcgen05.mma with the A operand in TMEM (K-major: lane = row, 8 columns per K=16 step)
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

// 16 consecutive 32-bit TMEM columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// half a 128-byte row (32 bf16, chunks c0 .. c0+3) of a K-major swizzle atom: chunk j of
// row r lives at (j ^ (r & 7))
__device__ __forceinline__ void st_row32(uint32_t atom, int r, int c0, const float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(atom + r * 128 + (((c0 + j) ^ (r & 7)) << 4)),
                 "r"(pack2(v[8 * j], v[8 * j + 1])), "r"(pack2(v[8 * j + 2], v[8 * j + 3])),
                 "r"(pack2(v[8 * j + 4], v[8 * j + 5])), "r"(pack2(v[8 * j + 6], v[8 * j + 7]))
                 : "memory");
}

template <int ST, int DQR>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_tc5_k(const __grid_constant__ CUtensorMap mQKV, const __grid_constant__ CUtensorMap mO,
                   const __grid_constant__ CUtensorMap mDQ, const int32_t* __restrict__ seq_start,
                   const float* __restrict__ lse, const float* __restrict__ Dsum, int nh, int nkv,
                   float* __restrict__ dkv32, float* __restrict__ dq32, float scale, float scale_log2,
                   int n_seq, int nkt2, int chunk) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // grid (sequence x kv head, key tile x 2): launch order puts every long (early) key tile
  // first. Key tiles with >= 3 causal query tiles split their query heads over two CTAs
  // (dK / dV of the halves are then reduce-added: two adds onto zero, order-independent),
  // which roughly halves the longest CTA and the tail of the last wave.
  // chunk > 0 (1-D grid): CTAs in chunks of `chunk` sequences, each chunk ordered longest key
  // tile first; the chunk's Q / dO / dQ rows stay in L2 while its CTAs run (the 2-D order
  // walks every sequence's tile 0 first, a working set of the whole micro-batch)
  int bx = blockIdx.x, by = blockIdx.y;
  if (chunk > 0) {
    const int per = chunk * nkv * nkt2, ch = bx / per, r = bx % per;
    const int cs = min(chunk, n_seq - ch * chunk) * nkv;  // (sequence, kv head) pairs in this chunk
    by = r / cs;
    bx = ch * chunk * nkv + r % cs;
  }
  const int kt = by >> 1, part = by & 1, sq = bx / nkv, kvh = bx % nkv;
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int k0 = kt * kKeys;
  if (k0 >= n) return;  // uniform for the CTA, before any barrier
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = nh / nkv, qd = nh * kHD, kvd = nkv * kHD;
  const int nq = (n + kQ - 1) / kQ - kt;  // causal query tiles per head: kt .. last
  const bool split = grp > 1 && nq >= 3;
  if (!split && part) return;
  const int h_lo = split && part ? (grp + 1) / 2 : 0, h_hi = split && !part ? (grp + 1) / 2 : grp;
  const int nit = (h_hi - h_lo) * nq;

  using Lay = dashcu::Lay<ST, DQR>;
  constexpr int kST = ST;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::BAR);
  uint64_t *kvfull = bar, *sfull = bar + 1, *sfree = bar + 2, *pready = bar + 3, *dqfull = bar + 4,
           *dqfree = bar + 5, *pfree = bar + 6, *qfull = bar + 7 /*[kST]*/, *qempty = bar + 7 + kST /*[kST]*/,
           *ldfull = bar + 7 + 2 * kST /*[kST]*/;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 7 + 3 * kST);
  float* sLD = reinterpret_cast<float*>(smem + Lay::LD);  // [2][sL 128 | sD 128]

  if (threadIdx.x == 0) {
    mbar_init(kvfull, 1);
    for (int s = 0; s < kST; ++s) mbar_init(&qfull[s], 1), mbar_init(&qempty[s], 1), mbar_init(&ldfull[s], 32);
    mbar_init(sfull, 1);
    mbar_init(sfree, 256);
    mbar_init(pready, 256);
    mbar_init(dqfull, 1);
    mbar_init(dqfree, 256);
    mbar_init(pfree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mQKV)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mO)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sK = smem_u32(smem + Lay::K), sV = smem_u32(smem + Lay::V), sQ = smem_u32(smem + Lay::Q),
                 sO = smem_u32(smem + Lay::O), sS = smem_u32(smem + Lay::S);

  if (warp == 0) {  // ------------------------------------------------------------------ loads
    if (lane == 0) {
      mbar_expect_tx(kvfull, 2 * kTile);
      tma_load_2d(smem + Lay::K, &mQKV, kvfull, qd + kvh * kHD, s0 + k0);
      tma_load_2d(smem + Lay::V, &mQKV, kvfull, qd + kvd + kvh * kHD, s0 + k0);
    }
    int h = kvh * grp + h_lo, qt = kt;
    for (int it = 0; it < nit; ++it) {
      const int st = it % kST, q0 = qt * kQ;
      mbar_wait_sleep(&qempty[st], ((it / kST) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&qfull[st], 2 * kTile);
        tma_load_2d(smem + Lay::Q + st * kTile, &mQKV, &qfull[st], h * kHD, s0 + q0);
        tma_load_2d(smem + Lay::O + st * kTile, &mO, &qfull[st], h * kHD, s0 + q0);
      }
      // log2-scaled LSE and D of the tile's 128 queries (the rows of lse / D are strided
      // by n_heads, so the warp gathers them rather than TMA)
      float* L = sLD + st * 256;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ql = lane + 32 * j, q = q0 + ql;
        const int64_t idx = static_cast<int64_t>(s0 + q) * nh + h;
        L[ql] = q < n ? -(lse[idx] * 1.4426950408889634f) : 0.f;  // stored negated: fma(s, c, -L)
        L[128 + ql] = q < n ? Dsum[idx] : 0.f;
      }
      mbar_arrive(&ldfull[st]);
      if (++qt * kQ >= n) qt = kt, ++h;
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------------------------- MMA
      constexpr uint32_t I_SS = idesc(128, false, false), I_KM = idesc(64, false, true), I_MM = idesc(64, true, true);
      mbar_wait_sleep(kvfull, 0);
      auto issue_s = [&](int it) {
        const int st = it % kST;
        mbar_wait_sleep(&qfull[st], (it / kST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t q = sQ + st * kTile, o = sO + st * kTile;
#pragma unroll
        for (int k = 0; k < kHD / 16; ++k)
          umma_bf16(tmem + kTS, smem_desc(sK + k * 32, 16, 1024), smem_desc(q + k * 32, 16, 1024), I_SS, k > 0);
#pragma unroll
        for (int k = 0; k < kHD / 16; ++k)
          umma_bf16(tmem + kTdP, smem_desc(sV + k * 32, 16, 1024), smem_desc(o + k * 32, 16, 1024), I_SS, k > 0);
        umma_commit(sfull);
      };
      issue_s(0);
      for (int it = 0; it < nit; ++it) {
        const int st = it % kST;
        if (it + 1 < nit) {  // S(it+1) as soon as the softmax warps hold S(it) in registers
          mbar_wait_sleep(sfree, it & 1);
          TR(it, 0);
          issue_s(it + 1);
          TR(it, 1);
        }
        mbar_wait_sleep(pready, it & 1);
        TR(it, 2);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t q = sQ + st * kTile, o = sO + st * kTile, ds = sS + (it & 1) * 2 * kTile;
        // dV first: its commit releases the single P^T buffer early for the next softmax
#pragma unroll
        for (int j = 0; j < kQ / 16; ++j)  // K = 128 queries: two 64-wide atoms of P^T / dS^T
          umma_bf16_ts(tmem + kTdV, tmem + kTP + 8 * j, smem_desc(o + j * 2048, kTile, 1024), I_KM,
                       (it > 0 || j > 0) ? 1u : 0u);
        umma_commit(pfree);
#pragma unroll
        for (int j = 0; j < kQ / 16; ++j)
          umma_bf16(tmem + kTdK, smem_desc(ds + (j >> 2) * kTile + (j & 3) * 32, 16, 1024),
                    smem_desc(q + j * 2048, kTile, 1024), I_KM, (it > 0 || j > 0) ? 1u : 0u);
        umma_commit(&qempty[st]);  // Q / dO of this stage are no longer read (S, dP, dV, dK issued)
        // dQ(it) overwrites the dQ accumulator: dQ(it-1) must have been read out (the
        // softmax warps do that while dV / dK of this iteration run)
        if (it > 0) mbar_wait_sleep(dqfree, (it - 1) & 1);
        TR(it, 3);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int j = 0; j < kKeys / 16; ++j)  // K = 128 keys; dS read MN-major (q is contiguous)
          umma_bf16(tmem + kTdQ, smem_desc(ds + j * 2048, kTile, 1024), smem_desc(sK + j * 2048, kTile, 1024), I_MM,
                    j > 0 ? 1u : 0u);
        umma_commit(dqfull);
      }
    }
  } else if (warp >= 4) {  // ---------------------------------------------------------- softmax
    const int ew = warp - 4, qq = ew & 3, hf = ew >> 2;
    const int key_l = qq * 32 + lane, key = k0 + key_l;
    const uint32_t lanes = static_cast<uint32_t>(qq * 32) << 16;
    const uint32_t stg = smem_u32(smem + Lay::DQ + ew * DQR * 128);
    // dQ of iteration `it` (rows q0 + 32 qq + lane, head columns hf*32 .. +31): TMEM ->
    // scale -> swizzled staging -> one bulk tensor reduce-add per warp. Call after
    // mbar_wait(dqfull, it & 1).
    auto dq_out = [&](int h, int q0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float dq[32];
      tmem_ld32(tmem + lanes + kTdQ + hf * 32, dq);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(dqfree);
#pragma unroll
      for (int j = 0; j < 32; ++j) dq[j] *= scale;
      if constexpr (DQR == 0) {  // fire-and-forget 16-byte fp32 reductions straight from registers
        if (q0 + qq * 32 + lane < n) {
          float* dst = dq32 + static_cast<int64_t>(s0 + q0 + qq * 32 + lane) * qd + h * kHD + hf * 32;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * j), "f"(dq[4 * j]),
                         "f"(dq[4 * j + 1]), "f"(dq[4 * j + 2]), "f"(dq[4 * j + 3])
                         : "memory");
        }
        return;
      }
#pragma unroll
      for (int half = 0; half < (DQR ? 32 / DQR : 0); ++half) {  // DQR-row boxes of the warp's 32 rows
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        if (lane / (DQR ? DQR : 1) == half) {
          const int r = lane % (DQR ? DQR : 1);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg + r * 128 + ((j ^ (r & 7)) << 4)),
                         "f"(dq[4 * j]), "f"(dq[4 * j + 1]), "f"(dq[4 * j + 2]), "f"(dq[4 * j + 3])
                         : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
#ifndef DASHCU_EXP_NO_DQ_STORE  // experiment builds only: time the kernel without the dQ reduce traffic
        if (lane == 0) {
#else
        if (false) {
#endif
          asm volatile(
              "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                  reinterpret_cast<uint64_t>(&mDQ)),
              "r"(stg), "r"(h * kHD + hf * 32), "r"(s0 + q0 + qq * 32 + half * (DQR ? DQR : 1))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    };
    int h = kvh * grp + h_lo, qt = kt, ph = 0, pq0 = 0;  // (head, tile) of this and the previous iteration
    for (int it = 0; it < nit; ++it) {
      const int st = it % kST, q0 = qt * kQ;
      mbar_wait_sleep(&ldfull[st], (it / kST) & 1);
      const float* L = sLD + st * 256 + hf * 64;
      const float* D = L + 128;
      if (warp == 4) TR(it, 4);
      mbar_wait_sleep(sfull, it & 1);
      if (warp == 4) TR(it, 5);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // masks only on the causal diagonal and at the sequence end (warp-uniform)
      const bool edge = qt == kt || q0 + kQ > n || k0 + kKeys > n;
      // two 32-column halves keep 64 registers of scores live; the second half's TMEM loads
      // release S^T / dP^T for the next iteration's MMAs
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t sr[32], dr[32];
        const uint32_t col = hf * 64 + hh * 32;
        tmem_ld32_async(tmem + lanes + kTS + col, sr);
        tmem_ld32_async(tmem + lanes + kTdP + col, dr);
        tmem_wait_ld();
        if (warp == 4) TR(it, 12 + hh);
        if (hh == 1) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mbar_arrive(sfree);
        }
        float* sv = reinterpret_cast<float*>(sr);  // P^T and dS^T overwrite S^T / dP^T in place
        float* dp = reinterpret_cast<float*>(dr);
        // element pairs on the packed fp32x2 pipe (FFMA2 / FADD2 / FMUL2): the softmax
        // warps are issue-bound, this removes a third of their instructions. Masks exist
        // only on edge tiles, in their own loop (predicated-off instructions still issue):
        // column c of this half is valid iff lo <= c < hi (causal key <= q, q < n, key < n).
        const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
        const int qb = q0 + col;
        const int lo = key - qb, hi = key < n ? max(lo, n - qb) : lo;  // empty range when key >= n
        auto body = [&](auto masked) {
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const float4 l4 = *reinterpret_cast<const float4*>(L + hh * 32 + c);  // -L (log2 units)
            const float4 d4 = *reinterpret_cast<const float4*>(D + hh * 32 + c);
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const uint64_t arg = f2_fma(f2_pack(sv[c + e], sv[c + e + 1]), sc2,
                                          e ? f2_pack(l4.z, l4.w) : f2_pack(l4.x, l4.y));
              float p0, p1;
              f2_unpack(arg, p0, p1);
              p0 = ex2(p0);
              p1 = (kSplitExp && ((c + e) & 3) == 0) ? ex2_poly(p1) : ex2(p1);  // 1 in 4 on the FMA pipe
              if constexpr (decltype(masked)::value) {
                const int cc = c + e;
                p0 = static_cast<unsigned>(cc - lo) < static_cast<unsigned>(hi - lo) ? p0 : 0.f;
                p1 = static_cast<unsigned>(cc + 1 - lo) < static_cast<unsigned>(hi - lo) ? p1 : 0.f;
              }
              sv[c + e] = p0;
              sv[c + e + 1] = p1;
              const uint64_t t =
                  f2_sub(f2_pack(dp[c + e], dp[c + e + 1]), e ? f2_pack(d4.z, d4.w) : f2_pack(d4.x, d4.y));
              f2_unpack(f2_mul(f2_pack(p0, p1), t), dp[c + e], dp[c + e + 1]);  // 1/sqrt(d) applied at readout
            }
          }
        };
        if (edge) body(std::true_type());
        else body(std::false_type());
        // P^T is single-buffered: dV(it-1) must have read it (pfree, committed first);
        // dS^T alternates between two buffers, the one of it-2 was released with dqfull(it-2)
        if (warp == 4) TR(it, 6 + hh * 4);
        if (hh == 0 && it > 0) mbar_wait_sleep(pfree, (it - 1) & 1);
        if (warp == 4) TR(it, 7 + hh * 4);
        {  // P^T: 32 queries -> 16 packed columns of this lane's TMEM row
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = pack2(sv[2 * i], sv[2 * i + 1]);
          tmem_st16(tmem + lanes + kTP + hf * 32 + hh * 16, pk);
        }
        st_row32(sS + (it & 1) * 2 * kTile + hf * kTile, key_l, hh * 4, dp);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // P^T stores landed in TMEM
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // dS^T visible to the MMAs
      mbar_arrive(pready);
      if (warp == 4) TR(it, 14);
      // dQ(it-1) (complete long ago) is read out while dV(it) / dK(it) run; its dqfree
      // gates only the dQ(it) MMA
      if (it > 0) {
        mbar_wait_sleep(dqfull, (it - 1) & 1);
        if (warp == 4) TR(it, 8);
        dq_out(ph, pq0);
        if (warp == 4) TR(it, 9);
      }
      ph = h, pq0 = q0;
      if (++qt * kQ >= n) qt = kt, ++h;
    }
    mbar_wait_sleep(dqfull, (nit - 1) & 1);
    dq_out(ph, pq0);
    // dK, dV of this thread's key row (all MMAs completed: the last dqfull covers them)
    float dk[32], dv[32];
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tmem_ld32(tmem + lanes + kTdK + hf * 32, dk);
    tmem_ld32(tmem + lanes + kTdV + hf * 32, dv);
#pragma unroll
    for (int i = 0; i < 32; ++i) dk[i] *= scale;
    if (key < n) {
      float* dkr = dkv32 + static_cast<int64_t>(s0 + key) * 2 * kvd + kvh * kHD + hf * 32;
      float* dvr = dkr + kvd;
      if (split) {  // dkv32 is zero: the two halves' sums are order-independent
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dkr + i), "f"(dk[i]), "f"(dk[i + 1]),
                       "f"(dk[i + 2]), "f"(dk[i + 3])
                       : "memory");
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dvr + i), "f"(dv[i]), "f"(dv[i + 1]),
                       "f"(dv[i + 2]), "f"(dv[i + 3])
                       : "memory");
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          *reinterpret_cast<float4*>(dkr + i) = make_float4(dk[i], dk[i + 1], dk[i + 2], dk[i + 3]);
          *reinterpret_cast<float4*>(dvr + i) = make_float4(dv[i], dv[i + 1], dv[i + 2], dv[i + 3]);
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// ---------------------------------------------------------------------------- head_dim 128
// The head_dim 64 layout (S^T, dP^T 128 x 128 each; dV, dK, dQ 64 columns each; P^T) needs
// 704 TMEM columns at head_dim 128, one CTA has 512. Query tiles of 64 instead, and dQ
// produced transposed so every MMA keeps M = 128:
//   (1) S^T  = K  Q^T      M128 N64  K128  A = K  (K-major, 2 atoms)  B = Q  (K-major, 2 atoms)
//   (2) dP^T = V  dO^T     M128 N64  K128  A = V                      B = dO
//   (4) dV  += P^T dO      M128 N128 K64   A = P^T (TMEM)             B = dO (MN-major, 2 atoms)
//   (5) dK  += dS^T Q      M128 N128 K64   A = dS^T (K-major)         B = Q  (MN-major, 2 atoms)
//   (6) dQ^T = K^T dS^T    M128 N64  K128  A = K  (MN-major, 2 atoms) B = dS^T (MN-major)
// TMEM: S^T 64 | dP^T 64 | dV 128 | dK 128 | dQ^T 64 | P^T 32 = 480 columns. dQ^T rows are
// head dims, so each softmax warp stages a [32 queries x 32 dims] fp32 box (transposing
// through shared memory) and reduce-adds it with one bulk tensor reduce.
constexpr int kQ64 = 64, kHD128 = 128;
constexpr int kAt = 16384;         // K / V atom: 128 key rows x 128 bytes
constexpr int kKV128 = 2 * kAt;    // K or V tile [128 keys x 128] bf16
constexpr int kQT = 2 * 8192;      // Q or dO tile [64 q x 128] bf16: two 8 KB atoms (64 rows x 128 bytes)
constexpr int kST128 = 2;

struct Lay128 {
  static constexpr int K = 0, V = kKV128, Q = 2 * kKV128 /*kST128 stages*/, O = Q + kST128 * kQT;
  static constexpr int S = O + kST128 * kQT;  // dS^T [128 keys x 64 q] bf16 (one atom) x 2 buffers
  static constexpr int DQ = S + 2 * kAt;      // 8 softmax warps x [32 x 32] fp32 dQ staging
  static constexpr int LD = DQ + 8 * 4096;    // per stage: -L[64], D[64]
  static constexpr int BAR = LD + kST128 * 512;
  static constexpr int BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "exceeds the 227 KB of opt-in shared memory per CTA");
};
constexpr uint32_t kT8S = 0, kT8dP = 64, kT8dV = 128, kT8dK = 256, kT8dQ = 384, kT8P = 448;

__global__ void __launch_bounds__(384, 1)
    attn_bwd_tc5_hd128_k(const __grid_constant__ CUtensorMap mKV, const __grid_constant__ CUtensorMap mQ,
                         const __grid_constant__ CUtensorMap mO, const __grid_constant__ CUtensorMap mDQ,
                         const int32_t* __restrict__ seq_start, const float* __restrict__ lse,
                         const float* __restrict__ Dsum, int nh, int nkv, float* __restrict__ dkv32, float scale,
                         float scale_log2, int n_seq, int nkt2, int chunk) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  int bx = blockIdx.x, by = blockIdx.y;  // CTA order as in attn_bwd_tc5_k
  if (chunk > 0) {
    const int per = chunk * nkv * nkt2, ch = bx / per, r = bx % per;
    const int cs = min(chunk, n_seq - ch * chunk) * nkv;
    by = r / cs;
    bx = ch * chunk * nkv + r % cs;
  }
  const int kt = by >> 1, part = by & 1, sq = bx / nkv, kvh = bx % nkv;
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int k0 = kt * kKeys;
  if (k0 >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = nh / nkv, qd = nh * kHD128, kvd = nkv * kHD128;
  const int qt0 = 2 * kt, nq = (n + kQ64 - 1) / kQ64 - qt0;  // causal 64-query tiles per head
  const bool split = grp > 1 && nq >= 6;
  if (!split && part) return;
  const int h_lo = split && part ? (grp + 1) / 2 : 0, h_hi = split && !part ? (grp + 1) / 2 : grp;
  const int nit = (h_hi - h_lo) * nq;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay128::BAR);
  uint64_t *kvfull = bar, *sfull = bar + 1, *sfree = bar + 2, *pready = bar + 3, *dqfull = bar + 4,
           *dqfree = bar + 5, *pfree = bar + 6, *qfull = bar + 7 /*[kST128]*/, *qempty = bar + 7 + kST128,
           *ldfull = bar + 7 + 2 * kST128;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 7 + 3 * kST128);
  float* sLD = reinterpret_cast<float*>(smem + Lay128::LD);

  if (threadIdx.x == 0) {
    mbar_init(kvfull, 1);
    for (int s = 0; s < kST128; ++s) mbar_init(&qfull[s], 1), mbar_init(&qempty[s], 1), mbar_init(&ldfull[s], 32);
    mbar_init(sfull, 1);
    mbar_init(sfree, 256);
    mbar_init(pready, 256);
    mbar_init(dqfull, 1);
    mbar_init(dqfree, 256);
    mbar_init(pfree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mKV)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mO)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sK = smem_u32(smem + Lay128::K), sV = smem_u32(smem + Lay128::V), sQ = smem_u32(smem + Lay128::Q),
                 sO = smem_u32(smem + Lay128::O), sS = smem_u32(smem + Lay128::S);

  if (warp == 0) {  // ------------------------------------------------------------------ loads
    if (lane == 0) {
      mbar_expect_tx(kvfull, 2 * kKV128);
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        tma_load_2d(smem + Lay128::K + a * kAt, &mKV, kvfull, qd + kvh * kHD128 + a * 64, s0 + k0);
        tma_load_2d(smem + Lay128::V + a * kAt, &mKV, kvfull, qd + kvd + kvh * kHD128 + a * 64, s0 + k0);
      }
    }
    int h = kvh * grp + h_lo, qt = qt0;
    for (int it = 0; it < nit; ++it) {
      const int st = it % kST128, q0 = qt * kQ64;
      mbar_wait_sleep(&qempty[st], ((it / kST128) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&qfull[st], 2 * kQT);
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          tma_load_2d(smem + Lay128::Q + st * kQT + a * 8192, &mQ, &qfull[st], h * kHD128 + a * 64, s0 + q0);
          tma_load_2d(smem + Lay128::O + st * kQT + a * 8192, &mO, &qfull[st], h * kHD128 + a * 64, s0 + q0);
        }
      }
      float* L = sLD + st * 128;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int ql = lane + 32 * j, q = q0 + ql;
        const int64_t idx = static_cast<int64_t>(s0 + q) * nh + h;
        L[ql] = q < n ? -(lse[idx] * 1.4426950408889634f) : 0.f;
        L[64 + ql] = q < n ? Dsum[idx] : 0.f;
      }
      mbar_arrive(&ldfull[st]);
      if (++qt * kQ64 >= n) qt = qt0, ++h;
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------------------------- MMA
      constexpr uint32_t I_S = idesc(64, false, false), I_KM = idesc(128, false, true), I_Q = idesc(64, true, true);
      mbar_wait_sleep(kvfull, 0);
      auto issue_s = [&](int it) {
        const int st = it % kST128;
        mbar_wait_sleep(&qfull[st], (it / kST128) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t q = sQ + st * kQT, o = sO + st * kQT;
#pragma unroll
        for (int k = 0; k < kHD128 / 16; ++k)  // head-dim step k: atom k / 4, 32-byte chunk k % 4
          umma_bf16(tmem + kT8S, smem_desc(sK + (k >> 2) * kAt + (k & 3) * 32, 16, 1024),
                    smem_desc(q + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024), I_S, k > 0);
#pragma unroll
        for (int k = 0; k < kHD128 / 16; ++k)
          umma_bf16(tmem + kT8dP, smem_desc(sV + (k >> 2) * kAt + (k & 3) * 32, 16, 1024),
                    smem_desc(o + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024), I_S, k > 0);
        umma_commit(sfull);
      };
      issue_s(0);
      for (int it = 0; it < nit; ++it) {
        const int st = it % kST128;
        if (it + 1 < nit) {
          mbar_wait_sleep(sfree, it & 1);
          issue_s(it + 1);
        }
        mbar_wait_sleep(pready, it & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t q = sQ + st * kQT, o = sO + st * kQT, ds = sS + (it & 1) * kAt;
#pragma unroll
        for (int j = 0; j < kQ64 / 16; ++j)  // K = 64 queries; B atoms (head dims 0-63, 64-127) 8 KB apart
          umma_bf16_ts(tmem + kT8dV, tmem + kT8P + 8 * j, smem_desc(o + j * 2048, 8192, 1024), I_KM,
                       (it > 0 || j > 0) ? 1u : 0u);
        umma_commit(pfree);
#pragma unroll
        for (int j = 0; j < kQ64 / 16; ++j)
          umma_bf16(tmem + kT8dK, smem_desc(ds + j * 32, 16, 1024), smem_desc(q + j * 2048, 8192, 1024), I_KM,
                    (it > 0 || j > 0) ? 1u : 0u);
        umma_commit(&qempty[st]);
        if (it > 0) mbar_wait_sleep(dqfree, (it - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int j = 0; j < kKeys / 16; ++j)  // K = 128 keys; K^T read MN-major (head dims contiguous)
          umma_bf16(tmem + kT8dQ, smem_desc(sK + j * 2048, kAt, 1024), smem_desc(ds + j * 2048, kAt, 1024), I_Q,
                    j > 0 ? 1u : 0u);
        umma_commit(dqfull);
      }
    }
  } else if (warp >= 4) {  // ---------------------------------------------------------- softmax
    const int ew = warp - 4, qq = ew & 3, hf = ew >> 2;
    const int key_l = qq * 32 + lane, key = k0 + key_l;
    const uint32_t lanes = static_cast<uint32_t>(qq * 32) << 16;
    const uint32_t stg = smem_u32(smem + Lay128::DQ + ew * 4096);
    // dQ^T of iteration `it`: TMEM lanes = head dims 32 qq + lane, columns = queries
    // 32 hf .. +31 -> [32 q x 32 dims] swizzled staging box -> one bulk reduce-add
    auto dq_out = [&](int h, int q0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float dq[32];
      tmem_ld32(tmem + lanes + kT8dQ + hf * 32, dq);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(dqfree);
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j)  // row j (query), column lane (head dim): chunk lane / 4 ^ (j & 7)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(stg + j * 128 + ((((lane >> 2) ^ j) & 7) << 4) + (lane & 3) * 4),
                     "f"(dq[j] * scale)
                     : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile(
            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                reinterpret_cast<uint64_t>(&mDQ)),
            "r"(stg), "r"(h * kHD128 + qq * 32), "r"(s0 + q0 + hf * 32)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    };
    const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
    int h = kvh * grp + h_lo, qt = qt0, ph = 0, pq0 = 0;
    for (int it = 0; it < nit; ++it) {
      const int st = it % kST128, q0 = qt * kQ64;
      mbar_wait_sleep(&ldfull[st], (it / kST128) & 1);
      const float* L = sLD + st * 128 + hf * 32;
      const float* D = L + 64;
      mbar_wait_sleep(sfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const bool edge = q0 < k0 + kKeys || q0 + kQ64 > n || k0 + kKeys > n;
      uint32_t sr[32], dr[32];
      tmem_ld32_async(tmem + lanes + kT8S + hf * 32, sr);
      tmem_ld32_async(tmem + lanes + kT8dP + hf * 32, dr);
      tmem_wait_ld();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(sfree);
      float* sv = reinterpret_cast<float*>(sr);
      float* dp = reinterpret_cast<float*>(dr);
      const int qb = q0 + hf * 32;
      const int lo = key - qb, hi = key < n ? max(lo, n - qb) : lo;
      auto body = [&](auto masked) {
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(L + c);
          const float4 d4 = *reinterpret_cast<const float4*>(D + c);
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const uint64_t arg =
                f2_fma(f2_pack(sv[c + e], sv[c + e + 1]), sc2, e ? f2_pack(l4.z, l4.w) : f2_pack(l4.x, l4.y));
            float p0, p1;
            f2_unpack(arg, p0, p1);
            p0 = ex2(p0);
            p1 = ex2(p1);
            if constexpr (decltype(masked)::value) {
              const int cc = c + e;
              p0 = static_cast<unsigned>(cc - lo) < static_cast<unsigned>(hi - lo) ? p0 : 0.f;
              p1 = static_cast<unsigned>(cc + 1 - lo) < static_cast<unsigned>(hi - lo) ? p1 : 0.f;
            }
            sv[c + e] = p0;
            sv[c + e + 1] = p1;
            const uint64_t t =
                f2_sub(f2_pack(dp[c + e], dp[c + e + 1]), e ? f2_pack(d4.z, d4.w) : f2_pack(d4.x, d4.y));
            f2_unpack(f2_mul(f2_pack(p0, p1), t), dp[c + e], dp[c + e + 1]);
          }
        }
      };
      if (edge) body(std::true_type());
      else body(std::false_type());
      if (it > 0) mbar_wait_sleep(pfree, (it - 1) & 1);  // dV(it-1) has read P^T
      {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack2(sv[2 * i], sv[2 * i + 1]);
        tmem_st16(tmem + lanes + kT8P + hf * 16, pk);
      }
      st_row32(sS + (it & 1) * kAt, key_l, hf * 4, dp);  // dS^T row: queries 32 hf .. (chunks 4 hf ..)
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(pready);
      if (it > 0) {
        mbar_wait_sleep(dqfull, (it - 1) & 1);
        dq_out(ph, pq0);
      }
      ph = h, pq0 = q0;
      if (++qt * kQ64 >= n) qt = qt0, ++h;
    }
    mbar_wait_sleep(dqfull, (nit - 1) & 1);
    dq_out(ph, pq0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
    for (int c = 0; c < 2; ++c) {  // dK, dV of this key row: head dims 64 hf + 32 c ..
      float dk[32], dv[32];
      tmem_ld32(tmem + lanes + kT8dK + hf * 64 + c * 32, dk);
      tmem_ld32(tmem + lanes + kT8dV + hf * 64 + c * 32, dv);
      if (key < n) {
        float* dkr = dkv32 + static_cast<int64_t>(s0 + key) * 2 * kvd + kvh * kHD128 + hf * 64 + c * 32;
        float* dvr = dkr + kvd;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          if (split) {
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dkr + i), "f"(dk[i] * scale),
                         "f"(dk[i + 1] * scale), "f"(dk[i + 2] * scale), "f"(dk[i + 3] * scale)
                         : "memory");
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dvr + i), "f"(dv[i]), "f"(dv[i + 1]),
                         "f"(dv[i + 2]), "f"(dv[i + 3])
                         : "memory");
          } else {
            *reinterpret_cast<float4*>(dkr + i) =
                make_float4(dk[i] * scale, dk[i + 1] * scale, dk[i + 2] * scale, dk[i + 3] * scale);
            *reinterpret_cast<float4*>(dvr + i) = make_float4(dv[i], dv[i + 1], dv[i + 2], dv[i + 3]);
          }
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
}  // namespace

#if defined(DASHCU_ATTN_TRACE) && DASHCU_ATTN_TRACE != 2
int attn_trace_read(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif

namespace {
template <int ST, int DQR>
void launch_bwd_tc5(cudaStream_t s, const CUtensorMap& mq, const CUtensorMap& mo, const CUtensorMap& mdq,
                    const int32_t* seq_start, const float* lse, const float* Dbuf, int n_seq, int max_len, int nh,
                    int nkv, float* dkv32, float* dq32, float sc) {
  auto k = attn_bwd_tc5_k<ST, DQR>;
  static bool attr = false;
  if (!attr) {
    DCU_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay<ST, DQR>::BYTES));
    attr = true;
  }
  const int nkt2 = 2 * ((max_len + kKeys - 1) / kKeys);
  // measured (C2 micro-batch, same box): 2-D order 0.508 ms, chunks of 2 / 4 / 8 sequences
  // 0.429 / 0.413 / 0.415 ms (DRAM reads of Q / dO / dQ fall once a chunk fits in L2)
  const int chunk = knob(KNOB_ATTN_BWD_CHUNK);
  dim3 grid = chunk > 0 ? dim3(n_seq * nkv * nkt2, 1) : dim3(n_seq * nkv, nkt2);
  k<<<grid, 384, Lay<ST, DQR>::BYTES, s>>>(mq, mo, mdq, seq_start, lse, Dbuf, nh, nkv, dkv32, dq32, sc,
                                             sc * 1.4426950408889634f, n_seq, nkt2, chunk);
  DCU_LAUNCHED();
}
}  // namespace

bool attn_bwd_tc5(cudaStream_t s, const bf16* qkv, const bf16* dctx, const float* lse, const float* Dbuf,
                  const int32_t* seq_start, int n_seq, int max_len, int rows, int nh, int nkv, int hd, float* dq32,
                  float* dkv32) {
  if ((hd != kHD && hd != kHD128) || nh % nkv) return false;
  if (knob(KNOB_ATTN_BWD) == 1) return false;
  const int qd = nh * hd, qkvd = qd + 2 * nkv * hd;
  if (hd == kHD128) {
    CUtensorMap mkv, mq, mo, mdq;
    if (!tma_map_2d(&mkv, qkv, rows, qkvd, qkvd, 64, 128, false, 128, true) ||
        !tma_map_2d(&mq, qkv, rows, qkvd, qkvd, 64, 64, false, 128, true) ||
        !tma_map_2d(&mo, dctx, rows, qd, qd, 64, 64, false, 128, true) ||
        !tma_map_2d(&mdq, dq32, rows, qd, qd, 32, 32, true, 128, false))
      return false;
    static bool attr = false;
    if (!attr) {
      DCU_CHECK(cudaFuncSetAttribute(attn_bwd_tc5_hd128_k, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay128::BYTES));
      attr = true;
    }
    const int nkt2 = 2 * ((max_len + kKeys - 1) / kKeys);
    const int chunk = knob(KNOB_ATTN_BWD_CHUNK);
    dim3 grid = chunk > 0 ? dim3(n_seq * nkv * nkt2, 1) : dim3(n_seq * nkv, nkt2);
    const float sc = 1.f / sqrtf(static_cast<float>(hd));
    attn_bwd_tc5_hd128_k<<<grid, 384, Lay128::BYTES, s>>>(mkv, mq, mo, mdq, seq_start, lse, Dbuf, nh, nkv, dkv32, sc,
                                                          sc * 1.4426950408889634f, n_seq, nkt2, chunk);
    DCU_LAUNCHED();
    return true;
  }
  CUtensorMap mq, mo, mdq;
  if (!tma_map_2d(&mq, qkv, rows, qkvd, qkvd, kHD, 128, false, 128, true) ||
      !tma_map_2d(&mo, dctx, rows, qd, qd, kHD, 128, false, 128, true) ||
      !tma_map_2d(&mdq, dq32, rows, qd, qd, 32, 32, true, 128, false))
    return false;
  const float sc = 1.f / sqrtf(static_cast<float>(hd));
  // dQ: bulk tensor reduce-adds of 32-row boxes staged in shared memory
  launch_bwd_tc5<2, 32>(s, mq, mo, mdq, seq_start, lse, Dbuf, n_seq, max_len, nh, nkv, dkv32, dq32, sc);
  return true;
}

}  // namespace dashcu
