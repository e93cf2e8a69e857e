// tcgen05 attention forward for head_dim 64 (teacher-forced causal attention of the
// training pass, policy.cpp:105-129; the mma.sync kernel in attention_tc.cu is the fallback).
//
// One CTA owns 128 queries of one (sequence, query head) and walks the causal key tiles
// (128 keys each) with an online softmax:
//   S_j = Q K_j^T          M128 N128 K64    A = Q (K-major)   B = K_j (K-major)   -> TMEM S[j&1]
//   softmax warps: m_j = max(m_{j-1}, rowmax(S_j)/sqrt(d)), P_j = exp(S_j/sqrt(d) - m_j) (bf16, smem)
//   O_j = P_j V_j          M128 N64  K128   A = P_j (K-major) B = V_j (MN-major)  -> TMEM O[j&1]
//   registers: acc = acc * 2^(m_{j-1} - m_j) + O_j,  l likewise; out = acc / l, LSE = m + log l.
// S and O are double-buffered in TMEM so the MMA of S_{j+1} and of O_j overlap the softmax.
// Warp roles: 0 TMA producer (Q once, K/V kST-stage ring), 1 MMA issuer, 2 TMEM allocator,
// 4..7 softmax (one thread per query row; TMEM lane quarter = warp % 4).
#include <cfloat>
#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "tc5.cuh"

namespace dashcu {

namespace {

constexpr int kQ = 128, kKeys = 128, kHD = 64;
constexpr int kTile = 128 * kHD * 2;  // 16 KB

constexpr int kST = 4;  // K/V pipeline depth: loads run 3 key tiles ahead of the MMAs

struct FLay {
  static constexpr int Q = 0, K = kTile /*kST stages*/, V = (1 + kST) * kTile /*kST stages*/;
  static constexpr int P = (1 + 2 * kST) * kTile;  // P [128 q x 128 keys] bf16: two 64-key swizzle atoms
  static constexpr int BAR = P + 2 * kTile;
  static constexpr int BYTES = BAR + 256 + 1024;
};

constexpr uint32_t kTS0 = 0, kTS1 = 128, kTO0 = 256, kTO1 = 320;

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

__global__ void __launch_bounds__(256, 1)
    attn_fwd_tc5_k(const __grid_constant__ CUtensorMap mQKV, const int32_t* __restrict__ seq_start, int nh, int nkv,
                   int nqt_max, bf16* __restrict__ ctx, float* __restrict__ lse, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // grid (sequence x head, query tile), the longest (last) query tiles launched first
  const int sq = blockIdx.x / nh, h = blockIdx.x % nh, qt = nqt_max - 1 - static_cast<int>(blockIdx.y);
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int q0 = qt * kQ;
  if (q0 >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = nh / nkv, kvh = h / grp, qd = nh * kHD, kvd = nkv * kHD;
  const int nkt = qt + 1;  // causal key tiles 0 .. qt

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FLay::BAR);
  uint64_t *qfull = bar, *sfull = bar + 1 /*[2]*/, *sfree = bar + 3 /*[2]*/, *pready = bar + 5,
           *ofull = bar + 6 /*[2]*/, *ofree = bar + 8 /*[2]*/, *kvfull = bar + 10 /*[kST]*/,
           *kvempty = bar + 10 + kST /*[kST]*/;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10 + 2 * kST);

  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int i = 0; i < kST; ++i) {
      mbar_init(&kvfull[i], 1);
      mbar_init(&kvempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sfree[i], 128);
      mbar_init(&ofull[i], 1);
      mbar_init(&ofree[i], 128);
    }
    mbar_init(pready, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mQKV)) : "memory");
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
  const uint32_t sQ = smem_u32(smem + FLay::Q), sK = smem_u32(smem + FLay::K), sV = smem_u32(smem + FLay::V),
                 sP = smem_u32(smem + FLay::P);

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------------------------- TMA
      mbar_expect_tx(qfull, kTile);
      tma_load_2d(smem + FLay::Q, &mQKV, qfull, h * kHD, s0 + q0);
      for (int j = 0; j < nkt; ++j) {
        const int st = j % kST;
        mbar_wait(&kvempty[st], ((j / kST) & 1) ^ 1);
        mbar_expect_tx(&kvfull[st], 2 * kTile);
        tma_load_2d(smem + FLay::K + st * kTile, &mQKV, &kvfull[st], qd + kvh * kHD, s0 + j * kKeys);
        tma_load_2d(smem + FLay::V + st * kTile, &mQKV, &kvfull[st], qd + kvd + kvh * kHD, s0 + j * kKeys);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------------------------- MMA
      constexpr uint32_t I_S = idesc(128, false, false), I_O = idesc(64, false, true);
      mbar_wait(qfull, 0);
      auto issue_s = [&](int j) {
        const int sb = j & 1, st = j % kST;
        if (j >= 2) mbar_wait(&sfree[sb], ((j >> 1) - 1) & 1);  // softmax holds S_{j-2} in registers
        mbar_wait(&kvfull[st], (j / kST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t k = sK + st * kTile;
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk)
          umma_bf16(tmem + (sb ? kTS1 : kTS0), smem_desc(sQ + kk * 32, 16, 1024), smem_desc(k + kk * 32, 16, 1024),
                    I_S, kk > 0);
        umma_commit(&sfull[sb]);
      };
      issue_s(0);
      for (int j = 0; j < nkt; ++j) {
        const int sb = j & 1, st = j % kST;
        if (j + 1 < nkt) issue_s(j + 1);
        mbar_wait(pready, j & 1);
        if (j >= 2) mbar_wait(&ofree[sb], ((j >> 1) - 1) & 1);  // O_{j-2} read out
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t v = sV + st * kTile;
#pragma unroll
        for (int kk = 0; kk < kKeys / 16; ++kk)
          umma_bf16(tmem + (sb ? kTO1 : kTO0), smem_desc(sP + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024),
                    smem_desc(v + kk * 2048, kTile, 1024), I_O, kk > 0);
        umma_commit(&kvempty[st]);
        umma_commit(&ofull[sb]);
      }
    }
  } else if (warp >= 4) {  // ---------------------------------------------------------- softmax
    const int qq = warp & 3, r = qq * 32 + lane, q = q0 + r;
    const uint32_t lanes = static_cast<uint32_t>(qq * 32) << 16;
    float acc[kHD];
#pragma unroll
    for (int i = 0; i < kHD; ++i) acc[i] = 0.f;
    float m = -FLT_MAX, m_prev = -FLT_MAX, l = 0.f;
    // O_j (TMEM) into the register accumulator: acc = acc * 2^(m_old - m_new) + O_j
    auto take_o = [&](int j, float m_old, float m_new) {
      const int st = j & 1;
      mbar_wait(&ofull[st], (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t o[kHD];
      tmem_ld32_async(tmem + lanes + (st ? kTO1 : kTO0), o);
      tmem_ld32_async(tmem + lanes + (st ? kTO1 : kTO0) + 32, o + 32);
      tmem_wait_ld();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&ofree[st]);
      const float c = ex2(m_old - m_new);
#pragma unroll
      for (int i = 0; i < kHD; ++i) acc[i] = __fmaf_rn(acc[i], c, __uint_as_float(o[i]));
    };
    for (int j = 0; j < nkt; ++j) {
      const int st = j & 1;
      mbar_wait(&sfull[st], (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t sr[kKeys];
#pragma unroll
      for (int c = 0; c < kKeys; c += 32) tmem_ld32_async(tmem + lanes + (st ? kTS1 : kTS0) + c, sr + c);
      tmem_wait_ld();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&sfree[st]);
      float* sv = reinterpret_cast<float*>(sr);  // raw scores; 1/sqrt(d) * log2(e) goes into the exponent
      if (j == qt) {  // causal diagonal: key j*128 + c > q is masked
#pragma unroll
        for (int c = 0; c < kKeys; ++c) sv[c] = (j * kKeys + c <= q) ? sv[c] : -FLT_MAX;
      }
      float t[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        t[i] = sv[i];
#pragma unroll
        for (int k = 1; k < 8; ++k) t[i] = fmaxf(t[i], sv[i + 16 * k]);
      }
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) t[i] = fmaxf(t[i], t[i + w]);
      const float m_new = fmaxf(m, t[0] * scale_log2);
      float rs[4] = {0.f, 0.f, 0.f, 0.f};
      uint32_t pk[kKeys / 2];
#pragma unroll
      for (int c = 0; c < kKeys; c += 2) {
        const float p0 = ex2(__fmaf_rn(sv[c], scale_log2, -m_new)), p1 = ex2(__fmaf_rn(sv[c + 1], scale_log2, -m_new));
        rs[(c >> 1) & 3] += p0 + p1;
        pk[c >> 1] = pack2(p0, p1);
      }
      l = l * ex2(m - m_new) + ((rs[0] + rs[1]) + (rs[2] + rs[3]));
      // P_j overwrites P_{j-1}: the MMA of O_{j-1} must be complete
      if (j > 0) {
        const int sp = (j - 1) & 1;
        mbar_wait(&ofull[sp], ((j - 1) >> 1) & 1);
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sP + a * kTile + r * 128 +
                                                                         ((ch ^ (r & 7)) << 4)),
                       "r"(pk[a * 32 + ch * 4]), "r"(pk[a * 32 + ch * 4 + 1]), "r"(pk[a * 32 + ch * 4 + 2]),
                       "r"(pk[a * 32 + ch * 4 + 3])
                       : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(pready);
      if (j > 0) take_o(j - 1, m_prev, m);
      m_prev = m;
      m = m_new;
    }
    take_o(nkt - 1, m_prev, m);
    if (q < n) {
      const float inv = 1.f / l;
      bf16* out = ctx + static_cast<int64_t>(s0 + q) * qd + h * kHD;
#pragma unroll
      for (int i = 0; i < kHD; i += 8) {
        uint4 v;
        v.x = pack2(acc[i] * inv, acc[i + 1] * inv);
        v.y = pack2(acc[i + 2] * inv, acc[i + 3] * inv);
        v.z = pack2(acc[i + 4] * inv, acc[i + 5] * inv);
        v.w = pack2(acc[i + 6] * inv, acc[i + 7] * inv);
        *reinterpret_cast<uint4*>(out + i) = v;
      }
      lse[static_cast<int64_t>(s0 + q) * nh + h] = (m + __log2f(l)) * 0.6931471805599453f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace

bool attn_fwd_tc5(cudaStream_t s, const bf16* qkv, const int32_t* seq_start, int n_seq, int max_len, int rows, int nh,
                  int nkv, int hd, bf16* ctx, float* lse) {
  if (hd != kHD || nh % nkv) return false;
  const char* force = getenv("DASHCU_ATTN_FWD");
  if (force && std::string(force) == "mma") return false;
  // one-tile sequences (the prompt prefill) amortise the per-CTA TMEM / barrier / first-load
  // latency poorly; the mma.sync kernel (several CTAs per SM) is faster there
  if (max_len <= 2 * kQ && !(force && std::string(force) == "tc5")) return false;
  const int qkvd = nh * hd + 2 * nkv * hd;
  CUtensorMap mq;
  if (!tma_map_2d(&mq, qkv, rows, qkvd, qkvd, kHD, 128, false, 128, true)) return false;
  static bool attr = false;
  if (!attr) {
    DCU_CHECK(cudaFuncSetAttribute(attn_fwd_tc5_k, cudaFuncAttributeMaxDynamicSharedMemorySize, FLay::BYTES));
    attr = true;
  }
  const int nqt = (max_len + kQ - 1) / kQ;
  dim3 grid(n_seq * nh, nqt);
  attn_fwd_tc5_k<<<grid, 256, FLay::BYTES, s>>>(mq, seq_start, nh, nkv, nqt, ctx, lse,
                                                1.4426950408889634f / sqrtf(static_cast<float>(hd)));
  DCU_LAUNCHED();
  return true;
}

}  // namespace dashcu
