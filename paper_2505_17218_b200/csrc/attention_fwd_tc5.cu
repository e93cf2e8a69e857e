// tcgen05 attention forward for head_dim 64 and 128 (teacher-forced causal attention of the
// training pass, policy.cpp:105-129; the mma.sync kernel in attention_tc.cu is the fallback).
//
// One CTA owns 128 queries of one sequence for every query head of a KV group (heads run
// back to back through one pipeline) and walks the causal key tiles (128 keys each) with an
// online softmax:
//   S_j = Q K_j^T          M128 N128 K=hd   A = Q (K-major, smem)  B = K_j (K-major)   -> TMEM S[j&1]
//   softmax warps: m = running row max of S/sqrt(d) (log2 domain), P_j = exp2(S_j/sqrt(d) - m)
//                  (bf16, written into TMEM with tcgen05.st)
//   O += P_j V_j           M128 N=hd K128   A = P_j (TMEM)          B = V_j (MN-major)  -> TMEM O
//   out = O / l, LSE = m + log l (l = sum of the bf16-rounded P the MMA consumed).
// Lazy rescaling: the max the exponentials use only moves when a row's true running max
// exceeds it by more than kRescale (log2 units); then that row's O (TMEM) and l are scaled
// by 2^(m_old - m_new) before the next PV. Otherwise P <= 2^kRescale, exact in the
// normalised result. No per-tile O round trip through registers, and P never touches
// shared memory. The MMA of S_{j+1} is issued as soon as the softmax warps hold S_j in
// registers, so it overlaps the softmax. Tiles of hd 128 are two 64-column swizzle atoms side
// by side (two TMA boxes).
// Warp roles: 0 TMA producer (Q once per head, K/V kST-stage ring), 1 TMEM allocator and
// MMA issuer, 2..9 softmax (TMEM lane quarter = warp % 4; two warps per quarter split the
// columns).
#include <cfloat>
#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "tc5.cuh"

namespace dashcu {

#if defined(DASHCU_ATTN_TRACE) && DASHCU_ATTN_TRACE == 2
// Debug builds only (-DDASHCU_ATTN_TRACE=2): clock64 timeline of CTA (0, 0), 16 slots per tile.
__device__ unsigned long long g_attn_trace[64 * 16];
#define TRF(t, k)                                                                             \
  do {                                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && (t) < 64)           \
      g_attn_trace[(t) * 16 + (k)] = clock64();                                               \
  } while (0)
int attn_trace_read(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#else
#define TRF(t, k) \
  do {            \
  } while (0)
#endif

namespace {

constexpr int kQ = 128, kKeys = 128;
// A quarter of the forward's exponentials via ex2_poly (tc5.cuh): its exp loop is bound by
// the MUFU unit (16 ex2 / clock / SM); measured -2.5 % (a half: +1.7 %, issue-bound).
// -DDASHCU_NO_SPLIT_EXP disables.
#ifndef DASHCU_NO_SPLIT_EXP
constexpr bool kSplitExp = true;
#else
constexpr bool kSplitExp = false;
#endif
#ifndef DASHCU_SPLIT_EVERY
#define DASHCU_SPLIT_EVERY 2
#endif
constexpr int kSplitEvery = DASHCU_SPLIT_EVERY;  // one pair in kSplitEvery uses ex2_poly for its odd element
constexpr int kAtom = 128 * 64 * 2;  // 16 KB: 128 rows x one 64-column (128-byte) swizzle atom

// hd 64: two CTAs per SM (~85 KB of shared memory and 256 TMEM columns each: one S buffer,
// O, P), so one CTA's exponentials run while the other's softmax warps load S, reduce the
// row max and store P (the exponential loop is MUFU-bound and the rest of a tile is not).
// hd 128: one CTA per SM with a double-buffered S.
template <int HD>
struct FLay {
  static constexpr int kCTAs = HD == 64 ? 2 : 1;  // CTAs per SM
  static constexpr int kTile = 128 * HD * 2;  // 16 / 32 KB: HD / 64 atoms
  static constexpr int kQS = 1;               // Q stages
  static constexpr int kST = 2;               // K/V pipeline depth (loads run kST - 1 key tiles ahead)
  static constexpr int kNSB = HD == 64 ? 1 : 2;  // S buffers in TMEM
  static constexpr int Q = 0, K = kQS * kTile, V = K + kST * kTile;
  static constexpr int XMAX = V + kST * kTile;  // row-max exchange [2][2][128] + row sums [2][128]
  static constexpr int BAR = XMAX + 4096;
  static constexpr int BYTES = BAR + 256 + 1024;
  static_assert(BYTES * kCTAs <= 232448, "exceeds the 227 KB of shared memory per SM");
  // TMEM columns: S buffer(s), O (HD columns), P (128 bf16 keys = 64 columns)
  static constexpr uint32_t TS1 = 128, TO = 128 * kNSB, TP = TO + HD;
  static constexpr uint32_t ALLOC = TP + 64 <= 256 ? 256 : 512;
  static_assert(ALLOC * kCTAs <= 512, "TMEM columns");
};
constexpr int kThreads = 320;  // warp 0 TMA, 1 TMEM allocation + MMA, 2..9 softmax

constexpr float kRescale = 8.f;  // lazy-rescale threshold (log2 units): P <= 256

// O += P V with A = P from TMEM (a_tmem: lane 0, first column of this K step)
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

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

template <int HD>
__global__ void __launch_bounds__(kThreads, FLay<HD>::kCTAs)
    attn_fwd_tc5_k(const __grid_constant__ CUtensorMap mQKV, const int32_t* __restrict__ seq_start, int nh, int nkv,
                   int nqt_max, bf16* __restrict__ ctx, float* __restrict__ lse, float scale_log2,
                   bf16* __restrict__ ctx_lo) {
  using FLay = dashcu::FLay<HD>;
  constexpr int kHD = HD, kTile = FLay::kTile, kST = FLay::kST, kQS = FLay::kQS, kNSB = FLay::kNSB;
  constexpr uint32_t kTS1 = FLay::TS1, kTO = FLay::TO, kTP = FLay::TP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // grid (sequence x KV head, query tile), the longest (last) query tiles launched first; the
  // CTA runs the tile for every query head of the KV group back to back, so the TMEM / barrier
  // set-up and the pipeline fill are paid once per group and K/V loads of the next head
  // stream in while the current head finishes
  // Query tiles with >= 3 causal key tiles split the group's heads over two CTAs (y = 2 qt'
  // + part), which halves the longest CTAs.
  const int sq = blockIdx.x / nkv, kvh = blockIdx.x % nkv;
  const int qt = nqt_max - 1 - static_cast<int>(blockIdx.y >> 1), part = blockIdx.y & 1;
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int q0 = qt * kQ;
  if (q0 >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp0 = nh / nkv, qd = nh * kHD, kvd = nkv * kHD;
  const int nkt = qt + 1;  // causal key tiles 0 .. qt per head
  const bool split = grp0 > 1 && nkt >= 3;
  if (!split && part) return;
  const int h_lo = split && part ? (grp0 + 1) / 2 : 0, h_hi = split && !part ? (grp0 + 1) / 2 : grp0;
  const int grp = h_hi - h_lo;     // heads run by this CTA: kvh * grp0 + h_lo + hh
  const int ntiles = grp * nkt;    // global tile counter t = head * nkt + key tile

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FLay::BAR);
  uint64_t *qfull = bar /*[2]*/, *qempty = bar + 2 /*[2]*/, *sfull = bar + 4 /*[2]*/, *sfree = bar + 6 /*[2]*/,
           *pready = bar + 8, *ofull = bar + 9 /*[1]*/, *kvfull = bar + 13 /*[kST]*/,
           *kvempty = bar + 13 + kST /*[kST]*/;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 13 + 2 * kST);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kST; ++i) {
      mbar_init(&kvfull[i], 1);
      mbar_init(&kvempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1);
      mbar_init(&sfull[i], 1);
      mbar_init(&sfree[i], 256);  // the 8 softmax warps
      mbar_init(&ofull[i], 1);
    }
    mbar_init(pready, 256);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mQKV)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(FLay::ALLOC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sQ = smem_u32(smem + FLay::Q), sK = smem_u32(smem + FLay::K), sV = smem_u32(smem + FLay::V);

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------------------------- TMA
      for (int hh = 0, t = 0; hh < grp; ++hh) {
        const int qs = hh % kQS;
        mbar_wait_sleep(&qempty[qs], ((hh / kQS) & 1) ^ 1);
        mbar_expect_tx(&qfull[qs], kTile);
#pragma unroll
        for (int a = 0; a < kHD / 64; ++a)
          tma_load_2d(smem + FLay::Q + qs * kTile + a * kAtom, &mQKV, &qfull[qs],
                      (kvh * grp0 + h_lo + hh) * kHD + a * 64, s0 + q0);
        for (int j = 0; j < nkt; ++j, ++t) {
          const int st = t % kST;
          mbar_wait_sleep(&kvempty[st], ((t / kST) & 1) ^ 1);
          mbar_expect_tx(&kvfull[st], 2 * kTile);
#pragma unroll
          for (int a = 0; a < kHD / 64; ++a) {
            tma_load_2d(smem + FLay::K + st * kTile + a * kAtom, &mQKV, &kvfull[st], qd + kvh * kHD + a * 64,
                        s0 + j * kKeys);
            tma_load_2d(smem + FLay::V + st * kTile + a * kAtom, &mQKV, &kvfull[st], qd + kvd + kvh * kHD + a * 64,
                        s0 + j * kKeys);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------------------------- MMA
      constexpr uint32_t I_S = idesc(128, false, false), I_O = idesc(kHD, false, true);
      auto issue_s = [&](int t) {
        const int sb = t % kNSB, st = t % kST, hh = t / nkt, j = t % nkt, qs = hh % kQS;
        if (t >= kNSB) mbar_wait_sleep(&sfree[sb], ((t / kNSB) - 1) & 1);  // softmax holds S_{t-kNSB} in registers
        if (j == 0) mbar_wait_sleep(&qfull[qs], (hh / kQS) & 1);
        mbar_wait_sleep(&kvfull[st], (t / kST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t k = sK + st * kTile, qa = sQ + qs * kTile;
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk) {  // 16-dim K step kk: atom kk / 4, 32-byte chunk kk % 4
          const uint32_t o = (kk >> 2) * kAtom + (kk & 3) * 32;
          umma_bf16(tmem + (sb ? kTS1 : 0u), smem_desc(qa + o, 16, 1024), smem_desc(k + o, 16, 1024), I_S, kk > 0);
        }
        umma_commit(&sfull[sb]);
        if (j == nkt - 1) umma_commit(&qempty[qs]);  // the head's last S: its Q tile is free
      };
      issue_s(0);
      for (int t = 0; t < ntiles; ++t) {
        const int st = t % kST, j = t % nkt;
        if (t + 1 < ntiles) issue_s(t + 1);
        TRF(t, 0);
        // P_t is in TMEM and every row of O is rescaled; the softmax waited for PV(t-1) (and
        // at a head's first tile it has read the previous head's O) before arriving
        mbar_wait_sleep(pready, t & 1);
        TRF(t, 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t v = sV + st * kTile;
#pragma unroll
        for (int kk = 0; kk < kKeys / 16; ++kk)  // 16 keys = 8 TMEM columns of P per K step
          umma_bf16_ts(tmem + kTO, tmem + kTP + kk * 8, smem_desc(v + kk * 2048, kAtom, 1024), I_O,
                       (j > 0 || kk > 0) ? 1u : 0u);  // V atoms kAtom apart along hd
        umma_commit(&kvempty[st]);
        umma_commit(&ofull[0]);
        TRF(t, 2);
      }
    }
  } else if (warp >= 2) {  // ---------------------------------------------------------- softmax
    // 8 warps: TMEM lane quarter qq = warp % 4 (query rows 32 qq ..), column half hf: keys
    // [64 hf, 64 hf + 64) of S and P, head dims [hd/2 hf, hd/2 hf + hd/2) of O. The two warps
    // of a quarter exchange their row maxima through shared memory once per tile (named
    // barrier 1 + qq, 64 threads); they take the same rescale decisions from the same maxima.
    const int qq = warp & 3, hf = (warp - 2) >> 2, r = qq * 32 + lane, q = q0 + r;
    const uint32_t lanes = static_cast<uint32_t>(qq * 32) << 16;
    const uint32_t o_cols = tmem + lanes + kTO + hf * (kHD / 2);
    float* xmax = reinterpret_cast<float*>(smem + FLay::XMAX);  // [2 parity][2 halves][128 rows]
    int t = 0;
    for (int hh = 0; hh < grp; ++hh) {
      const int h = kvh * grp0 + h_lo + hh;
      float m = -FLT_MAX, l = 0.f;  // the max the exponentials use (log2 domain), this half's sum
      for (int j = 0; j < nkt; ++j, ++t) {
        const int sb = t % kNSB;
        if (warp == 4) TRF(t, 4);
        mbar_wait_sleep(&sfull[sb], (t / kNSB) & 1);
        if (warp == 4) TRF(t, 5);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // S stays in TMEM until the exponentials are done: read once for the row max, then
        // again 32 keys at a time for the exponentials (64 live scores instead of 96+)
        const uint32_t s_cols = tmem + lanes + (sb ? kTS1 : 0u) + hf * 64;
        const bool diag = j == qt;  // causal diagonal: key j*128 + 64 hf + c > q is masked
        float tm[16];
        {
          uint32_t sr[64];
          tmem_ld32_async(s_cols, sr);
          tmem_ld32_async(s_cols + 32, sr + 32);
          tmem_wait_ld();
          float* sv = reinterpret_cast<float*>(sr);  // raw scores; 1/sqrt(d) * log2(e) goes into the exponent
          if (diag) {
#pragma unroll
            for (int c = 0; c < 64; ++c) sv[c] = (j * kKeys + hf * 64 + c <= q) ? sv[c] : -FLT_MAX;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) tm[i] = fmaxf(fmaxf(sv[i], sv[i + 16]), fmaxf(sv[i + 32], sv[i + 48]));
        }
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
          for (int i = 0; i < w; ++i) tm[i] = fmaxf(tm[i], tm[i + w]);
        // row max over both halves: publish, pair barrier, read the partner's
        float* xm = xmax + (t & 1) * 256;
        xm[hf * 128 + r] = tm[0];
        if (warp == 4) TRF(t, 6);
        asm volatile("bar.sync %0, 64;" ::"r"(1 + qq) : "memory");
        if (warp == 4) TRF(t, 7);
        const float m_true = fmaxf(m, fmaxf(tm[0], xm[(hf ^ 1) * 128 + r]) * scale_log2);
        const bool move = m_true > m + kRescale;  // first tile: m = -FLT_MAX
        const float m_new = move ? m_true : m;
        const float corr = move ? ex2(m - m_new) : 1.f;  // 0 on the first tile (l = 0)
        // PV(t-1) complete: P is free and O final for tile t-1 (normally long done: PV(t-1)
        // was issued when tile t-1's P arrived, before this tile's S load and row max)
        if (warp == 4) TRF(t, 8);
        if (t > 0) mbar_wait_sleep(&ofull[0], (t - 1) & 1);
        if (warp == 4) TRF(t, 9);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (j > 0 && __any_sync(0xffffffffu, move)) {  // rescale this half of the rows' O
#pragma unroll
          for (int ch = 0; ch < kHD / 64; ++ch) {
            uint32_t o[32];
            tmem_ld32_async(o_cols + ch * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
            tmem_st32(o_cols + ch * 32, o);
          }
        }
        uint64_t rs2[2] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
        const uint64_t sc2 = f2_pack(scale_log2, scale_log2), nm2 = f2_pack(-m_new, -m_new);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {  // 32 keys at a time: 16 TMEM columns of P per store
          uint32_t sr[32], pk[16];
          tmem_ld32_async(s_cols + 32 * h2, sr);
          tmem_wait_ld();
          float* sv = reinterpret_cast<float*>(sr) - 32 * h2;  // sv[c] for c in [32 h2, 32 h2 + 32)
          if (diag) {
#pragma unroll
            for (int c = 32 * h2; c < 32 * h2 + 32; ++c) sv[c] = (j * kKeys + hf * 64 + c <= q) ? sv[c] : -FLT_MAX;
          }
#pragma unroll
          for (int c = 32 * h2; c < 32 * h2 + 32; c += 2) {  // exponent arguments and row sums on the fp32x2 pipe
            float a0, a1;
            f2_unpack(f2_fma(f2_pack(sv[c], sv[c + 1]), sc2, nm2), a0, a1);
            const float p0 = ex2(a0);
            // a fraction of the exponentials on the FMA pipe (the exp loop is MUFU-bound)
            const float p1 = (kSplitExp && ((c >> 1) % kSplitEvery == 0)) ? ex2_poly(a1) : ex2(a1);
            const uint32_t pp = pack2(p0, p1);
            pk[(c >> 1) & 15] = pp;
            // the row sum adds the bf16-rounded values the PV product consumes (O / l consistent)
            rs2[(c >> 1) & 1] =
                f2_add(rs2[(c >> 1) & 1], f2_pack(__uint_as_float(pp << 16), __uint_as_float(pp & 0xffff0000u)));
          }
          tmem_st16(tmem + lanes + kTP + hf * 32 + h2 * 16, pk);  // keys [64 hf + 32 h2, +32)
        }
        float r0, r1, r2, r3;
        f2_unpack(rs2[0], r0, r1);
        f2_unpack(rs2[1], r2, r3);
        l = l * corr + ((r0 + r1) + (r2 + r3));  // this half's share of the row sum
        m = m_new;
        tmem_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&sfree[sb]);  // S read for the last time: the next S may overwrite it
        mbar_arrive(pready);
        if (warp == 4) TRF(t, 10);
      }
      // the head's O: wait for its last PV, read this half's head dims
      mbar_wait_sleep(&ofull[0], (t - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float acc[kHD / 2];
#pragma unroll
      for (int ch = 0; ch < kHD / 64; ++ch) {
        uint32_t o[32];
        tmem_ld32_async(o_cols + ch * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[ch * 32 + i] = __uint_as_float(o[i]);
      }
      // (the next head's first PV overwrites O only after this thread's next pready arrive)
      // full row sum = both halves' shares (same running max in both)
      float* xl = xmax + 512;
      xl[hf * 128 + r] = l;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + qq) : "memory");
      const float lt = l + xl[(hf ^ 1) * 128 + r];
      asm volatile("bar.sync %0, 64;" ::"r"(1 + qq) : "memory");  // xl reused by the next head
      if (q < n) {
        const float inv = 1.f / lt;
        bf16* out = ctx + static_cast<int64_t>(s0 + q) * qd + h * kHD + hf * (kHD / 2);
#pragma unroll
        for (int i = 0; i < kHD / 2; i += 8) {
          uint4 v;
          v.x = pack2(acc[i] * inv, acc[i + 1] * inv);
          v.y = pack2(acc[i + 2] * inv, acc[i + 3] * inv);
          v.z = pack2(acc[i + 4] * inv, acc[i + 5] * inv);
          v.w = pack2(acc[i + 6] * inv, acc[i + 7] * inv);
          *reinterpret_cast<uint4*>(out + i) = v;
          if (ctx_lo) {  // O - bf16(O), for the backward's D
            const uint32_t hv[4] = {v.x, v.y, v.z, v.w};
            uint32_t lv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              lv[k] = pack2(acc[i + 2 * k] * inv - __uint_as_float(hv[k] << 16),
                            acc[i + 2 * k + 1] * inv - __uint_as_float(hv[k] & 0xffff0000u));
            *reinterpret_cast<uint4*>(ctx_lo + (out - ctx) + i) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
          }
        }
        if (hf == 0) lse[static_cast<int64_t>(s0 + q) * nh + h] = (m + __log2f(lt)) * 0.6931471805599453f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(FLay::ALLOC));
}

}  // namespace

namespace {
template <int HD>
void launch_fwd_tc5(cudaStream_t s, const CUtensorMap& mq, const int32_t* seq_start, int n_seq, int nqt, int nh,
                    int nkv, bf16* ctx, float* lse, bf16* ctx_lo) {
  static bool attr = false;
  if (!attr) {
    DCU_CHECK(cudaFuncSetAttribute(attn_fwd_tc5_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, FLay<HD>::BYTES));
    attr = true;
  }
  dim3 grid(n_seq * nkv, 2 * nqt);
  attn_fwd_tc5_k<HD><<<grid, kThreads, FLay<HD>::BYTES, s>>>(mq, seq_start, nh, nkv, nqt, ctx, lse,
                                                        1.4426950408889634f / sqrtf(static_cast<float>(HD)), ctx_lo);
  DCU_LAUNCHED();
}
}  // namespace

bool attn_fwd_tc5(cudaStream_t s, const bf16* qkv, const int32_t* seq_start, int n_seq, int max_len, int rows, int nh,
                  int nkv, int hd, bf16* ctx, float* lse, bf16* ctx_lo) {
  if ((hd != 64 && hd != 128) || nh % nkv) return false;
  const int force = knob(KNOB_ATTN_FWD);
  if (force == 1) return false;
  // one-tile sequences (the prompt prefill) amortise the per-CTA TMEM / barrier / first-load
  // latency poorly; the mma.sync kernel (several CTAs per SM) is faster there
  if (max_len <= 2 * kQ && force != 2) return false;
  const int qkvd = nh * hd + 2 * nkv * hd;
  CUtensorMap mq;
  if (!tma_map_2d(&mq, qkv, rows, qkvd, qkvd, 64, 128, false, 128, true)) return false;  // one swizzle atom per box
  const int nqt = (max_len + kQ - 1) / kQ;
  if (hd == 64)
    launch_fwd_tc5<64>(s, mq, seq_start, n_seq, nqt, nh, nkv, ctx, lse, ctx_lo);
  else
    launch_fwd_tc5<128>(s, mq, seq_start, n_seq, nqt, nh, nkv, ctx, lse, ctx_lo);
  return true;
}

}  // namespace dashcu
