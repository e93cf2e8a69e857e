// Tensor-core attention for the bf16 path (sm_100a, mma.sync m16n8k16 tiles).
//
// decode  (policy.cpp:105-129 at one new position per sequence): one warp per
//         (sequence, kv head). The GRP query heads that share a KV head form one
//         16-row query tile, so every K/V byte of the cache is read from HBM once
//         (GQA); keys stream through a 3-stage cp.async ring in shared memory
//         (XOR-swizzled, ldmatrix), online softmax in fp32 registers.
#include <cfloat>

#include "kernels.cuh"
#include "mma.cuh"

namespace dashcu {

namespace {

constexpr float kLog2e = 1.4426950408889634f;

#ifndef DASHCU_DEC_ST
#define DASHCU_DEC_ST 2  // measured 3.6 % faster than 3 stages at 384 steps (r1)
#endif

// 32-key chunks, 2 warps per CTA (32 KB of ring at head_dim 64: 12 warps per SM). Same-box
// A/B at C2 (1024 decode steps, tools/ab_dec.sh): decode attention 4780 ms with 64-key
// chunks (6 warps per SM), 4637 ms with 32-key chunks, 4875 ms with 16-key chunks; two
// 64-key warps per item (split walk) or 3 stages lose 22 % (fewer warps per SM). Head_dim
// 128 with 16-key chunks (12 instead of 6 warps per SM, 168 registers): C3 decode attention
// 5357 -> 6092 ms, slower.
template <int HD>
struct DecCfg {
  static constexpr int KC = 32;                   // keys per chunk (divides kPage)
  static constexpr int ST = DASHCU_DEC_ST;       // pipeline stages (per warp)
  static constexpr int NW = 2;                    // warps per CTA
  static constexpr int UNITS = HD / 8;      // 16-byte units per key row
  static constexpr int CHUNK_BYTES = KC * HD * 2;
  static constexpr int WARP_BYTES = ST * 2 * CHUNK_BYTES;  // K and V
  static constexpr int SMEM = NW * WARP_BYTES;
};

// The completion KV stream (GBs per decode step) is loaded with an L2 evict-first policy so
// it does not evict the next GEMMs' weights and activations (-DDASHCU_DECODE_KV_NORMAL: A/B).
#ifndef DASHCU_DECODE_KV_NORMAL
constexpr bool kStreamKV = true;
#else
constexpr bool kStreamKV = false;
#endif

// append: the warp first stores its (row, kv head)'s new K / V row (qkv columns qd.. and
// qd + kvd..) into completion slot n_comp - 1, the separate kv_append kernel's work.
template <int HD>
__global__ void __launch_bounds__(DecCfg<HD>::NW * 32)
    attn_decode_tc_k(const bf16* __restrict__ qkv, const bf16* __restrict__ kp, const bf16* __restrict__ vp,
                     bf16* kc, bf16* vc, const int32_t* __restrict__ prompt_len, int S, int G, int pmax,
                     int n_comp, DecodeRows dr, int nh, int nkv, bf16* __restrict__ ctx, float scale_log2,
                     bool append) {
  using Cf = DecCfg<HD>;
  constexpr int KC = Cf::KC, ST = Cf::ST, UNITS = Cf::UNITS;
  pdl_wait();
  if (dr.step) n_comp = *dr.step;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * Cf::NW + warp;
  if (item >= S * nkv) return;
  const int s = item / nkv, kvh = item % nkv;  // s: decode row
  const int sq = dr_seq(dr, s);
  const int grp = nh / nkv, qd = nh * HD, kvd = nkv * HD, qkvd = qd + 2 * kvd;
  const int m = prompt_len[sq];
  const bf16* kpb = kp + (static_cast<int64_t>(sq / G) * nkv + kvh) * pmax * HD;
  const bf16* vpb = vp + (static_cast<int64_t>(sq / G) * nkv + kvh) * pmax * HD;
  // the sequence's page-table row, one entry per lane (completion <= 32 pages = 2048 slots);
  // longer rows read the table directly
  const bool shfl_pages = dr.max_pages <= 32;
  const uint64_t stream_pol = l2_policy_evict_first();
  const int32_t lane_page =
      shfl_pages && lane < dr.max_pages ? __ldg(dr.ptab + static_cast<int64_t>(sq) * dr.max_pages + lane) : 0;
  uint8_t* wsm = smem + warp * Cf::WARP_BYTES;
  const uint32_t wsm_a = smem_addr(wsm);
  if (append) {  // HD / 2 words of K and of V, one or two per lane
    const int slot = n_comp - 1;
    const int page = shfl_pages ? __shfl_sync(0xffffffffu, lane_page, (slot / kPage) & 31)
                                : __ldg(dr.ptab + static_cast<int64_t>(sq) * dr.max_pages + slot / kPage);
    const int64_t dst = ((static_cast<int64_t>(page) * nkv + kvh) * kPage + slot % kPage) * HD;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(qkv + static_cast<int64_t>(s) * qkvd + qd +
                                                            static_cast<int64_t>(kvh) * HD);
#pragma unroll
    for (int w = lane; w < HD / 2; w += 32) {
      reinterpret_cast<uint32_t*>(kc + dst)[w] = src[w];
      reinterpret_cast<uint32_t*>(vc + dst)[w] = src[w + kvd / 2];
    }
    __threadfence_block();  // the slot is read back below through cp.async by other lanes
    __syncwarp();
  }

  // Query tile: rows r < grp are the heads kvh*grp + r.
  const int g = lane >> 2, t = lane & 3;
  uint32_t qf[HD / 16][4];
  {
    const bf16* q0 = qkv + static_cast<int64_t>(s) * qkvd + static_cast<int64_t>(kvh) * grp * HD;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int c = kk * 16 + t * 2;
      auto ld = [&](int r, int col) -> uint32_t {
        return r < grp ? *reinterpret_cast<const uint32_t*>(q0 + static_cast<int64_t>(r) * HD + col) : 0u;
      };
      qf[kk][0] = ld(g, c);
      qf[kk][1] = ld(g + 8, c);
      qf[kk][2] = ld(g, c + 8);
      qf[kk][3] = ld(g + 8, c + 8);
    }
  }

  // chunks: cpm over the prompt keys [0, m), then chunks over the completion slots
  // [0, n_comp) aligned to slot 0, so a completion chunk (KC | kPage) lies in one page
  const int cpm = (m + KC - 1) / KC;
  auto chunk_keys = [&](int c, int* first) {  // first key / slot of chunk c and its bound
    *first = (c < cpm ? c : c - cpm) * KC;
    return c < cpm ? m : n_comp;
  };
  auto load_chunk = [&](int c, int stage) {
    const uint32_t kbase = wsm_a + stage * 2 * Cf::CHUNK_BYTES, vbase = kbase + Cf::CHUNK_BYTES;
    int first;
    const int lim = chunk_keys(c, &first);
    const bf16 *kb, *vb;
    if (c < cpm) {
      kb = kpb + static_cast<int64_t>(first) * HD;
      vb = vpb + static_cast<int64_t>(first) * HD;
    } else {
      const int page = shfl_pages ? __shfl_sync(0xffffffffu, lane_page, (first / kPage) & 31)
                                  : __ldg(dr.ptab + static_cast<int64_t>(sq) * dr.max_pages + first / kPage);
      const int64_t po = ((static_cast<int64_t>(page) * nkv + kvh) * kPage + first % kPage) * HD;
      kb = kc + po;
      vb = vc + po;
    }
#pragma unroll
    for (int i = 0; i < KC * UNITS / 32; ++i) {
      const int idx = lane + i * 32;
      const int r = idx / UNITS, u = idx % UNITS;
      const bool ok = first + r < lim;
      const int64_t ro = ok ? static_cast<int64_t>(r) * HD + u * 8 : 0;
      const int off = swz(r, u, UNITS);
      if (c < cpm || !kStreamKV) {  // the group's prompt KV: read by its G sequences, keep in L2
        cp_async16(kbase + off, kb + ro, ok ? 16 : 0);
        cp_async16(vbase + off, vb + ro, ok ? 16 : 0);
      } else {  // this sequence's completion KV: read once per step, evict first
        cp_async16_hint(kbase + off, kb + ro, ok ? 16 : 0, stream_pol);
        cp_async16_hint(vbase + off, vb + ro, ok ? 16 : 0, stream_pol);
      }
    }
  };

  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-FLT_MAX, -FLT_MAX}, lrow[2] = {0.f, 0.f};

  const int nch = cpm + (n_comp + KC - 1) / KC;
#pragma unroll
  for (int c = 0; c < ST - 1; ++c) {
    if (c < nch) load_chunk(c, c);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    __syncwarp();
    if (c + ST - 1 < nch) load_chunk(c + ST - 1, (c + ST - 1) % ST);
    cp_async_commit();
    cp_async_wait<ST - 1>();
    __syncwarp();
    const int stage = c % ST;
    const uint32_t kbase = wsm_a + stage * 2 * Cf::CHUNK_BYTES, vbase = kbase + Cf::CHUNK_BYTES;

    float sc[KC / 8][4];
#pragma unroll
    for (int nt = 0; nt < KC / 8; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; kk += 2) {
        const int key = nt * 8 + (lane & 7);
        const int u = kk * 2 + (lane >> 3);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kbase + swz(key, u, UNITS), b0, b1, b2, b3);
        mma_bf16_16816(sc[nt], qf[kk], b0, b1);
        mma_bf16_16816(sc[nt], qf[kk + 1], b2, b3);
      }
    }
    // scale into the log2 domain, mask keys past the end, online softmax
    float cmax[2] = {-FLT_MAX, -FLT_MAX};
    int cfirst;
    const int clim = chunk_keys(c, &cfirst);
#pragma unroll
    for (int nt = 0; nt < KC / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = cfirst + nt * 8 + t * 2 + (e & 1);
        const float v = key < clim ? sc[nt][e] * scale_log2 : -FLT_MAX;
        sc[nt][e] = v;
        cmax[e >> 1] = fmaxf(cmax[e >> 1], v);
      }
    }
    float corr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 1));
      cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 2));
      const float mn = fmaxf(mrow[h], cmax[h]);
      corr[h] = exp2f(mrow[h] - mn);
      mrow[h] = mn;
      lrow[h] *= corr[h];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
#pragma unroll
    for (int nt = 0; nt < KC / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(sc[nt][e] - mrow[e >> 1]);
        sc[nt][e] = p;
        lrow[e >> 1] += p;
      }
    }
    // O += P V
#pragma unroll
    for (int kc2 = 0; kc2 < KC / 16; ++kc2) {
      uint32_t a[4];
      a[0] = pack_bf16(sc[2 * kc2][0], sc[2 * kc2][1]);
      a[1] = pack_bf16(sc[2 * kc2][2], sc[2 * kc2][3]);
      a[2] = pack_bf16(sc[2 * kc2 + 1][0], sc[2 * kc2 + 1][1]);
      a[3] = pack_bf16(sc[2 * kc2 + 1][2], sc[2 * kc2 + 1][3]);
#pragma unroll
      for (int nt2 = 0; nt2 < HD / 8; nt2 += 2) {
        const int mi = lane >> 3;
        const int key = kc2 * 16 + (mi & 1) * 8 + (lane & 7);
        const int u = nt2 + (mi >> 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vbase + swz(key, u, UNITS), b0, b1, b2, b3);
        mma_bf16_16816(o[nt2], a, b0, b1);
        mma_bf16_16816(o[nt2 + 1], a, b2, b3);
      }
    }
  }
  cp_async_wait<0>();
  // every key is in: the next kernel (the W_o GEMM) may launch and set up on idle SMs; its
  // pdl_wait() still waits for this grid's ctx stores
  pdl_trigger();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 1);
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 2);
    lrow[h] = 1.f / lrow[h];
  }
  bf16* out = ctx + static_cast<int64_t>(s) * qd + static_cast<int64_t>(kvh) * grp * HD;
#pragma unroll
  for (int nt2 = 0; nt2 < HD / 8; ++nt2) {
    const int col = nt2 * 8 + t * 2;
    if (g < grp)
      *reinterpret_cast<uint32_t*>(out + static_cast<int64_t>(g) * HD + col) =
          pack_bf16(o[nt2][0] * lrow[0], o[nt2][1] * lrow[0]);
    if (g + 8 < grp)
      *reinterpret_cast<uint32_t*>(out + static_cast<int64_t>(g + 8) * HD + col) =
          pack_bf16(o[nt2][2] * lrow[1], o[nt2][3] * lrow[1]);
  }
}

template <int HD>
void launch_decode(cudaStream_t s, const bf16* qkv, const bf16* kp, const bf16* vp, bf16* kc, bf16* vc,
                   const int32_t* plen, int rows, int G, int pmax, int n_comp, const DecodeRows& dr, int nh, int nkv,
                   bf16* ctx, bool append) {
  using Cf = DecCfg<HD>;
  static bool attr = false;
  if (!attr) {
    DCU_CHECK(cudaFuncSetAttribute(attn_decode_tc_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    attr = true;
  }
  const int items = rows * nkv;
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(HD));
  launch_pdl(attn_decode_tc_k<HD>, dim3((items + Cf::NW - 1) / Cf::NW), dim3(Cf::NW * 32), Cf::SMEM, s, qkv, kp,
             vp, kc, vc, plen, rows, G, pmax, n_comp, dr, nh, nkv, ctx, scale_log2, append);
  DCU_LAUNCHED();
}

// ============================================================== forward (prefill / teacher-forced)
// grid (q tiles, sequences, query heads); 4 warps x 16 query rows. K/V tiles of
// 64 keys double-buffered through cp.async; causal + length masking; writes
// ctx (bf16) and the natural-log LSE per (row, head) for the backward pass.
template <int HD>
struct FwdCfg {
  static constexpr int BQ = 64, BKV = 64, UNITS = HD / 8;
  static constexpr int TILE = 64 * HD * 2;
  static constexpr int SMEM = TILE /*Q*/ + 2 * 2 * TILE /*K,V x 2 stages*/;
};

template <int HD>
__global__ void __launch_bounds__(128) attn_fwd_tc_k(const bf16* __restrict__ qkv, const int32_t* __restrict__ seq_start,
                                                     int nh, int nkv, bf16* __restrict__ ctx, float* __restrict__ lse,
                                                     float scale_log2, bf16* __restrict__ ctx_lo) {
  using Cf = FwdCfg<HD>;
  constexpr int UNITS = Cf::UNITS;
  extern __shared__ __align__(128) uint8_t smem[];
  const int qt = blockIdx.x, sq = blockIdx.y, h = blockIdx.z;
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int q0 = qt * 64;
  if (q0 >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int grp = nh / nkv, kvh = h / grp;
  const int qd = nh * HD, kvd = nkv * HD, qkvd = qd + 2 * kvd;
  const uint32_t sQ = smem_addr(smem), sKV = sQ + Cf::TILE;

  auto load_tile = [&](uint32_t dst, int row0, int col) {  // 64 rows x HD from qkv column `col`
#pragma unroll
    for (int i = 0; i < 64 * UNITS / 128; ++i) {
      const int idx = threadIdx.x + i * 128;
      const int r = idx / UNITS, u = idx % UNITS;
      const bool ok = row0 + r < n;
      const bf16* src = qkv + static_cast<int64_t>(s0 + (ok ? row0 + r : 0)) * qkvd + col + u * 8;
      cp_async16(dst + swz(r, u, UNITS), src, ok ? 16 : 0);
    }
  };
  const int nkt = (min(n, q0 + 64) + 63) / 64;  // causal: keys < q0 + 64
  load_tile(sQ, q0, h * HD);
  load_tile(sKV, 0, qd + kvh * HD);
  load_tile(sKV + Cf::TILE, 0, qd + kvd + kvh * HD);
  cp_async_commit();

  uint32_t qf[HD / 16][4];
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-FLT_MAX, -FLT_MAX}, lrow[2] = {0.f, 0.f};
  const int qr0 = q0 + warp * 16;  // this warp's first query row (sequence-relative)

  for (int kt = 0; kt < nkt; ++kt) {
    const int stage = kt & 1;
    if (kt + 1 < nkt) {
      const uint32_t nb = sKV + (stage ^ 1) * 2 * Cf::TILE;
      load_tile(nb, (kt + 1) * 64, qd + kvh * HD);
      load_tile(nb + Cf::TILE, (kt + 1) * 64, qd + kvd + kvh * HD);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int r = warp * 16 + (lane & 15), u = kk * 2 + (lane >> 4);
        ldsm_x4(sQ + swz(r, u, UNITS), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint32_t kb = sKV + stage * 2 * Cf::TILE, vb = kb + Cf::TILE;
    float sc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; kk += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kb + swz(nt * 8 + (lane & 7), kk * 2 + (lane >> 3), UNITS), b0, b1, b2, b3);
        mma_bf16_16816(sc[nt], qf[kk], b0, b1);
        mma_bf16_16816(sc[nt], qf[kk + 1], b2, b3);
      }
    }
    float cmax[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kt * 64 + nt * 8 + t * 2 + (e & 1);
        const int qr = qr0 + g + (e >> 1) * 8;
        const float v = (key <= qr && key < n) ? sc[nt][e] * scale_log2 : -FLT_MAX;
        sc[nt][e] = v;
        cmax[e >> 1] = fmaxf(cmax[e >> 1], v);
      }
    float corr[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      cmax[hh] = fmaxf(cmax[hh], __shfl_xor_sync(0xffffffffu, cmax[hh], 1));
      cmax[hh] = fmaxf(cmax[hh], __shfl_xor_sync(0xffffffffu, cmax[hh], 2));
      const float mn = fmaxf(mrow[hh], cmax[hh]);
      corr[hh] = exp2f(mrow[hh] - mn);
      mrow[hh] = mn;
      lrow[hh] *= corr[hh];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // rounded to bf16 here, as the PV product consumes it, so the normaliser matches O
        const float p = sc[nt][e] == -FLT_MAX ? 0.f : __bfloat162float(__float2bfloat16_rn(exp2f(sc[nt][e] - mrow[e >> 1])));
        sc[nt][e] = p;
        lrow[e >> 1] += p;
      }
#pragma unroll
    for (int kc2 = 0; kc2 < 4; ++kc2) {
      uint32_t a[4];
      a[0] = pack_bf16(sc[2 * kc2][0], sc[2 * kc2][1]);
      a[1] = pack_bf16(sc[2 * kc2][2], sc[2 * kc2][3]);
      a[2] = pack_bf16(sc[2 * kc2 + 1][0], sc[2 * kc2 + 1][1]);
      a[3] = pack_bf16(sc[2 * kc2 + 1][2], sc[2 * kc2 + 1][3]);
#pragma unroll
      for (int nt2 = 0; nt2 < HD / 8; nt2 += 2) {
        const int mi = lane >> 3;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vb + swz(kc2 * 16 + (mi & 1) * 8 + (lane & 7), nt2 + (mi >> 1), UNITS), b0, b1, b2, b3);
        mma_bf16_16816(o[nt2], a, b0, b1);
        mma_bf16_16816(o[nt2 + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    lrow[hh] += __shfl_xor_sync(0xffffffffu, lrow[hh], 1);
    lrow[hh] += __shfl_xor_sync(0xffffffffu, lrow[hh], 2);
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int qr = qr0 + g + hh * 8;
    if (qr >= n) continue;
    const float inv = 1.f / lrow[hh];
    bf16* out = ctx + static_cast<int64_t>(s0 + qr) * qd + h * HD;
#pragma unroll
    for (int nt2 = 0; nt2 < HD / 8; ++nt2) {
      const float v0 = o[nt2][2 * hh] * inv, v1 = o[nt2][2 * hh + 1] * inv;
      const uint32_t hi = pack_bf16(v0, v1);
      *reinterpret_cast<uint32_t*>(out + nt2 * 8 + t * 2) = hi;
      if (ctx_lo) {
        const __nv_bfloat162 h2 = *reinterpret_cast<const __nv_bfloat162*>(&hi);
        *reinterpret_cast<uint32_t*>(ctx_lo + (out - ctx) + nt2 * 8 + t * 2) =
            pack_bf16(v0 - __low2float(h2), v1 - __high2float(h2));
      }
    }
    if (t == 0) lse[static_cast<int64_t>(s0 + qr) * nh + h] = (mrow[hh] + log2f(lrow[hh])) * 0.6931471805599453f;
  }
}

// D[row][h] = sum_i dO[row][h][i] * O[row][h][i]   (the reference's wsum, policy.cpp:298-304)
__global__ void attn_bwd_dot_k(const bf16* __restrict__ dctx, const bf16* __restrict__ ctx,
                               const bf16* __restrict__ ctx_lo, int rows, int nh, int hd, float* __restrict__ D) {
  const int64_t n = static_cast<int64_t>(rows) * nh;
  const int lane = threadIdx.x & 31;
  if (hd % 8 == 0 && hd <= 256 && 32 % (hd / 8) == 0) {
    // 16-byte loads: hd / 8 lanes per (row, head), 32 / (hd / 8) pairs per warp iteration
    const int lpp = hd / 8, ppw = 32 / lpp, sub = lane / lpp, li = lane % lpp;
    for (int64_t w0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * ppw; w0 < n;
         w0 += ((gridDim.x * (int64_t)blockDim.x) >> 5) * ppw) {
      const int64_t w = w0 + sub;
      float s = 0.f;
      if (w < n) {
        const int64_t o = w * hd + li * 8;
        const uint4 ua = *reinterpret_cast<const uint4*>(dctx + o);
        const uint4 ub = *reinterpret_cast<const uint4*>(ctx + o);
        const uint4 uc = ctx_lo ? *reinterpret_cast<const uint4*>(ctx_lo + o) : make_uint4(0, 0, 0, 0);
        const bf16* a = reinterpret_cast<const bf16*>(&ua);
        const bf16* b = reinterpret_cast<const bf16*>(&ub);
        const bf16* c = reinterpret_cast<const bf16*>(&uc);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          s += __bfloat162float(a[i]) * (__bfloat162float(b[i]) + __bfloat162float(c[i]));
      }
      for (int off = lpp / 2; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (li == 0 && w < n) D[w] = s;
    }
    return;
  }
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * (int64_t)blockDim.x) >> 5) {
    const bf16* a = dctx + w * hd;
    const bf16* b = ctx + w * hd;
    float s = 0.f;
    for (int i = lane; i < hd; i += 32)
      s += __bfloat162float(a[i]) * (__bfloat162float(b[i]) + (ctx_lo ? __bfloat162float(ctx_lo[w * hd + i]) : 0.f));
    s = warp_sum(s);
    if (lane == 0) D[w] = s;
  }
}

// ============================================================== backward
// grid (key tiles, sequences, kv heads); 4 warps x 16 keys of a 64-key tile.
// For every query head of the KV group and every causal query tile:
//   S^T = K Q^T, P^T = exp(S^T - LSE), dV += P^T dO, dP^T = V dO^T,
//   dS^T = P^T (dP^T - D), dK += dS^T Q, dQ += dS K (fp32 atomics).
// dK/dV stay in registers across the whole group (GQA sum without atomics).
template <int HD>
struct BwdCfg {
  static constexpr int UNITS = HD / 8;
  static constexpr int TILE = 64 * HD * 2;
  static constexpr int SMEM = 4 * TILE /*K V Q dO*/ + 64 * 64 * 2 /*dS^T*/ + 2 * 64 * 4 /*lse, D*/;
};

template <int HD>
__global__ void __launch_bounds__(128) attn_bwd_tc_k(const bf16* __restrict__ qkv, const bf16* __restrict__ dctx,
                                                     const float* __restrict__ lse, const float* __restrict__ Dsum,
                                                     const int32_t* __restrict__ seq_start, int nh, int nkv,
                                                     float* __restrict__ dq32, float* __restrict__ dkv32, float scale,
                                                     float scale_log2) {
  using Cf = BwdCfg<HD>;
  constexpr int UNITS = Cf::UNITS;
  extern __shared__ __align__(128) uint8_t smem[];
  const int kt = blockIdx.x, sq = blockIdx.y, kvh = blockIdx.z;
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int k0 = kt * 64;
  if (k0 >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int grp = nh / nkv;
  const int qd = nh * HD, kvd = nkv * HD, qkvd = qd + 2 * kvd;
  const uint32_t sK = smem_addr(smem), sV = sK + Cf::TILE, sQ = sV + Cf::TILE, sO = sQ + Cf::TILE,
                 sS = sO + Cf::TILE;
  float* sL = reinterpret_cast<float*>(smem + 4 * Cf::TILE + 64 * 64 * 2);
  float* sD = sL + 64;

  auto load_tile = [&](uint32_t dst, const bf16* base, int64_t ld, int row0) {
#pragma unroll
    for (int i = 0; i < 64 * UNITS / 128; ++i) {
      const int idx = threadIdx.x + i * 128;
      const int r = idx / UNITS, u = idx % UNITS;
      const bool ok = row0 + r < n;
      const bf16* src = base + static_cast<int64_t>(s0 + (ok ? row0 + r : 0)) * ld + u * 8;
      cp_async16(dst + swz(r, u, UNITS), src, ok ? 16 : 0);
    }
  };
  load_tile(sK, qkv + qd + kvh * HD, qkvd, k0);
  load_tile(sV, qkv + qd + kvd + kvh * HD, qkvd, k0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int kr0 = k0 + warp * 16;  // this warp's first key (sequence-relative)
  const int nqt = (n + 63) / 64;

  for (int hh = 0; hh < grp; ++hh) {
    const int h = kvh * grp + hh;
    for (int qt = kt; qt < nqt; ++qt) {
      const int q0 = qt * 64;
      __syncthreads();  // previous iteration done with sQ / sO / sS
      load_tile(sQ, qkv + h * HD, qkvd, q0);
      load_tile(sO, dctx + h * HD, qd, q0);
      cp_async_commit();
      if (threadIdx.x < 64) {
        const int q = q0 + threadIdx.x;
        sL[threadIdx.x] = q < n ? lse[static_cast<int64_t>(s0 + q) * nh + h] * 1.4426950408889634f : 0.f;
        sD[threadIdx.x] = q < n ? Dsum[static_cast<int64_t>(s0 + q) * nh + h] : 0.f;
      }
      cp_async_wait<0>();
      __syncthreads();
      // S^T [16 keys x 64 q] and dP^T
      float st_[8][4], dp[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) st_[nt][e] = dp[nt][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        // this warp's 16 keys of K and V (A operands), re-read from smem to bound registers
        uint32_t kf[4], vf[4];
        const int ra = warp * 16 + (lane & 15), ua = kk * 2 + (lane >> 4);
        ldsm_x4(sK + swz(ra, ua, UNITS), kf[0], kf[1], kf[2], kf[3]);
        ldsm_x4(sV + swz(ra, ua, UNITS), vf[0], vf[1], vf[2], vf[3]);
#pragma unroll
        for (int nt = 0; nt < 8; nt += 2) {
          // B fragments for query n-tiles nt, nt+1 at k-chunk kk
          const int mi = lane >> 3;
          const int qrow = (nt + (mi >> 1)) * 8 + (lane & 7), ub = kk * 2 + (mi & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(sQ + swz(qrow, ub, UNITS), b0, b1, b2, b3);
          mma_bf16_16816(st_[nt], kf, b0, b1);
          mma_bf16_16816(st_[nt + 1], kf, b2, b3);
          ldsm_x4(sO + swz(qrow, ub, UNITS), b0, b1, b2, b3);
          mma_bf16_16816(dp[nt], vf, b0, b1);
          mma_bf16_16816(dp[nt + 1], vf, b2, b3);
        }
      }
      // P^T and dS^T (rows = keys g / g+8, cols = queries)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int qc = nt * 8 + t * 2 + (e & 1);
          const int q = q0 + qc;
          const int key = kr0 + g + (e >> 1) * 8;
          const bool ok = q < n && key <= q && key < n;
          const float p = ok ? exp2f(st_[nt][e] * scale_log2 - sL[qc]) : 0.f;
          st_[nt][e] = p;
          dp[nt][e] = p * (dp[nt][e] - sD[qc]) * scale;
        }
      // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
      for (int kc2 = 0; kc2 < 4; ++kc2) {
        uint32_t ap[4], as[4];
        ap[0] = pack_bf16(st_[2 * kc2][0], st_[2 * kc2][1]);
        ap[1] = pack_bf16(st_[2 * kc2][2], st_[2 * kc2][3]);
        ap[2] = pack_bf16(st_[2 * kc2 + 1][0], st_[2 * kc2 + 1][1]);
        ap[3] = pack_bf16(st_[2 * kc2 + 1][2], st_[2 * kc2 + 1][3]);
        as[0] = pack_bf16(dp[2 * kc2][0], dp[2 * kc2][1]);
        as[1] = pack_bf16(dp[2 * kc2][2], dp[2 * kc2][3]);
        as[2] = pack_bf16(dp[2 * kc2 + 1][0], dp[2 * kc2 + 1][1]);
        as[3] = pack_bf16(dp[2 * kc2 + 1][2], dp[2 * kc2 + 1][3]);
#pragma unroll
        for (int nt2 = 0; nt2 < HD / 8; nt2 += 2) {
          const int mi = lane >> 3;
          const int row = kc2 * 16 + (mi & 1) * 8 + (lane & 7);
          const int u = nt2 + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(sO + swz(row, u, UNITS), b0, b1, b2, b3);
          mma_bf16_16816(dv[nt2], ap, b0, b1);
          mma_bf16_16816(dv[nt2 + 1], ap, b2, b3);
          ldsm_x4_t(sQ + swz(row, u, UNITS), b0, b1, b2, b3);
          mma_bf16_16816(dk[nt2], as, b0, b1);
          mma_bf16_16816(dk[nt2 + 1], as, b2, b3);
        }
      }
      // dS^T -> smem [64 keys][64 q] (8 units of 16 B per row, swizzled)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int hh2 = 0; hh2 < 2; ++hh2) {
          const int r = warp * 16 + g + hh2 * 8;
          const int c = nt * 8 + t * 2;
          const uint32_t addr = sS + swz(r, c >> 3, 8) + (c & 7) * 2;
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(pack_bf16(dp[nt][2 * hh2], dp[nt][2 * hh2 + 1])));
        }
      __syncthreads();
      // dQ[16 q of this warp x HD] = dS[q x 64 keys] K[64 keys x HD]
      float dq[HD / 8][4];
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
#pragma unroll
      for (int kc2 = 0; kc2 < 4; ++kc2) {
        // A = dS[q rows warp*16.. +15][keys kc2*16 .. +15] from dS^T storage [key][q] (transposed load)
        uint32_t a[4];
        {
          const int mi = lane >> 3;
          const int key = kc2 * 16 + (mi >> 1) * 8 + (lane & 7);
          const int qc = warp * 16 + (mi & 1) * 8;
          ldsm_x4_t(sS + swz(key, qc >> 3, 8), a[0], a[1], a[2], a[3]);
        }
#pragma unroll
        for (int nt2 = 0; nt2 < HD / 8; nt2 += 2) {
          const int mi = lane >> 3;
          const int row = kc2 * 16 + (mi & 1) * 8 + (lane & 7);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(sK + swz(row, nt2 + (mi >> 1), UNITS), b0, b1, b2, b3);
          mma_bf16_16816(dq[nt2], a, b0, b1);
          mma_bf16_16816(dq[nt2 + 1], a, b2, b3);
        }
      }
#pragma unroll
      for (int hh2 = 0; hh2 < 2; ++hh2) {
        const int q = q0 + warp * 16 + g + hh2 * 8;
        if (q >= n) continue;
        float* dst = dq32 + static_cast<int64_t>(s0 + q) * qd + h * HD;
#pragma unroll
        for (int nt2 = 0; nt2 < HD / 8; ++nt2) {
          // one 8-byte vector reduction per column pair (sm_90+ red.v2.f32): half the L2 atomics
          asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dst + nt2 * 8 + t * 2),
                       "f"(dq[nt2][2 * hh2]), "f"(dq[nt2][2 * hh2 + 1])
                       : "memory");
        }
      }
    }
  }
  // dK, dV of this warp's 16 keys (the tile owns them for the whole KV group)
#pragma unroll
  for (int hh2 = 0; hh2 < 2; ++hh2) {
    const int key = kr0 + g + hh2 * 8;
    if (key >= n) continue;
    float* dkr = dkv32 + static_cast<int64_t>(s0 + key) * 2 * kvd + kvh * HD;
    float* dvr = dkr + kvd;
#pragma unroll
    for (int nt2 = 0; nt2 < HD / 8; ++nt2) {
      const int c = nt2 * 8 + t * 2;
      dkr[c] = dk[nt2][2 * hh2];
      dkr[c + 1] = dk[nt2][2 * hh2 + 1];
      dvr[c] = dv[nt2][2 * hh2];
      dvr[c + 1] = dv[nt2][2 * hh2 + 1];
    }
  }
}

template <class K>
void smem_attr(K k, int bytes) {
  if (bytes > 48 * 1024) DCU_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace

bool attn_fwd_tc(cudaStream_t s, const bf16* qkv, const int32_t* seq_start, int n_seq, int max_len, int rows, int nh,
                 int nkv, int hd, bf16* ctx, float* lse, double alg_flops, bf16* ctx_lo) {
  if (hd != 64 && hd != 128) return false;
  if (n_seq <= 0) return true;
  ProfScope ps(PROF_ATTN_FWD, s, alg_flops, 0);
  if (attn_fwd_tc5(s, qkv, seq_start, n_seq, max_len, rows, nh, nkv, hd, ctx, lse, ctx_lo)) return true;
  const float sl2 = kLog2e / sqrtf(static_cast<float>(hd));
  dim3 grid((max_len + 63) / 64, n_seq, nh);
  if (hd == 64) {
    smem_attr(attn_fwd_tc_k<64>, FwdCfg<64>::SMEM);
    attn_fwd_tc_k<64><<<grid, 128, FwdCfg<64>::SMEM, s>>>(qkv, seq_start, nh, nkv, ctx, lse, sl2, ctx_lo);
  } else {
    smem_attr(attn_fwd_tc_k<128>, FwdCfg<128>::SMEM);
    attn_fwd_tc_k<128><<<grid, 128, FwdCfg<128>::SMEM, s>>>(qkv, seq_start, nh, nkv, ctx, lse, sl2, ctx_lo);
  }
  DCU_LAUNCHED();
  return true;
}

bool attn_bwd_tc(cudaStream_t s, const bf16* qkv, const bf16* ctx, const bf16* dctx, const float* lse,
                 const int32_t* seq_start, int n_seq, int max_len, int rows, int nh, int nkv, int hd, float* Dbuf,
                 float* dq32, float* dkv32, double alg_flops, const bf16* ctx_lo) {
  if (hd != 64 && hd != 128) return false;
  if (n_seq <= 0) return true;
  ProfScope ps(PROF_ATTN_BWD, s, alg_flops, 0);
  attn_bwd_dot_k<<<kNumSMs * 8, 256, 0, s>>>(dctx, ctx, ctx_lo, rows, nh, hd, Dbuf);
  DCU_LAUNCHED();
  DCU_CHECK(cudaMemsetAsync(dq32, 0, sizeof(float) * static_cast<size_t>(rows) * nh * hd, s));
  if (attn_bwd_tc5(s, qkv, dctx, lse, Dbuf, seq_start, n_seq, max_len, rows, nh, nkv, hd, dq32, dkv32)) return true;
  const float sc = 1.f / sqrtf(static_cast<float>(hd));
  const float sl2 = kLog2e * sc;
  dim3 grid((max_len + 63) / 64, n_seq, nkv);
  if (hd == 64) {
    smem_attr(attn_bwd_tc_k<64>, BwdCfg<64>::SMEM);
    attn_bwd_tc_k<64><<<grid, 128, BwdCfg<64>::SMEM, s>>>(qkv, dctx, lse, Dbuf, seq_start, nh, nkv, dq32, dkv32, sc,
                                                          sl2);
  } else {
    smem_attr(attn_bwd_tc_k<128>, BwdCfg<128>::SMEM);
    attn_bwd_tc_k<128><<<grid, 128, BwdCfg<128>::SMEM, s>>>(qkv, dctx, lse, Dbuf, seq_start, nh, nkv, dq32, dkv32, sc,
                                                            sl2);
  }
  DCU_LAUNCHED();
  return true;
}

bool attn_decode_tc_supported(int nh, int nkv, int hd) { return nh / nkv <= 16 && (hd == 64 || hd == 128); }

bool attn_decode_tc(cudaStream_t s, const bf16* qkv, const bf16* kp, const bf16* vp, bf16* kc, bf16* vc,
                    const int32_t* plen, int rows, int G, int pmax, int n_comp, const DecodeRows& dr, int nh, int nkv,
                    int hd, bf16* ctx, double alg_bytes, bool append) {
  if (!attn_decode_tc_supported(nh, nkv, hd)) return false;
  ProfScope ps(PROF_ATTN_DECODE, s, 0, alg_bytes);
  if (hd == 64) launch_decode<64>(s, qkv, kp, vp, kc, vc, plen, rows, G, pmax, n_comp, dr, nh, nkv, ctx, append);
  else launch_decode<128>(s, qkv, kp, vp, kc, vc, plen, rows, G, pmax, n_comp, dr, nh, nkv, ctx, append);
  return true;
}

}  // namespace dashcu
