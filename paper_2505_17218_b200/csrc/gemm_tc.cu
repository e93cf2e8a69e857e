// tcgen05 tensor-core GEMM for sm_100a (bf16 x bf16 -> fp32 in TMEM), persistent.
//
//   C[M x N] = epilogue(A(m, k) . B(n, k)),  operands K-major or MN-major.
//
// One CTA per SM loops over 128 x BN output tiles (M fastest, so CTAs running
// together share the same B (weight) tile through L2). Warp roles:
//   warp 0      TMA producer: 128B-swizzled A/B k-blocks into a STAGES-deep
//               shared-memory ring that runs continuously across tiles
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=BN, K=16)
//               into one of TWO TMEM accumulators, so the epilogue of tile i
//               overlaps the MMAs of tile i+1; tcgen05.commit frees smem slots
//               and publishes finished accumulators
//   warp 2      TMEM allocator (2 x BN columns)
//   warps 4..   epilogue (EPW warps): tcgen05.ld 32 columns at a time -> bias /
//               tanh / dtanh / residual / fp32 accumulate (16-byte vector I/O),
//               or the fused LM-head sampling reduction (inverse-CDF slice sums + LSE)
// Operand major-ness is encoded in the UMMA instruction descriptor (bits 15/16)
// and the shared-memory descriptors (K-major: SBO = 1024 B between 8-row groups;
// MN-major: LBO = one 64-element TMA box, SBO = 1024 B between 8-k groups).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "gemm.cuh"
#include "rule.cuh"
#include "tc5.cuh"

namespace dashcu {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
// k-blocks per ring stage of the large-tile kernels (A/B builds; the skinny kernels use 4)
#ifndef DASHCU_KSUB_BIG
#define DASHCU_KSUB_BIG 1
#endif
constexpr int kKsubBig = DASHCU_KSUB_BIG;

// Producer / MMA-issuer waits on the operand ring. Default: tight try_wait loop; with
// -DDASHCU_GEMM_SLEEP_WAITS the suspend-hint form (frees issue slots for the epilogue
// warps sharing the SM sub-partition). A/B with tools builds.
__device__ __forceinline__ void mbar_wait_pipe(uint64_t* bar, uint32_t parity) {
#ifdef DASHCU_GEMM_SLEEP_WAITS
  mbar_wait_sleep(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}

// Persistent-schedule tile t -> (M tile, N tile), raster per GemmShape::n_fast.
__device__ __forceinline__ int tile_m(const GemmShape& g, int t, int tiles_m, int tiles_n) {
  return g.n_fast ? t / tiles_n : t % tiles_m;
}
__device__ __forceinline__ int tile_n(const GemmShape& g, int t, int tiles_m, int tiles_n) {
  return g.n_fast ? t % tiles_n : t / tiles_m;
}

// The W1 epilogue runs tanh on every element and its output is stored as bf16 (relative
// rounding 2^-9): the one-instruction MUFU tanh.approx (max relative error ~2^-11) is below
// that rounding and halves the epilogue's MUFU work against 1 - 2 / (exp(2x) + 1)
// (ex2 + rcp, ~1e-6 relative; -DDASHCU_TANH_ACCURATE selects it).
__device__ __forceinline__ float fast_tanh(float x) {
#ifdef DASHCU_TANH_ACCURATE
  const float e = __expf(2.f * fminf(fmaxf(x, -15.f), 15.f));
  return 1.f - __fdividef(2.f, e + 1.f);
#else
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- TMA-store epilogue -----------------------------------------------------------
// A thread owns one accumulator row, so direct 16-byte stores from a warp touch 32
// different rows per instruction (32 L1 wavefronts each). Instead every epilogue warp
// stages its 32 rows x 32 columns in a private 4 KB shared-memory buffer (in the TMA
// swizzle, so the 8 lanes of each store phase hit distinct banks) and one lane issues
// a bulk tensor store (or an fp32 reduce-add for EPI_ACCUM) of the 32 x 32 box; the
// tensor map clips rows >= M and columns >= N.
constexpr int kStageBytes = 4096;

// fp32 row of 32 (128 B, SWIZZLE_128B): 16-B chunk j of row r at r*128 + (j ^ (r & 7))*16
__device__ __forceinline__ void stage_f32(uint32_t buf, int lane, const float* v) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 128 + ((j ^ (lane & 7)) << 4)),
                 "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                 : "memory");
}
// bf16 row of 32 (64 B, SWIZZLE_64B): chunk j of row r at r*64 + (j ^ ((r >> 1) & 3))*16
__device__ __forceinline__ void stage_b16(uint32_t buf, int lane, const float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)),
                 "r"(pack2(v[8 * j], v[8 * j + 1])), "r"(pack2(v[8 * j + 2], v[8 * j + 3])),
                 "r"(pack2(v[8 * j + 4], v[8 * j + 5])), "r"(pack2(v[8 * j + 6], v[8 * j + 7]))
                 : "memory");
}
// Before overwriting the warp's buffer: the previous bulk store has finished reading it.
__device__ __forceinline__ void stage_acquire(int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
}
// After all lanes staged: make the writes visible to the async proxy, one lane stores.
__device__ __forceinline__ void stage_release(int lane, const CUtensorMap* map, uint32_t buf, int col, int row,
                                              bool reduce_add) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    if (reduce_add)
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(map)),
                   "r"(buf), "r"(col), "r"(row)
                   : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(map)),
                   "r"(buf), "r"(col), "r"(row)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}
__device__ __forceinline__ void stage_drain(int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

// Split-K ordering: the epilogue warp owning (tile, sub-block) for K slice s waits until
// slices 0..s-1 have reduced into C (flag == s), so the fp32 sums happen in a fixed
// order (deterministic). Items are dealt round-robin to co-resident persistent CTAs and
// only ever wait on lower-numbered items, so the chain cannot deadlock.
__device__ __forceinline__ void split_wait(const uint32_t* flag, uint32_t s, int lane) {
  if (lane == 0) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    } while (v < s);
    asm volatile("fence.proxy.async.global;" ::: "memory");  // later bulk reduces are ordered after
  }
  __syncwarp();
}
__device__ __forceinline__ void split_signal(uint32_t* flag, int lane) {
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // this slice's reduces performed
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
  }
}

// Output maps of the TMA-store epilogue (Epi::tma bits 0 / 1).
struct OutMaps {
  CUtensorMap f32;  // 32 x 32 fp32 box, SWIZZLE_128B: c32 / logits
  CUtensorMap b16;  // 32 x 32 bf16 box, SWIZZLE_64B: cT / dz
  CUtensorMap rs;   // input: fp32 residual (Epi::tma bit 2)
  CUtensorMap ax;   // input: bf16 tanh activations of EPI_DTANH (bit 3)
};

// AR: rows of the A box a stage holds (BM, or 32 / 64 for the skinny decode GEMMs: the MMA
// still reads 128 rows, the rows past AR are stale shared memory whose accumulator rows
// (>= M) are never stored, and the TMA no longer writes 96 zero-filled rows per k-block).
// KSUB: k-blocks per ring stage (one full-barrier wait + fence + commit per stage: that
// sequence costs the MMA issuer ~190 cycles, which is 2.4 x the four MMAs of a k-block
// at N <= 64, tools/mma_probe.cu; the MMA order over K is the same for every KSUB).
// MM: MMA M (128, or 64 for skinny tiles of <= 64 rows: half the A operand read per MMA;
// the accumulator then sits in TMEM lanes 0-15 of each 32-lane quarter, row 16 q + lane).
template <int BN, int STAGES, bool AK, bool BKM, int EPW, int AR = BM, int KSUB = 1, int MM = BM>
struct Cfg {
  static constexpr int A_BYTES = AR * BK * 2;
  static constexpr int BNS = BN;
  static constexpr int B_BYTES = BNS * BK * 2;
  static constexpr int B_LOAD = BN * BK * 2;  // bytes the B loads of a k-block deliver
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int KB_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGE_BYTES = KSUB * KB_BYTES;
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;  // EPW x 4 KB epilogue staging
  static constexpr int BAR_OFF = STG_OFF + EPW * kStageBytes;
  static constexpr int SMEM = BAR_OFF + 1024 /*align*/ + (2 * STAGES + 4 + EPW) * 8 + 16 /*barriers, TMEM slot*/;
  static constexpr int THREADS = 128 + EPW * 32;
  // kind::f16 instruction descriptor: D f32, A/B bf16, majors, N>>3, M>>4
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((AK ? 0u : 1u) << 15) |
                                    ((BKM ? 0u : 1u) << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(MM >> 4) << 24);
};

// 32 bias values of columns [nb, nb + 32) (0 past N); issued before the TMEM load so
// the (broadcast) global loads overlap it.
__device__ __forceinline__ void load_bias32(const float* bias, int nb, int N, float* b) {
  if (nb + 32 <= N && (reinterpret_cast<uintptr_t>(bias + nb) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(bias + nb + i));
      b[i] = x.x, b[i + 1] = x.y, b[i + 2] = x.z, b[i + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) b[i] = nb + i < N ? __ldg(bias + nb + i) : 0.f;
  }
}

__device__ __forceinline__ float max32(const float* x) {  // tree: max is exact in any order
  float t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = fmaxf(x[i], x[i + 16]);
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) t[i] = fmaxf(t[i], t[i + w]);
  return t[0];
}

// Generic epilogue on columns [c_lo, c_hi) of one accumulator row.
__device__ __forceinline__ void epilogue_store(const GemmShape& g, const Epi& e, uint32_t taddr, int row, int n0,
                                               int c_lo, int c_hi, bool vec) {
  float v[32];
#pragma unroll 1
  for (int c = c_lo; c < c_hi; c += 32) {
    tmem_ld32(taddr + c, v);
    if (row >= g.M) continue;
    const int nb = n0 + c;
    if (vec && nb + 32 <= g.N) {
      const int64_t r64 = row;
      if (e.bias) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 b = *reinterpret_cast<const float4*>(e.bias + nb + i);
          v[i] = __fmaf_rn(v[i], e.alpha, b.x), v[i + 1] = __fmaf_rn(v[i + 1], e.alpha, b.y);
          v[i + 2] = __fmaf_rn(v[i + 2], e.alpha, b.z), v[i + 3] = __fmaf_rn(v[i + 3], e.alpha, b.w);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __fmul_rn(v[i], e.alpha);
      }
      if (e.kind == EPI_TANH) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fast_tanh(v[i]);
      }
      if (e.kind == EPI_DTANH) {
        const bf16* ap = static_cast<const bf16*>(e.aux) + r64 * e.ld_aux + nb;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const uint4 raw = *reinterpret_cast<const uint4*>(ap + i);
          const bf16* a8 = reinterpret_cast<const bf16*>(&raw);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float a = __bfloat162float(a8[k]);
            v[i + k] *= (1.f - a * a);
          }
        }
      }
      if (e.resid) {
        const float* rp = e.resid + r64 * e.ldr + nb;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 x = *reinterpret_cast<const float4*>(rp + i);
          v[i] += x.x, v[i + 1] += x.y, v[i + 2] += x.z, v[i + 3] += x.w;
        }
      }
      if (e.kind == EPI_ACCUM) {
        float* cp = e.c32 + r64 * e.ldc32 + nb;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          float4 x = *reinterpret_cast<float4*>(cp + i);
          x.x += v[i], x.y += v[i + 1], x.z += v[i + 2], x.w += v[i + 3];
          *reinterpret_cast<float4*>(cp + i) = x;
        }
        continue;
      }
      if (e.c32) {
        float* cp = e.c32 + r64 * e.ldc32 + nb;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(cp + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
      if (e.cT) {
        bf16* cp = static_cast<bf16*>(e.cT) + r64 * e.ldcT + nb;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 o;
          o.x = pack2(v[i], v[i + 1]);
          o.y = pack2(v[i + 2], v[i + 3]);
          o.z = pack2(v[i + 4], v[i + 5]);
          o.w = pack2(v[i + 6], v[i + 7]);
          *reinterpret_cast<uint4*>(cp + i) = o;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int n = nb + i;
        if (n < g.N) epi_apply<bf16>(e, row, n, v[i]);
      }
    }
  }
}

// Row `lane` of a staged 32 x 32 box (the layouts of stage_f32 / stage_b16).
__device__ __forceinline__ void unstage_f32(uint32_t buf, int lane, float* x) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(x[4 * j]), "=f"(x[4 * j + 1]), "=f"(x[4 * j + 2]), "=f"(x[4 * j + 3])
                 : "r"(buf + lane * 128 + ((j ^ (lane & 7)) << 4))
                 : "memory");
}
__device__ __forceinline__ void unstage_b16(uint32_t buf, int lane, float* x) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t r[4];
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4))
                 : "memory");
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[8 * j + 2 * k] = __uint_as_float(r[k] << 16);
      x[8 * j + 2 * k + 1] = __uint_as_float(r[k] & 0xffff0000u);
    }
  }
}

// Generic epilogue through the TMA path (Epi::tma != 0): same math as epilogue_store.
// The fp32 residual (bit 2) or the bf16 tanh activations of EPI_DTANH (bit 3) arrive
// as a 32 x 32 box in the warp's staging buffer (TMA load, zero-filled past M / N,
// issued before the TMEM load); outputs leave through the same buffer as bulk stores.
// `bias` is e.bias, or null for K slices after the first of a split-K accumulate (the
// bias is added once per output element).
__device__ __forceinline__ void epilogue_store_tma(const GemmShape& g, const Epi& e, const OutMaps& om, uint32_t taddr,
                                                   int row, int r0, int n0, int c_lo, int c_hi, uint32_t stg,
                                                   int lane, uint64_t* ebar, uint32_t& ephase, const float* bias) {
  float v[32], b[32];
  const bool live = row < g.M;
  const int64_t r64 = row;
  const bool tres = (e.tma & 4) != 0, taux = (e.tma & 8) != 0;
  uint8_t* stg_ptr = reinterpret_cast<uint8_t*>(__cvta_shared_to_generic(stg));
#pragma unroll 1
  for (int c = c_lo; c < c_hi; c += 32) {
    const int nb = n0 + c;
    if (nb >= g.N) {  // warp-uniform
      tmem_ld32(taddr + c, v);
      continue;
    }
    if (tres || taux) {
      stage_acquire(lane);  // the previous bulk store has finished reading the buffer
      if (lane == 0) {
        mbar_expect_tx(ebar, tres ? 4096u : 2048u);
        tma_load_2d(stg_ptr, tres ? &om.rs : &om.ax, ebar, nb, r0);
      }
    }
    if (bias) load_bias32(bias, nb, g.N, b);  // broadcast loads, overlap the TMEM load
    tmem_ld32(taddr + c, v);
    const bool full = nb + 32 <= g.N;
    if (bias) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __fmaf_rn(v[i], e.alpha, b[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __fmul_rn(v[i], e.alpha);
    }
    if (e.kind == EPI_TANH) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fast_tanh(v[i]);
    }
    if (tres || taux) {
      mbar_wait(ebar, ephase);
      ephase ^= 1u;
    }
    if (e.kind == EPI_DTANH) {
      if (taux) {
        unstage_b16(stg, lane, b);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= (1.f - b[i] * b[i]);
      } else if (live) {
        const bf16* ap = static_cast<const bf16*>(e.aux) + r64 * e.ld_aux + nb;
        for (int i = 0; i < 32; ++i)
          if (full || nb + i < g.N) {
            const float a = __bfloat162float(ap[i]);
            v[i] *= (1.f - a * a);
          }
      }
    }
    if (e.resid) {
      if (tres) {
        unstage_f32(stg, lane, b);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += b[i];
      } else if (live) {
        const float* rp = e.resid + r64 * e.ldr + nb;
        for (int i = 0; i < 32; ++i)
          if (full || nb + i < g.N) v[i] += rp[i];
      }
    }
    if (tres || taux) __syncwarp();  // every lane has read the box before it is overwritten
    if (e.tma & 1) {
      stage_acquire(lane);
      stage_f32(stg, lane, v);
      stage_release(lane, &om.f32, stg, nb, r0, e.kind == EPI_ACCUM);
    }
    if (e.tma & 2) {
      stage_acquire(lane);
      stage_b16(stg, lane, v);
      stage_release(lane, &om.b16, stg, nb, r0, false);
    }
  }
}

// Residual epilogue with the next chunk's residual box prefetched (CTA-pair kernel, DB
// variant): per warp two 4 KB residual / fp32-output buffers used alternately and one 2 KB
// bf16-output buffer. Chunk k adds the residual staged in buf[k & 1], writes the fp32 sum
// back into the same buffer and bulk-stores it, while the TMA load of chunk k+1's residual
// is already in flight into buf[(k+1) & 1]. Bulk stores are committed one group each, so
// "wait_group.read 1" = every store but the newest has finished reading its buffer.
__device__ __forceinline__ void epilogue_resid_db(const GemmShape& g, const Epi& e, const OutMaps& om, uint32_t taddr,
                                                  int r0, int n0, int c_lo, int c_hi, uint32_t stg, int lane,
                                                  uint64_t* ebar2, uint32_t* eph2) {
  float v[32], b[32];
  const uint32_t buf[2] = {stg, stg + 4096}, tbuf = stg + 8192;
  auto load = [&](int k) {  // residual box of chunk k into buf[k & 1]
    const int nb = n0 + c_lo + 32 * k;
    if (lane == 0) {
      mbar_expect_tx(&ebar2[k & 1], 4096u);
      tma_load_2d(reinterpret_cast<uint8_t*>(__cvta_shared_to_generic(buf[k & 1])), &om.rs, &ebar2[k & 1], nb, r0);
    }
  };
  const int nk = min((c_hi - c_lo) / 32, (g.N - n0 - c_lo + 31) / 32);
  if (nk <= 0) return;
  // buf[0]'s last store (previous tile) has been read before the first load reuses it
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
  load(0);
#pragma unroll 1
  for (int k = 0; k < nk; ++k) {
    const int nb = n0 + c_lo + 32 * k;
    if (k + 1 < nk) {  // buf[(k+1)&1] held chunk k-1's fp32 output: wait until read, then prefetch
      if (lane == 0) {  // chunk k-1 committed c32 then (optionally) cT: the newest may stay pending
        if (e.tma & 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
      load(k + 1);
    }
    if (e.bias) load_bias32(e.bias, nb, g.N, b);
    tmem_ld32(taddr + c_lo + 32 * k, v);
    if (e.bias) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __fmaf_rn(v[i], e.alpha, b[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __fmul_rn(v[i], e.alpha);
    }
    if (e.kind == EPI_TANH) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fast_tanh(v[i]);
    }
    mbar_wait(&ebar2[k & 1], eph2[k & 1]);
    eph2[k & 1] ^= 1u;
    unstage_f32(buf[k & 1], lane, b);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += b[i];
    __syncwarp();  // every lane has read the residual before the buffer is overwritten
    if (e.tma & 1) {
      stage_f32(buf[k & 1], lane, v);
      stage_release(lane, &om.f32, buf[k & 1], nb, r0, false);
    }
    if (e.tma & 2) {  // cT(k-1) read; c32(k), committed just now, may stay pending
      if (lane == 0) {
        if (e.tma & 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
      stage_b16(tbuf, lane, v);
      stage_release(lane, &om.b16, tbuf, nb, r0, false);
    }
  }
}

#ifndef DASHCU_NO_AUX_DB  // A/B builds: -DDASHCU_NO_AUX_DB keeps the single-buffered dtanh epilogue
constexpr bool kAuxDb = true;
#else
constexpr bool kAuxDb = false;
#endif
// dtanh epilogue (EPI_DTANH, bf16 output only) with the next chunk's tanh-activation box
// prefetched (CTA-pair kernel): the warp's 4 KB buffer holds two 2 KB bf16 boxes used
// alternately. Chunk k reads aux(k) from buf[k & 1], writes its bf16 result into the same
// buffer and bulk-stores it; aux(k+1) is already loading into buf[(k+1) & 1] (whose
// previous store, chunk k-1's, must have been read first).
__device__ __forceinline__ void epilogue_aux_db(const GemmShape& g, const Epi& e, const OutMaps& om, uint32_t taddr,
                                                int r0, int n0, int c_lo, int c_hi, uint32_t stg, int lane,
                                                uint64_t* ebar2, uint32_t* eph2) {
  float v[32], a[32];
  const uint32_t buf[2] = {stg, stg + 2048};
  auto load = [&](int k) {  // tanh activations of chunk k into buf[k & 1]
    if (lane == 0) {
      mbar_expect_tx(&ebar2[k & 1], 2048u);
      tma_load_2d(reinterpret_cast<uint8_t*>(__cvta_shared_to_generic(buf[k & 1])), &om.ax, &ebar2[k & 1],
                  n0 + c_lo + 32 * k, r0);
    }
  };
  const int nk = min((c_hi - c_lo) / 32, (g.N - n0 - c_lo + 31) / 32);
  if (nk <= 0) return;
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous tile's stores
  __syncwarp();
  load(0);
#pragma unroll 1
  for (int k = 0; k < nk; ++k) {
    const int nb = n0 + c_lo + 32 * k;
    if (k + 1 < nk) {  // buf[(k+1)&1] held chunk k-1's output: read by its store before reuse
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      load(k + 1);
    }
    tmem_ld32(taddr + c_lo + 32 * k, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __fmul_rn(v[i], e.alpha);
    mbar_wait(&ebar2[k & 1], eph2[k & 1]);
    eph2[k & 1] ^= 1u;
    unstage_b16(buf[k & 1], lane, a);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= (1.f - a[i] * a[i]);
    __syncwarp();  // every lane has read its activations before the buffer is overwritten
    stage_b16(buf[k & 1], lane, v);
    stage_release(lane, &om.b16, buf[k & 1], nb, r0, false);
  }
}

// LM-head sampling epilogue (inverse-CDF contract, rule.cuh): per 32-id slice the
// epilogue stores the fp32 logits (the scan needs the chosen slice's ids) and one
// 4-float record {m_s, Z_s, m1_s, Z1_s}: the contract's max / sexp2-sum at 1/T and
// the T=1 log-sum-exp partials for the recorded log-prob. Slices without BOS and
// inside V (all but two per row) take a branch-free path: tree max, then 32
// independent sexp2 chains feeding the contract's 4 interleaved partial sums.
__device__ __forceinline__ void epilogue_sample(const GemmShape& g, const Epi& e, const SampleArgs& sa,
                                                const OutMaps& om, uint32_t taddr, int row, int r0, int n0, int c_lo,
                                                int c_hi, uint32_t stg, int lane) {
  float v[32], b[32];
  const bool live = row < g.M;
  const bool t1 = sa.inv_t == 1.f;
#pragma unroll 1
  for (int c = c_lo; c < c_hi; c += 32) {
    const int nb = n0 + c;
    if (nb < g.N) load_bias32(e.bias, nb, g.N, b);
    tmem_ld32(taddr + c, v);
    if (nb >= g.N) continue;  // ragged last tile (warp-uniform): no slice record past V
    const bool full = nb + 32 <= g.N;
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __fadd_rn(v[i], b[i]);
    if (sa.logits) {  // fp32 logits only for the parity dump (the scan recomputes its slice)
      stage_acquire(lane);
      stage_f32(stg, lane, v);
      stage_release(lane, &om.f32, stg, nb, r0, false);
    }
    if (!live) continue;
    float m, m1, Z, Z1;
    if (full && (sa.bos < nb || sa.bos >= nb + 32)) {
      float x[32];
      if (t1) {  // v * 1.0 == v
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = v[i];
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = __fmul_rn(v[i], sa.inv_t);
      }
      m = max32(x);
      // the contract's e_i = sexp2((x_i - m) * log2e) and the 4 interleaved partial sums,
      // element pairs on the packed fp32x2 pipe (per lane the same roundings: bit-exact)
      float a[4] = {0.f, 0.f, 0.f, 0.f};
      const uint64_t m2 = f2_pack(m, m), l2 = f2_pack(kLog2e, kLog2e);
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float y0, y1, e0, e1;
        f2_unpack(f2_mul(f2_sub(f2_pack(x[i], x[i + 1]), m2), l2), y0, y1);
        sexp2_x2(y0, y1, e0, e1);
        const int j = i & 3;  // 0 or 2: accumulators (a_j, a_j+1) get (e_i, e_i+1)
        f2_unpack(f2_add(f2_pack(a[j], a[j + 1]), f2_pack(e0, e1)), a[j], a[j + 1]);
      }
      Z = __fadd_rn(__fadd_rn(a[0], a[1]), __fadd_rn(a[2], a[3]));
      if (t1) {
        m1 = m, Z1 = Z;
      } else {
        m1 = max32(v);
        float b4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 32; ++i) b4[i & 3] += __expf(v[i] - m1);
        Z1 = (b4[0] + b4[1]) + (b4[2] + b4[3]);
      }
    } else {  // the slice holding BOS, or the ragged end of V
      float x[32];
      m = -FLT_MAX, m1 = -FLT_MAX;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const bool ok = nb + i < g.N && nb + i != sa.bos;
        x[i] = ok ? __fmul_rn(v[i], sa.inv_t) : -FLT_MAX;
        m = fmaxf(m, x[i]);
        m1 = fmaxf(m1, ok ? v[i] : -FLT_MAX);
      }
      float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float ei = x[i] == -FLT_MAX ? 0.f : sexp2(__fmul_rn(__fsub_rn(x[i], m), kLog2e));
        a[i & 3] = __fadd_rn(a[i & 3], ei);
      }
      Z = __fadd_rn(__fadd_rn(a[0], a[1]), __fadd_rn(a[2], a[3]));
      Z1 = Z;
      if (!t1) {
        float b4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 32; ++i) b4[i & 3] += x[i] == -FLT_MAX ? 0.f : __expf(v[i] - m1);
        Z1 = (b4[0] + b4[1]) + (b4[2] + b4[3]);
      } else {
        m1 = m;
      }
    }
    if (t1) {  // m1 = m, Z1 = Z: the compact 8-byte record halves the scan's traffic
      float2* pp = reinterpret_cast<float2*>(sa.part + (static_cast<int64_t>(row) * sa.ntiles + (nb / kSlice)) * 2);
      *pp = make_float2(m, Z);
    } else {
      float4* pp = reinterpret_cast<float4*>(sa.part + (static_cast<int64_t>(row) * sa.ntiles + (nb / kSlice)) * 4);
      *pp = make_float4(m, Z, m1, Z1);
    }
  }
}

// LM-head backward pass 1: per (row, slice) {max, sum exp} of the non-BOS logits.
__device__ __forceinline__ void epilogue_lse(const GemmShape& g, const Epi& e, const SampleArgs& sa, uint32_t taddr,
                                             int row, int n0, int c_lo, int c_hi, int slice) {
  float v[32], b[32];
  const bool live = row < g.M;
  float mx = -FLT_MAX, se = 0.f;
#pragma unroll 1
  for (int c = c_lo; c < c_hi; c += 32) {
    const int nb = n0 + c;
    if (nb < g.N) load_bias32(e.bias, nb, g.N, b);
    tmem_ld32(taddr + c, v);
    if (!live || nb >= g.N) continue;
    if (nb + 32 <= g.N && (sa.bos < nb || sa.bos >= nb + 32)) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += b[i];
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int n = nb + i;
        v[i] = (n < g.N && n != sa.bos) ? v[i] + b[i] : -FLT_MAX;
      }
    }
    const float cm = max32(v);
    if (cm > -FLT_MAX) {
      const float nm = fmaxf(mx, cm);
      float a4[4] = {se * __expf(mx - nm), 0.f, 0.f, 0.f};  // 4 chains: the adds overlap
#pragma unroll
      for (int i = 0; i < 32; ++i) a4[i & 3] += v[i] > -FLT_MAX ? __expf(v[i] - nm) : 0.f;
      se = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      mx = nm;
    }
  }
  if (live) {
    float* pp = sa.part + (static_cast<int64_t>(row) * sa.ntiles + slice) * 2;
    pp[0] = mx;
    pp[1] = se;
  }
}

// LM-head backward pass 2: dz = w_r (onehot(y_r) - exp(logit - lse_r)), BOS column 0, bf16.
__device__ __forceinline__ void epilogue_dz(const GemmShape& g, const Epi& e, const SampleArgs& sa, const OutMaps& om,
                                            uint32_t taddr, int row, int r0, int n0, int c_lo, int c_hi, uint32_t stg,
                                            int lane) {
  float v[32], b[32];
  const bool live = row < g.M;
  const float lse = live ? sa.lse[row] : 0.f;
  const float w = live ? sa.weight[row] : 0.f;
  const int y = live ? sa.target[row] : -1;
#pragma unroll 1
  for (int c = c_lo; c < c_hi; c += 32) {
    const int nb = n0 + c;
    if (nb < g.N) load_bias32(e.bias, nb, g.N, b);
    tmem_ld32(taddr + c, v);
    if (nb >= g.N) continue;  // warp-uniform
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int n = nb + i;
      const float p = __expf(v[i] + b[i] - lse);
      v[i] = (n == sa.bos) ? 0.f : w * ((n == y ? 1.f : 0.f) - p);
    }
    stage_acquire(lane);
    stage_b16(stg, lane, v);
    stage_release(lane, &om.b16, stg, nb, r0, false);
  }
}

// Chosen-slice recompute (MODE 4, gemm_tc_slice): tile (row block mb, nt) multiplies the 128
// rows of the block with the W_out rows of the slices chosen by its rows 8 nt .. 8 nt + 7
// (B staged as eight 32-row boxes); row 8 nt + j keeps columns [32 j, 32 j + 32): its own
// slice. Same instruction sequence as the MODE 1 sampling GEMM (128 x 256 tiles, BK 64, the
// same K order), so the 32 logits equal the ones the sampling epilogue saw, bit for bit.
__device__ __forceinline__ void epilogue_slice(const GemmShape& g, const Epi& e, const SampleArgs& sa,
                                               uint32_t taddr, int row, int nt, int q, int c_lo, int c_hi,
                                               int lane) {
  float v[32];
  const int base = nt * 8 - q * 32;  // lane of the tile's first useful row within this quarter
  const bool mine = lane >= base && lane < base + 8 && row < g.M;
  const int j = lane - base;
  const int sb = mine ? sa.sel[row].sb : -1;
#pragma unroll 1
  for (int c = c_lo; c < c_hi; c += 32) {
    tmem_ld32(taddr + c, v);  // warp-collective
    if (!mine || c != 32 * j || sb < 0) continue;
    float* out = sa.logits + static_cast<int64_t>(row) * kSlice;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int id = sb * kSlice + i;
      out[i] = id < g.N ? __fadd_rn(v[i], __ldg(e.bias + id)) : 0.f;
    }
  }
}

#ifdef DASHCU_GEMM_TRACE
// experiment builds: CTA 0's per-k-block clocks (producer issue, MMA data-ready) of the
// last launch, read with dashcu_debug_gemm_trace
__device__ long long g_trace[3][512];
#define GEMM_TRACE(i, k) \
  if (blockIdx.x == 0 && (k) < 512) g_trace[i][k] = clock64()
// phase marks of CTA 0 (thread-0 / warp-leader clocks) in g_trace[2][500 + ...]
#define GEMM_MARK(k) \
  if (blockIdx.x == 0) g_trace[2][500 + (k)] = clock64()
// per-tile epilogue start / end of CTA 0's first epilogue warp: g_trace[2][300 + 2 i + k]
#define GEMM_TILE(i, k) \
  if (blockIdx.x == 0 && threadIdx.x == 128 && (i) < 90) g_trace[2][300 + 2 * (i) + (k)] = clock64()
#else
#define GEMM_TILE(i, k)
#define GEMM_MARK(k)
#define GEMM_TRACE(i, k)
#endif

// MODE: 0 generic store epilogue, 1 fused sampling, 2 LSE partials, 3 dz, 4 chosen-slice recompute
template <int BN, int STAGES, bool AK, bool BKM, int EPW, int MODE, int AR = BM, int KSUB = 1, int MM = BM>
__global__ void __launch_bounds__(Cfg<BN, STAGES, AK, BKM, EPW, AR, KSUB, MM>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ OutMaps om, GemmShape g, Epi e, SampleArgs sa) {
  static_assert(AR == BM || AK, "partial A boxes are K-major only");
  static_assert(KSUB == 1 || MODE == 0, "multi-k-block stages: generic GEMMs only");
  static_assert(MM == BM || (MODE == 0 && AR <= MM), "M = 64 MMAs: generic GEMMs with <= 64-row A boxes");
  using C = Cfg<BN, STAGES, AK, BKM, EPW, AR, KSUB, MM>;
  constexpr int TM = MODE == 0 ? MM : BM;  // rows per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* ebar = tempty + 2;       // [EPW] epilogue TMA-load barriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + EPW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GEMM_MARK(0);
  const int nkb = (g.K + BK - 1) / BK;
  const int tiles_m = (g.M + TM - 1) / TM, tiles_n = MODE == 4 ? BM / 8 : (g.N + BN - 1) / BN;
  const int ntile = tiles_m * tiles_n;
  // split-K (EPI_ACCUM only): work item w = (tile w % ntile, K slice w / ntile), slices of kps
  // k-blocks. Slice-major: a tile's slices run about a round apart, so each slice's ordered
  // reduce finds its predecessor done instead of all of them finishing together and queueing
  const int S = MODE == 0 ? e.splits : 1;
  const int kps = (nkb + S - 1) / S;
  const int nitem = ntile * S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPW * 32);
    }
    for (int w = 0; w < EPW; ++w) mbar_init(&ebar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) GEMM_MARK(1);
  pdl_wait();  // set-up above overlapped the previous kernel; its outputs are visible now
  if (threadIdx.x == 0) GEMM_MARK(2);

  if (warp == 0) {
    if (lane == 0) {
      int st_all = 0;
      for (int w = blockIdx.x; w < nitem; w += gridDim.x) {
        const int t = w % ntile, sp = w / ntile;
        const int m0 = (MODE == 4 ? t / tiles_n : tile_m(g, t, tiles_m, tiles_n)) * TM,
                  n0 = MODE == 4 ? t % tiles_n : tile_n(g, t, tiles_m, tiles_n) * BN;
        int slice_row[8];  // MODE 4: W_out row of each 32-row B box
        if constexpr (MODE == 4) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int r = m0 + n0 * 8 + j;
            slice_row[j] = r < g.M ? max(sa.sel[r].sb, 0) * kSlice : 0;
          }
        }
        const int kb_lo = sp * kps, kb_hi = min(nkb, kb_lo + kps);
        for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KSUB, ++st_all) {
          const int s = st_all % STAGES;
          const uint32_t ph = (st_all / STAGES) & 1;
          mbar_wait_pipe(&empty[s], ph ^ 1);
          GEMM_TRACE(0, st_all);
          const int cnt = min(KSUB, kb_hi - kb0);
          mbar_expect_tx(&full[s], cnt * (C::A_BYTES + C::B_LOAD));
          for (int sub = 0; sub < cnt; ++sub) {
            const int kb = kb0 + sub;
            uint8_t* sa_ = smem + s * C::STAGE_BYTES + sub * C::KB_BYTES;
            uint8_t* sb_ = sa_ + C::A_BYTES;
            const int k0 = kb * BK;
            if (AK) {
              tma_load_2d(sa_, &mapA, &full[s], k0, m0);
            } else {
              tma_load_2d(sa_, &mapA, &full[s], m0, k0);
              tma_load_2d(sa_ + 64 * BK * 2, &mapA, &full[s], m0 + 64, k0);
            }
            if constexpr (MODE == 4) {
#pragma unroll
              for (int j = 0; j < 8; ++j) tma_load_2d(sb_ + j * kSlice * BK * 2, &mapB, &full[s], k0, slice_row[j]);
            } else if (BKM) {
              tma_load_2d(sb_, &mapB, &full[s], k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < C::BNS / 64; ++j) tma_load_2d(sb_ + j * 64 * BK * 2, &mapB, &full[s], n0 + 64 * j, k0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int st_all = 0, i = 0;
      for (int w = blockIdx.x; w < nitem; w += gridDim.x, ++i) {
        const int kb_lo = (w / ntile) * kps, kb_hi = min(nkb, kb_lo + kps);
        const int acc = i & 1;
        const uint32_t aph = (i >> 1) & 1;
        mbar_wait_pipe(&tempty[acc], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KSUB, ++st_all) {
          const int s = st_all % STAGES;
          const uint32_t ph = (st_all / STAGES) & 1;
          GEMM_TRACE(1, st_all);
          mbar_wait_pipe(&full[s], ph);
          GEMM_TRACE(2, st_all);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int cnt = min(KSUB, kb_hi - kb0);
#pragma unroll 1
          for (int sub = 0; sub < cnt; ++sub) {
            const int kb = kb0 + sub;
            const uint32_t sa_ = smem_u32(smem + s * C::STAGE_BYTES + sub * C::KB_BYTES);
            const uint32_t sb_ = sa_ + C::A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // K-major: advance 32 B inside the swizzle row; MN-major: advance 16 k-rows (2 x 1024 B)
              const uint64_t da = AK ? smem_desc(sa_ + k * 32, 16, 1024) : smem_desc(sa_ + k * 2048, 64 * BK * 2, 1024);
              const uint64_t db = BKM ? smem_desc(sb_ + k * 32, 16, 1024) : smem_desc(sb_ + k * 2048, 64 * BK * 2, 1024);
              umma_bf16(d, da, db, C::IDESC, (kb > kb_lo || k > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
      // every MMA is issued: the next kernel may launch now (its CTAs land on the SMs this
      // grid leaves idle and set up while our epilogues drain; its pdl_wait() still waits
      // for this whole grid)
      pdl_trigger();
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = ew & 3;                  // TMEM lane quarter (warp % 4 rule)
    const int slice = ew >> 2;             // column slice handled by this warp
    constexpr int NSL = EPW / 4;
    constexpr int CW = (BN / 32 + NSL - 1) / NSL * 32;  // 32-column chunks per slice (224: 128 + 96)
    const int c_lo = min(BN, slice * CW), c_hi = min(BN, (slice + 1) * CW);
    auto al = [](const void* p, int64_t ld, int esz) {
      return p == nullptr || (((reinterpret_cast<uintptr_t>(p) | static_cast<uintptr_t>(ld * esz)) & 15) == 0);
    };
    const bool vec = al(e.c32, e.ldc32, 4) && al(e.cT, e.ldcT, 2) && al(e.resid, e.ldr, 4) &&
                     al(e.aux, e.ld_aux, 2) && al(e.bias, 0, 4);
    const uint32_t stg = smem_u32(smem + C::STG_OFF + ew * kStageBytes);
    uint32_t ephase = 0;
    int i = 0;
    for (int w = blockIdx.x; w < nitem; w += gridDim.x, ++i) {
      const int t = w % ntile, sp = w / ntile;
      const int m0 = (MODE == 4 ? t / tiles_n : tile_m(g, t, tiles_m, tiles_n)) * TM,
                n0 = MODE == 4 ? t % tiles_n : tile_n(g, t, tiles_m, tiles_n) * BN;
      const int acc = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      mbar_wait_sleep(&tfull[acc], aph);
      if (threadIdx.x == 128 && i == 0) GEMM_MARK(3);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t* flag = S > 1 ? e.split_flags + t * EPW + ew : nullptr;
      if (flag && sp > 0) split_wait(flag, sp, lane);  // K slices reduce into C in slice order
      const uint32_t taddr = tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      const int r0 = m0 + q * 32;
      // M = 64: rows 16 q .. 16 q + 15 in lanes 0-15 of the quarter (lanes 16-31 hold none)
      const int row = MM == 64 ? (lane < 16 ? m0 + q * 16 + lane : g.M) : r0 + lane;
      if constexpr (MM == 64)
        epilogue_store(g, e, taddr, row, n0, c_lo, c_hi, vec);
      else if constexpr (MODE == 1)
        epilogue_sample(g, e, sa, om, taddr, row, r0, n0, c_lo, c_hi, stg, lane);
      else if constexpr (MODE == 2)
        epilogue_lse(g, e, sa, taddr, row, n0, c_lo, c_hi, tile_n(g, t, tiles_m, tiles_n) * NSL + slice);
      else if constexpr (MODE == 3)
        epilogue_dz(g, e, sa, om, taddr, row, r0, n0, c_lo, c_hi, stg, lane);
      else if constexpr (MODE == 4)
        epilogue_slice(g, e, sa, taddr, row, n0, q, c_lo, c_hi, lane);
      else if (e.tma)
        epilogue_store_tma(g, e, om, taddr, row, r0, n0, c_lo, c_hi, stg, lane, &ebar[ew], ephase,
                           sp > 0 ? nullptr : e.bias);
      else
        epilogue_store(g, e, taddr, row, n0, c_lo, c_hi, vec);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[acc]);
      if (flag) split_signal(flag, lane);
    }
    if (threadIdx.x == 128) GEMM_MARK(4);
    stage_drain(lane);  // bulk stores complete before the CTA's shared memory goes away
    if (threadIdx.x == 128) GEMM_MARK(5);
  }
  pdl_trigger();  // this CTA's work is done: the next kernel may be scheduled
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

// 2-D bf16 operand map (128-byte swizzle) over a row-major [rows x cols] matrix.
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_cols, int box_rows) {
  return tma_map_2d(m, base, rows, cols, ld, box_cols, box_rows, false, 128, true);
}

// 32 x 32 output box for the TMA-store epilogue over a row-major [rows x cols] matrix.
bool make_out_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, bool f32) {
  return tma_map_2d(m, base, rows, cols, ld, 32, 32, f32, f32 ? 128 : 64, false);
}

// Epilogue outputs through bulk tensor stores when both outputs are TMA-legal
// (the generic EPI kinds only; returns the Epi::tma bits, 0 = direct stores).
int out_maps_for(const GemmShape& g, const Epi& e, OutMaps* om) {
  if (knob(KNOB_NO_TMA_STORE)) return 0;
  int bits = 0;
  if (e.c32) {
    if (!make_out_map(&om->f32, e.c32, g.M, g.N, e.ldc32, true)) return 0;
    bits |= 1;
  }
  if (e.cT && e.kind != EPI_ACCUM) {
    if (!make_out_map(&om->b16, e.cT, g.M, g.N, e.ldcT, false)) return 0;
    bits |= 2;
  }
  if (!bits) return 0;
  if (e.resid && make_out_map(&om->rs, e.resid, g.M, g.N, e.ldr, true)) bits |= 4;
  else if (!e.resid && e.kind == EPI_DTANH && e.aux && make_out_map(&om->ax, e.aux, g.M, g.N, e.ld_aux, false))
    bits |= 8;
  return bits;
}

// Per-device split-K flag words (one per tile x epilogue warp), zeroed before each use.
uint32_t* split_flag_buffer(int n) {
  static std::mutex mu;
  static uint32_t* buf[16] = {};
  static int cap[16] = {};
  int dev = 0;
  DCU_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (cap[dev] < n) {
    if (buf[dev]) DCU_CHECK(cudaFree(buf[dev]));
    const int c = std::max(n, 1 << 16);
    DCU_CHECK(cudaMalloc(&buf[dev], sizeof(uint32_t) * c));
    cap[dev] = c;
  }
  return buf[dev];
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
  }
  return n;
}

template <int BN, int STAGES, bool AK, bool BKM, int EPW, int MODE, int AR = BM, int KSUB = 1, int MM = BM>
void launch(cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& om, const GemmShape& g,
            const Epi& e, const SampleArgs& sa) {
  using C = Cfg<BN, STAGES, AK, BKM, EPW, AR, KSUB, MM>;
  static_assert(C::SMEM <= 232448, "shared memory");
  auto k = gemm_tc_kernel<BN, STAGES, AK, BKM, EPW, MODE, AR, KSUB, MM>;
  static bool attr = false;
  if (!attr) {
    DCU_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  constexpr int TM = MODE == 0 ? MM : BM;
  const int nitem = ((g.M + TM - 1) / TM) * (MODE == 4 ? BM / 8 : (g.N + BN - 1) / BN) * (MODE == 0 ? e.splits : 1);
  const int cap = num_sms();
  const int grid = nitem < cap ? nitem : cap;  // persistent: all CTAs co-resident
  ProfScope ps(MODE == 1 || MODE == 4 ? PROF_SAMPLE : MODE >= 2 ? PROF_LM_ROWS : PROF_GEMM_TC, s,
               MODE == 4 ? 2.0 * g.M * kSlice * static_cast<double>(g.K) : 2.0 * g.M * g.N * static_cast<double>(g.K),
               0);
  if (ps.keyed())
    snprintf(ps.key, sizeof(ps.key), "mode%d %dx%d/%d M%d N%d K%d %c%c epi%d split%d", MODE, AR, BN, KSUB, g.M, g.N,
             g.K, AK ? 'k' : 'm', BKM ? 'k' : 'm', e.kind, MODE == 0 ? e.splits : 1);
  launch_pdl(k, dim3(grid), dim3(C::THREADS), C::SMEM, s, ma, mb, om, g, e, sa);
  DCU_LAUNCHED();
}

template <int BN, int STAGES_KB, int KSUB = 1>
void dispatch_majors(cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& om,
                     const GemmShape& g, const Epi& e) {
  const SampleArgs none;
  constexpr int STAGES = STAGES_KB / KSUB < 2 ? 2 : STAGES_KB / KSUB;
  // 8 epilogue warps (two per SM sub-partition, each owning half of the tile's columns)
  if (g.a_kmajor && g.b_kmajor) launch<BN, STAGES, true, true, 8, 0, BM, KSUB>(s, ma, mb, om, g, e, none);
  else if (g.a_kmajor) launch<BN, STAGES, true, false, 8, 0, BM, KSUB>(s, ma, mb, om, g, e, none);
  else if (g.b_kmajor) launch<BN, STAGES, false, true, 8, 0, BM, KSUB>(s, ma, mb, om, g, e, none);
  else launch<BN, STAGES, false, false, 8, 0, BM, KSUB>(s, ma, mb, om, g, e, none);
}

}  // namespace
extern "C" __attribute__((visibility("default"))) int dashcu_debug_gemm_trace(long long* out) {
#ifdef DASHCU_GEMM_TRACE
  return cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)) == cudaSuccess ? 0 : 4;
#else
  (void)out;
  return 1;
#endif
}
namespace {

bool legal(const GemmShape& g) {
  if (g.K <= 0 || g.M <= 0 || g.N <= 0) return false;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(g.A), pb = reinterpret_cast<uintptr_t>(g.B);
  return !((pa & 15) || (pb & 15) || ((g.lda * 2) & 15) || ((g.ldb * 2) & 15));
}

constexpr int kSampleBN = 256;
constexpr int kSampleEPW = 8;  // two 128-column halves per accumulator row

// ======================================================= CTA-pair (cta_group::2) variant
// A cluster of two CTAs on one TPC computes a 256 x BN tile: each CTA stages its own 128
// rows of A and HALF of B (BN/2 rows), and the leader's single thread issues
// tcgen05.mma.cta_group::2 (M = 256), which reads both CTAs' shared memory. Per SM
// this halves the B traffic through shared memory (the 1-CTA 128x256 tile needs
// 192 B/clk of smem read+fill at full MMA rate, the pair 128 B/clk). Each CTA's TMEM
// holds its own 128 accumulator rows, so the epilogue is unchanged.
//   full[s]   leader only: expect_tx(both CTAs' bytes); both CTAs' TMA complete on it
//   empty[s]  both: multicast tcgen05.commit from the leader
//   tfull[a]  both: multicast commit; tempty[a] leader: arrivals from both epilogues
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void* p) {  // same smem offset in CTA rank 0
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

template <int BN, int STAGES, bool AK, bool BKM, int EPW, bool DB = false, int KSUB = kKsubBig>
struct Cfg2 {
  static constexpr int BNH = BN / 2;  // B rows staged per CTA
  // BN = 224 (N = 896 = 4 x 224 without the half-empty fourth 256 tile): the B stage keeps
  // the 128-row footprint (K-major loads 112 rows; MN-major loads two 64-column swizzle
  // atoms, the MMA reads 112 of their columns), TMEM buffers sit 224 columns apart
  static constexpr int BNS = BN == 224 ? 128 : BNH;  // staged B footprint (rows / columns)
  static constexpr int TMEM_COLS = BN == 224 ? 512 : 2 * BN;  // alloc: power of two
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = BNS * BK * 2;
  static constexpr int B_LOAD = (BKM ? BNH : BNS) * BK * 2;  // bytes the B loads of a k-block deliver
  static constexpr int KB_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGE_BYTES = KSUB * KB_BYTES;
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;
  static constexpr int STG_WARP = DB ? 10240 : kStageBytes;  // DB: 2 residual/fp32 + 1 bf16 buffer
  static constexpr int BAR_OFF = STG_OFF + EPW * STG_WARP;
  static constexpr int SMEM = BAR_OFF + 1024 + 512;
  static constexpr int THREADS = 128 + EPW * 32;
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((AK ? 0u : 1u) << 15) |
                                    ((BKM ? 0u : 1u) << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(256 >> 4) << 24);
};

template <int BN, int STAGES, bool AK, bool BKM, int EPW, bool DB>
__global__ void __launch_bounds__(Cfg2<BN, STAGES, AK, BKM, EPW, DB>::THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ OutMaps om, GemmShape g, Epi e) {
  using C = Cfg2<BN, STAGES, AK, BKM, EPW, DB>;
  constexpr int KSUB = kKsubBig;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* ebar = tempty + 2;       // [2 * EPW] epilogue TMA-load barriers (2 per warp in DB)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + 2 * EPW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GEMM_MARK(0);
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nkb = (g.K + BK - 1) / BK;
  const int tiles_m = (g.M + 255) / 256, tiles_n = (g.N + BN - 1) / BN;
  const int ntile = tiles_m * tiles_n;
  // split-K (EPI_ACCUM only), as in the single-CTA kernel: item w = (tile w % ntile, K slice
  // w / ntile); each CTA's epilogue warps reduce their 128-row half in slice order
  const int S = e.splits > 1 ? e.splits : 1;
  const int kps = (nkb + S - 1) / S;
  const int nitem = ntile * S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPW * 32);
    }
    for (int w = 0; w < 2 * EPW; ++w) mbar_init(&ebar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / TMA
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) GEMM_MARK(1);
  pdl_wait();  // set-up above overlapped the previous kernel; its outputs are visible now
  if (threadIdx.x == 0) GEMM_MARK(2);

  if (warp == 0) {
    if (lane == 0) {
      int kb_all = 0;
      for (int w = pair; w < nitem; w += npairs) {
        const int t = w % ntile, kb_lo = (w / ntile) * kps, kb_hi = min(nkb, kb_lo + kps);
        const int m0 = tile_m(g, t, tiles_m, tiles_n) * 256 + static_cast<int>(rank) * 128;
        const int n0 = tile_n(g, t, tiles_m, tiles_n) * BN + static_cast<int>(rank) * C::BNH;
        for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KSUB, ++kb_all) {
          const int s = kb_all % STAGES;
          const uint32_t ph = (kb_all / STAGES) & 1;
          mbar_wait_pipe(&empty[s], ph ^ 1);
          GEMM_TRACE(0, kb_all);
          const int cnt = min(KSUB, kb_hi - kb0);
          const uint32_t lb = leader_addr(&full[s]);
          if (leader) mbar_expect_tx(&full[s], 2 * cnt * (C::A_BYTES + C::B_LOAD));
          for (int sub = 0; sub < cnt; ++sub) {
            const int kb = kb0 + sub;
            uint8_t* sa_ = smem + s * C::STAGE_BYTES + sub * C::KB_BYTES;
            uint8_t* sb_ = sa_ + C::A_BYTES;
            const int k0 = kb * BK;
            if (AK) {
              tma_load_2d_pair(sa_, &mapA, lb, k0, m0);
            } else {
              tma_load_2d_pair(sa_, &mapA, lb, m0, k0);
              tma_load_2d_pair(sa_ + 64 * BK * 2, &mapA, lb, m0 + 64, k0);
            }
            if (BKM) {
              tma_load_2d_pair(sb_, &mapB, lb, k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < C::BNS / 64; ++j) tma_load_2d_pair(sb_ + j * 64 * BK * 2, &mapB, lb, n0 + 64 * j, k0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      int kb_all = 0, i = 0;
      for (int w = pair; w < nitem; w += npairs, ++i) {
        const int kb_lo = (w / ntile) * kps, kb_hi = min(nkb, kb_lo + kps);
        const int acc = i & 1;
        const uint32_t aph = (i >> 1) & 1;
        mbar_wait_cluster(&tempty[acc], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KSUB, ++kb_all) {
          const int s = kb_all % STAGES;
          const uint32_t ph = (kb_all / STAGES) & 1;
          GEMM_TRACE(1, kb_all);
          mbar_wait_pipe(&full[s], ph);
          GEMM_TRACE(2, kb_all);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int cnt = min(KSUB, kb_hi - kb0);
#pragma unroll 1
          for (int sub = 0; sub < cnt; ++sub) {
            const int kb = kb0 + sub;
            const uint32_t sa_ = smem_u32(smem + s * C::STAGE_BYTES + sub * C::KB_BYTES);
            const uint32_t sb_ = sa_ + C::A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t da = AK ? smem_desc(sa_ + k * 32, 16, 1024) : smem_desc(sa_ + k * 2048, 64 * BK * 2, 1024);
              const uint64_t db = BKM ? smem_desc(sb_ + k * 32, 16, 1024) : smem_desc(sb_ + k * 2048, 64 * BK * 2, 1024);
              umma_bf16_pair(d, da, db, C::IDESC, (kb > kb_lo || k > 0) ? 1u : 0u);
            }
          }
          umma_commit_pair(&empty[s]);
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = ew & 3;
    const int slice = ew >> 2;
    constexpr int NSL = EPW / 4;
    constexpr int CW = (BN / 32 + NSL - 1) / NSL * 32;  // 32-column chunks per slice (224: 128 + 96)
    const int c_lo = min(BN, slice * CW), c_hi = min(BN, (slice + 1) * CW);
    auto al = [](const void* p, int64_t ld, int esz) {
      return p == nullptr || (((reinterpret_cast<uintptr_t>(p) | static_cast<uintptr_t>(ld * esz)) & 15) == 0);
    };
    const bool vec = al(e.c32, e.ldc32, 4) && al(e.cT, e.ldcT, 2) && al(e.resid, e.ldr, 4) &&
                     al(e.aux, e.ld_aux, 2) && al(e.bias, 0, 4);
    const uint32_t tempty_leader0 = leader_addr(&tempty[0]), tempty_leader1 = leader_addr(&tempty[1]);
    const uint32_t stg = smem_u32(smem + C::STG_OFF + ew * C::STG_WARP);
    uint32_t ephase = 0, eph2[2] = {0, 0};
    int i = 0;
    for (int w = pair; w < nitem; w += npairs, ++i) {
      const int t = w % ntile, sp = w / ntile;
      const int m0 = tile_m(g, t, tiles_m, tiles_n) * 256 + static_cast<int>(rank) * 128,
                n0 = tile_n(g, t, tiles_m, tiles_n) * BN;
      const int acc = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      mbar_wait_sleep(&tfull[acc], aph);
      GEMM_TILE(i, 0);
      if (threadIdx.x == 128 && i == 0) GEMM_MARK(3);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t* flag = S > 1 ? e.split_flags + (t * 2 + static_cast<int>(rank)) * EPW + ew : nullptr;
      if (flag && sp > 0) split_wait(flag, sp, lane);  // K slices reduce into C in slice order
      const uint32_t taddr = tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      if (DB && (e.tma & 4))
        epilogue_resid_db(g, e, om, taddr, m0 + q * 32, n0, c_lo, c_hi, stg, lane, &ebar[2 * ew], eph2);
      else if (kAuxDb && e.kind == EPI_DTANH && e.tma == (2 | 8) && !e.bias)
        epilogue_aux_db(g, e, om, taddr, m0 + q * 32, n0, c_lo, c_hi, stg, lane, &ebar[2 * ew], eph2);
      else if (e.tma)
        epilogue_store_tma(g, e, om, taddr, m0 + q * 32 + lane, m0 + q * 32, n0, c_lo, c_hi, stg, lane,
                           &ebar[2 * ew], ephase, sp > 0 ? nullptr : e.bias);
      else
        epilogue_store(g, e, taddr, m0 + q * 32 + lane, n0, c_lo, c_hi, vec);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acc ? tempty_leader1
                                                                                            : tempty_leader0)
                   : "memory");
      if (flag) split_signal(flag, lane);
      GEMM_TILE(i, 1);
    }
    if (threadIdx.x == 128) GEMM_MARK(4);
    stage_drain(lane);
    if (threadIdx.x == 128) GEMM_MARK(5);
  }
  pdl_trigger();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

template <int BN, int STAGES, bool AK, bool BKM, bool DB = false, int EPW = 8>
void launch2(cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& om, const GemmShape& g,
             const Epi& e) {
  // STAGES counts k-blocks; the ring holds STAGES / KSUB stages of KSUB k-blocks
  constexpr int NST = STAGES / kKsubBig < 2 ? 2 : STAGES / kKsubBig;
  using C = Cfg2<BN, NST, AK, BKM, EPW, DB>;
  static_assert(C::SMEM <= 232448, "shared memory");
  auto k = gemm_tc2_kernel<BN, NST, AK, BKM, EPW, DB>;
  static bool attr = false;
  if (!attr) {
    DCU_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int ntile = ((g.M + 255) / 256) * ((g.N + BN - 1) / BN) * (e.splits > 1 ? e.splits : 1);
  const int pcap = num_sms() / 2;
  const int npairs = ntile < pcap ? ntile : pcap;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * npairs);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr_c[2];
  attr_c[0].id = cudaLaunchAttributeClusterDimension;
  attr_c[0].val.clusterDim.x = 2;
  attr_c[0].val.clusterDim.y = 1;
  attr_c[0].val.clusterDim.z = 1;
  attr_c[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_c[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_c;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  ProfScope ps(PROF_GEMM_TC, s, 2.0 * g.M * g.N * static_cast<double>(g.K), 0);
  if (ps.keyed())
    snprintf(ps.key, sizeof(ps.key), "pair 256x%d M%d N%d K%d %c%c epi%d", BN, g.M, g.N, g.K, AK ? 'k' : 'm',
             BKM ? 'k' : 'm', e.kind);
  DCU_CHECK(cudaLaunchKernelEx(&cfg, k, ma, mb, om, g, e));
  DCU_LAUNCHED();
}

}  // namespace

// cta_group::2 GEMM for 256-row-multiple-friendly shapes. Returns false if not TMA-legal.
template <int BN, int STAGES, bool DB = false, int EPW = 8>
void dispatch_pair(cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& om, const GemmShape& g,
                   const Epi& e) {
  if (g.a_kmajor && g.b_kmajor) launch2<BN, STAGES, true, true, DB, EPW>(s, ma, mb, om, g, e);
  else if (g.a_kmajor) launch2<BN, STAGES, true, false, DB, EPW>(s, ma, mb, om, g, e);
  else if (g.b_kmajor) launch2<BN, STAGES, false, true, DB, EPW>(s, ma, mb, om, g, e);
  else launch2<BN, STAGES, false, false, DB, EPW>(s, ma, mb, om, g, e);
}

// cta_group::2 GEMM with 256 x BN tiles (BN 256 or 128). Returns false if not TMA-legal.
bool gemm_tc_pair(cudaStream_t s, const GemmShape& g, const Epi& e, int BN, int splits = 1) {
  if (!legal(g)) return false;
  CUtensorMap ma, mb;
  bool ok = g.a_kmajor ? make_map(&ma, g.A, g.M, g.K, g.lda, BK, 128) : make_map(&ma, g.A, g.K, g.M, g.lda, 64, BK);
  ok = ok && (g.b_kmajor ? make_map(&mb, g.B, g.N, g.K, g.ldb, BK, BN / 2) : make_map(&mb, g.B, g.K, g.N, g.ldb, 64, BK));
  if (!ok) return false;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  Epi et = e;
  et.tma = out_maps_for(g, e, &om);
  if (splits > 1 && e.kind == EPI_ACCUM && (et.tma & 1)) {  // ordered split-K (weight gradients)
    const int tiles = ((g.M + 255) / 256) * ((g.N + BN - 1) / BN);
    et.splits = splits;
    et.split_flags = split_flag_buffer(tiles * 16);  // (tile, CTA of the pair, epilogue warp)
    DCU_CHECK(cudaMemsetAsync(et.split_flags, 0, sizeof(uint32_t) * tiles * 16, s));
  } else {
    et.splits = 1;
  }
  // residual epilogues (fp32 resid in, fp32 + bf16 out): 4 x 32 KB stages and the
  // double-buffered residual prefetch (DASHCU_GEMM_RESID_DB=0 disables)
  // Long-K residual GEMMs (K >= 2048) take 5 stages with 4 epilogue warps: their mainloop
  // needs the deeper ring more than their epilogue needs 8 warps (measured +6 % at K = 4864,
  // -10 % at K = 896). KNOB_GEMM_RESID_DEEP forces either.
  const int rdeep = knob(KNOB_GEMM_RESID_DEEP);
  const bool deep = rdeep >= 0 ? rdeep == 1 : g.K >= 2048;
  const bool rdbl = (et.tma & 4) && knob(KNOB_GEMM_RESID_DB) != 0;
  if (BN == 224) {  // N = 4 x 224 (e.g. d = 896) without the half-empty 256 tile
    if (rdbl && deep) dispatch_pair<224, 5, true, 4>(s, ma, mb, om, g, et);
    else if (rdbl) dispatch_pair<224, 4, true>(s, ma, mb, om, g, et);
    else dispatch_pair<224, 6>(s, ma, mb, om, g, et);
  } else if (BN == 256 && rdbl && deep)
    dispatch_pair<256, 5, true, 4>(s, ma, mb, om, g, et);
  else if (BN == 256 && rdbl) dispatch_pair<256, 4, true>(s, ma, mb, om, g, et);
  else if (BN == 256) dispatch_pair<256, 6>(s, ma, mb, om, g, et);  // 6 x 32 KB stages
  else dispatch_pair<128, 8>(s, ma, mb, om, g, et);            // 8 x 24 KB stages
  return true;
}

// Raster of the persistent tile schedule: N tiles fastest when A is the operand that
// cannot stay in L2 (an A panel is then read from HBM once and shared by the CTAs working
// on its N tiles), M tiles fastest otherwise. DASHCU_GEMM_RASTER=0/1 forces m / n fast.
bool raster_n_fast(const GemmShape& g) {
  const int r = knob(KNOB_GEMM_RASTER);
  if (r >= 0) return r == 1;
  const double a = 2.0 * g.M * g.K, b = 2.0 * g.N * g.K;
  return a > 2.0 * b && a > 48e6;
}

// Skinny GEMMs (at most one 128-row tile: small-batch decode, e.g. the GRPO-style arm's 32
// sequences) stream their weight matrix through every SM only with narrow N tiles: one
// 128 x 64 (N >= 4096) or 128 x 32 tile per CTA, the whole K per tile, so the per-element
// accumulation order stays that of every other tile shape (scheduling independence).
bool gemm_tc_skinny(cudaStream_t s, const GemmShape& g, const Epi& e) {
  const int BN = g.N >= 64 * 64 ? 64 : 32;
  // A box rows: the batch rounded up to 32 / 64 / 128 (both operands K-major: the decode)
  const int AR = !(g.a_kmajor && g.b_kmajor) || knob(KNOB_GEMM_SKINNY_AR) == 0 ? BM : g.M <= 32 ? 32 : g.M <= 64 ? 64 : BM;
  CUtensorMap ma, mb;
  bool ok = g.a_kmajor ? make_map(&ma, g.A, g.M, g.K, g.lda, BK, AR) : make_map(&ma, g.A, g.K, g.M, g.lda, 64, BK);
  ok = ok && (g.b_kmajor ? make_map(&mb, g.B, g.N, g.K, g.ldb, BK, BN) : make_map(&mb, g.B, g.K, g.N, g.ldb, 64, BK));
  if (!ok) return false;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  Epi et = e;
  et.tma = out_maps_for(g, e, &om);
  et.splits = 1;
  const SampleArgs none;
  // four k-blocks per ring stage (one barrier round trip per 16 MMAs), ~192 KB of ring;
  // KNOB_GEMM_SKINNY_M64: M = 64 MMAs for <= 64 rows (direct-store epilogue)
  if (AR <= 64 && knob(KNOB_GEMM_SKINNY_M64) == 1) {
    et.tma = 0;
    if (AR == 32) {
      if (BN == 64) launch<64, 4, true, true, 8, 0, 32, 4, 64>(s, ma, mb, om, g, et, none);
      else launch<32, 6, true, true, 8, 0, 32, 4, 64>(s, ma, mb, om, g, et, none);
    } else {
      if (BN == 64) launch<64, 3, true, true, 8, 0, 64, 4, 64>(s, ma, mb, om, g, et, none);
      else launch<32, 4, true, true, 8, 0, 64, 4, 64>(s, ma, mb, om, g, et, none);
    }
  } else if (AR == 32) {
    if (BN == 64) launch<64, 4, true, true, 8, 0, 32, 4>(s, ma, mb, om, g, et, none);  // 4 x 48 KB
    else launch<32, 6, true, true, 8, 0, 32, 4>(s, ma, mb, om, g, et, none);           // 6 x 32 KB
  } else if (AR == 64) {
    if (BN == 64) launch<64, 3, true, true, 8, 0, 64, 4>(s, ma, mb, om, g, et, none);  // 3 x 64 KB
    else launch<32, 4, true, true, 8, 0, 64, 4>(s, ma, mb, om, g, et, none);           // 4 x 48 KB
  } else if (g.a_kmajor && g.b_kmajor && knob(KNOB_GEMM_SKINNY_AR) != 0) {
    if (BN == 64) launch<64, 4, true, true, 8, 0, BM, 2>(s, ma, mb, om, g, et, none);  // 4 x 48 KB
    else launch<32, 4, true, true, 8, 0, BM, 2>(s, ma, mb, om, g, et, none);           // 4 x 40 KB
  } else if (BN == 64) {
    dispatch_majors<64, 8>(s, ma, mb, om, g, et);  // 8 x 24 KB stages
  } else {
    dispatch_majors<32, 8>(s, ma, mb, om, g, et);  // 8 x 20 KB stages
  }
  return true;
}

bool gemm_tc(cudaStream_t s, const GemmShape& g_in, const Epi& e) {
  if (!legal(g_in)) return false;
  GemmShape g = g_in;
  g.n_fast = raster_n_fast(g);
  if (g.M <= BM && g.b_kmajor && e.kind != EPI_ACCUM && knob(KNOB_GEMM_PAIR) == 0 && g.N <= 16384 &&
      gemm_tc_skinny(s, g, e))
    return true;
  // Tile shape by the persistent schedule: time ~ rounds x per-tile cost, rounds =
  // ceil(tiles / concurrent CTAs). Measured per-SM efficiencies: 128x128 tiles 0.76
  // (shared-memory bound), 128x256 1.0, CTA-pair 256x256 1.12 (B staged half per SM).
  const int tm = (g.M + BM - 1) / BM, tm2 = (g.M + 255) / 256;
  const double sms = static_cast<double>(num_sms());
  const double r128 = std::ceil(tm * ((g.N + 127) / 128) / sms);
  const double r256 = std::ceil(tm * ((g.N + 255) / 256) / sms);
  const double rpair = std::ceil(tm2 * ((g.N + 255) / 256) / std::floor(sms / 2));
  const double rpair128 = std::ceil(tm2 * ((g.N + 127) / 128) / std::floor(sms / 2));
  double c128 = r128 * 0.5 / 0.76, c256 = r256;
  // the 256 x 128 pair tile: half the N granularity, but measured at ~0.68 of the 128 x 256
  // per-SM rate (fwd_w2 771 vs 1166 TF/s), so it rarely wins
  const double cpair = rpair / 1.12, cpair128 = rpair128 * 0.5 / 0.68;
  // 256 x 224 pair tiles: same tile count as 256 x 256 when N is a multiple of 224 but not
  // of 256 (N = 896: 4 full tiles instead of 3.5), 7/8 of the MMA work per tile
  int pbn = 256;
  double pscale = 1.0;
  {
    const double c = std::ceil(tm2 * ((g.N + 223) / 224) / std::floor(sms / 2)) * 224 / 256.0;
    if (c < rpair * 0.98) pbn = 224, pscale = c / rpair;
  }
  const bool use224 = pbn != 256;
  // ordered split-K for accumulating pair GEMMs with few tiles (the weight gradients, e.g.
  // dW1 = 19 x 4 pair tiles for 74 pairs: 2 rounds of which one is 3 % full), same cost
  // model as the single-CTA split below
  int splitp = 1;
  double cpair_s = rpair * pscale;
  if (e.kind == EPI_ACCUM && e.c32 && !knob(KNOB_NO_SPLITK)) {
    const int tp = tm2 * ((g.N + pbn - 1) / pbn), nkb_ = (g.K + BK - 1) / BK;
    for (int S = 2; S <= knob(KNOB_SPLITK_MAX) && nkb_ / S >= 16; ++S) {
      const double c = std::ceil(tp * S / std::floor(sms / 2)) / S * (pbn / 256.0) * (1.0 + 0.03 * (S - 1));
      if (c < cpair_s * 0.97) cpair_s = c, splitp = S;
    }
  }
  // Split-K for accumulating GEMMs with few output tiles (weight gradients over a long
  // token axis): S K slices per tile fill the machine; each extra slice costs one more
  // ordered fp32 reduce of the tile (~3%). Slices keep >= 16 k-blocks. S <= 4
  // (KNOB_SPLITK_MAX): the slices of a tile run in the same round and reduce one after the
  // other, so more slices serialise more epilogues (wgrad_qkv 93.6 -> 78.2 us at <= 4)
  int split128 = 1, split256 = 1;
  const int nkb = (g.K + BK - 1) / BK;
  if (e.kind == EPI_ACCUM && e.c32 && !knob(KNOB_NO_SPLITK)) {
    auto best = [&](int tiles, double unit, double* cost) {
      int sb = 1;
      for (int S = 2; S <= knob(KNOB_SPLITK_MAX) && nkb / S >= 16; ++S) {
        const double c = std::ceil(tiles * S / sms) / S * unit * (1.0 + 0.03 * (S - 1));
        if (c < *cost * 0.97) *cost = c, sb = S;
      }
      return sb;
    };
    split128 = best(tm * ((g.N + 127) / 128), 0.5 / 0.76, &c128);
    split256 = best(tm * ((g.N + 255) / 256), 1.0, &c256);
  }
  // KNOB_GEMM_PAIR: 1 force the 256x256 pair, 2 force the 256x128 pair, 3 force the
  // 256x224 pair, 0 model, -1 never
  const int forced = knob(KNOB_GEMM_PAIR);
  if (forced != -1) {
    const double cp = cpair_s / 1.12;
    const bool p256 = forced == 1 || forced == 3 || (forced == 0 && cp < c256 && cp < c128 && cp <= cpair128);
    const bool p128 = forced == 2 || (forced == 0 && !p256 && cpair128 < c256 && cpair128 < c128);
    const int bn = forced == 3 ? 224 : (forced != 1 && use224) ? pbn : 256;
    if ((p256 && gemm_tc_pair(s, g, e, bn, bn == pbn ? splitp : 1)) || (p128 && gemm_tc_pair(s, g, e, 128)))
      return true;
  }
  const int BN = c256 <= c128 ? 256 : 128;
  CUtensorMap ma, mb;
  bool ok = g.a_kmajor ? make_map(&ma, g.A, g.M, g.K, g.lda, BK, BM) : make_map(&ma, g.A, g.K, g.M, g.lda, 64, BK);
  ok = ok && (g.b_kmajor ? make_map(&mb, g.B, g.N, g.K, g.ldb, BK, BN) : make_map(&mb, g.B, g.K, g.N, g.ldb, 64, BK));
  if (!ok) return false;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  Epi et = e;
  et.tma = out_maps_for(g, e, &om);
  et.splits = 1;
  const int S = BN == 256 ? split256 : split128;
  if (S > 1 && (et.tma & 1)) {
    const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
    et.splits = S;
    et.split_flags = split_flag_buffer(tiles * 8);
    DCU_CHECK(cudaMemsetAsync(et.split_flags, 0, sizeof(uint32_t) * tiles * 8, s));
  }
  if (BN == 256) dispatch_majors<256, 4, kKsubBig>(s, ma, mb, om, g, et);  // 4 x 48 KB stages
  else dispatch_majors<128, 6, kKsubBig>(s, ma, mb, om, g, et);             // 6 x 32 KB stages
  return true;
}

int gemm_tc_sample_tiles(int N) { return (N + kSlice - 1) / kSlice; }  // one record per 32-id slice

int gemm_tc_sample(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa) {
  if (!legal(g) || !g.a_kmajor || !g.b_kmajor) return 0;
  CUtensorMap ma, mb;
  if (!make_map(&ma, g.A, g.M, g.K, g.lda, BK, BM) || !make_map(&mb, g.B, g.N, g.K, g.ldb, BK, kSampleBN)) return 0;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  if (sa.logits && !make_out_map(&om.f32, sa.logits, g.M, g.N, sa.logits_ld, true)) return 0;
  Epi e;
  e.bias = bias;
  SampleArgs a = sa;
  a.ntiles = gemm_tc_sample_tiles(g.N);
  launch<kSampleBN, 4, true, true, kSampleEPW, 1>(s, ma, mb, om, g, e, a);
  return a.ntiles;
}

bool gemm_tc_slice(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa) {
  if (!legal(g) || !g.a_kmajor || !g.b_kmajor) return false;
  CUtensorMap ma, mb;
  if (!make_map(&ma, g.A, g.M, g.K, g.lda, BK, BM) || !make_map(&mb, g.B, g.N, g.K, g.ldb, BK, kSlice)) return false;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  Epi e;
  e.bias = bias;
  launch<kSampleBN, 4, true, true, kSampleEPW, 4>(s, ma, mb, om, g, e, sa);
  return true;
}

int gemm_tc_lse_tiles(int N) { return ((N + 255) / 256) * 2; }  // two column slices per tile (8 epilogue warps)

int gemm_tc_lse(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa) {
  if (!legal(g) || !g.a_kmajor || !g.b_kmajor) return 0;
  CUtensorMap ma, mb;
  if (!make_map(&ma, g.A, g.M, g.K, g.lda, BK, BM) || !make_map(&mb, g.B, g.N, g.K, g.ldb, BK, 256)) return 0;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  Epi e;
  e.bias = bias;
  SampleArgs a = sa;
  a.ntiles = gemm_tc_lse_tiles(g.N);
  launch<256, 4, true, true, 8, 2>(s, ma, mb, om, g, e, a);
  return a.ntiles;
}

bool gemm_tc_dz(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa) {
  if (!legal(g) || !g.a_kmajor || !g.b_kmajor) return false;
  CUtensorMap ma, mb;
  if (!make_map(&ma, g.A, g.M, g.K, g.lda, BK, BM) || !make_map(&mb, g.B, g.N, g.K, g.ldb, BK, 256)) return false;
  OutMaps om;
  memset(&om, 0, sizeof(om));
  if (!make_out_map(&om.b16, sa.dz, g.M, g.N, sa.ld_dz, false)) return false;
  Epi e;
  e.bias = bias;
  launch<256, 4, true, true, 8, 3>(s, ma, mb, om, g, e, sa);
  return true;
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
}  // namespace

namespace {
// Encoded maps by (base, shape, box, type): the decode re-launches the same ~8 GEMM shapes on
// the same buffers every step, and cuTensorMapEncodeTiled costs more host time than the
// launch itself at small batch. Per thread, bounded (cleared when it fills up).
struct MapKey {
  const void* base;
  int64_t rows, cols, ld;
  int box_cols, box_rows, flags;
  bool operator==(const MapKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && ld == o.ld && box_cols == o.box_cols &&
           box_rows == o.box_rows && flags == o.flags;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = reinterpret_cast<uint64_t>(k.base) * 0x9E3779B97F4A7C15ull;
    for (int64_t v : {k.rows, k.cols, k.ld, static_cast<int64_t>(k.box_cols) << 20 | k.box_rows << 4 | k.flags})
      h = (h ^ static_cast<uint64_t>(v)) * 0xBF58476D1CE4E5B9ull;
    return static_cast<size_t>(h ^ (h >> 31));
  }
};
thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> t_maps;
}  // namespace

bool tma_map_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_cols, int box_rows,
                bool f32, int swizzle_bytes, bool l2_promote) {
  const MapKey key{base, rows, cols, ld, box_cols, box_rows, (f32 ? 1 : 0) | (l2_promote ? 2 : 0) | (swizzle_bytes << 2)};
  auto it = t_maps.find(key);
  if (it != t_maps.end()) {
    *m = it->second;
    return true;
  }
  auto fn = encode_fn();
  const int esz = f32 ? 4 : 2;
  if (!fn || !base || ((reinterpret_cast<uintptr_t>(base) | static_cast<uintptr_t>(ld * esz)) & 15)) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esz)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  l2_promote ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (t_maps.size() >= 4096) t_maps.clear();
  t_maps.emplace(key, *m);
  return true;
}


}  // namespace dashcu
