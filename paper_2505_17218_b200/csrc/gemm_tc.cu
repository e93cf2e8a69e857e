// tcgen05 tensor-core GEMM for sm_100a (bf16 x bf16 -> fp32 in TMEM).
//
//   C[M x N] = epilogue(A(m, k) . B(n, k)),  operands K-major or MN-major.
//
// Warp roles per CTA (256 threads, one 128 x BN output tile):
//   warp 0      TMA producer: 128B-swizzled tiles of A and B into a STAGES-deep
//               shared-memory ring (cp.async.bulk.tensor + mbarrier complete_tx)
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128, N=BN,
//               K=16) into a TMEM accumulator; tcgen05.commit frees the smem slot
//   warp 2      TMEM allocator (BN columns)
//   warps 4..7  epilogue: tcgen05.ld 32 columns at a time -> bias / tanh /
//               dtanh / residual / fp32 accumulate -> global
// Operand major-ness is encoded in the UMMA instruction descriptor (bits 15/16)
// and the shared-memory descriptors (K-major: SBO = 1024 B between 8-row groups;
// MN-major: LBO = one 64-element TMA box, SBO = 1024 B between 8-k groups).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm.cuh"

namespace dashcu {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fff) | (static_cast<uint64_t>((lbo >> 4) & 0x3fff) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int BN, int STAGES, bool AK, bool BKM>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  // kind::f16 instruction descriptor: D f32, A/B bf16, majors, N>>3, M>>4
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((AK ? 0u : 1u) << 15) |
                                    ((BKM ? 0u : 1u) << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(BM >> 4) << 24);
};

template <int BN, int STAGES, bool AK, bool BKM>
__global__ void __launch_bounds__(256, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, GemmShape g,
                   Epi e) {
  using C = Cfg<BN, STAGES, AK, BKM>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nkb = (g.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * C::STAGE_BYTES;
        uint8_t* sb = sa + C::A_BYTES;
        mbar_expect_tx(&full[s], C::STAGE_BYTES);
        const int k0 = kb * BK;
        if (AK) {
          tma_load_2d(sa, &mapA, &full[s], k0, m0);
        } else {
          tma_load_2d(sa, &mapA, &full[s], m0, k0);
          tma_load_2d(sa + 64 * BK * 2, &mapA, &full[s], m0 + 64, k0);
        }
        if (BKM) {
          tma_load_2d(sb, &mapB, &full[s], k0, n0);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 64 * BK * 2, &mapB, &full[s], n0 + 64 * j, k0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // K-major: advance 32 B inside the swizzle row; MN-major: advance 16 k-rows (2 x 1024 B)
          const uint64_t da = AK ? smem_desc(sa + k * 32, 16, 1024) : smem_desc(sa + k * 2048, 64 * BK * 2, 1024);
          const uint64_t db = BKM ? smem_desc(sb + k * 32, 16, 1024) : smem_desc(sb + k * 2048, 64 * BK * 2, 1024);
          umma_bf16(tmem, da, db, C::IDESC, (kb > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tfull);
    }
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lane quarter
    const int row = m0 + q * 32 + lane;
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float v[32];
    // 16-byte vector path: every pointer / leading dim the epilogue touches is 16-B aligned
    auto al = [](const void* p, int64_t ld, int esz) {
      return p == nullptr || (((reinterpret_cast<uintptr_t>(p) | static_cast<uintptr_t>(ld * esz)) & 15) == 0);
    };
    const bool vec = al(e.c32, e.ldc32, 4) && al(e.cT, e.ldcT, 2) && al(e.resid, e.ldr, 4) && al(e.aux, e.ld_aux, 2) &&
                     al(e.bias, 0, 4);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
      if (row >= g.M) continue;
      const int nb = n0 + c;
      if (vec && nb + 32 <= g.N) {
        const int64_t r64 = row;
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= e.alpha;
        if (e.bias) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = *reinterpret_cast<const float4*>(e.bias + nb + i);
            v[i] += b.x, v[i + 1] += b.y, v[i + 2] += b.z, v[i + 3] += b.w;
          }
        }
        if (e.kind == EPI_TANH) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = tanhf(v[i]);
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
          for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(cp + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
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
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

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

// 2-D bf16 tensor map over a row-major [rows x cols] matrix with leading dim ld.
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int STAGES, bool AK, bool BKM>
void launch(cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, const GemmShape& g, const Epi& e) {
  using C = Cfg<BN, STAGES, AK, BKM>;
  auto k = gemm_tc_kernel<BN, STAGES, AK, BKM>;
  static bool attr = false;
  if (!attr) {
    DCU_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM);
  ProfScope ps(PROF_GEMM_TC, s, 2.0 * g.M * g.N * static_cast<double>(g.K), 0);
  k<<<grid, 256, C::SMEM, s>>>(ma, mb, g, e);
  DCU_LAUNCHED();
}

}  // namespace

bool gemm_tc(cudaStream_t s, const GemmShape& g, const Epi& e) {
  if (g.K <= 0 || g.M <= 0 || g.N <= 0) return false;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(g.A), pb = reinterpret_cast<uintptr_t>(g.B);
  if ((pa & 15) || (pb & 15) || ((g.lda * 2) & 15) || ((g.ldb * 2) & 15)) return false;
  constexpr int BN = 128;
  CUtensorMap ma, mb;
  bool ok = g.a_kmajor ? make_map(&ma, g.A, g.M, g.K, g.lda, BK, BM) : make_map(&ma, g.A, g.K, g.M, g.lda, 64, BK);
  ok = ok && (g.b_kmajor ? make_map(&mb, g.B, g.N, g.K, g.ldb, BK, BN) : make_map(&mb, g.B, g.K, g.N, g.ldb, 64, BK));
  if (!ok) return false;
  // 3 stages x 32 KB: two CTAs per SM, so one CTA's epilogue overlaps the other's mainloop
  if (g.a_kmajor && g.b_kmajor) launch<BN, 3, true, true>(s, ma, mb, g, e);
  else if (g.a_kmajor) launch<BN, 3, true, false>(s, ma, mb, g, e);
  else if (g.b_kmajor) launch<BN, 3, false, true>(s, ma, mb, g, e);
  else launch<BN, 3, false, false>(s, ma, mb, g, e);
  return true;
}

}  // namespace dashcu
