// CUDA-core tiled GEMM: the fp32 parity path (SURVEY App.B D9: "SIMT fp32 FMA,
// no TF32") and the fallback for operand strides TMA cannot describe.
// 64x64 tile, BK = 16, 256 threads, 4x4 outputs per thread, fp32 accumulate.
#include "gemm.cuh"

namespace dashcu {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <class T, bool AK, bool BKM>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmShape g, Epi e) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const T* A = static_cast<const T*>(g.A);
  const T* B = static_cast<const T*>(g.B);
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int idx = tid + r * 256;
      int mm, kk;
      if (AK) {
        mm = idx / BK;
        kk = idx % BK;
      } else {
        mm = idx % BM;
        kk = idx / BM;
      }
      const int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < g.M && gk < g.K) v = tof<T>(AK ? A[static_cast<int64_t>(gm) * g.lda + gk] : A[static_cast<int64_t>(gk) * g.lda + gm]);
      As[kk][mm] = v;
      int nn;
      if (BKM) {
        nn = idx / BK;
        kk = idx % BK;
      } else {
        nn = idx % BN;
        kk = idx / BN;
      }
      const int gn = n0 + nn, gk2 = k0 + kk;
      float w = 0.f;
      if (gn < g.N && gk2 < g.K) w = tof<T>(BKM ? B[static_cast<int64_t>(gn) * g.ldb + gk2] : B[static_cast<int64_t>(gk2) * g.ldb + gn]);
      Bs[kk][nn] = w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < g.N) epi_apply<T>(e, m, n, acc[i][j]);
    }
  }
}

}  // namespace

template <class T>
void gemm_simt(cudaStream_t s, const GemmShape& g, const Epi& e) {
  if (g.M <= 0 || g.N <= 0) return;
  dim3 grid(cdiv(g.N, BN), cdiv(g.M, BM));
  ProfScope ps(PROF_GEMM_SIMT, s, 2.0 * g.M * g.N * static_cast<double>(g.K), 0);
  if (g.a_kmajor && g.b_kmajor) gemm_simt_kernel<T, true, true><<<grid, 256, 0, s>>>(g, e);
  else if (g.a_kmajor && !g.b_kmajor) gemm_simt_kernel<T, true, false><<<grid, 256, 0, s>>>(g, e);
  else if (!g.a_kmajor && g.b_kmajor) gemm_simt_kernel<T, false, true><<<grid, 256, 0, s>>>(g, e);
  else gemm_simt_kernel<T, false, false><<<grid, 256, 0, s>>>(g, e);
  DCU_LAUNCHED();
}

template void gemm_simt<float>(cudaStream_t, const GemmShape&, const Epi&);
template void gemm_simt<bf16>(cudaStream_t, const GemmShape&, const Epi&);

void gemm(cudaStream_t s, int dtype, const GemmShape& g, const Epi& e) {
  if (g.M <= 0 || g.N <= 0) return;
  if (dtype == 0) {
    gemm_simt<float>(s, g, e);
    return;
  }
  if (!gemm_tc(s, g, e)) gemm_simt<bf16>(s, g, e);
}

}  // namespace dashcu
