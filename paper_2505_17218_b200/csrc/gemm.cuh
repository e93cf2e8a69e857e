// GEMM interface shared by the CUDA-core (parity) and tcgen05 (production) kernels.
//
//   C[M x N] = epilogue( alpha * sum_k A(m, k) * B(n, k) )
//
// A(m, k) = a_kmajor ? A[m*lda + k] : A[k*lda + m]
// B(n, k) = b_kmajor ? B[n*ldb + k] : B[k*ldb + n]
//
// Forward projections are (K, K) (x @ W^T with W row-major [out x in], the
// reference's y = W x, policy.cpp:21-28); input gradients are (K, MN)
// (dX = dY @ W); weight gradients are (MN, MN) (dW += dY^T @ X), accumulated
// in place into the fp32 gradient (the reference's add_scaled, tensors.cpp:109).
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace dashcu {

enum EpiKind : int {
  EPI_STORE = 0,  // out = v (+bias) (+resid)
  EPI_TANH = 1,   // out = tanh(v + bias)                       policy.cpp:137
  EPI_DTANH = 2,  // out = v * (1 - aux^2)                      policy.cpp:261
  EPI_ACCUM = 3,  // c32 += v                                   wgrad, beta = 1
};

struct Epi {
  int kind = EPI_STORE;
  float alpha = 1.f;
  const float* bias = nullptr;   // [N]
  const float* resid = nullptr;  // fp32 [M x ldr]
  int64_t ldr = 0;
  const void* aux = nullptr;     // T [M x ld_aux] (EPI_DTANH)
  int64_t ld_aux = 0;
  float* c32 = nullptr;          // fp32 output / accumulator
  int64_t ldc32 = 0;
  void* cT = nullptr;            // T output (operand copy for the next GEMM)
  int64_t ldcT = 0;
  int tma = 0;                   // set by the tcgen05 launcher: bit 0 c32, bit 1 cT via bulk tensor stores
  int splits = 1;                // set by the tcgen05 launcher: split-K slices (EPI_ACCUM only)
  uint32_t* split_flags = nullptr;
};

struct GemmShape {
  int M, N, K;
  const void* A;
  int64_t lda;
  bool a_kmajor;
  const void* B;
  int64_t ldb;
  bool b_kmajor;
  // tile raster of the persistent schedule (set by the dispatcher): false = M tiles vary
  // fastest (a B panel is shared by the CTAs of a round), true = N tiles vary fastest (an
  // A panel is shared, so an A larger than L2 streams from HBM once instead of once per
  // N tile)
  bool n_fast = false;
};

// LM-head sampling epilogue (policy.cpp:148-151 + :399-424 with the DESIGN.md §4 rule):
// per (row, 32-id slice) the epilogue writes one float4 {m_s, Z_s, m1_s, Z1_s}: the slice
// max and sexp2 sum at 1/T and at T = 1 over non-BOS ids, plus the fp32 logits;
// sample_scan walks the slice sums of a row (inverse CDF) and picks the token.
// The same tile machinery also runs the LM-head backward without ever storing
// fp32 logits (policy.cpp:471-483): pass 1 (LSE mode) writes per (row, slice)
// {max, sum exp} partials, lse_reduce makes the row LSE; pass 2 (DZ mode)
// recomputes the logits and writes dz = w_r (onehot(y_r) - softmax) in bf16.
struct SampleArgs {
  const uint64_t* keys = nullptr;  // per-row sequence key derive_seed(round, "sample", m, g)
  int step = 0;
  float inv_t = 1.f;
  int bos = -1;
  float* part = nullptr;  // [rows][ntiles][4] (sample: per 32-id slice) or [rows][ntiles][2] (lse)
  int ntiles = 0;
  float* logits = nullptr;  // sample: fp32 logits row r at logits + r * logits_ld (the scan
  int64_t logits_ld = 0;    //   reads the chosen slice; also the parity dump)
  const float* lse = nullptr;      // DZ: per-row log-sum-exp over non-BOS logits
  const int32_t* target = nullptr; // DZ: per-row target id
  const float* weight = nullptr;   // DZ: per-row weight w_r = A_n / N
  bf16* dz = nullptr;              // DZ: [rows][ld_dz]
  int64_t ld_dz = 0;
  const SliceSel* sel = nullptr;   // SLICE: per-row chosen slice (sample_scan phase 1)
};
int gemm_tc_lse(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa);
bool gemm_tc_dz(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa);
int gemm_tc_lse_tiles(int N);

// dtype: 0 fp32 (CUDA cores), 1 bf16 (tcgen05 when the operands are TMA-legal)
void gemm(cudaStream_t s, int dtype, const GemmShape& g, const Epi& e);
template <class T>
void gemm_simt(cudaStream_t s, const GemmShape& g, const Epi& e);
// tcgen05 path; returns false if the shape is not TMA-legal (strides must be 16-byte multiples).
bool gemm_tc(cudaStream_t s, const GemmShape& g, const Epi& e);
// Fused LM head + sampling partials; returns the number of N tiles (0 if not TMA-legal).
int gemm_tc_sample(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa);
int gemm_tc_sample_tiles(int N);
// The chosen 32-id slice of every row recomputed on the sampling GEMM's instruction sequence:
// sa.logits[row * 32 + i] = logit of id 32 sel[row].sb + i (bias added), bit-identical to the
// sampling epilogue's value; g = the sampling GEMM's shape (A = the rows, B = W_out).
bool gemm_tc_slice(cudaStream_t s, const GemmShape& g, const float* bias, const SampleArgs& sa);

template <class T>
__device__ __forceinline__ void epi_apply(const Epi& e, int m, int n, float acc) {
  float v = e.alpha * acc;
  if (e.bias) v += e.bias[n];
  if (e.kind == EPI_TANH) v = tanhf(v);
  if (e.kind == EPI_DTANH) {
    const float a = tof<T>(static_cast<const T*>(e.aux)[static_cast<int64_t>(m) * e.ld_aux + n]);
    v *= (1.f - a * a);
  }
  if (e.resid) v += e.resid[static_cast<int64_t>(m) * e.ldr + n];
  if (e.kind == EPI_ACCUM) {
    e.c32[static_cast<int64_t>(m) * e.ldc32 + n] += v;
    return;
  }
  if (e.c32) e.c32[static_cast<int64_t>(m) * e.ldc32 + n] = v;
  if (e.cT) static_cast<T*>(e.cT)[static_cast<int64_t>(m) * e.ldcT + n] = fromf<T>(v);
}

}  // namespace dashcu
