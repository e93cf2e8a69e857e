// Memory-bound kernels of the DASH step: parameter init/casts, the optimizer,
// embeddings, bias-gradient column sums, LM-head loss rows, the sampling step
// (non-fused form), KV-cache plumbing and the advantage/filter + compaction.
#include <cub/device/device_radix_sort.cuh>
#include <cfloat>

#include "kernels.cuh"
#include "tc5.cuh"
#include "rule.cuh"

namespace dashcu {

int64_t g_launches = 0;

namespace {

inline int grid1d(int64_t n, int bs = 256) {
  const int64_t b = (n + bs - 1) / bs;
  return static_cast<int>(b < kNumSMs * 32 ? (b < 1 ? 1 : b) : kNumSMs * 32);
}

// ---------------------------------------------------------------- init / casts

__global__ void init_normal_ctr_k(float* w, int64_t n, double scale, uint64_t key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = static_cast<uint64_t>(i >> 1);
    const uint64_t h1 = splitmix64(key ^ (2 * k));
    const uint64_t h2 = splitmix64(key ^ (2 * k + 1));
    const double u1 = (static_cast<double>(h1 >> 11) + 0.5) * 1.1102230246251565e-16;  // 2^-53
    const double u2 = static_cast<double>(h2 >> 11) * 1.1102230246251565e-16;
    const double r = sqrt(-2.0 * log(u1));
    const double t = 6.283185307179586 * u2;
    w[i] = static_cast<float>(scale * ((i & 1) ? r * sin(t) : r * cos(t)));
  }
}

__global__ void f64_to_f32_k(const double* in, float* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}
__global__ void f32_to_f64_k(const float* in, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}
__global__ void cast_bf16_k(const float* in, bf16* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}
// 8 elements per thread iteration: two 16-byte loads, one 16-byte store (n % 8 == 0, aligned)
__global__ void cast_bf16_v8_k(const float4* __restrict__ in, uint4* __restrict__ out, int64_t n8) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = in[2 * i], b = in[2 * i + 1];
    __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w),
                   p2 = __floats2bfloat162_rn(b.x, b.y), p3 = __floats2bfloat162_rn(b.z, b.w);
    out[i] = make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                        *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
  }
}
__global__ void fill_k(float* p, float v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Adam / SGD ascent on fp32 master weights; 4 elements per
// thread iteration with 16-byte accesses where aligned.
__global__ void optimizer_k(int kind, float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, bf16* __restrict__ wT, int64_t n, float lr, float b1, float b2,
                            float eps, float c1, float c2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float wi = opt_update(kind, w[i], g[i], m + i, v + i, lr, b1, b2, eps, c1, c2);
    w[i] = wi;
    if (wT) wT[i] = __float2bfloat16_rn(wi);
  }
}

// ------------------------------------------------------------------ embeddings

template <class T>
__global__ void embed_fwd_k(const T* E, const T* P, const int32_t* tok, const int32_t* pos, int rows, int d,
                            float* x32, T* xT) {
  const int64_t n = static_cast<int64_t>(rows) * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / d), c = static_cast<int>(i % d);
    const float v = tof<T>(E[static_cast<int64_t>(tok[r]) * d + c]) + tof<T>(P[static_cast<int64_t>(pos[r]) * d + c]);
    x32[i] = v;
    xT[i] = fromf<T>(v);
  }
}

template <class T>
__global__ void embed_decode_k(const T* E, const T* P, const int32_t* tok, const int32_t* plen, int step, int rows,
                               int d, float* x32, T* xT, const int32_t* row_seq, const int* step_dev) {
  pdl_wait();
  if (step_dev) step = *step_dev;
  const int64_t n = static_cast<int64_t>(rows) * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / d), c = static_cast<int>(i % d);
    const int sq = row_seq ? row_seq[r] : r;
    const int p = plen[sq] + step - 1;
    const float v = tof<T>(E[static_cast<int64_t>(tok[sq]) * d + c]) + tof<T>(P[static_cast<int64_t>(p) * d + c]);
    x32[i] = v;
    xT[i] = fromf<T>(v);
  }
}

// Embedding backward (policy.cpp:335-344: dtok[tok_t] += dx_t, dpos[pos_t] += dx_t),
// deterministic: the rows are stably sorted by id (CUB radix sort of (id, row) pairs), and
// the block that owns the first row of an id's run sums the run in row order and adds the
// sum to that id's gradient row. No floating-point atomics, so the result does not depend
// on scheduling.
__global__ void embed_seg_mark_k(const int32_t* ids, int rows, int32_t* keys, int32_t* vals) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) keys[r] = ids[r], vals[r] = r;
}

// Pass 1: window w holds sorted positions [w kEmbWin, (w+1) kEmbWin); every run of equal
// ids inside it is summed in row order into part[position of the run's first row in the
// window]. Pass 2: the block owning the head of an id's run adds that run's window partials
// in window order to the id's gradient row. Long runs (a token repeated thousands of times
// in a micro-batch) spread over many blocks in pass 1 instead of one serial loop.
constexpr int kEmbWin = 64;
__global__ void embed_win_k(const float* __restrict__ dx, const int32_t* __restrict__ skey,
                            const int32_t* __restrict__ srow, int rows, int d, float* __restrict__ part) {
  const int w0 = blockIdx.x * kEmbWin, w1 = min(rows, w0 + kEmbWin);
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (c >= d) return;
  const bool v4 = (d & 3) == 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int start = w0;
  for (int i = w0; i < w1; ++i) {
    const float* src = dx + static_cast<int64_t>(srow[i]) * d + c;
    if (v4) {
      const float4 v = *reinterpret_cast<const float4*>(src);
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    } else {
      acc.x += src[0];
      if (c + 1 < d) acc.y += src[1];
      if (c + 2 < d) acc.z += src[2];
      if (c + 3 < d) acc.w += src[3];
    }
    if (i + 1 == w1 || skey[i + 1] != skey[i]) {
      float* dst = part + static_cast<int64_t>(start) * d + c;
      if (v4) {
        *reinterpret_cast<float4*>(dst) = acc;
      } else {
        dst[0] = acc.x;
        if (c + 1 < d) dst[1] = acc.y;
        if (c + 2 < d) dst[2] = acc.z;
        if (c + 3 < d) dst[3] = acc.w;
      }
      acc = make_float4(0.f, 0.f, 0.f, 0.f);
      start = i + 1;
    }
  }
}

__global__ void embed_run_k(const float* __restrict__ part, const int32_t* __restrict__ skey, int rows, int d,
                            float* __restrict__ g) {
  const int i = blockIdx.x;
  const int key = skey[i];
  if (i > 0 && skey[i - 1] == key) return;  // not the head of its run
  float* gr = g + static_cast<int64_t>(key) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = part[static_cast<int64_t>(i) * d + c];
    // the run's later windows start at multiples of kEmbWin while the id is unchanged
    for (int p = (i / kEmbWin + 1) * kEmbWin; p < rows && skey[p] == key; p += kEmbWin)
      acc += part[static_cast<int64_t>(p) * d + c];
    gr[c] += acc;
  }
}

// Column sums (bias gradients, policy.cpp:250-262 db = sum_rows dY), deterministic and
// coalesced: pass 1 — thread = VEC consecutive columns (one 16-byte load per row) over
// one row segment, partial sums to tmp[segment][N]; pass 2 — out[n] += the segments
// in order. No atomics, so the result does not depend on scheduling.
template <class T, int VEC>
__global__ void colsum_part_k(const T* __restrict__ X, int64_t ld, int M, int N, int seg_rows, bool vec,
                              float* __restrict__ tmp) {
  const int n0 = (blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  if (n0 >= N) return;
  const int r_begin = blockIdx.y * seg_rows, r_end = min(M, r_begin + seg_rows);
  float acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
  if (vec && n0 + VEC <= N) {
#pragma unroll 4
    for (int r = r_begin; r < r_end; ++r) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(X + static_cast<int64_t>(r) * ld + n0));
      const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int i = 0; i < VEC; ++i) acc[i] += tof<T>(e[i]);
    }
  } else {
    for (int r = r_begin; r < r_end; ++r)
#pragma unroll
      for (int i = 0; i < VEC; ++i)
        if (n0 + i < N) acc[i] += tof<T>(X[static_cast<int64_t>(r) * ld + n0 + i]);
  }
  float* t = tmp + static_cast<int64_t>(blockIdx.y) * N + n0;
#pragma unroll
  for (int i = 0; i < VEC; ++i)
    if (n0 + i < N) t[i] = acc[i];
}

// block (32 columns x 32 segment lanes): lane y sums segments y, y+32, ... in order, then
// a fixed-shape tree over the 32 lanes — deterministic for a given (M, N).
__global__ void colsum_fin_k(const float* __restrict__ tmp, int nseg, int N, float* __restrict__ out) {
  __shared__ float red[32][33];
  const int n = blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (n < N)
    for (int y = threadIdx.y; y < nseg; y += 32) s += tmp[static_cast<int64_t>(y) * N + n];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  for (int w = 16; w >= 1; w >>= 1) {
    if (threadIdx.y < w) red[threadIdx.y][threadIdx.x] += red[threadIdx.y + w][threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.y == 0 && n < N) out[n] += red[0][threadIdx.x];
}

// ----------------------------------------------------------- sampling / loss rows

struct ArgBest {
  float s;
  int i;
};

__device__ __forceinline__ ArgBest block_argmax(ArgBest b, float* ss, int* si) {
  // warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float s2 = __shfl_xor_sync(0xffffffffu, b.s, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, b.i, o);
    if (better(s2, i2, b.s, b.i)) {
      b.s = s2;
      b.i = i2;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    ss[w] = b.s;
    si[w] = b.i;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    b.s = l < nw ? ss[l] : -FLT_MAX;
    b.i = l < nw ? si[l] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float s2 = __shfl_xor_sync(0xffffffffu, b.s, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, b.i, o);
      if (better(s2, i2, b.s, b.i)) {
        b.s = s2;
        b.i = i2;
      }
    }
    if (l == 0) {
      ss[0] = b.s;
      si[0] = b.i;
    }
  }
  __syncthreads();
  ArgBest r{ss[0], si[0]};
  __syncthreads();
  return r;
}

__device__ __forceinline__ float block_reduce(float v, float* sm, bool is_max) {
  v = is_max ? warp_max(v) : warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    float t = l < nw ? sm[l] : (is_max ? -FLT_MAX : 0.f);
    t = is_max ? warp_max(t) : warp_sum(t);
    if (l == 0) sm[0] = t;
  }
  __syncthreads();
  const float r = sm[0];
  __syncthreads();
  return r;
}

// Sampling partials from fp32 logits (the fp32 parity path; the bf16 path computes the
// same records in the LM-head GEMM epilogue): one thread per (row, 32-id slice),
// operations in the order of the contract (rule.cuh).
__global__ void sample_partials_k(const float* __restrict__ logits, int rows, int V, int bos, float inv_t,
                                  float* __restrict__ part, int nslices) {
  const int64_t n = static_cast<int64_t>(rows) * nslices;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(w / nslices), s = static_cast<int>(w % nslices);
    const float* l = logits + static_cast<int64_t>(r) * V + s * kSlice;
    float x[kSlice];
    float m = -FLT_MAX, m1 = -FLT_MAX;
#pragma unroll
    for (int i = 0; i < kSlice; ++i) {
      const int id = s * kSlice + i;
      const bool ok = id < V && id != bos;
      x[i] = ok ? __fmul_rn(l[i], inv_t) : -FLT_MAX;
      m = fmaxf(m, x[i]);
      m1 = fmaxf(m1, ok ? l[i] : -FLT_MAX);
    }
    float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < kSlice; ++i)
      a[i & 3] = __fadd_rn(a[i & 3], x[i] == -FLT_MAX ? 0.f : sexp2(__fmul_rn(__fsub_rn(x[i], m), kLog2e)));
    const float Z = __fadd_rn(__fadd_rn(a[0], a[1]), __fadd_rn(a[2], a[3]));
    float Z1 = Z;
    if (inv_t != 1.f) {
      Z1 = 0.f;
      for (int i = 0; i < kSlice; ++i)
        if (x[i] != -FLT_MAX) Z1 += __expf(l[i] - m1);
    } else {
      m1 = m;
    }
    reinterpret_cast<float4*>(part)[w] = make_float4(m, Z, m1, Z1);
  }
}

constexpr int kScanMaxB = 192;

// id search inside the chosen slice sb (the contract's last level) + the token bookkeeping
// of policy.cpp:423-426 (EOS stops, cap, logp at T = 1); l = the slice's 32 fp32 logits
__device__ __forceinline__ void scan_finish(const SliceSel& q, const float* l, int sq, int V, int bos, int eos,
                                            float inv_t, int step, uint8_t* finished, int32_t* comp, float* logp,
                                            int32_t* len, int32_t* tok_next, int max_len, float* lse_out) {
  int tk = -1, last_i = -1;
  float r = q.sbase;
  for (int i = 0; i < kSlice; ++i) {
    const int id = q.sb * kSlice + i;
    if (id >= V || id == bos) continue;
    const float e = sexp2(__fmul_rn(__fsub_rn(__fmul_rn(l[i], inv_t), q.ms), kLog2e));
    r = __fmaf_rn(e, q.scale, r);
    last_i = id;
    if (q.target < r) {
      tk = id;
      break;
    }
  }
  if (tk < 0) tk = last_i;
  comp[static_cast<int64_t>(sq) * max_len + step] = tk;
  logp[static_cast<int64_t>(sq) * max_len + step] = l[tk - q.sb * kSlice] - q.lse1;
  if (lse_out) lse_out[static_cast<int64_t>(sq) * max_len + step] = q.lse1;
  len[sq] = step + 1;
  if (tk == eos) finished[sq] = 1;
  tok_next[sq] = tk;
}  // slices per lane block staged in shared memory (V <= 196608)

// The inverse-CDF walk of the sampling contract (rule.cuh), one warp per row: lane j
// owns a block of consecutive slices; block, slice and id sums are accumulated in the
// contract's order, so the chosen id is a pure function of the fp32 logits, 1/T and the
// row key. Then the token bookkeeping of policy.cpp:423-426 (EOS stops, cap, logp at T=1).
// The row's slice records (38 KB at V = 151,936, T = 1) are first copied into the warp's
// shared-memory window with coalesced, independent vector loads: the lane-blocked walk
// reads lane-strided records, which straight from global memory was a chain of ~300
// dependent-latency loads per lane (33 us per decode step at any batch size).
__global__ void __launch_bounds__(256) sample_scan_k(const float* __restrict__ part, int nslices,
                                                     const float* __restrict__ logits, int64_t logits_ld, int rows,
                                                     int V, int bos, int eos, float inv_t, const uint64_t* keys,
                                                     int step, const int32_t* cap, uint8_t* finished, int32_t* comp,
                                                     float* logp, int32_t* len, int32_t* tok_next, int max_len,
                                                     bool compact, float* lse_out, const int32_t* row_seq, int phase,
                                                     SliceSel* sel, const float* dump, int64_t dump_ld,
                                                     int* mismatches, const int* step_dev) {
  pdl_wait();
  if (step_dev) step = *step_dev;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int sq = row_seq ? row_seq[row] : row;  // per-sequence state below, per-row records above
  if (phase == 2) {  // finish: the chosen slice's logits, recomputed by gemm_tc_slice (row-major [rows x 32])
    if (lane != 0) return;
    const SliceSel q = sel[row];
    if (q.sb < 0) return;
    const float* l = logits + static_cast<int64_t>(row) * kSlice;
    if (dump && mismatches) {  // parity runs: the recomputed slice must equal the GEMM's logits bit for bit
      const float* ref = dump + static_cast<int64_t>(row) * dump_ld + q.sb * kSlice;
      int bad = 0;
      for (int i = 0; i < kSlice && q.sb * kSlice + i < V; ++i)
        bad += __float_as_uint(ref[i]) != __float_as_uint(l[i]);
      if (bad) atomicAdd(mismatches, bad);
    }
    scan_finish(q, l, sq, V, bos, eos, inv_t, step, finished, comp, logp, len, tok_next, max_len, lse_out);
    return;
  }
  const bool active = !finished[sq] && step < cap[sq];
  if (!active) {
    if (lane == 0) {
      tok_next[sq] = eos;
      if (phase == 1) sel[row].sb = -1;
    }
    return;
  }
  // records {m, Z, m1, Z1}; at T = 1 the fused epilogue stores only {m, Z} (m1 = m, Z1 = Z)
  extern __shared__ float4 s_rec[];  // [warps per block][nslices records]
  __shared__ uint64_t s_bar[8];
  const int recf = compact ? 2 : 4;  // floats per record
  float* srow = reinterpret_cast<float*>(s_rec) + static_cast<int64_t>(threadIdx.x >> 5) * nslices * recf;
  {
    const float* grow = part + static_cast<int64_t>(row) * nslices * recf;
    const uint32_t bytes = static_cast<uint32_t>(nslices) * recf * 4;
    if (((reinterpret_cast<uintptr_t>(grow) | bytes) & 15) == 0) {  // one bulk (TMA) copy per row
      uint64_t* bar = &s_bar[threadIdx.x >> 5];
      if (lane == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(bar, bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(srow)),
            "l"(grow), "r"(bytes), "r"(smem_u32(bar))
            : "memory");
      }
      __syncwarp();
      mbar_wait(bar, 0);
    } else {
      const int n2 = nslices * recf / 2;  // float2 units (rows are 8-byte aligned)
      const float2* g2 = reinterpret_cast<const float2*>(grow);
      float2* s2 = reinterpret_cast<float2*>(srow);
#pragma unroll 8
      for (int i = lane; i < n2; i += 32) s2[i] = __ldg(g2 + i);
      __syncwarp();
    }
  }
  const float4* P4 = reinterpret_cast<const float4*>(srow);
  const float2* P2 = reinterpret_cast<const float2*>(srow);
  auto rec = [&](int s) -> float4 {
    if (compact) {
      const float2 q = P2[s];
      return make_float4(q.x, q.y, q.x, q.y);
    }
    return P4[s];
  };
  const int B = (nslices + 31) / 32;
  const int s0 = lane * B, s1 = min(nslices, s0 + B);
  float M = -FLT_MAX, M1 = -FLT_MAX;
  for (int s = s0; s < s1; ++s) {
    const float4 p = rec(s);
    M = fmaxf(M, p.x);
    M1 = fmaxf(M1, p.z);
  }
  M = warp_max(M);
  M1 = warp_max(M1);
  float T = 0.f, L1 = 0.f;
  for (int s = s0; s < s1; ++s) {
    const float4 p = rec(s);
    T = __fadd_rn(T, __fmul_rn(p.y, sexp2(__fmul_rn(__fsub_rn(p.x, M), kLog2e))));
    L1 += p.w * __expf(p.z - M1);
  }
  L1 = warp_sum(L1);
  // lane 0: total and block search in lane order
  float Tj[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) Tj[j] = __shfl_sync(0xffffffffu, T, j);
  // slice sums of every block, computed by the whole warp into shared memory (the same
  // fp32 operations as the sequential definition; only the walk below is sequential)
  __shared__ float sS[8][kScanMaxB];
  float* Sw = sS[threadIdx.x >> 5];
  const bool staged = B <= kScanMaxB;
  float total = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) total = __fadd_rn(total, Tj[j]);
  const float target = __fmul_rn(row_uniform(keys[sq], step), total);
  int jb = -1;
  float base = 0.f;
  {
    float cum = 0.f, last_base = 0.f;
    int last_j = -1;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float prev = cum;
      cum = __fadd_rn(cum, Tj[j]);
      if (Tj[j] > 0.f) {
        last_j = j;
        last_base = prev;
      }
      if (jb < 0 && target < cum) {
        jb = j;
        base = prev;
      }
    }
    if (jb < 0) {
      jb = last_j;
      base = last_base;
    }
  }
  if (staged) {
    for (int k = lane; k < B; k += 32) {
      const int s = jb * B + k;
      float v = 0.f;
      if (s < nslices) {
        const float4 p = rec(s);
        v = __fmul_rn(p.y, sexp2(__fmul_rn(__fsub_rn(p.x, M), kLog2e)));
      }
      Sw[k] = v;
    }
    __syncwarp();
  }
  if (lane != 0) return;
  // slice search inside block jb
  int sb = -1, last_s = -1;
  float sbase = 0.f, last_sbase = 0.f, r = base;
  for (int s = jb * B; s < min(nslices, (jb + 1) * B); ++s) {
    float Ss;
    if (staged) {
      Ss = Sw[s - jb * B];
    } else {
      const float4 p = rec(s);
      Ss = __fmul_rn(p.y, sexp2(__fmul_rn(__fsub_rn(p.x, M), kLog2e)));
    }
    const float prev = r;
    r = __fadd_rn(r, Ss);
    if (Ss > 0.f) {
      last_s = s;
      last_sbase = prev;
    }
    if (target < r) {
      sb = s;
      sbase = prev;
      break;
    }
  }
  if (sb < 0) {
    sb = last_s;
    sbase = last_sbase;
  }
  SliceSel q;
  const float4 p = rec(sb);
  q.sb = sb;
  q.target = target;
  q.sbase = sbase;
  q.ms = p.x;
  q.scale = sexp2(__fmul_rn(__fsub_rn(p.x, M), kLog2e));
  q.lse1 = M1 + logf(L1);  // T = 1 log-sum-exp over non-BOS ids (policy.cpp:424)
  if (phase == 1) {  // select: the slice is recomputed by gemm_tc_slice, the walk finishes in phase 2
    sel[row] = q;
    return;
  }
  scan_finish(q, logits + static_cast<int64_t>(row) * logits_ld + sb * kSlice, sq, V, bos, eos, inv_t, step, finished,
              comp, logp, len, tok_next, max_len, lse_out);
}

// Row LSE from the LSE-mode GEMM partials; optionally logp = logit[y] - lse with the
// target logit recomputed as a bf16 dot product in fp32 (one warp per row).
__global__ void __launch_bounds__(256) lse_reduce_k(const float* __restrict__ part, int ntiles, int rows,
                                                    float* __restrict__ lse, const bf16* __restrict__ Y, int d,
                                                    const bf16* __restrict__ W, const float* __restrict__ bias,
                                                    const int32_t* __restrict__ target, float* __restrict__ logp) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  float mx = -FLT_MAX, se = 0.f;
  for (int t = lane; t < ntiles; t += 32) {
    const float m2 = part[(static_cast<int64_t>(row) * ntiles + t) * 2];
    const float s2 = part[(static_cast<int64_t>(row) * ntiles + t) * 2 + 1];
    if (m2 > -FLT_MAX) {
      const float nm = fmaxf(mx, m2);
      se = se * __expf(mx - nm) + s2 * __expf(m2 - nm);
      mx = nm;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, se, o);
    const float nm = fmaxf(mx, m2);
    if (nm > -FLT_MAX) {
      se = se * __expf(mx - nm) + s2 * __expf(m2 - nm);
      mx = nm;
    }
  }
  const float L = mx + logf(se);
  if (lane == 0) lse[row] = L;
  if (logp) {
    const int y = target[row];
    const bf16* yr = Y + static_cast<int64_t>(row) * d;
    const bf16* wr = W + static_cast<int64_t>(y) * d;
    float a = 0.f;
    for (int i = lane; i < d; i += 32) a += __bfloat162float(yr[i]) * __bfloat162float(wr[i]);
    a = warp_sum(a);
    if (lane == 0) logp[row] = a + bias[y] - L;
  }
}

template <class T>
__global__ void __launch_bounds__(256) lm_rows_k(const float* logits, int V, int bos, const int32_t* target,
                                                 const float* weight, float* logp, T* dz) {
  __shared__ float sm[32];
  const int r = blockIdx.x;
  const float* lg = logits + static_cast<int64_t>(r) * V;
  float mx = -FLT_MAX;
  for (int i = threadIdx.x; i < V; i += blockDim.x)
    if (i != bos) mx = fmaxf(mx, lg[i]);
  mx = block_reduce(mx, sm, true);
  float sum = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x)
    if (i != bos) sum += expf(lg[i] - mx);
  sum = block_reduce(sum, sm, false);
  const float lse = mx + logf(sum);
  const int y = target[r];
  if (threadIdx.x == 0 && logp) logp[r] = lg[y] - lse;
  if (dz) {
    const float w = weight ? weight[r] : 1.f;
    T* out = dz + static_cast<int64_t>(r) * V;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      float v = 0.f;
      if (i != bos) v = w * ((i == y ? 1.f : 0.f) - expf(lg[i] - lse));
      out[i] = fromf<T>(v);
    }
  }
}

// KL term rows (kl_term, policy.cpp:487-522): per completion row r with current logits lc and
// base logits lb (fp32, BOS excluded): value[r] = sum_i pb_i ((lb_i - lse_b) - (lc_i - lse_c))
// = KL(base || current) at this context, and dz[r][i] = w_r (pc_i - pb_i) (the reference's
// dlogits, BOS column 0). The value is formed as sum_i pb_i (lb_i - lc_i) - (lse_b - lse_c)
// with fp64 sums and lse_b - lse_c = (mb - mc) + log(Sb / Sc): near base == current the two
// log-sum-exps share their rounding, so the difference is not swamped by it.
template <class T>
__global__ void __launch_bounds__(256) kl_rows_k(const float* lc_all, const float* lb_all, int V, int bos,
                                                 const float* weight, double* value, T* dz) {
  __shared__ float sm[32];
  __shared__ double smd[3][32];
  const int r = blockIdx.x;
  const float* lc = lc_all + static_cast<int64_t>(r) * V;
  const float* lb = lb_all + static_cast<int64_t>(r) * V;
  float mc = -FLT_MAX, mb = -FLT_MAX;
  for (int i = threadIdx.x; i < V; i += blockDim.x)
    if (i != bos) mc = fmaxf(mc, lc[i]), mb = fmaxf(mb, lb[i]);
  mc = block_reduce(mc, sm, true);
  mb = block_reduce(mb, sm, true);
  double sc = 0.0, sb = 0.0, sd = 0.0;  // sum e^(lc-mc), sum e^(lb-mb), sum e^(lb-mb) (lb - lc)
  for (int i = threadIdx.x; i < V; i += blockDim.x)
    if (i != bos) {
      const double eb = expf(lb[i] - mb);
      sc += expf(lc[i] - mc);
      sb += eb;
      sd += eb * static_cast<double>(lb[i] - lc[i]);
    }
  double v3[3] = {sc, sb, sd};
  for (int k = 0; k < 3; ++k) {
    v3[k] = warp_sum_d(v3[k]);
    if ((threadIdx.x & 31) == 0) smd[k][threadIdx.x >> 5] = v3[k];
  }
  __syncthreads();
  double t3[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k)
    for (int w = 0; w < (blockDim.x >> 5); ++w) t3[k] += smd[k][w];
  sc = t3[0], sb = t3[1], sd = t3[2];
  const float lse_c = mc + static_cast<float>(log(sc)), lse_b = mb + static_cast<float>(log(sb));
  if (threadIdx.x == 0 && value)
    value[r] = sd / sb - ((static_cast<double>(mb) - mc) + log(sb / sc));
  if (!dz) return;
  const float w = weight ? weight[r] : 1.f;
  T* out = dz + static_cast<int64_t>(r) * V;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    float v = 0.f;
    if (i != bos) v = w * (expf(lc[i] - lse_c) - expf(lb[i] - lse_b));
    out[i] = fromf<T>(v);
  }
}

// ------------------------------------------------------------------- KV plumbing

template <class T>
__global__ void kv_store_prompt_k(const T* qkv, const int32_t* start, int n_prompts, int pmax, int qd, int kvd,
                                  int nkv, int hd, T* ks, T* vs) {
  const int p = blockIdx.y;
  const int s0 = start[p], len = start[p + 1] - s0;
  const int qkvd = qd + 2 * kvd;
  const int64_t n = static_cast<int64_t>(len) * kvd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = static_cast<int>(i / kvd), c = static_cast<int>(i % kvd);
    const int h = c / hd, dd = c % hd;
    const int64_t src = static_cast<int64_t>(s0 + t) * qkvd + qd + c;
    const int64_t dst = ((static_cast<int64_t>(p) * nkv + h) * pmax + t) * hd + dd;
    ks[dst] = qkv[src];
    vs[dst] = qkv[src + kvd];
  }
}

template <class T>
__global__ void kv_append_k(const T* qkv, int rows, int qd, int kvd, int nkv, int hd, int slot, DecodeRows dr, T* ks,
                            T* vs) {
  pdl_wait();
  if (dr.step) slot = *dr.step - 1;
  const int qkvd = qd + 2 * kvd;
  const int64_t n = static_cast<int64_t>(rows) * kvd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / kvd), c = static_cast<int>(i % kvd);
    const int h = c / hd, dd = c % hd;
    const int64_t src = static_cast<int64_t>(r) * qkvd + qd + c;
    const int64_t dst = kv_slot_off(dr, dr_seq(dr, r), h, nkv, slot, hd) + dd;
    ks[dst] = qkv[src];
    vs[dst] = qkv[src + kvd];
  }
}

template <class T>
__global__ void pack_dqkv_k(const float* dq, const float* dkv, int rows, int qd, int kvd, T* out) {
  const int w = qd + 2 * kvd;
  const int64_t n = static_cast<int64_t>(rows) * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / w), c = static_cast<int>(i % w);
    const float v = c < qd ? dq[static_cast<int64_t>(r) * qd + c] : dkv[static_cast<int64_t>(r) * 2 * kvd + (c - qd)];
    out[i] = fromf<T>(v);
  }
}

// bf16 fast path: 8 columns per thread (two 16-byte fp32 loads, one 16-byte store), 2-D grid
// (row blocks x 8-column groups) so no per-element 64-bit division. qd, kvd multiples of 8.
__global__ void pack_dqkv8_k(const float* __restrict__ dq, const float* __restrict__ dkv, int rows, int qd, int kvd,
                             bf16* __restrict__ out) {
  const int w8 = (qd + 2 * kvd) / 8;
  const int c8 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c8 >= w8) return;
  const int c = c8 * 8;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    const float* src = c < qd ? dq + static_cast<int64_t>(r) * qd + c : dkv + static_cast<int64_t>(r) * 2 * kvd + (c - qd);
    const float4 a = __ldg(reinterpret_cast<const float4*>(src));
    const float4 b = __ldg(reinterpret_cast<const float4*>(src + 4));
    uint4 o;
    __nv_bfloat162 t;
    t = __floats2bfloat162_rn(a.x, a.y); o.x = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(a.z, a.w); o.y = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(b.x, b.y); o.z = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(b.z, b.w); o.w = *reinterpret_cast<uint32_t*>(&t);
    *reinterpret_cast<uint4*>(out + static_cast<int64_t>(r) * (qd + 2 * kvd) + c) = o;
  }
}

template <class T>
__global__ void gather_rows_k(const T* src, int64_t ld, const int32_t* idx, int rows, int width, T* dst) {
  const int64_t n = static_cast<int64_t>(rows) * width;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / width), c = static_cast<int>(i % width);
    dst[i] = src[static_cast<int64_t>(idx[r]) * ld + c];
  }
}

__global__ void scatter_rows_k(const float* src, int rows, int width, const int32_t* idx, float* dst) {
  const int64_t n = static_cast<int64_t>(rows) * width;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / width), c = static_cast<int>(i % width);
    dst[static_cast<int64_t>(idx[r]) * width + c] = src[i];
  }
}

// ------------------------------------------------------------ advantage / filter

// One thread per group, sequential fp64 sums in index order: bit-identical to
// advantage.cpp (group_advantage :80-94, leave_one_out :96-112, normalize_std
// :114-133, filter :135-140) for any rewards, not just binary ones.
__global__ void advantage_k(const double* r, int n, int G, int kind, int normalize, double eps, double tau,
                            double* adv, uint8_t* kept) {
  const int gs = kind == 0 ? n : G;
  const int ngroups = n / gs;
  for (int grp = blockIdx.x * blockDim.x + threadIdx.x; grp < ngroups; grp += gridDim.x * blockDim.x) {
    const int s = grp * gs;
    double sum = 0.0;
    for (int i = s; i < s + gs; ++i) sum += r[i];
    if (kind == 3) {
      // given advantages (adv holds them already): normalize_std / filter only
    } else if (kind == 2) {
      const double den = static_cast<double>(gs - 1);
      for (int i = s; i < s + gs; ++i) adv[i] = r[i] - (sum - r[i]) / den;
    } else {
      const double mean = sum / static_cast<double>(gs);
      for (int i = s; i < s + gs; ++i) adv[i] = r[i] - mean;
    }
    if (normalize) {
      double mean = 0.0;
      for (int i = s; i < s + gs; ++i) mean += r[i];
      mean /= static_cast<double>(gs);
      double var = 0.0;
      for (int i = s; i < s + gs; ++i) {
        const double dv = __dsub_rn(r[i], mean);
        var = __dadd_rn(var, __dmul_rn(dv, dv));  // no FMA contraction: bit-equal to the reference
      }
      var /= static_cast<double>(gs);
      const double den = sqrt(var) + eps;
      for (int i = s; i < s + gs; ++i) adv[i] = adv[i] / den;
    }
    for (int i = s; i < s + gs; ++i) kept[i] = fabs(adv[i]) > tau ? 1 : 0;
  }
}

// Single-block ballot + prefix-sum stream compaction: ascending kept indices.
__global__ void __launch_bounds__(1024) compact_k(const uint8_t* kept, int n, int32_t* idx, int32_t* n_kept) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = 0; c < n; c += 1024) {
    const int i = c + threadIdx.x;
    const bool k = i < n && kept[i];
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    if (lane == 0) warp_tot[w] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int j = 0; j < w; ++j) off += warp_tot[j];
    if (k) idx[base + off + __popc(bal & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int j = 0; j < 32; ++j) t += warp_tot[j];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_kept = base;
}

}  // namespace

// ------------------------------------------------------------------- wrappers

void init_normal_ctr(cudaStream_t s, float* w, int64_t n, double scale, uint64_t seed) {
  init_normal_ctr_k<<<grid1d(n), 256, 0, s>>>(w, n, scale, splitmix64(seed ^ 0x5DEECE66Dull));
  DCU_LAUNCHED();
}
void f64_to_f32(cudaStream_t s, const double* in, float* out, int64_t n) {
  f64_to_f32_k<<<grid1d(n), 256, 0, s>>>(in, out, n);
  DCU_LAUNCHED();
}
void f32_to_f64(cudaStream_t s, const float* in, double* out, int64_t n) {
  f32_to_f64_k<<<grid1d(n), 256, 0, s>>>(in, out, n);
  DCU_LAUNCHED();
}
void cast_f32_bf16(cudaStream_t s, const float* in, bf16* out, int64_t n) {
  if (n % 8 == 0 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    cast_bf16_v8_k<<<grid1d(n / 8), 256, 0, s>>>(reinterpret_cast<const float4*>(in), reinterpret_cast<uint4*>(out),
                                                  n / 8);
  } else {
    cast_bf16_k<<<grid1d(n), 256, 0, s>>>(in, out, n);
  }
  DCU_LAUNCHED();
}
void fill_f32(cudaStream_t s, float* p, float v, int64_t n) {
  if (n <= 0) return;
  fill_k<<<grid1d(n), 256, 0, s>>>(p, v, n);
  DCU_LAUNCHED();
}
void optimizer_update(cudaStream_t s, int kind, float* w, const float* g, float* m, float* v, bf16* wT, int64_t n,
                      float lr, float b1, float b2, float eps, float c1, float c2) {
  ProfScope ps(PROF_OPTIMIZER, s, 0, 30.0 * static_cast<double>(n));
  optimizer_k<<<grid1d(n), 256, 0, s>>>(kind, w, g, m, v, wT, n, lr, b1, b2, eps, c1, c2);
  DCU_LAUNCHED();
}

template <class T>
void embed_fwd(cudaStream_t s, const T* E, const T* P, const int32_t* tok, const int32_t* pos, int rows, int d,
               float* x32, T* xT) {
  if (rows <= 0) return;
  embed_fwd_k<T><<<grid1d(static_cast<int64_t>(rows) * d), 256, 0, s>>>(E, P, tok, pos, rows, d, x32, xT);
  DCU_LAUNCHED();
}
template <class T>
void embed_decode(cudaStream_t s, const T* E, const T* P, const int32_t* tok, const int32_t* plen, int step,
                  int rows, int d, float* x32, T* xT, const int32_t* row_seq, const int* step_dev) {
  launch_pdl(embed_decode_k<T>, dim3(grid1d(static_cast<int64_t>(rows) * d)), dim3(256), 0, s, E, P, tok, plen, step,
             rows, d, x32, xT, row_seq, step_dev);
  DCU_LAUNCHED();
}
size_t embed_bwd_tmp_bytes(int rows) {
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), rows);
  return 4 * sizeof(int32_t) * static_cast<size_t>(rows) + (cub_bytes + 255) / 256 * 256 + 256;
}
size_t embed_bwd_part_floats(int rows, int d) { return static_cast<size_t>(rows) * d; }

void embed_bwd(cudaStream_t s, const float* dx, const int32_t* tok, const int32_t* pos, int rows, int d, int n_tok,
               int n_pos, float* gt, float* gp, void* tmp, float* part) {
  if (rows <= 0) return;
  int32_t* keys = static_cast<int32_t*>(tmp);
  int32_t* vals = keys + rows;
  int32_t* skeys = vals + rows;
  int32_t* svals = skeys + rows;
  void* cub_tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(svals + rows) + 255) & ~uintptr_t(255));
  const int bits_needed[2] = {32 - __builtin_clz(static_cast<unsigned>(std::max(n_tok, 2) - 1)),
                              32 - __builtin_clz(static_cast<unsigned>(std::max(n_pos, 2) - 1))};
  const int32_t* ids[2] = {tok, pos};
  float* grads[2] = {gt, gp};
  const int bs = d >= 1024 ? 256 : 128;
  for (int w = 0; w < 2; ++w) {
    embed_seg_mark_k<<<cdiv(rows, 256), 256, 0, s>>>(ids[w], rows, keys, vals);
    DCU_LAUNCHED();
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, keys, skeys, vals, svals, rows, 0, bits_needed[w], s);
    DCU_CHECK(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys, skeys, vals, svals, rows, 0, bits_needed[w],
                                              s));
    embed_win_k<<<dim3(cdiv(rows, kEmbWin), cdiv(d, 4 * 128)), 128, 0, s>>>(dx, skeys, svals, rows, d, part);
    DCU_LAUNCHED();
    embed_run_k<<<rows, bs, 0, s>>>(part, skeys, rows, d, grads[w]);
    DCU_LAUNCHED();
  }
}
namespace {
// nseg <= want, and want is non-decreasing in M (so a buffer sized for M covers any M' <= M)
template <class T>
void colsum_geom(int M, int N, int* gx, int* nseg, int* seg_rows, int* want_out = nullptr) {
  constexpr int VEC = 16 / sizeof(T);
  *gx = cdiv(cdiv(N, VEC), 256);
  int want = std::max(1, (kNumSMs * 8) / *gx);  // ~8 blocks per SM
  want = std::min(want, std::max(1, M / 16));   // at least 16 rows per segment
  *seg_rows = cdiv(M, want);
  *nseg = cdiv(M, *seg_rows);
  if (want_out) *want_out = want;
}
}  // namespace

template <class T>
size_t colsum_tmp_floats(int M, int N) {
  int gx, nseg, seg_rows, want;
  colsum_geom<T>(M, N, &gx, &nseg, &seg_rows, &want);
  return static_cast<size_t>(want) * N;
}

template <class T>
void colsum_acc(cudaStream_t s, const T* X, int64_t ld, int M, int N, float* out, float* tmp) {
  if (M <= 0 || N <= 0) return;
  constexpr int VEC = 16 / sizeof(T);
  int gx, nseg, seg_rows;
  colsum_geom<T>(M, N, &gx, &nseg, &seg_rows);
  const bool vec = ((reinterpret_cast<uintptr_t>(X) | static_cast<uintptr_t>(ld * sizeof(T))) & 15) == 0;
  colsum_part_k<T, VEC><<<dim3(gx, nseg), 256, 0, s>>>(X, ld, M, N, seg_rows, vec, tmp);
  DCU_LAUNCHED();
  colsum_fin_k<<<cdiv(N, 32), dim3(32, 32), 0, s>>>(tmp, nseg, N, out);
  DCU_LAUNCHED();
}
void colsum_acc_f32(cudaStream_t s, const float* X, int64_t ld, int M, int N, float* out, float* tmp) {
  colsum_acc<float>(s, X, ld, M, N, out, tmp);
}

void sample_rows(cudaStream_t s, const float* logits, int rows, int V, int bos, int eos, float inv_t,
                 const uint64_t* keys, int step, const int32_t* cap, uint8_t* finished, int32_t* comp, float* logp,
                 int32_t* len, int32_t* tok_next, int max_len, float* part, const int32_t* row_seq) {
  const int ns = (V + kSlice - 1) / kSlice;
  {
    ProfScope ps(PROF_SAMPLE, s, 0, 4.0 * rows * static_cast<double>(V));
    sample_partials_k<<<grid1d(static_cast<int64_t>(rows) * ns), 256, 0, s>>>(logits, rows, V, bos, inv_t, part, ns);
    DCU_LAUNCHED();
  }
  sample_scan(s, part, ns, logits, V, rows, V, bos, eos, inv_t, keys, step, cap, finished, comp, logp, len, tok_next,
              max_len, false, nullptr, row_seq);
}


void lse_reduce(cudaStream_t s, const float* part, int ntiles, int rows, float* lse, const bf16* Y, int d,
                const bf16* W, const float* bias, const int32_t* target, float* logp) {
  if (rows <= 0) return;
  lse_reduce_k<<<cdiv(rows, 8), 256, 0, s>>>(part, ntiles, rows, lse, Y, d, W, bias, target, logp);
  DCU_LAUNCHED();
}

void sample_scan(cudaStream_t s, const float* part, int nslices, const float* logits, int64_t logits_ld, int rows,
                 int V, int bos, int eos, float inv_t, const uint64_t* keys, int step, const int32_t* cap,
                 uint8_t* finished, int32_t* comp, float* logp, int32_t* len, int32_t* tok_next, int max_len,
                 bool compact, float* lse_out, const int32_t* row_seq, int phase, SliceSel* sel, const float* dump,
                 int64_t dump_ld, int* mismatches, const int* step_dev) {
  // phases 0 / 1 stage each row's records in shared memory (one bulk copy per row): one
  // warp per CTA, as many CTAs per SM as the row windows fit (5 at V = 151,936, T = 1)
  const size_t row_bytes = static_cast<size_t>(nslices) * (compact ? 8 : 16);
  if (phase != 2 && row_bytes > 200 * 1024) throw Error(1, "sample_scan: vocabulary too large for the staged walk");
  const int wpb = phase == 2 ? 8 : 1;
  const size_t smem = phase == 2 ? 0 : row_bytes;
  static size_t smem_set = 0;
  if (smem > 48 * 1024 && smem > smem_set) {
    DCU_CHECK(cudaFuncSetAttribute(sample_scan_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 16));
    smem_set = 200 * 1024 + 16;
  }
  launch_pdl(sample_scan_k, dim3(cdiv(rows, wpb)), dim3(32 * wpb), smem, s, part, nslices, logits, logits_ld, rows, V,
             bos, eos, inv_t, keys, step, cap, finished, comp, logp, len, tok_next, max_len, compact, lse_out, row_seq,
             phase, sel, dump, dump_ld, mismatches, step_dev);
  DCU_LAUNCHED();
}

// Micro-batch packing on the device (forward_for_loss, policy.cpp:350-358): CTA k writes
// sequence k's packed tokens (prompt, then completion[:-1]) and positions, and its loss
// rows (packed row of the token predicting completion j, the target id, the sampler-LSE cell
// s * max_len + j, the row weight). info[8k..]: s, m, len, token offset in the round / in
// its micro-batch, loss-row offset, prompt offset lo / hi (31 bits each).
__global__ void pack_batch_rows_k(const int32_t* __restrict__ info, const float* __restrict__ wq,
                                  const int32_t* __restrict__ ptok, const int32_t* __restrict__ comp, int max_len,
                                  int32_t* __restrict__ tok, int32_t* __restrict__ pos, int32_t* __restrict__ rows,
                                  int32_t* __restrict__ tgt, int32_t* __restrict__ lsei, float* __restrict__ w) {
  const int32_t* f = info + 8 * static_cast<int64_t>(blockIdx.x);
  const int s = f[0], m = f[1], len = f[2], tg = f[3], tl = f[4], rg = f[5];
  const int64_t po = static_cast<int64_t>(f[6]) | (static_cast<int64_t>(f[7]) << 31);
  const int32_t* cs = comp + static_cast<int64_t>(s) * max_len;
  const int n = m + len - 1;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    tok[tg + t] = t < m ? ptok[po + t] : cs[t - m];
    pos[tg + t] = t;
  }
  const float wk = wq[blockIdx.x];
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    rows[rg + j] = tl + m - 1 + j;
    tgt[rg + j] = cs[j];
    lsei[rg + j] = static_cast<int32_t>(static_cast<int64_t>(s) * max_len + j);
    w[rg + j] = wk;
  }
}
void pack_batch_rows(cudaStream_t s, int nseq, const int32_t* info, const float* wq, const int32_t* ptok,
                     const int32_t* comp, int max_len, int32_t* tok, int32_t* pos, int32_t* rows, int32_t* tgt,
                     int32_t* lsei, float* w) {
  if (nseq <= 0) return;
  pack_batch_rows_k<<<nseq, 256, 0, s>>>(info, wq, ptok, comp, max_len, tok, pos, rows, tgt, lsei, w);
  DCU_LAUNCHED();
}

__global__ void step_advance_k(int* step) {
  pdl_wait();
  *step += 1;
}
void step_advance(cudaStream_t s, int* step_dev) {
  launch_pdl(step_advance_k, dim3(1), dim3(1), 0, s, step_dev);
  DCU_LAUNCHED();
}

// PPO clipped-surrogate weights: one thread per sequence of the micro-batch.
// Sequence-level ratio rho = exp(sum_j logp_j - old_lp) with the per-token teacher-forced
// log-probs summed in row order in fp64 (the snapshot sums the same fp32 values in the same
// order, so at theta == theta_old rho is exactly 1). The gradient of
// min(rho A, clip(rho, 1-eps, 1+eps) A) is rho A grad log pi on the unclipped branch and 0
// where the clipped (constant) branch is the minimum: A > 0 and rho > 1+eps, or A < 0 and
// rho < 1-eps. Every loss row of the sequence gets the weight; stats[i] = {rho, clipped,
// surrogate term}.
__global__ void ppo_weights_k(const float* __restrict__ logp, const int32_t* __restrict__ row_start, int nseq,
                              const double* __restrict__ old_lp, const double* __restrict__ adv, double eps,
                              float* __restrict__ w, double* __restrict__ stats) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nseq) return;
  double sum = 0.0;
  for (int r = row_start[i]; r < row_start[i + 1]; ++r) sum += static_cast<double>(logp[r]);
  const double rho = exp(sum - old_lp[i]);
  const double a = adv[i];
  const bool clipped = (a > 0.0 && rho > 1.0 + eps) || (a < 0.0 && rho < 1.0 - eps);
  const double wi = clipped ? 0.0 : a * rho;
  const double clip_rho = fmin(fmax(rho, 1.0 - eps), 1.0 + eps);
  for (int r = row_start[i]; r < row_start[i + 1]; ++r) w[r] = static_cast<float>(wi);
  if (stats) {
    stats[3 * i] = rho;
    stats[3 * i + 1] = clipped ? 1.0 : 0.0;
    stats[3 * i + 2] = fmin(rho * a, clip_rho * a);
  }
}

void ppo_weights(cudaStream_t s, const float* logp, const int32_t* row_start, int nseq, const double* old_lp,
                 const double* adv, double eps, float* w, double* stats) {
  if (nseq <= 0) return;
  ppo_weights_k<<<cdiv(nseq, 128), 128, 0, s>>>(logp, row_start, nseq, old_lp, adv, eps, w, stats);
  DCU_LAUNCHED();
}

__global__ void gather_f32_k(const float* __restrict__ src, const int32_t* __restrict__ idx, int n,
                             float* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

void gather_f32(cudaStream_t s, const float* src, const int32_t* idx, int n, float* dst) {
  if (n <= 0) return;
  gather_f32_k<<<cdiv(n, 256), 256, 0, s>>>(src, idx, n, dst);
  DCU_LAUNCHED();
}

template <class T>
void lm_rows(cudaStream_t s, const float* logits, int rows, int V, int bos, const int32_t* target,
             const float* weight, float* logp, T* dz) {
  if (rows <= 0) return;
  ProfScope ps(PROF_LM_ROWS, s, 0, static_cast<double>(rows) * V * (4.0 + (dz ? sizeof(T) : 0)));
  lm_rows_k<T><<<rows, 256, 0, s>>>(logits, V, bos, target, weight, logp, dz);
  DCU_LAUNCHED();
}

template <class T>
void kl_rows(cudaStream_t s, const float* lc, const float* lb, int rows, int V, int bos, const float* weight,
             double* value, T* dz) {
  if (rows <= 0) return;
  ProfScope ps(PROF_LM_ROWS, s, 0, static_cast<double>(rows) * V * (8.0 + (dz ? sizeof(T) : 0)));
  kl_rows_k<T><<<rows, 256, 0, s>>>(lc, lb, V, bos, weight, value, dz);
  DCU_LAUNCHED();
}
template void kl_rows<float>(cudaStream_t, const float*, const float*, int, int, int, const float*, double*, float*);
template void kl_rows<bf16>(cudaStream_t, const float*, const float*, int, int, int, const float*, double*, bf16*);

template <class T>
void kv_store_prompt(cudaStream_t s, const T* qkv, const int32_t* start, int n_prompts, int pmax, int qd, int kvd,
                     int nkv, int hd, T* ks, T* vs) {
  kv_store_prompt_k<T><<<dim3(cdiv(static_cast<int64_t>(pmax) * kvd, 256), n_prompts), 256, 0, s>>>(
      qkv, start, n_prompts, pmax, qd, kvd, nkv, hd, ks, vs);
  DCU_LAUNCHED();
}
template <class T>
void kv_append(cudaStream_t s, const T* qkv, int rows, int qd, int kvd, int nkv, int hd, int slot,
               const DecodeRows& dr, T* ks, T* vs) {
  launch_pdl(kv_append_k<T>, dim3(grid1d(static_cast<int64_t>(rows) * kvd)), dim3(256), 0, s, qkv, rows, qd, kvd, nkv,
             hd, slot, dr, ks, vs);
  DCU_LAUNCHED();
}
template <class T>
void pack_dqkv(cudaStream_t s, const float* dq, const float* dkv, int rows, int qd, int kvd, T* out) {
  if constexpr (sizeof(T) == 2) {
    if (qd % 8 == 0 && kvd % 8 == 0) {
      const int w8 = (qd + 2 * kvd) / 8;
      dim3 grid(cdiv(w8, 128), std::min(rows, kNumSMs * 16));
      pack_dqkv8_k<<<grid, 128, 0, s>>>(dq, dkv, rows, qd, kvd, reinterpret_cast<bf16*>(out));
      DCU_LAUNCHED();
      return;
    }
  }
  pack_dqkv_k<T><<<grid1d(static_cast<int64_t>(rows) * (qd + 2 * kvd)), 256, 0, s>>>(dq, dkv, rows, qd, kvd, out);
  DCU_LAUNCHED();
}
template <class T>
void gather_rows(cudaStream_t s, const T* src, int64_t ld, const int32_t* idx, int rows, int width, T* dst) {
  if (rows <= 0) return;
  gather_rows_k<T><<<grid1d(static_cast<int64_t>(rows) * width), 256, 0, s>>>(src, ld, idx, rows, width, dst);
  DCU_LAUNCHED();
}
void scatter_rows_f32(cudaStream_t s, const float* src, int rows, int width, const int32_t* idx, float* dst) {
  if (rows <= 0) return;
  scatter_rows_k<<<grid1d(static_cast<int64_t>(rows) * width), 256, 0, s>>>(src, rows, width, idx, dst);
  DCU_LAUNCHED();
}

void advantage_filter(cudaStream_t s, const double* r, int n, int G, int kind, int normalize, double eps, double tau,
                      double* adv, uint8_t* kept, int32_t* kept_idx, int32_t* n_kept) {
  const int ngroups = kind == 0 ? 1 : n / G;
  advantage_k<<<cdiv(ngroups, 128), 128, 0, s>>>(r, n, G, kind, normalize, eps, tau, adv, kept);
  DCU_LAUNCHED();
  compact_k<<<1, 1024, 0, s>>>(kept, n, kept_idx, n_kept);
  DCU_LAUNCHED();
}

#define INST(T)                                                                                                   \
  template void embed_fwd<T>(cudaStream_t, const T*, const T*, const int32_t*, const int32_t*, int, int, float*, T*); \
  template void embed_decode<T>(cudaStream_t, const T*, const T*, const int32_t*, const int32_t*, int, int, int,     \
                                float*, T*, const int32_t*, const int*);                                          \
  template void colsum_acc<T>(cudaStream_t, const T*, int64_t, int, int, float*, float*);                        \
  template size_t colsum_tmp_floats<T>(int, int);                                                                 \
  template void lm_rows<T>(cudaStream_t, const float*, int, int, int, const int32_t*, const float*, float*, T*);  \
  template void kv_store_prompt<T>(cudaStream_t, const T*, const int32_t*, int, int, int, int, int, int, T*, T*); \
  template void kv_append<T>(cudaStream_t, const T*, int, int, int, int, int, int, const DecodeRows&, T*, T*);   \
  template void pack_dqkv<T>(cudaStream_t, const float*, const float*, int, int, int, T*);                        \
  template void gather_rows<T>(cudaStream_t, const T*, int64_t, const int32_t*, int, int, T*);
INST(float)
INST(bf16)
#undef INST

}  // namespace dashcu
