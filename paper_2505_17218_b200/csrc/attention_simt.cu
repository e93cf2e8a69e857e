// CUDA-core attention kernels (parity path; also the bf16 path until the
// tensor-core kernels take over). Causal single-position softmax attention of
// the reference (policy.cpp:105-129, scale 1/sqrt(head_dim)) generalised to GQA,
// its reverse pass (policy.cpp:292-322) and the decode form over the KV store.
#include <cfloat>

#include "kernels.cuh"

namespace dashcu {

namespace {

constexpr int kWarps = 8;

// grid (n_seq, nh); 8 warps; each warp owns query rows r = warp, warp+8, ...
// dynamic smem: kWarps * (max_len + hd) floats.
template <class T>
__global__ void __launch_bounds__(256) attn_fwd_k(const T* __restrict__ qkv, const int32_t* seq_start, int max_len,
                                                  int nh, int nkv, int hd, T* __restrict__ ctx, float* __restrict__ lse) {
  extern __shared__ float sm[];
  const int sq = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int qd = nh * hd, kvd = nkv * hd, qkvd = qd + 2 * kvd;
  const int kvh = h / (nh / nkv);
  float* sc = sm + warp * (max_len + hd);
  float* qs = sc + max_len;
  const float scale = rsqrtf(static_cast<float>(hd));
  for (int r = warp; r < n; r += kWarps) {
    const T* q = qkv + static_cast<int64_t>(s0 + r) * qkvd + h * hd;
    for (int i = lane; i < hd; i += 32) qs[i] = tof<T>(q[i]);
    __syncwarp();
    float mx = -FLT_MAX;
    for (int j = lane; j <= r; j += 32) {
      const T* k = qkv + static_cast<int64_t>(s0 + j) * qkvd + qd + kvh * hd;
      float a = 0.f;
      for (int i = 0; i < hd; ++i) a = fmaf(qs[i], tof<T>(k[i]), a);
      a *= scale;
      sc[j] = a;
      mx = fmaxf(mx, a);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j <= r; j += 32) {
      const float p = expf(sc[j] - mx);
      sc[j] = p;
      sum += p;
    }
    sum = warp_sum(sum);
    __syncwarp();
    const float inv = 1.f / sum;
    for (int i = lane; i < hd; i += 32) {
      float a = 0.f;
      for (int j = 0; j <= r; ++j) a = fmaf(sc[j], tof<T>(qkv[static_cast<int64_t>(s0 + j) * qkvd + qd + kvd + kvh * hd + i]), a);
      ctx[static_cast<int64_t>(s0 + r) * qd + h * hd + i] = fromf<T>(a * inv);
    }
    if (lane == 0) lse[static_cast<int64_t>(s0 + r) * nh + h] = mx + logf(sum);
    __syncwarp();
  }
}

// Reverse pass. dq32 [T x qd] written; dkv32 [T x 2kvd] accumulated with atomics
// (k part then v part), summing over the query heads of each KV group.
template <class T>
__global__ void __launch_bounds__(256) attn_bwd_k(const T* __restrict__ qkv, const T* __restrict__ dctx,
                                                  const float* __restrict__ lse, const int32_t* seq_start, int max_len,
                                                  int nh, int nkv, int hd, float* __restrict__ dq32,
                                                  float* __restrict__ dkv32) {
  extern __shared__ float sm[];
  const int sq = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = seq_start[sq], n = seq_start[sq + 1] - s0;
  const int qd = nh * hd, kvd = nkv * hd, qkvd = qd + 2 * kvd;
  const int kvh = h / (nh / nkv);
  float* P = sm + warp * (2 * max_len + 2 * hd);
  float* DS = P + max_len;
  float* qs = DS + max_len;
  float* dos = qs + hd;
  const float scale = rsqrtf(static_cast<float>(hd));
  for (int r = warp; r < n; r += kWarps) {
    const int64_t row = s0 + r;
    for (int i = lane; i < hd; i += 32) {
      qs[i] = tof<T>(qkv[row * qkvd + h * hd + i]);
      dos[i] = tof<T>(dctx[row * qd + h * hd + i]);
    }
    __syncwarp();
    const float L = lse[row * nh + h];
    float D = 0.f;
    for (int j = lane; j <= r; j += 32) {
      const T* k = qkv + static_cast<int64_t>(s0 + j) * qkvd + qd + kvh * hd;
      const T* v = k + kvd;
      float a = 0.f, da = 0.f;
      for (int i = 0; i < hd; ++i) {
        a = fmaf(qs[i], tof<T>(k[i]), a);
        da = fmaf(dos[i], tof<T>(v[i]), da);
      }
      const float p = expf(a * scale - L);
      P[j] = p;
      DS[j] = da;
      D += p * da;
    }
    D = warp_sum(D);
    __syncwarp();
    for (int j = lane; j <= r; j += 32) DS[j] = P[j] * (DS[j] - D) * scale;
    __syncwarp();
    for (int i = lane; i < hd; i += 32) {
      float a = 0.f;
      for (int j = 0; j <= r; ++j) a = fmaf(DS[j], tof<T>(qkv[static_cast<int64_t>(s0 + j) * qkvd + qd + kvh * hd + i]), a);
      dq32[row * qd + h * hd + i] = a;
    }
    for (int j = 0; j <= r; ++j) {
      const float ds = DS[j], p = P[j];
      float* dk = dkv32 + static_cast<int64_t>(s0 + j) * 2 * kvd + kvh * hd;
      float* dv = dk + kvd;
      for (int i = lane; i < hd; i += 32) {
        atomicAdd(&dk[i], ds * qs[i]);
        atomicAdd(&dv[i], p * dos[i]);
      }
    }
    __syncwarp();
  }
}

// Decode: one warp per (sequence, query head). Keys: the group's prompt KV
// (shared by its G sequences) then the sequence's own completion KV.
// dynamic smem: (pmax + max_len + hd) floats per warp; block = 1 warp.
template <class T>
__global__ void __launch_bounds__(32) attn_decode_k(const T* __restrict__ qkv, const T* __restrict__ kp,
                                                    const T* __restrict__ vp, const T* __restrict__ kc,
                                                    const T* __restrict__ vc, const int32_t* prompt_len, int G, int pmax,
                                                    int n_comp, int max_len, DecodeRows dr, int nh, int nkv, int hd,
                                                    T* __restrict__ ctx) {
  extern __shared__ float sm[];
  const int s = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;  // s: decode row
  const int qd = nh * hd, kvd = nkv * hd, qkvd = qd + 2 * kvd;
  const int kvh = h / (nh / nkv);
  const int sq = dr_seq(dr, s);
  if (dr.step) n_comp = *dr.step;
  const int p = sq / G, m = prompt_len[sq];
  const int nk = m + n_comp;
  float* sc = sm;
  float* qs = sm + pmax + max_len;
  const T* kpb = kp + (static_cast<int64_t>(p) * nkv + kvh) * pmax * hd;
  const T* vpb = vp + (static_cast<int64_t>(p) * nkv + kvh) * pmax * hd;
  for (int i = lane; i < hd; i += 32) qs[i] = tof<T>(qkv[static_cast<int64_t>(s) * qkvd + h * hd + i]);
  __syncwarp();
  const float scale = rsqrtf(static_cast<float>(hd));
  float mx = -FLT_MAX;
  for (int j = lane; j < nk; j += 32) {
    const T* k = j < m ? kpb + static_cast<int64_t>(j) * hd : kc + kv_slot_off(dr, sq, kvh, nkv, j - m, hd);
    float a = 0.f;
    for (int i = 0; i < hd; ++i) a = fmaf(qs[i], tof<T>(k[i]), a);
    a *= scale;
    sc[j] = a;
    mx = fmaxf(mx, a);
  }
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < nk; j += 32) {
    const float e = expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  __syncwarp();
  const float inv = 1.f / sum;
  for (int i = lane; i < hd; i += 32) {
    float a = 0.f;
    for (int j = 0; j < nk; ++j) {
      const T* v = j < m ? vpb + static_cast<int64_t>(j) * hd : vc + kv_slot_off(dr, sq, kvh, nkv, j - m, hd);
      a = fmaf(sc[j], tof<T>(v[i]), a);
    }
    ctx[static_cast<int64_t>(s) * qd + h * hd + i] = fromf<T>(a * inv);
  }
}

void set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) DCU_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

template <class T>
void attn_fwd_varlen(cudaStream_t s, const T* qkv, const int32_t* seq_start, int n_seq, int max_len, int nh, int nkv,
                     int hd, T* ctx, float* lse, double alg_flops) {
  if (n_seq <= 0) return;
  ProfScope ps(PROF_ATTN_FWD, s, alg_flops, 0);
  const size_t smem = sizeof(float) * kWarps * (max_len + hd);
  set_smem((const void*)attn_fwd_k<T>, smem);
  attn_fwd_k<T><<<dim3(n_seq, nh), 256, smem, s>>>(qkv, seq_start, max_len, nh, nkv, hd, ctx, lse);
  DCU_LAUNCHED();
}

template <class T>
void attn_bwd_varlen(cudaStream_t s, const T* qkv, const T* dctx, const float* lse, const int32_t* seq_start, int n_seq,
                     int max_len, int nh, int nkv, int hd, float* dq32, float* dkv32, double alg_flops) {
  if (n_seq <= 0) return;
  ProfScope ps(PROF_ATTN_BWD, s, alg_flops, 0);
  const size_t smem = sizeof(float) * kWarps * (2 * max_len + 2 * hd);
  set_smem((const void*)attn_bwd_k<T>, smem);
  attn_bwd_k<T><<<dim3(n_seq, nh), 256, smem, s>>>(qkv, dctx, lse, seq_start, max_len, nh, nkv, hd, dq32, dkv32);
  DCU_LAUNCHED();
}

template <class T>
void attn_decode(cudaStream_t s, const T* qkv, const T* kp, const T* vp, const T* kc, const T* vc,
                 const int32_t* prompt_len, int rows, int G, int pmax, int n_comp, int max_len, const DecodeRows& dr,
                 int nh, int nkv, int hd, T* ctx, double alg_bytes) {
  ProfScope ps(PROF_ATTN_DECODE, s, 0, alg_bytes);
  const size_t smem = sizeof(float) * (pmax + max_len + hd);
  set_smem((const void*)attn_decode_k<T>, smem);
  attn_decode_k<T><<<dim3(rows, nh), 32, smem, s>>>(qkv, kp, vp, kc, vc, prompt_len, G, pmax, n_comp, max_len, dr, nh,
                                                    nkv, hd, ctx);
  DCU_LAUNCHED();
}

#define INST(T)                                                                                                     \
  template void attn_fwd_varlen<T>(cudaStream_t, const T*, const int32_t*, int, int, int, int, int, T*, float*,     \
                                   double);                                                                         \
  template void attn_bwd_varlen<T>(cudaStream_t, const T*, const T*, const float*, const int32_t*, int, int, int, int, \
                                   int, float*, float*, double);                                                    \
  template void attn_decode<T>(cudaStream_t, const T*, const T*, const T*, const T*, const T*, const int32_t*, int, \
                               int, int, int, int, const DecodeRows&, int, int, int, T*, double);
INST(float)
INST(bf16)
#undef INST

}  // namespace dashcu
