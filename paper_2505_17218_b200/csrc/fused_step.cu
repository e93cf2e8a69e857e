// Fused ZeRO-1 update over NVLink peer memory: one kernel per rank does the
// reduce-scatter of the fp32 gradient, the Adam / SGD update of the rank's slice and the
// all-gather of the updated fp32 master + bf16 working weights, instead of ncclReduceScatter
// + an update kernel + ncclAllGather (dashcu_sharded_step). Peer buffers come from CUDA IPC
// handles exchanged once per policy (policy.cu); see FusedStepArgs (kernels.cuh).
#include "kernels.cuh"

namespace dashcu {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// until every word[i] (i < n) has reached epoch; false on timeout (~4 s at 1.9 GHz)
__device__ bool wait_flags(const uint32_t* words, int n, uint32_t epoch) {
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i)
    while (static_cast<int32_t>(ld_acquire_sys(words + i) - epoch) < 0) {
      if (clock64() - t0 > 8000000000ll) return false;
      __nanosleep(256);
    }
  return true;
}

__global__ void __launch_bounds__(256) fused_step_k(FusedStepArgs a) {
  // entry: every block announces this rank's gradient is final (idempotent), then waits for
  // all ranks' announcements before reading their gradients
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < a.world; ++p) st_release_sys(a.flags[p] + a.rank, a.epoch);
    if (!wait_flags(a.flags[a.rank], a.world, a.epoch)) atomicExch(a.err, 1);
  }
  __syncthreads();
  // this rank's slice: gradient summed over ranks in rank order, update, write to every rank
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = a.off + i;
    float gs = a.g[0][k];
    for (int p = 1; p < a.world; ++p) gs += a.g[p][k];
    const float wi = opt_update(a.kind, a.w[a.rank][k], gs, a.m + i, a.v + i, a.lr, a.b1, a.b2, a.eps, a.c1, a.c2);
    const bf16 wb = __float2bfloat16_rn(wi);
    for (int p = 0; p < a.world; ++p) {
      a.w[p][k] = wi;
      if (a.wT[p]) a.wT[p][k] = wb;
    }
  }
  // exit: the last block of this rank announces completion to every rank and waits for all
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
      for (int p = 0; p < a.world; ++p) st_release_sys(a.flags[p] + a.world + a.rank, a.epoch);
      if (!wait_flags(a.flags[a.rank] + a.world, a.world, a.epoch)) atomicExch(a.err, 1);
      *a.done = 0;
      __threadfence_system();
    }
  }
}

}  // namespace

void fused_step(cudaStream_t s, const FusedStepArgs& a, int grid) {
  ProfScope ps(PROF_OPTIMIZER, s, 0, 30.0 * static_cast<double>(a.len));
  fused_step_k<<<grid, 256, 0, s>>>(a);
  DCU_LAUNCHED();
}

}  // namespace dashcu
