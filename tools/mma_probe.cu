// tcgen05.mma issue-rate probe: one CTA issues NMMA kind::f16 MMAs (M = 128, N, K = 16,
// both operands in shared memory) into NACC accumulators round-robin, then commits and
// waits; prints cycles per MMA. Separates the per-instruction throughput floor from the
// latency of a chain of dependent accumulations into one accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe tools/mma_probe.cu
#include <cstdio>

#include "../paper_2505_17218_b200/csrc/tc5.cuh"

using namespace dashcu;

// MODE 0: back-to-back MMAs; 1: + tcgen05.commit to a second barrier every 4 MMAs;
// 2: + a wait on an already-completed barrier every 4 MMAs (the GEMM's per-k-block
// full-wait / fence / commit sequence); 3: fresh operands per k-block (walks a 160 KB
// region of 4 KB A + BN x 128 B B blocks instead of re-reading one k-block)
template <int N, int NACC, int MODE = 0>
__global__ void probe(int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2, done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                             (static_cast<uint32_t>(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    if (MODE == 2) mbar_arrive(&done);  // phase 0 complete
    long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const int k = i & 3;
      if (MODE == 2 && k == 0) {
        mbar_wait(&done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const uint32_t blk = MODE == 3 ? static_cast<uint32_t>((i >> 2) % 16) * (4096 + N * 128) : 0u;
      const uint32_t a0 = MODE == 3 ? sa + blk : sa, b0 = MODE == 3 ? sa + blk + 4096 : sb;
      const uint64_t da = smem_desc(a0 + k * 32, 16, 1024), db = smem_desc(b0 + k * 32, 16, 1024);
      umma_bf16(tmem + (i % NACC) * N, da, db, IDESC, i >= NACC ? 1u : 0u);
      if (MODE >= 1 && k == 3) umma_commit(&bar2);
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int NACC, int MODE = 0>
void run(long long* d) {
  static_assert(N * NACC <= 512, "TMEM columns");
  auto k = probe<N, NACC, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long h[2];
  for (int nmma : {64, 1024}) {
    k<<<1, 128, 200 * 1024>>>(nmma, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    k<<<1, 128, 200 * 1024>>>(nmma, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d N=%3d acc=%d mma=%5d  issue %7.1f cyc/mma  complete %7.1f cyc/mma\n", MODE, N, NACC, nmma,
           double(h[0]) / nmma, double(h[1]) / nmma);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<16, 1>(d);
  run<32, 1>(d);
  run<32, 2>(d);
  run<32, 4>(d);
  run<64, 1>(d);
  run<64, 4>(d);
  run<128, 1>(d);
  run<128, 2>(d);
  run<256, 1>(d);
  run<256, 2>(d);
  run<32, 1, 1>(d);
  run<32, 1, 2>(d);
  run<64, 1, 2>(d);
  run<256, 1, 2>(d);
  run<32, 1, 3>(d);
  run<64, 1, 3>(d);
  run<128, 1, 3>(d);
  run<256, 1, 3>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
