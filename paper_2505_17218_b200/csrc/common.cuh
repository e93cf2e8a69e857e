// Shared device/host helpers for libdashcu (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

namespace dashcu {

// Status-carrying exception used inside the library; converted to a status
// code at the C-ABI boundary (api.cu). Codes follow include/dashcu.h.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw Error(4, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what + " (" + file + ":" +
                     std::to_string(line) + ")");
}

#define DCU_CHECK(x)                                          \
  do {                                                        \
    cudaError_t e__ = (x);                                    \
    if (e__ != cudaSuccess) throw_cuda(e__, #x, __FILE__, __LINE__); \
  } while (0)

// Every kernel launch in the library goes through this counter so the bench
// can report how many of OUR kernels ran (gpu_launches).
extern int64_t g_launches;
#define DCU_LAUNCHED() \
  do {                 \
    ++::dashcu::g_launches; \
    DCU_CHECK(cudaGetLastError()); \
  } while (0)

// Programmatic dependent launch (PDL). Kernels launched with launch_pdl may start (on SMs
// the previous kernel has left) while it is still finishing: everything before pdl_wait()
// (barrier init, TMEM allocation, tensor-map prefetch) overlaps the previous kernel's tail;
// pdl_wait() blocks until the previous grid has completed and its writes are visible, so
// it must precede every global read of upstream data and every global write. pdl_trigger()
// lets the next kernel be scheduled early (its CTAs still wait in its own pdl_wait()).
// On by default (KNOB_PDL; the kernels trigger at their end): same-box A/B at C2 shapes,
// sampling -1.0 %, accumulate -0.6 % (tools/ab_pdl.sh).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Kernel-variant knobs (test coverage of forced variants and same-box A/B runs). Read from
// the environment ONCE at library load and settable through dashcu_set_knob; the hot
// dispatch reads this array, never getenv.
enum Knob : int {
  KNOB_GEMM_PAIR = 0,    // 0 tile model, 1 force 256x256 pair, 2 force 256x128 pair, 3 force 256x224, -1 never
  KNOB_GEMM_RASTER,      // -1 model, 0 M tiles fastest, 1 N tiles fastest
  KNOB_NO_SPLITK,        // 1: no split-K (single-CTA and pair)
  KNOB_NO_TMA_STORE,     // 1: per-thread epilogue stores instead of bulk tensor stores
  KNOB_GEMM_RESID_DB,    // 0: no double-buffered residual prefetch in the pair epilogue
  KNOB_GEMM_RESID_DEEP,  // -1 model (K >= 2048), 0 / 1 force the 5-stage / 4-epilogue-warp ring
  KNOB_ATTN_FWD,         // 0 auto, 1 mma.sync kernel, 2 tcgen05 kernel even for one-tile sequences
  KNOB_ATTN_BWD,         // 0 auto, 1 mma.sync kernel
  KNOB_ATTN_BWD_CHUNK,   // sequences per CTA chunk in the tcgen05 backward (0: 2-D grid order)
  KNOB_LSE_RECOMPUTE,    // 1: the backward recomputes the LM-head LSE instead of reusing the sampler's
  KNOB_PDL,              // 1: programmatic dependent launch
  KNOB_DECODE_GRAPH,     // 0: no CUDA-graph replay of decode steps
  KNOB_DECODE_COMPACT,   // 0: finished sequences keep their decode rows until the round ends
  KNOB_GEMM_SKINNY_AR,   // 0: skinny GEMMs (M <= 128) stage full 128-row A boxes
  KNOB_GEMM_SKINNY_M64,  // 0: skinny GEMMs with <= 64 rows issue M = 128 MMAs (default: M = 64)
  KNOB_SPLITK_MAX,       // largest ordered split-K slice count the tile model may pick
  KNOB_COMM_WORLD1,      // 1: dashcu_ctx_init_comm creates a 1-rank NCCL communicator at world 1 (tests)
  KNOB_NUM
};
extern int g_knob[KNOB_NUM];
inline int knob(Knob k) { return g_knob[k]; }

inline bool pdl_enabled() { return knob(KNOB_PDL) == 1; }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  DCU_CHECK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// Kernel-class profiler: when a class is enabled, its launches are bracketed by
// CUDA events on the launching stream and charged with their ALGORITHMIC flops
// and bytes (not measured traffic), so bench.py can report achieved / roofline.
enum ProfClass : int {
  PROF_GEMM_TC = 0,
  PROF_GEMM_SIMT = 1,
  PROF_ATTN_DECODE = 2,
  PROF_ATTN_FWD = 3,
  PROF_ATTN_BWD = 4,
  PROF_SAMPLE = 5,
  PROF_LM_ROWS = 6,
  PROF_OPTIMIZER = 7,
  PROF_NUM = 8
};
extern const char* const kProfNames[PROF_NUM];
extern unsigned g_prof_mask;
extern int g_prof_period;              // >= 1: bracket one launch in g_prof_period per class
extern int64_t g_prof_seen[PROF_NUM];  // launches of each enabled class since the last reset
void prof_begin(int cls, cudaStream_t s, cudaEvent_t* ev);
void prof_end(int cls, cudaStream_t s, cudaEvent_t ev0, double flops, double bytes, const char* key);
// mask bit 31: also aggregate per launch key (kernel variant + shape), see dashcu_profile_keys
constexpr unsigned kProfKeysBit = 1u << 31;

struct ProfScope {
  int cls;
  cudaStream_t s;
  double flops, bytes;
  cudaEvent_t ev = nullptr;
  bool on;
  char key[96];
  ProfScope(int c, cudaStream_t st, double f, double b) : cls(c), s(st), flops(f), bytes(b) {
    // every launch of an enabled class is counted; one in g_prof_period is bracketed with
    // events (profile_read scales the sampled time / flops / bytes to the class totals)
    on = (g_prof_mask >> c) & 1u;
    if (on) on = (g_prof_seen[c]++ % g_prof_period) == 0;
    key[0] = 0;
    if (on) prof_begin(c, s, &ev);
  }
  bool keyed() const { return on && (g_prof_mask & kProfKeysBit); }
  ~ProfScope() {
    if (on) prof_end(cls, s, ev, flops, bytes, key[0] ? key : nullptr);
  }
};

typedef __nv_bfloat16 bf16;

template <class T>
struct Cvt;
template <>
struct Cvt<float> {
  static __device__ __forceinline__ float to_f(float x) { return x; }
  static __device__ __forceinline__ float from_f(float x) { return x; }
};
template <>
struct Cvt<bf16> {
  static __device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ bf16 from_f(float x) { return __float2bfloat16_rn(x); }
};

template <class T>
__device__ __forceinline__ float tof(T x) { return Cvt<T>::to_f(x); }
template <class T>
__device__ __forceinline__ T fromf(float x) { return Cvt<T>::from_f(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int cdiv(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

constexpr int kNumSMs = 148;

// SM count of the current device (host side, cached after the first query)
inline int num_sms_host() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
  }
  return n;
}

}  // namespace dashcu
