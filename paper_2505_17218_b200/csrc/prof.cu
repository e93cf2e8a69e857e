// Kernel-class profiler (see common.cuh ProfScope) + its C-ABI readers.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dashcu.h"
#include "common.cuh"

namespace dashcu {

const char* const kProfNames[PROF_NUM] = {"gemm_tc",   "gemm_simt", "attn_decode", "attn_fwd",
                                          "attn_bwd",  "sample",    "lm_rows",     "optimizer"};
unsigned g_prof_mask = 0;
int g_prof_period = 1;
int64_t g_prof_seen[PROF_NUM] = {};

// ------------------------------------------------------------------- knobs
namespace {
struct KnobDef {
  const char* name;
  int def;
};
// env name = "DASHCU_" + name
const KnobDef kKnobs[KNOB_NUM] = {
    {"GEMM_PAIR", 0},       {"GEMM_RASTER", -1},    {"NO_SPLITK", 0},  {"NO_TMA_STORE", 0},
    {"GEMM_RESID_DB", 1},   {"GEMM_RESID_DEEP", -1}, {"ATTN_FWD", 0},  {"ATTN_BWD", 0},
    {"ATTN_BWD_CHUNK", 4},  {"LSE_RECOMPUTE", 0},   {"PDL", 1},        {"DECODE_GRAPH", 1},
    {"DECODE_COMPACT", 1},  {"GEMM_SKINNY_AR", 1},  {"GEMM_SKINNY_M64", 1},
    {"SPLITK_MAX", 4},      {"COMM_WORLD1", 0},
};
int knob_index(const char* name) {
  if (!name) return -1;
  if (!strncmp(name, "DASHCU_", 7)) name += 7;
  for (int i = 0; i < KNOB_NUM; ++i)
    if (!strcmp(name, kKnobs[i].name)) return i;
  return -1;
}
// string values of the old environment knobs ("mma", "tc5")
int knob_value(int i, const char* v) {
  if (i == KNOB_ATTN_FWD || i == KNOB_ATTN_BWD) {
    if (!strcmp(v, "mma")) return 1;
    if (!strcmp(v, "tc5")) return 2;
  }
  return atoi(v);
}
}  // namespace

int g_knob[KNOB_NUM] = {};
namespace {
struct KnobInit {
  KnobInit() {
    for (int i = 0; i < KNOB_NUM; ++i) {
      g_knob[i] = kKnobs[i].def;
      const std::string env = std::string("DASHCU_") + kKnobs[i].name;
      if (const char* v = getenv(env.c_str())) g_knob[i] = knob_value(i, v);
    }
  }
} g_knob_init;
}  // namespace

namespace {

struct Pending {
  int cls;
  cudaEvent_t a, b;
  double flops, bytes;
  std::string key;
};

struct Agg {
  double ms = 0, flops = 0, bytes = 0;
  int64_t launches = 0;
};

struct Prof {
  std::mutex mu;
  std::vector<cudaEvent_t> pool;
  std::vector<Pending> pending;
  double ms[PROF_NUM] = {};
  double flops[PROF_NUM] = {};
  double bytes[PROF_NUM] = {};
  int64_t launches[PROF_NUM] = {};
  std::map<std::string, Agg> keys;

  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    DCU_CHECK(cudaEventCreate(&e));
    return e;
  }
  void drain() {
    for (auto& p : pending) {
      DCU_CHECK(cudaEventSynchronize(p.b));
      float t = 0.f;
      DCU_CHECK(cudaEventElapsedTime(&t, p.a, p.b));
      ms[p.cls] += t;
      flops[p.cls] += p.flops;
      bytes[p.cls] += p.bytes;
      launches[p.cls] += 1;
      if (!p.key.empty()) {
        Agg& a = keys[p.key];
        a.ms += t;
        a.flops += p.flops;
        a.bytes += p.bytes;
        a.launches += 1;
      }
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
};

Prof& prof() {
  static Prof p;
  return p;
}

}  // namespace

void prof_begin(int, cudaStream_t s, cudaEvent_t* ev) {
  Prof& p = prof();
  std::lock_guard<std::mutex> lk(p.mu);
  *ev = p.get();
  DCU_CHECK(cudaEventRecord(*ev, s));
}

void prof_end(int cls, cudaStream_t s, cudaEvent_t ev0, double flops, double bytes, const char* key) {
  Prof& p = prof();
  std::lock_guard<std::mutex> lk(p.mu);
  cudaEvent_t e = p.get();
  DCU_CHECK(cudaEventRecord(e, s));
  p.pending.push_back({cls, ev0, e, flops, bytes, key ? std::string(kProfNames[cls]) + " " + key : std::string()});
  if (p.pending.size() > 65536) p.drain();
}

}  // namespace dashcu

extern "C" {

// Kernel-variant knobs (tests / A-B tools): name with or without the DASHCU_ prefix.
// value INT32_MIN restores the default. Returns the previous value, or INT32_MIN for an
// unknown name.
DASHCU_API int dashcu_set_knob(const char* name, int value) {
  using namespace dashcu;
  const int i = knob_index(name);
  if (i < 0) return INT32_MIN;
  const int old = g_knob[i];
  g_knob[i] = value == INT32_MIN ? kKnobs[i].def : value;
  return old;
}

DASHCU_API int dashcu_profile_sampling(int period) {
  std::lock_guard<std::mutex> lk(dashcu::prof().mu);
  dashcu::g_prof_period = period < 1 ? 1 : period;
  return 0;
}

DASHCU_API int dashcu_profile_enable(unsigned class_mask) {
  std::lock_guard<std::mutex> lk(dashcu::prof().mu);
  dashcu::g_prof_mask = class_mask;
  return 0;
}

DASHCU_API int dashcu_profile_read(dashcu_kprof* out, int max, int reset) {
  using namespace dashcu;
  try {
    Prof& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    p.drain();
    int n = 0;
    for (int c = 0; c < PROF_NUM && n < max; ++c, ++n) {
      // sampled launches scaled to the class totals (exact when the sampling period is 1)
      const int64_t total = std::max<int64_t>(g_prof_seen[c], p.launches[c]);
      const double f = p.launches[c] ? static_cast<double>(total) / p.launches[c] : 0.0;
      snprintf(out[n].name, sizeof(out[n].name), "%s", kProfNames[c]);
      out[n].launches = total;
      out[n].ms = p.ms[c] * f;
      out[n].flops = p.flops[c] * f;
      out[n].bytes = p.bytes[c] * f;
    }
    if (reset) {
      for (int c = 0; c < PROF_NUM; ++c) p.ms[c] = p.flops[c] = p.bytes[c] = 0, p.launches[c] = 0, g_prof_seen[c] = 0;
      p.keys.clear();
    }
    return n;
  } catch (...) {
    return -1;
  }
}

// One line per launch key: "<class> <key>\t<launches>\t<ms>\t<flops>\t<bytes>\n".
// Returns the bytes needed (excluding the NUL); writes at most cap-1 of them.
DASHCU_API int64_t dashcu_profile_keys(char* buf, int64_t cap) {
  using namespace dashcu;
  try {
    Prof& p = prof();
    std::lock_guard<std::mutex> lk(p.mu);
    p.drain();
    std::string out;
    char line[256];
    for (auto& kv : p.keys) {
      snprintf(line, sizeof(line), "%s\t%lld\t%.6f\t%.6e\t%.6e\n", kv.first.c_str(),
               static_cast<long long>(kv.second.launches), kv.second.ms, kv.second.flops, kv.second.bytes);
      out += line;
    }
    if (buf && cap > 0) {
      const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(out.size()));
      memcpy(buf, out.data(), n);
      buf[n] = 0;
    }
    return static_cast<int64_t>(out.size());
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
