// dash_b200.hpp — reference-facing C++ API of the B200 DASH step.
//
// Compiles against the reference's own headers (proj/include/dash/*.hpp) and
// forwards to the C ABI in dashcu.h. The per-trajectory functions keep the exact
// signatures of proj/include/dash/policy.hpp / advantage.hpp, in namespace
// dash::b200, so a trainer switches a call site by qualifying it (or with
// `namespace dash { using namespace b200; }` in a translation unit that does not
// link policy.cpp). The batch functions are the SPEC-level entry points the
// reference specifies but never implemented.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "dash/advantage.hpp"
#include "dash/policy.hpp"
#include "dash/tensors.hpp"
#include "dash/trajectory.hpp"

namespace dash::b200 {

// Device and precision of the process-wide B200 context (default: device 0, bf16).
void configure(int device, bool fp32_parity_mode);

// ---- policy.hpp:24-51 (hot-path subset) ----
LogProbResult log_prob(const PolicyParams& params, const Trajectory& traj);        // policy.cpp:362-377
Trajectory sample(const PolicyParams& params, const std::vector<int>& prompt,     // policy.cpp:379-429
                  int max_len, double temperature, std::uint64_t seed);
GradientVector grad_log_prob(const PolicyParams& params, const Trajectory& traj);  // policy.cpp:463-485
KlResult kl_term(const PolicyParams& params, const PolicyParams& base,            // policy.cpp:487-522
                 const Trajectory& traj);

// ---- advantage.hpp:36-50 ----
AdvantageBatch single_path_advantage(const std::vector<double>& rewards);
AdvantageBatch group_advantage(const std::vector<double>& rewards, const GroupIndex& groups);
AdvantageBatch leave_one_out(const std::vector<double>& rewards, const GroupIndex& groups);
AdvantageBatch normalize_std(const AdvantageBatch& adv, const std::vector<double>& rewards,
                             const GroupIndex& groups, double eps);
AdvantageBatch filter_by_threshold(const AdvantageBatch& adv, double tau);

// ---- SPEC-level batch entry points ----
struct SamplingPlan {  // SPEC.md:368-371 (H = GPUs; one rank handles its own shard)
  int M = 0, G = 4, max_len = 0;
  double temperature = 1.0;
  std::uint64_t round_seed = 0;
  std::int64_t prompt_index_base = 0;
};
// preemptive_sample: M*G trajectories, group-contiguous.
std::vector<Trajectory> preemptive_sample(const SamplingPlan& plan, const PolicyParams& snapshot,
                                          const std::vector<std::vector<int>>& prompts);
// pg_gradient + run_schedule(DASH): mean over the round
// (1/N, N = batch size) of kept A_n * grad log pi, accumulated in micro-batches.
GradientVector pg_gradient(const std::vector<Trajectory>& batch, const AdvantageBatch& adv,
                           const PolicyParams& params, int micro_batch = 32);
struct OptState {
  bool adam = true;
  double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};
// optimizer_step: ascent on the device master weights, written back.
void optimizer_step(PolicyParams& params, const GradientVector& grad, OptState& st, double lr);
// Checkpoint container (dashcu_policy_save / _load: named f64 tensors in the
// views() order with the reference's content_hash).
void save_checkpoint(const PolicyParams& params, const std::string& path);
PolicyParams load_checkpoint(const ArchConfig& arch, const std::string& path);

}  // namespace dash::b200
