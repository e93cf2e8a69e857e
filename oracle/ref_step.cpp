// TEST / BASELINE INFRASTRUCTURE ONLY — never linked into the product.
//
// One DASH step driven through the UNMODIFIED reference library on all host
// cores: this is the "reference CPU path" that bench.py --impl reference and
// the cpu_baseline leg time. The composition follows SURVEY §3.3 / SPEC:461:
//   preemptive_sample  -> dash::sample per (m, g) with
//                         derive_seed(round, "sample", m, g)   (rng.hpp:29-35)
//   reward             -> synthetic Bernoulli or
//                         tasks::reward for the ADD task (tasks.cpp:155-175)
//   group_advantage    -> advantage.cpp:80-94, filter_by_threshold :135-140
//   pg accumulate      -> sum_kept (A_n / N) * grad_log_prob (policy.cpp:463, SPEC:284-292,
//                         ParamTensors::add_scaled tensors.cpp:109-115)
//   optimizer_step     -> SGD via add_scaled, or Adam over views()
// Work is split over a thread-per-trajectory work queue; the reference
// functions are pure on an immutable snapshot.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <thread>
#include <vector>

#include "dash/advantage.hpp"
#include "dash/policy.hpp"
#include "dash/rng.hpp"
#include "dash/tasks.hpp"
#include "dash/tensors.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class F>
void parallel_for(int n, int threads, F&& f) {
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  const int t = threads < 1 ? 1 : threads;
  for (int w = 0; w < t; ++w)
    pool.emplace_back([&, w] {
      for (;;) {
        const int i = next.fetch_add(1);
        if (i >= n) break;
        f(i, w);
      }
    });
  for (auto& th : pool) th.join();
}

double u01(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

}  // namespace

struct RefStepStats {
  double sample_s, reward_adv_s, grad_s, update_s, total_s;
  int64_t tokens_sampled;
  int32_t kept;
  int32_t n_seq;
  double mean_reward;
};

// arch: int32[7]. params: flat views() order, updated in place.
// prompts: concatenated token ids, prompt_offsets[n_prompts+1].
// reward_mode 0: synthetic Bernoulli(p_m) keyed by reward_seed,
//             1: ADD-task reward with instance seed instance_seeds[m] (difficulty 2).
// opt 0 SGD ascent, 1 Adam ascent (m, v buffers of num_params, *adam_t in/out).
REF_API int ref_dash_step(const int32_t* arch_i, double* params, const int32_t* prompts,
                          const int64_t* prompt_offsets, int n_prompts, int G, int max_len,
                          double temperature, uint64_t round_seed, int64_t prompt_index_base,
                          int reward_mode, uint64_t reward_seed, const uint64_t* instance_seeds,
                          double tau, int opt, double lr, double* adam_m, double* adam_v,
                          int64_t* adam_t, int n_threads, RefStepStats* st) {
  dash::ArchConfig a;
  a.vocab_size = arch_i[0];
  a.embed_dim = arch_i[1];
  a.context_len = arch_i[2];
  a.ffn_hidden = arch_i[3];
  a.n_layers = arch_i[4];
  a.bos_id = arch_i[5];
  a.eos_id = arch_i[6];
  try {
    const double t0 = now_s();
    dash::PolicyParams p = dash::PolicyParams::zeros(a);
    {
      std::size_t off = 0;
      for (auto& t : p.views()) {
        std::memcpy(t.data, params + off, t.size * sizeof(double));
        off += t.size;
      }
    }
    const int n = n_prompts * G;
    std::vector<dash::Trajectory> trajs(n);
    parallel_for(n, n_threads, [&](int i, int) {
      const int m = i / G, g = i % G;
      std::vector<int> prompt(prompts + prompt_offsets[m], prompts + prompt_offsets[m + 1]);
      const uint64_t gm = static_cast<uint64_t>(prompt_index_base + m);
      trajs[i] = dash::sample(p, prompt, max_len, temperature,
                              dash::derive_seed(round_seed, "sample", gm, static_cast<uint64_t>(g)));
    });
    const double t1 = now_s();
    std::vector<double> r(n);
    int64_t tokens = 0;
    for (int i = 0; i < n; ++i) {
      const int m = i / G, g = i % G;
      const uint64_t gm = static_cast<uint64_t>(prompt_index_base + m);
      tokens += trajs[i].generation_length();
      if (reward_mode == 0) {
        const double pm = u01(dash::derive_seed(reward_seed, "reward_p", gm, 0));
        r[i] = u01(dash::derive_seed(reward_seed, "reward", gm, static_cast<uint64_t>(g))) < pm ? 1.0 : 0.0;
      } else {
        std::vector<std::string> toks{"<s>", "</s>"};
        for (int b = 2; b < 256; ++b) toks.emplace_back(1, static_cast<char>(b));
        dash::TaskSpec task{dash::TaskKind::Add, 2,
                            dash::Vocab::from_tokens(std::move(toks), "<s>", "</s>", "#")};
        auto inst = dash::generate_instance(task, instance_seeds[m]);
        r[i] = dash::reward(task, inst, trajs[i]).r;
      }
    }
    // tau = -inf: no filter_by_threshold call (GRPO-style arm), group_advantage keeps all
    auto adv = dash::group_advantage(r, dash::GroupIndex::contiguous(n, G));
    if (!(std::isinf(tau) && tau < 0)) adv = dash::filter_by_threshold(adv, tau);
    std::vector<int> kept_idx;
    for (int i = 0; i < n; ++i)
      if (adv.kept[i]) kept_idx.push_back(i);
    const double t2 = now_s();

    // One accumulator guarded by a mutex: per-thread accumulators would need
    // threads x num_params doubles (67 GB at the 0.5B shape on 16 threads).
    const int nt = n_threads < 1 ? 1 : n_threads;
    std::vector<dash::GradientVector> acc(1, dash::GradientVector::zeros(a));
    std::mutex acc_mu;
    parallel_for(static_cast<int>(kept_idx.size()), nt, [&](int k, int) {
      const int i = kept_idx[k];
      dash::GradientVector gi = dash::grad_log_prob(p, trajs[i]);
      std::lock_guard<std::mutex> lk(acc_mu);
      acc[0].add_scaled(gi, adv.advantages[i] / static_cast<double>(n));
    });
    const double t3 = now_s();

    if (opt == 0) {
      p.add_scaled(acc[0], lr);
    } else {
      const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
      const int64_t t = ++(*adam_t);
      const double c1 = 1.0 - std::pow(b1, static_cast<double>(t));
      const double c2 = 1.0 - std::pow(b2, static_cast<double>(t));
      auto pv = p.views();
      auto gv = acc[0].views();
      std::vector<std::size_t> base(pv.size(), 0);
      for (std::size_t ti = 1; ti < pv.size(); ++ti) base[ti] = base[ti - 1] + pv[ti - 1].size;
      // elementwise, so chunked over threads (the reference has no optimizer code)
      constexpr std::size_t kChunk = 1 << 20;
      std::vector<std::pair<std::size_t, std::size_t>> work;  // (tensor, start)
      for (std::size_t ti = 0; ti < pv.size(); ++ti)
        for (std::size_t j = 0; j < pv[ti].size; j += kChunk) work.emplace_back(ti, j);
      parallel_for(static_cast<int>(work.size()), nt, [&](int w, int) {
        const std::size_t ti = work[w].first, j0 = work[w].second;
        const std::size_t j1 = std::min(pv[ti].size, j0 + kChunk);
        for (std::size_t j = j0; j < j1; ++j) {
          const std::size_t off = base[ti] + j;
          const double g = gv[ti].data[j];
          adam_m[off] = b1 * adam_m[off] + (1.0 - b1) * g;
          adam_v[off] = b2 * adam_v[off] + (1.0 - b2) * g * g;
          pv[ti].data[j] += lr * (adam_m[off] / c1) / (std::sqrt(adam_v[off] / c2) + eps);
        }
      });
    }
    {
      std::size_t off = 0;
      for (const auto& t : p.views()) {
        std::memcpy(params + off, t.data, t.size * sizeof(double));
        off += t.size;
      }
    }
    const double t4 = now_s();
    double rs = 0.0;
    for (double v : r) rs += v;
    st->sample_s = t1 - t0;
    st->reward_adv_s = t2 - t1;
    st->grad_s = t3 - t2;
    st->update_s = t4 - t3;
    st->total_s = t4 - t0;
    st->tokens_sampled = tokens;
    st->kept = static_cast<int32_t>(kept_idx.size());
    st->n_seq = n;
    st->mean_reward = rs / n;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}
