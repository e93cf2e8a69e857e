// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library compiled in place from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load the resulting libdash_ref.so, and only as the checker / CPU baseline.
//
// Every entry point forwards to the reference function named beside it; the
// flat parameter buffers follow ParamTensors::views() order
// (reference proj/src/tensors.cpp:49-71).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "dash/advantage.hpp"
#include "dash/errors.hpp"
#include "dash/policy.hpp"
#include "dash/rng.hpp"
#include "dash/tasks.hpp"
#include "dash/tensors.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

// 0 ok, 1 InputError, 2 CapacityError, 3 OnPolicyViolation, 9 other
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const dash::InputError& e) {
    g_err = e.what();
    return 1;
  } catch (const dash::CapacityError& e) {
    g_err = e.what();
    return 2;
  } catch (const dash::OnPolicyViolation& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

dash::ArchConfig arch_of(const int32_t* a) {
  dash::ArchConfig c;
  c.vocab_size = a[0];
  c.embed_dim = a[1];
  c.context_len = a[2];
  c.ffn_hidden = a[3];
  c.n_layers = a[4];
  c.bos_id = a[5];
  c.eos_id = a[6];
  return c;
}

dash::PolicyParams params_of(const int32_t* a, const double* flat) {
  dash::PolicyParams p = dash::PolicyParams::zeros(arch_of(a));
  std::size_t off = 0;
  for (auto& t : p.views()) {
    std::memcpy(t.data, flat + off, t.size * sizeof(double));
    off += t.size;
  }
  return p;
}

void flatten(const dash::ParamTensors& p, double* out) {
  std::size_t off = 0;
  for (const auto& t : p.views()) {
    std::memcpy(out + off, t.data, t.size * sizeof(double));
    off += t.size;
  }
}

std::vector<int> ivec(const int32_t* p, int n) { return std::vector<int>(p, p + n); }

// Byte vocab of SURVEY App.B D7: id 0 "<s>", id 1 "</s>", id b = byte b for
// b in [2, 255]; delimiter "#".
dash::TaskSpec byte_add_task(int difficulty) {
  std::vector<std::string> toks{"<s>", "</s>"};
  for (int b = 2; b < 256; ++b) toks.emplace_back(1, static_cast<char>(b));
  dash::Vocab v = dash::Vocab::from_tokens(std::move(toks), "<s>", "</s>", "#");
  return dash::TaskSpec{dash::TaskKind::Add, difficulty, std::move(v)};
}

// TaskSpec of kind k (0 add, 1 mod, 2 reverse, 3 parity, 4 micro) over the task's own
// vocabulary (TaskSpec::make) or, vocab == 1, the byte vocabulary above.
dash::TaskSpec task_of(int kind, int difficulty, int vocab) {
  static const dash::TaskKind kinds[5] = {dash::TaskKind::Add, dash::TaskKind::Mod, dash::TaskKind::Reverse,
                                          dash::TaskKind::Parity, dash::TaskKind::Micro};
  if (kind < 0 || kind > 4) throw dash::InputError("unknown task kind");
  if (vocab == 0) return dash::TaskSpec::make(kinds[kind], difficulty);
  dash::TaskSpec t = byte_add_task(difficulty);
  t.kind = kinds[kind];
  return t;
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// arch = int32[7] {vocab, embed_dim, context_len, ffn_hidden, n_layers, bos, eos}
REF_API int ref_num_params(const int32_t* arch, int64_t* n) {
  return guarded([&] { *n = static_cast<int64_t>(dash::PolicyParams::zeros(arch_of(arch)).num_params()); });
}

// PolicyParams::init (tensors.cpp:150-158)
REF_API int ref_init_params(const int32_t* arch, double scale, uint64_t seed, double* out) {
  return guarded([&] { flatten(dash::PolicyParams::init(arch_of(arch), scale, seed), out); });
}

// ParamTensors::content_hash (tensors.cpp:95-107)
REF_API int ref_content_hash(const int32_t* arch, const double* flat, uint64_t* h) {
  return guarded([&] { *h = params_of(arch, flat).content_hash(); });
}

// sample (policy.cpp:379-429). out_completion/out_logp sized >= max_len.
REF_API int ref_sample(const int32_t* arch, const double* flat, const int32_t* prompt, int m,
                       int max_len, double temperature, uint64_t seed, int32_t* out_completion,
                       double* out_logp, int32_t* out_len) {
  return guarded([&] {
    auto p = params_of(arch, flat);
    dash::Trajectory t = dash::sample(p, ivec(prompt, m), max_len, temperature, seed);
    *out_len = t.generation_length();
    for (int i = 0; i < *out_len; ++i) {
      out_completion[i] = t.completion[i];
      out_logp[i] = t.log_probs[i];
    }
  });
}

// log_prob (policy.cpp:362-377)
REF_API int ref_log_prob(const int32_t* arch, const double* flat, const int32_t* prompt, int m,
                         const int32_t* completion, int len, double* per_token, double* total) {
  return guarded([&] {
    auto p = params_of(arch, flat);
    dash::Trajectory t;
    t.prompt = ivec(prompt, m);
    t.completion = ivec(completion, len);
    dash::LogProbResult r = dash::log_prob(p, t);
    for (int i = 0; i < len; ++i) per_token[i] = r.per_token[i];
    *total = r.total;
  });
}

// grad_log_prob (policy.cpp:463-485), flat gradient in views() order.
REF_API int ref_grad_log_prob(const int32_t* arch, const double* flat, const int32_t* prompt, int m,
                              const int32_t* completion, int len, double* grad_out) {
  return guarded([&] {
    auto p = params_of(arch, flat);
    dash::Trajectory t;
    t.prompt = ivec(prompt, m);
    t.completion = ivec(completion, len);
    flatten(dash::grad_log_prob(p, t), grad_out);
  });
}

// kl_term (policy.cpp:487-522): value and flat gradient in views() order.
REF_API int ref_kl_term(const int32_t* arch, const double* flat, const double* base_flat, const int32_t* prompt,
                        int m, const int32_t* completion, int len, double* value, double* grad_out) {
  return guarded([&] {
    auto p = params_of(arch, flat);
    auto b = params_of(arch, base_flat);
    dash::Trajectory t;
    t.prompt = ivec(prompt, m);
    t.completion = ivec(completion, len);
    auto r = dash::kl_term(p, b, t);
    *value = r.value;
    flatten(r.grad, grad_out);
  });
}

// next_token_probs (policy.cpp:524-537)
REF_API int ref_next_token_probs(const int32_t* arch, const double* flat, const int32_t* ctx, int n,
                                 double* probs) {
  return guarded([&] {
    auto p = params_of(arch, flat);
    auto v = dash::next_token_probs(p, ivec(ctx, n));
    std::memcpy(probs, v.data(), v.size() * sizeof(double));
  });
}

// greedy_decode (policy.cpp:431-461)
REF_API int ref_greedy_decode(const int32_t* arch, const double* flat, const int32_t* prompt, int m,
                              int max_len, int32_t* out, int32_t* out_len) {
  return guarded([&] {
    auto p = params_of(arch, flat);
    auto v = dash::greedy_decode(p, ivec(prompt, m), max_len);
    *out_len = static_cast<int32_t>(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  });
}

// ---- advantage.cpp -------------------------------------------------------
// kind: 0 single_path (:67-78), 1 group (:80-94), 2 leave_one_out (:96-112)
REF_API int ref_advantage(const double* rewards, int n, int group_size, int kind, double* out) {
  return guarded([&] {
    std::vector<double> r(rewards, rewards + n);
    dash::AdvantageBatch a;
    if (kind == 0) a = dash::single_path_advantage(r);
    else if (kind == 1) a = dash::group_advantage(r, dash::GroupIndex::contiguous(n, group_size));
    else a = dash::leave_one_out(r, dash::GroupIndex::contiguous(n, group_size));
    std::memcpy(out, a.advantages.data(), n * sizeof(double));
  });
}

// normalize_std (advantage.cpp:114-133)
REF_API int ref_normalize_std(const double* adv, const double* rewards, int n, int group_size,
                              double eps, double* out) {
  return guarded([&] {
    dash::AdvantageBatch a;
    a.advantages.assign(adv, adv + n);
    a.kept.assign(n, 1);
    std::vector<double> r(rewards, rewards + n);
    auto o = dash::normalize_std(a, r, dash::GroupIndex::contiguous(n, group_size), eps);
    std::memcpy(out, o.advantages.data(), n * sizeof(double));
  });
}

// filter_by_threshold (advantage.cpp:135-140) + kept_count/filtered_fraction/mean_abs_kept (:44-65)
REF_API int ref_filter_by_threshold(const double* adv, int n, double tau, uint8_t* kept,
                                    int32_t* kept_count, double* filtered_fraction,
                                    double* mean_abs_kept) {
  return guarded([&] {
    dash::AdvantageBatch a;
    a.advantages.assign(adv, adv + n);
    a.kept.assign(n, 1);
    auto o = dash::filter_by_threshold(a, tau);
    for (int i = 0; i < n; ++i) kept[i] = static_cast<uint8_t>(o.kept[i] != 0);
    *kept_count = o.kept_count();
    *filtered_fraction = o.filtered_fraction();
    *mean_abs_kept = o.mean_abs_kept();
  });
}

// ---- rng.hpp ---------------------------------------------------------------
REF_API uint64_t ref_splitmix64(uint64_t x) { return dash::splitmix64(x); }
REF_API uint64_t ref_fnv1a(const char* s) { return dash::fnv1a(s); }
REF_API uint64_t ref_derive_seed(uint64_t base, const char* tag, uint64_t a, uint64_t b) {
  return dash::derive_seed(base, tag, a, b);
}
// kind 0: next_u64, 1: uniform01 (as bits of double), 2: normal (as bits of double)
REF_API void ref_rng_draws(uint64_t seed, int kind, int n, uint64_t* out) {
  dash::Rng r(seed);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) {
      out[i] = r.next_u64();
    } else {
      double v = kind == 1 ? r.uniform01() : r.normal();
      std::memcpy(&out[i], &v, sizeof(double));
    }
  }
}

// ---- tasks.cpp (host-side prompt/reward source for config 1) ---------------
// generate_instance (tasks.cpp:105-153) for ADD over the byte vocab (D7).
REF_API int ref_add_instance(int difficulty, uint64_t seed, int32_t* prompt, int32_t* m,
                             char* answer, int answer_cap) {
  return guarded([&] {
    auto task = byte_add_task(difficulty);
    auto inst = dash::generate_instance(task, seed);
    *m = static_cast<int32_t>(inst.prompt.size());
    for (std::size_t i = 0; i < inst.prompt.size(); ++i) prompt[i] = inst.prompt[i];
    std::snprintf(answer, answer_cap, "%s", inst.answer.c_str());
  });
}

// reward (tasks.cpp:155-175) for the ADD/byte-vocab instance with `seed`.
REF_API int ref_add_reward(int difficulty, uint64_t seed, const int32_t* completion, int len,
                           double* r) {
  return guarded([&] {
    auto task = byte_add_task(difficulty);
    auto inst = dash::generate_instance(task, seed);
    dash::Trajectory t;
    t.prompt = inst.prompt;
    t.completion = ivec(completion, len);
    *r = dash::reward(task, inst, t).r;
  });
}

// generate_instance (tasks.cpp:105-153) for any task kind and either vocabulary.
REF_API int ref_task_instance(int kind, int difficulty, int vocab, uint64_t seed, int32_t* prompt, int32_t* m,
                              char* answer, int answer_cap) {
  return guarded([&] {
    auto task = task_of(kind, difficulty, vocab);
    auto inst = dash::generate_instance(task, seed);
    *m = static_cast<int32_t>(inst.prompt.size());
    for (std::size_t i = 0; i < inst.prompt.size(); ++i) prompt[i] = inst.prompt[i];
    std::snprintf(answer, answer_cap, "%s", inst.answer.c_str());
  });
}

// reward (tasks.cpp:155-175) for any task kind and either vocabulary.
REF_API int ref_task_reward(int kind, int difficulty, int vocab, uint64_t seed, const int32_t* completion, int len,
                            double* r) {
  return guarded([&] {
    auto task = task_of(kind, difficulty, vocab);
    auto inst = dash::generate_instance(task, seed);
    dash::Trajectory t;
    t.prompt = inst.prompt;
    t.completion = ivec(completion, len);
    *r = dash::reward(task, inst, t).r;
  });
}

// expert_trajectory (tasks.cpp:177-...) completion: always rewarded 1.
REF_API int ref_task_expert(int kind, int difficulty, int vocab, uint64_t seed, int stepwise, int32_t* completion,
                            int cap, int32_t* len) {
  return guarded([&] {
    auto task = task_of(kind, difficulty, vocab);
    auto inst = dash::generate_instance(task, seed);
    auto tr = dash::expert_trajectory(task, inst, stepwise ? dash::Verbosity::Stepwise : dash::Verbosity::Terse);
    if (static_cast<int>(tr.completion.size()) > cap) throw dash::CapacityError("completion buffer too small");
    *len = static_cast<int32_t>(tr.completion.size());
    for (std::size_t i = 0; i < tr.completion.size(); ++i) completion[i] = tr.completion[i];
  });
}
