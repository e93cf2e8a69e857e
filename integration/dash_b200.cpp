// Reference-facing C++ API (include/dash_b200.hpp) implemented over the C ABI.
//
// Built against the reference's headers (proj/include) — this is the code a
// maintainer adds to the reference build to route the DASH hot path to the B200
// (INTEGRATION.md). It owns one process-wide dashcu context + policy handle;
// PolicyParams are uploaded only when their content_hash (tensors.cpp:95-107)
// changes, so a round that samples, computes advantages and accumulates on one
// snapshot uploads the weights once.
#include "dash_b200.hpp"

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "dash/errors.hpp"
#include "dashcu.h"

namespace dash::b200 {
namespace {

struct State {
  std::mutex mu;
  int device = 0;
  int dtype = DASHCU_BF16;
  dashcu_ctx* ctx = nullptr;
  dashcu_policy* pol = nullptr;
  dashcu_policy* base = nullptr;  // kl_term's base policy
  std::uint64_t base_hash = 0;
  ArchConfig arch{};
  bool have_arch = false;
  std::uint64_t hash = 0;
  bool have_params = false;
};

State& S() {
  static State s;
  return s;
}

// status code -> the reference's exception classes (errors.hpp:10-23)
void check(int rc) {
  if (rc == DASHCU_OK) return;
  const std::string msg = std::string("dashcu: ") + dashcu_last_error();
  if (rc == DASHCU_E_INPUT) throw InputError(msg);
  if (rc == DASHCU_E_CAPACITY) throw CapacityError(msg);
  if (rc == DASHCU_E_ON_POLICY) throw OnPolicyViolation(msg);
  throw std::runtime_error(msg);
}

std::vector<double> flatten(const ParamTensors& p) {
  std::vector<double> out;
  out.reserve(p.num_params());
  for (const auto& t : p.views()) out.insert(out.end(), t.data, t.data + t.size);
  return out;
}

void unflatten(const std::vector<double>& flat, ParamTensors& p) {
  std::size_t off = 0;
  for (auto& t : p.views()) {
    std::memcpy(t.data, flat.data() + off, t.size * sizeof(double));
    off += t.size;
  }
}

dashcu_arch to_c(const ArchConfig& a) {
  dashcu_arch c{};
  c.vocab_size = a.vocab_size;
  c.embed_dim = a.embed_dim;
  c.context_len = a.context_len;
  c.ffn_hidden = a.ffn_hidden;
  c.n_layers = a.n_layers;
  c.bos_id = a.bos_id;
  c.eos_id = a.eos_id;
  return c;  // n_heads = n_kv_heads = head_dim = 0: the reference single-head geometry
}

// Make the device policy hold `params` (caller holds the lock).
dashcu_policy* bind(const PolicyParams& params) {
  State& s = S();
  if (!s.ctx) check(dashcu_ctx_create(s.device, &s.ctx));
  if (!s.pol || !s.have_arch || !(s.arch == params.arch)) {
    if (s.pol) dashcu_policy_destroy(s.pol);
    s.pol = nullptr;
    const dashcu_arch a = to_c(params.arch);
    check(dashcu_policy_create(s.ctx, &a, s.dtype, &s.pol));
    s.arch = params.arch;
    s.have_arch = true;
    s.have_params = false;
  }
  const std::uint64_t h = params.content_hash();
  if (!s.have_params || h != s.hash) {
    const auto flat = flatten(params);
    check(dashcu_policy_upload(s.pol, flat.data(), static_cast<std::int64_t>(flat.size())));
    s.hash = h;
    s.have_params = true;
  }
  return s.pol;
}

void load(dashcu_policy* pol, const std::vector<const Trajectory*>& ts) {
  std::vector<int32_t> ptok, ctok;
  std::vector<int64_t> poff{0}, coff{0};
  for (const Trajectory* t : ts) {
    ptok.insert(ptok.end(), t->prompt.begin(), t->prompt.end());
    poff.push_back(static_cast<int64_t>(ptok.size()));
    ctok.insert(ctok.end(), t->completion.begin(), t->completion.end());
    coff.push_back(static_cast<int64_t>(ctok.size()));
  }
  if (ctok.empty()) ctok.push_back(0);
  check(dashcu_rollout_load(pol, ptok.data(), poff.data(), static_cast<int32_t>(ts.size()), 1, ctok.data(),
                            coff.data()));
}

GradientVector download_grad(dashcu_policy* pol, const ArchConfig& a) {
  GradientVector g = GradientVector::zeros(a);
  std::vector<double> flat(g.num_params());
  check(dashcu_grad_download(pol, flat.data(), static_cast<std::int64_t>(flat.size())));
  unflatten(flat, g);
  return g;
}

// contiguous equal-size groups only (the DASH layout: G duplicates of each prompt)
int group_size(const GroupIndex& groups, int n) {
  groups.validate(n);
  const int G = static_cast<int>(groups.groups.front().size());
  int next = 0;
  for (const auto& g : groups.groups) {
    if (static_cast<int>(g.size()) != G) throw InputError("b200: groups must have equal size");
    for (int i : g)
      if (i != next++) throw InputError("b200: groups must be contiguous index ranges");
  }
  return G;
}

AdvantageBatch run_adv(const std::vector<double>* rewards, const std::vector<double>* given, int n, int G, int kind,
                       bool normalize, double eps, double tau, BaselineKind bk) {
  State& s = S();
  if (!s.ctx) check(dashcu_ctx_create(s.device, &s.ctx));
  AdvantageBatch out;
  out.baseline = bk;
  out.advantages.assign(n, 0.0);
  if (given) out.advantages = *given;
  std::vector<uint8_t> kept(n);
  int32_t nk = 0;
  check(dashcu_advantage_filter(s.ctx, rewards ? rewards->data() : nullptr, n, G, kind, normalize ? 1 : 0, eps, tau,
                                out.advantages.data(), kept.data(), nullptr, &nk));
  out.kept.assign(kept.begin(), kept.end());
  return out;
}

}  // namespace

void configure(int device, bool fp32_parity_mode) {
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  s.device = device;
  s.dtype = fp32_parity_mode ? DASHCU_F32 : DASHCU_BF16;
  if (s.pol) dashcu_policy_destroy(s.pol);
  if (s.base) dashcu_policy_destroy(s.base);
  if (s.ctx) dashcu_ctx_destroy(s.ctx);
  s.pol = nullptr;
  s.base = nullptr;
  s.ctx = nullptr;
  s.have_arch = s.have_params = false;
}

LogProbResult log_prob(const PolicyParams& params, const Trajectory& traj) {
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  dashcu_policy* pol = bind(params);
  load(pol, {&traj});
  LogProbResult r;
  const int len = traj.generation_length();
  std::vector<float> per(len > 0 ? len : 1);
  if (len > 0) check(dashcu_rollout_log_prob(pol, per.data(), len));
  r.per_token.assign(per.begin(), per.begin() + len);
  for (double v : r.per_token) r.total += v;
  return r;
}

Trajectory sample(const PolicyParams& params, const std::vector<int>& prompt, int max_len, double temperature,
                  std::uint64_t seed) {
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  dashcu_policy* pol = bind(params);
  dashcu_plan plan{1, 1, max_len, temperature, 0, 0};
  std::vector<int32_t> ptok(prompt.begin(), prompt.end());
  int64_t poff[2] = {0, static_cast<int64_t>(ptok.size())};
  const int ml = max_len > 0 ? max_len : 1;
  std::vector<int32_t> comp(ml);
  std::vector<float> lp(ml);
  int32_t len = 0;
  check(dashcu_sample_keyed(pol, &plan, ptok.data(), poff, &seed, comp.data(), &len, lp.data()));
  Trajectory t;
  t.prompt = prompt;
  t.completion.assign(comp.begin(), comp.begin() + len);
  t.log_probs.assign(lp.begin(), lp.begin() + len);
  return t;
}

GradientVector grad_log_prob(const PolicyParams& params, const Trajectory& traj) {
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  dashcu_policy* pol = bind(params);
  load(pol, {&traj});
  check(dashcu_grad_zero(pol));
  const double w = 1.0;
  check(dashcu_accumulate_weighted(pol, &w, 1, 0));
  return download_grad(pol, params.arch);
}

KlResult kl_term(const PolicyParams& params, const PolicyParams& base, const Trajectory& traj) {
  if (!(params.arch == base.arch)) throw InputError("kl_term: parameter sets have different architectures");
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  dashcu_policy* pol = bind(params);
  const std::uint64_t bh = base.content_hash();
  if (!s.base || bh != s.base_hash) {
    if (s.base) dashcu_policy_destroy(s.base);
    s.base = nullptr;
    const dashcu_arch a = to_c(base.arch);
    check(dashcu_policy_create(s.ctx, &a, s.dtype, &s.base));
    const auto flat = flatten(base);
    check(dashcu_policy_upload(s.base, flat.data(), static_cast<std::int64_t>(flat.size())));
    s.base_hash = bh;
  }
  load(pol, {&traj});
  check(dashcu_grad_zero(pol));
  KlResult r;
  check(dashcu_accumulate_kl(pol, s.base, 1.0, 0, nullptr, 0, &r.value));
  r.grad = download_grad(pol, params.arch);
  return r;
}

AdvantageBatch single_path_advantage(const std::vector<double>& rewards) {
  if (rewards.empty()) throw InputError("advantage of an empty batch");
  std::lock_guard<std::mutex> lk(S().mu);
  const int n = static_cast<int>(rewards.size());
  return run_adv(&rewards, nullptr, n, n, DASHCU_ADV_SINGLE_PATH, false, 0.0, 0.0, BaselineKind::Batch);
}

AdvantageBatch group_advantage(const std::vector<double>& rewards, const GroupIndex& groups) {
  if (rewards.empty()) throw InputError("advantage of an empty batch");
  const int n = static_cast<int>(rewards.size());
  const int G = group_size(groups, n);
  std::lock_guard<std::mutex> lk(S().mu);
  return run_adv(&rewards, nullptr, n, G, DASHCU_ADV_GROUP, false, 0.0, 0.0, BaselineKind::Group);
}

AdvantageBatch leave_one_out(const std::vector<double>& rewards, const GroupIndex& groups) {
  if (rewards.empty()) throw InputError("advantage of an empty batch");
  const int n = static_cast<int>(rewards.size());
  const int G = group_size(groups, n);
  std::lock_guard<std::mutex> lk(S().mu);
  return run_adv(&rewards, nullptr, n, G, DASHCU_ADV_LEAVE_ONE_OUT, false, 0.0, 0.0, BaselineKind::Group);
}

AdvantageBatch normalize_std(const AdvantageBatch& adv, const std::vector<double>& rewards, const GroupIndex& groups,
                             double eps) {
  if (adv.normalized) throw InputError("advantages are already normalized");
  if (static_cast<int>(rewards.size()) != adv.size())
    throw InputError("rewards and advantages disagree on batch size");
  const int n = adv.size();
  const int G = group_size(groups, n);
  std::lock_guard<std::mutex> lk(S().mu);
  AdvantageBatch out = run_adv(&rewards, &adv.advantages, n, G, DASHCU_ADV_GIVEN, true, eps, 0.0, adv.baseline);
  out.kept = adv.kept;  // only filter_by_threshold clears entries (advantage.hpp:25)
  out.normalized = true;
  return out;
}

AdvantageBatch filter_by_threshold(const AdvantageBatch& adv, double tau) {
  if (!(tau >= 0.0)) throw InputError("filter threshold must be >= 0");
  std::lock_guard<std::mutex> lk(S().mu);
  AdvantageBatch out = run_adv(nullptr, &adv.advantages, adv.size(), adv.size(), DASHCU_ADV_GIVEN, false, 0.0, tau,
                               adv.baseline);
  out.normalized = adv.normalized;
  return out;
}

std::vector<Trajectory> preemptive_sample(const SamplingPlan& plan, const PolicyParams& snapshot,
                                          const std::vector<std::vector<int>>& prompts) {
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  dashcu_policy* pol = bind(snapshot);
  if (plan.M != static_cast<int>(prompts.size())) throw InputError("plan.M must equal the number of prompts");
  std::vector<int32_t> ptok;
  std::vector<int64_t> poff{0};
  for (const auto& p : prompts) {
    ptok.insert(ptok.end(), p.begin(), p.end());
    poff.push_back(static_cast<int64_t>(ptok.size()));
  }
  if (ptok.empty()) ptok.push_back(0);
  const int S_ = plan.M * plan.G, ml = plan.max_len > 0 ? plan.max_len : 1;
  std::vector<int32_t> comp(static_cast<size_t>(S_) * ml), lens(S_);
  std::vector<float> lp(static_cast<size_t>(S_) * ml);
  dashcu_plan cp{plan.M, plan.G, plan.max_len, plan.temperature, plan.round_seed, plan.prompt_index_base};
  check(dashcu_sample(pol, &cp, ptok.data(), poff.data(), comp.data(), lens.data(), lp.data()));
  std::vector<Trajectory> out(S_);
  for (int i = 0; i < S_; ++i) {
    out[i].prompt = prompts[i / plan.G];
    out[i].completion.assign(comp.begin() + static_cast<size_t>(i) * ml, comp.begin() + static_cast<size_t>(i) * ml + lens[i]);
    out[i].log_probs.assign(lp.begin() + static_cast<size_t>(i) * ml, lp.begin() + static_cast<size_t>(i) * ml + lens[i]);
  }
  return out;
}

GradientVector pg_gradient(const std::vector<Trajectory>& batch, const AdvantageBatch& adv, const PolicyParams& params,
                           int micro_batch) {
  if (static_cast<int>(batch.size()) != adv.size()) throw InputError("batch and advantages disagree on size");
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  dashcu_policy* pol = bind(params);
  std::vector<const Trajectory*> ts;
  for (const auto& t : batch) ts.push_back(&t);
  load(pol, ts);
  const double N = static_cast<double>(batch.size());  // 1/N over the whole round (SURVEY App.B D4)
  std::vector<double> w(batch.size(), 0.0);
  for (size_t i = 0; i < batch.size(); ++i)
    if (adv.kept.empty() || adv.kept[i]) w[i] = adv.advantages[i] / N;
  check(dashcu_grad_zero(pol));
  check(dashcu_accumulate_weighted(pol, w.data(), static_cast<int32_t>(w.size()), micro_batch));
  return download_grad(pol, params.arch);
}

void optimizer_step(PolicyParams& params, const GradientVector& grad, OptState& st, double lr) {
  if (!(params.arch == grad.arch)) throw InputError("tensor arch mismatch in optimizer_step");
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  dashcu_policy* pol = bind(params);
  const auto g = flatten(grad);
  check(dashcu_grad_upload(pol, g.data(), static_cast<std::int64_t>(g.size())));
  dashcu_opt o{st.adam ? DASHCU_OPT_ADAM : DASHCU_OPT_SGD, lr, st.beta1, st.beta2, st.eps};
  check(dashcu_optimizer_step(pol, &o));
  std::vector<double> flat(params.num_params());
  check(dashcu_policy_download(pol, flat.data(), static_cast<std::int64_t>(flat.size())));
  unflatten(flat, params);
  s.hash = params.content_hash();  // device already holds exactly these (fp32-rounded) weights
}

void save_checkpoint(const PolicyParams& params, const std::string& path) {
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  check(dashcu_policy_save(bind(params), path.c_str(), 0));
}

PolicyParams load_checkpoint(const ArchConfig& arch, const std::string& path) {
  State& s = S();
  std::lock_guard<std::mutex> lk(s.mu);
  PolicyParams p = PolicyParams::zeros(arch);
  dashcu_policy* pol = bind(p);
  check(dashcu_policy_load(pol, path.c_str(), 0));
  std::vector<double> flat(p.num_params());
  check(dashcu_policy_download(pol, flat.data(), static_cast<std::int64_t>(flat.size())));
  unflatten(flat, p);
  s.hash = p.content_hash();
  return p;
}

}  // namespace dash::b200
