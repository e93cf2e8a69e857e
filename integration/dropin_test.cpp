// Drop-in check: the reference's own types and CPU functions (proj/src, linked
// unmodified) side by side with dash::b200 (the B200 path through libdashcu.so).
// Built by oracle/Makefile into oracle/_ref/dropin_test (it contains reference
// objects, so it is test infrastructure); run by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "dash/advantage.hpp"
#include "dash/errors.hpp"
#include "dash/policy.hpp"
#include "dash/rng.hpp"
#include "dash/tensors.hpp"
#include "dash_b200.hpp"

using namespace dash;

static int failures = 0;
static void expect(bool ok, const std::string& what, double v = 0.0) {
  std::printf("%s %s %.3e\n", ok ? "PASS" : "FAIL", what.c_str(), v);
  if (!ok) ++failures;
}

static double rel(const ParamTensors& a, const ParamTensors& b) {
  double num = 0, den = 0;
  auto va = a.views();
  auto vb = b.views();
  for (size_t t = 0; t < va.size(); ++t)
    for (size_t i = 0; i < va[t].size; ++i) {
      const double d = va[t].data[i] - vb[t].data[i];
      num += d * d;
      den += vb[t].data[i] * vb[t].data[i];
    }
  return std::sqrt(num / (den > 0 ? den : 1e-300));
}

static PolicyParams fp32_round(PolicyParams p) {
  for (auto& t : p.views())
    for (size_t i = 0; i < t.size; ++i) t.data[i] = static_cast<double>(static_cast<float>(t.data[i]));
  return p;
}

int main() {
  ArchConfig a;
  a.vocab_size = 256;
  a.embed_dim = 128;
  a.context_len = 64;
  a.ffn_hidden = 512;
  a.n_layers = 2;
  a.bos_id = 0;
  a.eos_id = 1;
  for (int mode = 0; mode < 2; ++mode) {
    const bool f32 = mode == 0;
    const double tol = f32 ? 1e-3 : 2e-2;
    const std::string tag = f32 ? "[f32] " : "[bf16] ";
    b200::configure(0, f32);
    PolicyParams p = fp32_round(PolicyParams::init(a, 0.02, 1));
    Trajectory t;
    t.prompt = {0, 50, 51, 43, 52, 53, 61};
    t.completion = {66, 75, 40, 115, 241, 20, 64, 51};
    const double lr = log_prob(p, t).total, lg = b200::log_prob(p, t).total;
    expect(std::fabs(lg - lr) <= tol * std::fabs(lr), tag + "log_prob vs reference (golden completion)",
           std::fabs(lg - lr) / std::fabs(lr));
    expect(rel(b200::grad_log_prob(p, t), grad_log_prob(p, t)) <= tol, tag + "grad_log_prob vs reference",
           rel(b200::grad_log_prob(p, t), grad_log_prob(p, t)));
    // advantage / filter: bit-exact
    std::vector<double> r;
    for (int i = 0; i < 64; ++i) r.push_back(static_cast<double>((i * 7 + i / 8) % 3 == 0));
    const auto gi = GroupIndex::contiguous(64, 8);
    const auto ga = group_advantage(r, gi), gb = b200::group_advantage(r, gi);
    expect(ga.advantages == gb.advantages, tag + "group_advantage bit-exact");
    const auto fa = filter_by_threshold(ga, 0.1), fb = b200::filter_by_threshold(gb, 0.1);
    expect(fa.kept == fb.kept, tag + "filter_by_threshold bit-exact");
    expect(normalize_std(ga, r, gi, 1e-6).advantages == b200::normalize_std(gb, r, gi, 1e-6).advantages,
           tag + "normalize_std bit-exact");
    expect(leave_one_out(r, gi).advantages == b200::leave_one_out(r, gi).advantages, tag + "leave_one_out bit-exact");
    expect(single_path_advantage(r).advantages == b200::single_path_advantage(r).advantages,
           tag + "single_path_advantage bit-exact");
    // one DASH round through the SPEC-level batch API
    b200::SamplingPlan plan;
    plan.M = 8;
    plan.G = 8;
    plan.max_len = 24;
    plan.round_seed = 3;
    std::vector<std::vector<int>> prompts;
    for (int m = 0; m < plan.M; ++m) prompts.push_back({0, 50 + m, 43, 52, 61});
    const auto batch = b200::preemptive_sample(plan, p, prompts);
    expect(static_cast<int>(batch.size()) == plan.M * plan.G, tag + "preemptive_sample count");
    std::vector<double> rw;
    for (int i = 0; i < plan.M * plan.G; ++i)
      rw.push_back(std::fmod(static_cast<double>(splitmix64(i * 977 + 5) % 1000), 2.0));
    const auto adv = b200::filter_by_threshold(
        b200::group_advantage(rw, GroupIndex::contiguous(plan.M * plan.G, plan.G)), 0.1);
    const GradientVector gb200 = b200::pg_gradient(batch, adv, p, 16);
    GradientVector gref = GradientVector::zeros(a);
    for (size_t i = 0; i < batch.size(); ++i)
      if (adv.kept[i]) gref.add_scaled(grad_log_prob(p, batch[i]), adv.advantages[i] / batch.size());
    expect(rel(gb200, gref) <= tol, tag + "pg_gradient vs reference sum of A/N grad_log_prob", rel(gb200, gref));
    // recorded log-probs replay within tolerance
    double worst = 0;
    for (int i = 0; i < 4; ++i) {
      const auto lpr = log_prob(p, batch[i]);
      for (int j = 0; j < batch[i].generation_length(); ++j)
        worst = std::fmax(worst, std::fabs(lpr.per_token[j] - batch[i].log_probs[j]));
    }
    expect(worst <= (f32 ? 1e-3 : 5e-2), tag + "sampled log-probs replay under the reference log_prob", worst);
    // optimizer: SGD ascent equals add_scaled(grad, lr)
    PolicyParams q = p;
    b200::OptState os;
    os.adam = false;
    b200::optimizer_step(q, gb200, os, 1e-2);
    PolicyParams qr = p;
    qr.add_scaled(gb200, 1e-2);
    expect(q.max_abs_diff(qr) <= 1e-6, tag + "optimizer_step (SGD) vs add_scaled", q.max_abs_diff(qr));
    // determinism + error mapping
    const auto s1 = b200::sample(p, t.prompt, 10, 1.0, 77), s2 = b200::sample(p, t.prompt, 10, 1.0, 77);
    expect(s1.completion == s2.completion, tag + "sample deterministic per seed");
    bool threw = false;
    try {
      b200::sample(p, t.prompt, 10, 0.0, 1);
    } catch (const InputError&) {
      threw = true;
    }
    expect(threw, tag + "nonpositive temperature -> InputError");
    threw = false;
    try {
      Trajectory bad = t;
      bad.completion.push_back(0);
      b200::log_prob(p, bad);
    } catch (const InputError&) {
      threw = true;
    }
    expect(threw, tag + "BOS in completion -> InputError");
    // kl_term against the reference's (value and gradient), and kl(p, p) = 0
    PolicyParams base = p;
    {
      Rng br(5);
      for (auto& v : base.views())
        for (size_t i = 0; i < v.size; ++i) v.data[i] = static_cast<double>(static_cast<float>(v.data[i] + 0.01 * br.normal()));
    }
    const KlResult kr = kl_term(p, base, t), kb = b200::kl_term(p, base, t);
    expect(std::fabs(kb.value - kr.value) <= (f32 ? 1e-3 : 2e-2) * std::fabs(kr.value), tag + "kl_term value vs reference",
           std::fabs(kb.value - kr.value) / std::fabs(kr.value));
    expect(rel(kb.grad, kr.grad) <= tol, tag + "kl_term gradient vs reference", rel(kb.grad, kr.grad));
    const KlResult k0 = b200::kl_term(p, p, t);
    expect(std::fabs(k0.value) <= 1e-6 && k0.grad.max_abs() <= 1e-6, tag + "kl_term(p, p) = 0", std::fabs(k0.value));
    // checkpoint round trip through the container (bitwise)
    const std::string ck = "/tmp/dropin_ckpt_" + std::to_string(mode) + ".bin";
    b200::save_checkpoint(p, ck);
    const PolicyParams pl = b200::load_checkpoint(p.arch, ck);
    expect(pl.content_hash() == p.content_hash(), tag + "checkpoint save/load bitwise (content_hash)");
  }
  std::printf("%s (%d failures)\n", failures ? "DROPIN FAIL" : "DROPIN OK", failures);
  return failures ? 1 : 0;
}
