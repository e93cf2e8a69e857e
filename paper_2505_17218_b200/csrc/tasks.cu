// Synthetic verifiable tasks on the host: the prompt feeder and the trajectory reward of the
// DASH step (tasks.cpp:105-175). Host-only C++ (no device work): prompts
// are generated per instance seed exactly as generate_instance does (std::mt19937_64 with
// the reference's rejection-sampled below(), rng.hpp:36-60) and rewarded exactly as
// reward() does (text after the last '#' up to EOS, trimmed of spaces / tabs, compared with
// the canonical answer).
//
// Two vocabularies: the task's own (build_vocab, tasks.cpp:23-53: "<s>", "</s>", then the
// task's characters) and the byte vocabulary of BASELINE configs[0] (SURVEY App.B D7:
// id 0 "<s>", id 1 "</s>", ids 2..255 the single bytes 2..255, delimiter "#").
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/dashcu.h"
#include "common.cuh"

namespace dashcu {
extern thread_local std::string g_last_error;  // policy.cu (dashcu_last_error)
namespace {

// Rng::below (rng.hpp:44-52): rejection sampling without modulo bias
uint64_t below(std::mt19937_64& e, uint64_t n) {
  const uint64_t limit = n * (UINT64_MAX / n);
  uint64_t x;
  do {
    x = e();
  } while (x >= limit);
  return x % n;
}

// uniform_with_digits (tasks.cpp:55-62)
uint64_t uniform_with_digits(std::mt19937_64& e, int digits) {
  if (digits == 1) return below(e, 10);
  uint64_t lo = 1;
  for (int i = 1; i < digits; ++i) lo *= 10;
  const uint64_t hi = lo * 10 - 1;
  return lo + below(e, hi - lo + 1);
}

const char* task_chars(int kind) {  // build_vocab (tasks.cpp:23-53), after <s> and </s>
  switch (kind) {
    case DASHCU_TASK_ADD: return "0123456789+=,#";
    case DASHCU_TASK_MOD: return "0123456789%=,#";
    case DASHCU_TASK_REVERSE: return "abcd>,#";
    case DASHCU_TASK_PARITY: return "01=,#";
    case DASHCU_TASK_MICRO: return "#ab";
  }
  return nullptr;
}

struct Vocab {
  int kind = 0, vocab = 0;  // vocab: DASHCU_VOCAB_TASK or DASHCU_VOCAB_BYTE
  int bos = 0, eos = 1;
  int id(char c) const {
    if (vocab == DASHCU_VOCAB_BYTE) {
      const int b = static_cast<unsigned char>(c);
      return b >= 2 ? b : -1;
    }
    const char* p = std::strchr(task_chars(kind), c);
    return p && c ? 2 + static_cast<int>(p - task_chars(kind)) : -1;
  }
  int size() const { return vocab == DASHCU_VOCAB_BYTE ? 256 : 2 + static_cast<int>(std::strlen(task_chars(kind))); }
  int delim() const { return id('#'); }
  // token text of a completion id (Vocab::token); BOS / EOS never appear in answers
  std::string token(int t) const {
    if (t == bos) return "<s>";
    if (t == eos) return "</s>";
    if (t < 0 || t >= size()) return "?";
    if (vocab == DASHCU_VOCAB_BYTE) return std::string(1, static_cast<char>(t));
    return std::string(1, task_chars(kind)[t - 2]);
  }
};

Vocab vocab_of(int kind, int vocab) {
  if (!task_chars(kind)) throw Error(1, "unknown task kind");
  if (vocab != DASHCU_VOCAB_TASK && vocab != DASHCU_VOCAB_BYTE) throw Error(1, "unknown vocabulary");
  Vocab v;
  v.kind = kind;
  v.vocab = vocab;
  return v;
}

// generate_instance (tasks.cpp:105-153): prompt body text and answer
void instance(int kind, int difficulty, uint64_t seed, std::string* body, std::string* answer) {
  std::mt19937_64 e(seed);
  switch (kind) {
    case DASHCU_TASK_ADD: {
      const uint64_t a = uniform_with_digits(e, difficulty);
      const uint64_t b = uniform_with_digits(e, difficulty);
      *body = std::to_string(a) + "+" + std::to_string(b) + "=";
      *answer = std::to_string(a + b);
      break;
    }
    case DASHCU_TASK_MOD: {
      const uint64_t a = uniform_with_digits(e, difficulty);
      const uint64_t m = 2 + below(e, 8);
      *body = std::to_string(a) + "%" + std::to_string(m) + "=";
      *answer = std::to_string(a % m);
      break;
    }
    case DASHCU_TASK_REVERSE: {
      std::string s;
      for (int i = 0; i < difficulty; ++i) s += static_cast<char>('a' + below(e, 4));
      *body = s + ">";
      *answer = std::string(s.rbegin(), s.rend());
      break;
    }
    case DASHCU_TASK_PARITY: {
      std::string s;
      int ones = 0;
      for (int i = 0; i < difficulty; ++i) {
        const int bit = static_cast<int>(below(e, 2));
        ones += bit;
        s += static_cast<char>('0' + bit);
      }
      *body = s + "=";
      *answer = ones % 2 == 1 ? "1" : "0";
      break;
    }
    case DASHCU_TASK_MICRO: {
      const char q = below(e, 2) == 0 ? 'a' : 'b';
      *body = std::string(1, q);
      *answer = std::string(1, q);
      break;
    }
  }
}

// reward (tasks.cpp:155-175)
double reward_of(const Vocab& v, const std::string& answer, const int32_t* comp, int len) {
  int last = -1, end = len;
  for (int i = 0; i < len; ++i) {
    if (comp[i] == v.eos) {
      end = i;
      break;
    }
    if (comp[i] == v.delim()) last = i;
  }
  if (last < 0) return 0.0;
  std::string text;
  for (int i = last + 1; i < end; ++i) text += v.token(comp[i]);
  const auto first = text.find_first_not_of(" \t");
  const auto lastc = text.find_last_not_of(" \t");
  text = first == std::string::npos ? "" : text.substr(first, lastc - first + 1);
  return text == answer ? 1.0 : 0.0;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return DASHCU_E_DEVICE;
  }
  return DASHCU_OK;
}

}  // namespace

}  // namespace dashcu

using namespace dashcu;

extern "C" {

int dashcu_task_vocab_size(int32_t kind, int32_t vocab, int32_t* size) {
  return guarded([&] {
    if (!size) throw Error(1, "null argument");
    *size = vocab_of(kind, vocab).size();
  });
}

int dashcu_task_instances(int32_t kind, int32_t difficulty, int32_t vocab, const uint64_t* seeds, int32_t n,
                          int32_t* prompt_tokens, int64_t prompt_cap, int64_t* prompt_offsets, char* answers,
                          int32_t answer_stride) {
  return guarded([&] {
    if (difficulty < 1) throw Error(1, "task difficulty must be >= 1");  // TaskSpec::make
    if (!seeds || !prompt_offsets || n < 0) throw Error(1, "null argument");
    const Vocab v = vocab_of(kind, vocab);
    prompt_offsets[0] = 0;
    for (int i = 0; i < n; ++i) {
      std::string body, ans;
      instance(kind, difficulty, seeds[i], &body, &ans);
      const int64_t o = prompt_offsets[i];
      const int64_t m = 1 + static_cast<int64_t>(body.size());
      if (prompt_tokens && o + m > prompt_cap) throw Error(2, "prompt buffer too small");
      if (prompt_tokens) {
        prompt_tokens[o] = v.bos;
        for (size_t c = 0; c < body.size(); ++c) {
          const int id = v.id(body[c]);
          if (id < 0) throw Error(1, std::string("character not in vocab: ") + body[c]);
          prompt_tokens[o + 1 + static_cast<int64_t>(c)] = id;
        }
      }
      prompt_offsets[i + 1] = o + m;
      if (answers && answer_stride > 0)
        std::snprintf(answers + static_cast<int64_t>(i) * answer_stride, answer_stride, "%s", ans.c_str());
    }
  });
}

int dashcu_task_rewards(int32_t kind, int32_t difficulty, int32_t vocab, const uint64_t* seeds, int32_t n_prompts,
                        int32_t group_size, const int32_t* completions, int32_t stride, const int32_t* lengths,
                        double* rewards) {
  return guarded([&] {
    if (difficulty < 1) throw Error(1, "task difficulty must be >= 1");
    if (!seeds || !completions || !lengths || !rewards || n_prompts < 0 || group_size < 1)
      throw Error(1, "null argument");
    const Vocab v = vocab_of(kind, vocab);
    for (int m = 0; m < n_prompts; ++m) {
      std::string body, ans;
      instance(kind, difficulty, seeds[m], &body, &ans);
      for (int g = 0; g < group_size; ++g) {
        const int64_t s = static_cast<int64_t>(m) * group_size + g;
        rewards[s] = reward_of(v, ans, completions + s * stride, lengths[s]);
      }
    }
  });
}

}  // extern "C"
