/* TEST INFRASTRUCTURE ONLY — the CPU oracle (see dash_oracle.h). Never linked into
 * the product; the product path fails loudly without its CUDA library.
 *
 * Reference anchors (paths under /root/reference/proj):
 *   rng                  include/dash/rng.hpp:10-82
 *   layout / init        src/tensors.cpp:49-71, :150-158
 *   forward (advance)    src/policy.cpp:80-153     lse/softmax :156-181
 *   log_prob             src/policy.cpp:362-377    sample :379-429
 *   grad_log_prob        src/policy.cpp:463-485    backward :201-346
 *   advantage / filter   src/advantage.cpp:9-140
 *   pg / optimizer
 * Compiled with -ffp-contract=off (oracle/Makefile).
 */
#include "dash_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */

uint64_t dor_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t dor_fnv1a(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (const unsigned char* p = (const unsigned char*)s; *p; ++p) {
    h ^= *p;
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t dor_derive_seed(uint64_t base, const char* tag, uint64_t a, uint64_t b) {
  uint64_t h = dor_splitmix64(base ^ dor_fnv1a(tag));
  h = dor_splitmix64(h ^ (a + 0x9e3779b97f4a7c15ull));
  return dor_splitmix64(h ^ (b + 0x7f4a7c159e3779b9ull));
}

/* std::mt19937_64 (the engine behind dash::Rng, rng.hpp:40-82) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

typedef struct {
  mt64 eng;
  int has_spare;
  double spare;
} drng;

static double drng_u01(drng* r) { return (double)(mt64_next(&r->eng) >> 11) * 0x1.0p-53; }

/* Marsaglia polar, second value cached (rng.hpp:61-76) */
static double drng_normal(drng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u, v, s;
  do {
    u = 2.0 * drng_u01(r) - 1.0;
    v = 2.0 * drng_u01(r) - 1.0;
    s = u * u + v * v;
  } while (s >= 1.0 || s == 0.0);
  const double m = sqrt(-2.0 * log(s) / s);
  r->spare = v * m;
  r->has_spare = 1;
  return u * m;
}

void dor_rng_draws(uint64_t seed, int kind, int n, uint64_t* out) {
  drng r;
  mt64_seed(&r.eng, seed);
  r.has_spare = 0;
  for (int i = 0; i < n; ++i) {
    if (kind == 0) {
      out[i] = mt64_next(&r.eng);
    } else {
      double v = kind == 1 ? drng_u01(&r) : drng_normal(&r);
      memcpy(&out[i], &v, sizeof v);
    }
  }
}

/* --------------------------------------------------------------- layout */

typedef struct {
  int V, d, ctx, H, L, bos, eos, nh, nkv, hd, qd, kvd, grp;
} geo;

static geo geo_of(const dor_arch* a) {
  geo g;
  g.V = a->vocab_size;
  g.d = a->embed_dim;
  g.ctx = a->context_len;
  g.H = a->ffn_hidden;
  g.L = a->n_layers;
  g.bos = a->bos_id;
  g.eos = a->eos_id;
  g.nh = a->n_heads > 0 ? a->n_heads : 1;
  g.nkv = a->n_kv_heads > 0 ? a->n_kv_heads : 1;
  g.hd = a->head_dim > 0 ? a->head_dim : a->embed_dim;
  g.qd = g.nh * g.hd;
  g.kvd = g.nkv * g.hd;
  g.grp = g.nh / g.nkv;
  return g;
}

void dor_layout_of(const dor_arch* a, dor_layout* o) {
  const geo g = geo_of(a);
  int64_t off = 0;
  o->token_embed = off;
  off += (int64_t)g.V * g.d;
  o->pos_embed = off;
  off += (int64_t)g.ctx * g.d;
  o->layer0 = off;
  int64_t lo = 0;
  o->wq = lo;
  lo += (int64_t)g.qd * g.d;
  o->wk = lo;
  lo += (int64_t)g.kvd * g.d;
  o->wv = lo;
  lo += (int64_t)g.kvd * g.d;
  o->wo = lo;
  lo += (int64_t)g.d * g.qd;
  o->w1 = lo;
  lo += (int64_t)g.H * g.d;
  o->b1 = lo;
  lo += g.H;
  o->w2 = lo;
  lo += (int64_t)g.d * g.H;
  o->b2 = lo;
  lo += g.d;
  o->layer_stride = lo;
  off += lo * g.L;
  o->w_out = off;
  off += (int64_t)g.V * g.d;
  o->b_out = off;
  off += g.V;
  o->total = off;
}

int64_t dor_num_params(const dor_arch* a) {
  dor_layout l;
  dor_layout_of(a, &l);
  return l.total;
}

void dor_init_params(const dor_arch* a, double scale, uint64_t seed, double* out) {
  const int64_t n = dor_num_params(a);
  if (scale == 0.0) {
    memset(out, 0, (size_t)n * sizeof(double));
    return;
  }
  drng r;
  mt64_seed(&r.eng, seed);
  r.has_spare = 0;
  for (int64_t i = 0; i < n; ++i) out[i] = scale * drng_normal(&r);
}

/* Restates the device kernel init_normal_ctr (paper_2505_17218_b200/csrc/kernels_misc.cu):
 * Box-Muller on a counter hash, pair k = i/2 -> (cos, sin). */
void dor_init_params_ctr(const dor_arch* a, double scale, uint64_t seed, double* out) {
  const int64_t n = dor_num_params(a);
  const uint64_t key = dor_splitmix64(seed ^ 0x5DEECE66Dull);
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t k = (uint64_t)(i >> 1);
    const uint64_t h1 = dor_splitmix64(key ^ (2 * k));
    const uint64_t h2 = dor_splitmix64(key ^ (2 * k + 1));
    const double u1 = ((double)(h1 >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double t = 6.283185307179586 * u2;
    out[i] = scale * ((i & 1) ? r * sin(t) : r * cos(t));
  }
}

/* ------------------------------------------------------------- forward */

/* Activations of one sequence at every position (the reference Cache,
 * policy.cpp:45-78, generalised to GQA). */
typedef struct {
  int n;
  double *x, *q, *k, *v, *ctx, *h, *u, *y; /* [L][n][*] */
  double* att;                            /* [L][nh][n][n] */
  double* logits;                         /* [n][V] */
} acts;

static void acts_alloc(const geo* g, int n, acts* s) {
  s->n = n;
  const size_t L = (size_t)g->L, N = (size_t)n;
  s->x = calloc(L * N * g->d, sizeof(double));
  s->q = calloc(L * N * g->qd, sizeof(double));
  s->k = calloc(L * N * g->kvd, sizeof(double));
  s->v = calloc(L * N * g->kvd, sizeof(double));
  s->ctx = calloc(L * N * g->qd, sizeof(double));
  s->h = calloc(L * N * g->d, sizeof(double));
  s->u = calloc(L * N * g->H, sizeof(double));
  s->y = calloc(L * N * g->d, sizeof(double));
  s->att = calloc(L * g->nh * N * N, sizeof(double));
  s->logits = calloc(N * g->V, sizeof(double));
}

static void acts_free(acts* s) {
  free(s->x);
  free(s->q);
  free(s->k);
  free(s->v);
  free(s->ctx);
  free(s->h);
  free(s->u);
  free(s->y);
  free(s->att);
  free(s->logits);
}

/* y[o] = sum_i W[o][i] x[i], summed in index order (policy.cpp:21-28) */
static void mv(const double* w, const double* x, double* y, int out, int in) {
  for (int o = 0; o < out; ++o) {
    const double* r = w + (size_t)o * in;
    double s = 0.0;
    for (int i = 0; i < in; ++i) s += r[i] * x[i];
    y[o] = s;
  }
}

#define AT(base, l, t, w) ((base) + ((size_t)(l) * (size_t)NPOS + (size_t)(t)) * (size_t)(w))

/* Forward over tokens[0..n) (advance() per position, policy.cpp:80-153). */
static void forward(const geo* g, const dor_layout* lay, const double* P, const int32_t* tok, acts* s) {
  const int n = s->n, d = g->d, hd = g->hd;
  const int NPOS = n;
  const double scale = 1.0 / sqrt((double)hd);
  double* row = malloc(sizeof(double) * (size_t)n);
  for (int t = 0; t < n; ++t) {
    const double* e = P + lay->token_embed + (size_t)tok[t] * d;
    const double* pe = P + lay->pos_embed + (size_t)t * d;
    double* x = AT(s->x, 0, t, d);
    for (int i = 0; i < d; ++i) x[i] = e[i] + pe[i];
  }
  for (int l = 0; l < g->L; ++l) {
    const double* B = P + lay->layer0 + (size_t)l * lay->layer_stride;
    for (int t = 0; t < n; ++t) {
      const double* x = AT(s->x, l, t, d);
      mv(B + lay->wq, x, AT(s->q, l, t, g->qd), g->qd, d);
      mv(B + lay->wk, x, AT(s->k, l, t, g->kvd), g->kvd, d);
      mv(B + lay->wv, x, AT(s->v, l, t, g->kvd), g->kvd, d);
    }
    for (int t = 0; t < n; ++t) {
      double* c = AT(s->ctx, l, t, g->qd);
      for (int hh = 0; hh < g->nh; ++hh) {
        const int kv = hh / g->grp;
        const double* q = AT(s->q, l, t, g->qd) + hh * hd;
        double* a = s->att + (((size_t)l * g->nh + hh) * n + t) * n;
        double mx = -INFINITY;
        for (int j = 0; j <= t; ++j) {
          const double* kj = AT(s->k, l, j, g->kvd) + kv * hd;
          double sc = 0.0;
          for (int i = 0; i < hd; ++i) sc += q[i] * kj[i];
          sc *= scale;
          a[j] = sc;
          if (sc > mx) mx = sc;
        }
        double den = 0.0;
        for (int j = 0; j <= t; ++j) {
          a[j] = exp(a[j] - mx);
          den += a[j];
        }
        const double inv = 1.0 / den;
        for (int j = 0; j <= t; ++j) a[j] *= inv;
        double* ch = c + hh * hd;
        for (int i = 0; i < hd; ++i) ch[i] = 0.0;
        for (int j = 0; j <= t; ++j) {
          const double w = a[j];
          const double* vj = AT(s->v, l, j, g->kvd) + kv * hd;
          for (int i = 0; i < hd; ++i) ch[i] += w * vj[i];
        }
      }
      const double* x = AT(s->x, l, t, d);
      double* h = AT(s->h, l, t, d);
      mv(B + lay->wo, c, h, d, g->qd);
      for (int i = 0; i < d; ++i) h[i] += x[i];
      double* u = AT(s->u, l, t, g->H);
      mv(B + lay->w1, h, u, g->H, d);
      for (int j = 0; j < g->H; ++j) u[j] = tanh(u[j] + B[lay->b1 + j]);
      double* y = AT(s->y, l, t, d);
      mv(B + lay->w2, u, y, d, g->H);
      for (int i = 0; i < d; ++i) y[i] += B[lay->b2 + i] + h[i];
      if (l + 1 < g->L) memcpy(AT(s->x, l + 1, t, d), y, sizeof(double) * (size_t)d);
    }
  }
  for (int t = 0; t < n; ++t) {
    double* lg = s->logits + (size_t)t * g->V;
    mv(P + lay->w_out, AT(s->y, g->L - 1, t, d), lg, g->V, d);
    for (int o = 0; o < g->V; ++o) lg[o] += P[lay->b_out + o];
  }
  free(row);
}

/* log-sum-exp over non-BOS ids (policy.cpp:156-164) */
static double lse_nobos(const double* lg, int V, int bos) {
  double mx = -INFINITY;
  for (int i = 0; i < V; ++i)
    if (i != bos && lg[i] > mx) mx = lg[i];
  double den = 0.0;
  for (int i = 0; i < V; ++i)
    if (i != bos) den += exp(lg[i] - mx);
  return mx + log(den);
}

static int32_t* concat(const int32_t* a, int na, const int32_t* b, int nb) {
  int32_t* out = malloc(sizeof(int32_t) * (size_t)(na + nb + 1));
  memcpy(out, a, sizeof(int32_t) * (size_t)na);
  if (nb > 0) memcpy(out + na, b, sizeof(int32_t) * (size_t)nb);
  return out;
}

double dor_log_prob(const dor_arch* a, const double* params, const int32_t* prompt, int m,
                    const int32_t* completion, int len, double* per_token) {
  if (len == 0) return 0.0;
  const geo g = geo_of(a);
  dor_layout lay;
  dor_layout_of(a, &lay);
  const int n = m + len - 1; /* the last completion token is never fed (policy.cpp:350-358) */
  int32_t* tok = concat(prompt, m, completion, len - 1);
  acts s;
  acts_alloc(&g, n, &s);
  forward(&g, &lay, params, tok, &s);
  double total = 0.0;
  for (int j = 0; j < len; ++j) {
    const double* lg = s.logits + (size_t)(m - 1 + j) * g.V;
    const double v = lg[completion[j]] - lse_nobos(lg, g.V, g.bos);
    if (per_token) per_token[j] = v;
    total += v;
  }
  acts_free(&s);
  free(tok);
  return total;
}

void dor_next_logits(const dor_arch* a, const double* params, const int32_t* ctx, int n,
                     double* logits) {
  const geo g = geo_of(a);
  dor_layout lay;
  dor_layout_of(a, &lay);
  acts s;
  acts_alloc(&g, n, &s);
  forward(&g, &lay, params, ctx, &s);
  memcpy(logits, s.logits + (size_t)(n - 1) * g.V, sizeof(double) * (size_t)g.V);
  acts_free(&s);
}

/* ------------------------------------------------------------- backward */

/* out[o][i] += s * a[o] * b[i] */
static void outer_acc(double* out, const double* a, const double* b, int no, int ni) {
  for (int o = 0; o < no; ++o) {
    const double ao = a[o];
    if (ao == 0.0) continue;
    double* r = out + (size_t)o * ni;
    for (int i = 0; i < ni; ++i) r[i] += ao * b[i];
  }
}

/* y[i] += sum_o W[o][i] a[o] */
static void mtv_acc(const double* w, const double* a, double* y, int no, int ni) {
  for (int o = 0; o < no; ++o) {
    const double ao = a[o];
    if (ao == 0.0) continue;
    const double* r = w + (size_t)o * ni;
    for (int i = 0; i < ni; ++i) y[i] += ao * r[i];
  }
}

/* grad_log_prob (policy.cpp:463-485) or, with base != NULL, the gradient of kl_term
 * (policy.cpp:487-522: dlogits = softmax(current) - softmax(base) at every completion
 * position, value = sum_j sum_i pb_i ((lb_i - lse_b) - (lc_i - lse_c))), scaled into grad. */
static void grad_core(const dor_arch* a, const double* P, const double* base, const int32_t* prompt, int m,
                      const int32_t* completion, int len, double scale, double* grad, double* kl_value) {
  if (kl_value) *kl_value = 0.0;
  if (len == 0 || (scale == 0.0 && !kl_value)) return;
  const geo g = geo_of(a);
  dor_layout lay;
  dor_layout_of(a, &lay);
  const int n = m + len - 1, d = g.d, hd = g.hd, V = g.V;
  const int NPOS = n;
  const double att_scale = 1.0 / sqrt((double)hd);
  int32_t* tok = concat(prompt, m, completion, len - 1);
  acts s;
  acts_alloc(&g, n, &s);
  forward(&g, &lay, P, tok, &s);

  double* G = calloc((size_t)lay.total, sizeof(double)); /* this trajectory's gradient */
  double* dz = calloc((size_t)V, sizeof(double));
  double* dy = calloc((size_t)n * d, sizeof(double));
  double* dx = calloc((size_t)n * d, sizeof(double));
  double* dh = calloc((size_t)n * d, sizeof(double));
  double* dctx = calloc((size_t)n * g.qd, sizeof(double));
  double* dq = calloc((size_t)n * g.qd, sizeof(double));
  double* dk = calloc((size_t)n * g.kvd, sizeof(double));
  double* dv = calloc((size_t)n * g.kvd, sizeof(double));
  double* du = calloc((size_t)g.H, sizeof(double));
  double* da = calloc((size_t)n, sizeof(double));

  acts sb;
  if (base) {
    acts_alloc(&g, n, &sb);
    forward(&g, &lay, base, tok, &sb);
  }
  /* LM head: dlogits = onehot(y) - softmax_nobos (policy.cpp:471-483), or the KL term's
   * pc - pb (policy.cpp:509-518) */
  for (int j = 0; j < len; ++j) {
    const int t = m - 1 + j;
    const double* lg = s.logits + (size_t)t * V;
    const double lse = lse_nobos(lg, V, g.bos);
    if (base) {
      const double* lb = sb.logits + (size_t)t * V;
      const double lse_b = lse_nobos(lb, V, g.bos);
      for (int i = 0; i < V; ++i) {
        if (i == g.bos) {
          dz[i] = 0.0;
          continue;
        }
        const double pb = exp(lb[i] - lse_b), pc = exp(lg[i] - lse);
        if (kl_value) *kl_value += pb * ((lb[i] - lse_b) - (lg[i] - lse));
        dz[i] = pc - pb;
      }
    } else {
      for (int i = 0; i < V; ++i) dz[i] = (i == g.bos) ? 0.0 : -exp(lg[i] - lse);
      dz[completion[j]] += 1.0;
    }
    const double* yt = AT(s.y, g.L - 1, t, d);
    outer_acc(G + lay.w_out, dz, yt, V, d);
    for (int i = 0; i < V; ++i) G[lay.b_out + i] += dz[i];
    mtv_acc(P + lay.w_out, dz, dy + (size_t)t * d, V, d);
  }

  for (int l = g.L - 1; l >= 0; --l) {
    const double* B = P + lay.layer0 + (size_t)l * lay.layer_stride;
    double* GB = G + lay.layer0 + (size_t)l * lay.layer_stride;
    memset(dx, 0, sizeof(double) * (size_t)n * d);
    memset(dctx, 0, sizeof(double) * (size_t)n * g.qd);
    memset(dq, 0, sizeof(double) * (size_t)n * g.qd);
    memset(dk, 0, sizeof(double) * (size_t)n * g.kvd);
    memset(dv, 0, sizeof(double) * (size_t)n * g.kvd);
    for (int t = 0; t < n; ++t) {
      /* y = h + W2 tanh(W1 h + b1) + b2 */
      const double* dyt = dy + (size_t)t * d;
      const double* u = AT(s.u, l, t, g.H);
      const double* h = AT(s.h, l, t, d);
      outer_acc(GB + lay.w2, dyt, u, d, g.H);
      for (int i = 0; i < d; ++i) GB[lay.b2 + i] += dyt[i];
      memset(du, 0, sizeof(double) * (size_t)g.H);
      mtv_acc(B + lay.w2, dyt, du, d, g.H);
      for (int j = 0; j < g.H; ++j) du[j] *= (1.0 - u[j] * u[j]);
      outer_acc(GB + lay.w1, du, h, g.H, d);
      for (int j = 0; j < g.H; ++j) GB[lay.b1 + j] += du[j];
      double* dht = dh + (size_t)t * d;
      memcpy(dht, dyt, sizeof(double) * (size_t)d);
      mtv_acc(B + lay.w1, du, dht, g.H, d);
      /* h = x + Wo ctx */
      double* dxt = dx + (size_t)t * d;
      for (int i = 0; i < d; ++i) dxt[i] += dht[i];
      outer_acc(GB + lay.wo, dht, AT(s.ctx, l, t, g.qd), d, g.qd);
      mtv_acc(B + lay.wo, dht, dctx + (size_t)t * g.qd, d, g.qd);
    }
    /* attention: ctx_t = sum_j a_tj v_j, a_t = softmax(q_t.k_j * scale) (policy.cpp:292-322) */
    for (int hh = 0; hh < g.nh; ++hh) {
      const int kv = hh / g.grp;
      for (int t = 0; t < n; ++t) {
        const double* arow = s.att + (((size_t)l * g.nh + hh) * n + t) * n;
        const double* dct = dctx + (size_t)t * g.qd + hh * hd;
        const double* qt = AT(s.q, l, t, g.qd) + hh * hd;
        double wsum = 0.0;
        for (int j = 0; j <= t; ++j) {
          const double* vj = AT(s.v, l, j, g.kvd) + kv * hd;
          double acc = 0.0;
          for (int i = 0; i < hd; ++i) acc += vj[i] * dct[i];
          da[j] = acc;
          wsum += arow[j] * acc;
          double* dvj = dv + (size_t)j * g.kvd + kv * hd;
          for (int i = 0; i < hd; ++i) dvj[i] += arow[j] * dct[i];
        }
        double* dqt = dq + (size_t)t * g.qd + hh * hd;
        for (int j = 0; j <= t; ++j) {
          const double ds = arow[j] * (da[j] - wsum) * att_scale;
          if (ds == 0.0) continue;
          const double* kj = AT(s.k, l, j, g.kvd) + kv * hd;
          double* dkj = dk + (size_t)j * g.kvd + kv * hd;
          for (int i = 0; i < hd; ++i) {
            dqt[i] += ds * kj[i];
            dkj[i] += ds * qt[i];
          }
        }
      }
    }
    for (int t = 0; t < n; ++t) {
      const double* x = AT(s.x, l, t, d);
      double* dxt = dx + (size_t)t * d;
      outer_acc(GB + lay.wq, dq + (size_t)t * g.qd, x, g.qd, d);
      outer_acc(GB + lay.wk, dk + (size_t)t * g.kvd, x, g.kvd, d);
      outer_acc(GB + lay.wv, dv + (size_t)t * g.kvd, x, g.kvd, d);
      mtv_acc(B + lay.wq, dq + (size_t)t * g.qd, dxt, g.qd, d);
      mtv_acc(B + lay.wk, dk + (size_t)t * g.kvd, dxt, g.kvd, d);
      mtv_acc(B + lay.wv, dv + (size_t)t * g.kvd, dxt, g.kvd, d);
    }
    memcpy(dy, dx, sizeof(double) * (size_t)n * d);
  }
  /* embeddings (policy.cpp:335-344) */
  for (int t = 0; t < n; ++t) {
    double* e = G + lay.token_embed + (size_t)tok[t] * d;
    double* pe = G + lay.pos_embed + (size_t)t * d;
    const double* dxt = dx + (size_t)t * d;
    for (int i = 0; i < d; ++i) {
      e[i] += dxt[i];
      pe[i] += dxt[i];
    }
  }
  for (int64_t i = 0; i < lay.total; ++i) grad[i] += scale * G[i];

  free(G);
  free(dz);
  free(dy);
  free(dx);
  free(dh);
  free(dctx);
  free(dq);
  free(dk);
  free(dv);
  free(du);
  free(da);
  acts_free(&s);
  if (base) acts_free(&sb);
  free(tok);
}

void dor_grad_log_prob_acc(const dor_arch* a, const double* P, const int32_t* prompt, int m,
                           const int32_t* completion, int len, double scale, double* grad) {
  grad_core(a, P, NULL, prompt, m, completion, len, scale, grad, NULL);
}

/* kl_term (policy.cpp:487-522): returns KL(base || current) summed over the completion
 * positions; grad += scale * its gradient w.r.t. the current parameters P. */
double dor_kl_term_acc(const dor_arch* a, const double* P, const double* base, const int32_t* prompt, int m,
                       const int32_t* completion, int len, double scale, double* grad) {
  double v = 0.0;
  grad_core(a, P, base, prompt, m, completion, len, scale, grad, &v);
  return v;
}

/* ------------------------------------------------------ sampling contract */
/* DESIGN.md §4. Every fp32 operation is a single IEEE operation (fmaf, or one
 * rounded * / + with contraction off), so the device evaluates it identically. */

static uint32_t fmix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}

float dor_soft_logf(float x) {
  uint32_t bits;
  memcpy(&bits, &x, 4);
  int e = (int)((bits >> 23) & 0xffu) - 127;
  uint32_t mb = (bits & 0x7fffffu) | 0x3f800000u;
  float mant;
  memcpy(&mant, &mb, 4);
  if (mant > 1.41421356f) {
    mant = mant * 0.5f;
    e += 1;
  }
  const float f = mant - 1.0f;
  const float s = f / (2.0f + f);
  const float z = s * s;
  float p = fmaf(z, 0.11111111f, 0.14285715f);
  p = fmaf(z, p, 0.2f);
  p = fmaf(z, p, 0.33333334f);
  p = fmaf(z, p, 1.0f);
  const float r = (2.0f * s) * p;
  return fmaf((float)e, 0.6931472f, r);
}

uint32_t dor_row_key(uint64_t seq_key, int32_t step) {
  return (uint32_t)(dor_splitmix64(seq_key + 0x9e3779b97f4a7c15ull * (uint64_t)(uint32_t)(step + 1)) >> 32);
}

float dor_gumbel(uint32_t row_key, int32_t token) {
  const uint32_t h = fmix32(((uint32_t)token * 0x9e3779b1u) ^ row_key);
  const float u = (float)((h >> 9) * 2u + 1u) * 0x1.0p-24f;
  const float e = -dor_soft_logf(u);
  return -dor_soft_logf(e);
}

/* Gumbel-max form (kept as an independent reference distribution in the tests). */
int32_t dor_sample_rule_gumbel(const float* logits, int vocab, int bos, float inv_t, uint64_t seq_key,
                               int32_t step) {
  const uint32_t rk = dor_row_key(seq_key, step);
  int32_t best = -1;
  float bs = -INFINITY;
  for (int i = 0; i < vocab; ++i) {
    if (i == bos) continue;
    const float sc = fmaf(logits[i], inv_t, dor_gumbel(rk, i));
    if (best < 0 || sc > bs) {
      bs = sc;
      best = i;
    }
  }
  return best;
}

/* ---- the inverse-CDF contract (device: csrc/rule.cuh, kernels_misc.cu
 * sample_scan_k, gemm_tc.cu epilogue_sample). The reference scans cum += exp(l/T - max)
 * in id order and takes the first id with u*den < cum (policy.cpp:402-422); this is the
 * same scan with the sums organised in 32-id slices and 32 blocks of slices. Every
 * operation is one IEEE rounding (contraction off), so it matches the GPU bit-for-bit. */
#define DOR_SLICE 32
static const float kLOG2E = 1.4426950408889634f;

float dor_sexp2(float x) {
  x = fmaxf(x, -125.f);
  const float fl = floorf(x);
  const float f = x - fl;
  float p = 1.5252734e-05f;
  p = fmaf(p, f, 1.5403530e-04f);
  p = fmaf(p, f, 1.3333558e-03f);
  p = fmaf(p, f, 9.6181291e-03f);
  p = fmaf(p, f, 5.5504109e-02f);
  p = fmaf(p, f, 2.4022651e-01f);
  p = fmaf(p, f, 6.9314718e-01f);
  p = fmaf(p, f, 1.0f);
  int32_t bits;
  memcpy(&bits, &p, 4);
  bits += (int32_t)fl * (1 << 23);
  memcpy(&p, &bits, 4);
  return p;
}

int32_t dor_sample_rule(const float* logits, int vocab, int bos, float inv_t, uint64_t seq_key, int32_t step) {
  const int S = (vocab + DOR_SLICE - 1) / DOR_SLICE;
  float* ms = malloc(sizeof(float) * (size_t)S);
  float* Zs = malloc(sizeof(float) * (size_t)S);
  float M = -FLT_MAX;
  for (int s = 0; s < S; ++s) {
    float x[DOR_SLICE], m = -FLT_MAX, a[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < DOR_SLICE; ++i) {
      const int id = s * DOR_SLICE + i;
      x[i] = (id < vocab && id != bos) ? logits[id] * inv_t : -FLT_MAX;
      m = fmaxf(m, x[i]);
    }
    for (int i = 0; i < DOR_SLICE; ++i) a[i & 3] = a[i & 3] + (x[i] == -FLT_MAX ? 0.f : dor_sexp2((x[i] - m) * kLOG2E));
    ms[s] = m;
    Zs[s] = (a[0] + a[1]) + (a[2] + a[3]);
    M = fmaxf(M, m);
  }
  const int B = (S + 31) / 32;
  float T[32];
  for (int j = 0; j < 32; ++j) {
    T[j] = 0.f;
    for (int s = j * B; s < S && s < (j + 1) * B; ++s) T[j] = T[j] + Zs[s] * dor_sexp2((ms[s] - M) * kLOG2E);
  }
  float total = 0.f;
  for (int j = 0; j < 32; ++j) total = total + T[j];
  const uint32_t rk = dor_row_key(seq_key, step);
  const float u = (float)((rk >> 9) * 2u + 1u) * 0x1.0p-24f;
  const float target = u * total;
  int jb = -1, last_j = -1;
  float base = 0.f, cum = 0.f, last_base = 0.f;
  for (int j = 0; j < 32; ++j) {
    const float prev = cum;
    cum = cum + T[j];
    if (T[j] > 0.f) {
      last_j = j;
      last_base = prev;
    }
    if (jb < 0 && target < cum) {
      jb = j;
      base = prev;
    }
  }
  if (jb < 0) {
    jb = last_j;
    base = last_base;
  }
  int sb = -1, last_s = -1;
  float sbase = 0.f, last_sbase = 0.f, r = base;
  for (int s = jb * B; s < S && s < (jb + 1) * B; ++s) {
    const float Ss = Zs[s] * dor_sexp2((ms[s] - M) * kLOG2E);
    const float prev = r;
    r = r + Ss;
    if (Ss > 0.f) {
      last_s = s;
      last_sbase = prev;
    }
    if (target < r) {
      sb = s;
      sbase = prev;
      break;
    }
  }
  if (sb < 0) {
    sb = last_s;
    sbase = last_sbase;
  }
  const float scale = dor_sexp2((ms[sb] - M) * kLOG2E);
  int tk = -1, last_i = -1;
  r = sbase;
  for (int i = 0; i < DOR_SLICE; ++i) {
    const int id = sb * DOR_SLICE + i;
    if (id >= vocab || id == bos) continue;
    const float e = dor_sexp2((logits[id] * inv_t - ms[sb]) * kLOG2E);
    r = fmaf(e, scale, r);
    last_i = id;
    if (target < r) {
      tk = id;
      break;
    }
  }
  if (tk < 0) tk = last_i;
  free(ms);
  free(Zs);
  return tk;
}

int dor_sample(const dor_arch* a, const double* params, const int32_t* prompt, int m, int max_len,
               double temperature, uint64_t seq_key, int32_t* completion, double* logp) {
  const geo g = geo_of(a);
  int cap = max_len < g.ctx - m ? max_len : g.ctx - m;
  if (cap <= 0) return 0;
  const float inv_t = (float)(1.0 / temperature);
  int32_t* ctx = malloc(sizeof(int32_t) * (size_t)(m + cap));
  memcpy(ctx, prompt, sizeof(int32_t) * (size_t)m);
  double* lg = malloc(sizeof(double) * (size_t)g.V);
  float* lf = malloc(sizeof(float) * (size_t)g.V);
  int len = 0;
  for (int step = 0; step < cap; ++step) {
    dor_next_logits(a, params, ctx, m + step, lg);
    for (int i = 0; i < g.V; ++i) lf[i] = (float)lg[i];
    const int32_t tk = dor_sample_rule(lf, g.V, g.bos, inv_t, seq_key, step);
    completion[len] = tk;
    if (logp) logp[len] = lg[tk] - lse_nobos(lg, g.V, g.bos);
    ++len;
    if (tk == g.eos) break;
    ctx[m + step] = tk;
  }
  free(ctx);
  free(lg);
  free(lf);
  return len;
}

/* ------------------------------------------------------------ advantage */

int dor_advantage_filter(const double* r, int n, int G, int kind, int normalize, double eps,
                         double tau, double* adv, uint8_t* kept, int32_t* kept_idx, int32_t* n_kept) {
  if (n <= 0) return 1;                                   /* advantage.cpp:68 */
  if (kind != 0 && (G <= 0 || n % G != 0)) return 1;     /* :10-11 */
  if (kind == 2 && G < 2) return 1;                       /* :100-101 */
  /* tau = -INFINITY: no filter_by_threshold call at all, kept stays all 1 as
   * group_advantage / single_path_advantage leave it (advantage.cpp:77, :92) */
  const int no_filter = isinf(tau) && tau < 0;
  if (!no_filter && !(tau >= 0.0)) return 1;              /* :136 */
  if (kind == 0) {
    double mean = 0.0;
    for (int i = 0; i < n; ++i) mean += r[i];
    mean /= (double)n;
    for (int i = 0; i < n; ++i) adv[i] = r[i] - mean;
  } else {
    for (int s = 0; s < n; s += G) {
      double sum = 0.0;
      for (int i = s; i < s + G; ++i) sum += r[i];
      if (kind == 1) {
        const double mean = sum / (double)G;
        for (int i = s; i < s + G; ++i) adv[i] = r[i] - mean;
      } else {
        const double den = (double)(G - 1);
        for (int i = s; i < s + G; ++i) adv[i] = r[i] - (sum - r[i]) / den;
      }
    }
  }
  if (normalize) { /* normalize_std: population std of rewards, / (std + eps) (:114-133) */
    const int gs = kind == 0 ? n : G;
    for (int s = 0; s < n; s += gs) {
      double mean = 0.0;
      for (int i = s; i < s + gs; ++i) mean += r[i];
      mean /= (double)gs;
      double var = 0.0;
      for (int i = s; i < s + gs; ++i) var += (r[i] - mean) * (r[i] - mean);
      var /= (double)gs;
      const double den = sqrt(var) + eps;
      for (int i = s; i < s + gs; ++i) adv[i] = adv[i] / den;
    }
  }
  int32_t k = 0;
  for (int i = 0; i < n; ++i) {
    kept[i] = (uint8_t)(no_filter || fabs(adv[i]) > tau);
    if (kept[i]) kept_idx[k++] = i;
  }
  *n_kept = k;
  return 0;
}

/* -------------------------------------------------------------- updates */

void dor_pg_accumulate(const dor_arch* a, const double* params, int n_traj, const int32_t* prompts,
                       const int64_t* p_off, const int32_t* completions, const int64_t* c_off,
                       const double* weight, double* grad) {
  for (int i = 0; i < n_traj; ++i)
    dor_grad_log_prob_acc(a, params, prompts + p_off[i], (int)(p_off[i + 1] - p_off[i]),
                          completions + c_off[i], (int)(c_off[i + 1] - c_off[i]), weight[i], grad);
}

void dor_adam_step(double* p, const double* g, double* m, double* v, int64_t n, int64_t t, double lr,
                   double b1, double b2, double eps) {
  const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
  for (int64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    p[i] += lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
  }
}

void dor_sgd_step(double* p, const double* g, int64_t n, double lr) {
  for (int64_t i = 0; i < n; ++i) p[i] += lr * g[i];
}

/* ------------------------------------------------------ synthetic workload */

static double u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

double dor_synthetic_reward(uint64_t reward_seed, int64_t m, int32_t g) {
  const double pm = u01(dor_derive_seed(reward_seed, "reward_p", (uint64_t)m, 0));
  return u01(dor_derive_seed(reward_seed, "reward", (uint64_t)m, (uint64_t)g)) < pm ? 1.0 : 0.0;
}

void dor_synthetic_prompt(uint64_t seed, int64_t m, int len, int vocab, int bos, int eos,
                          int32_t* out) {
  const uint64_t key = dor_derive_seed(seed, "prompt", (uint64_t)m, 0);
  int j0 = 0;
  if (bos >= 0 && len > 0) out[j0++] = bos;
  const int nspecial = (bos >= 0 ? 1 : 0) + 1;
  const int lo = bos < eos ? bos : eos, hi = bos < eos ? eos : bos;
  for (int j = j0; j < len; ++j) {
    int id = (int)(dor_splitmix64(key + 0x9e3779b97f4a7c15ull * (uint64_t)j) % (uint64_t)(vocab - nspecial));
    /* map to the ascending list of non-special ids */
    if (lo >= 0 && id >= lo) ++id;
    if (id >= hi) ++id;
    out[j] = id;
  }
}
