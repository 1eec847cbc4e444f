/*
 * sxen_oracle.c -- CPU restatement of the reference hot path (see sxen_oracle.h).
 * TEST INFRASTRUCTURE ONLY; parity PINNED against the reference (header comment).
 * Citations are file:line under /root/reference/proj/.
 */
#include "sxen_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ rng */

static const uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

/* include/sxen/rng.hpp:9-14 (splitmix64 finalizer) */
uint64_t sxo_mix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* include/sxen/rng.hpp:16-18 */
uint64_t sxo_hash_combine(uint64_t a, uint64_t b) {
  return sxo_mix64(a ^ (b + kGolden + (a << 6) + (a >> 2)));
}

/* include/sxen/rng.hpp:26-27 */
uint64_t sxo_rng_key(uint64_t seed, int has_stream, uint64_t stream) {
  const uint64_t k = sxo_mix64(seed);
  return has_stream ? sxo_hash_combine(k, stream) : k;
}

/* include/sxen/rng.hpp:31 : draw i (1-based) = mix64(key + phi*i) */
uint64_t sxo_rng_u64(uint64_t key, uint64_t counter) { return sxo_mix64(key + kGolden * counter); }

/* include/sxen/rng.hpp:35 */
double sxo_rng_double(uint64_t key, uint64_t counter) {
  return (double)(sxo_rng_u64(key, counter) >> 11) * 0x1.0p-53;
}

/* include/sxen/rng.hpp:37 */
void sxo_rng_fill_double(uint64_t key, uint64_t first_counter, size_t n, double lo, double hi,
                         double* out) {
  for (size_t i = 0; i < n; ++i) {
    const double u = sxo_rng_double(key, first_counter + i);
    const double span = hi - lo;
    const double prod = span * u;
    out[i] = lo + prod;
  }
}

/* ------------------------------------------------------------------ config */

static int is_pow2(uint32_t v) { return v != 0 && (v & (v - 1)) == 0; }

/* src/encoding.cpp:60-66 */
double sxo_equal_memory_multiplier(int n) {
  return pow((double)(n + 1), (double)(n - 1) / (2.0 * (double)n));
}

/* src/encoding.cpp:68-82 */
uint32_t sxo_level_resolution(const sxo_config* cfg, int level) {
  double r = (double)cfg->base_resolution * pow(cfg->growth, (double)level);
  if (cfg->level_scale == SXO_SCALE_EQUAL_MEMORY && cfg->backend == SXO_BACKEND_SIMPLEX) {
    r *= sxo_equal_memory_multiplier(cfg->dim);
  }
  const double floored = floor(r);
  if (floored < 1.0) return 1;
  if (floored > (double)SXO_MAX_RES) return SXO_MAX_RES + 1;
  return (uint32_t)floored;
}

/* src/encoding.cpp:28-58 ; code = ordinal of the rejected check */
int sxo_validate(const sxo_config* cfg) {
  if (cfg->dim < 1 || cfg->dim > SXO_MAX_DIM) return 1;
  if (cfg->levels < 1) return 2;
  if (!is_pow2(cfg->table_size)) return 3;
  if (cfg->features < 1 || cfg->features > SXO_MAX_FEATURES) return 4;
  if (cfg->base_resolution < 1) return 5;
  if (!(cfg->growth > 1.0) || !isfinite(cfg->growth)) return 6;
  if (sxo_level_resolution(cfg, cfg->levels - 1) > SXO_MAX_RES) return 7;
  return 0;
}

/* src/lattice.cpp:21-30 */
void sxo_skew_constants(int n, double out[3]) {
  const double root = sqrt((double)n + 1.0);
  out[0] = (root - 1.0) / (double)n;
  out[1] = (1.0 - 1.0 / root) / (double)n;
  out[2] = root;
}

/* ------------------------------------------------------------------ lattice */

/* src/lattice.cpp:82-102 : stable descending insertion sort carrying axis ids */
void sxo_subdivide(int n, const double* fracs, uint8_t* perm, double* sorted) {
  for (int i = 0; i < n; ++i) {
    perm[i] = (uint8_t)i;
    sorted[i] = fracs[i];
  }
  for (int i = 1; i < n; ++i) {
    const double v = sorted[i];
    const uint8_t a = perm[i];
    int j = i - 1;
    while (j >= 0 && sorted[j] < v) {
      sorted[j + 1] = sorted[j];
      perm[j + 1] = perm[j];
      --j;
    }
    sorted[j + 1] = v;
    perm[j + 1] = a;
  }
}

/* src/lattice.cpp:139-147 */
void sxo_barycentric(int n, const double* sorted, double* weights) {
  weights[0] = 1.0 - sorted[0];
  for (int i = 1; i < n; ++i) weights[i] = sorted[i - 1] - sorted[i];
  weights[n] = sorted[n - 1];
}

/* ------------------------------------------------------------------ hash */

/* include/sxen/hashing.hpp:16-18 */
static const uint32_t kPrimes[SXO_MAX_DIM] = {1u,          2654435761u, 805459861u,  3674653429u,
                                              2097192037u, 1434869437u, 2165219737u, 4294967291u};

/* src/encoding.cpp:17-20 */
static uint32_t axis_term(int axis, int64_t coord) { return (uint32_t)(uint64_t)coord * kPrimes[axis]; }

/* include/sxen/hashing.hpp:23-29 */
uint32_t sxo_hash_coords(int n, const int64_t* coords) {
  uint32_t h = 0;
  for (int i = 0; i < n; ++i) h ^= axis_term(i, coords[i]);
  return h;
}

/* ------------------------------------------------------------------ tables */

/* src/encoding.cpp:169-176 */
void sxo_init_tables(const sxo_config* cfg, uint64_t seed, float* tables) {
  const size_t per_level = (size_t)cfg->table_size * (size_t)cfg->features;
  for (int l = 0; l < cfg->levels; ++l) {
    const uint64_t key = sxo_rng_key(seed, 1, (uint64_t)l);
    float* t = tables + (size_t)l * per_level;
    for (size_t i = 0; i < per_level; ++i) {
      const double u = sxo_rng_double(key, (uint64_t)i + 1);
      const double span = 1e-4 - (-1e-4);
      const double prod = span * u;
      t[i] = (float)(-1e-4 + prod);
    }
  }
}

/* ------------------------------------------------------------------ gather */

static double clampd(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }
static int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

/* src/encoding.cpp:196-242 */
static int gather_simplex(const sxo_config* cfg, uint32_t nl, const double* x, uint32_t* idx,
                          double* w, int64_t* base_out, uint8_t* perm_out, int* oob_out) {
  const int n = cfg->dim;
  double sc[3];
  sxo_skew_constants(n, sc);
  const double s = (double)nl / sc[2];
  const double one_below = nextafter(1.0, 0.0);

  double y[SXO_MAX_DIM];
  for (int i = 0; i < n; ++i) {
    const double xi = (one_below < x[i]) ? one_below : x[i]; /* std::min(x, one_below) */
    y[i] = xi * s;
  }
  /* skew_in_place, src/lattice.cpp:40-45 */
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += y[i];
  const double shift = sc[0] * sum;
  for (int i = 0; i < n; ++i) y[i] += shift;

  int64_t base[SXO_MAX_DIM];
  double fracs[SXO_MAX_DIM];
  int oob = 0;
  const int64_t limit = (int64_t)nl;
  for (int i = 0; i < n; ++i) {
    const double f = floor(y[i]);
    int64_t b = (int64_t)f;
    if (b < 0 || b + 1 > limit) {
      oob = 1;
      b = clampi(b, 0, limit - 1);
    }
    base[i] = b;
    fracs[i] = clampd(y[i] - (double)b, 0.0, one_below);
  }

  uint8_t perm[SXO_MAX_DIM];
  double sorted[SXO_MAX_DIM];
  double wts[SXO_MAX_DIM + 1];
  sxo_subdivide(n, fracs, perm, sorted);
  sxo_barycentric(n, sorted, wts);

  const uint32_t mask = cfg->table_size - 1u;
  int64_t coords[SXO_MAX_DIM];
  memcpy(coords, base, sizeof(coords));
  uint32_t h = sxo_hash_coords(n, base);
  idx[0] = h & mask;
  w[0] = wts[0];
  for (int k = 0; k < n; ++k) {
    const int axis = perm[k];
    h ^= axis_term(axis, coords[axis]);
    coords[axis] += 1;
    h ^= axis_term(axis, coords[axis]);
    idx[k + 1] = h & mask;
    w[k + 1] = wts[k + 1];
  }
  if (base_out) memcpy(base_out, base, (size_t)n * sizeof(int64_t));
  if (perm_out) memcpy(perm_out, perm, (size_t)n);
  if (oob_out) *oob_out = oob;
  return n + 1;
}

/* src/encoding.cpp:244-285 */
static int gather_grid(const sxo_config* cfg, uint32_t nl, const double* x, uint32_t* idx,
                       double* w, int64_t* base_out, int* oob_out) {
  const int n = cfg->dim;
  const double one_below = nextafter(1.0, 0.0);
  int64_t base[SXO_MAX_DIM];
  double w0[SXO_MAX_DIM], w1[SXO_MAX_DIM];
  int oob = 0;
  const int64_t limit = (int64_t)nl;
  for (int i = 0; i < n; ++i) {
    const double xi = (one_below < x[i]) ? one_below : x[i];
    const double y = xi * (double)nl;
    const double f = floor(y);
    int64_t b = (int64_t)f;
    if (b < 0 || b + 1 > limit) {
      oob = 1;
      b = clampi(b, 0, limit - 1);
    }
    const double frac = clampd(y - (double)b, 0.0, one_below);
    base[i] = b;
    w1[i] = frac;
    w0[i] = 1.0 - frac;
  }
  const int corners = 1 << n;
  int64_t c[SXO_MAX_DIM];
  for (int m = 0; m < corners; ++m) {
    double weight = 1.0;
    for (int d = 0; d < n; ++d) {
      const int bit = (m >> d) & 1;
      c[d] = base[d] + bit;
      weight *= bit ? w1[d] : w0[d];
    }
    idx[m] = sxo_hash_coords(n, c) & (cfg->table_size - 1u);
    w[m] = weight;
  }
  if (base_out) memcpy(base_out, base, (size_t)n * sizeof(int64_t));
  if (oob_out) *oob_out = oob;
  return corners;
}

int sxo_gather(const sxo_config* cfg, uint32_t res, const double* x, uint32_t* idx, double* w,
               int64_t* base_out, uint8_t* perm_out, int* oob) {
  if (cfg->backend == SXO_BACKEND_SIMPLEX) return gather_simplex(cfg, res, x, idx, w, base_out, perm_out, oob);
  return gather_grid(cfg, res, x, idx, w, base_out, oob);
}

static int vertex_count(const sxo_config* cfg) {
  return cfg->backend == SXO_BACKEND_SIMPLEX ? cfg->dim + 1 : (1 << cfg->dim);
}

/* src/encoding.cpp:183-194 : !(x >= 0 && x <= 1) rejects NaN too */
static int input_ok(const sxo_config* cfg, const double* x) {
  for (int i = 0; i < cfg->dim; ++i) {
    if (!(x[i] >= 0.0 && x[i] <= 1.0)) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------ encode */

/* src/encoding.cpp:295-315 */
long sxo_encode(const sxo_config* cfg, const float* tables, const double* x, size_t n_samples,
                float* out, uint64_t* counters) {
  const int n = cfg->dim, L = cfg->levels, F = cfg->features;
  const size_t per_level = (size_t)cfg->table_size * (size_t)F;
  uint32_t res[64];
  uint32_t* resp = res;
  if (L > 64) resp = (uint32_t*)malloc((size_t)L * sizeof(uint32_t));
  for (int l = 0; l < L; ++l) resp[l] = sxo_level_resolution(cfg, l);
  uint32_t idx[1 << SXO_MAX_DIM];
  double w[1 << SXO_MAX_DIM];
  double acc[SXO_MAX_FEATURES];
  long bad = -1;
  for (size_t s = 0; s < n_samples; ++s) {
    const double* xs = x + s * (size_t)n;
    if (!input_ok(cfg, xs)) {
      bad = (long)s;
      break;
    }
    float* dst = out + s * (size_t)L * (size_t)F;
    for (int l = 0; l < L; ++l) {
      int oob = 0;
      const int count = sxo_gather(cfg, resp[l], xs, idx, w, NULL, NULL, &oob);
      if (counters) {
        counters[0] += (uint64_t)count;
        counters[1] += (uint64_t)oob;
      }
      for (int f = 0; f < F; ++f) acc[f] = 0.0;
      const float* tab = tables + (size_t)l * per_level;
      for (int i = 0; i < count; ++i) {
        const double wi = w[i];
        const float* entry = tab + (size_t)idx[i] * (size_t)F;
        for (int f = 0; f < F; ++f) {
          const double prod = wi * (double)entry[f];
          acc[f] += prod;
        }
      }
      for (int f = 0; f < F; ++f) dst[(size_t)l * (size_t)F + (size_t)f] = (float)acc[f];
    }
  }
  if (resp != res) free(resp);
  return bad;
}

long sxo_encode_debug(const sxo_config* cfg, const double* x, size_t n_samples, uint32_t* idx,
                      double* w, int64_t* base, uint8_t* perm) {
  const int n = cfg->dim, L = cfg->levels;
  const int V = vertex_count(cfg);
  for (size_t s = 0; s < n_samples; ++s) {
    const double* xs = x + s * (size_t)n;
    if (!input_ok(cfg, xs)) return (long)s;
    for (int l = 0; l < L; ++l) {
      const size_t o = (s * (size_t)L + (size_t)l);
      sxo_gather(cfg, sxo_level_resolution(cfg, l), xs, idx + o * (size_t)V, w + o * (size_t)V,
                 base ? base + o * (size_t)n : NULL, perm ? perm + o * (size_t)n : NULL, NULL);
    }
  }
  return -1;
}

/* src/encoding.cpp:317-335, EncoderGradient::add :110-120 */
long sxo_encode_backward(const sxo_config* cfg, const double* x, const double* upstream,
                         size_t n_samples, double* grad, uint8_t* touched) {
  const int n = cfg->dim, L = cfg->levels, F = cfg->features;
  const size_t T = cfg->table_size;
  uint32_t idx[1 << SXO_MAX_DIM];
  double w[1 << SXO_MAX_DIM];
  uint32_t* res = (uint32_t*)malloc((size_t)L * sizeof(uint32_t));
  for (int l = 0; l < L; ++l) res[l] = sxo_level_resolution(cfg, l);
  long bad = -1;
  for (size_t s = 0; s < n_samples; ++s) {
    const double* xs = x + s * (size_t)n;
    if (!input_ok(cfg, xs)) {
      bad = (long)s;
      break;
    }
    const double* up = upstream + s * (size_t)L * (size_t)F;
    for (int l = 0; l < L; ++l) {
      const int count = sxo_gather(cfg, res[l], xs, idx, w, NULL, NULL, NULL);
      for (int i = 0; i < count; ++i) {
        if (touched) touched[(size_t)l * T + idx[i]] = 1;
        double* dst = grad + ((size_t)l * T + idx[i]) * (size_t)F;
        for (int f = 0; f < F; ++f) {
          const double prod = w[i] * up[(size_t)l * (size_t)F + (size_t)f];
          dst[f] += prod;
        }
      }
    }
  }
  free(res);
  return bad;
}

/* ------------------------------------------------------------------ MLP */

static int layer_count(const sxo_mlp_config* c) { return c->hidden_layers + 1; }
static int layer_in(const sxo_mlp_config* c, int l) { return l == 0 ? c->input_width : c->hidden_width; }
static int layer_out(const sxo_mlp_config* c, int l) {
  return l == layer_count(c) - 1 ? c->output_width : c->hidden_width;
}

/* src/mlp.cpp:35-52 */
int sxo_mlp_validate(const sxo_mlp_config* c) {
  const int kMaxWidth = 1 << 14;
  if (c->input_width < 1 || c->input_width > kMaxWidth) return 1;
  if (c->output_width < 1 || c->output_width > kMaxWidth) return 2;
  if (c->hidden_layers < 0) return 3;
  if (c->hidden_layers > 0 && (c->hidden_width < 1 || c->hidden_width > kMaxWidth)) return 4;
  return 0;
}

/* src/mlp.cpp:19-32 : per layer, weights (out x in, row-major) then biases */
size_t sxo_mlp_param_count(const sxo_mlp_config* c) {
  size_t total = 0;
  for (int l = 0; l < layer_count(c); ++l) {
    total += (size_t)layer_in(c, l) * (size_t)layer_out(c, l) + (size_t)layer_out(c, l);
  }
  return total;
}

size_t sxo_mlp_act_width(const sxo_mlp_config* c) {
  size_t w = (size_t)c->input_width;
  for (int l = 0; l < layer_count(c); ++l) w += (size_t)layer_out(c, l);
  return w;
}

/* src/mlp.cpp:106-113 */
void sxo_mlp_init(const sxo_mlp_config* c, uint64_t seed, float* params) {
  size_t off = 0;
  for (int l = 0; l < layer_count(c); ++l) {
    const uint64_t key = sxo_rng_key(seed, 1, (uint64_t)l);
    const double bound = sqrt(6.0 / (double)layer_in(c, l));
    const size_t nw = (size_t)layer_in(c, l) * (size_t)layer_out(c, l);
    for (size_t i = 0; i < nw; ++i) {
      const double u = sxo_rng_double(key, (uint64_t)i + 1);
      const double span = bound - (-bound);
      const double prod = span * u;
      params[off + i] = (float)(-bound + prod);
    }
    off += nw;
    for (int o = 0; o < layer_out(c, l); ++o) params[off + (size_t)o] = 0.0f;
    off += (size_t)layer_out(c, l);
  }
}

/* src/mlp.cpp:137-162 */
void sxo_mlp_forward(const sxo_mlp_config* c, const float* params, const float* input,
                     size_t n_samples, float* acts, float* out) {
  const size_t aw = sxo_mlp_act_width(c);
  for (size_t s = 0; s < n_samples; ++s) {
    float* a = acts + s * aw;
    memcpy(a, input + s * (size_t)c->input_width, (size_t)c->input_width * sizeof(float));
    const float* src = a;
    float* dst = a + c->input_width;
    size_t poff = 0;
    for (int l = 0; l < layer_count(c); ++l) {
      const int in = layer_in(c, l), ow = layer_out(c, l);
      const float* w = params + poff;
      const float* b = w + (size_t)in * (size_t)ow;
      const int relu = l + 1 < layer_count(c);
      for (int o = 0; o < ow; ++o) {
        double acc = (double)b[o];
        const float* row = w + (size_t)o * (size_t)in;
        for (int i = 0; i < in; ++i) {
          const double prod = (double)row[i] * (double)src[i];
          acc += prod;
        }
        if (relu && acc < 0.0) acc = 0.0;
        dst[o] = (float)acc;
      }
      poff += (size_t)in * (size_t)ow + (size_t)ow;
      src = dst;
      dst += ow;
    }
    if (out) memcpy(out + s * (size_t)c->output_width, src, (size_t)c->output_width * sizeof(float));
  }
}

/* src/mlp.cpp:164-202 */
void sxo_mlp_backward(const sxo_mlp_config* c, const float* params, const float* acts,
                      const double* upstream, size_t n_samples, double* grad, double* input_grad) {
  const size_t aw = sxo_mlp_act_width(c);
  const int LC = layer_count(c);
  int maxw = c->input_width;
  for (int l = 0; l < LC; ++l)
    if (layer_out(c, l) > maxw) maxw = layer_out(c, l);
  double* cur = (double*)malloc((size_t)maxw * sizeof(double));
  double* nxt = (double*)malloc((size_t)maxw * sizeof(double));
  size_t* w_off = (size_t*)malloc((size_t)LC * sizeof(size_t));
  size_t* a_off = (size_t*)malloc(((size_t)LC + 1) * sizeof(size_t));
  size_t po = 0, ao = 0;
  for (int l = 0; l < LC; ++l) {
    w_off[l] = po;
    po += (size_t)layer_in(c, l) * (size_t)layer_out(c, l) + (size_t)layer_out(c, l);
    a_off[l] = ao;
    ao += (size_t)layer_in(c, l);
  }
  a_off[LC] = ao;
  for (size_t s = 0; s < n_samples; ++s) {
    const float* a = acts + s * aw;
    for (int o = 0; o < c->output_width; ++o) cur[o] = upstream[s * (size_t)c->output_width + (size_t)o];
    for (int l = LC - 1; l >= 0; --l) {
      const int in = layer_in(c, l), ow = layer_out(c, l);
      const float* w = params + w_off[l];
      const float* src = a + a_off[l];
      double* dw = grad + w_off[l];
      double* db = dw + (size_t)in * (size_t)ow;
      for (int o = 0; o < ow; ++o) {
        const double d = cur[o];
        db[o] += d;
        double* dw_row = dw + (size_t)o * (size_t)in;
        for (int i = 0; i < in; ++i) {
          const double prod = d * (double)src[i];
          dw_row[i] += prod;
        }
      }
      double* downstream = nxt;
      for (int i = 0; i < in; ++i) {
        double acc = 0.0;
        for (int o = 0; o < ow; ++o) {
          const double prod = cur[o] * (double)w[(size_t)o * (size_t)in + (size_t)i];
          acc += prod;
        }
        if (l > 0 && src[i] <= 0.0f) acc = 0.0;
        downstream[i] = acc;
      }
      if (l > 0) {
        double* t = cur;
        cur = nxt;
        nxt = t;
      } else if (input_grad) {
        memcpy(input_grad + s * (size_t)c->input_width, nxt, (size_t)in * sizeof(double));
      }
    }
  }
  free(cur);
  free(nxt);
  free(w_off);
  free(a_off);
}

/* ------------------------------------------------------------------ optimizers */

/* src/optimizer.cpp:9-15 */
static double adam_delta(double g, double* m, double* v, const sxo_adam_config* cfg, double bc1,
                         double bc2) {
  const double a = cfg->beta1 * *m;
  const double b = (1.0 - cfg->beta1) * g;
  *m = a + b;
  const double c = cfg->beta2 * *v;
  const double d = (1.0 - cfg->beta2) * g * g;
  *v = c + d;
  const double m_hat = *m / bc1;
  const double v_hat = *v / bc2;
  return -cfg->lr * m_hat / (sqrt(v_hat) + cfg->epsilon);
}

/* src/optimizer.cpp:25-41 */
long sxo_adam_step(float* params, const double* grads, double* m, double* v, size_t n, int64_t t,
                   const sxo_adam_config* cfg) {
  const double bc1 = 1.0 - pow(cfg->beta1, (double)t);
  const double bc2 = 1.0 - pow(cfg->beta2, (double)t);
  for (size_t i = 0; i < n; ++i) {
    const double g = grads[i];
    if (!isfinite(g)) return (long)i;
    params[i] = (float)((double)params[i] + adam_delta(g, &m[i], &v[i], cfg, bc1, bc2));
  }
  return -1;
}

/* src/optimizer.cpp:54-84 (dense scan of the touched map instead of the touch-order list:
 * per-entry updates are independent, so visiting order does not change results) */
long sxo_sparse_adam_step(const sxo_config* cfg, float* tables, const double* grad,
                          const uint8_t* touched, double* m, double* v, int64_t t,
                          const sxo_adam_config* acfg) {
  const double bc1 = 1.0 - pow(acfg->beta1, (double)t);
  const double bc2 = 1.0 - pow(acfg->beta2, (double)t);
  const size_t T = cfg->table_size;
  const int F = cfg->features;
  for (int l = 0; l < cfg->levels; ++l) {
    for (size_t r = 0; r < T; ++r) {
      if (!touched[(size_t)l * T + r]) continue;
      for (int f = 0; f < F; ++f) {
        const size_t i = ((size_t)l * T + r) * (size_t)F + (size_t)f;
        const double g = grad[i];
        if (!isfinite(g)) return (long)i;
        tables[i] = (float)((double)tables[i] + adam_delta(g, &m[i], &v[i], acfg, bc1, bc2));
      }
    }
  }
  return -1;
}

/* ------------------------------------------------------------------ training grads */

/* src/trainer.cpp:20-49 (run_chunk) + loss reduction :118-120, aux_dims = 0 */
double sxo_train_grads(const sxo_config* ecfg, const sxo_mlp_config* mcfg, const float* tables,
                       const float* mlp_params, const double* coords, const double* targets,
                       size_t n_samples, size_t global_batch, double* table_grad, uint8_t* touched,
                       double* mlp_grad, double* sample_loss) {
  const int enc_w = ecfg->levels * ecfg->features;
  const int out_w = mcfg->output_width;
  const size_t aw = sxo_mlp_act_width(mcfg);
  float* input = (float*)malloc((size_t)enc_w * sizeof(float));
  float* acts = (float*)malloc(aw * sizeof(float));
  double* upstream = (double*)malloc((size_t)out_w * sizeof(double));
  double* input_grad = (double*)malloc((size_t)mcfg->input_width * sizeof(double));
  const double upstream_scale = 2.0 / (double)(global_batch * (size_t)out_w);
  double total = 0.0;
  for (size_t s = 0; s < n_samples; ++s) {
    const double* x = coords + s * (size_t)ecfg->dim;
    sxo_encode(ecfg, tables, x, 1, input, NULL);
    sxo_mlp_forward(mcfg, mlp_params, input, 1, acts, NULL);
    const float* pred = acts + (aw - (size_t)out_w);
    double loss = 0.0;
    for (int o = 0; o < out_w; ++o) {
      const double e = (double)pred[o] - targets[s * (size_t)out_w + (size_t)o];
      const double sq = e * e;
      loss += sq;
      upstream[o] = upstream_scale * e;
    }
    if (sample_loss) sample_loss[s] = loss;
    total += loss;
    sxo_mlp_backward(mcfg, mlp_params, acts, upstream, 1, mlp_grad, input_grad);
    sxo_encode_backward(ecfg, x, input_grad, 1, table_grad, touched);
  }
  free(input);
  free(acts);
  free(upstream);
  free(input_grad);
  return total / ((double)global_batch * (double)out_w);
}

/* ------------------------------------------------------------------ CPU baseline timing */

typedef struct {
  const sxo_config* cfg;
  const float* tables;
  const double* x;
  const double* upstream;
  size_t begin, end;
  double* grad;
  uint8_t* touched;
  float* out;
} bench_job;

static void* bench_worker(void* p) {
  bench_job* j = (bench_job*)p;
  const size_t LF = (size_t)j->cfg->levels * (size_t)j->cfg->features;
  for (size_t s = j->begin; s < j->end; ++s) {
    sxo_encode(j->cfg, j->tables, j->x + s * (size_t)j->cfg->dim, 1, j->out, NULL);
    sxo_encode_backward(j->cfg, j->x + s * (size_t)j->cfg->dim, j->upstream + s * LF, 1, j->grad,
                        j->touched);
  }
  return NULL;
}

double sxo_bench_fwd_bwd(const sxo_config* cfg, const float* tables, const double* x,
                         const double* upstream, size_t n_samples, int threads) {
  if (threads < 1) threads = 1;
  const size_t per = (size_t)cfg->levels * (size_t)cfg->table_size;
  bench_job* jobs = (bench_job*)calloc((size_t)threads, sizeof(bench_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const size_t chunk = (n_samples + (size_t)threads - 1) / (size_t)threads;
  for (int t = 0; t < threads; ++t) {
    jobs[t].cfg = cfg;
    jobs[t].tables = tables;
    jobs[t].x = x;
    jobs[t].upstream = upstream;
    jobs[t].begin = (size_t)t * chunk < n_samples ? (size_t)t * chunk : n_samples;
    jobs[t].end = jobs[t].begin + chunk < n_samples ? jobs[t].begin + chunk : n_samples;
    jobs[t].grad = (double*)calloc(per * (size_t)cfg->features, sizeof(double));
    jobs[t].touched = (uint8_t*)calloc(per, 1);
    jobs[t].out = (float*)calloc((size_t)cfg->levels * (size_t)cfg->features, sizeof(float));
  }
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, bench_worker, &jobs[t]);
  bench_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  for (int t = 0; t < threads; ++t) {
    free(jobs[t].grad);
    free(jobs[t].touched);
    free(jobs[t].out);
  }
  free(jobs);
  free(tids);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
