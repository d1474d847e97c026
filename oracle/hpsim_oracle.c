/*
 * hpsim_oracle.c — CPU restatement of the reference hot path (TEST
 * INFRASTRUCTURE ONLY; see hpsim_oracle.h). Every function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/core/. Loop nests and accumulation orders follow the
 * reference exactly; OpenMP only splits loops over independent outputs, so
 * per-element summation order (and therefore every bit) is unchanged.
 */
#include "hpsim_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* or_last_error(void) { return g_err; }

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ---------------------------------------------------------------- rng
 * std::mt19937_64 (C++ [rand.eng.mers], default parameters) and the
 * reference's GaussianSampler (include/hpsim/rng.hpp:26-56). */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int i;
  double spare;
  int have_spare;
} gauss_t;

static void mt_seed(gauss_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = MT_N;
  g->have_spare = 0;
  g->spare = 0.0;
}

static uint64_t mt_next(gauss_t* g) {
  if (g->i >= MT_N) {
    for (int k = 0; k < MT_N; ++k) {
      uint64_t x = (g->mt[k] & 0xFFFFFFFF80000000ULL) | (g->mt[(k + 1) % MT_N] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[k] = g->mt[(k + MT_M) % MT_N] ^ xa;
    }
    g->i = 0;
  }
  uint64_t x = g->mt[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:45-47 */
static double uniform01(gauss_t* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }

/* rng.hpp:30-43 */
static double gauss_next(gauss_t* g) {
  if (g->have_spare) {
    g->have_spare = 0;
    return g->spare;
  }
  const double u1 = 1.0 - uniform01(g);
  const double u2 = uniform01(g);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.14159265358979323846 * u2;
  g->spare = radius * sin(angle);
  g->have_spare = 1;
  return radius * cos(angle);
}

void or_gaussian_fill(uint64_t seed, double* out, int64_t n) {
  gauss_t g;
  mt_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = gauss_next(&g);
}

void or_uniform_u64(uint64_t seed, uint64_t* out, int64_t n) {
  gauss_t g;
  mt_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&g);
}

/* ---------------------------------------------------------------- geometry
 * model.cpp:25-35 (exact division) + floor-mode superset. */
static int conv_out_dim(int64_t in, int k, int s, int p, int floor_mode, int64_t* out) {
  const int64_t num = in + 2 * (int64_t)p - k;
  if (num < 0 || (!floor_mode && num % s != 0)) return 0;
  *out = num / s + 1;
  return 1;
}

static int pool_out_dim(int64_t in, int k, int s, int64_t* out) {
  if (in < k) return 0;
  *out = (in - k) / s + 1;
  return 1;
}

typedef struct {
  int64_t c, h, w;      /* stage input */
  int64_t f, ho, wo;    /* conv output */
  int64_t hp, wp;       /* stage output (after pool, == ho/wo without pool) */
} geom_t;

/* ModelSpec::validate (model.cpp:39-91) */
static int compute_geometry(const or_model_spec* s, geom_t* g) {
  if (s->n_conv < 1) return fail(1, "model.conv_layers: at least one conv layer required");
  if (s->n_fc < 1) return fail(1, "model.fc_layers: at least one fc layer required");
  for (int i = 0; i < 3; ++i)
    if (s->input_shape[i] <= 0) return fail(1, "model.input_shape: dimensions must be positive");
  int64_t c = s->input_shape[0], h = s->input_shape[1], w = s->input_shape[2];
  for (int i = 0; i < s->n_conv; ++i) {
    const or_conv_layer* l = &s->conv[i];
    if (l->in_channels != c)
      return fail(1, "model.conv_layers[%d].in_channels: expected %lld, got %lld", i, (long long)c,
                  (long long)l->in_channels);
    if (l->out_channels <= 0 || l->kernel <= 0 || l->stride <= 0 || l->pad < 0)
      return fail(1,
                  "model.conv_layers[%d]: out_channels/kernel/stride must be positive, pad "
                  "non-negative",
                  i);
    geom_t* gi = g ? &g[i] : NULL;
    int64_t ho, wo;
    if (!conv_out_dim(h, l->kernel, l->stride, l->pad, l->floor_mode, &ho))
      return fail(1, "model.conv_layers[%d] (height): output dimension (%lld+2*%d-%d)/%d+1 is not a positive integer",
                  i, (long long)h, l->pad, l->kernel, l->stride);
    if (!conv_out_dim(w, l->kernel, l->stride, l->pad, l->floor_mode, &wo))
      return fail(1, "model.conv_layers[%d] (width): output dimension (%lld+2*%d-%d)/%d+1 is not a positive integer",
                  i, (long long)w, l->pad, l->kernel, l->stride);
    int64_t hp = ho, wp = wo;
    if (l->lrn_size < 0) return fail(1, "model.conv_layers[%d].lrn_size: must be >= 0", i);
    if (l->pool_kernel > 0) {
      if (l->pool_stride <= 0) return fail(1, "model.conv_layers[%d].pool_stride: must be positive", i);
      if (!pool_out_dim(ho, l->pool_kernel, l->pool_stride, &hp) ||
          !pool_out_dim(wo, l->pool_kernel, l->pool_stride, &wp))
        return fail(1, "model.conv_layers[%d].pool_kernel: larger than the conv output", i);
    }
    if (gi) {
      gi->c = c; gi->h = h; gi->w = w;
      gi->f = l->out_channels; gi->ho = ho; gi->wo = wo; gi->hp = hp; gi->wp = wp;
    }
    c = l->out_channels;
    h = hp;
    w = wp;
  }
  int64_t dim = c * h * w;
  for (int i = 0; i < s->n_fc; ++i) {
    const or_fc_layer* l = &s->fc[i];
    if (l->in_dim != dim)
      return fail(1, "model.fc_layers[%d].in_dim: expected %lld (flattened preceding output), got %lld", i,
                  (long long)dim, (long long)l->in_dim);
    if (l->out_dim <= 0) return fail(1, "model.fc_layers[%d].out_dim: must be positive", i);
    dim = l->out_dim;
  }
  if (s->num_classes <= 0) return fail(1, "model.num_classes: must be positive");
  if (dim != s->num_classes)
    return fail(1, "model.fc_layers: last out_dim %lld does not match num_classes %lld", (long long)dim,
                (long long)s->num_classes);
  return 0;
}

int or_validate(const or_model_spec* spec) { return compute_geometry(spec, NULL); }

int or_conv_output_sizes(const or_model_spec* spec, int64_t* hw) {
  geom_t* g = calloc((size_t)spec->n_conv, sizeof(geom_t));
  int rc = compute_geometry(spec, g);
  if (rc == 0)
    for (int i = 0; i < spec->n_conv; ++i) {
      hw[2 * i] = g[i].hp;
      hw[2 * i + 1] = g[i].wp;
    }
  free(g);
  return rc;
}

int64_t or_flattened_conv_size(const or_model_spec* spec) {
  geom_t* g = calloc((size_t)spec->n_conv, sizeof(geom_t));
  int64_t r = -1;
  if (compute_geometry(spec, g) == 0) {
    const geom_t* l = &g[spec->n_conv - 1];
    r = l->f * l->hp * l->wp;
  }
  free(g);
  return r;
}

/* ---------------------------------------------------------------- kernels */

/* conv2d_forward_impl (tensor.cpp:419-451) */
static void conv_fwd(const double* x, const double* k, double* y, int64_t B, int64_t C, int64_t H,
                     int64_t W, int64_t F, int64_t R, int64_t S, int64_t OH, int64_t OW, int stride,
                     int pad) {
  const int64_t out_hw = OH * OW;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < B; ++b)
    for (int64_t f = 0; f < F; ++f)
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow) {
          double acc = 0;
          for (int64_t c = 0; c < C; ++c)
            for (int64_t r = 0; r < R; ++r) {
              const int64_t h = oh * stride - pad + r;
              if (h < 0 || h >= H) continue;
              for (int64_t s = 0; s < S; ++s) {
                const int64_t w = ow * stride - pad + s;
                if (w < 0 || w >= W) continue;
                acc += x[((b * C + c) * H + h) * W + w] * k[((f * C + c) * R + r) * S + s];
              }
            }
          y[(b * F + f) * out_hw + oh * OW + ow] = acc;
        }
}

/* conv2d_backward_impl (tensor.cpp:453-516). gx may be NULL (conv1: the
 * reference computes and discards it, model.cpp:277-280). */
static void conv_bwd(const double* x, const double* k, const double* gy, double* gx, double* gk,
                     int64_t B, int64_t C, int64_t H, int64_t W, int64_t F, int64_t R, int64_t S,
                     int64_t OH, int64_t OW, int stride, int pad) {
  const int64_t out_hw = OH * OW;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t f = 0; f < F; ++f)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t r = 0; r < R; ++r)
        for (int64_t s = 0; s < S; ++s) {
          double acc = 0;
          for (int64_t b = 0; b < B; ++b)
            for (int64_t oh = 0; oh < OH; ++oh) {
              const int64_t h = oh * stride - pad + r;
              if (h < 0 || h >= H) continue;
              for (int64_t ow = 0; ow < OW; ++ow) {
                const int64_t w = ow * stride - pad + s;
                if (w < 0 || w >= W) continue;
                acc += gy[(b * F + f) * out_hw + oh * OW + ow] * x[((b * C + c) * H + h) * W + w];
              }
            }
          gk[((f * C + c) * R + r) * S + s] = acc;
        }
  if (!gx) return;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < B; ++b)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t h = 0; h < H; ++h)
        for (int64_t w = 0; w < W; ++w) {
          double acc = 0;
          for (int64_t f = 0; f < F; ++f)
            for (int64_t r = 0; r < R; ++r) {
              const int64_t oh_num = h + pad - r;
              if (oh_num < 0 || oh_num % stride != 0) continue;
              const int64_t oh = oh_num / stride;
              if (oh >= OH) continue;
              for (int64_t s = 0; s < S; ++s) {
                const int64_t ow_num = w + pad - s;
                if (ow_num < 0 || ow_num % stride != 0) continue;
                const int64_t ow = ow_num / stride;
                if (ow >= OW) continue;
                acc += gy[(b * F + f) * out_hw + oh * OW + ow] * k[((f * C + c) * R + r) * S + s];
              }
            }
          gx[((b * C + c) * H + h) * W + w] = acc;
        }
}

int or_conv2d_forward(const double* x, int64_t B, int64_t C, int64_t H, int64_t W, const double* k,
                      int64_t F, int64_t R, int64_t S, int stride, int pad, int floor_mode,
                      double* y) {
  int64_t OH, OW;
  if (!conv_out_dim(H, (int)R, stride, pad, floor_mode, &OH) ||
      !conv_out_dim(W, (int)S, stride, pad, floor_mode, &OW))
    return fail(1, "conv2d: output dimension (H+2*pad-R)/stride+1 is not a positive integer");
  conv_fwd(x, k, y, B, C, H, W, F, R, S, OH, OW, stride, pad);
  return 0;
}

int or_conv2d_backward(const double* x, int64_t B, int64_t C, int64_t H, int64_t W,
                       const double* k, int64_t F, int64_t R, int64_t S, int stride, int pad,
                       int floor_mode, const double* gy, double* gx, double* gk) {
  int64_t OH, OW;
  if (!conv_out_dim(H, (int)R, stride, pad, floor_mode, &OH) ||
      !conv_out_dim(W, (int)S, stride, pad, floor_mode, &OW))
    return fail(1, "conv2d: output dimension (H+2*pad-R)/stride+1 is not a positive integer");
  conv_bwd(x, k, gy, gx, gk, B, C, H, W, F, R, S, OH, OW, stride, pad);
  return 0;
}

/* matmul_impl (tensor.cpp:254-269): c[m x n] = a[m x p] b[p x n] */
void or_matmul(const double* a, const double* b, double* c, int64_t m, int64_t p, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (int64_t k = 0; k < p; ++k) acc += a[i * p + k] * b[k * n + j];
      c[i * n + j] = acc;
    }
}

/* matmul_tn_impl (tensor.cpp:271-287): c[m x n] = a^T b, a is [p x m] */
void or_matmul_tn(const double* a, const double* b, double* c, int64_t p, int64_t m, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (int64_t k = 0; k < p; ++k) acc += a[k * m + i] * b[k * n + j];
      c[i * n + j] = acc;
    }
}

/* matmul_nt_impl (tensor.cpp:289-305): c[m x n] = a b^T, b is [n x p] */
void or_matmul_nt(const double* a, const double* b, double* c, int64_t m, int64_t p, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (int64_t k = 0; k < p; ++k) acc += a[i * p + k] * b[j * p + k];
      c[i * n + j] = acc;
    }
}

/* logistic_xent_impl (tensor.cpp:587-614) */
int or_logistic_xent(const double* z, const double* t, int64_t B, int64_t L, double* grad,
                     double* loss_out) {
  if (B == 0) return fail(2, "logistic_xent: empty batch");
  const double inv_b = 1.0 / (double)B;
  double loss = 0.0;
  for (int64_t i = 0; i < B * L; ++i) {
    const double zi = z[i], ti = t[i];
    if (ti < 0.0 || ti > 1.0)
      return fail(3, "logistic_xent: target %f outside [0,1] at flat index %lld", ti, (long long)i);
    const double softplus_neg = (-zi > 0.0 ? -zi : 0.0) + log1p(exp(-fabs(zi)));
    loss += softplus_neg + (1.0 - ti) * zi;
    const double sigma = zi >= 0.0 ? 1.0 / (1.0 + exp(-zi)) : exp(zi) / (1.0 + exp(zi));
    grad[i] = inv_b * (sigma - ti);
  }
  *loss_out = loss * inv_b;
  return 0;
}

/* momentum_update (optimizer.cpp:19-31) via Tensor::scale / add_scaled / add
 * (tensor.cpp:195-229), double storage. */
void or_momentum_update(double* w, double* delta, const double* g, int64_t n, double lr,
                        double momentum, double weight_decay) {
  const double s1 = -lr, s2 = -lr * weight_decay;
  for (int64_t i = 0; i < n; ++i) delta[i] *= momentum;
  for (int64_t i = 0; i < n; ++i) delta[i] += s1 * g[i];
  for (int64_t i = 0; i < n; ++i) delta[i] += s2 * w[i];
  for (int64_t i = 0; i < n; ++i) w[i] += delta[i];
}

/* Same, float storage: scalars formed in double, rounded to float once
 * (tensor.cpp:197, 222). */
void or_momentum_update_f32(float* w, float* delta, const float* g, int64_t n, double lr,
                            double momentum, double weight_decay) {
  const float fm = (float)momentum, s1 = (float)(-lr), s2 = (float)(-lr * weight_decay);
  for (int64_t i = 0; i < n; ++i) delta[i] *= fm;
  for (int64_t i = 0; i < n; ++i) delta[i] += s1 * g[i];
  for (int64_t i = 0; i < n; ++i) delta[i] += s2 * w[i];
  for (int64_t i = 0; i < n; ++i) w[i] += delta[i];
}

/* ---- extensions (not in the reference; parity unpinned, torch-checked) --- */

/* Overlapping max-pool, floor mode, no padding. Ties: first maximum in
 * row-major window order (strict >); NaN wins (torch CPU convention). idx is
 * the argmax's h*W+w inside its (b,c) plane. */
void or_maxpool_forward(const double* x, int64_t B, int64_t C, int64_t H, int64_t W, int k, int s,
                        double* y, int32_t* idx) {
  const int64_t OH = (H - k) / s + 1, OW = (W - k) / s + 1;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < B; ++b)
    for (int64_t c = 0; c < C; ++c) {
      const double* xp = x + (b * C + c) * H * W;
      for (int64_t oh = 0; oh < OH; ++oh)
        for (int64_t ow = 0; ow < OW; ++ow) {
          int64_t best_i = (oh * s) * W + ow * s;
          double best = -INFINITY;
          for (int r = 0; r < k; ++r)
            for (int q = 0; q < k; ++q) {
              const int64_t ii = (oh * s + r) * W + (ow * s + q);
              const double v = xp[ii];
              if (v > best || isnan(v)) {
                best = v;
                best_i = ii;
                if (isnan(v)) goto done;
              }
            }
        done:
          y[((b * C + c) * OH + oh) * OW + ow] = best;
          idx[((b * C + c) * OH + oh) * OW + ow] = (int32_t)best_i;
        }
    }
}

/* Gradient routed to each window's argmax, accumulated over windows in
 * row-major output order. */
void or_maxpool_backward(const double* gy, const int32_t* idx, int64_t B, int64_t C, int64_t H,
                         int64_t W, int k, int s, double* gx) {
  const int64_t OH = (H - k) / s + 1, OW = (W - k) / s + 1;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < B; ++b)
    for (int64_t c = 0; c < C; ++c) {
      double* gp = gx + (b * C + c) * H * W;
      for (int64_t i = 0; i < H * W; ++i) gp[i] = 0.0;
      for (int64_t o = 0; o < OH * OW; ++o) gp[idx[(b * C + c) * OH * OW + o]] += gy[(b * C + c) * OH * OW + o];
    }
}

/* Krizhevsky et al. 2012 local response normalisation across channels:
 *   d_i = k + alpha * sum_{j=i-n/2}^{i+(n-1)/2} a_j^2   (alpha NOT divided by n)
 *   b_i = a_i * d_i^(-beta)
 * scale receives d. Sum in ascending channel order. */
void or_lrn_forward(const double* a, int64_t B, int64_t C, int64_t HW, int n, double alpha,
                    double beta, double k, double* b, double* scale) {
  const int lo = n / 2, hi = (n - 1) / 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t bb = 0; bb < B; ++bb)
    for (int64_t c = 0; c < C; ++c) {
      const int64_t j0 = c - lo < 0 ? 0 : c - lo;
      const int64_t j1 = c + hi > C - 1 ? C - 1 : c + hi;
      for (int64_t p = 0; p < HW; ++p) {
        double sum = 0.0;
        for (int64_t j = j0; j <= j1; ++j) {
          const double v = a[(bb * C + j) * HW + p];
          sum += v * v;
        }
        const double d = k + alpha * sum;
        const int64_t at = (bb * C + c) * HW + p;
        scale[at] = d;
        b[at] = a[at] * pow(d, -beta);
      }
    }
}

/* ga_j = gb_j d_j^-beta - 2 alpha beta a_j sum_{i: j in N(i)} gb_i a_i d_i^(-beta-1) */
void or_lrn_backward(const double* a, const double* scale, const double* gb, int64_t B, int64_t C,
                     int64_t HW, int n, double alpha, double beta, double* ga) {
  const int lo = n / 2, hi = (n - 1) / 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t bb = 0; bb < B; ++bb)
    for (int64_t c = 0; c < C; ++c) {
      /* i ranges over channels whose window contains c: i in [c-hi, c+lo] */
      const int64_t i0 = c - hi < 0 ? 0 : c - hi;
      const int64_t i1 = c + lo > C - 1 ? C - 1 : c + lo;
      for (int64_t p = 0; p < HW; ++p) {
        double acc = 0.0;
        for (int64_t i = i0; i <= i1; ++i) {
          const int64_t ai = (bb * C + i) * HW + p;
          acc += gb[ai] * a[ai] * pow(scale[ai], -beta - 1.0);
        }
        const int64_t at = (bb * C + c) * HW + p;
        ga[at] = gb[at] * pow(scale[at], -beta) - 2.0 * alpha * beta * a[at] * acc;
      }
    }
}

/* ---------------------------------------------------------------- cluster */

typedef struct {
  double* k;
  double* b;
} conv_p;
typedef struct {
  double* w; /* [in][out_i] */
  double* b; /* [out_i] */
  int64_t c0, c1;
} fc_p;

typedef struct {
  conv_p* conv;
  conv_p* conv_m;
  fc_p* fc;
  fc_p* fc_m;
  int64_t sent[4], recv[4];
} worker_t;

typedef struct {
  double* input;
  int input_owned;
  const uint8_t** mask; /* forced ReLU masks (NULL: pre > 0) */
  double** pre;
  double** act;
  double** lrn;
  double** lrn_d;
  double** pool;
  int32_t** pidx;
} cache_t;

struct or_cluster {
  or_model_spec spec;
  or_conv_layer* conv;
  or_fc_layer* fc;
  or_cluster_config cfg;
  geom_t* g;
  int64_t flat;
  int skip_sync_broadcast;
  int storage_bf16; /* test-only: round stored tensors to bf16 where the B200 bf16 path stores them */
  /* test-only decision replay (or_cluster_force_decisions): per worker x conv
   * layer ReLU masks / pool argmax, per fc layer ReLU masks (K == 1); and the
   * last step's disagreement statistics against the oracle's own decisions */
  uint8_t** f_cmask;
  int32_t** f_pidx;
  uint8_t** f_fmask;
  int64_t* st_mis;  /* [3][K * max(nc, nf)] */
  double* st_gap;
  worker_t* w;
  or_trace_event* events;
  int n_events, cap_events;
};

static int stat_layers(const or_cluster* c) {
  const int a = c->spec.n_conv, b = c->cfg.workers * c->spec.n_fc;
  return a > b ? a : b;
}

static double* dalloc(int64_t n) { return calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

static void shard_range(int64_t total, int parts, int idx, int64_t* b, int64_t* e) {
  const int64_t base = total / parts; /* cluster.cpp:69-75 */
  *b = base * idx;
  *e = idx == parts - 1 ? total : *b + base;
}

static int64_t conv_k_size(const or_cluster* c, int l) {
  const or_conv_layer* L = &c->conv[l];
  return L->out_channels * L->in_channels * L->kernel * L->kernel;
}

/* ClusterConfig::validate (cluster.cpp:50-67) + Cluster::Cluster (:394-415)
 * + init_model (model.cpp:133-162). */
or_cluster* or_cluster_create(const or_model_spec* spec, const or_cluster_config* cfg, int* status) {
  *status = 0;
  geom_t* g = calloc((size_t)(spec->n_conv > 0 ? spec->n_conv : 1), sizeof(geom_t));
  int rc = compute_geometry(spec, g);
  if (rc) {
    free(g);
    *status = rc;
    return NULL;
  }
  if (cfg->workers < 1) {
    free(g);
    *status = fail(1, "cluster.workers: must be >= 1");
    return NULL;
  }
  if (cfg->per_worker_batch < 1) {
    free(g);
    *status = fail(1, "cluster.per_worker_batch: must be >= 1");
    return NULL;
  }
  if (cfg->scheme == 2 && cfg->per_worker_batch % cfg->workers != 0) {
    free(g);
    *status = fail(1,
                   "cluster.per_worker_batch: scheme C scatters b/K examples per worker per turn; "
                   "%lld is not divisible by %d",
                   (long long)cfg->per_worker_batch, cfg->workers);
    return NULL;
  }
  if (cfg->variable_batch && cfg->scheme == 0) {
    free(g);
    *status = fail(1,
                   "cluster.variable_batch: scheme A has a single fc pass per step; per-sub-batch "
                   "updates require scheme B or C");
    return NULL;
  }
  or_cluster* c = calloc(1, sizeof(or_cluster));
  c->cfg = *cfg;
  c->g = g;
  c->conv = malloc(sizeof(or_conv_layer) * (size_t)spec->n_conv);
  memcpy(c->conv, spec->conv, sizeof(or_conv_layer) * (size_t)spec->n_conv);
  c->fc = malloc(sizeof(or_fc_layer) * (size_t)spec->n_fc);
  memcpy(c->fc, spec->fc, sizeof(or_fc_layer) * (size_t)spec->n_fc);
  c->spec = *spec;
  c->spec.conv = c->conv;
  c->spec.fc = c->fc;
  const geom_t* last = &g[spec->n_conv - 1];
  c->flat = last->f * last->hp * last->wp;

  /* init_model: one GaussianSampler stream; conv kernels in layer order,
   * then fc weights; biases zero; value = 0.01 * N(0,1). Single precision
   * rounds each value to float as Tensor::set_value does. */
  const int single = cfg->precision == 0;
  gauss_t gs;
  mt_seed(&gs, cfg->seed);
  const int nc = spec->n_conv, nf = spec->n_fc, K = cfg->workers;
  double** mk = malloc(sizeof(double*) * (size_t)nc);
  double** mw = malloc(sizeof(double*) * (size_t)nf);
  for (int l = 0; l < nc; ++l) {
    const int64_t n = conv_k_size(c, l);
    mk[l] = dalloc(n);
    for (int64_t i = 0; i < n; ++i) {
      double v = 0.01 * gauss_next(&gs);
      mk[l][i] = single ? (double)(float)v : v;
    }
  }
  for (int l = 0; l < nf; ++l) {
    const int64_t n = c->fc[l].in_dim * c->fc[l].out_dim;
    mw[l] = dalloc(n);
    for (int64_t i = 0; i < n; ++i) {
      double v = 0.01 * gauss_next(&gs);
      mw[l][i] = single ? (double)(float)v : v;
    }
  }
  c->w = calloc((size_t)K, sizeof(worker_t));
  for (int i = 0; i < K; ++i) {
    worker_t* w = &c->w[i];
    w->conv = calloc((size_t)nc, sizeof(conv_p));
    w->conv_m = calloc((size_t)nc, sizeof(conv_p));
    for (int l = 0; l < nc; ++l) {
      const int64_t n = conv_k_size(c, l), f = c->conv[l].out_channels;
      w->conv[l].k = dalloc(n);
      memcpy(w->conv[l].k, mk[l], sizeof(double) * (size_t)n);
      w->conv[l].b = dalloc(f);
      w->conv_m[l].k = dalloc(n);
      w->conv_m[l].b = dalloc(f);
    }
    w->fc = calloc((size_t)nf, sizeof(fc_p));
    w->fc_m = calloc((size_t)nf, sizeof(fc_p));
    for (int l = 0; l < nf; ++l) {
      const int64_t in = c->fc[l].in_dim, out = c->fc[l].out_dim;
      int64_t c0, c1;
      shard_range(out, K, i, &c0, &c1);
      const int64_t ns = c1 - c0;
      w->fc[l].c0 = w->fc_m[l].c0 = c0;
      w->fc[l].c1 = w->fc_m[l].c1 = c1;
      w->fc[l].w = dalloc(in * ns);
      for (int64_t r = 0; r < in; ++r)
        for (int64_t q = 0; q < ns; ++q) w->fc[l].w[r * ns + q] = mw[l][r * out + c0 + q];
      w->fc[l].b = dalloc(ns);
      w->fc_m[l].w = dalloc(in * ns);
      w->fc_m[l].b = dalloc(ns);
    }
  }
  for (int l = 0; l < nc; ++l) free(mk[l]);
  for (int l = 0; l < nf; ++l) free(mw[l]);
  free(mk);
  free(mw);
  c->cap_events = 8 + 2 * K;
  c->events = calloc((size_t)c->cap_events, sizeof(or_trace_event));
  {
    const int L = nc > K * nf ? nc : K * nf;
    c->f_cmask = calloc((size_t)(K * nc + 1), sizeof(uint8_t*));
    c->f_pidx = calloc((size_t)(K * nc + 1), sizeof(int32_t*));
    c->f_fmask = calloc((size_t)(K * nf + 1), sizeof(uint8_t*));
    c->st_mis = calloc((size_t)(3 * K * L + 1), sizeof(int64_t));
    c->st_gap = calloc((size_t)(3 * K * L + 1), sizeof(double));
  }
  return c;
}

void or_cluster_destroy(or_cluster* c) {
  if (!c) return;
  for (int i = 0; i < c->cfg.workers; ++i) {
    worker_t* w = &c->w[i];
    for (int l = 0; l < c->spec.n_conv; ++l) {
      free(w->conv[l].k); free(w->conv[l].b); free(w->conv_m[l].k); free(w->conv_m[l].b);
    }
    for (int l = 0; l < c->spec.n_fc; ++l) {
      free(w->fc[l].w); free(w->fc[l].b); free(w->fc_m[l].w); free(w->fc_m[l].b);
    }
    free(w->conv); free(w->conv_m); free(w->fc); free(w->fc_m);
  }
  for (int t = 0; t < c->cfg.workers * c->spec.n_conv; ++t) { free(c->f_cmask[t]); free(c->f_pidx[t]); }
  for (int t = 0; t < c->cfg.workers * c->spec.n_fc; ++t) free(c->f_fmask[t]);
  free(c->f_cmask); free(c->f_pidx); free(c->f_fmask); free(c->st_mis); free(c->st_gap);
  free(c->w); free(c->conv); free(c->fc); free(c->g); free(c->events);
  free(c);
}

void or_cluster_set_skip_sync_broadcast(or_cluster* c, int v) { c->skip_sync_broadcast = v; }

/* ---- bf16 storage emulation (test infrastructure; not in the reference) ----
 * The B200 bf16 math mode keeps fp32 master weights / momenta and accumulates
 * every GEMM, LRN and reduction in fp32, but STORES operands as bf16: the input
 * batch, the conv / fc operand copies of the weights, every post-ReLU
 * activation and stage output (pooled LRN output), the logit gradient, the
 * fc-internal input gradients and every conv-layer dz / dgrad output. The
 * logits and the boundary gradient stay fp32. A forward decision taken on a
 * bf16-rounded value (pool argmax, ReLU mask) differs from the all-double one
 * whenever rounding reorders or ties two window values, which changes whole
 * gradient entries, not just their low bits. With storage_bf16 set, this
 * oracle rounds (to nearest even, via float like the GPU's fp32 -> bf16 store)
 * at exactly those points and computes everything else in double, so the GPU
 * step is compared with the same decisions; the pure-double mode stays the
 * reference restatement. */
static double q_bf16(double v) {
  float f = (float)v;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) {
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
  }
  memcpy(&f, &u, 4);
  return (double)f;
}
static void q_arr(const or_cluster* c, double* a, int64_t n) {
  if (c->storage_bf16 != 1) return;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) a[i] = q_bf16(a[i]);
}
static void f_arr(const or_cluster* c, double* a, int64_t n) { /* fp32 storage */
  if (c->storage_bf16 != 1) return;
  for (int64_t i = 0; i < n; ++i) a[i] = (double)(float)a[i];
}
/* Operand copy (bf16 mode) or the array itself. Caller frees when != src. */
static const double* q_copy(const or_cluster* c, const double* src, int64_t n) {
  if (c->storage_bf16 != 1) return src;
  double* d = dalloc(n);
  memcpy(d, src, sizeof(double) * (size_t)n);
  q_arr(c, d, n);
  return d;
}
/* bf16 mode: the LRN scale in fp32 with the B200 kernels' pinned arithmetic
 * (lrn_pool_fwd_kernel: s = fma(a_j, a_j, s) over the window in ascending
 * channel order from s = 0, d = fma(alpha, s, k)), then b = a * d^-beta in
 * double. The scale decides pool ties: at AlexNet's k = 2 most pixels have
 * alpha * sum below half an fp32 ulp of 2, so d is exactly 2.0f on the GPU and
 * two pixels with the same bf16 activation tie (first maximum wins), where the
 * all-double scale would break the tie. */
static void lrn_forward_f32_scale(const double* a, int64_t B, int64_t C, int64_t HW, int n, double alpha,
                                  double beta, double k, double* b) {
  const int lo = n / 2, hi = (n - 1) / 2;
  const float af = (float)alpha, kf = (float)k;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t bb = 0; bb < B; ++bb)
    for (int64_t c = 0; c < C; ++c) {
      const int64_t j0 = c - lo < 0 ? 0 : c - lo;
      const int64_t j1 = c + hi > C - 1 ? C - 1 : c + hi;
      for (int64_t p = 0; p < HW; ++p) {
        float sum = 0.f;
        for (int64_t j = j0; j <= j1; ++j) {
          const float v = (float)a[(bb * C + j) * HW + p];
          sum = fmaf(v, v, sum);
        }
        const float d = fmaf(af, sum, kf);
        const int64_t at = (bb * C + c) * HW + p;
        b[at] = a[at] * pow((double)d, -beta);
      }
    }
}

/* Decision replay (test infrastructure): the next run_step takes these ReLU
 * masks / pool argmax instead of its own (kind 0: conv ReLU mask uint8
 * [b][F][OH][OW]; kind 1: conv pool argmax int32 [b][F][PH][PW], plane index;
 * kind 2: fc ReLU mask uint8 [n][out] of turn j, layer = j * n_fc + l, the
 * gathered activation's mask -- worker i uses its shard's columns) and records, per forced
 * decision set, how many differ from its own and by how much. src NULL clears. */
int or_cluster_force_decisions(or_cluster* c, int worker, int kind, int layer, const void* src, int64_t n) {
  const int nc = c->spec.n_conv, nf = c->spec.n_fc, K = c->cfg.workers;
  const int64_t b = c->cfg.per_worker_batch;
  if (worker < 0 || worker >= K || kind < 0 || kind > 2) return fail(4, "force_decisions: bad worker/kind");
  if (kind < 2 && (layer < 0 || layer >= nc)) return fail(4, "force_decisions: bad conv layer");
  const int nsub = c->cfg.scheme == 0 ? 1 : K;
  if (kind == 2 && (layer < 0 || layer >= nsub * nf)) return fail(4, "force_decisions: bad fc turn/layer");
  int64_t want;
  void** slot;
  size_t es;
  if (kind == 0) {
    want = b * c->g[layer].f * c->g[layer].ho * c->g[layer].wo;
    slot = (void**)&c->f_cmask[worker * nc + layer];
    es = 1;
  } else if (kind == 1) {
    if (c->conv[layer].pool_kernel <= 0) return fail(4, "force_decisions: layer has no pool");
    want = b * c->g[layer].f * c->g[layer].hp * c->g[layer].wp;
    slot = (void**)&c->f_pidx[worker * nc + layer];
    es = 4;
  } else {
    const int64_t rows = c->cfg.scheme == 0 ? (int64_t)K * b : b;
    want = rows * c->fc[layer % nf].out_dim;
    slot = (void**)&c->f_fmask[layer];
    es = 1;
  }
  free(*slot);
  *slot = NULL;
  if (!src) return 0;
  if (n != want) return fail(2, "force_decisions: size %lld, expected %lld", (long long)n, (long long)want);
  *slot = malloc((size_t)n * es);
  memcpy(*slot, src, (size_t)n * es);
  return 0;
}

int or_cluster_decision_stats(const or_cluster* c, int worker, int kind, int layer, int64_t* mismatches,
                              double* max_gap) {
  const int L = stat_layers(c);
  if (worker < 0 || worker >= c->cfg.workers || kind < 0 || kind > 2 || layer < 0 || layer >= L)
    return fail(4, "decision_stats: bad worker/kind/layer");
  const int64_t at = ((int64_t)kind * c->cfg.workers + worker) * L + layer;
  *mismatches = c->st_mis[at];
  *max_gap = c->st_gap[at];
  return 0;
}

int or_cluster_set_storage_rounding(or_cluster* c, int mode) {
  if (mode < 0 || mode > 1) return fail(4, "storage rounding: mode must be 0 (double) or 1 (bf16)");
  c->storage_bf16 = mode;
  return 0;
}

/* conv_forward (model.cpp:225-243) + add_channel_bias (:166-182) + relu
 * (tensor.cpp:556-564), then the LRN / pool superset. */
static void decision_stat(const or_cluster* c, int kind, int worker, int layer, int64_t mis, double gap) {
  const int L = stat_layers(c);
  const int64_t at = ((int64_t)kind * c->cfg.workers + worker) * L + layer;
  c->st_mis[at] = mis;
  c->st_gap[at] = gap;
}

/* ReLU with an optional forced mask: out = mask ? z : 0; records the
 * disagreements with the oracle's own decision (z > 0) and the largest |z| /
 * rms(z) among them. */
static void relu_forced(const or_cluster* c, int kind, int worker, int layer, const double* z, double* a,
                        int64_t n, const uint8_t* mask) {
  if (!mask) {
    for (int64_t i = 0; i < n; ++i) a[i] = z[i] > 0.0 ? z[i] : 0.0;
    return;
  }
  int64_t mis = 0;
  double gap = 0.0, ss = 0.0;
  for (int64_t i = 0; i < n; ++i) ss += z[i] * z[i];
  const double rms = sqrt(ss / (double)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    a[i] = mask[i] ? z[i] : 0.0;
    if ((mask[i] != 0) != (z[i] > 0.0)) {
      ++mis;
      const double g = fabs(z[i]) / (rms > 0.0 ? rms : 1.0);
      if (g > gap) gap = g;
    }
  }
  decision_stat(c, kind, worker, layer, mis, gap);
}

static void conv_forward(const or_cluster* c, const conv_p* p, const double* batch, int64_t B,
                         cache_t* cache, int worker) {
  const int nc = c->spec.n_conv;
  cache->input = (double*)q_copy(c, batch, B * c->g[0].c * c->g[0].h * c->g[0].w);
  cache->input_owned = cache->input != batch;
  cache->pre = calloc((size_t)nc, sizeof(double*));
  cache->mask = calloc((size_t)nc, sizeof(uint8_t*));
  cache->act = calloc((size_t)nc, sizeof(double*));
  cache->lrn = calloc((size_t)nc, sizeof(double*));
  cache->lrn_d = calloc((size_t)nc, sizeof(double*));
  cache->pool = calloc((size_t)nc, sizeof(double*));
  cache->pidx = calloc((size_t)nc, sizeof(int32_t*));
  const double* x = batch;
  for (int l = 0; l < nc; ++l) {
    const or_conv_layer* L = &c->conv[l];
    const geom_t* g = &c->g[l];
    const int64_t hw = g->ho * g->wo, n = B * g->f * hw;
    double* z = dalloc(n);
    const double* kq = q_copy(c, p[l].k, conv_k_size(c, l));
    conv_fwd(l == 0 ? cache->input : x, kq, z, B, g->c, g->h, g->w, g->f, L->kernel, L->kernel, g->ho, g->wo,
             L->stride, L->pad);
    if (kq != p[l].k) free((void*)kq);
    for (int64_t b = 0; b < B; ++b)
      for (int64_t f = 0; f < g->f; ++f)
        for (int64_t q = 0; q < hw; ++q) z[(b * g->f + f) * hw + q] += p[l].b[f];
    cache->pre[l] = z;
    double* a = dalloc(n);
    const uint8_t* fm = c->f_cmask[worker * nc + l];
    if (L->relu) {
      relu_forced(c, 0, worker, l, z, a, n, fm);
      cache->mask[l] = fm;
    } else {
      for (int64_t i = 0; i < n; ++i) a[i] = z[i];
    }
    q_arr(c, a, n);
    cache->act[l] = a;
    const double* out = a;
    if (L->lrn_size > 0) {
      cache->lrn[l] = dalloc(n);
      cache->lrn_d[l] = dalloc(n);
      or_lrn_forward(a, B, g->f, hw, L->lrn_size, L->lrn_alpha, L->lrn_beta, L->lrn_k,
                     cache->lrn[l], cache->lrn_d[l]);
      if (c->storage_bf16 == 1)
        lrn_forward_f32_scale(a, B, g->f, hw, L->lrn_size, L->lrn_alpha, L->lrn_beta, L->lrn_k,
                              cache->lrn[l]);
      out = cache->lrn[l];
    }
    if (L->pool_kernel > 0) {
      const int64_t np = B * g->f * g->hp * g->wp;
      cache->pool[l] = dalloc(np);
      cache->pidx[l] = calloc((size_t)np, sizeof(int32_t));
      or_maxpool_forward(out, B, g->f, g->ho, g->wo, L->pool_kernel, L->pool_stride,
                         cache->pool[l], cache->pidx[l]);
      const int32_t* fi = c->f_pidx[worker * nc + l];
      if (fi) { /* replay the forced argmax; record the near-tie gaps where it differs */
        int64_t mis = 0;
        double gap = 0.0, ss = 0.0;
        const int64_t plane = g->ho * g->wo, pp = g->hp * g->wp;
        for (int64_t t = 0; t < n; ++t) ss += out[t] * out[t];
        const double rms = sqrt(ss / (double)(n > 0 ? n : 1));
        for (int64_t o = 0; o < np; ++o) {
          const double* xp = out + (o / pp) * plane;
          const double own = cache->pool[l][o], forced = xp[fi[o]];
          if (fi[o] != cache->pidx[l][o]) { /* gap: the value given up, in units of the layer's rms */
            ++mis;
            const double gg = fabs(own - forced) / (rms > 0.0 ? rms : 1.0);
            if (gg > gap) gap = gg;
          }
          cache->pool[l][o] = forced;
          cache->pidx[l][o] = fi[o];
        }
        decision_stat(c, 1, worker, l, mis, gap);
      }
      out = cache->pool[l];
      q_arr(c, cache->pool[l], np);
    } else if (L->lrn_size > 0) {
      q_arr(c, cache->lrn[l], n);
    }
    x = out;
  }
}

static const double* stage_out(const or_cluster* c, const cache_t* cache, int l) {
  if (c->conv[l].pool_kernel > 0) return cache->pool[l];
  if (c->conv[l].lrn_size > 0) return cache->lrn[l];
  return cache->act[l];
}

static void cache_free(const or_cluster* c, cache_t* cache) {
  for (int l = 0; l < c->spec.n_conv; ++l) {
    free(cache->pre[l]); free(cache->act[l]); free(cache->lrn[l]); free(cache->lrn_d[l]);
    free(cache->pool[l]); free(cache->pidx[l]);
  }
  free(cache->pre); free((void*)cache->mask); free(cache->act); free(cache->lrn); free(cache->lrn_d); free(cache->pool);
  free(cache->pidx);
  if (cache->input_owned) free(cache->input);
}

/* conv_backward_from_flat (model.cpp:259-283) + channel_sums (:184-202) +
 * relu_backward (tensor.cpp:566-583), with the pool / LRN superset. */
static void conv_backward(const or_cluster* c, const conv_p* p, const cache_t* cache, int64_t B,
                          const double* flat_grad, conv_p* grads) {
  const int nc = c->spec.n_conv;
  const geom_t* gl = &c->g[nc - 1];
  double* grad = dalloc(B * gl->f * gl->hp * gl->wp);
  memcpy(grad, flat_grad, sizeof(double) * (size_t)(B * gl->f * gl->hp * gl->wp));
  for (int l = nc - 1; l >= 0; --l) {
    const or_conv_layer* L = &c->conv[l];
    const geom_t* g = &c->g[l];
    const int64_t hw = g->ho * g->wo, n = B * g->f * hw;
    if (L->pool_kernel > 0) {
      double* gx = dalloc(n);
      or_maxpool_backward(grad, cache->pidx[l], B, g->f, g->ho, g->wo, L->pool_kernel,
                          L->pool_stride, gx);
      free(grad);
      grad = gx;
    }
    if (L->lrn_size > 0) {
      double* ga = dalloc(n);
      or_lrn_backward(cache->act[l], cache->lrn_d[l], grad, B, g->f, hw, L->lrn_size,
                      L->lrn_alpha, L->lrn_beta, ga);
      free(grad);
      grad = ga;
    }
    if (L->relu) {
      const uint8_t* fm = cache->mask[l];
      for (int64_t i = 0; i < n; ++i)
        if (fm ? !fm[i] : !(cache->pre[l][i] > 0.0)) grad[i] = 0.0;
    }
    q_arr(c, grad, n);
    for (int64_t f = 0; f < g->f; ++f) grads[l].b[f] = 0.0;
    for (int64_t b = 0; b < B; ++b)
      for (int64_t f = 0; f < g->f; ++f)
        for (int64_t q = 0; q < hw; ++q) grads[l].b[f] += grad[(b * g->f + f) * hw + q];
    const double* input = l == 0 ? cache->input : stage_out(c, cache, l - 1);
    double* gx = l > 0 ? dalloc(B * g->c * g->h * g->w) : NULL;
    const double* kq = q_copy(c, p[l].k, conv_k_size(c, l));
    conv_bwd(input, kq, grad, gx, grads[l].k, B, g->c, g->h, g->w, g->f, L->kernel, L->kernel,
             g->ho, g->wo, L->stride, L->pad);
    if (kq != p[l].k) free((void*)kq);
    if (gx) q_arr(c, gx, B * g->c * g->h * g->w);
    free(grad);
    grad = gx;
  }
  free(grad);
}

static void push_event(or_cluster* c, int phase, int sub, int worker, int64_t total, int64_t maxs) {
  or_trace_event* e = &c->events[c->n_events++];
  e->phase = phase;
  e->sub_batch = sub;
  e->worker = worker;
  e->bytes_total = total;
  e->bytes_max_sender = maxs;
}

/* Cluster::run_step (cluster.cpp:439-711) */
int or_cluster_run_step(or_cluster* c, const double* const* batches, const double* const* targets,
                        const or_hyper* hp, double lr, or_step_metrics* out) {
  const int K = c->cfg.workers, scheme = c->cfg.scheme, nf = c->spec.n_fc, nc = c->spec.n_conv;
  const int64_t b = c->cfg.per_worker_batch, A = c->flat, L = c->spec.num_classes;
  const int64_t elt = c->cfg.precision == 0 ? 4 : 8;
  const int64_t row_bytes = A * elt;
  const int variable = c->cfg.variable_batch;
  const double fc_lr = variable ? (hp->has_fc_partial_lr ? hp->fc_partial_lr : lr) : lr;
  memset(out, 0, sizeof *out);
  c->n_events = 0;
  for (int i = 0; i < K; ++i)
    if (!batches[i] || !targets[i])
      return fail(4, "run_step: expected %d batches and targets", K);

  /* charge lambda, cluster.cpp:466-471 */
#define CHARGE(wi, cls, s_, r_)              \
  do {                                       \
    c->w[wi].sent[cls] += (s_);              \
    c->w[wi].recv[cls] += (r_);              \
    out->bytes_sent[cls] += (s_);            \
  } while (0)

  cache_t* caches = calloc((size_t)K, sizeof(cache_t));
  for (int i = 0; i < K; ++i) conv_forward(c, c->w[i].conv, batches[i], b, &caches[i], i);

  /* exchange_activations / assemble_rows (cluster.cpp:113-194) */
  const int num_sub = scheme == 0 ? 1 : K;
  const int64_t n = scheme == 0 ? (int64_t)K * b : b;
  double** assembled = calloc((size_t)num_sub, sizeof(double*));
  double** sub_t = calloc((size_t)num_sub, sizeof(double*));
  int64_t* sent = calloc((size_t)num_sub * K, sizeof(int64_t));
  for (int j = 0; j < num_sub; ++j) {
    assembled[j] = dalloc(n * A);
    sub_t[j] = dalloc(n * L);
  }
  const int64_t slice = scheme == 2 ? b / K : 0;
  for (int i = 0; i < K; ++i) {
    const double* top = stage_out(c, &caches[i], nc - 1);
    if (scheme == 0) {
      memcpy(assembled[0] + i * b * A, top, sizeof(double) * (size_t)(b * A));
      memcpy(sub_t[0] + i * b * L, targets[i], sizeof(double) * (size_t)(b * L));
    } else if (scheme == 1) {
      memcpy(assembled[i], top, sizeof(double) * (size_t)(b * A));
      memcpy(sub_t[i], targets[i], sizeof(double) * (size_t)(b * L));
    } else {
      for (int j = 0; j < K; ++j) {
        memcpy(assembled[j] + i * slice * A, top + j * slice * A, sizeof(double) * (size_t)(slice * A));
        memcpy(sub_t[j] + i * slice * L, targets[i] + j * slice * L, sizeof(double) * (size_t)(slice * L));
      }
    }
  }
  if (K > 1)
    for (int j = 0; j < num_sub; ++j)
      for (int i = 0; i < K; ++i) {
        int64_t s = 0;
        if (scheme == 0) s = (K - 1) * b * row_bytes;
        else if (scheme == 1) s = i == j ? (K - 1) * b * row_bytes : 0;
        else s = (K - 1) * (b / K) * row_bytes;
        sent[j * K + i] = s;
      }

  /* uniform-mode accumulators, zero_like (cluster.cpp:372-390) */
  fc_p** acc = calloc((size_t)K, sizeof(fc_p*));
  fc_p** pass = calloc((size_t)K, sizeof(fc_p*));
  for (int i = 0; i < K; ++i) {
    acc[i] = calloc((size_t)nf, sizeof(fc_p));
    pass[i] = calloc((size_t)nf, sizeof(fc_p));
    for (int l = 0; l < nf; ++l) {
      const int64_t ns = c->w[i].fc[l].c1 - c->w[i].fc[l].c0;
      acc[i][l].w = dalloc(c->fc[l].in_dim * ns);
      acc[i][l].b = dalloc(ns);
      pass[i][l].w = dalloc(c->fc[l].in_dim * ns);
      pass[i][l].b = dalloc(ns);
    }
  }

  or_trace_event* fwd_ev = calloc((size_t)num_sub, sizeof(or_trace_event));
  double** boundary = calloc((size_t)num_sub, sizeof(double*));
  double loss_weighted = 0.0;
  double** layer_in = calloc((size_t)nf, sizeof(double*));
  double** pre = calloc((size_t)nf * K, sizeof(double*));

  for (int j = 0; j < num_sub; ++j) {
    { /* cluster.cpp:511-528 */
      int64_t total = 0, maxs = 0;
      for (int i = 0; i < K; ++i) {
        int64_t inbound = 0;
        if (K > 1) inbound = scheme == 1 ? (i == j ? 0 : b * row_bytes) : sent[j * K + i];
        CHARGE(i, 0, sent[j * K + i], inbound);
        total += sent[j * K + i];
        if (sent[j * K + i] > maxs) maxs = sent[j * K + i];
      }
      fwd_ev[j].phase = 1; fwd_ev[j].sub_batch = j; fwd_ev[j].worker = scheme == 1 ? j : -1;
      fwd_ev[j].bytes_total = total; fwd_ev[j].bytes_max_sender = maxs;
    }
    /* model-parallel fc forward (cluster.cpp:534-553) */
    double* x = assembled[j];
    for (int l = 0; l < nf; ++l) {
      const int64_t in = c->fc[l].in_dim, outd = c->fc[l].out_dim;
      layer_in[l] = x;
      double* gathered = dalloc(n * outd);
      for (int i = 0; i < K; ++i) {
        const fc_p* p = &c->w[i].fc[l];
        const int64_t ns = p->c1 - p->c0;
        double* z = dalloc(n * ns);
        const double* wq = q_copy(c, p->w, in * ns);
        or_matmul(x, wq, z, n, in, ns); /* fc_affine model.cpp:219-223 */
        if (wq != p->w) free((void*)wq);
        for (int64_t r = 0; r < n; ++r)
          for (int64_t q = 0; q < ns; ++q) z[r * ns + q] += p->b[q];
        const uint8_t* fg = c->f_fmask[j * nf + l];
        if (fg && c->fc[l].relu) { /* forced: this shard's columns of the turn's gathered mask */
          uint8_t* fm = malloc((size_t)(n * ns));
          for (int64_t r = 0; r < n; ++r)
            for (int64_t q = 0; q < ns; ++q) fm[r * ns + q] = fg[r * outd + p->c0 + q];
          double* a = dalloc(n * ns);
          relu_forced(c, 2, i, j * nf + l, z, a, n * ns, fm);
          for (int64_t r = 0; r < n; ++r)
            for (int64_t q = 0; q < ns; ++q) gathered[r * outd + p->c0 + q] = a[r * ns + q];
          free(a);
          free(fm);
        } else {
          for (int64_t r = 0; r < n; ++r)
            for (int64_t q = 0; q < ns; ++q) {
              const double v = z[r * ns + q];
              gathered[r * outd + p->c0 + q] = c->fc[l].relu ? (v > 0.0 ? v : 0.0) : v;
            }
        }
        pre[l * K + i] = z;
        const int64_t shard_bytes = n * ns * elt;
        CHARGE(i, 2, (K - 1) * shard_bytes, n * (outd - ns) * elt);
      }
      if (l + 1 < nf) q_arr(c, gathered, n * outd);
      else f_arr(c, gathered, n * outd);
      x = gathered;
    }
    double* grad = dalloc(n * L);
    double loss = 0.0;
    int rc = or_logistic_xent(x, sub_t[j], n, L, grad, &loss);
    if (rc) return rc; /* DomainError propagates (test-only oracle: leaks on error) */
    q_arr(c, grad, n * L);
    loss_weighted += loss * (double)n;
    free(x);
    /* fc backward (cluster.cpp:562-584) */
    for (int li = nf - 1; li >= 0; --li) {
      const int64_t in = c->fc[li].in_dim, outd = c->fc[li].out_dim;
      double* dx = dalloc(n * in);
      for (int i = 0; i < K; ++i) {
        const fc_p* p = &c->w[i].fc[li];
        const int64_t ns = p->c1 - p->c0;
        double* dz = dalloc(n * ns);
        for (int64_t r = 0; r < n; ++r)
          for (int64_t q = 0; q < ns; ++q) dz[r * ns + q] = grad[r * outd + p->c0 + q];
        if (c->fc[li].relu) {
          const uint8_t* fg = c->f_fmask[j * nf + li];
          for (int64_t r = 0; r < n; ++r)
            for (int64_t q = 0; q < ns; ++q)
              if (fg ? !fg[r * outd + p->c0 + q] : !(pre[li * K + i][r * ns + q] > 0.0)) dz[r * ns + q] = 0.0;
        }
        or_matmul_tn(layer_in[li], dz, pass[i][li].w, n, in, ns);
        for (int64_t q = 0; q < ns; ++q) pass[i][li].b[q] = 0.0;
        for (int64_t r = 0; r < n; ++r)
          for (int64_t q = 0; q < ns; ++q) pass[i][li].b[q] += dz[r * ns + q];
        double* partial = dalloc(n * in);
        const double* wq = q_copy(c, p->w, in * ns);
        or_matmul_nt(dz, wq, partial, n, ns, in);
        if (wq != p->w) free((void*)wq);
        for (int64_t t = 0; t < n * in; ++t) dx[t] += partial[t];
        free(partial);
        free(dz);
        if (li > 0) {
          const int64_t part_bytes = n * in * elt;
          CHARGE(i, 2, (K - 1) * part_bytes, (K - 1) * part_bytes);
        }
      }
      free(grad);
      if (li > 0) q_arr(c, dx, n * in);
      else f_arr(c, dx, n * in);
      grad = dx;
    }
    boundary[j] = grad;
    for (int l = 1; l < nf; ++l) free(layer_in[l]);
    for (int t = 0; t < nf * K; ++t) {
      free(pre[t]);
      pre[t] = NULL;
    }
    if (variable) { /* cluster.cpp:586-601 */
      for (int i = 0; i < K; ++i)
        for (int l = 0; l < nf; ++l) {
          fc_p* p = &c->w[i].fc[l];
          fc_p* m = &c->w[i].fc_m[l];
          const int64_t ns = p->c1 - p->c0;
          or_momentum_update(p->w, m->w, pass[i][l].w, c->fc[l].in_dim * ns, fc_lr, hp->momentum,
                             hp->weight_decay);
          or_momentum_update(p->b, m->b, pass[i][l].b, ns, fc_lr, hp->momentum, hp->weight_decay);
        }
      out->fc_update_count += 1;
    } else { /* :602-609 */
      for (int i = 0; i < K; ++i)
        for (int l = 0; l < nf; ++l) {
          const int64_t ns = c->w[i].fc[l].c1 - c->w[i].fc[l].c0;
          for (int64_t t = 0; t < c->fc[l].in_dim * ns; ++t) acc[i][l].w[t] += pass[i][l].w[t];
          for (int64_t t = 0; t < ns; ++t) acc[i][l].b[t] += pass[i][l].b[t];
        }
    }
  }

  /* return_gradients (cluster.cpp:196-269) + accounting (:613-633) */
  double** own = calloc((size_t)K, sizeof(double*));
  for (int i = 0; i < K; ++i) own[i] = dalloc(b * A);
  int64_t* rsent = calloc((size_t)num_sub * K, sizeof(int64_t));
  if (scheme == 0) {
    for (int i = 0; i < K; ++i) {
      memcpy(own[i], boundary[0] + i * b * A, sizeof(double) * (size_t)(b * A));
      if (K > 1) rsent[i] = (K - 1) * b * row_bytes;
    }
  } else if (scheme == 1) {
    for (int j = 0; j < K; ++j) {
      memcpy(own[j], boundary[j], sizeof(double) * (size_t)(b * A));
      for (int i = 0; i < K; ++i)
        if (i != j) rsent[j * K + i] = b * row_bytes;
    }
  } else {
    for (int j = 0; j < K; ++j)
      for (int i = 0; i < K; ++i) {
        memcpy(own[i] + j * slice * A, boundary[j] + i * slice * A, sizeof(double) * (size_t)(slice * A));
        if (K > 1) rsent[j * K + i] = (K - 1) * slice * row_bytes;
      }
  }
  push_event(c, 0, -1, -1, 0, 0);
  for (int j = 0; j < num_sub; ++j) {
    int64_t total = 0, maxs = 0;
    for (int i = 0; i < K; ++i) {
      const int64_t s = rsent[j * K + i];
      int64_t r = s;
      if (scheme == 1) r = (i == j && K > 1) ? (K - 1) * b * row_bytes : 0;
      CHARGE(i, 1, s, r);
      total += s;
      if (s > maxs) maxs = s;
    }
    c->events[c->n_events++] = fwd_ev[j];
    push_event(c, 2, j, scheme == 1 ? j : -1, total, maxs);
  }

  /* conv backward per worker (cluster.cpp:647-656) */
  conv_p** cg = calloc((size_t)K, sizeof(conv_p*));
  for (int i = 0; i < K; ++i) {
    if (scheme == 0 && K > 1)
      for (int64_t t = 0; t < b * A; ++t) own[i][t] *= (double)K;
    cg[i] = calloc((size_t)nc, sizeof(conv_p));
    for (int l = 0; l < nc; ++l) {
      cg[i][l].k = dalloc(conv_k_size(c, l));
      cg[i][l].b = dalloc(c->conv[l].out_channels);
    }
    conv_backward(c, c->w[i].conv, &caches[i], b, own[i], cg[i]);
  }
  push_event(c, 3, -1, -1, 0, 0);

  /* flatten / sync / unflatten (cluster.cpp:273-354, 660-675) */
  int64_t G = 0;
  for (int l = 0; l < nc; ++l) G += conv_k_size(c, l) + c->conv[l].out_channels;
  {
    int64_t total = 0, maxs = 0;
    if (K > 1) {
      double* mean = dalloc(G);
      double** flat = calloc((size_t)K, sizeof(double*));
      for (int i = 0; i < K; ++i) {
        flat[i] = dalloc(G);
        int64_t at = 0;
        for (int l = 0; l < nc; ++l) {
          memcpy(flat[i] + at, cg[i][l].k, sizeof(double) * (size_t)conv_k_size(c, l));
          at += conv_k_size(c, l);
          memcpy(flat[i] + at, cg[i][l].b, sizeof(double) * (size_t)c->conv[l].out_channels);
          at += c->conv[l].out_channels;
        }
      }
      for (int w = 0; w < K; ++w)
        for (int64_t t = 0; t < G; ++t) mean[t] += flat[w][t];
      const double inv = 1.0 / (double)K;
      for (int64_t t = 0; t < G; ++t) mean[t] *= inv;
      for (int i = 0; i < K; ++i) {
        int64_t s0, s1;
        shard_range(G, K, i, &s0, &s1);
        const int64_t shard_bytes = (s1 - s0) * elt;
        const int64_t s = (G * elt - shard_bytes) + (K - 1) * shard_bytes;
        CHARGE(i, 3, s, s);
        total += s;
        if (s > maxs) maxs = s;
        if (c->skip_sync_broadcast) {
          for (int64_t t = s0; t < s1; ++t) flat[i][t] = mean[t];
        } else {
          memcpy(flat[i], mean, sizeof(double) * (size_t)G);
        }
      }
      for (int i = 0; i < K; ++i) {
        int64_t at = 0;
        for (int l = 0; l < nc; ++l) {
          memcpy(cg[i][l].k, flat[i] + at, sizeof(double) * (size_t)conv_k_size(c, l));
          at += conv_k_size(c, l);
          memcpy(cg[i][l].b, flat[i] + at, sizeof(double) * (size_t)c->conv[l].out_channels);
          at += c->conv[l].out_channels;
        }
        free(flat[i]);
      }
      free(flat);
      free(mean);
    } else {
      CHARGE(0, 3, 0, 0);
    }
    push_event(c, 4, -1, -1, total, maxs);
  }

  /* updates (cluster.cpp:680-708) */
  if (!variable) {
    const double inv_subs = 1.0 / (double)num_sub;
    for (int i = 0; i < K; ++i)
      for (int l = 0; l < nf; ++l) {
        fc_p* p = &c->w[i].fc[l];
        fc_p* m = &c->w[i].fc_m[l];
        const int64_t ns = p->c1 - p->c0, nw = c->fc[l].in_dim * ns;
        for (int64_t t = 0; t < nw; ++t) acc[i][l].w[t] *= inv_subs;
        for (int64_t t = 0; t < ns; ++t) acc[i][l].b[t] *= inv_subs;
        or_momentum_update(p->w, m->w, acc[i][l].w, nw, lr, hp->momentum, hp->weight_decay);
        or_momentum_update(p->b, m->b, acc[i][l].b, ns, lr, hp->momentum, hp->weight_decay);
      }
    out->fc_update_count = 1;
  }
  for (int i = 0; i < K; ++i)
    for (int l = 0; l < nc; ++l) {
      or_momentum_update(c->w[i].conv[l].k, c->w[i].conv_m[l].k, cg[i][l].k, conv_k_size(c, l), lr,
                         hp->momentum, hp->weight_decay);
      or_momentum_update(c->w[i].conv[l].b, c->w[i].conv_m[l].b, cg[i][l].b,
                         c->conv[l].out_channels, lr, hp->momentum, hp->weight_decay);
    }
  out->conv_update_count = 1;
  out->loss = loss_weighted / (double)(K * b);
  out->n_events = c->n_events;
#undef CHARGE

  for (int i = 0; i < K; ++i) {
    cache_free(c, &caches[i]);
    for (int l = 0; l < nc; ++l) { free(cg[i][l].k); free(cg[i][l].b); }
    free(cg[i]);
    for (int l = 0; l < nf; ++l) { free(acc[i][l].w); free(acc[i][l].b); free(pass[i][l].w); free(pass[i][l].b); }
    free(acc[i]); free(pass[i]); free(own[i]);
  }
  for (int j = 0; j < num_sub; ++j) { free(assembled[j]); free(sub_t[j]); free(boundary[j]); }
  free(caches); free(cg); free(acc); free(pass); free(own); free(assembled); free(sub_t);
  free(boundary); free(sent); free(rsent); free(fwd_ev); free(layer_in); free(pre);
  return 0;
}

int or_cluster_trace(const or_cluster* c, or_trace_event* out, int cap) {
  for (int i = 0; i < c->n_events && i < cap; ++i) out[i] = c->events[i];
  return c->n_events;
}

int or_cluster_worker_bytes(const or_cluster* c, int worker, int64_t sent[4], int64_t received[4]) {
  if (worker < 0 || worker >= c->cfg.workers) return fail(4, "worker index out of range");
  for (int i = 0; i < 4; ++i) {
    sent[i] = c->w[worker].sent[i];
    received[i] = c->w[worker].recv[i];
  }
  return 0;
}

static double* param_ptr(const or_cluster* c, int worker, int which, int layer, int64_t* n) {
  if (worker < 0 || worker >= c->cfg.workers) return NULL;
  const worker_t* w = &c->w[worker];
  const int mom = which >= 4;
  which &= 3;
  if (which <= 1) {
    if (layer < 0 || layer >= c->spec.n_conv) return NULL;
    const conv_p* p = mom ? &w->conv_m[layer] : &w->conv[layer];
    *n = which == 0 ? conv_k_size(c, layer) : c->conv[layer].out_channels;
    return which == 0 ? p->k : p->b;
  }
  if (layer < 0 || layer >= c->spec.n_fc) return NULL;
  const fc_p* p = mom ? &w->fc_m[layer] : &w->fc[layer];
  const int64_t ns = p->c1 - p->c0;
  *n = which == 2 ? c->fc[layer].in_dim * ns : ns;
  return which == 2 ? p->w : p->b;
}

int64_t or_cluster_param_size(const or_cluster* c, int worker, int which, int layer) {
  int64_t n = -1;
  return param_ptr(c, worker, which, layer, &n) ? n : -1;
}

int or_cluster_read_param(const or_cluster* c, int worker, int which, int layer, double* dst,
                          int64_t n) {
  int64_t want = 0;
  double* p = param_ptr(c, worker, which, layer, &want);
  if (!p) return fail(4, "read_param: bad worker/which/layer");
  if (n != want) return fail(2, "read_param: size %lld, expected %lld", (long long)n, (long long)want);
  memcpy(dst, p, sizeof(double) * (size_t)n);
  return 0;
}

int or_cluster_write_param(or_cluster* c, int worker, int which, int layer, const double* src,
                           int64_t n) {
  int64_t want = 0;
  double* p = param_ptr(c, worker, which, layer, &want);
  if (!p) return fail(4, "write_param: bad worker/which/layer");
  if (n != want) return fail(2, "write_param: size %lld, expected %lld", (long long)n, (long long)want);
  memcpy(p, src, sizeof(double) * (size_t)n);
  return 0;
}
