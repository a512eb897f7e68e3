/* TEST INFRASTRUCTURE — the parity oracle, NOT part of the product.
 * See pgb_oracle.h. Plain C restatement of the reference DPSGD path;
 * pinned against oracle/_ref (the compiled reference) by
 * tests/test_oracle.py and tests/golden/gen_golden.py. */
#include "pgb_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---- rng: proj/core/include/pegrad/rng.hpp:35-62 ----------------------- */

uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_rng_value_at(uint64_t seed, uint64_t stream, uint64_t i) {
  const uint64_t g = 0x9E3779B97F4A7C15ull;
  return orc_mix64(orc_mix64(seed + g * (stream + 1)) + g * (i + 1));
}

typedef struct { uint64_t seed, stream, counter; } rng_t;

static double rng_unit(rng_t* r) { /* [0,1): rng.hpp:55-57 */
  return (double)(orc_rng_value_at(r->seed, r->stream, r->counter++) >> 11) *
         0x1.0p-53;
}
static double rng_uniform(rng_t* r, double lo, double hi) { /* rng.hpp:59-61 */
  return lo + (hi - lo) * rng_unit(r);
}

/* Box-Muller over pair-indexed uniforms in (0,1] (kernels.hpp:597-614). */
static void gauss_pair(uint64_t seed, uint64_t stream, int64_t pair,
                       double* c, double* s) {
  const double two_pi = 6.283185307179586476925286766559;
  const double u1 =
      (double)((orc_rng_value_at(seed, stream, 2 * (uint64_t)pair) >> 11) + 1) *
      0x1.0p-53;
  const double u2 =
      (double)((orc_rng_value_at(seed, stream, 2 * (uint64_t)pair + 1) >> 11) + 1) *
      0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  *c = r * cos(two_pi * u2);
  *s = r * sin(two_pi * u2);
}

void orc_gaussian_f64(uint64_t seed, uint64_t stream, int64_t n, double* out) {
  for (int64_t q = 0; 2 * q < n; ++q) {
    double c, s;
    gauss_pair(seed, stream, q, &c, &s);
    out[2 * q] = c;
    if (2 * q + 1 < n) out[2 * q + 1] = s;
  }
}

void orc_gaussian_f32(uint64_t seed, uint64_t stream, int64_t n, float* out) {
  for (int64_t q = 0; 2 * q < n; ++q) {
    double c, s;
    gauss_pair(seed, stream, q, &c, &s);
    out[2 * q] = (float)c;
    if (2 * q + 1 < n) out[2 * q + 1] = (float)s;
  }
}

/* ---- model descriptions: models.cpp:50-167 ----------------------------- */

static void add_layer(orc_desc* d, int32_t kind, int64_t in, int64_t out,
                      int64_t k, int64_t stride, int64_t pad) {
  orc_layer* l = &d->layers[d->n_layers++];
  l->kind = kind;
  l->in = in;
  l->out = out;
  l->k = k;
  l->stride = stride;
  l->pad = pad;
}

int orc_finish_desc(orc_desc* d) { /* register_params, models.cpp:50-83 */
  d->n_blocks = 0;
  for (int i = 0; i < d->n_layers; ++i) {
    const orc_layer* l = &d->layers[i];
    if (d->n_blocks + 3 > ORC_MAX_BLOCKS) return fail(ORC_CONFIG, "too many params");
    switch (l->kind) {
      case ORC_DENSE:
        d->block_size[d->n_blocks] = l->in * l->out;
        d->fan_in[d->n_blocks++] = l->in;
        d->block_size[d->n_blocks] = l->out;
        d->fan_in[d->n_blocks++] = 0;
        break;
      case ORC_CONV:
        d->block_size[d->n_blocks] = l->out * l->in * l->k * l->k;
        d->fan_in[d->n_blocks++] = l->in * l->k * l->k;
        d->block_size[d->n_blocks] = l->out;
        d->fan_in[d->n_blocks++] = 0;
        break;
      case ORC_EMBEDDING:
        d->block_size[d->n_blocks] = l->in * l->out;
        d->fan_in[d->n_blocks++] = l->out;
        break;
      case ORC_LSTM:
        d->block_size[d->n_blocks] = 4 * l->out * l->in;
        d->fan_in[d->n_blocks++] = l->in;
        d->block_size[d->n_blocks] = 4 * l->out * l->out;
        d->fan_in[d->n_blocks++] = l->out;
        d->block_size[d->n_blocks] = 4 * l->out;
        d->fan_in[d->n_blocks++] = 0;
        break;
      default:
        break;
    }
  }
  return ORC_OK;
}

int orc_build_desc(int32_t kind, int64_t seq_len, int64_t vocab, int64_t hidden,
                   orc_desc* d) { /* build_desc, models.cpp:87-167 */
  memset(d, 0, sizeof *d);
  d->model_kind = kind;
  const int64_t L = seq_len > 0 ? seq_len : 256;
  const int64_t V = vocab > 0 ? vocab : 10004;
  const int64_t H = hidden > 0 ? hidden : 100;
  switch (kind) {
    case ORC_LOGREG:
      add_layer(d, ORC_DENSE, 104, 1, 0, 1, 0);
      d->in_rank = 1; d->in_shape[0] = 104; d->classes = 1;
      break;
    case ORC_FCNN:
      add_layer(d, ORC_DENSE, 104, 50, 0, 1, 0);
      add_layer(d, ORC_RELU, 0, 0, 0, 1, 0);
      add_layer(d, ORC_DENSE, 50, 10, 0, 1, 0);
      d->in_rank = 1; d->in_shape[0] = 104; d->classes = 10;
      break;
    case ORC_MNIST_CNN:
      add_layer(d, ORC_CONV, 1, 16, 8, 2, 3);
      add_layer(d, ORC_RELU, 0, 0, 0, 1, 0);
      add_layer(d, ORC_MAXPOOL, 0, 0, 2, 2, 0);
      add_layer(d, ORC_CONV, 16, 32, 4, 1, 0);
      add_layer(d, ORC_RELU, 0, 0, 0, 1, 0);
      add_layer(d, ORC_FLATTEN, 0, 0, 0, 1, 0);
      add_layer(d, ORC_DENSE, 512, 32, 0, 1, 0);
      add_layer(d, ORC_RELU, 0, 0, 0, 1, 0);
      add_layer(d, ORC_DENSE, 32, 10, 0, 1, 0);
      d->in_rank = 3; d->in_shape[0] = 1; d->in_shape[1] = 28; d->in_shape[2] = 28;
      d->classes = 10;
      break;
    case ORC_CIFAR_CNN: {
      const int64_t ch[][2] = {{3, 32}, {32, 32}, {32, 64}, {64, 64},
                               {64, 128}, {128, 128}, {128, 256}, {256, 10}};
      for (int i = 0; i < 8; ++i) {
        add_layer(d, ORC_CONV, ch[i][0], ch[i][1], 3, 1, 1);
        add_layer(d, ORC_RELU, 0, 0, 0, 1, 0);
        if (i == 1 || i == 3 || i == 5) add_layer(d, ORC_AVGPOOL, 0, 0, 2, 2, 0);
      }
      d->n_layers--; /* the last conv has no relu: models.cpp:140-141 */
      add_layer(d, ORC_GLOBAL_AVGPOOL, 0, 0, 0, 1, 0);
      d->in_rank = 3; d->in_shape[0] = 3; d->in_shape[1] = 32; d->in_shape[2] = 32;
      d->classes = 10;
      break;
    }
    case ORC_EMBED: {
      const int64_t E = hidden > 0 ? hidden : 16;
      add_layer(d, ORC_EMBEDDING, V, E, 0, 1, 0);
      add_layer(d, ORC_SEQ_AVGPOOL, 0, 0, 0, 1, 0);
      add_layer(d, ORC_DENSE, E, 2, 0, 1, 0);
      d->in_rank = 1; d->in_shape[0] = L; d->classes = 2; d->token_input = 1;
      break;
    }
    case ORC_LSTM_MODEL:
      add_layer(d, ORC_EMBEDDING, V, H, 0, 1, 0);
      add_layer(d, ORC_LSTM, H, H, 0, 1, 0);
      add_layer(d, ORC_SEQ_AVGPOOL, 0, 0, 0, 1, 0);
      add_layer(d, ORC_DENSE, H, 2, 0, 1, 0);
      d->in_rank = 1; d->in_shape[0] = L; d->classes = 2; d->token_input = 1;
      break;
    default:
      return fail(ORC_CONFIG, "unknown model kind %d", kind);
  }
  return orc_finish_desc(d);
}

int64_t orc_param_count(const orc_desc* d) {
  int64_t n = 0;
  for (int p = 0; p < d->n_blocks; ++p) n += d->block_size[p];
  return n;
}

static int64_t in_numel(const orc_desc* d) {
  int64_t n = 1;
  for (int i = 0; i < d->in_rank; ++i) n *= d->in_shape[i];
  return n;
}

/* Fan-in uniform init, one stream per parameter (models.cpp:359-375). */
void orc_init_params_f64(const orc_desc* d, uint64_t seed, double* flat) {
  for (int p = 0; p < d->n_blocks; ++p) {
    rng_t r = {seed, (uint64_t)p, 0};
    const int64_t n = d->block_size[p];
    if (d->fan_in[p] == 0) {
      memset(flat, 0, sizeof(double) * n);
    } else {
      const double bound = 1.0 / sqrt((double)d->fan_in[p]);
      for (int64_t j = 0; j < n; ++j) flat[j] = rng_uniform(&r, -bound, bound);
    }
    flat += n;
  }
}

void orc_init_params_f32(const orc_desc* d, uint64_t seed, float* flat) {
  for (int p = 0; p < d->n_blocks; ++p) {
    rng_t r = {seed, (uint64_t)p, 0};
    const int64_t n = d->block_size[p];
    if (d->fan_in[p] == 0) {
      memset(flat, 0, sizeof(float) * n);
    } else {
      const float bound = (float)(1.0 / sqrt((double)d->fan_in[p]));
      for (int64_t j = 0; j < n; ++j)
        flat[j] = (float)rng_uniform(&r, (double)(-bound), (double)bound);
    }
    flat += n;
  }
}

/* ---- synthetic data: dataset.cpp:126-237 -------------------------------- */

#define SYNTH_BODY(T)                                                          \
  const int64_t row = in_numel(d);                                             \
  switch (d->model_kind) {                                                     \
    case ORC_LOGREG:                                                           \
    case ORC_FCNN: { /* synth_adult, dataset.cpp:126-159 */                    \
      const int64_t F = d->in_shape[0];                                        \
      double* w = malloc(sizeof(double) * F);                                  \
      double* rowv = malloc(sizeof(double) * F);                               \
      rng_t wr = {seed, 1, 0};                                                 \
      double wn = 0;                                                           \
      for (int64_t f = 0; f < F; ++f) { w[f] = rng_uniform(&wr, -1, 1); }      \
      for (int64_t f = 0; f < F; ++f) wn += w[f] * w[f];                       \
      wn = sqrt(wn);                                                           \
      rng_t xr = {seed, 2, 0};                                                 \
      for (int64_t i = 0; i < n; ++i) {                                        \
        double score = 0;                                                      \
        for (int attempt = 0;; ++attempt) {                                    \
          score = 0;                                                           \
          for (int64_t f = 0; f < F; ++f) {                                    \
            rowv[f] = rng_uniform(&xr, -1, 1);                                 \
            score += rowv[f] * w[f];                                           \
          }                                                                    \
          if (fabs(score) / wn >= 0.05 || attempt > 64) break;                 \
        }                                                                      \
        for (int64_t f = 0; f < F; ++f) x[i * F + f] = (T)rowv[f];             \
        y[i] = score > 0 ? (T)1 : (T)0;                                        \
      }                                                                        \
      free(w);                                                                 \
      free(rowv);                                                              \
      return ORC_OK;                                                           \
    }                                                                          \
    case ORC_EMBED:                                                            \
    case ORC_LSTM_MODEL: { /* synth_tokens, dataset.cpp:161-181 */             \
      const int64_t V = d->layers[0].in;                                       \
      rng_t r = {seed, 3, 0};                                                  \
      for (int64_t i = 0; i < n; ++i) {                                        \
        double mean = 0;                                                       \
        for (int64_t t = 0; t < row; ++t) {                                    \
          const double id = floor(rng_uniform(&r, 0, (double)V));              \
          x[i * row + t] = (T)id;                                              \
          mean += id;                                                          \
        }                                                                      \
        mean /= (double)row;                                                   \
        y[i] = mean > (V - 1) / 2.0 ? (T)1 : (T)0;                             \
      }                                                                        \
      return ORC_OK;                                                           \
    }                                                                          \
    case ORC_MNIST_CNN:                                                        \
    case ORC_CIFAR_CNN: { /* synth_images, dataset.cpp:183-201 */              \
      GAUSS(seed, 4, n * row, x);                                              \
      rng_t lr = {seed, 5, 0};                                                 \
      for (int64_t i = 0; i < n; ++i)                                          \
        y[i] = (T)floor(rng_uniform(&lr, 0, 10));                              \
      return ORC_OK;                                                           \
    }                                                                          \
  }                                                                            \
  return fail(ORC_CONFIG, "synth: bad model kind");

int orc_synth_f64(const orc_desc* d, int64_t n, uint64_t seed, double* x, double* y) {
  if (n <= 0) return fail(ORC_CONFIG, "synth: n must be positive");
#define GAUSS orc_gaussian_f64
  SYNTH_BODY(double)
#undef GAUSS
}

int orc_synth_f32(const orc_desc* d, int64_t n, uint64_t seed, float* x, float* y) {
  if (n <= 0) return fail(ORC_CONFIG, "synth: n must be positive");
#define GAUSS orc_gaussian_f32
  SYNTH_BODY(float)
#undef GAUSS
}

/* ---- per-example forward/backward (fp64) -------------------------------- */
/* Layer semantics: trace_forward, models.cpp:169-296; VJPs autodiff.cpp:
 * 121-124 (relu gt-mask), 155-159 (matmul), 160-174 (bmm), 183-185
 * (reduce_max -> first-max routing, kernels.hpp:377-396), 186-192
 * (im2col <-> col2im); per-example extraction strategies.cpp:136-188. */

typedef struct { int rank; int64_t d[3]; } shp;

static int64_t shp_numel(shp s) {
  int64_t n = 1;
  for (int i = 0; i < s.rank; ++i) n *= s.d[i];
  return n;
}

static int conv_extent(int64_t in, int64_t k, int64_t stride, int64_t pad,
                       int64_t* out) { /* kernels.hpp:400-410 */
  const int64_t span = in + 2 * pad - k;
  if (span < 0 || stride <= 0 || span % stride != 0)
    return fail(ORC_SHAPE,
                "conv window %lld stride %lld pad %lld does not produce an "
                "integral extent over %lld",
                (long long)k, (long long)stride, (long long)pad, (long long)in);
  *out = span / stride + 1;
  return ORC_OK;
}

typedef struct {
  shp s[ORC_MAX_LAYERS + 1]; /* s[l] = shape entering layer l */
  int64_t poff[ORC_MAX_LAYERS]; /* offset of layer's first param in flat */
  int pblock[ORC_MAX_LAYERS];   /* first param block ordinal, -1 if none */
  int64_t off_block[ORC_MAX_BLOCKS];
  int64_t max_act;
} plan_t;

static int make_plan(const orc_desc* d, plan_t* P) {
  memset(P, 0, sizeof *P);
  P->s[0].rank = d->in_rank;
  for (int i = 0; i < d->in_rank; ++i) P->s[0].d[i] = d->in_shape[i];
  int64_t off = 0;
  int blk = 0;
  for (int p = 0; p < d->n_blocks; ++p) {
    P->off_block[p] = off;
    off += d->block_size[p];
  }
  off = 0;
  P->max_act = shp_numel(P->s[0]);
  for (int l = 0; l < d->n_layers; ++l) {
    const orc_layer* L = &d->layers[l];
    shp in = P->s[l], out = in;
    P->pblock[l] = -1;
    P->poff[l] = off;
    int rc;
    switch (L->kind) {
      case ORC_DENSE:
        if (in.rank != 1 || in.d[0] != L->in)
          return fail(ORC_SHAPE, "dense layer %d: input does not match in=%lld", l,
                      (long long)L->in);
        out.rank = 1;
        out.d[0] = L->out;
        P->pblock[l] = blk;
        blk += 2;
        off += L->in * L->out + L->out;
        break;
      case ORC_CONV: {
        if (in.rank != 3 || in.d[0] != L->in)
          return fail(ORC_SHAPE, "conv layer %d: channel mismatch", l);
        int64_t ho = 0, wo = 0;
        if ((rc = conv_extent(in.d[1], L->k, L->stride, L->pad, &ho))) return rc;
        if ((rc = conv_extent(in.d[2], L->k, L->stride, L->pad, &wo))) return rc;
        out.d[0] = L->out;
        out.d[1] = ho;
        out.d[2] = wo;
        P->pblock[l] = blk;
        blk += 2;
        off += L->out * L->in * L->k * L->k + L->out;
        break;
      }
      case ORC_MAXPOOL:
      case ORC_AVGPOOL: {
        if (in.rank != 3) return fail(ORC_SHAPE, "pool2d expects (N,C,H,W)");
        int64_t ho = 0, wo = 0;
        if ((rc = conv_extent(in.d[1], L->k, L->stride, 0, &ho))) return rc;
        if ((rc = conv_extent(in.d[2], L->k, L->stride, 0, &wo))) return rc;
        out.d[1] = ho;
        out.d[2] = wo;
        break;
      }
      case ORC_GLOBAL_AVGPOOL:
        if (in.rank != 3) return fail(ORC_SHAPE, "global_avgpool expects (N,C,H,W)");
        out.rank = 1;
        out.d[0] = in.d[0];
        break;
      case ORC_FLATTEN:
        out.rank = 1;
        out.d[0] = shp_numel(in);
        break;
      case ORC_RELU:
        break;
      case ORC_EMBEDDING:
        if (in.rank != 1 || l != 0)
          return fail(ORC_SHAPE, "embedding expects token ids");
        out.rank = 2;
        out.d[0] = in.d[0];
        out.d[1] = L->out;
        P->pblock[l] = blk;
        blk += 1;
        off += L->in * L->out;
        break;
      case ORC_SEQ_AVGPOOL:
        if (in.rank != 2) return fail(ORC_SHAPE, "seq_avgpool expects (N,L,E)");
        out.rank = 1;
        out.d[0] = in.d[1];
        break;
      default:
        return fail(ORC_UNSUPPORTED, "unsupported layer: kind %d", L->kind);
    }
    P->s[l + 1] = out;
    if (shp_numel(out) > P->max_act) P->max_act = shp_numel(out);
  }
  const shp last = P->s[d->n_layers];
  if (last.rank != 1 || last.d[0] != (d->classes == 1 ? 1 : d->classes))
    return fail(ORC_SHAPE, "logits do not match classes");
  return ORC_OK;
}

static int checked_id(double raw, int64_t V, int64_t pos, const char* what,
                      int64_t* id) { /* kernels.hpp:475-489 */
  const int64_t v = (int64_t)llround(raw);
  if ((double)v != raw)
    return fail(ORC_INDEX, "%s: non-integral id at position %lld", what, (long long)pos);
  if (v < 0 || v >= V)
    return fail(ORC_INDEX, "%s: id %lld out of range [0,%lld) at position %lld", what,
                (long long)v, (long long)V, (long long)pos);
  *id = v;
  return ORC_OK;
}

/* One example: forward, loss, backward; writes this example's gradient
 * for every param block into g_flat (P). */
static int example_grad(const orc_desc* d, const plan_t* P, const double* x,
                        double label, const double* params, double* g_flat,
                        double** acts, double* gA, double* gB, double* loss) {
  const int nl = d->n_layers;
  memcpy(acts[0], x, sizeof(double) * shp_numel(P->s[0]));
  int rc;
  /* forward */
  for (int l = 0; l < nl; ++l) {
    const orc_layer* L = &d->layers[l];
    const shp in = P->s[l], out = P->s[l + 1];
    const double* a = acts[l];
    double* z = acts[l + 1];
    const double* W = params + P->poff[l];
    switch (L->kind) {
      case ORC_DENSE: {
        const double* b = W + L->in * L->out;
        for (int64_t o = 0; o < L->out; ++o) {
          double acc = 0;
          for (int64_t i = 0; i < L->in; ++i) acc += a[i] * W[i * L->out + o];
          z[o] = acc + b[o];
        }
        break;
      }
      case ORC_CONV: {
        const int64_t C = in.d[0], H = in.d[1], Wd = in.d[2];
        const int64_t D = out.d[0], Ho = out.d[1], Wo = out.d[2], k = L->k;
        const double* b = W + D * C * k * k;
        for (int64_t dd = 0; dd < D; ++dd)
          for (int64_t oy = 0; oy < Ho; ++oy)
            for (int64_t ox = 0; ox < Wo; ++ox) {
              double acc = 0;
              for (int64_t c = 0; c < C; ++c)
                for (int64_t u = 0; u < k; ++u) {
                  const int64_t iy = oy * L->stride + u - L->pad;
                  if (iy < 0 || iy >= H) continue;
                  for (int64_t v = 0; v < k; ++v) {
                    const int64_t ix = ox * L->stride + v - L->pad;
                    if (ix < 0 || ix >= Wd) continue;
                    acc += W[((dd * C + c) * k + u) * k + v] * a[(c * H + iy) * Wd + ix];
                  }
                }
              z[(dd * Ho + oy) * Wo + ox] = acc + b[dd];
            }
        break;
      }
      case ORC_MAXPOOL:
      case ORC_AVGPOOL: {
        const int64_t C = in.d[0], H = in.d[1], Wd = in.d[2];
        const int64_t Ho = out.d[1], Wo = out.d[2], k = L->k, s = L->stride;
        for (int64_t c = 0; c < C; ++c)
          for (int64_t oy = 0; oy < Ho; ++oy)
            for (int64_t ox = 0; ox < Wo; ++ox) {
              double m = 0, sum = 0;
              int first = 1;
              for (int64_t u = 0; u < k; ++u)
                for (int64_t v = 0; v < k; ++v) {
                  const double val = a[(c * H + oy * s + u) * Wd + ox * s + v];
                  sum += val;
                  if (first || val > m) m = val;
                  first = 0;
                }
              z[(c * Ho + oy) * Wo + ox] =
                  L->kind == ORC_MAXPOOL ? m : sum * (1.0 / (double)(k * k));
            }
        break;
      }
      case ORC_GLOBAL_AVGPOOL: {
        const int64_t C = in.d[0], HW = in.d[1] * in.d[2];
        for (int64_t c = 0; c < C; ++c) {
          double sum = 0;
          for (int64_t j = 0; j < HW; ++j) sum += a[c * HW + j];
          z[c] = sum * (1.0 / (double)HW);
        }
        break;
      }
      case ORC_FLATTEN:
        memcpy(z, a, sizeof(double) * shp_numel(in));
        break;
      case ORC_RELU: {
        const int64_t n = shp_numel(in);
        for (int64_t j = 0; j < n; ++j) z[j] = a[j] > 0 ? a[j] : 0;
        break;
      }
      case ORC_EMBEDDING: {
        const int64_t Lq = in.d[0], E = L->out;
        for (int64_t t = 0; t < Lq; ++t) {
          int64_t id;
          if ((rc = checked_id(a[t], L->in, t, "gather_rows", &id))) return rc;
          memcpy(z + t * E, W + id * E, sizeof(double) * E);
        }
        break;
      }
      case ORC_SEQ_AVGPOOL: {
        const int64_t Lq = in.d[0], E = in.d[1];
        for (int64_t e = 0; e < E; ++e) {
          double sum = 0;
          for (int64_t t = 0; t < Lq; ++t) sum += a[t * E + e];
          z[e] = sum * (1.0 / (double)Lq);
        }
        break;
      }
      default:
        return fail(ORC_UNSUPPORTED, "unsupported layer");
    }
  }
  /* loss + dlogits: softmax_xent(_grad), kernels.hpp:516-566 */
  const double* zl = acts[nl];
  double* g = gA;
  const int64_t K = d->classes;
  if (K == 1) {
    int64_t yv;
    if ((rc = checked_id(label, 2, 0, "softmax_xent label", &yv))) return rc;
    const double z = zl[0], az = fabs(z);
    *loss = (z > 0 ? z : 0) - z * (double)yv + log1p(exp(-az));
    g[0] = 1.0 / (1.0 + exp(-z)) - (double)yv;
  } else {
    int64_t yv;
    if ((rc = checked_id(label, K, 0, "softmax_xent label", &yv))) return rc;
    double m = zl[0];
    for (int64_t k = 1; k < K; ++k) if (zl[k] > m) m = zl[k];
    double s = 0;
    for (int64_t k = 0; k < K; ++k) s += exp(zl[k] - m);
    *loss = m + log(s) - zl[yv];
    for (int64_t k = 0; k < K; ++k) g[k] = exp(zl[k] - m) / s - (k == yv ? 1.0 : 0.0);
  }
  /* backward */
  for (int l = nl - 1; l >= 0; --l) {
    const orc_layer* L = &d->layers[l];
    const shp in = P->s[l], out = P->s[l + 1];
    const double* a = acts[l];
    const double* W = params + P->poff[l];
    double* gW = g_flat + P->poff[l];
    double* gx = gB;
    const int64_t nin = shp_numel(in);
    const int need_gx = l > 0; /* the first layer's input gradient is dead */
    switch (L->kind) {
      case ORC_DENSE: {
        for (int64_t i = 0; i < L->in; ++i)
          for (int64_t o = 0; o < L->out; ++o) gW[i * L->out + o] = a[i] * g[o];
        for (int64_t o = 0; o < L->out; ++o) gW[L->in * L->out + o] = g[o];
        if (need_gx)
          for (int64_t i = 0; i < L->in; ++i) {
            double acc = 0;
            for (int64_t o = 0; o < L->out; ++o) acc += g[o] * W[i * L->out + o];
            gx[i] = acc;
          }
        break;
      }
      case ORC_CONV: {
        const int64_t C = in.d[0], H = in.d[1], Wd = in.d[2];
        const int64_t D = out.d[0], Ho = out.d[1], Wo = out.d[2], k = L->k;
        double* gb = gW + D * C * k * k;
        memset(gW, 0, sizeof(double) * (D * C * k * k + D));
        if (need_gx) memset(gx, 0, sizeof(double) * nin);
        for (int64_t dd = 0; dd < D; ++dd)
          for (int64_t oy = 0; oy < Ho; ++oy)
            for (int64_t ox = 0; ox < Wo; ++ox) {
              const double gv = g[(dd * Ho + oy) * Wo + ox];
              gb[dd] += gv;
              for (int64_t c = 0; c < C; ++c)
                for (int64_t u = 0; u < k; ++u) {
                  const int64_t iy = oy * L->stride + u - L->pad;
                  if (iy < 0 || iy >= H) continue;
                  for (int64_t v = 0; v < k; ++v) {
                    const int64_t ix = ox * L->stride + v - L->pad;
                    if (ix < 0 || ix >= Wd) continue;
                    const int64_t wi = ((dd * C + c) * k + u) * k + v;
                    const int64_t xi = (c * H + iy) * Wd + ix;
                    gW[wi] += gv * a[xi];
                    if (need_gx) gx[xi] += gv * W[wi];
                  }
                }
            }
        break;
      }
      case ORC_MAXPOOL:
      case ORC_AVGPOOL: {
        const int64_t C = in.d[0], H = in.d[1], Wd = in.d[2];
        const int64_t Ho = out.d[1], Wo = out.d[2], k = L->k, s = L->stride;
        memset(gx, 0, sizeof(double) * nin);
        for (int64_t c = 0; c < C; ++c)
          for (int64_t oy = 0; oy < Ho; ++oy)
            for (int64_t ox = 0; ox < Wo; ++ox) {
              const double gv = g[(c * Ho + oy) * Wo + ox];
              if (L->kind == ORC_AVGPOOL) {
                for (int64_t u = 0; u < k; ++u)
                  for (int64_t v = 0; v < k; ++v)
                    gx[(c * H + oy * s + u) * Wd + ox * s + v] += gv * (1.0 / (double)(k * k));
              } else {
                int64_t best = -1;
                double bv = 0;
                for (int64_t u = 0; u < k; ++u)
                  for (int64_t v = 0; v < k; ++v) {
                    const int64_t xi = (c * H + oy * s + u) * Wd + ox * s + v;
                    if (best < 0 || a[xi] > bv) { bv = a[xi]; best = xi; }
                  }
                gx[best] += gv;
              }
            }
        break;
      }
      case ORC_GLOBAL_AVGPOOL: {
        const int64_t C = in.d[0], HW = in.d[1] * in.d[2];
        for (int64_t c = 0; c < C; ++c)
          for (int64_t j = 0; j < HW; ++j) gx[c * HW + j] = g[c] * (1.0 / (double)HW);
        break;
      }
      case ORC_FLATTEN:
        memcpy(gx, g, sizeof(double) * nin);
        break;
      case ORC_RELU:
        for (int64_t j = 0; j < nin; ++j) gx[j] = a[j] > 0 ? g[j] : 0;
        break;
      case ORC_EMBEDDING: {
        const int64_t Lq = in.d[0], E = L->out;
        memset(gW, 0, sizeof(double) * L->in * E);
        for (int64_t t = 0; t < Lq; ++t) {
          const int64_t id = (int64_t)llround(a[t]);
          for (int64_t e = 0; e < E; ++e) gW[id * E + e] += g[t * E + e];
        }
        break;
      }
      case ORC_SEQ_AVGPOOL: {
        const int64_t Lq = in.d[0], E = in.d[1];
        for (int64_t t = 0; t < Lq; ++t)
          for (int64_t e = 0; e < E; ++e) gx[t * E + e] = g[e] * (1.0 / (double)Lq);
        break;
      }
      default:
        return fail(ORC_UNSUPPORTED, "unsupported layer");
    }
    /* swap cotangent buffers */
    double* t = gA;
    gA = gB;
    gB = t;
    g = gA;
  }
  return ORC_OK;
}

int orc_per_example_grads(const orc_desc* d, int64_t B, const double* x,
                          const double* y, const double* params,
                          double* stacks, double* normsq, double* losses) {
  plan_t P;
  int rc = make_plan(d, &P);
  if (rc) return rc;
  if (B <= 0) return fail(ORC_CONTRACT, "batch must be positive");
  const int64_t Ptot = orc_param_count(d);
  const int64_t row = in_numel(d);
  double* buf = malloc(sizeof(double) * (P.max_act * (d->n_layers + 3) + Ptot));
  double* acts[ORC_MAX_LAYERS + 1];
  for (int l = 0; l <= d->n_layers; ++l) acts[l] = buf + l * P.max_act;
  double* gA = buf + (d->n_layers + 1) * P.max_act;
  double* gB = gA + P.max_act;
  double* gi = gB + P.max_act;
  for (int64_t i = 0; i < B && rc == ORC_OK; ++i) {
    double loss = 0;
    rc = example_grad(d, &P, x + i * row, y[i], params, gi, acts, gA, gB, &loss);
    if (rc) break;
    if (losses) losses[i] = loss;
    if (stacks)
      for (int p = 0; p < d->n_blocks; ++p)
        memcpy(stacks + P.off_block[p] * B + i * d->block_size[p],
               gi + P.off_block[p], sizeof(double) * d->block_size[p]);
    if (normsq) {
      double acc = 0;
      for (int64_t j = 0; j < Ptot; ++j) acc += gi[j] * gi[j];
      normsq[i] = acc;
    }
  }
  free(buf);
  return rc;
}

static uint64_t noise_stream(int64_t step, int p) { /* dpsgd.cpp:27-32 */
  return ((uint64_t)1 << 32) + (uint64_t)step * 4096 + (uint64_t)p;
}

int orc_dpsgd_step(const orc_desc* d, int64_t B, const double* x,
                   const double* y, double* params, double clip, double sigma,
                   double lr, int64_t m, uint64_t seed, int64_t step,
                   double* norms, int64_t* clipped, double* clipped_sum) {
  /* validate, dpsgd.cpp:36-51 */
  if (!(clip > 0)) return fail(ORC_CONFIG, "DpConfig: clip norm must be positive");
  if (sigma < 0) return fail(ORC_CONFIG, "DpConfig: noise multiplier must be non-negative");
  if (!(lr > 0)) return fail(ORC_CONFIG, "DpConfig: learning rate must be positive");
  if (m < 1 || B % m != 0)
    return fail(ORC_CONFIG, "DpConfig: microbatch size %lld must divide the batch size %lld",
                (long long)m, (long long)B);
  const int64_t Ptot = orc_param_count(d);
  plan_t P;
  int rc = make_plan(d, &P);
  if (rc) return rc;
  double* stacks = malloc(sizeof(double) * Ptot * B);
  rc = orc_per_example_grads(d, B, x, y, params, stacks, NULL, NULL);
  if (rc) { free(stacks); return rc; }
  /* microbatch means (dpsgd.cpp:102-132); m = 1 is the identity */
  const int64_t U = B / m;
  double* units = stacks;
  if (m > 1) {
    units = calloc((size_t)(Ptot * U), sizeof(double));
    for (int p = 0; p < d->n_blocks; ++p) {
      const int64_t per = d->block_size[p];
      const double* src = stacks + P.off_block[p] * B;
      double* dst = units + P.off_block[p] * U;
      for (int64_t u = 0; u < U; ++u) {
        for (int64_t j = 0; j < m; ++j)
          for (int64_t e = 0; e < per; ++e) dst[u * per + e] += src[(u * m + j) * per + e];
        for (int64_t e = 0; e < per; ++e) dst[u * per + e] *= 1.0 / (double)m;
      }
    }
  }
  /* norms + clip factors (dpsgd.cpp:54-99, 254-275) */
  double* s = malloc(sizeof(double) * U);
  int64_t nclip = 0;
  for (int64_t u = 0; u < U; ++u) {
    double acc = 0;
    for (int p = 0; p < d->n_blocks; ++p) {
      const int64_t per = d->block_size[p];
      const double* v = units + P.off_block[p] * U + u * per;
      for (int64_t e = 0; e < per; ++e) acc += v[e] * v[e];
    }
    const double n = sqrt(acc);
    if (norms) norms[u] = n;
    s[u] = n > clip ? clip / n : 1.0;
    if (n > clip) ++nclip;
  }
  if (clipped) *clipped = nclip;
  /* clipped sum, noise, mean, update (dpsgd.cpp:135-183, 277-322) */
  double* noise = NULL;
  for (int p = 0; p < d->n_blocks; ++p) {
    const int64_t per = d->block_size[p];
    const double* src = units + P.off_block[p] * U;
    double* prm = params + P.off_block[p];
    double* acc = calloc((size_t)per, sizeof(double));
    for (int64_t u = 0; u < U; ++u)
      for (int64_t e = 0; e < per; ++e) acc[e] += src[u * per + e] * s[u];
    if (clipped_sum) memcpy(clipped_sum + P.off_block[p], acc, sizeof(double) * per);
    if (sigma > 0) {
      noise = realloc(noise, sizeof(double) * per);
      orc_gaussian_f64(seed, noise_stream(step, p), per, noise);
      for (int64_t e = 0; e < per; ++e) acc[e] += sigma * clip * noise[e];
    }
    for (int64_t e = 0; e < per; ++e) prm[e] -= lr * (acc[e] * (1.0 / (double)U));
    free(acc);
  }
  free(noise);
  free(s);
  if (units != stacks) free(units);
  free(stacks);
  return ORC_OK;
}

int orc_sgd_step(const orc_desc* d, int64_t B, const double* x,
                 const double* y, double* params, double lr) {
  const int64_t Ptot = orc_param_count(d);
  plan_t P;
  int rc = make_plan(d, &P);
  if (rc) return rc;
  double* stacks = malloc(sizeof(double) * Ptot * B);
  rc = orc_per_example_grads(d, B, x, y, params, stacks, NULL, NULL);
  if (!rc) {
    for (int p = 0; p < d->n_blocks; ++p) {
      const int64_t per = d->block_size[p];
      const double* src = stacks + P.off_block[p] * B;
      for (int64_t e = 0; e < per; ++e) {
        double acc = 0;
        for (int64_t i = 0; i < B; ++i) acc += src[i * per + e];
        params[P.off_block[p] + e] -= lr * (acc * (1.0 / (double)B));
      }
    }
  }
  free(stacks);
  return rc;
}

/* ---- fp32 views-path tail, exact reference op order -------------------- */

static double sumsq_lanes_f32(const float* p, int64_t n) { /* kernels.hpp:573-589 */
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    const double v0 = p[i], v1 = p[i + 1], v2 = p[i + 2], v3 = p[i + 3];
    a0 += v0 * v0;
    a1 += v1 * v1;
    a2 += v2 * v2;
    a3 += v3 * v3;
  }
  for (; i < n; ++i) {
    const double v = p[i];
    a0 += v * v;
  }
  return (a0 + a1) + (a2 + a3);
}

int orc_aggregate_f32(int64_t B, int32_t n_blocks, const int64_t* bs,
                      const float* stacks, float* params, float clip,
                      float sigma, float lr, uint64_t seed, int64_t step,
                      float* norms, int64_t* clipped) {
  float* s = malloc(sizeof(float) * B);
  int64_t nclip = 0;
  for (int64_t i = 0; i < B; ++i) { /* dpsgd.cpp:254-270 */
    double acc = 0;
    const float* blk = stacks;
    for (int p = 0; p < n_blocks; ++p) {
      acc += sumsq_lanes_f32(blk + i * bs[p], bs[p]);
      blk += bs[p] * B;
    }
    const float n = (float)sqrt(acc);
    if (norms) norms[i] = n;
    s[i] = n > clip ? clip / n : 1.0f;
    if (n > clip) ++nclip;
  }
  if (clipped) *clipped = nclip;
  const float inv = 1.0f / (float)B;
  const float scale = sigma * clip;
  const float* blk = stacks;
  for (int p = 0; p < n_blocks; ++p) { /* dpsgd.cpp:277-322 */
    const int64_t per = bs[p];
    float* a = calloc((size_t)per, sizeof(float));
    for (int64_t i = 0; i < B; ++i) {
      const float si = s[i];
      for (int64_t j = 0; j < per; ++j) {
        const float scaled = blk[i * per + j] * si;
        a[j] += scaled;
      }
    }
    if (sigma > 0) {
      float* n = malloc(sizeof(float) * per);
      orc_gaussian_f32(seed, noise_stream(step, p), per, n);
      for (int64_t j = 0; j < per; ++j) {
        const float t = scale * n[j];
        a[j] += t;
      }
      free(n);
    }
    for (int64_t j = 0; j < per; ++j) a[j] *= inv;
    for (int64_t j = 0; j < per; ++j) { /* apply_update, dpsgd.cpp:173-183 */
      const float t = lr * a[j];
      params[j] = params[j] - t;
    }
    params += per;
    blk += per * B;
    free(a);
  }
  free(s);
  return ORC_OK;
}
