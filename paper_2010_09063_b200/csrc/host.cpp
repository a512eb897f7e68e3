// Host side of libpegrad_b200.so: model descriptions, parameter init,
// synthetic datasets, config validation and the error channel. Everything
// here is bit-compatible with the reference's host code it replaces:
//   build_desc / register_params   proj/core/src/models.cpp:50-167
//   build_from_desc (init)          proj/core/src/models.cpp:359-375
//   synth_for_model                 proj/core/src/dataset.cpp:126-237
//   validate (DpConfig)             proj/core/src/dpsgd.cpp:36-51
//   check_strategy_support          proj/core/src/strategies.cpp:76-113
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <thread>
#include <vector>

#include "pgb_internal.h"

namespace pgb {

namespace {
thread_local std::string g_last_error;

struct Rng {  // RngState (rng.hpp:25-32) with sequential draws
  uint64_t key, counter = 0;
  Rng(uint64_t seed, uint64_t stream) : key(stream_key(seed, stream)) {}
  double unit() { return double(value_at(key, counter++) >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
};

void add_layer(pgb_model_desc& d, int32_t kind, int64_t in = 0, int64_t out = 0,
               int64_t k = 0, int64_t stride = 1, int64_t pad = 0) {
  if (d.n_layers >= PGB_MAX_LAYERS) raise(PGB_ERR_CONFIG, "too many layers");
  d.layers[d.n_layers++] = pgb_layer_spec{kind, in, out, k, stride, pad};
}

// Box-Muller pair (kernels.hpp:597-614) on the host, for synthetic images.
void gaussian_fill(uint64_t seed, uint64_t stream, float* out, int64_t n) {
  const uint64_t key = stream_key(seed, stream);
  const int64_t pairs = (n + 1) / 2;
  auto body = [&](int64_t lo, int64_t hi) {
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    for (int64_t q = lo; q < hi; ++q) {
      const double u1 = double((value_at(key, 2 * q) >> 11) + 1) * 0x1.0p-53;
      const double u2 = double((value_at(key, 2 * q + 1) >> 11) + 1) * 0x1.0p-53;
      const double r = std::sqrt(-2.0 * std::log(u1));
      out[2 * q] = static_cast<float>(r * std::cos(kTwoPi * u2));
      if (2 * q + 1 < n) out[2 * q + 1] = static_cast<float>(r * std::sin(kTwoPi * u2));
    }
  };
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = pairs < (1 << 16) ? 1 : std::min<int64_t>(hw, 16);
  if (nt == 1) {
    body(0, pairs);
    return;
  }
  std::vector<std::thread> ts;
  for (int64_t t = 0; t < nt; ++t)
    ts.emplace_back(body, pairs * t / nt, pairs * (t + 1) / nt);
  for (auto& t : ts) t.join();
}

}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

const char* layer_kind_name(int32_t k) {
  static const char* names[] = {"dense", "conv", "maxpool", "avgpool", "global_avgpool",
                                "flatten", "relu", "embedding", "seq_avgpool", "lstm"};
  return (k >= 0 && k < 10) ? names[k] : "?";
}

static const char* model_name(int32_t k) {
  static const char* names[] = {"logreg", "fcnn", "mnist_cnn", "cifar_cnn", "embed", "lstm"};
  return (k >= 0 && k < 6) ? names[k] : "?";
}

static const char* strategy_name(int32_t s) {
  static const char* names[] = {"naive", "vmap", "outer", "norms", "groupconv", "jacmm"};
  return (s >= 0 && s < 6) ? names[s] : "?";
}

int64_t conv_out_extent(int64_t in, int64_t k, int64_t stride, int64_t pad) {
  const int64_t span = in + 2 * pad - k;
  if (span < 0 || stride <= 0 || span % stride != 0)
    raise(PGB_ERR_SHAPE, "conv window " + std::to_string(k) + " stride " +
                             std::to_string(stride) + " pad " + std::to_string(pad) +
                             " does not produce an integral extent over " +
                             std::to_string(in));
  return span / stride + 1;
}

void layer_shapes(const pgb_model_desc& d, ExShape* s) {
  s[0].rank = d.input_rank;
  for (int i = 0; i < d.input_rank; ++i) s[0].d[i] = d.input_shape[i];
  for (int l = 0; l < d.n_layers; ++l) {
    const pgb_layer_spec& L = d.layers[l];
    const ExShape in = s[l];
    ExShape out = in;
    switch (L.kind) {
      case PGB_DENSE:
        if (in.rank != 1 || in.d[0] != L.in)
          raise(PGB_ERR_SHAPE, "dense layer " + std::to_string(l) + ": input " +
                                   std::to_string(in.numel()) + " features, layer expects " +
                                   std::to_string(L.in));
        out.rank = 1;
        out.d[0] = L.out;
        break;
      case PGB_CONV:
        if (in.rank != 3 || in.d[0] != L.in)
          raise(PGB_ERR_SHAPE, "conv layer " + std::to_string(l) + ": channel mismatch");
        out.d[0] = L.out;
        out.d[1] = conv_out_extent(in.d[1], L.k, L.stride, L.pad);
        out.d[2] = conv_out_extent(in.d[2], L.k, L.stride, L.pad);
        break;
      case PGB_MAXPOOL:
      case PGB_AVGPOOL:
        if (in.rank != 3) raise(PGB_ERR_SHAPE, "pool2d expects (N,C,H,W)");
        out.d[1] = conv_out_extent(in.d[1], L.k, L.stride, 0);
        out.d[2] = conv_out_extent(in.d[2], L.k, L.stride, 0);
        break;
      case PGB_GLOBAL_AVGPOOL:
        if (in.rank != 3) raise(PGB_ERR_SHAPE, "global_avgpool expects (N,C,H,W)");
        out.rank = 1;
        out.d[0] = in.d[0];
        break;
      case PGB_FLATTEN:
        out.rank = 1;
        out.d[0] = in.numel();
        break;
      case PGB_RELU:
        break;
      case PGB_EMBEDDING:
        if (in.rank != 1 || l != 0) raise(PGB_ERR_SHAPE, "embedding expects token ids");
        out.rank = 2;
        out.d[0] = in.d[0];
        out.d[1] = L.out;
        break;
      case PGB_SEQ_AVGPOOL:
        if (in.rank != 2) raise(PGB_ERR_SHAPE, "seq_avgpool expects (N,L,E)");
        out.rank = 1;
        out.d[0] = in.d[1];
        break;
      default:
        raise(PGB_ERR_UNSUPPORTED, std::string("unsupported layer: ") + layer_kind_name(L.kind));
    }
    s[l + 1] = out;
  }
  const ExShape& last = s[d.n_layers];
  if (last.rank != 1 || last.d[0] != d.classes)
    raise(PGB_ERR_SHAPE, "logits (" + std::to_string(last.numel()) +
                             ") do not match the class count " + std::to_string(d.classes));
}

void validate_dp_config(const pgb_dp_config& c, int64_t batch) {  // dpsgd.cpp:36-51
  if (!(c.clip_norm > 0.0f)) raise(PGB_ERR_CONFIG, "DpConfig: clip norm must be positive");
  if (c.noise_multiplier < 0.0f)
    raise(PGB_ERR_CONFIG, "DpConfig: noise multiplier must be non-negative");
  if (!(c.learning_rate > 0.0f)) raise(PGB_ERR_CONFIG, "DpConfig: learning rate must be positive");
  if (c.microbatch < 1 || batch % c.microbatch != 0)
    raise(PGB_ERR_CONFIG, "DpConfig: microbatch size " + std::to_string(c.microbatch) +
                              " must divide the batch size " + std::to_string(batch));
}

void check_strategy_support(int32_t s, const pgb_model_desc& d) {  // strategies.cpp:76-113
  if (s < 0 || s > PGB_JACMM) raise(PGB_ERR_CONFIG, "unknown strategy " + std::to_string(s));
  for (int i = 0; i < d.n_layers; ++i) {
    const int32_t k = d.layers[i].kind;
    bool ok = true;
    switch (s) {
      case PGB_NAIVE:
      case PGB_VMAP:
        ok = true;
        break;
      case PGB_OUTER:
      case PGB_NORMS:
        ok = k == PGB_DENSE || k == PGB_RELU;
        break;
      case PGB_GROUPCONV:
        ok = k == PGB_DENSE || k == PGB_RELU || k == PGB_CONV || k == PGB_MAXPOOL ||
             k == PGB_AVGPOOL || k == PGB_GLOBAL_AVGPOOL || k == PGB_FLATTEN;
        break;
      case PGB_JACMM:
        ok = k != PGB_LSTM;
        break;
    }
    if (!ok)
      raise(PGB_ERR_UNSUPPORTED, std::string("unsupported layer: ") + layer_kind_name(k) +
                                     " (strategy " + strategy_name(s) + ", model " +
                                     model_name(d.model_kind) + ")");
  }
}

}  // namespace pgb

using namespace pgb;

extern "C" {

const char* pgb_last_error(void) { return g_last_error.c_str(); }
const char* pgb_version(void) { return "pegrad_b200 0.1 (sm_100a)"; }

pgb_status pgb_finish_desc(pgb_model_desc* d) {  // register_params, models.cpp:50-83
  return guarded([&] {
    if (!d) raise(PGB_ERR_CONTRACT, "null desc");
    d->n_params = 0;
    auto add = [&](int64_t size, int64_t fan) {
      if (d->n_params >= PGB_MAX_PARAMS) raise(PGB_ERR_CONFIG, "too many parameters");
      d->param_size[d->n_params] = size;
      d->param_fan_in[d->n_params++] = fan;
    };
    for (int i = 0; i < d->n_layers; ++i) {
      const pgb_layer_spec& l = d->layers[i];
      switch (l.kind) {
        case PGB_DENSE:
          add(l.in * l.out, l.in);
          add(l.out, 0);
          break;
        case PGB_CONV:
          add(l.out * l.in * l.k * l.k, l.in * l.k * l.k);
          add(l.out, 0);
          break;
        case PGB_EMBEDDING:
          add(l.in * l.out, l.out);
          break;
        case PGB_LSTM:
          add(4 * l.out * l.in, l.in);
          add(4 * l.out * l.out, l.out);
          add(4 * l.out, 0);
          break;
        default:
          break;
      }
    }
  });
}

pgb_status pgb_build_desc(int32_t kind, const pgb_model_options* opts, pgb_model_desc* out) {
  return guarded([&] {  // models.cpp:87-167
    if (!out) raise(PGB_ERR_CONTRACT, "null desc");
    pgb_model_desc d;
    std::memset(&d, 0, sizeof d);
    d.model_kind = kind;
    const int64_t L = opts && opts->seq_len > 0 ? opts->seq_len : 256;
    const int64_t V = opts && opts->vocab > 0 ? opts->vocab : 10004;
    const int64_t H = opts && opts->hidden > 0 ? opts->hidden : 100;
    switch (kind) {
      case PGB_LOGREG:
        add_layer(d, PGB_DENSE, 104, 1);
        d.input_rank = 1;
        d.input_shape[0] = 104;
        d.classes = 1;
        break;
      case PGB_FCNN:
        add_layer(d, PGB_DENSE, 104, 50);
        add_layer(d, PGB_RELU);
        add_layer(d, PGB_DENSE, 50, 10);
        d.input_rank = 1;
        d.input_shape[0] = 104;
        d.classes = 10;
        break;
      case PGB_MNIST_CNN:
        add_layer(d, PGB_CONV, 1, 16, 8, 2, 3);
        add_layer(d, PGB_RELU);
        add_layer(d, PGB_MAXPOOL, 0, 0, 2, 2);
        add_layer(d, PGB_CONV, 16, 32, 4, 1, 0);
        add_layer(d, PGB_RELU);
        add_layer(d, PGB_FLATTEN);
        add_layer(d, PGB_DENSE, 512, 32);
        add_layer(d, PGB_RELU);
        add_layer(d, PGB_DENSE, 32, 10);
        d.input_rank = 3;
        d.input_shape[0] = 1;
        d.input_shape[1] = 28;
        d.input_shape[2] = 28;
        d.classes = 10;
        break;
      case PGB_CIFAR_CNN: {
        const int64_t ch[8][2] = {{3, 32},   {32, 32},   {32, 64},   {64, 64},
                                  {64, 128}, {128, 128}, {128, 256}, {256, 10}};
        for (int i = 0; i < 8; ++i) {
          add_layer(d, PGB_CONV, ch[i][0], ch[i][1], 3, 1, 1);
          if (i < 7) add_layer(d, PGB_RELU);
          if (i == 1 || i == 3 || i == 5) add_layer(d, PGB_AVGPOOL, 0, 0, 2, 2);
        }
        add_layer(d, PGB_GLOBAL_AVGPOOL);
        d.input_rank = 3;
        d.input_shape[0] = 3;
        d.input_shape[1] = 32;
        d.input_shape[2] = 32;
        d.classes = 10;
        break;
      }
      case PGB_EMBED: {
        const int64_t E = opts && opts->hidden > 0 ? opts->hidden : 16;
        add_layer(d, PGB_EMBEDDING, V, E);
        add_layer(d, PGB_SEQ_AVGPOOL);
        add_layer(d, PGB_DENSE, E, 2);
        d.input_rank = 1;
        d.input_shape[0] = L;
        d.classes = 2;
        d.token_input = 1;
        break;
      }
      case PGB_LSTM_MODEL:
        add_layer(d, PGB_EMBEDDING, V, H);
        add_layer(d, PGB_LSTM, H, H);
        add_layer(d, PGB_SEQ_AVGPOOL);
        add_layer(d, PGB_DENSE, H, 2);
        d.input_rank = 1;
        d.input_shape[0] = L;
        d.classes = 2;
        d.token_input = 1;
        break;
      default:
        raise(PGB_ERR_CONFIG, "unknown model kind " + std::to_string(kind) +
                                  " (expected one of logreg, fcnn, mnist_cnn, cifar_cnn, "
                                  "embed, lstm)");
    }
    *out = d;
    const pgb_status st = pgb_finish_desc(out);
    if (st != PGB_OK) raise(st, g_last_error);
  });
}

int64_t pgb_param_count(const pgb_model_desc* d) {
  int64_t n = 0;
  for (int i = 0; d && i < d->n_params; ++i) n += d->param_size[i];
  return n;
}

pgb_status pgb_init_params(const pgb_model_desc* d, uint64_t seed, float* flat) {
  return guarded([&] {  // build_from_desc, models.cpp:359-375
    if (!d || !flat) raise(PGB_ERR_CONTRACT, "null argument");
    for (int p = 0; p < d->n_params; ++p) {
      const int64_t n = d->param_size[p];
      if (d->param_fan_in[p] == 0) {
        std::memset(flat, 0, sizeof(float) * n);
      } else {
        Rng rng(seed, uint64_t(p));
        const float bound = static_cast<float>(1.0 / std::sqrt(double(d->param_fan_in[p])));
        const double lo = static_cast<double>(-bound), hi = static_cast<double>(bound);
        for (int64_t j = 0; j < n; ++j) flat[j] = static_cast<float>(rng.uniform(lo, hi));
      }
      flat += n;
    }
  });
}

pgb_status pgb_synth(const pgb_model_desc* d, int64_t n, uint64_t seed, float* x, float* y) {
  return guarded([&] {  // dataset.cpp:126-237
    if (!d || !x || !y) raise(PGB_ERR_CONTRACT, "null argument");
    if (n <= 0) raise(PGB_ERR_CONFIG, "synth: n must be positive");
    int64_t row = 1;
    for (int i = 0; i < d->input_rank; ++i) row *= d->input_shape[i];
    switch (d->model_kind) {
      case PGB_LOGREG:
      case PGB_FCNN: {  // synth_adult: planted rule with a margin
        const int64_t F = d->input_shape[0];
        Rng wr(seed, 1);
        std::vector<double> w(F), r(F);
        for (auto& v : w) v = wr.uniform(-1, 1);
        double wn = 0;
        for (double v : w) wn += v * v;
        wn = std::sqrt(wn);
        Rng xr(seed, 2);
        for (int64_t i = 0; i < n; ++i) {
          double score = 0;
          for (int attempt = 0;; ++attempt) {
            score = 0;
            for (int64_t f = 0; f < F; ++f) {
              r[f] = xr.uniform(-1, 1);
              score += r[f] * w[f];
            }
            if (std::abs(score) / wn >= 0.05 || attempt > 64) break;
          }
          for (int64_t f = 0; f < F; ++f) x[i * F + f] = static_cast<float>(r[f]);
          y[i] = score > 0 ? 1.0f : 0.0f;
        }
        break;
      }
      case PGB_EMBED:
      case PGB_LSTM_MODEL: {  // synth_tokens
        const int64_t V = d->layers[0].in;
        Rng r(seed, 3);
        for (int64_t i = 0; i < n; ++i) {
          double mean = 0;
          for (int64_t t = 0; t < row; ++t) {
            const double id = std::floor(r.uniform(0, double(V)));
            x[i * row + t] = static_cast<float>(id);
            mean += id;
          }
          mean /= double(row);
          y[i] = mean > (V - 1) / 2.0 ? 1.0f : 0.0f;
        }
        break;
      }
      case PGB_MNIST_CNN:
      case PGB_CIFAR_CNN: {  // synth_images: N(0,1) pixels, uniform labels
        gaussian_fill(seed, 4, x, n * row);
        Rng lr(seed, 5);
        for (int64_t i = 0; i < n; ++i) y[i] = static_cast<float>(std::floor(lr.uniform(0, 10)));
        break;
      }
      default:
        raise(PGB_ERR_CONFIG, "synth_for_model: bad model kind");
    }
  });
}

// ---- bench::train's shuffle (proj/core/src/harness.cpp:337-343) ---------------
pgb_status pgb_shuffle_order(uint64_t seed, int64_t epoch, int64_t n, int64_t* order) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !order)) raise(PGB_ERR_CONTRACT, "shuffle_order: bad arguments");
    const uint64_t key = pgb::stream_key(seed, (uint64_t(1) << 40) + (uint64_t)epoch);
    uint64_t ctr = 0;
    for (int64_t i = n - 1; i > 0; --i) {
      const double u = static_cast<double>(pgb::value_at(key, ctr++) >> 11) * 0x1.0p-53;
      const int64_t j = static_cast<int64_t>(0.0 + (static_cast<double>(i + 1) - 0.0) * u);
      std::swap(order[i], order[j]);
    }
  });
}

// ---- IDX containers (io::load_idx, proj/core/src/dataset.cpp:35-82) -----------
pgb_status pgb_idx_info(const char* path, int32_t* rank, int64_t* dims, int64_t* count) {
  return guarded([&] {
    if (!path || !rank || !dims || !count) raise(PGB_ERR_CONTRACT, "null argument");
    pgb::IdxArray a = pgb::read_idx(path);
    *rank = (int32_t)a.dims.size();
    for (size_t d = 0; d < a.dims.size(); ++d) dims[d] = a.dims[d];
    *count = (int64_t)(a.bytes.size() - a.offset);
  });
}

pgb_status pgb_load_idx(const char* path, float scale_div, float* out, int64_t capacity) {
  return guarded([&] {
    if (!path || !out) raise(PGB_ERR_CONTRACT, "null argument");
    pgb::IdxArray a = pgb::read_idx(path);
    const size_t n = a.bytes.size() - a.offset;
    if (capacity < 0 || n > static_cast<size_t>(capacity))
      raise(PGB_ERR_CONTRACT, "load_idx: payload of " + std::to_string(n) +
                                  " elements exceeds the output capacity " +
                                  std::to_string(capacity));
    const unsigned char* b = a.bytes.data() + a.offset;
    for (size_t i = 0; i < n; ++i) {
      const float v = static_cast<float>(b[i]);
      out[i] = scale_div > 0.0f ? v / scale_div : v;
    }
  });
}

}  // extern "C"

namespace pgb {

namespace {
uint32_t be32(const unsigned char* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
}
}  // namespace

// Same checks and error offsets as the reference's loader.
IdxArray read_idx(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) raise(PGB_ERR_IO, "load_idx: cannot open '" + path + "'");
  IdxArray a;
  a.bytes.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
  if (a.bytes.size() < 4)
    raise(PGB_ERR_FORMAT, "load_idx: '" + path + "' truncated at offset 0 (" +
                              std::to_string(a.bytes.size()) + " bytes)");
  const uint32_t magic = be32(a.bytes.data());
  if ((magic >> 16) != 0 || ((magic >> 8) & 0xff) != 0x08) {
    char buf[16];
    std::snprintf(buf, sizeof(buf), "%08x", magic);
    raise(PGB_ERR_FORMAT, std::string("load_idx: bad magic 0x") + buf +
                              " at offset 0 (expected an unsigned-byte IDX array)");
  }
  const uint32_t ndim = magic & 0xff;
  if (ndim < 1 || ndim > 4)
    raise(PGB_ERR_FORMAT, "load_idx: unsupported rank " + std::to_string(ndim) + " at offset 3");
  size_t offset = 4;
  int64_t total = 1;
  for (uint32_t d = 0; d < ndim; ++d) {
    if (a.bytes.size() < offset + 4)
      raise(PGB_ERR_FORMAT, "load_idx: truncated dims at offset " + std::to_string(offset));
    const int64_t extent = be32(a.bytes.data() + offset);
    a.dims.push_back(extent);
    // the dimension product must fit the payload arithmetic (and size_t)
    if (extent != 0 && total > (int64_t(1) << 62) / extent)
      raise(PGB_ERR_FORMAT, "load_idx: dimension product overflows at offset " +
                                std::to_string(offset));
    total *= extent;
    offset += 4;
  }
  if (a.bytes.size() != offset + static_cast<size_t>(total))
    raise(PGB_ERR_FORMAT, "load_idx: payload size mismatch at offset " + std::to_string(offset) +
                              " (want " + std::to_string(total) + " bytes, have " +
                              std::to_string(a.bytes.size() - offset) + ")");
  a.offset = offset;
  return a;
}

}  // namespace pgb
