// pegrad_b200.hpp -- the reference's C++ API shapes over the C ABI.
//
// A pegrad user (proj/core/include/pegrad/{models,strategies,dpsgd}.hpp)
// switches by including this header and linking libpegrad_b200.so:
//
//   pegrad::models::build<float>(kind, seed)        -> pegrad_b200::models::build(kind, seed)
//   pegrad::GradEngine<float>(model, s, B, graph)   -> pegrad_b200::GradEngine(model, s, B)
//   pegrad::dpsgd_step(model, engine, x, y, cfg, i) -> pegrad_b200::dpsgd_step(...)  (same
//                                                      argument meaning, StepReport, errors)
//   pegrad::io::synth_for_model<float>(desc, n, s)  -> pegrad_b200::io::synth_for_model(...)
//
// Header-only; every call goes through include/pegrad_b200.h. Status codes
// are rethrown as the reference's exception types (common.hpp:56-114).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pegrad_b200.h"

namespace pegrad_b200 {

// ---- errors: pegrad::Error hierarchy ------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct IndexError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct UnsupportedError : Error { using Error::Error; };
struct TraceError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };
struct NcclError : Error { using Error::Error; };
struct OutOfMemoryError : Error { using Error::Error; };

inline void check(pgb_status s) {
  if (s == PGB_OK) return;
  const std::string m = pgb_last_error();
  switch (s) {
    case PGB_ERR_SHAPE: throw ShapeError(m);
    case PGB_ERR_DOMAIN: throw DomainError(m);
    case PGB_ERR_INDEX: throw IndexError(m);
    case PGB_ERR_CONFIG: throw ConfigError(m);
    case PGB_ERR_CONTRACT: throw ContractError(m);
    case PGB_ERR_UNSUPPORTED: throw UnsupportedError(m);
    case PGB_ERR_TRACE: throw TraceError(m);
    case PGB_ERR_FORMAT: throw FormatError(m);
    case PGB_ERR_IO: throw IoError(m);
    case PGB_ERR_CUDA: throw CudaError(m);
    case PGB_ERR_NCCL: throw NcclError(m);
    case PGB_ERR_OOM: throw OutOfMemoryError(m);
    default: throw Error(m);
  }
}

// ---- models (models.hpp:24-88) ---------------------------------------------------
namespace models {

enum class ModelKind { logreg = 0, fcnn, mnist_cnn, cifar_cnn, embed, lstm };
enum class LayerKind {
  dense = 0, conv, maxpool, avgpool, global_avgpool, flatten, relu, embedding, seq_avgpool, lstm
};

struct LayerSpec {
  LayerKind kind;
  int64_t in = 0, out = 0, k = 0, stride = 1, pad = 0;
};

struct ModelOptions {
  int64_t seq_len = -1, vocab = -1, hidden = -1;
};

struct ModelDesc {
  pgb_model_desc c{};
  ModelKind kind() const { return static_cast<ModelKind>(c.model_kind); }
  int64_t classes() const { return c.classes; }
  std::vector<int64_t> input_shape() const {
    return std::vector<int64_t>(c.input_shape, c.input_shape + c.input_rank);
  }
  std::vector<LayerSpec> layers() const {
    std::vector<LayerSpec> v;
    for (int i = 0; i < c.n_layers; ++i) {
      const pgb_layer_spec& l = c.layers[i];
      v.push_back({static_cast<LayerKind>(l.kind), l.in, l.out, l.k, l.stride, l.pad});
    }
    return v;
  }
  int n_params() const { return c.n_params; }
  int64_t param_size(int p) const { return c.param_size[p]; }
  int64_t param_count() const { return pgb_param_count(&c); }
  int64_t input_numel() const {
    int64_t n = 1;
    for (int i = 0; i < c.input_rank; ++i) n *= c.input_shape[i];
    return n;
  }
};

inline ModelDesc build_desc(ModelKind kind, const ModelOptions& o = {}) {
  ModelDesc d;
  pgb_model_options co{o.seq_len, o.vocab, o.hidden};
  check(pgb_build_desc(static_cast<int32_t>(kind), &co, &d.c));
  return d;
}

// A custom layer list (e.g. the 104-50-2 FFNN of BASELINE config 2).
inline ModelDesc custom_desc(ModelKind kind, const std::vector<LayerSpec>& layers,
                             const std::vector<int64_t>& input_shape, int64_t classes,
                             bool token_input = false) {
  ModelDesc d;
  if (layers.size() > PGB_MAX_LAYERS || input_shape.size() > 3)
    throw ConfigError("custom_desc: too many layers or input dimensions");
  d.c.model_kind = static_cast<int32_t>(kind);
  d.c.n_layers = static_cast<int32_t>(layers.size());
  for (size_t i = 0; i < layers.size(); ++i)
    d.c.layers[i] = {static_cast<int32_t>(layers[i].kind), layers[i].in, layers[i].out,
                     layers[i].k, layers[i].stride, layers[i].pad};
  d.c.input_rank = static_cast<int32_t>(input_shape.size());
  for (size_t i = 0; i < input_shape.size(); ++i) d.c.input_shape[i] = input_shape[i];
  d.c.classes = classes;
  d.c.token_input = token_input ? 1 : 0;
  check(pgb_finish_desc(&d.c));
  return d;
}

// models::Model<float>: parameters in registry order, one flat block each.
struct Model {
  ModelDesc desc;
  std::vector<std::vector<float>> params;
  std::vector<float> flat() const {
    std::vector<float> f;
    for (const auto& p : params) f.insert(f.end(), p.begin(), p.end());
    return f;
  }
  void set_flat(const std::vector<float>& f) {
    size_t o = 0;
    for (auto& p : params) {
      std::copy(f.begin() + o, f.begin() + o + p.size(), p.begin());
      o += p.size();
    }
  }
};

inline Model build_from_desc(const ModelDesc& d, uint64_t seed) {
  Model m;
  m.desc = d;
  std::vector<float> flat(d.param_count());
  check(pgb_init_params(&d.c, seed, flat.data()));
  for (int p = 0, o = 0; p < d.n_params(); ++p) {
    m.params.emplace_back(flat.begin() + o, flat.begin() + o + d.param_size(p));
    o += static_cast<int>(d.param_size(p));
  }
  return m;
}

inline Model build(ModelKind kind, uint64_t seed, const ModelOptions& o = {}) {
  return build_from_desc(build_desc(kind, o), seed);
}

}  // namespace models

// ---- strategies / engine (strategies.hpp:34-100) -----------------------------------
enum class Strategy { naive = 0, vmap, outer, norms, groupconv, jacmm };
enum class ExecMode { eager = 0, graph };

template <typename T = float>
struct DpConfig {  // dpsgd.hpp:24-31
  T clip_norm = T(1);
  T noise_multiplier = T(0);
  T learning_rate = T(0.1);
  int64_t microbatch = 1;
  uint64_t seed = 0;
};

struct StepReport {  // dpsgd.hpp:36-41
  std::vector<float> pre_clip_norms;
  int64_t clipped_count = 0;
  std::vector<uint64_t> noise_streams;
};

class GradEngine {
 public:
  GradEngine(const models::Model& model, Strategy strategy, int64_t batch,
             ExecMode mode = ExecMode::graph, int device = 0)
      : batch_(batch), strategy_(strategy) {
    pgb_engine* h = nullptr;
    check(pgb_engine_create(&model.desc.c, static_cast<int32_t>(strategy), batch, device, &h));
    h_.reset(h);
    check(pgb_engine_set_graph(h, mode == ExecMode::graph ? 1 : 0));
    upload(model);
  }
  int64_t batch() const { return batch_; }
  Strategy strategy() const { return strategy_; }
  pgb_engine* handle() const { return h_.get(); }
  void upload(const models::Model& m) {
    std::vector<float> f = m.flat();
    check(pgb_set_params(h_.get(), f.data()));
    bound_ = &m;
    synced_ = std::move(f);
    device_ahead_ = false;
  }
  void download(models::Model& m) {
    std::vector<float> f(m.desc.param_count());
    check(pgb_get_params(h_.get(), f.data()));
    m.set_flat(f);
    bound_ = &m;
    synced_ = std::move(f);
    device_ahead_ = false;
  }
  // The reference's dpsgd_step reads model.params on every call
  // (dpsgd.cpp:188-331): upload when the device does not hold exactly this
  // model's host parameters (another model was stepped on this engine, or the
  // host copy was edited since the last sync). After a step with
  // sync_params = false the device copy is the newer one and is kept.
  void bind(const models::Model& m) {
    if (bound_ == &m && (device_ahead_ || m.flat() == synced_)) return;
    upload(m);
  }
  void mark_device_ahead(const models::Model& m) {
    bound_ = &m;
    device_ahead_ = true;
  }
  // strategies.cpp:432-450 / 453-458: sum_i w_i g_i (flat parameter order)
  std::vector<float> weighted_grad_sum(const float* x, const float* y, const float* w) const {
    std::vector<float> out(param_count());
    check(pgb_weighted_grad_sum(h_.get(), x, y, w, out.data()));
    return out;
  }
  std::vector<float> batch_grad_sum(const float* x, const float* y) const {
    std::vector<float> out(param_count());
    check(pgb_batch_grad_sum(h_.get(), x, y, out.data()));
    return out;
  }
  int64_t param_count() const {
    pgb_engine_info info{};
    check(pgb_engine_info_get(h_.get(), &info));
    return info.param_count;
  }
  int64_t footprint_bytes() const {
    pgb_engine_info info{};
    check(pgb_engine_info_get(h_.get(), &info));
    return info.workspace_bytes;
  }

 private:
  struct Del {
    void operator()(pgb_engine* e) const { pgb_engine_destroy(e); }
  };
  std::unique_ptr<pgb_engine, Del> h_;
  int64_t batch_;
  Strategy strategy_;
  const models::Model* bound_ = nullptr;  // the model whose parameters the device holds
  std::vector<float> synced_;             // its host parameters at the last sync
  bool device_ahead_ = false;             // device newer than the host copy
};

inline void validate(const DpConfig<float>& cfg, int64_t batch) {  // dpsgd.cpp:36-51
  if (!(cfg.clip_norm > 0.0f)) throw ConfigError("DpConfig: clip norm must be positive");
  if (cfg.noise_multiplier < 0.0f)
    throw ConfigError("DpConfig: noise multiplier must be non-negative");
  if (!(cfg.learning_rate > 0.0f)) throw ConfigError("DpConfig: learning rate must be positive");
  if (cfg.microbatch < 1 || batch % cfg.microbatch != 0)
    throw ConfigError("DpConfig: microbatch size " + std::to_string(cfg.microbatch) +
                      " must divide the batch size " + std::to_string(batch));
}

// dpsgd_step (dpsgd.hpp:70-73): x is batch*numel(input) floats, y batch
// floats. The device keeps the parameters; with sync_params (default, the
// reference's contract) model.params are refreshed after the step.
inline StepReport dpsgd_step(models::Model& model, GradEngine& engine, const float* x,
                             const float* y, const DpConfig<float>& cfg, int64_t step_index,
                             bool sync_params = true) {
  validate(cfg, engine.batch());
  StepReport rep;
  rep.pre_clip_norms.resize(engine.batch() / cfg.microbatch);
  pgb_dp_config c{cfg.clip_norm, cfg.noise_multiplier, cfg.learning_rate, cfg.microbatch,
                  cfg.seed};
  pgb_step_report r{};
  engine.bind(model);
  check(pgb_dpsgd_step(engine.handle(), x, y, &c, step_index, rep.pre_clip_norms.data(), &r));
  rep.clipped_count = r.clipped_count;
  rep.noise_streams.assign(r.noise_streams, r.noise_streams + r.n_streams);
  if (sync_params) engine.download(model);
  else engine.mark_device_ahead(model);
  return rep;
}

inline StepReport dpsgd_step(models::Model& model, GradEngine& engine,
                             const std::vector<float>& x, const std::vector<float>& y,
                             const DpConfig<float>& cfg, int64_t step_index,
                             bool sync_params = true) {
  if ((int64_t)y.size() != engine.batch() ||
      (int64_t)x.size() != engine.batch() * model.desc.input_numel())
    throw ContractError("GradEngine: batch extent mismatch (engine built for " +
                        std::to_string(engine.batch()) + ")");
  return dpsgd_step(model, engine, x.data(), y.data(), cfg, step_index, sync_params);
}

// sgd_step (dpsgd.hpp:76-78)
inline void sgd_step(models::Model& model, GradEngine& engine, const std::vector<float>& x,
                     const std::vector<float>& y, float learning_rate, bool sync_params = true) {
  engine.bind(model);
  check(pgb_sgd_step(engine.handle(), x.data(), y.data(), learning_rate));
  if (sync_params) engine.download(model);
  else engine.mark_device_ahead(model);
}

// ---- data (dataset.hpp:36-69) -----------------------------------------------------
namespace io {
struct Dataset {
  std::vector<float> inputs, labels;
  int64_t count = 0;
};
inline Dataset synth_for_model(const models::ModelDesc& d, int64_t n, uint64_t seed) {
  Dataset ds;
  ds.count = n;
  ds.inputs.resize(n * d.input_numel());
  ds.labels.resize(n);
  check(pgb_synth(&d.c, n, seed, ds.inputs.data(), ds.labels.data()));
  return ds;
}

// io::load_idx (dataset.cpp:35-82): values of one unsigned-byte IDX array and
// its dims; FormatError / IoError with the reference's messages.
struct IdxArray {
  std::vector<float> values;
  std::vector<int64_t> dims;
};
inline IdxArray load_idx(const std::string& path, float scale_div = 0.0f) {
  int32_t rank = 0;
  int64_t dims[4] = {0, 0, 0, 0}, count = 0;
  check(pgb_idx_info(path.c_str(), &rank, dims, &count));
  IdxArray a;
  a.dims.assign(dims, dims + rank);
  a.values.resize((size_t)count);
  check(pgb_load_idx(path.c_str(), scale_div, a.values.data(), (int64_t)a.values.size()));
  return a;
}

// io::load_mnist (dataset.cpp:84-112): images scaled to [0,1], (N,1,28,28)
inline Dataset load_mnist(const std::string& dir, const std::string& prefix = "train") {
  IdxArray img = load_idx(dir + "/" + prefix + "-images-idx3-ubyte", 255.0f);
  IdxArray lab = load_idx(dir + "/" + prefix + "-labels-idx1-ubyte");
  if (img.dims.size() != 3) throw FormatError("load_mnist: expected rank-3 image array");
  if (lab.dims.size() != 1 || lab.dims[0] != img.dims[0])
    throw FormatError("load_mnist: image/label count mismatch");
  Dataset ds;
  ds.count = img.dims[0];
  ds.inputs = std::move(img.values);
  ds.labels = std::move(lab.values);
  return ds;
}
}  // namespace io

// ---- epoch driver (harness.hpp:75-80): N/B sequential slices ----------------------
namespace bench {
struct EpochResult {
  double seconds = 0;
  int64_t clipped_total = 0;
};
inline EpochResult run_epoch(models::Model& model, GradEngine& engine, const io::Dataset& data,
                             const DpConfig<float>& cfg, int64_t step0) {
  pgb_dp_config c{cfg.clip_norm, cfg.noise_multiplier, cfg.learning_rate, cfg.microbatch,
                  cfg.seed};
  EpochResult r;
  engine.bind(model);
  check(pgb_run_epoch(engine.handle(), data.inputs.data(), data.labels.data(), data.count, &c,
                      step0, nullptr, &r.clipped_total, &r.seconds));
  engine.download(model);
  return r;
}

// The step loop of run_bench (harness.cpp:147-151) over batches already on the
// device (d_x: n_batches * B examples): step step0 + i reads batch
// (step0 + i) mod n_batches; static multi-step CUDA graphs, asynchronous.
inline int64_t run_steps_device(GradEngine& engine, const float* d_x, const float* d_y,
                                int64_t n_batches, int64_t n_steps, const DpConfig<float>& cfg,
                                int64_t step0) {
  pgb_dp_config c{cfg.clip_norm, cfg.noise_multiplier, cfg.learning_rate, cfg.microbatch,
                  cfg.seed};
  int64_t launches = 0;
  check(pgb_run_steps_device(engine.handle(), d_x, d_y, n_batches, n_steps, &c, step0,
                             &launches));
  return launches;
}
// bench::train (harness.cpp:319-382): seeded per-epoch shuffle
// (pgb_shuffle_order), DPSGD (or SGD) steps, the mean evaluation loss over the
// first min(N, 1024) examples per epoch, the final accuracy over the whole set
// (first maximum; K = 1: logit > 0).
struct TrainResult {
  std::vector<double> epoch_mean_loss;
  double final_train_accuracy = 0;
  int64_t steps = 0;
};

inline TrainResult train(models::Model& model, const io::Dataset& data, Strategy strategy,
                         ExecMode mode, const DpConfig<float>& cfg, int64_t batch,
                         int64_t epochs, bool private_training) {
  if (batch <= 0 || batch > data.count) throw ConfigError("train: bad batch size");
  GradEngine engine(model, strategy, batch, mode);
  TrainResult res;
  const int64_t steps = data.count / batch, row = model.desc.input_numel();
  const int64_t K = model.desc.c.classes;
  std::vector<int64_t> order((size_t)data.count);
  for (int64_t i = 0; i < data.count; ++i) order[(size_t)i] = i;  // reshuffled every epoch
  std::vector<float> x((size_t)(batch * row)), y((size_t)batch);
  // forward-only losses / logits of examples [0, n) in engine-batch chunks
  auto evaluate = [&](int64_t n, std::vector<float>& losses, std::vector<float>& logits) {
    losses.assign((size_t)n, 0.0f);
    logits.assign((size_t)(n * K), 0.0f);
    std::vector<float> lo((size_t)batch), lg((size_t)(batch * K));
    engine.bind(model);
    for (int64_t s0 = 0; s0 < n; s0 += batch) {
      const int64_t cnt = std::min(batch, n - s0);
      for (int64_t i = 0; i < batch; ++i) {  // the tail chunk repeats its last example
        const int64_t src = s0 + std::min(i, cnt - 1);
        std::copy(data.inputs.begin() + src * row, data.inputs.begin() + (src + 1) * row,
                  x.begin() + i * row);
        y[(size_t)i] = data.labels[(size_t)src];
      }
      check(pgb_forward(engine.handle(), x.data(), y.data(), lo.data(), lg.data()));
      std::copy(lo.begin(), lo.begin() + cnt, losses.begin() + s0);
      std::copy(lg.begin(), lg.begin() + cnt * K, logits.begin() + s0 * K);
    }
  };
  std::vector<float> losses, logits;
  const int64_t eval_n = std::min<int64_t>(data.count, 1024);
  for (int64_t epoch = 0; epoch < epochs; ++epoch) {
    check(pgb_shuffle_order(cfg.seed, epoch, data.count, order.data()));
    for (int64_t s = 0; s < steps; ++s) {
      for (int64_t i = 0; i < batch; ++i) {
        const int64_t src = order[(size_t)(s * batch + i)];
        std::copy(data.inputs.begin() + src * row, data.inputs.begin() + (src + 1) * row,
                  x.begin() + i * row);
        y[(size_t)i] = data.labels[(size_t)src];
      }
      if (private_training) dpsgd_step(model, engine, x, y, cfg, epoch * steps + s);
      else sgd_step(model, engine, x, y, cfg.learning_rate);
      ++res.steps;
    }
    evaluate(eval_n, losses, logits);
    double tot = 0;
    for (float l : losses) tot += l;
    res.epoch_mean_loss.push_back(tot / (double)eval_n);
  }
  evaluate(data.count, losses, logits);
  int64_t correct = 0;
  for (int64_t i = 0; i < data.count; ++i) {
    int64_t pred = 0;
    if (K == 1) {
      pred = logits[(size_t)i] > 0.0f ? 1 : 0;
    } else {
      for (int64_t k = 1; k < K; ++k)
        if (logits[(size_t)(i * K + k)] > logits[(size_t)(i * K + pred)]) pred = k;
    }
    correct += pred == (int64_t)data.labels[(size_t)i];
  }
  res.final_train_accuracy = (double)correct / (double)data.count;
  return res;
}
}  // namespace bench

}  // namespace pegrad_b200
