// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// A thin extern "C" shim around the *unmodified* reference library
// ("pegrad", compiled from /root/reference/proj/core/src by oracle/Makefile
// into oracle/_ref/libpegrad_ref.so). It exists so the Python test-suite,
// tests/golden/gen_golden.py and bench.py's cpu_baseline / --impl reference
// legs can drive the reference's own public API:
//   models::build / build_desc           (proj/core/src/models.cpp:87-167,359-380)
//   io::synth_for_model                   (proj/core/src/dataset.cpp:219-237)
//   GradEngine<T>::compute                (proj/core/src/strategies.cpp:330-397)
//   dpsgd_step                            (proj/core/src/dpsgd.cpp:188-331)
//   gaussian<T>                           (proj/core/src/tensor_ops.cpp:292-296)
//   bench::run_bench                      (proj/core/src/harness.cpp:85-167)
//   io::load_idx                          (proj/core/src/dataset.cpp:35-82)
//   bench::records_from_json / records_to_json (proj/core/src/harness.cpp:219-274)
// Only tests/, __graft_entry__.smoke() and bench.py's reference legs load it.

#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "pegrad/dataset.hpp"
#include "pegrad/dpsgd.hpp"
#include "pegrad/harness.hpp"
#include "pegrad/models.hpp"
#include "pegrad/strategies.hpp"
#include "pegrad/tensor_ops.hpp"

using namespace pegrad;

namespace {

thread_local std::string g_err;

// Error codes mirror include/pegrad_b200.h's pgb_status ordering.
int code_of(const std::exception& e) {
  if (dynamic_cast<const ShapeError*>(&e)) return 1;
  if (dynamic_cast<const DomainError*>(&e)) return 2;
  if (dynamic_cast<const IndexError*>(&e)) return 3;
  if (dynamic_cast<const ConfigError*>(&e)) return 4;
  if (dynamic_cast<const ContractError*>(&e)) return 5;
  if (dynamic_cast<const UnsupportedError*>(&e)) return 6;
  if (dynamic_cast<const TraceError*>(&e)) return 7;
  if (dynamic_cast<const FormatError*>(&e)) return 8;
  if (dynamic_cast<const IoError*>(&e)) return 9;
  return 99;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// The reference keeps register_params() private to models.cpp; custom
// descriptions (e.g. the 104-50-2 FFNN of BASELINE config 2) therefore fill
// the registry here following the documented layout rules
// (proj/core/src/models.cpp:50-83).
void fill_registry(models::ModelDesc& d) {
  using models::LayerKind;
  d.param_names.clear();
  d.param_shapes.clear();
  d.param_fan_in.clear();
  int li = 0;
  for (const auto& l : d.layers) {
    const std::string pre = "l" + std::to_string(li) + ".";
    auto add = [&](const std::string& n, Shape s, int64_t f) {
      d.param_names.push_back(pre + n);
      d.param_shapes.push_back(std::move(s));
      d.param_fan_in.push_back(f);
    };
    switch (l.kind) {
      case LayerKind::dense:
        add("W", {l.in, l.out}, l.in);
        add("b", {l.out}, 0);
        break;
      case LayerKind::conv:
        add("W", {l.out, l.in, l.k, l.k}, l.in * l.k * l.k);
        add("b", {l.out}, 0);
        break;
      case LayerKind::embedding:
        add("table", {l.in, l.out}, l.out);
        break;
      case LayerKind::lstm:
        add("Wx", {4 * l.out, l.in}, l.in);
        add("Wh", {4 * l.out, l.out}, l.out);
        add("b", {4 * l.out}, 0);
        break;
      default:
        break;
    }
    ++li;
  }
}

template <typename T>
std::vector<Tensor<T>> unflatten(const models::ModelDesc& d, const T* flat) {
  std::vector<Tensor<T>> out;
  for (const Shape& s : d.param_shapes) {
    const int64_t n = numel(s);
    out.push_back(Tensor<T>::from(s, std::vector<T>(flat, flat + n)));
    flat += n;
  }
  return out;
}

template <typename T>
void flatten_into(const std::vector<Tensor<T>>& ps, T* flat) {
  for (const auto& t : ps) {
    std::memcpy(flat, t.data(), sizeof(T) * t.size());
    flat += t.size();
  }
}

template <typename T>
Shape batch_shape(const models::ModelDesc& d, int64_t B) {
  Shape s = d.input_shape;
  s.insert(s.begin(), B);
  return s;
}

template <typename T>
struct RefEngine {
  models::Model<T> model;
  std::unique_ptr<GradEngine<T>> engine;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_desc_builtin(int kind, int64_t seq_len, int64_t vocab,
                       int64_t hidden) {
  models::ModelDesc* d = nullptr;
  int rc = guarded([&] {
    models::ModelOptions o;
    o.seq_len = seq_len;
    o.vocab = vocab;
    o.hidden = hidden;
    d = new models::ModelDesc(
        models::build_desc(static_cast<models::ModelKind>(kind), o));
  });
  return rc == 0 ? d : nullptr;
}

// l6: n_layers rows of (kind, in, out, k, stride, pad)
void* ref_desc_custom(int model_kind, int n_layers, const int64_t* l6,
                      int in_rank, const int64_t* in_shape, int64_t classes,
                      int token_input) {
  auto* d = new models::ModelDesc();
  d->kind = static_cast<models::ModelKind>(model_kind);
  for (int i = 0; i < n_layers; ++i) {
    models::LayerSpec s;
    s.kind = static_cast<models::LayerKind>(l6[6 * i]);
    s.in = l6[6 * i + 1];
    s.out = l6[6 * i + 2];
    s.k = l6[6 * i + 3];
    s.stride = l6[6 * i + 4];
    s.pad = l6[6 * i + 5];
    d->layers.push_back(s);
  }
  d->input_shape.assign(in_shape, in_shape + in_rank);
  d->classes = classes;
  d->token_input = token_input != 0;
  fill_registry(*d);
  return d;
}

void ref_desc_free(void* d) { delete static_cast<models::ModelDesc*>(d); }

int64_t ref_desc_param_count(void* d) {
  return static_cast<models::ModelDesc*>(d)->param_count();
}
int ref_desc_num_blocks(void* d) {
  return static_cast<int>(
      static_cast<models::ModelDesc*>(d)->param_shapes.size());
}
int64_t ref_desc_block_size(void* d, int p) {
  return numel(static_cast<models::ModelDesc*>(d)->param_shapes[p]);
}

#define REF_TYPED(T, SFX)                                                     \
  int ref_init_params_##SFX(void* dv, uint64_t seed, T* flat) {               \
    return guarded([&] {                                                      \
      auto m = models::build_from_desc<T>(*static_cast<models::ModelDesc*>(dv), \
                                          seed);                              \
      flatten_into(m.params, flat);                                           \
    });                                                                       \
  }                                                                           \
  int ref_synth_##SFX(void* dv, int64_t n, uint64_t seed, T* x, T* y) {       \
    return guarded([&] {                                                      \
      auto ds = io::synth_for_model<T>(*static_cast<models::ModelDesc*>(dv),  \
                                       n, seed);                              \
      std::memcpy(x, ds.inputs.data(), sizeof(T) * ds.inputs.size());         \
      std::memcpy(y, ds.labels.data(), sizeof(T) * ds.labels.size());         \
    });                                                                       \
  }                                                                           \
  int ref_gaussian_##SFX(uint64_t seed, uint64_t stream, int64_t n, T* out) { \
    return guarded([&] {                                                      \
      RngState rng(seed, stream);                                             \
      auto t = gaussian<T>({n}, rng);                                         \
      std::memcpy(out, t.data(), sizeof(T) * n);                              \
    });                                                                       \
  }                                                                           \
  void* ref_engine_new_##SFX(void* dv, int strategy, int64_t B,              \
                             const T* params) {                               \
    RefEngine<T>* e = nullptr;                                                \
    int rc = guarded([&] {                                                    \
      const auto& d = *static_cast<models::ModelDesc*>(dv);                   \
      auto* ne = new RefEngine<T>();                                          \
      ne->model.desc = d;                                                     \
      ne->model.params = unflatten<T>(d, params);                             \
      ne->engine = std::make_unique<GradEngine<T>>(                           \
          ne->model, static_cast<Strategy>(strategy), B, ExecMode::graph);    \
      e = ne;                                                                 \
    });                                                                       \
    return rc == 0 ? e : nullptr;                                             \
  }                                                                           \
  void ref_engine_free_##SFX(void* h) { delete static_cast<RefEngine<T>*>(h); } \
  int ref_engine_get_params_##SFX(void* h, T* flat) {                         \
    return guarded([&] {                                                      \
      flatten_into(static_cast<RefEngine<T>*>(h)->model.params, flat);        \
    });                                                                       \
  }                                                                           \
  int ref_engine_set_params_##SFX(void* h, const T* flat) {                   \
    return guarded([&] {                                                      \
      auto* e = static_cast<RefEngine<T>*>(h);                                \
      e->model.params = unflatten<T>(e->model.desc, flat);                    \
    });                                                                       \
  }                                                                           \
  /* stacks: block-major, block p is (B, numel(shape_p)); norms (B) */        \
  int ref_engine_per_example_##SFX(void* h, const T* x, const T* y,           \
                                   T* stacks, T* norms) {                     \
    return guarded([&] {                                                      \
      auto* e = static_cast<RefEngine<T>*>(h);                                \
      const auto& d = e->model.desc;                                          \
      const int64_t B = e->engine->batch();                                   \
      const int64_t row = numel(d.input_shape);                               \
      auto xt = Tensor<T>::from(batch_shape<T>(d, B),                         \
                                std::vector<T>(x, x + B * row));              \
      auto yt = Tensor<T>::from({B}, std::vector<T>(y, y + B));               \
      auto g = e->engine->compute(xt, yt, e->model.params);                   \
      if (stacks) {                                                           \
        if (g.norms_only) throw ContractError("norms-only strategy");         \
        for (const auto& s : g.stacks) {                                      \
          std::memcpy(stacks, s.data(), sizeof(T) * s.size());                \
          stacks += s.size();                                                 \
        }                                                                     \
      }                                                                       \
      if (norms) {                                                            \
        auto n = per_example_global_norms(g);                                 \
        std::memcpy(norms, n.data(), sizeof(T) * B);                          \
      }                                                                       \
    });                                                                       \
  }                                                                           \
  int ref_engine_step_##SFX(void* h, const T* x, const T* y, T clip,          \
                            T sigma, T lr, int64_t m, uint64_t seed,          \
                            int64_t step, T* norms, int64_t* clipped) {       \
    return guarded([&] {                                                      \
      auto* e = static_cast<RefEngine<T>*>(h);                                \
      const auto& d = e->model.desc;                                          \
      const int64_t B = e->engine->batch();                                   \
      const int64_t row = numel(d.input_shape);                               \
      auto xt = Tensor<T>::from(batch_shape<T>(d, B),                         \
                                std::vector<T>(x, x + B * row));              \
      auto yt = Tensor<T>::from({B}, std::vector<T>(y, y + B));               \
      DpConfig<T> cfg;                                                        \
      cfg.clip_norm = clip;                                                   \
      cfg.noise_multiplier = sigma;                                           \
      cfg.learning_rate = lr;                                                 \
      cfg.microbatch = m;                                                     \
      cfg.seed = seed;                                                        \
      auto rep = dpsgd_step(e->model, *e->engine, xt, yt, cfg, step);         \
      if (norms)                                                              \
        std::memcpy(norms, rep.pre_clip_norms.data(),                         \
                    sizeof(T) * rep.pre_clip_norms.size());                   \
      if (clipped) *clipped = rep.clipped_count;                              \
    });                                                                       \
  }                                                                           \
  int ref_engine_sgd_step_##SFX(void* h, const T* x, const T* y, T lr) {      \
    return guarded([&] {                                                      \
      auto* e = static_cast<RefEngine<T>*>(h);                                \
      const auto& d = e->model.desc;                                          \
      const int64_t B = e->engine->batch();                                   \
      const int64_t row = numel(d.input_shape);                               \
      auto xt = Tensor<T>::from(batch_shape<T>(d, B),                         \
                                std::vector<T>(x, x + B * row));              \
      auto yt = Tensor<T>::from({B}, std::vector<T>(y, y + B));               \
      sgd_step(e->model, *e->engine, xt, yt, lr);                             \
    });                                                                       \
  }                                                                           \
  /* GradEngine::weighted_grad_sum: sum_i w_i g_i, flat parameter order */    \
  int ref_engine_weighted_sum_##SFX(void* h, const T* x, const T* y,          \
                                    const T* w, T* out) {                     \
    return guarded([&] {                                                      \
      auto* e = static_cast<RefEngine<T>*>(h);                                \
      const auto& d = e->model.desc;                                          \
      const int64_t B = e->engine->batch();                                   \
      const int64_t row = numel(d.input_shape);                               \
      auto xt = Tensor<T>::from(batch_shape<T>(d, B),                         \
                                std::vector<T>(x, x + B * row));              \
      auto yt = Tensor<T>::from({B}, std::vector<T>(y, y + B));               \
      auto wt = Tensor<T>::from({B}, std::vector<T>(w, w + B));               \
      flatten_into(e->engine->weighted_grad_sum(xt, yt, wt, e->model.params), \
                   out);                                                      \
    });                                                                       \
  }

REF_TYPED(float, f32)
REF_TYPED(double, f64)

// bench::train (harness.cpp:319-382) over caller data: the model starts at
// `params` and ends in them; per-epoch mean evaluation losses, final accuracy.
int ref_train_f32(void* dv, float* params, const float* x, const float* y, int64_t n,
                  int strategy, double clip, double sigma, double lr, int64_t m,
                  uint64_t seed, int64_t batch, int64_t epochs, int private_training,
                  double* epoch_loss, double* accuracy, int64_t* steps) {
  return guarded([&] {
    const auto& d = *static_cast<models::ModelDesc*>(dv);
    models::Model<float> model;
    model.desc = d;
    model.params = unflatten<float>(d, params);
    io::Dataset<float> data;
    const int64_t row = numel(d.input_shape);
    data.inputs = Tensor<float>::from(batch_shape<float>(d, n), std::vector<float>(x, x + n * row));
    data.labels = Tensor<float>::from({n}, std::vector<float>(y, y + n));
    data.count = n;
    DpConfig<float> cfg;
    cfg.clip_norm = (float)clip;
    cfg.noise_multiplier = (float)sigma;
    cfg.learning_rate = (float)lr;
    cfg.microbatch = m;
    cfg.seed = seed;
    auto r = bench::train(model, data, static_cast<Strategy>(strategy), ExecMode::graph, cfg,
                          batch, epochs, private_training != 0);
    for (size_t e = 0; e < r.epoch_mean_loss.size(); ++e) epoch_loss[e] = r.epoch_mean_loss[e];
    *accuracy = r.final_train_accuracy;
    *steps = r.steps;
    flatten_into(model.params, params);
  });
}

// bench::run_bench over synth_for_model data; returns the median epoch time.
int ref_run_bench_f32(int kind, int strategy, int64_t B, int64_t N,
                      int64_t epochs, double clip, double sigma, double lr,
                      uint64_t seed, double* median_seconds) {
  return guarded([&] {
    auto desc = models::build_desc(static_cast<models::ModelKind>(kind));
    auto data = io::synth_for_model<float>(desc, N, seed);
    bench::RunOptions o;
    o.batch_sizes = {B};
    o.epochs = epochs;
    o.clip_norm = clip;
    o.noise_multiplier = sigma;
    o.learning_rate = lr;
    o.seed = seed;
    auto recs = bench::run_bench<float>(static_cast<models::ModelKind>(kind),
                                        data, static_cast<Strategy>(strategy),
                                        o);
    if (recs.empty() || recs[0].status != "ok")
      throw ContractError("run_bench: " +
                          (recs.empty() ? std::string("no record")
                                        : recs[0].status + " " + recs[0].reason));
    *median_seconds = recs[0].median_epoch_seconds;
  });
}

// io::load_idx<float>: element count into *n, the rank and dims, and (when
// out is non-null and cap suffices) the values.
int ref_load_idx_f32(const char* path, float* out, int64_t cap, int64_t* n, int* rank,
                     int64_t* dims) {
  return guarded([&] {
    Tensor<float> t = io::load_idx<float>(path);
    *n = t.size();
    *rank = (int)t.rank();
    for (int d = 0; d < (int)t.rank(); ++d) dims[d] = t.dim(d);
    if (out && cap >= t.size()) std::memcpy(out, t.data(), sizeof(float) * t.size());
  });
}

// Parse BenchRecord JSON with the reference's parser and re-emit it with the
// reference's writer (records_from_json -> records_to_json).
int ref_records_json_roundtrip(const char* text, char* out, int64_t cap, int64_t* len) {
  return guarded([&] {
    const std::string s = bench::records_to_json(bench::records_from_json(text));
    *len = (int64_t)s.size();
    if (out && cap > (int64_t)s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

}  // extern "C"
