// Reference-style C++ test of the drop-in shim (include/pegrad_b200.hpp),
// mirroring proj/tests/test_dpsgd.cpp's contracts on the GPU engine:
// config validation, StepReport fields, noise streams, determinism of
// identical seeds, sigma=0 + loose C == plain SGD, label IndexError and the
// strategy support matrix. Prints "OK" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <unistd.h>

#include "pegrad_b200.hpp"

using namespace pegrad_b200;

#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      std::exit(1);                                                  \
    }                                                                \
  } while (0)

template <typename E, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "unexpected exception: %s\n", e.what());
    return false;
  } catch (...) {
    std::fprintf(stderr, "unexpected non-std exception\n");
    return false;
  }
  std::fprintf(stderr, "no exception\n");
  return false;
}

int main() {
  using models::ModelKind;
  const int64_t B = 16;
  // parameter counts (test_models.cpp:26-35)
  CHECK(models::build_desc(ModelKind::mnist_cnn).param_count() == 26010);
  CHECK(models::build_desc(ModelKind::cifar_cnn).param_count() == 605226);

  auto model = models::build(ModelKind::mnist_cnn, 0);
  auto data = io::synth_for_model(model.desc, B, 0);
  GradEngine engine(model, Strategy::groupconv, B);

  // config validation (test_dpsgd.cpp:285-296)
  DpConfig<float> bad;
  bad.clip_norm = 0;
  CHECK(throws<ConfigError>([&] { dpsgd_step(model, engine, data.inputs, data.labels, bad, 0); }));
  bad.clip_norm = 1;
  bad.microbatch = 3;
  CHECK(throws<ConfigError>([&] { dpsgd_step(model, engine, data.inputs, data.labels, bad, 0); }));

  // a noisy step: report fields and noise stream ids (dpsgd.cpp:27-32)
  DpConfig<float> cfg;
  cfg.clip_norm = 1.0f;
  cfg.noise_multiplier = 1.1f;
  cfg.learning_rate = 0.1f;
  auto rep = dpsgd_step(model, engine, data.inputs, data.labels, cfg, 7);
  CHECK((int64_t)rep.pre_clip_norms.size() == B);
  int64_t above = 0;
  for (float n : rep.pre_clip_norms) {
    CHECK(std::isfinite(n) && n > 0);
    above += n > cfg.clip_norm;
  }
  CHECK(rep.clipped_count == above);
  CHECK((int)rep.noise_streams.size() == model.desc.n_params());
  CHECK(rep.noise_streams[0] == (uint64_t(1) << 32) + 7 * 4096);

  // identical seeds -> identical trajectories (test_dpsgd.cpp:263-283)
  auto a = models::build(ModelKind::mnist_cnn, 1);
  auto b = models::build(ModelKind::mnist_cnn, 1);
  GradEngine ea(a, Strategy::groupconv, B), eb(b, Strategy::groupconv, B);
  for (int s = 0; s < 3; ++s) {
    dpsgd_step(a, ea, data.inputs, data.labels, cfg, s);
    dpsgd_step(b, eb, data.inputs, data.labels, cfg, s);
  }
  CHECK(a.flat() == b.flat());

  // sigma = 0 and a loose C is plain SGD (test_dpsgd.cpp:204-226)
  auto c = models::build(ModelKind::fcnn, 11);
  auto d = models::build(ModelKind::fcnn, 11);
  auto fd = io::synth_for_model(c.desc, 8, 3);
  GradEngine ec(c, Strategy::vmap, 8), ed(d, Strategy::vmap, 8);
  DpConfig<float> loose;
  loose.clip_norm = 1e6f;
  loose.noise_multiplier = 0.0f;
  loose.learning_rate = 0.5f;
  auto r2 = dpsgd_step(c, ec, fd.inputs, fd.labels, loose, 0);
  CHECK(r2.clipped_count == 0 && r2.noise_streams.empty());
  sgd_step(d, ed, fd.inputs, fd.labels, 0.5f);
  const auto fc = c.flat(), fdd = d.flat();
  for (size_t i = 0; i < fc.size(); ++i)
    CHECK(std::fabs(fc[i] - fdd[i]) <= 1e-6f * (1.0f + std::fabs(fdd[i])));

  // the norms-only two-pass branch (dpsgd.cpp:194-230): weighted sums through
  // the shim, batch_grad_sum = weighted_grad_sum(1), sum_i w g_i linear in w,
  // and microbatch != 1 refused
  {
    auto e = models::build(ModelKind::fcnn, 5);
    auto fe = io::synth_for_model(e.desc, 8, 1);
    GradEngine en(e, Strategy::norms, 8);
    std::vector<float> ones(8, 1.0f), halves(8, 0.5f);
    const auto g1 = en.batch_grad_sum(fe.inputs.data(), fe.labels.data());
    const auto w1 = en.weighted_grad_sum(fe.inputs.data(), fe.labels.data(), ones.data());
    const auto wh = en.weighted_grad_sum(fe.inputs.data(), fe.labels.data(), halves.data());
    CHECK(g1 == w1);
    for (size_t i = 0; i < g1.size(); ++i) CHECK(std::fabs(wh[i] - 0.5f * g1[i]) <= 1e-6f * (1.0f + std::fabs(g1[i])));
    DpConfig<float> mb = cfg;
    mb.microbatch = 2;
    CHECK(throws<ConfigError>([&] { dpsgd_step(e, en, fe.inputs, fe.labels, mb, 0); }));
  }

  // labels outside [0, classes) are an IndexError; parameters untouched
  auto before = model.flat();
  auto badlab = data.labels;
  badlab[3] = 12.0f;
  CHECK(throws<IndexError>([&] { dpsgd_step(model, engine, data.inputs, badlab, cfg, 8); }));
  engine.download(model);
  CHECK(model.flat() == before);

  // dpsgd_step reads model.params on every call (dpsgd.cpp:188-331): a host
  // edit of the parameters, and a second model stepped on the same engine,
  // both reach the device (two engines built from the edited models agree)
  {
    auto m1 = models::build(ModelKind::fcnn, 21);
    auto m2 = models::build(ModelKind::fcnn, 22);
    auto fx = io::synth_for_model(m1.desc, 8, 4);
    GradEngine shared(m1, Strategy::vmap, 8);
    m1.params[0][0] += 0.25f;  // host edit after the engine took its copy
    auto r1 = m1, r2 = m2;
    GradEngine e1(r1, Strategy::vmap, 8), e2(r2, Strategy::vmap, 8);
    dpsgd_step(m1, shared, fx.inputs, fx.labels, cfg, 0);
    dpsgd_step(r1, e1, fx.inputs, fx.labels, cfg, 0);
    CHECK(m1.flat() == r1.flat());
    dpsgd_step(m2, shared, fx.inputs, fx.labels, cfg, 0);  // another model, same engine
    dpsgd_step(r2, e2, fx.inputs, fx.labels, cfg, 0);
    CHECK(m2.flat() == r2.flat());
    // sync_params = false keeps the newer device copy for the next step
    dpsgd_step(m1, shared, fx.inputs, fx.labels, cfg, 1, false);
    dpsgd_step(m1, shared, fx.inputs, fx.labels, cfg, 2);
    dpsgd_step(r1, e1, fx.inputs, fx.labels, cfg, 1);
    dpsgd_step(r1, e1, fx.inputs, fx.labels, cfg, 2);
    CHECK(m1.flat() == r1.flat());
  }

  // the strategy support matrix (strategies.cpp:76-113)
  CHECK(throws<UnsupportedError>([&] { GradEngine bad_e(model, Strategy::outer, B); }));

  // one epoch driver pass (harness.cpp:85-167 shape)
  auto ep = io::synth_for_model(model.desc, 4 * B, 5);
  auto res = bench::run_epoch(model, engine, ep, cfg, 100);
  CHECK(res.seconds > 0 && res.clipped_total >= 0);

  // bench::train (harness.cpp:319-382): steps, one mean loss per epoch,
  // accuracy in [0, 1], deterministic for a fixed seed
  {
    auto t1 = models::build(ModelKind::fcnn, 2), t2 = models::build(ModelKind::fcnn, 2);
    auto td = io::synth_for_model(t1.desc, 96, 6);
    DpConfig<float> tc;
    tc.clip_norm = 1.0f;
    tc.noise_multiplier = 1.1f;
    tc.seed = 9;
    auto r1 = bench::train(t1, td, Strategy::vmap, ExecMode::graph, tc, 32, 2, true);
    auto r2 = bench::train(t2, td, Strategy::vmap, ExecMode::graph, tc, 32, 2, true);
    CHECK(r1.steps == 6 && r1.epoch_mean_loss.size() == 2);
    CHECK(r1.final_train_accuracy >= 0.0 && r1.final_train_accuracy <= 1.0);
    CHECK(r1.epoch_mean_loss == r2.epoch_mean_loss && t1.flat() == t2.flat());
    CHECK(throws<ConfigError>([&] { bench::train(t1, td, Strategy::vmap, ExecMode::graph, tc, 0, 1, true); }));
  }

  // IDX ingest (dataset.cpp:35-112): a small MNIST pair written here
  {
    const char* dir = std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp";
    const std::string base = std::string(dir) + "/pgb_shim_" + std::to_string(::getpid());
    auto write = [](const std::string& path, uint32_t magic, std::vector<uint32_t> dims,
                    const std::vector<unsigned char>& payload) {
      FILE* f = std::fopen(path.c_str(), "wb");
      auto be = [&](uint32_t v) {
        unsigned char b[4] = {(unsigned char)(v >> 24), (unsigned char)(v >> 16),
                              (unsigned char)(v >> 8), (unsigned char)v};
        std::fwrite(b, 1, 4, f);
      };
      be(magic);
      for (uint32_t d : dims) be(d);
      std::fwrite(payload.data(), 1, payload.size(), f);
      std::fclose(f);
    };
    std::vector<unsigned char> img(3 * 28 * 28), lab = {7, 0, 9};
    for (size_t i = 0; i < img.size(); ++i) img[i] = (unsigned char)(i * 37 % 256);
    write(base + "-images-idx3-ubyte", 0x803, {3, 28, 28}, img);
    write(base + "-labels-idx1-ubyte", 0x801, {3}, lab);
    auto mn = io::load_mnist(dir, "pgb_shim_" + std::to_string(::getpid()));
    CHECK(mn.count == 3 && mn.inputs.size() == 3 * 784 && mn.labels[2] == 9.0f);
    CHECK(mn.inputs[5] == (float)(5 * 37 % 256) / 255.0f);
    write(base + "-bad", 0x0D02, {2, 2}, {1, 2, 3, 4});
    CHECK(throws<FormatError>([&] { io::load_idx(base + "-bad"); }));
    CHECK(throws<IoError>([&] { io::load_idx(base + "-missing"); }));
    std::remove((base + "-images-idx3-ubyte").c_str());
    std::remove((base + "-labels-idx1-ubyte").c_str());
    std::remove((base + "-bad").c_str());
  }
  std::printf("OK\n");
  return 0;
}
