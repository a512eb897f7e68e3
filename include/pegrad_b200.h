/* pegrad_b200 — B200-native (sm_100a) DPSGD step engine, C ABI.
 *
 * The reference ("pegrad", /root/reference/proj) has no FFI: its step path is
 * the in-process C++ API
 *     dpsgd_step(Model<T>&, GradEngine<T>&, x, y, DpConfig<T>, step_index)
 *         -> StepReport<T>                      (core/include/pegrad/dpsgd.hpp:70-73)
 *     GradEngine<T>(model, Strategy, batch, ExecMode)
 *         compute / compute_views               (core/include/pegrad/strategies.hpp:58-100)
 *     models::build_desc / build                (core/include/pegrad/models.hpp:75-88)
 *     bench::run_bench / train                  (core/include/pegrad/harness.hpp:75-115)
 * This header is the drop-in boundary for that path: plain pointers and
 * sizes, no torch or C++ types. include/pegrad_b200.hpp wraps it back into
 * the reference's C++ shapes (Model, DpConfig, StepReport, exceptions).
 *
 * Layout contract (same as the reference's Tensor<float>): row-major NCHW
 * fp32 inputs, ids/labels as integral floats, parameters flattened in
 * parameter-registry order (models.cpp:50-83); per-example gradient stacks
 * are block-major: block p is (B, numel(shape_p)), blocks concatenated.
 */
#ifndef PEGRAD_B200_H
#define PEGRAD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGB_MAX_LAYERS 32
#define PGB_MAX_PARAMS 64

/* 1:1 with the pegrad exception hierarchy (common.hpp:56-114), plus device
 * failures the reference cannot have. */
typedef enum pgb_status {
  PGB_OK = 0,
  PGB_ERR_SHAPE = 1,       /* ShapeError */
  PGB_ERR_DOMAIN = 2,      /* DomainError */
  PGB_ERR_INDEX = 3,       /* IndexError: ids / labels */
  PGB_ERR_CONFIG = 4,      /* ConfigError: DpConfig, unknown names */
  PGB_ERR_CONTRACT = 5,    /* ContractError: batch mismatch, bad handle */
  PGB_ERR_UNSUPPORTED = 6, /* UnsupportedError: "unsupported layer" */
  PGB_ERR_TRACE = 7,
  PGB_ERR_FORMAT = 8,
  PGB_ERR_IO = 9,
  PGB_ERR_CUDA = 10,
  PGB_ERR_NCCL = 11,
  PGB_ERR_OOM = 12
} pgb_status;

/* pegrad::models::ModelKind (models.hpp:24) */
enum { PGB_LOGREG = 0, PGB_FCNN, PGB_MNIST_CNN, PGB_CIFAR_CNN, PGB_EMBED, PGB_LSTM_MODEL };
/* pegrad::models::LayerKind (models.hpp:29-40) */
enum {
  PGB_DENSE = 0, PGB_CONV, PGB_MAXPOOL, PGB_AVGPOOL, PGB_GLOBAL_AVGPOOL,
  PGB_FLATTEN, PGB_RELU, PGB_EMBEDDING, PGB_SEQ_AVGPOOL, PGB_LSTM
};
/* pegrad::Strategy (strategies.hpp:34) */
enum { PGB_NAIVE = 0, PGB_VMAP, PGB_OUTER, PGB_NORMS, PGB_GROUPCONV, PGB_JACMM };

/* pegrad::models::LayerSpec (models.hpp:42-49) */
typedef struct pgb_layer_spec {
  int32_t kind;
  int64_t in, out, k, stride, pad;
} pgb_layer_spec;

/* pegrad::models::ModelOptions (models.hpp:52-56); -1 keeps the default */
typedef struct pgb_model_options {
  int64_t seq_len, vocab, hidden;
} pgb_model_options;

/* pegrad::models::ModelDesc (models.hpp:58-73); the registry part
 * (param_size / param_fan_in) is filled by pgb_finish_desc. */
typedef struct pgb_model_desc {
  int32_t model_kind;
  int32_t n_layers;
  pgb_layer_spec layers[PGB_MAX_LAYERS];
  int32_t input_rank;
  int64_t input_shape[3];
  int64_t classes; /* 1 selects the binary sigmoid head */
  int32_t token_input;
  int32_t n_params;
  int64_t param_size[PGB_MAX_PARAMS];
  int64_t param_fan_in[PGB_MAX_PARAMS];
} pgb_model_desc;

/* pegrad::DpConfig<float> (dpsgd.hpp:24-31) */
typedef struct pgb_dp_config {
  float clip_norm;        /* C > 0 */
  float noise_multiplier; /* sigma >= 0, noise stddev sigma*C */
  float learning_rate;
  int64_t microbatch;     /* m, divides the batch */
  uint64_t seed;
} pgb_dp_config;

/* pegrad::StepReport<float> (dpsgd.hpp:36-41); pre_clip_norms are returned
 * through a caller buffer of B/m floats. */
typedef struct pgb_step_report {
  int64_t clipped_count;
  int32_t n_streams;
  uint64_t noise_streams[PGB_MAX_PARAMS];
} pgb_step_report;

typedef struct pgb_unique_id {
  char internal[128];
} pgb_unique_id;

typedef struct pgb_engine_info {
  int64_t batch;          /* local examples per step */
  int64_t global_batch;   /* batch * world */
  int64_t param_count;
  int32_t n_params;
  int32_t world, rank, device;
  int64_t workspace_bytes; /* device arena */
  int32_t kernels_per_step;
  int32_t graph_enabled;
} pgb_engine_info;

typedef struct pgb_engine pgb_engine;

const char* pgb_last_error(void);
const char* pgb_version(void);

/* ---- models (host) : models.cpp:50-167, 359-380 ------------------------- */
pgb_status pgb_build_desc(int32_t model_kind, const pgb_model_options* opts,
                          pgb_model_desc* out);
pgb_status pgb_finish_desc(pgb_model_desc* desc);
int64_t pgb_param_count(const pgb_model_desc* desc);
pgb_status pgb_init_params(const pgb_model_desc* desc, uint64_t seed,
                           float* flat_out);
/* The per-epoch example order of bench::train (harness.cpp:330-343): one
 * Fisher-Yates pass with RngState(seed, 2^40 + epoch), j = (int64)(0 + (i + 1)
 * * rng_next_unit) for i = n-1 .. 1, applied IN PLACE to `order` -- the
 * reference initialises the order to 0..n-1 once and reshuffles it every
 * epoch, so epoch e's order is the composition of passes 0..e. */
pgb_status pgb_shuffle_order(uint64_t seed, int64_t epoch, int64_t n, int64_t* order);
/* io::synth_for_model<float> (dataset.cpp:219-237), x (n, input_shape), y (n) */
pgb_status pgb_synth(const pgb_model_desc* desc, int64_t n, uint64_t seed,
                     float* x_out, float* y_out);

/* ---- engine : GradEngine + dpsgd_step ------------------------------------ */
pgb_status pgb_engine_create(const pgb_model_desc* desc, int32_t strategy,
                             int64_t batch, int32_t device, pgb_engine** out);
/* Data-parallel: one engine per GPU/process; `local_batch` examples each,
 * one NCCL all-reduce of the clipped sum per step. Collective over `world`. */
pgb_status pgb_nccl_unique_id(pgb_unique_id* out);
pgb_status pgb_engine_create_dist(const pgb_model_desc* desc, int32_t strategy,
                                  int64_t local_batch, int32_t device,
                                  int32_t rank, int32_t world,
                                  const pgb_unique_id* id, pgb_engine** out);
void pgb_engine_destroy(pgb_engine* e);
pgb_status pgb_engine_info_get(pgb_engine* e, pgb_engine_info* out);
pgb_status pgb_engine_set_graph(pgb_engine* e, int32_t enable);

pgb_status pgb_set_params(pgb_engine* e, const float* flat);
pgb_status pgb_get_params(pgb_engine* e, float* flat);

/* One DPSGD step from HOST buffers (x: batch*numel(input), y: batch).
 * Synchronous; norms_out (batch/m floats) and report may be NULL. */
pgb_status pgb_dpsgd_step(pgb_engine* e, const float* x, const float* y,
                          const pgb_dp_config* cfg, int64_t step_index,
                          float* norms_out, pgb_step_report* report);
/* Same step from DEVICE pointers, enqueued on the engine stream; returns
 * without synchronizing. pgb_synchronize waits and reports the last step. */
pgb_status pgb_dpsgd_step_device(pgb_engine* e, const float* d_x,
                                 const float* d_y, const pgb_dp_config* cfg,
                                 int64_t step_index);
pgb_status pgb_synchronize(pgb_engine* e, float* norms_out,
                           pgb_step_report* report);
/* sgd_step (dpsgd.cpp:334-346) */
pgb_status pgb_sgd_step(pgb_engine* e, const float* x, const float* y,
                        float learning_rate);

/* compute_views probe: per-example gradient stacks (block-major, B*P) and
 * pre-clip norms (B) for the current parameters. Either may be NULL. */
pgb_status pgb_per_example_grads(pgb_engine* e, const float* x, const float* y,
                                 float* stacks_out, float* norms_out);
/* Noise-free clipped sum  sum_i min(1, C/||g_i||) g_i  (P floats, no update),
 * pre-clip norms (batch) and clipped count: the parity probe of north-star
 * items (2)-(3). Any output may be NULL. */
pgb_status pgb_clipped_sum(pgb_engine* e, const float* x, const float* y, float clip_norm,
                           float* sum_out, float* norms_out, int64_t* clipped_out);
/* GradEngine::weighted_grad_sum (strategies.hpp:79-83, strategies.cpp:432-450):
 * sum_i w_i g_i over the batch (P floats, flat parameter order, no update);
 * w has batch entries. The second pass of the norms-only two-pass step
 * (dpsgd.cpp:194-230) with w = clip factors. One-process engines. */
pgb_status pgb_weighted_grad_sum(pgb_engine* e, const float* x, const float* y, const float* w,
                                 float* sum_out);
/* GradEngine::batch_grad_sum (strategies.hpp:85-87, strategies.cpp:453-458):
 * weighted_grad_sum with every weight 1. */
pgb_status pgb_batch_grad_sum(pgb_engine* e, const float* x, const float* y, float* sum_out);
/* Forward only: per-example losses (batch) and logits (batch*classes). */
pgb_status pgb_forward(pgb_engine* e, const float* x, const float* y, float* losses_out,
                       float* logits_out);
/* The views-path tail over caller-supplied stacks: norms, clip, clipped sum,
 * noise, mean, update (dpsgd.cpp:232-322). Updates the engine parameters. */
pgb_status pgb_aggregate(pgb_engine* e, const float* stacks,
                         const pgb_dp_config* cfg, int64_t step_index,
                         float* norms_out, pgb_step_report* report);
/* gaussian<float>(n, RngState(seed, stream)) generated on the device. */
pgb_status pgb_gaussian(int32_t device, uint64_t seed, uint64_t stream,
                        int64_t n, float* out);

/* run_bench-shaped epoch driver (harness.cpp:85-167): n/batch sequential
 * slices of host x/y, step_index = step0 + s; batches streamed H2D on a copy
 * stream (double-buffered) while the previous step computes. Per-step norms
 * (steps*batch floats) are copied back when norms_out != NULL. */
pgb_status pgb_run_epoch(pgb_engine* e, const float* x, const float* y,
                         int64_t n_examples, const pgb_dp_config* cfg,
                         int64_t step0, float* norms_out,
                         int64_t* clipped_total, double* seconds_out);

/* n_steps DPSGD steps over a device-resident ring of n_batches batches
 * (d_x: (n_batches * B, ...) device pointer); step step0 + i reads batch
 * (step0 + i) mod n_batches. Asynchronous on the engine stream; the fused
 * MNIST schedule runs as static multi-step CUDA graphs. *launches_out (nullable)
 * = kernels launched. Same semantics as n calls of pgb_dpsgd_step_device.
 * Replaces the step loop of proj/core/src/harness.cpp:147-151 on resident data. */
pgb_status pgb_run_steps_device(pgb_engine* e, const float* d_x, const float* d_y,
                                int64_t n_batches, int64_t n_steps, const pgb_dp_config* cfg,
                                int64_t step0, int64_t* launches_out);
/* Builds (captures and instantiates, without running) every CUDA graph that
 * pgb_run_steps_device(e, d_x, d_y, n_batches, n_steps, cfg, ...) will launch,
 * so a timed run that follows contains no one-time setup. Synchronous. */
pgb_status pgb_prepare_steps(pgb_engine* e, const float* d_x, const float* d_y,
                             int64_t n_batches, int64_t n_steps, const pgb_dp_config* cfg);
/* Unsigned-byte IDX containers (io::load_idx / load_mnist,
 * proj/core/src/dataset.cpp:35-112): same validation and FormatError / IoError
 * byte-offset messages. pgb_idx_info: rank (<= 4), dims, element count.
 * pgb_load_idx: float(byte) / scale_div (scale_div <= 0: no division) into a
 * host buffer of `capacity` floats; pgb_load_idx_device: the bytes cross PCIe
 * as bytes and are decoded on `device` into d_out (`capacity` floats) with the
 * same arithmetic. A payload larger than `capacity` (e.g. the file grew since
 * pgb_idx_info) fails with PGB_ERR_CONTRACT and writes nothing. */
pgb_status pgb_idx_info(const char* path, int32_t* rank, int64_t* dims, int64_t* count);
pgb_status pgb_load_idx(const char* path, float scale_div, float* out, int64_t capacity);
pgb_status pgb_load_idx_device(const char* path, int32_t device, float scale_div, float* d_out,
                               int64_t capacity);
/* Device addresses for zero-copy interop (torch, benchmarks). */
pgb_status pgb_device_params(pgb_engine* e, float** d_params);
pgb_status pgb_device_stream(pgb_engine* e, void** cuda_stream);
/* Per-kernel device time of the (non-graph) step schedule, averaged over
 * n_steps (<= 32) steps, measured with CUDA events on the engine stream
 * while the launches run back to back. names_out holds 32 chars/kernel. */
pgb_status pgb_profile_steps(pgb_engine* e, const float* d_x, const float* d_y,
                             const pgb_dp_config* cfg, int64_t step0, int32_t n_steps,
                             int32_t max_kernels, float* ms_out, char* names_out,
                             int32_t* n_kernels_out);
/* Self-test of the tcgen05 3xTF32 GEMM block: C (MxN) = A (MxK) . B (NxK)^T,
 * host buffers. */
pgb_status pgb_debug_tc_gemm(int32_t device, int32_t M, int32_t N, int32_t K, const float* A,
                             const float* B, float* C);
/* Self-test of the TMA-fed tcgen05 GEMM (tensor maps, 128-B swizzle, 3xTF32
 * with the hi/lo split on the CUDA cores): C (M x N) = A (M x K) . B (N x K)^T,
 * row-major, K a multiple of 4. */
/* self-test: one 32 x 4 TMA box at (x0, y0) of a (height, width) fp32 array */
pgb_status pgb_debug_tma_box(int32_t device, const float* src, int32_t width, int32_t height,
                             int32_t x0, int32_t y0, float* out);
pgb_status pgb_debug_tma_gemm(int32_t device, int32_t M, int32_t N, int32_t K, const float* A,
                              const float* B, float* C);
/* Self-test of the UMMA operand layouts (K-major / MN-major, no swizzle) and
 * the TMEM accumulator row map: raw TMEM dump (128 lanes x N) of
 * A (MxK) . B (NxK)^T, M in {64, 128}, K <= 32. */
pgb_status pgb_debug_umma_probe(int32_t device, int32_t M, int32_t N, int32_t K, int32_t a_mn,
                                int32_t b_mn, const float* A, const float* B, float* D_raw);
/* tcgen05 issue-rate microbenchmark: cycles for `reps` M x N x 8 tf32 MMAs;
 * strides = {a_lbo, a_sbo, b_lbo, b_sbo} bytes; mode bit 0: two accumulators. */
pgb_status pgb_debug_umma_rate(int32_t device, int32_t M, int32_t N, int32_t reps,
                               const uint32_t* strides, int32_t mode, int64_t* cycles);
/* Kernel launches recorded for the last step (profiling/evidence). */
int32_t pgb_kernels_per_step(pgb_engine* e);

#ifdef __cplusplus
}
#endif
#endif /* PEGRAD_B200_H */
