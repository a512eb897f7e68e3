/* TEST INFRASTRUCTURE — the parity oracle, NOT part of the product.
 *
 * A plain-C restatement of the reference ("pegrad", /root/reference/proj)
 * DPSGD step path, written from the reference's documented algorithm and
 * pinned against the compiled reference (oracle/_ref and the fixtures in tests/golden).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it; the product (libpegrad_b200.so) never links or calls it.
 *
 * Every function cites the reference file:line it restates.
 */
#ifndef PGB_ORACLE_H
#define PGB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same ordinals as pegrad::models::LayerKind (proj/core/include/pegrad/models.hpp:29-40). */
enum {
  ORC_DENSE = 0, ORC_CONV, ORC_MAXPOOL, ORC_AVGPOOL, ORC_GLOBAL_AVGPOOL,
  ORC_FLATTEN, ORC_RELU, ORC_EMBEDDING, ORC_SEQ_AVGPOOL, ORC_LSTM
};
/* Same ordinals as pegrad::models::ModelKind (models.hpp:24). */
enum { ORC_LOGREG = 0, ORC_FCNN, ORC_MNIST_CNN, ORC_CIFAR_CNN, ORC_EMBED, ORC_LSTM_MODEL };

/* Status codes: the pegrad exception hierarchy (common.hpp:56-114). */
enum {
  ORC_OK = 0, ORC_SHAPE = 1, ORC_DOMAIN = 2, ORC_INDEX = 3, ORC_CONFIG = 4,
  ORC_CONTRACT = 5, ORC_UNSUPPORTED = 6
};

#define ORC_MAX_LAYERS 32
#define ORC_MAX_BLOCKS 64

typedef struct {
  int32_t kind;
  int64_t in, out, k, stride, pad;
} orc_layer;

typedef struct {
  int32_t model_kind;
  int32_t n_layers;
  orc_layer layers[ORC_MAX_LAYERS];
  int32_t in_rank;
  int64_t in_shape[3];
  int64_t classes;
  int32_t token_input;
  /* registry, filled by orc_finish_desc (models.cpp:50-83) */
  int32_t n_blocks;
  int64_t block_size[ORC_MAX_BLOCKS];
  int64_t fan_in[ORC_MAX_BLOCKS];
} orc_desc;

const char* orc_last_error(void);

int orc_build_desc(int32_t model_kind, int64_t seq_len, int64_t vocab,
                   int64_t hidden, orc_desc* d);
int orc_finish_desc(orc_desc* d);
int64_t orc_param_count(const orc_desc* d);

uint64_t orc_mix64(uint64_t z);
uint64_t orc_rng_value_at(uint64_t seed, uint64_t stream, uint64_t i);
void orc_gaussian_f64(uint64_t seed, uint64_t stream, int64_t n, double* out);
void orc_gaussian_f32(uint64_t seed, uint64_t stream, int64_t n, float* out);

void orc_init_params_f64(const orc_desc* d, uint64_t seed, double* flat);
void orc_init_params_f32(const orc_desc* d, uint64_t seed, float* flat);
int orc_synth_f64(const orc_desc* d, int64_t n, uint64_t seed, double* x, double* y);
int orc_synth_f32(const orc_desc* d, int64_t n, uint64_t seed, float* x, float* y);

/* Per-example gradients of loss_i (block-major stacks: block p is
 * (B, block_size[p])), squared global norms and per-example losses. Any
 * output may be NULL. */
int orc_per_example_grads(const orc_desc* d, int64_t B, const double* x,
                          const double* y, const double* params,
                          double* stacks, double* normsq, double* losses);

/* One dpsgd_step (dpsgd.cpp:188-331) in fp64. params updated in place.
 * clipped_sum (P, nullable) receives the noise-free sum of clipped units. */
int orc_dpsgd_step(const orc_desc* d, int64_t B, const double* x,
                   const double* y, double* params, double clip, double sigma,
                   double lr, int64_t microbatch, uint64_t seed, int64_t step,
                   double* norms, int64_t* clipped, double* clipped_sum);

/* Plain SGD (dpsgd.cpp:334-346). */
int orc_sgd_step(const orc_desc* d, int64_t B, const double* x,
                 const double* y, double* params, double lr);

/* The fp32 views-path tail (dpsgd.cpp:232-322) over given fp32 stacks:
 * fp64 4-lane norms, scales, ascending-i clipped sum, noise, mean, update,
 * in the reference's exact fp32 operation order. */
int orc_aggregate_f32(int64_t B, int32_t n_blocks, const int64_t* block_size,
                      const float* stacks, float* params, float clip,
                      float sigma, float lr, uint64_t seed, int64_t step,
                      float* norms, int64_t* clipped);

#ifdef __cplusplus
}
#endif
#endif
