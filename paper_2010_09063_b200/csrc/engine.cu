// The DPSGD step engine: lowers a ModelDesc to a fixed sm_100a kernel
// schedule (no tape, no interpreter), keeps parameters and every workspace
// resident in one device arena, and replays the step as a CUDA graph.
//
// Replaces, for the GPU: GradEngine<float> (proj/core/src/strategies.cpp:
// 221-495) + the dpsgd_step views path (proj/core/src/dpsgd.cpp:188-331) +
// the run_bench epoch loop (proj/core/src/harness.cpp:85-167).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "mnist_fused.cuh"
#include "mnist_tc.cuh"
#include "mlp_fused.cuh"
#include "tc.cuh"
#include "conv_tc.cuh"
#include "pgb_internal.h"
#include "tma_gemm.cuh"

namespace pgb {

#define PGB_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      const pgb_status st_ = (e_ == cudaErrorMemoryAllocation) ? PGB_ERR_OOM : PGB_ERR_CUDA; \
      raise(st_, std::string(#call) + ": " + cudaGetErrorString(e_));                   \
    }                                                                                   \
  } while (0)

// ---- NCCL, resolved at runtime so single-GPU use never needs libnccl ------
struct Nccl {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  static Nccl& get() {
    static Nccl n = [] {
      Nccl r;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) return r;
      r.getUniqueId = (decltype(r.getUniqueId))dlsym(h, "ncclGetUniqueId");
      r.commInitRank = (decltype(r.commInitRank))dlsym(h, "ncclCommInitRank");
      r.allReduce = (decltype(r.allReduce))dlsym(h, "ncclAllReduce");
      r.commDestroy = (decltype(r.commDestroy))dlsym(h, "ncclCommDestroy");
      r.errStr = (decltype(r.errStr))dlsym(h, "ncclGetErrorString");
      r.groupStart = (decltype(r.groupStart))dlsym(h, "ncclGroupStart");
      r.groupEnd = (decltype(r.groupEnd))dlsym(h, "ncclGroupEnd");
      return r;
    }();
    if (!n.allReduce) raise(PGB_ERR_NCCL, "libnccl.so.2 could not be loaded");
    return n;
  }
};

#define PGB_NCCL(call)                                                                  \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      raise(PGB_ERR_NCCL, std::string(#call) + ": " + Nccl::get().errStr(r_));          \
  } while (0)

// ---- launch helpers -----------------------------------------------------------
inline int grid_for(size_t n, int threads = 256) {
  size_t g = (n + threads - 1) / threads;
  return (int)std::min<size_t>(std::max<size_t>(g, 1), 148 * 16);
}

template <class Op>
void launch_gemm(const Op& op, int batch, cudaStream_t s) {
  if (op.M >= 64) {
    dim3 grid((op.N + 63) / 64, (op.M + 63) / 64, batch);
    tile_gemm_kernel<Op, 64, 64, 16, 4, 4><<<grid, 256, 0, s>>>(op);
  } else if (op.M >= 32) {
    dim3 grid((op.N + 63) / 64, (op.M + 31) / 32, batch);
    tile_gemm_kernel<Op, 32, 64, 16, 4, 4><<<grid, 128, 0, s>>>(op);
  } else {
    dim3 grid((op.N + 127) / 128, (op.M + 15) / 16, batch);
    tile_gemm_kernel<Op, 16, 128, 16, 4, 4><<<grid, 128, 0, s>>>(op);
  }
}

struct Layer {
  pgb_layer_spec spec;
  ExShape in, out;
  int pblock = -1;       // first parameter block
  float* act_in = nullptr;
  float* act_out = nullptr;
  float* gout = nullptr;  // cotangent of this layer's output (backward)
  bool alias = false;    // flatten / fused relu / fused seq_avgpool: no kernel
  bool fused_relu = false;      // producer applies relu
  bool fused_pool = false;      // embedding fused with the following seq_avgpool
  bool skip_bwd = false;        // handled by a neighbour in the backward pass
  bool needs_gx = false;        // input gradient needed upstream
  const float* bwd_mask = nullptr;  // relu output to gate gx with
  // 3x3 conv on a 4x4 / 8x8 map: on the step path its weight block's
  // per-example norm is a Gram (ghost) norm and its clipped sum one
  // clip-scaled GEMM over the batch -- no per-example stack
  bool ghost = false;
  int ghost_splits = 0;         // example splits of the summed dW GEMM
};

struct Engine {
  pgb_model_desc desc{};
  int strategy = 0;
  int64_t B = 0;
  int device = 0, rank = 0, world = 1;
  // the data-parallel schedule (local clipped sum -> NCCL all-reduce ->
  // noise + update): world > 1, or a one-rank communicator forced with
  // PGB_FORCE_DIST=1 at pgb_engine_create_dist (tests drive the multi-GPU
  // kernels and the captured all-reduce on one GPU that way)
  bool dist = false;
  ncclComm_t comm = nullptr;

  std::vector<Layer> layers;
  BlockTable bt{};       // live per-example gradient sources (ghost dense blocks)
  BlockTable bt_stack{}; // the same blocks materialised in d_stacks (block-major)
  // sparse per-example embedding gradients on the step path (embedding ->
  // seq_avgpool): distinct tokens + counts per example and per-row example
  // bitmaps instead of the dense (B, V, E) stack (embed_index/agg kernels)
  int emb_layer = -1;          // the embedding layer, when the sparse path applies
  bool sparse_embed_next = false;
  bool ghost_next = false;      // this step's conv blocks go through the ghost path
  bool mlp_noise_next = false;  // this step's mlp_kernel draws the noise (dense-only models)
  bool any_ghost = false;
  bool ghost_enabled = true;    // PGB_NO_GHOST=1: per-example conv dW stacks throughout
  float* d_dw_ws = nullptr;     // split workspace of the summed dW GEMMs
  float* d_split_ws = nullptr;  // K-split workspace of the forward / input-gradient GEMMs
  bool no_ksplit = false;       // PGB_NO_KSPLIT=1: no K splits
  bool no_halo = false;         // PGB_NO_HALO=1: one TMA box per tap
  int* d_emb_tok = nullptr;    // (B, L)
  int* d_emb_cnt = nullptr;    // (B, L)
  int* d_emb_nd = nullptr;     // (B)
  unsigned* d_emb_bits = nullptr;  // (V, words)
  int emb_words = 0;
  int nparts = 1;        // fp64 norm partials per example
  bool norms_fused = false;  // per-example norms produced by the gradient kernel
  bool fused_mnist = false;  // whole per-example pass in one kernel
  bool mlp_fused = false;    // dense-only models: one warp-per-example kernel (mlp_fused.cuh)
  bool mlp_attr = false;
  bool emb_head = false;     // embedding models: dense head in mlp_kernel on the sparse path
  bool mnist_tc = false;     // ... with the conv GEMMs on tcgen05 (mnist_tc.cuh)
  bool agg_in_kernel = false;  // ... and the aggregation after an in-kernel grid barrier
  bool fuse_agg_next = false;  // set by enqueue_step for the fused launch it makes
  // multi-step graph capture, steps after the first: the tensor-core kernel
  // follows the previous step's aggregation kernel on the stream
  bool cap_pdl_tc = false;
  // conv2 W leaves the MNIST kernel as clipped pair rows (PGB_C2_PAIRS=0: per example)
  bool c2_pairs = true;
  bool pairs_next = false;     // ... for the launch enqueue_step is making
  unsigned long long* d_grid_ctr = nullptr;
  bool use_tc = true;        // conv GEMMs on tcgen05 (PGB_NO_TC=1: CUDA-core tiles)
  // 3x3 / stride-1 convolutions on the TMA-fed tcgen05 GEMM (tma_gemm.cuh;
  // PGB_NO_TMA=1: the register-gather tcgen05 GEMM of conv_tc.cuh)
  bool use_tma = true;
  // per GEMM kind, measured on the CIFAR layers (profiles/r02_cifar_*):
  // forward for C >= 16 inputs (C = 3 pads to 32 channels per tap); every
  // input gradient (since the persistent engine and the epilogue's mask loads
  // ahead of its stores: 826 -> 580 us per CIFAR step); per-example dW stays
  // on the gather GEMM (its 9 x C row tiles scatter stride-9 stores; the
  // 4x4 / 8x8 layers take the ghost path anyway). PGB_TMA_ALL=1 takes every
  // eligible GEMM (parity tests).
  bool tma_all = false;
  bool emb_agg_scalar = false;
  bool pool_generic = false;    // PGB_POOL_GENERIC=1: the generic pooling kernels  // PGB_EMB_AGG_SCALAR=1: the scalar embedding aggregation
  bool tma_fwd(const ConvGeom& g) const { return use_tma && tg::conv_ok(g) && (tma_all || g.C >= 16); }
  bool tma_dx(const ConvGeom& g) const { return use_tma && tg::conv_ok(g); }
  // few-channel 3x3 forward directly on the CUDA cores (conv3x3_smallc_fwd_kernel;
  // PGB_NO_DIRECT_CONV=1: the gather GEMM)
  bool direct_conv = true;
  bool direct_dw = true;  // PGB_NO_DIRECT_DW=1: the first layer's dW on the gather GEMM
  bool smallc_dw(const ConvGeom& g) const {
    return direct_conv && direct_dw && g.C <= 4 && g.k == 3 && g.stride == 1 && g.pad == 1 && g.Ho == g.H &&
           g.Wo == g.W && g.W == 32 &&
           smallc_dw_smem_floats<4, 2>(g.H, 8) * sizeof(float) <= 110 * 1024;
  }
  bool smallc_fwd(const ConvGeom& g) const {
    return direct_conv && g.C <= 4 && g.k == 3 && g.stride == 1 && g.pad == 1 && g.Ho == g.H &&
           g.Wo == g.W && g.W % 4 == 0 && g.D % 16 == 0;
  }
  bool tma_dw(const ConvGeom& g) const {
    return use_tma && tg::conv_ok(g) && (tma_all || dwh_sel(g));
  }
  // per-example dW on the halo kernel (tma_dw_halo_kernel) for C >= dwh_min_c
  // (PGB_NO_DW_HALO=1: off; PGB_DWH_MIN_C; PGB_DWH_ROT: accumulators per
  // kernel row, 1 or 2)
  bool dw_halo = true;
  int dwh_min_c = 16, dwh_rot = 1;
  bool dwh_raw = true;     // PGB_DWH_SPLIT=1: hi / lo operand tensors split by the layout kernels
  // conv weight-gradient work on a forked graph branch beside the input
  // gradient (PGB_NO_DW_FORK=1: in line); needs its own shifted-copy scratch
  // and a cotangent buffer per layer (no ping-pong)
  bool dw_fork = true, fork_dw_now = false;
  // the ghost layers' clip-scaled dW GEMMs on parallel branches: per-layer
  // scratch (shift copies, scaled cotangent pair, split workspace)
  static constexpr int kGhostBranches = 4;
  cudaStream_t ghost_streams[kGhostBranches - 1] = {};
  cudaEvent_t ev_gfork = nullptr, ev_gjoin[kGhostBranches - 1] = {};
  std::vector<float*> d_gcp, d_gwt, d_gwt_lo, d_gws;
  float* d_nhwc_dw = nullptr;
  bool dw_fork_ok() const { return dw_fork && dwh_raw && use_tma && !tma_all && !fused_mnist; }
  // forward / input-gradient / clipped-sum dW GEMMs: operand A as plain fp32,
  // its lo half split in the kernel (PGB_TMA_SPLIT=1: hi / lo tensors)
  bool raw_a = true;
  int dw_prep_kernels = 2;  // layout kernels of the last tma_conv_dw
  bool dwh_sel(const ConvGeom& g) const { return dw_halo && tg::dwh_ok(g) && g.C >= dwh_min_c; }
  // scratch operands of the TMA GEMMs, each as its 3xTF32 (hi, lo) pair: the
  // A operand (NHWC copy / shifted copies), the B operand (permuted weights /
  // the dW cotangent)
  float* d_nhwc = nullptr;
  float* d_nhwc_lo = nullptr;
  float* d_wt = nullptr;
  float* d_wt_lo = nullptr;
  // every TMA conv layer's weight operands, written once per step (conv_wt_all_kernel)
  float* d_wall = nullptr;
  float* d_wall_lo = nullptr;
  std::vector<long long> wall_fwd, wall_dx;  // per layer: element offset, or -1
  std::vector<int64_t> param_off;
  int64_t P = 0;
  int64_t in_row = 0;
  int first_param_layer = 0;

  static constexpr int kSlots = 3;  // epoch driver: input / result ring depth
  cudaStream_t stream = nullptr, copy_stream = nullptr, out_stream = nullptr;
  cudaStream_t side_stream = nullptr;  // fork / join branch of the embedding step
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool emb_fork = true;  // PGB_NO_EMB_FORK=1: the head's aggregation in line
  // epoch-driver staging (pinned, grown on demand) and events
  float* h_norm_stage = nullptr;
  int* h_clip_stage = nullptr;
  int64_t stage_steps = 0, stage_units = 0;
  // per-step results (norms, clip count) land in a ring of kResSlots device
  // slots read back on out_stream; the ring is deep so the compute stream
  // never waits on a read-back queued behind a large input copy
  static constexpr int kResSlots = 64;
  cudaEvent_t ev_copied[kSlots] = {}, ev_consumed[kSlots] = {}, ev_done[kResSlots] = {},
              ev_read[kResSlots] = {};
  // per-batch copies of the first chunk of a chunked epoch (its steps start as
  // soon as their own batch has landed instead of waiting for the whole chunk)
  static constexpr int kHeadSlots = kResSlots / kSlots;
  cudaEvent_t ev_head[kHeadSlots] = {};
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;

  void ensure_host_stage(int64_t steps, int64_t units) {
    if (steps <= stage_steps && units <= stage_units) return;
    if (h_norm_stage) cudaFreeHost(h_norm_stage);
    if (h_clip_stage) cudaFreeHost(h_clip_stage);
    if (h_step_base) cudaFreeHost(h_step_base);
    h_norm_stage = nullptr;
    h_clip_stage = nullptr;
    h_step_base = nullptr;
    stage_steps = std::max(steps, stage_steps);
    stage_units = std::max(units, stage_units);
    PGB_CUDA(cudaMallocHost(&h_norm_stage, sizeof(float) * stage_steps * stage_units));
    PGB_CUDA(cudaMallocHost(&h_clip_stage, sizeof(int) * 2 * stage_steps));
    // one step index per chunk (never rewritten while its copy may be pending)
    PGB_CUDA(cudaMallocHost(&h_step_base, sizeof(long long) * (stage_steps + 1)));
  }
  // epoch-driver input chunks (device, grown on demand): a pinned H2D copy
  // moves ~15-30 GB/s at one batch (0.8 MB) but ~40-50 GB/s at >= 12 MB, so
  // the driver copies several steps' batches per transfer
  float* d_xc[kSlots] = {};
  float* d_yc[kSlots] = {};
  int64_t chunk_cap = 0;
  // multi-step graphs of the epoch driver (fused MNIST): chunk slot sl runs C
  // steps from d_xc[sl]; their step indices are *d_step_base[sl] + j, so the
  // graph is static and the host only writes one value per chunk
  long long* d_step_base = nullptr;  // (kSlots + 1): chunk slots + the resident-data graph
  long long* h_step_base = nullptr;  // pinned (kSlots)
  const long long* cap_step_base = nullptr;  // set while capturing
  int cap_step_off = 0;
  const float* cap_xring = nullptr;  // resident-data ring (run_steps_device)
  const float* cap_yring = nullptr;
  int cap_ring_n = 0;
  const float* cap_x_next = nullptr;  // next step's batch inside a chunk graph
  struct ChunkGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    StepArgs args{};
    int64_t C = 0;
    int nk = 0;  // kernels per step
  };
  ChunkGraph chunk_graphs[kSlots];
  // C steps over a device-resident batch ring, one graph per C (the full
  // chunk and the remainder of a run); rebuilt when the ring or the DP
  // configuration changes
  std::map<int64_t, ChunkGraph> resident;
  const float* resident_x = nullptr;
  const float* resident_y = nullptr;
  int resident_n = 0;
  void ensure_chunk_ring(int64_t steps_per_chunk) {
    if (steps_per_chunk <= chunk_cap) return;
    for (int i = 0; i < kSlots; ++i) {
      if (d_xc[i]) cudaFree(d_xc[i]);
      if (d_yc[i]) cudaFree(d_yc[i]);
      d_xc[i] = d_yc[i] = nullptr;
    }
    chunk_cap = 0;
    for (int i = 0; i < kSlots; ++i) {
      PGB_CUDA(cudaMalloc(&d_xc[i], sizeof(float) * steps_per_chunk * B * in_row));
      PGB_CUDA(cudaMalloc(&d_yc[i], sizeof(float) * steps_per_chunk * B));
    }
    chunk_cap = steps_per_chunk;
  }
  // arena
  char* arena = nullptr;
  size_t arena_bytes = 0;
  float* d_params = nullptr;
  float* d_x = nullptr;
  float* d_y = nullptr;
  float* d_xb[kSlots] = {};
  float* d_yb[kSlots] = {};
  float* d_norms_ring = nullptr;    // (kResSlots, B)
  int* d_clip_ring = nullptr;       // (kResSlots, 2)
  // where the next launched step writes its norms / clip count
  float* norms_dst = nullptr;
  int* clipped_dst = nullptr;
  float* d_stacks = nullptr;
  float* d_wts = nullptr;  // (B) weights of pgb_weighted_grad_sum
  float* d_xin = nullptr;  // (B, in) inputs as the fused dense kernel read them
  double* d_tile_sq = nullptr;  // (B, tiles) squared sums of the conv dW GEMM tiles
  float* d_units = nullptr;
  double* d_parts = nullptr;
  float* d_cot[2] = {nullptr, nullptr};
  std::vector<float*> d_ghost_g;  // per layer: output cotangent of a ghost conv
  float* d_loss = nullptr;
  float* d_norms = nullptr;
  float* d_sum = nullptr;
  int* d_clipped = nullptr;
  DevError* d_err = nullptr;
  // fused MNIST factors
  float *d_a2 = nullptr, *d_dz1 = nullptr, *d_h = nullptr, *d_dz2 = nullptr;
  float* d_w2t = nullptr;  // conv2 weights kept transposed [k][d] for the fused kernel
  float* d_w1t = nullptr;  // conv1 weights kept transposed [(u,v)][d]
  float* d_tcw = nullptr;  // hi/lo UMMA operands of the conv weights (mnist_tc.cuh)
  float* d_noise = nullptr;   // (P) the step's normals, drawn by the fused kernel
  float* d_scale = nullptr;   // (B) clip factors, finalised by the fused kernel
  int* d_clipflag = nullptr;  // (B)
  std::vector<float*> d_dense_g;  // per dense layer: output cotangent (B, out)

  // pinned host staging
  StepArgs cur_args{};  // the step's DP arguments, passed by value to the kernels
  float* h_norms = nullptr;
  int* h_clipped = nullptr;
  DevError* h_err = nullptr;

  bool graph_enabled = true;
  bool pdl_enabled = std::getenv("PGB_NO_PDL") == nullptr;
  // One CUDA graph per schedule variant. Per-step arguments reach the graph as
  // kernel-node parameter updates (the aggregation / noise-update launch
  // structs, and the fused MNIST kernel's input pointers), so a replay needs
  // no host-to-device copy on the stream.
  struct StepGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t agg = nullptr, noise = nullptr, fused = nullptr;
    AggLaunch agg_args{};
    NoiseLaunch noise_args{};
    mnist::Params fused_args{};
    AggLaunch fused_agg{};  // the tc_kernel's in-kernel aggregation arguments
    bool fused_tc = false;
    cudaGraphNode_t emb = nullptr;  // the sparse embedding aggregation
    EmbAggLaunch emb_args{};
    cudaGraphNode_t mlp = nullptr;  // the fused dense-model kernel (inputs per step)
    mlp::Params mlp_args{};
    cudaGraphNode_t scales = nullptr;  // clip factors of a ghost-conv step
    ScalesLaunch scales_args{};
  };
  // key: (schedule variant and input slot, exact microbatch): the graph bakes
  // m and U = B/m into its microbatch / sumsq / aggregation launches
  std::map<std::pair<int, int64_t>, StepGraph> graphs;
  int kernels_last = 0;
  pgb_dp_config last_cfg{};
  int64_t last_step = 0;

  ~Engine() {
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto& kv : graphs) cudaGraphDestroy(kv.second.graph);
    if (comm) Nccl::get().commDestroy(comm);
    if (arena) cudaFree(arena);
    if (h_norms) cudaFreeHost(h_norms);
    if (h_clipped) cudaFreeHost(h_clipped);
    if (h_err) cudaFreeHost(h_err);
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (out_stream) cudaStreamDestroy(out_stream);
    if (side_stream) cudaStreamDestroy(side_stream);
    for (int i = 0; i < kGhostBranches - 1; ++i) {
      if (ghost_streams[i]) cudaStreamDestroy(ghost_streams[i]);
      if (ev_gjoin[i]) cudaEventDestroy(ev_gjoin[i]);
    }
    if (ev_gfork) cudaEventDestroy(ev_gfork);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (h_norm_stage) cudaFreeHost(h_norm_stage);
    if (h_clip_stage) cudaFreeHost(h_clip_stage);
    for (int i = 0; i < kSlots; ++i) {
      if (d_xc[i]) cudaFree(d_xc[i]);
      if (d_yc[i]) cudaFree(d_yc[i]);
      if (chunk_graphs[i].exec) cudaGraphExecDestroy(chunk_graphs[i].exec);
      if (chunk_graphs[i].graph) cudaGraphDestroy(chunk_graphs[i].graph);
    }
    for (auto& kv : resident) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
    }
    if (h_step_base) cudaFreeHost(h_step_base);
    for (int i = 0; i < kSlots; ++i)
      for (cudaEvent_t ev : {ev_copied[i], ev_consumed[i]})
        if (ev) cudaEventDestroy(ev);
    for (int i = 0; i < kResSlots; ++i)
      for (cudaEvent_t ev : {ev_done[i], ev_read[i]})
        if (ev) cudaEventDestroy(ev);
    for (int i = 0; i < kHeadSlots; ++i)
      if (ev_head[i]) cudaEventDestroy(ev_head[i]);
    if (ev_t0) cudaEventDestroy(ev_t0);
    if (ev_t1) cudaEventDestroy(ev_t1);
  }

  // 2x2 / stride-2 pooling that tiles its input exactly (pool2_*_kernel)
  bool pool2(const Layer& L) const {
    const pgb_layer_spec& sp = L.spec;
    return !pool_generic && sp.k == 2 && sp.stride == 2 && sp.pad == 0 &&
           L.in.d[1] == 2 * L.out.d[1] && L.in.d[2] == 2 * L.out.d[2] &&
           B * L.out.numel() < (1ll << 31);
  }

  static ConvGeom conv_geom(const Layer& L) {
    const pgb_layer_spec& sp = L.spec;
    return ConvGeom{(int)L.in.d[0], (int)L.in.d[1], (int)L.in.d[2], (int)L.out.d[0],
                    (int)L.out.d[1], (int)L.out.d[2], (int)sp.k, (int)sp.stride, (int)sp.pad};
  }

  // ---- convolutions on the TMA-fed tcgen05 GEMM (tma_gemm.cuh) --------------
  // forward: out (B, D, H, W) = conv(x) + bias (+ relu)
  int tma_conv_fwd(cudaStream_t s, const ConvGeom& g, int Bi, const float* x, const float* W,
                   const float* bias, float* out, bool relu, int layer = -1) {
    const int Cp = tg::round32(g.C), HW = g.H * g.W, bn = tg::pick_bn(g.D);
    tg::nchw_to_nhwc(x, d_nhwc, raw_a ? nullptr : d_nhwc_lo, g.C, HW, Cp, Bi, s);
    const bool pre = layer >= 0 && d_wall && wall_fwd[layer] >= 0;
    float* wt = pre ? d_wall + wall_fwd[layer] : d_wt;
    float* wt_lo = pre ? d_wall_lo + wall_fwd[layer] : d_wt_lo;
    if (!pre)
      tg::conv_wt_fwd_kernel<<<grid_for((size_t)g.D * 9 * Cp), 256, 0, s>>>(W, d_wt, d_wt_lo, g.D,
                                                                           g.C, Cp);
    tg::Params p{};
    int by, bnimg;
    tg::fwd_box(g, by, bnimg);
    const bool halo = halo_ok(g, bn);
    const uint64_t da[4] = {(uint64_t)Cp, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)Bi};
    const uint64_t sa[3] = {4ull * Cp, 4ull * Cp * g.W, 4ull * Cp * HW};
    const uint32_t ba[4] = {32, (uint32_t)g.W, (uint32_t)(halo ? by + 2 : by), (uint32_t)bnimg};
    tg::make_map(&p.ta, d_nhwc, 4, da, sa, ba);
    tg::make_map(&p.ta_lo, d_nhwc_lo, 4, da, sa, ba);
    p.halo = halo ? 1 : 0;
    const uint64_t db[2] = {(uint64_t)9 * Cp, (uint64_t)g.D};
    const uint64_t sb[1] = {4ull * 9 * Cp};
    const uint32_t bb[2] = {32, (uint32_t)bn};
    tg::make_map(&p.tb, wt, 2, db, sb, bb);
    tg::make_map(&p.tb_lo, wt_lo, 2, db, sb, bb);
    p.mode = tg::kConvFwd;
    p.raw = raw_a ? 1 : 0;
    p.M = Bi * HW;
    p.N = g.D;
    p.nchunks = (halo ? 3 : 9) * Cp / 32;
    p.C = g.C, p.H = g.H, p.W = g.W, p.D = g.D;
    p.Cg = Cp / 32;
    p.by = by, p.bn = bnimg;
    p.out = out;
    p.bias = bias;
    p.relu = relu ? 1 : 0;
    return (pre ? 2 : 3) + tma_launch_split(p, bn, (g.D + bn - 1) / bn, (p.M + 127) / 128, s);
  }

  // K splits of a forward / input-gradient GEMM: the tensor core's fp32
  // accumulation truncates, so each split keeps every TMEM accumulator chain
  // short (the hi.hi products rotate over tg::nacc accumulators) and the
  // splits are added in order in fp32 (round to nearest). Depends on K and
  // the tile width only -- never on the batch -- so an output element gets
  // the same arithmetic at every batch size. Chain lengths (chunks per
  // accumulator; PGB_KSPLIT_CHAIN[_FWD|_DX]) measured on the CIFAR B = 256
  // clipped sum against the reference's fp64 fixture, blocks 1-10 (block 0
  // is cancellation-bound, 7.5e-4 for every setting; the reference's own fp32
  // build is off by up to 4.6e-4): no split 1-4e-4 at 133k ex/s; forward 8
  // 1-7e-4 at 129k; forward 4 / dx 8 <= 1.0e-5 at 128k (default); 4 / 4
  // <= 9.9e-6 at 125k; 2 / 2 <= 1.6e-6 at 113k.
  static int ksplit_for(int bn, int nchunks, bool fwd = false) {
    static const int chain_fwd = env_int("PGB_KSPLIT_CHAIN_FWD", env_int("PGB_KSPLIT_CHAIN", 4));
    static const int chain_dx = env_int("PGB_KSPLIT_CHAIN_DX", env_int("PGB_KSPLIT_CHAIN", 8));
    const int nacc = bn == 16 ? 8 : bn == 32 ? 4 : bn == 64 ? 2 : 3;
    const int per = (fwd ? chain_fwd : chain_dx) * nacc;
    return std::max(1, (nchunks + per - 1) / per);
  }
  static int ksplit_mi(int nchunks, bool fwd) {
    static const int chain_fwd = env_int("PGB_KSPLIT_CHAIN_FWD", env_int("PGB_KSPLIT_CHAIN", 4));
    static const int chain_dx = env_int("PGB_KSPLIT_CHAIN_DX", env_int("PGB_KSPLIT_CHAIN", 8));
    const int chain = fwd ? chain_fwd : chain_dx;
    return std::max(1, (nchunks + chain - 1) / chain);
  }
  static int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::max(1, std::atoi(v)) : dflt;
  }


  // halo stages for the forward / input gradient: 16- and 32-wide maps whose
  // 128-position tiles are whole rows of one image, N <= 64 (PGB_NO_HALO=1: off)
  bool halo_ok(const ConvGeom& g, int bn) const {
    return !no_halo && bn <= 64 && (g.W == 16 || g.W == 32) && 128 % g.W == 0 &&
           g.H % (128 / g.W) == 0;
  }

  // launch a forward / input-gradient GEMM, split over K when it under-fills
  // the SMs (raw splits to d_split_ws, added in order by the epilogue kernel)
  int tma_launch_split(tg::Params& p, int bn, int ntn, int ntm, cudaStream_t s) {
    // (a halo chunk is three taps: the chain counts taps)
    // (halo tiles with BN <= 32: one accumulator per kernel row, so the
    // chain is the split's chunk count)
    const bool fwd = p.mode == tg::kConvFwd;
    const int S = no_ksplit ? 1
                  : p.halo && bn <= 32
                      ? std::min(p.nchunks, ksplit_mi(p.nchunks, fwd))
                      : std::min(p.nchunks, ksplit_for(bn, p.nchunks * (p.halo ? 3 : 1), fwd));
    if (S <= 1 || !d_split_ws) {
      tg::launch(p, bn, dim3(ntn, ntm, 1), s);
      return 0;
    }
    p.ksplit = S;
    p.ws = d_split_ws;
    tg::launch(p, bn, dim3(ntn, ntm, S), s);
    tg::Params q = p;
    q.ntn = ntn;
    q.ntm = ntm;
    const long long per = (long long)ntm * ntn * bn * 128;
    tg::splitk_epilogue_kernel<<<grid_for((size_t)per / 4), 256, 0, s>>>(q);
    return 1;
  }

  // input gradient: gx (B, C, H, W) = conv^T(gout) * [mask > 0]
  int tma_conv_dx(cudaStream_t s, const ConvGeom& g, int Bi, const float* gout, const float* W,
                  const float* mask, float* gx, int layer = -1) {
    const int Dp = tg::round32(g.D), HW = g.H * g.W, bn = tg::pick_bn(g.C);
    tg::nchw_to_nhwc(gout, d_nhwc, raw_a ? nullptr : d_nhwc_lo, g.D, HW, Dp, Bi, s);
    const bool pre = layer >= 0 && d_wall && wall_dx[layer] >= 0;
    float* wt = pre ? d_wall + wall_dx[layer] : d_wt;
    float* wt_lo = pre ? d_wall_lo + wall_dx[layer] : d_wt_lo;
    if (!pre)
      tg::conv_wt_dx_kernel<<<grid_for((size_t)g.C * 9 * Dp), 256, 0, s>>>(W, d_wt, d_wt_lo, g.D,
                                                                          g.C, Dp);
    tg::Params p{};
    int by, bnimg;
    tg::fwd_box(g, by, bnimg);
    const bool halo = halo_ok(g, bn);
    const uint64_t da[4] = {(uint64_t)Dp, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)Bi};
    const uint64_t sa[3] = {4ull * Dp, 4ull * Dp * g.W, 4ull * Dp * HW};
    const uint32_t ba[4] = {32, (uint32_t)g.W, (uint32_t)(halo ? by + 2 : by), (uint32_t)bnimg};
    tg::make_map(&p.ta, d_nhwc, 4, da, sa, ba);
    tg::make_map(&p.ta_lo, d_nhwc_lo, 4, da, sa, ba);
    p.halo = halo ? 1 : 0;
    const uint64_t db[2] = {(uint64_t)9 * Dp, (uint64_t)g.C};
    const uint64_t sb[1] = {4ull * 9 * Dp};
    const uint32_t bb[2] = {32, (uint32_t)bn};
    tg::make_map(&p.tb, wt, 2, db, sb, bb);
    tg::make_map(&p.tb_lo, wt_lo, 2, db, sb, bb);
    p.mode = tg::kConvDx;
    p.raw = raw_a ? 1 : 0;
    p.M = Bi * HW;
    p.N = g.C;
    p.nchunks = (halo ? 3 : 9) * Dp / 32;
    p.C = g.C, p.H = g.H, p.W = g.W, p.D = g.D;
    p.Cg = Dp / 32;
    p.by = by, p.bn = bnimg;
    p.out = gx;
    p.mask = mask;
    return (pre ? 2 : 3) + tma_launch_split(p, bn, (g.C + bn - 1) / bn, (p.M + 127) / 128, s);
  }

  // per-example weight gradient stacks (B, D, C, 3, 3) + each tile's squared
  // sum; returns the tiles per example (the tile_sq row length)
  int tma_conv_dw(cudaStream_t s, const ConvGeom& g, int Bi, const float* x, const float* gout,
                  float* stack, double* tile_sq) {
    const bool halo = dwh_sel(g);
    const int HW = g.H * g.W, bn = halo ? tg::kDwhBN : tg::pick_bn(g.D);
    int Cr, T, big, mtiles;
    if (halo)
      tg::dwh_tiling(g.C, Cr, T, mtiles), big = 0;
    else
      tg::dw_tiling(g.C, Cr, T, big, mtiles);
    const int bx = g.W, by = 32 / g.W;
    const long long total = (long long)Bi * g.C * HW;
    // halo kernel with plain fp32 operands (it splits the lo halves itself):
    // the shifted copies only, the cotangent read in place
    const bool raw = halo && dwh_raw;
    float* cp = fork_dw_now ? d_nhwc_dw : d_nhwc;  // (the forked branch has its own)
    tg::shift3_kernel<<<grid_for((size_t)total), 256, 0, s>>>(x, cp, raw ? nullptr : d_nhwc_lo,
                                                              total, g.W);
    const long long gt = (long long)Bi * g.D * HW;
    if (!raw) tg::split_kernel<<<grid_for((size_t)gt), 256, 0, s>>>(gout, d_wt, d_wt_lo, gt);
    dw_prep_kernels = raw ? 1 : 2;
    tg::Params p{};
    // A: the shifted copies [v][n][c][p] (positions flattened); B: gout [n][d][p]
    const uint64_t da[4] = {(uint64_t)HW, (uint64_t)g.C, (uint64_t)Bi, 3};
    const uint64_t sa[3] = {4ull * HW, 4ull * HW * g.C, 4ull * total};
    const uint32_t ba[4] = {32, (uint32_t)Cr, 1, 1};
    tg::make_map(&p.ta, cp, 4, da, sa, ba);
    tg::make_map(&p.ta_lo, d_nhwc_lo, 4, da, sa, ba);
    const uint64_t db[3] = {(uint64_t)HW, (uint64_t)g.D, (uint64_t)Bi};
    const uint64_t sb[2] = {4ull * HW, 4ull * HW * g.D};
    const uint32_t bb[3] = {32, (uint32_t)bn, 1};
    tg::make_map(&p.tb, raw ? gout : d_wt, 3, db, sb, bb);
    tg::make_map(&p.tb_lo, raw ? gout : d_wt_lo, 3, db, sb, bb);
    p.raw = raw ? 1 : 0;
    p.mode = tg::kConvDw;
    p.M = mtiles * 128;
    p.N = g.D;
    p.nchunks = (HW + 31) / 32;
    p.C = g.C, p.H = g.H, p.W = g.W, p.D = g.D;
    p.Cr = Cr, p.T = T, p.big_c = big;
    p.bx = bx, p.dw_by = by;
    const int ntiles = (g.D + bn - 1) / bn;
    p.tiles = ntiles * mtiles;
    p.out = stack;
    p.tile_sq = tile_sq;
    if (halo) {
      p.rot = dwh_rot;
      tg::launch_dwh(p, dim3(ntiles, mtiles, Bi), s);
      return p.tiles;
    }
    tg::launch(p, bn, dim3(ntiles, mtiles, Bi), s);
    return p.tiles;
  }

  // The reference MNIST CNN (models.cpp:107-121) runs as one fused kernel.
  static bool is_mnist(const pgb_model_desc& d) {
    const int64_t want[9][6] = {{PGB_CONV, 1, 16, 8, 2, 3},   {PGB_RELU, 0, 0, 0, 1, 0},
                                {PGB_MAXPOOL, 0, 0, 2, 2, 0}, {PGB_CONV, 16, 32, 4, 1, 0},
                                {PGB_RELU, 0, 0, 0, 1, 0},    {PGB_FLATTEN, 0, 0, 0, 1, 0},
                                {PGB_DENSE, 512, 32, 0, 1, 0}, {PGB_RELU, 0, 0, 0, 1, 0},
                                {PGB_DENSE, 32, 10, 0, 1, 0}};
    if (d.n_layers != 9 || d.input_rank != 3 || d.input_shape[0] != 1 ||
        d.input_shape[1] != 28 || d.input_shape[2] != 28 || d.classes != 10)
      return false;
    for (int l = 0; l < 9; ++l) {
      const pgb_layer_spec& L = d.layers[l];
      const bool has_geom = L.kind == PGB_CONV || L.kind == PGB_MAXPOOL;
      if (L.kind != want[l][0]) return false;
      if ((L.kind == PGB_CONV || L.kind == PGB_DENSE) && (L.in != want[l][1] || L.out != want[l][2]))
        return false;
      if (has_geom && (L.k != want[l][3] || L.stride != want[l][4] || L.pad != want[l][5]))
        return false;
    }
    return true;
  }

  // ---- planning ------------------------------------------------------------
  void plan() {
    ExShape s[PGB_MAX_LAYERS + 1];
    layer_shapes(desc, s);
    const int n = desc.n_layers;
    layers.resize(n);
    int blk = 0;
    first_param_layer = n;
    for (int l = 0; l < n; ++l) {
      Layer& L = layers[l];
      L.spec = desc.layers[l];
      L.in = s[l];
      L.out = s[l + 1];
      const int k = L.spec.kind;
      if (k == PGB_LSTM) raise(PGB_ERR_UNSUPPORTED, "unsupported layer: lstm (GPU engine)");
      if (k == PGB_DENSE || k == PGB_CONV || k == PGB_EMBEDDING) {
        L.pblock = blk;
        blk += (k == PGB_EMBEDDING) ? 1 : 2;
        if (first_param_layer == n) first_param_layer = l;
      }
      if (k == PGB_EMBEDDING && (l + 1 >= n || desc.layers[l + 1].kind != PGB_SEQ_AVGPOOL))
        raise(PGB_ERR_UNSUPPORTED,
              "unsupported layer: embedding must feed seq_avgpool (GPU engine)");
    }
    if (blk != desc.n_params) raise(PGB_ERR_CONTRACT, "parameter registry does not match layers");
    for (int l = 0; l < n; ++l) {
      Layer& L = layers[l];
      const int k = L.spec.kind;
      if (k == PGB_FLATTEN) L.alias = true;
      if (k == PGB_RELU && l > 0 &&
          (layers[l - 1].spec.kind == PGB_DENSE || layers[l - 1].spec.kind == PGB_CONV)) {
        L.alias = true;
        layers[l - 1].fused_relu = true;
      }
      if (k == PGB_SEQ_AVGPOOL && l > 0 && layers[l - 1].spec.kind == PGB_EMBEDDING) {
        L.alias = true;
        layers[l - 1].fused_pool = true;
      }
      if (k == PGB_FLATTEN || k == PGB_RELU || k == PGB_SEQ_AVGPOOL) L.skip_bwd = true;
      L.needs_gx = l > first_param_layer;
    }
    param_off.assign(desc.n_params + 1, 0);
    for (int p = 0; p < desc.n_params; ++p) param_off[p + 1] = param_off[p] + desc.param_size[p];
    P = param_off[desc.n_params];
    in_row = s[0].numel();
    fused_mnist = is_mnist(desc) && std::getenv("PGB_NO_FUSED") == nullptr;
    mnist_tc = fused_mnist && std::getenv("PGB_MNIST_SIMT") == nullptr;
    use_tc = std::getenv("PGB_NO_TC") == nullptr;
    use_tma = use_tc && std::getenv("PGB_NO_TMA") == nullptr;
    tma_all = std::getenv("PGB_TMA_ALL") != nullptr;
    emb_agg_scalar = std::getenv("PGB_EMB_AGG_SCALAR") != nullptr;
    pool_generic = std::getenv("PGB_POOL_GENERIC") != nullptr;
    ghost_enabled = std::getenv("PGB_NO_GHOST") == nullptr;
    no_ksplit = std::getenv("PGB_NO_KSPLIT") != nullptr;
    no_halo = std::getenv("PGB_NO_HALO") != nullptr;
    dw_halo = std::getenv("PGB_NO_DW_HALO") == nullptr;
    dwh_min_c = env_int("PGB_DWH_MIN_C", 16);
    dwh_rot = std::min(2, env_int("PGB_DWH_ROT", 1));
    dwh_raw = std::getenv("PGB_DWH_SPLIT") == nullptr;
    dw_fork = std::getenv("PGB_NO_DW_FORK") == nullptr;
    raw_a = std::getenv("PGB_TMA_SPLIT") == nullptr;
    direct_conv = std::getenv("PGB_NO_DIRECT_CONV") == nullptr;
    direct_dw = std::getenv("PGB_NO_DIRECT_DW") == nullptr;
    if (const char* cp = std::getenv("PGB_C2_PAIRS")) c2_pairs = std::atoi(cp) != 0;
    // dense / relu / flatten only, dense first, widths and depth within the
    // fused kernel's per-warp buffers
    {
      int nd = 0;
      bool ok = !fused_mnist && std::getenv("PGB_NO_MLP_FUSED") == nullptr && n > 0 &&
                desc.layers[0].kind == PGB_DENSE && desc.classes <= mlp::kMaxClasses;
      for (int l = 0; l < n && ok; ++l) {
        const pgb_layer_spec& sp = desc.layers[l];
        if (sp.kind == PGB_DENSE) {
          ++nd;
          ok = sp.in <= mlp::kMaxWidth && sp.out <= mlp::kMaxWidth;
        } else if (sp.kind == PGB_RELU) {
          ok = layers[l].alias;
        } else {
          ok = sp.kind == PGB_FLATTEN;
        }
      }
      mlp_fused = ok && nd >= 1 && nd <= mlp::kMaxLayers &&
                  desc.layers[n - 1].kind == PGB_DENSE && P <= mlp::kMaxParams;
    }
  }

  void allocate() {
    // size every buffer, then carve one arena (256-byte aligned slices)
    const int n = desc.n_layers;
    std::vector<std::pair<void**, size_t>> req;
    auto want = [&](void** p, size_t bytes) { req.emplace_back(p, (bytes + 255) & ~size_t(255)); };
    want((void**)&d_params, sizeof(float) * P);
    want((void**)&d_x, sizeof(float) * B * in_row);
    want((void**)&d_y, sizeof(float) * B);
    for (int i = 0; i < kSlots; ++i) {
      want((void**)&d_xb[i], sizeof(float) * B * in_row);
      want((void**)&d_yb[i], sizeof(float) * B);
    }
    want((void**)&d_norms_ring, sizeof(float) * B * kResSlots);
    want((void**)&d_clip_ring, sizeof(int) * 2 * kResSlots);
    want((void**)&d_step_base, sizeof(long long) * (kSlots + 1));
    want((void**)&d_grid_ctr, sizeof(unsigned long long));
    want((void**)&d_stacks, sizeof(float) * B * P);
    want((void**)&d_wts, sizeof(float) * B);
    want((void**)&d_xin, sizeof(float) * B * in_row);
    {
      int tiles = 1;
      for (int l = 0; l < n; ++l)
        if (desc.layers[l].kind == PGB_CONV) {
          const ExShape& in = layers[l].in;
          tiles = std::max(tiles, tc::tile_count((int)(in.d[0] * desc.layers[l].k * desc.layers[l].k),
                                                 (int)desc.layers[l].out));
        }
      int64_t nhwc = 1, wt = 1;
      for (int l = 0; l < n; ++l)
        if (desc.layers[l].kind == PGB_CONV && use_tma) {
          const ConvGeom g = conv_geom(layers[l]);
          if (!tg::conv_ok(g)) continue;
          int Cr, T, big, mt;
          tg::dw_tiling(g.C, Cr, T, big, mt);
          tiles = std::max(tiles, mt * ((g.D + tg::pick_bn(g.D) - 1) / tg::pick_bn(g.D)));
          if (tg::dwh_ok(g)) {
            tg::dwh_tiling(g.C, Cr, T, mt);
            tiles = std::max(tiles, mt * ((g.D + tg::kDwhBN - 1) / tg::kDwhBN));
          }
          const int64_t hw = (int64_t)g.H * g.W;
          nhwc = std::max(nhwc, B * hw * std::max(tg::round32(g.C), tg::round32(g.D)));
          nhwc = std::max(nhwc, 3 * B * hw * g.C);  // the dW input's shifted copies
          wt = std::max(wt, (int64_t)9 * std::max((int64_t)g.D * tg::round32(g.C),
                                                  (int64_t)g.C * tg::round32(g.D)));
          wt = std::max(wt, B * hw * g.D);  // the dW cotangent
        }
      want((void**)&d_tile_sq, sizeof(double) * B * tiles);
      int64_t split_ws = 0;
      for (int l = 0; l < n; ++l)
        if (desc.layers[l].kind == PGB_CONV && use_tma) {
          const ConvGeom g = conv_geom(layers[l]);
          if (!tg::conv_ok(g)) continue;
          const int64_t M = B * g.H * g.W, ntm = (M + 127) / 128;
          for (int side = 0; side < 2; ++side) {  // forward (N = D), input gradient (N = C)
            const int N = side ? g.C : g.D, K = side ? g.D : g.C;
            const int bn = tg::pick_bn(N), ntn = (N + bn - 1) / bn;
            const int S = std::max(ksplit_for(bn, 9 * tg::round32(K) / 32, side == 0),
                                   ksplit_mi(3 * tg::round32(K) / 32, side == 0));
            if (S > 1) split_ws = std::max<int64_t>(split_ws, (int64_t)S * ntm * ntn * bn * 128);
          }
        }
      if (split_ws) want((void**)&d_split_ws, sizeof(float) * split_ws);
      if (use_tma) {
        want((void**)&d_nhwc, sizeof(float) * nhwc);
        want((void**)&d_nhwc_lo, sizeof(float) * nhwc);
        want((void**)&d_wt, sizeof(float) * wt);
        want((void**)&d_wt_lo, sizeof(float) * wt);
        // per-layer weight operands of the forward / input-gradient GEMMs
        wall_fwd.assign(n, -1);
        wall_dx.assign(n, -1);
        long long wall = 0;
        int segs = 0;
        for (int l = 0; l < n; ++l) {
          if (desc.layers[l].kind != PGB_CONV) continue;
          const ConvGeom g = conv_geom(layers[l]);
          // (layers past conv_wt_all_kernel's segment table keep the per-GEMM
          // weight kernels)
          if (!tg::conv_ok(g) || segs + 2 > tg::kMaxWtSegs) continue;
          segs += 2;
          wall_fwd[l] = wall;
          wall += (long long)g.D * 9 * tg::round32(g.C);
          wall_dx[l] = wall;
          wall += (long long)g.C * 9 * tg::round32(g.D);
        }
        if (wall > 0) {
          want((void**)&d_wall, sizeof(float) * wall);
          want((void**)&d_wall_lo, sizeof(float) * wall);
        }
      }
    }
    want((void**)&d_units, sizeof(float) * B * P);  // microbatch means (only m>1)
    want((void**)&d_parts, sizeof(double) * B * std::max(1, desc.n_params));
    int64_t max_act = 0;
    for (int l = 0; l < n; ++l) max_act = std::max(max_act, layers[l].out.numel());
    max_act = std::max(max_act, in_row);
    want((void**)&d_cot[0], sizeof(float) * B * max_act);
    want((void**)&d_cot[1], sizeof(float) * B * max_act);
    want((void**)&d_loss, sizeof(float) * B);
    want((void**)&d_norms, sizeof(float) * B);
    want((void**)&d_sum, sizeof(float) * (P + 2));
    want((void**)&d_clipped, sizeof(int) * 2);
    want((void**)&d_err, sizeof(DevError));
    if (fused_mnist) {
      want((void**)&d_a2, sizeof(float) * B * 512);
      want((void**)&d_dz1, sizeof(float) * B * 32);
      want((void**)&d_h, sizeof(float) * B * 32);
      want((void**)&d_dz2, sizeof(float) * B * 10);
      want((void**)&d_w2t, sizeof(float) * 32 * 256);
      want((void**)&d_w1t, sizeof(float) * 16 * 64);
      want((void**)&d_tcw, sizeof(float) * kTcwFloats);
      want((void**)&d_noise, sizeof(float) * P);
      want((void**)&d_scale, sizeof(float) * B);
      want((void**)&d_clipflag, sizeof(int) * B);
    }
    if (mlp_fused && !fused_mnist) want((void**)&d_noise, sizeof(float) * P);
    for (int l = 0; l < n; ++l) {
      const Layer& L = layers[l];
      if (L.spec.kind == PGB_EMBEDDING && L.fused_pool && B <= 1024 && L.in.d[0] <= kEmbMaxL) {
        emb_layer = l;
        emb_words = (int)((B + 31) / 32);
        const int64_t Lq = L.in.d[0];
        want((void**)&d_emb_tok, sizeof(int) * B * Lq);
        want((void**)&d_emb_cnt, sizeof(int) * B * Lq);
        want((void**)&d_emb_nd, sizeof(int) * B);
        // (two bitmaps: the rows each example holds, and those it holds twice or more)
        want((void**)&d_emb_bits, sizeof(unsigned) * 2 * L.spec.in * emb_words);
        // the dense head after the pool through mlp_kernel (dense / relu only,
        // within its widths; the embedding first)
        bool ok = l == 0 && std::getenv("PGB_NO_EMB_HEAD") == nullptr &&
                  desc.classes <= mlp::kMaxClasses && L.spec.out <= mlp::kMaxWidth;
        int nd = 0, firstp = -1;
        for (int j = l + 2; j < n && ok; ++j) {
          const pgb_layer_spec& sp = desc.layers[j];
          if (sp.kind == PGB_DENSE) {
            ok = sp.in <= mlp::kMaxWidth && sp.out <= mlp::kMaxWidth;
            if (firstp < 0) firstp = layers[j].pblock;
            ++nd;
          } else {
            ok = sp.kind == PGB_RELU && layers[j].alias;
          }
        }
        emb_head = ok && nd >= 1 && nd <= mlp::kMaxLayers && l + 1 < n &&
                   desc.layers[l + 1].kind == PGB_SEQ_AVGPOOL &&
                   desc.layers[n - 1].kind == PGB_DENSE &&
                   P - param_off[firstp] <= mlp::kMaxParams;
      }
    }
    // ghost conv layers (4x4 / 8x8 maps on the TMA engine): dedicated output
    // cotangents (kept until the clip factors are known) and the split
    // workspace of their summed weight-gradient GEMMs
    d_ghost_g.assign(n, nullptr);
    any_ghost = false;
    {
      int64_t ws = 0;
      for (int l = 0; l < n; ++l) {
        Layer& L = layers[l];
        L.ghost = false;
        if (L.spec.kind != PGB_CONV || !ghost_enabled || !use_tc || !use_tma || fused_mnist)
          continue;
        // a conv reading the step input itself keeps per-example stacks (the
        // summed dW GEMM reads the layer input after the backward, when only
        // the layers' own activation buffers are stable)
        bool reads_input = true;
        for (int j = 0; j < l; ++j)
          if (!layers[j].alias) reads_input = false;
        if (reads_input) continue;
        const ConvGeom g = conv_geom(L);
        const int hw = g.H * g.W;
        if (!tg::conv_ok(g) || (hw != 16 && hw != 64)) continue;
        // shared memory of the Gram kernel: x, g and the input Gram
        if ((size_t)(g.C + g.D + hw) * hw * sizeof(float) > 160 * 1024) continue;
        L.ghost = true;
        any_ghost = true;
        want((void**)&d_ghost_g[l], sizeof(float) * B * L.out.numel());
        int Cr, T, big, mtiles;
        tg::dw_tiling(g.C, Cr, T, big, mtiles);
        const int bn = tg::pick_bn(g.D), ntiles = (g.D + bn - 1) / bn;
        const int tiles = mtiles * ntiles;
        // enough example splits to fill the SMs, at least 4 examples each
        int splits = std::max(1, std::min<int>(148 / tiles, (int)(B / 4)));
        L.ghost_splits = splits;
        ws = std::max<int64_t>(ws, (int64_t)splits * mtiles * ntiles * bn * 128);
        if (dw_fork) {
          d_gcp.resize(n, nullptr), d_gwt.resize(n, nullptr), d_gwt_lo.resize(n, nullptr);
          d_gws.resize(n, nullptr);
          want((void**)&d_gcp[l], sizeof(float) * 3 * B * hw * g.C);
          want((void**)&d_gwt[l], sizeof(float) * B * hw * g.D);
          want((void**)&d_gwt_lo[l], sizeof(float) * B * hw * g.D);
          want((void**)&d_gws[l], sizeof(float) * splits * mtiles * ntiles * bn * 128);
        }
      }
      if (any_ghost) {
        want((void**)&d_dw_ws, sizeof(float) * ws);
        if (!fused_mnist) {
          want((void**)&d_scale, sizeof(float) * B);
          want((void**)&d_clipflag, sizeof(int) * B);
        }
      }
    }
    if (dw_fork_ok()) {
      // forked weight-gradient branch: a cotangent buffer per conv layer and
      // its own shifted-copy scratch
      int64_t cp = 0;
      for (int l = 0; l < n; ++l) {
        const Layer& L = layers[l];
        if (L.spec.kind != PGB_CONV || L.ghost || L.skip_bwd) continue;
        want((void**)&d_ghost_g[l], sizeof(float) * B * L.out.numel());
        const ConvGeom g = conv_geom(L);
        if (tg::dwh_ok(g)) cp = std::max<int64_t>(cp, 3 * B * (int64_t)g.H * g.W * g.C);
      }
      if (cp) want((void**)&d_nhwc_dw, sizeof(float) * cp);
    }
    d_dense_g.assign(n, nullptr);
    for (int l = 0; l < n; ++l)
      if (layers[l].spec.kind == PGB_DENSE)
        want((void**)&d_dense_g[l], sizeof(float) * B * layers[l].spec.out);
    std::vector<float*> owned(n + 1, nullptr);
    for (int l = 0; l < n; ++l) {
      const Layer& L = layers[l];
      if (L.alias) continue;
      // embedding+seq_avgpool is one kernel writing the pooled (B, E) output
      const int64_t numel = L.fused_pool ? layers[l + 1].out.numel() : L.out.numel();
      want((void**)&owned[l + 1], sizeof(float) * B * numel);
    }
    arena_bytes = 0;
    for (auto& r : req) arena_bytes += r.second;
    PGB_CUDA(cudaMalloc(&arena, arena_bytes));
    PGB_CUDA(cudaMemset(arena, 0, arena_bytes));
    size_t o = 0;
    for (auto& r : req) {
      *r.first = arena + o;
      o += r.second;
    }
    norms_dst = d_norms;
    clipped_dst = d_clipped;
    // activation chain: act_in(0) = null = the step's input slot
    float* cur = nullptr;
    for (int l = 0; l < n; ++l) {
      Layer& L = layers[l];
      L.act_in = cur;
      L.act_out = L.alias ? cur : owned[l + 1];
      cur = L.act_out;
    }
    // masks: relu output gating the input gradient of the next real layer
    for (int l = 0; l < n; ++l) {
      Layer& L = layers[l];
      if (L.skip_bwd) continue;
      bool relu = false;
      for (int j = l - 1; j >= 0; --j) {
        const int k = layers[j].spec.kind;
        if (k == PGB_RELU) relu = true;
        if (k != PGB_RELU && k != PGB_FLATTEN) break;
      }
      L.bwd_mask = relu ? L.act_in : nullptr;
    }
    // output cotangent buffers: dense layers keep theirs (the ghost factors
    // of their weight blocks); everything else ping-pongs
    int pp = 0;
    for (int l = n - 1; l >= 0; --l) {
      Layer& L = layers[l];
      if (L.skip_bwd) continue;
      if (L.spec.kind == PGB_DENSE) {
        L.gout = d_dense_g[l];
      } else if (L.ghost) {
        L.gout = d_ghost_g[l];
      } else if (d_ghost_g[l]) {
        // (a forked weight-gradient branch may still read it when the
        // ping-pong would hand the buffer to a layer further down)
        L.gout = d_ghost_g[l];
      } else {
        L.gout = d_cot[pp];
        pp ^= 1;
      }
    }
    build_tables();
  }

  void set_block(BlockTable& t, int p, int kind, const float* base, long long stride,
                 const float* a = nullptr, long long a_stride = 0, int out = 1) {
    t.kind[p] = kind;
    t.base[p] = base;
    t.stride[p] = stride;
    t.a[p] = a;
    t.a_stride[p] = a_stride;
    t.out[p] = out;
  }

  void build_tables() {
    BlockTable t{};
    t.n = desc.n_params;
    long long pairs = 0;
    for (int p = 0; p < t.n; ++p) {
      t.size[p] = desc.param_size[p];
      t.param_off[p] = param_off[p];
      t.pair_off[p] = pairs;
      pairs += (desc.param_size[p] + 1) / 2;
    }
    t.pair_off[t.n] = pairs;
    bt_stack = t;
    for (int p = 0; p < t.n; ++p)
      set_block(bt_stack, p, 0, d_stacks + param_off[p] * B, desc.param_size[p]);
    bt = bt_stack;
    if (fused_mnist) {
      // conv blocks materialised by the fused kernel; dense blocks factored
      set_block(bt, 4, 1, d_dz1, 32, d_a2, 512, 32);
      set_block(bt, 5, 0, d_dz1, 32);
      set_block(bt, 6, 1, d_dz2, 10, d_h, 32, 10);
      set_block(bt, 7, 0, d_dz2, 10);
      // conv2 W (32, 256) -> swizzled [256][32]; conv1 W (16, 64) -> [64][16]
      for (BlockTable* t : {&bt, &bt_stack}) {
        t->shadow[2] = d_w2t;
        t->shadow_rows[2] = 32;
        t->shadow_swz[2] = 31;
        t->shadow[0] = d_w1t;
        t->shadow_rows[0] = 16;
        t->shadow_swz[0] = 0;
        if (mnist_tc) {
          t->tcw[0] = d_tcw;
          t->tcw_kind[0] = 1;
          t->tcw[2] = d_tcw;
          t->tcw_kind[2] = 2;
        }
      }
      norms_fused = true;
      nparts = 1;
    } else {
      for (int l = 0; l < desc.n_layers; ++l) {
        const Layer& L = layers[l];
        if (L.spec.kind != PGB_DENSE) continue;
        const int o = (int)L.spec.out;
        // act_in null means the step input: dense as the first layer keeps
        // its weight block materialised (the input slot is not stable)
        if (L.act_in) {
          set_block(bt, L.pblock, 1, L.gout, o, L.act_in, L.spec.in, o);
        }
        set_block(bt, L.pblock + 1, 0, L.gout, o);
      }
      // conv dW blocks: the per-example norm comes from the dW GEMM's tile sums
      if (use_tc)
        for (int l = 0; l < desc.n_layers; ++l)
          if (layers[l].spec.kind == PGB_CONV) bt.norm_pre[layers[l].pblock] = 1;
      norms_fused = false;
      nparts = t.n;
    }
  }

  // The gradient-source table for a step whose input sits at x_slot: a dense
  // first layer is factored over the input itself.
  BlockTable table_for(const float* x_slot, bool sparse = false) const {
    BlockTable t = bt;
    if (fused_mnist) return t;
    if (sparse && emb_layer >= 0) t.kind[layers[emb_layer].pblock] = 2;
    for (int l = 0; l < desc.n_layers; ++l) {
      const Layer& L = layers[l];
      if (L.spec.kind != PGB_DENSE || L.act_in) continue;
      const int o = (int)L.spec.out;
      t.kind[L.pblock] = 1;
      t.base[L.pblock] = L.gout;
      t.stride[L.pblock] = o;
      t.a[L.pblock] = mlp_fused ? d_xin : x_slot;
      t.a_stride[L.pblock] = L.spec.in;
      t.out[L.pblock] = o;
    }
    return t;
  }

  void init(const pgb_model_desc& d, int strat, int64_t batch, int dev) {
    desc = d;
    strategy = strat;
    B = batch;
    device = dev;
    if (B <= 0) raise(PGB_ERR_CONTRACT, "GradEngine: batch must be positive");
    check_strategy_support(strat, desc);
    plan();
    PGB_CUDA(cudaSetDevice(device));
    // Opt-in (PGB_GRID_SYNC=1): the aggregation inside the tensor-core kernel
    // after a grid barrier. Measured slower than the PDL-launched aggregation
    // kernel (the barrier costs ~1.3 us and the tiles run ~2x slower at the
    // kernel's 64-register budget), so the separate kernel is the default.
    if (mnist_tc && !dist && std::getenv("PGB_GRID_SYNC") != nullptr) {
      // the in-kernel grid barrier needs every CTA resident: one per SM
      int sms = 0;
      PGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      agg_in_kernel = (B + 1) / 2 <= sms;
    }
    PGB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    PGB_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    PGB_CUDA(cudaStreamCreateWithFlags(&out_stream, cudaStreamNonBlocking));
    PGB_CUDA(cudaStreamCreateWithFlags(&side_stream, cudaStreamNonBlocking));
    PGB_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    PGB_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    PGB_CUDA(cudaEventCreateWithFlags(&ev_gfork, cudaEventDisableTiming));
    for (int i = 0; i < kGhostBranches - 1; ++i) {
      PGB_CUDA(cudaStreamCreateWithFlags(&ghost_streams[i], cudaStreamNonBlocking));
      PGB_CUDA(cudaEventCreateWithFlags(&ev_gjoin[i], cudaEventDisableTiming));
    }
    emb_fork = std::getenv("PGB_NO_EMB_FORK") == nullptr;
    for (int i = 0; i < kSlots; ++i)
      for (cudaEvent_t* ev : {&ev_copied[i], &ev_consumed[i]})
        PGB_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    for (int i = 0; i < kResSlots; ++i)
      for (cudaEvent_t* ev : {&ev_done[i], &ev_read[i]})
        PGB_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    for (int i = 0; i < kHeadSlots; ++i)
      PGB_CUDA(cudaEventCreateWithFlags(&ev_head[i], cudaEventDisableTiming));
    PGB_CUDA(cudaEventCreate(&ev_t0));
    PGB_CUDA(cudaEventCreate(&ev_t1));
    allocate();
    PGB_CUDA(cudaMallocHost(&h_norms, sizeof(float) * B));
    PGB_CUDA(cudaMallocHost(&h_clipped, sizeof(int) * 2));
    PGB_CUDA(cudaMallocHost(&h_err, sizeof(DevError)));
    {
      // process-wide function attribute: allow the largest batch any engine
      // may use (the opt-in maximum), never a per-engine value
      int optin = 0;
      PGB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
      cudaFuncAttributes fa{};
      PGB_CUDA(cudaFuncGetAttributes(&fa, aggregate_kernel));
      const int room = optin - (int)fa.sharedSizeBytes;
      if ((int)agg_smem((int)B) > room)
        raise(PGB_ERR_OOM, "batch " + std::to_string(B) +
                               " exceeds the aggregation kernel's shared-memory budget");
      PGB_CUDA(cudaFuncSetAttribute(aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    room));
    }
    if (fused_mnist) {
      PGB_CUDA(cudaFuncSetAttribute(mnist::fused_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(mnist::Smem)));
      PGB_CUDA(cudaFuncSetAttribute(mnist::tc_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(mnist::TcSmem)));
      PGB_CUDA(cudaFuncSetAttribute(mnist::tc_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(mnist::TcSmem)));
    }
    // reference init is the default parameter state (models::build, seed 0)
    std::vector<float> p0(P);
    if (pgb_init_params(&desc, 0, p0.data()) != PGB_OK) raise(PGB_ERR_CONTRACT, "init failed");
    PGB_CUDA(cudaMemcpy(d_params, p0.data(), sizeof(float) * P, cudaMemcpyHostToDevice));
    refresh_shadows(stream);
    PGB_CUDA(cudaStreamSynchronize(stream));
  }

  // Keep transposed shadows in step with host-uploaded parameters.
  void refresh_shadows(cudaStream_t s) {
    for (int p = 0; p < bt.n; ++p)
      if (bt.shadow[p]) {
        const int rows = bt.shadow_rows[p], cols = (int)(bt.size[p] / rows),
                  swz = bt.shadow_swz[p];
        transpose_kernel<<<grid_for((size_t)rows * cols), 256, 0, s>>>(
            d_params + param_off[p], rows, cols, swz, bt.shadow[p]);
      }
    if (mnist_tc)
      mnist::tc_shadow_kernel<<<36, 256, 0, s>>>(d_params + param_off[0], d_params + param_off[2],
                                                 d_tcw);
  }

  // ---- profiling hook: an event after every launch while profiling --------
  std::vector<std::pair<cudaEvent_t, const char*>>* prof = nullptr;
  int mark(cudaStream_t s, const char* name) {
    static const bool debug_sync = std::getenv("PGB_DEBUG_LAUNCH") != nullptr;
    if (debug_sync) {
      cudaError_t e = cudaGetLastError();
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (e == cudaSuccess) cudaStreamIsCapturing(s, &cs);
      if (e == cudaSuccess && cs == cudaStreamCaptureStatusNone) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess)
        raise(PGB_ERR_CUDA, std::string("launch of ") + name + ": " + cudaGetErrorString(e));
    }
    if (prof) {
      cudaEvent_t ev;
      PGB_CUDA(cudaEventCreate(&ev));
      PGB_CUDA(cudaEventRecord(ev, s));
      prof->emplace_back(ev, name);
    }
    return 1;
  }

  // ---- schedule ------------------------------------------------------------
  int enqueue_forward(cudaStream_t s, const float* x_slot, const float* y_slot) {
    int nk = 0;
    const int n = desc.n_layers;
    const int Bi = (int)B;
    if (d_wall) {  // the step's weight operands for every TMA conv GEMM, one launch
      tg::WtAll A{};
      for (int l = 0; l < n && A.n + 2 <= tg::kMaxWtSegs; ++l) {
        if (wall_fwd[l] < 0) continue;
        const ConvGeom g = conv_geom(layers[l]);
        for (int kind = 0; kind < 2; ++kind) {
          const int k = A.n++;
          A.W[k] = d_params + param_off[layers[l].pblock];
          A.D[k] = g.D;
          A.C[k] = g.C;
          A.P[k] = tg::round32(kind == 0 ? g.C : g.D);
          A.kind[k] = kind;
          A.off[k] = kind == 0 ? wall_fwd[l] : wall_dx[l];
          A.off[k + 1] = A.off[k] + (long long)(kind == 0 ? g.D : g.C) * 9 * A.P[k];
        }
      }
      A.hi = d_wall;
      A.lo = d_wall_lo;
      tg::conv_wt_all_kernel<<<grid_for((size_t)A.off[A.n]), 256, 0, s>>>(A);
      nk += mark(s, "conv_wt_all");
    }
    for (int l = 0; l < n; ++l) {
      Layer& L = layers[l];
      const float* in = L.act_in ? L.act_in : x_slot;
      const pgb_layer_spec& sp = L.spec;
      const float* W = L.pblock >= 0 ? d_params + param_off[L.pblock] : nullptr;
      switch (sp.kind) {
        case PGB_DENSE: {
          DenseFwdOp op{Bi, (int)sp.out, (int)sp.in, in, W, W + sp.in * sp.out, L.act_out,
                        L.fused_relu ? 1 : 0};
          launch_gemm(op, 1, s);
          nk += mark(s, "dense_fwd");
          break;
        }
        case PGB_CONV: {
          ConvGeom g{(int)L.in.d[0], (int)L.in.d[1], (int)L.in.d[2], (int)L.out.d[0],
                     (int)L.out.d[1], (int)L.out.d[2], (int)sp.k, (int)sp.stride, (int)sp.pad};
          const int K = g.C * g.k * g.k;
          if (tma_fwd(g)) {
            const int kk = tma_conv_fwd(s, g, Bi, in, W, W + (size_t)g.D * K, L.act_out,
                                        L.fused_relu, l);
            nk += mark(s, "conv_fwd_tma") + kk - 1;
          } else if (smallc_fwd(g)) {
            const size_t sm = sizeof(float) * (size_t)(g.C * 9 + 1) * g.D;
            const long long thr = (long long)Bi * g.H * (g.W / 4);
            const int blocks = (int)std::min<long long>((thr + 255) / 256, 148ll * 8);
            switch (g.C) {
              case 1: conv3x3_smallc_fwd_kernel<1><<<blocks, 256, sm, s>>>(in, W, W + (size_t)g.D * K, L.act_out, Bi, g.D, g.H, g.W, L.fused_relu ? 1 : 0); break;
              case 2: conv3x3_smallc_fwd_kernel<2><<<blocks, 256, sm, s>>>(in, W, W + (size_t)g.D * K, L.act_out, Bi, g.D, g.H, g.W, L.fused_relu ? 1 : 0); break;
              case 3: conv3x3_smallc_fwd_kernel<3><<<blocks, 256, sm, s>>>(in, W, W + (size_t)g.D * K, L.act_out, Bi, g.D, g.H, g.W, L.fused_relu ? 1 : 0); break;
              default: conv3x3_smallc_fwd_kernel<4><<<blocks, 256, sm, s>>>(in, W, W + (size_t)g.D * K, L.act_out, Bi, g.D, g.H, g.W, L.fused_relu ? 1 : 0); break;
            }
            nk += mark(s, "conv_fwd_direct");
          } else if (use_tc) {
            tc::TcConvFwdOp op{Bi * g.Ho * g.Wo, g.D, K, g, in, W, W + (size_t)g.D * K,
                               L.act_out, L.fused_relu ? 1 : 0};
            tc::launch(op, 1, s);
            nk += mark(s, "conv_fwd_tc");
          } else {
            ConvFwdOp op{g.D, Bi * g.Ho * g.Wo, K, g, in, W, W + (size_t)g.D * K, L.act_out,
                         L.fused_relu ? 1 : 0};
            launch_gemm(op, 1, s);
            nk += mark(s, "conv_fwd");
          }
          break;
        }
        case PGB_MAXPOOL:
        case PGB_AVGPOOL: {
          const size_t tot = (size_t)B * L.out.numel();
          if (pool2(L))
            pool2_fwd_kernel<<<grid_for(tot), 256, 0, s>>>(in, L.act_out, Bi * (int)L.in.d[0],
                                                          (int)L.out.d[1], (int)L.out.d[2],
                                                          sp.kind == PGB_MAXPOOL);
          else
            pool_fwd_kernel<<<grid_for(tot), 256, 0, s>>>(
                in, L.act_out, Bi * (int)L.in.d[0], (int)L.in.d[1], (int)L.in.d[2],
                (int)L.out.d[1], (int)L.out.d[2], (int)sp.k, (int)sp.stride,
                sp.kind == PGB_MAXPOOL);
          nk += mark(s, "pool_fwd");
          break;
        }
        case PGB_GLOBAL_AVGPOOL: {
          const int BC = Bi * (int)L.in.d[0];
          gap_fwd_kernel<<<(BC * 32 + 255) / 256, 256, 0, s>>>(in, L.act_out, BC,
                                                              (int)(L.in.d[1] * L.in.d[2]));
          nk += mark(s, "gap_fwd");
          break;
        }
        case PGB_RELU:
          if (!L.alias) {
            relu_fwd_kernel<<<grid_for((size_t)B * L.in.numel()), 256, 0, s>>>(
                in, L.act_out, (size_t)B * L.in.numel());
            nk += mark(s, "relu_fwd");
          }
          break;
        case PGB_EMBEDDING: {
          const int E = (int)sp.out;
          embed_pool_fwd_kernel<<<Bi, std::min(1024, kPoolGroups * ((E + 31) / 32) * 32), 0, s>>>(
              in, W, L.act_out, Bi, (int)L.in.d[0], E, (int)sp.in, d_err);
          nk += mark(s, "embed_pool_fwd");
          break;
        }
        default:
          break;  // flatten / fused relu / fused seq_avgpool
      }
    }
    // loss and dlogits, into the cotangent buffer of the last real layer
    const Layer* top = nullptr;
    for (int l = n - 1; l >= 0 && !top; --l)
      if (!layers[l].skip_bwd) top = &layers[l];
    xent_kernel<<<(Bi + 127) / 128, 128, 0, s>>>(logits_buffer(), y_slot, Bi, (int)desc.classes,
                                                 d_loss, top->gout, d_err);
    nk += mark(s, "xent");
    return nk;
  }

  const float* logits_buffer() const { return layers.back().act_out; }

  int enqueue_fused_mnist(cudaStream_t s, const float* x_slot, const float* y_slot) {
    mnist::Params prm{};
    prm.x = x_slot;
    prm.y = y_slot;
    prm.w = d_params;
    prm.w2t = d_w2t;
    prm.w1t = d_w1t;
    for (int p = 0; p < 8; ++p) prm.off[p] = param_off[p];
    prm.st_c1w = d_stacks + param_off[0] * B;
    prm.st_c1b = d_stacks + param_off[1] * B;
    prm.st_c2w = d_stacks + param_off[2] * B;
    prm.st_c2b = d_stacks + param_off[3] * B;
    prm.a2 = d_a2;
    prm.dz1 = d_dz1;
    prm.h = d_h;
    prm.dz2 = d_dz2;
    prm.loss = d_loss;
    prm.normsq = d_parts;
    prm.err = d_err;
    prm.B = (int)B;
    prm.a = cur_args;
    prm.norms = norms_dst;
    prm.scale = d_scale;
    prm.clipped = d_clipflag;
    prm.noise = d_noise;
    long long pairs = 0;
    for (int p = 0; p < 8; ++p) {
      prm.size[p] = desc.param_size[p];
      prm.pair_off[p] = pairs;
      pairs += (desc.param_size[p] + 1) / 2;
    }
    prm.pair_off[8] = pairs;
    prm.tcw = d_tcw;
    prm.step_base = cap_step_base;
    prm.step_off = cap_step_off;
    prm.xring = cap_xring;
    prm.yring = cap_yring;
    prm.ring_origin = 0;
    prm.ring_n = cap_ring_n;
    prm.x_next = cap_x_next;
    if (mnist_tc && pairs_next) prm.c2_pairs = prm.st_c2w;
    if (mnist_tc) {
      AggLaunch L{};
      if (fuse_agg_next) {
        L = agg_launch(bt, nparts, (int)B, 0, true);
        agg_plan(L.bt, L.plan, kAggRows);  // the in-kernel tiles (agg_tile_run<.., kAggRows>)
        prm.grid_ctr = d_grid_ctr;
        prm.agg_tiles = L.plan.tile_start[L.plan.n];
      }
      if (cap_pdl_tc && pdl_enabled && !fuse_agg_next) {
        // a programmatic dependent of the previous step's aggregation
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)((B + 1) / 2));
        cfg.blockDim = dim3(mnist::TNT);
        cfg.dynamicSmemBytes = sizeof(mnist::TcSmem);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        PGB_CUDA(cudaLaunchKernelEx(&cfg, mnist::tc_kernel<false>, prm, L));
      } else {
        if (fuse_agg_next)
          mnist::tc_kernel<true><<<(unsigned)((B + 1) / 2), mnist::TNT, sizeof(mnist::TcSmem), s>>>(
              prm, L);
        else
          mnist::tc_kernel<false><<<(unsigned)((B + 1) / 2), mnist::TNT, sizeof(mnist::TcSmem), s>>>(
              prm, L);
      }
      return mark(s, fuse_agg_next ? "mnist_tc_step" : "mnist_tc");
    }
    mnist::fused_kernel<<<(unsigned)B, mnist::NT, sizeof(mnist::Smem), s>>>(prm);
    return mark(s, "mnist_fused");
  }

  // dense-only models: the whole per-example pass in mlp::mlp_kernel
  // head: the dense layers after an embedding + seq_avgpool (their input is
  // the pooled activation, their input cotangent feeds the embedding block)
  int enqueue_mlp(cudaStream_t s, const float* x_slot, const float* y_slot, bool head = false) {
    mlp::Params prm{};
    int first = -1;
    for (const Layer& L : layers) {
      if (L.spec.kind != PGB_DENSE) continue;
      if (first < 0) first = L.pblock;
      mlp::DenseLayer& D = prm.L[prm.n++];
      D.in = (int)L.spec.in;
      D.out = (int)L.spec.out;
      D.relu = L.fused_relu ? 1 : 0;
      D.pW = L.pblock;
      D.pb = L.pblock + 1;
      D.act = L.act_out;
      D.gout = L.gout;
    }
    // the dense blocks are the tail of the parameter vector (layer order)
    const long long off0 = param_off[first];
    for (int l = 0; l < prm.n; ++l) {
      prm.L[l].offW = (int)(param_off[prm.L[l].pW] - off0);
      prm.L[l].offb = (int)(param_off[prm.L[l].pb] - off0);
    }
    prm.params = d_params;
    prm.stage_off = (int)off0;
    prm.P = (int)(P - off0);
    prm.xin = head ? nullptr : d_xin;
    prm.gin = head ? layers[emb_layer].gout : nullptr;
    prm.step_base = cap_step_base;
    prm.step_off = cap_step_off;
    prm.xring = cap_xring;
    prm.yring = cap_yring;
    prm.ring_origin = 0;
    prm.ring_n = cap_ring_n;
    prm.x = x_slot;
    prm.y = y_slot;
    prm.loss = d_loss;
    prm.parts = d_parts;
    prm.nparts = nparts;
    prm.B = (int)B;
    prm.classes = (int)desc.classes;
    prm.err = d_err;
    if (head) {
      prm.x = layers[emb_layer].act_out;  // pooled (B, E)
      prm.xring = nullptr;
    }
    // dense-only models: the extra CTAs draw the step's noise for the
    // aggregation (its epilogue then only loads it)
    if (!head && d_noise && cur_args.add_noise) {
      prm.a = cur_args;
      prm.noise = d_noise;
      prm.nb_first = first;
      prm.nnb = desc.n_params - first;
      long long pairs = 0;
      for (int b = 0; b < prm.nnb; ++b) {
        prm.nb_off[b] = param_off[first + b];
        prm.nb_size[b] = desc.param_size[first + b];
        prm.nb_pair[b] = pairs;
        pairs += (prm.nb_size[b] + 1) / 2;
      }
      prm.nb_pair[prm.nnb] = pairs;
      prm.noise_ctas = (int)((pairs + 32 * mlp::kWarps - 1) / (32 * mlp::kWarps));
      mlp_noise_next = true;
    }
    const size_t smem = sizeof(float) * (size_t)prm.P;
    if (!mlp_attr) {  // once per engine (the attribute is per device)
      PGB_CUDA(cudaFuncSetAttribute(mlp::mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(sizeof(float) * mlp::kMaxParams)));
      mlp_attr = true;
    }
    mlp::mlp_kernel<<<(unsigned)((B + mlp::kWarps - 1) / mlp::kWarps + prm.noise_ctas),
                      32 * mlp::kWarps, smem, s>>>(prm);
    return mark(s, head ? "embed_head" : "mlp_fused");
  }

  // embedding models on the sparse step path: pooled forward, the dense head
  // in one kernel (forward, loss, backward to the pooled cotangent, ghost
  // norms), then the sparse embedding index
  int enqueue_embed_head_grads(cudaStream_t s, const float* x_slot, const float* y_slot) {
    int nk = 0;
    const Layer& Le = layers[emb_layer];
    const int E = (int)Le.spec.out, V = (int)Le.spec.in, Bi = (int)B;
    const float* Wt = d_params + param_off[Le.pblock];
    if (E % 4 == 0 && E <= 128 && param_off[Le.pblock] % 4 == 0 && Le.in.d[0] <= kPoolMaxL &&
        !pool_generic)
      embed_pool4_fwd_kernel<<<Bi, 32 * kPool4Groups, 0, s>>>(x_slot, Wt, Le.act_out, Bi,
                                                             (int)Le.in.d[0], E, V, d_err);
    else
      embed_pool_fwd_kernel<<<Bi, std::min(1024, kPoolGroups * ((E + 31) / 32) * 32), 0, s>>>(
          x_slot, Wt, Le.act_out, Bi, (int)Le.in.d[0], E, V, d_err);
    nk += mark(s, "embed_pool_fwd");
    nk += enqueue_mlp(s, x_slot, y_slot, true);
    embed_index_kernel<<<Bi, 256, 0, s>>>(x_slot, Le.gout, (int)Le.in.d[0], E, V, emb_words,
                                          d_emb_tok, d_emb_cnt, d_emb_nd, d_emb_bits, d_parts,
                                          nparts, Le.pblock);
    nk += mark(s, "embed_index");
    return nk;
  }

  // Per-example gradient sources for the batch (the reference's
  // compute_views); norms land in d_parts. Returns kernels launched.
  int enqueue_grads(cudaStream_t s, const float* x_slot, const float* y_slot) {
    if (fused_mnist) return enqueue_fused_mnist(s, x_slot, y_slot);
    if (mlp_fused) return enqueue_mlp(s, x_slot, y_slot);
    if (emb_head && sparse_embed_next) return enqueue_embed_head_grads(s, x_slot, y_slot);
    int nk = enqueue_forward(s, x_slot, y_slot);
    const int n = desc.n_layers;
    const int Bi = (int)B;
    const Layer* below = nullptr;
    fork_dw_now = dw_fork_ok() && !prof && d_nhwc_dw;
    bool forked = false;
    for (int l = n - 1; l >= first_param_layer; --l) {
      Layer& L = layers[l];
      if (L.skip_bwd) continue;
      // the next real layer down receives this layer's input gradient
      below = nullptr;
      for (int j = l - 1; j >= 0 && !below; --j)
        if (!layers[j].skip_bwd) below = &layers[j];
      const pgb_layer_spec& sp = L.spec;
      const float* in = L.act_in ? L.act_in : x_slot;
      const float* W = L.pblock >= 0 ? d_params + param_off[L.pblock] : nullptr;
      float* gcur = L.gout;
      float* gnext = below ? below->gout : nullptr;
      switch (sp.kind) {
        case PGB_DENSE: {
          if (L.needs_gx) {
            DenseBwdXOp op{Bi, (int)sp.in, (int)sp.out, gcur, W, L.bwd_mask, gnext};
            launch_gemm(op, 1, s);
            nk += mark(s, "dense_bwd_x");
          }
          break;
        }
        case PGB_CONV: {
          ConvGeom gg{(int)L.in.d[0], (int)L.in.d[1], (int)L.in.d[2], (int)L.out.d[0],
                      (int)L.out.d[1], (int)L.out.d[2], (int)sp.k, (int)sp.stride,
                      (int)sp.pad};
          const int K = gg.C * gg.k * gg.k, Pp = gg.Ho * gg.Wo;
          float* sW = d_stacks + param_off[L.pblock] * B;
          float* sb = d_stacks + param_off[L.pblock + 1] * B;
          // the weight-gradient work of this layer reads only its input and
          // output cotangent: on a forked branch beside the input gradient
          // (fills the SMs the other's tail leaves idle; joined after the loop)
          cudaStream_t sd = s;
          if (fork_dw_now) {
            PGB_CUDA(cudaEventRecord(ev_fork, s));
            PGB_CUDA(cudaStreamWaitEvent(side_stream, ev_fork, 0));
            sd = side_stream;
            forked = true;
          }
          if (ghost_next && L.ghost) {
            // the block's per-example norm only (ghost Gram norm); its
            // clipped sum comes later from enqueue_ghost_sums
            const int hw = gg.H * gg.W;
            const size_t sm = sizeof(float) * (size_t)(gg.C + gg.D + hw) * hw;
            if (hw == 64) {
              gram_attr(conv_gram_norm_kernel<64>, sm);
              conv_gram_norm_kernel<64><<<Bi, 256, sm, sd>>>(in, gcur, gg.C, gg.D, gg.W, d_parts,
                                                           nparts, L.pblock, sb);
            } else {
              gram_attr(conv_gram_norm_kernel<16>, sm);
              conv_gram_norm_kernel<16><<<Bi, 256, sm, sd>>>(in, gcur, gg.C, gg.D, gg.W, d_parts,
                                                           nparts, L.pblock, sb);
            }
            nk += mark(sd, "conv_dw_gram");
          } else if (smallc_dw(gg)) {
            // input rows + per-warp cotangent slices (8 warps x 2 channels, two
            // passes; two blocks per SM so one block's loads overlap the other's sums)
            auto launch = [&](auto kern, size_t floats) {
              const size_t sm = sizeof(float) * floats;
              gram_attr(kern, sm);
              kern<<<Bi, 256, sm, sd>>>(in, gcur, sW, gg.D, gg.H, d_parts, nparts, L.pblock, sb);
            };
            switch (gg.C) {
              case 1: launch(conv3x3_smallc_dw_kernel<1, 2>, smallc_dw_smem_floats<1, 2>(gg.H, 8)); break;
              case 2: launch(conv3x3_smallc_dw_kernel<2, 2>, smallc_dw_smem_floats<2, 2>(gg.H, 8)); break;
              case 3: launch(conv3x3_smallc_dw_kernel<3, 2>, smallc_dw_smem_floats<3, 2>(gg.H, 8)); break;
              default: launch(conv3x3_smallc_dw_kernel<4, 2>, smallc_dw_smem_floats<4, 2>(gg.H, 8)); break;
            }
            nk += mark(sd, "conv_dw_pex_direct");
          } else if (tma_dw(gg)) {
            const int tiles = tma_conv_dw(sd, gg, Bi, in, gcur, sW, d_tile_sq);
            nk += mark(sd, "conv_dw_pex_tma") + dw_prep_kernels;
            tile_sq_reduce_kernel<<<(Bi + 127) / 128, 128, 0, sd>>>(d_tile_sq, tiles, Bi, d_parts,
                                                                   nparts, L.pblock);
            nk += mark(sd, "conv_dw_norm");
          } else if (use_tc) {
            tc::TcConvDWOp dw{K, gg.D, Pp, gg, in, gcur, sW, d_tile_sq};
            tc::launch(dw, Bi, sd);
            nk += mark(sd, "conv_dw_pex_tc");
            // the block's per-example norm from the GEMM's tile sums (sumsq skips it)
            tile_sq_reduce_kernel<<<(Bi + 127) / 128, 128, 0, sd>>>(
                d_tile_sq, tc::tile_count(K, gg.D), Bi, d_parts, nparts, L.pblock);
            nk += mark(sd, "conv_dw_norm");
          } else {
            ConvDWOp dw{gg.D, K, Pp, gg, gcur, in, sW};
            launch_gemm(dw, Bi, sd);
            nk += mark(sd, "conv_dw_pex");
          }
          // (the Gram kernel wrote the ghost layers' bias rows, the direct dW kernel the
          // few-channel first layer's)
          if (!(ghost_next && L.ghost) && !smallc_dw(gg)) {
            conv_db_pex_kernel<<<(Bi * gg.D * 32 + 255) / 256, 256, 0, sd>>>(gcur, Bi * gg.D, Pp,
                                                                           sb);
            nk += mark(sd, "conv_db_pex");
          }
          if (L.needs_gx && tma_dx(gg)) {
            const int kk = tma_conv_dx(s, gg, Bi, gcur, W, L.bwd_mask, gnext, l);
            nk += mark(s, "conv_bwd_x_tma") + kk - 1;
          } else if (L.needs_gx && use_tc && gg.stride == 1) {
            tc::TcConvBwdXS1Op op{Bi * gg.H * gg.W, gg.C, gg.D * gg.k * gg.k, gg, gcur, W,
                                  L.bwd_mask, gnext};
            tc::launch(op, 1, s);
            nk += mark(s, "conv_bwd_x_tc");
          } else if (L.needs_gx && use_tc) {
            tc::TcConvBwdXOp op{Bi * gg.H * gg.W, gg.C, gg.D * gg.k * gg.k, gg, gcur, W,
                                L.bwd_mask, gnext};
            tc::launch(op, 1, s);
            nk += mark(s, "conv_bwd_x_tc");
          } else if (L.needs_gx) {
            ConvBwdXOp op{gg.C, Bi * gg.H * gg.W, gg.D * gg.k * gg.k, gg, gcur, W,
                          L.bwd_mask, gnext};
            launch_gemm(op, 1, s);
            nk += mark(s, "conv_bwd_x");
          }
          break;
        }
        case PGB_MAXPOOL:
        case PGB_AVGPOOL: {
          const size_t tot = (size_t)B * L.in.numel();
          if (pool2(L))
            pool2_bwd_kernel<<<grid_for((size_t)B * L.out.numel()), 256, 0, s>>>(
                in, gcur, L.bwd_mask, gnext, Bi * (int)L.in.d[0], (int)L.out.d[1],
                (int)L.out.d[2], sp.kind == PGB_MAXPOOL);
          else
            pool_bwd_kernel<<<grid_for(tot), 256, 0, s>>>(
                in, gcur, L.bwd_mask, gnext, Bi * (int)L.in.d[0], (int)L.in.d[1],
                (int)L.in.d[2], (int)L.out.d[1], (int)L.out.d[2], (int)sp.k, (int)sp.stride,
                sp.kind == PGB_MAXPOOL);
          nk += mark(s, "pool_bwd");
          break;
        }
        case PGB_GLOBAL_AVGPOOL: {
          const size_t tot = (size_t)B * L.in.numel();
          gap_bwd_kernel<<<grid_for(tot), 256, 0, s>>>(gcur, L.bwd_mask, gnext,
                                                      Bi * (int)L.in.d[0],
                                                      (int)(L.in.d[1] * L.in.d[2]));
          nk += mark(s, "gap_bwd");
          break;
        }
        case PGB_EMBEDDING: {
          const int E = (int)sp.out, V = (int)sp.in;
          if (sparse_embed_next && l == emb_layer) {
            // distinct tokens, counts, row bitmaps and the block's norm
            embed_index_kernel<<<Bi, 256, 0, s>>>(in, gcur, (int)L.in.d[0], E, V, emb_words,
                                                  d_emb_tok, d_emb_cnt, d_emb_nd, d_emb_bits,
                                                  d_parts, nparts, L.pblock);
            nk += mark(s, "embed_index");
            break;
          }
          float* st = d_stacks + param_off[L.pblock] * B;
          PGB_CUDA(cudaMemsetAsync(st, 0, sizeof(float) * B * V * E, s));
          embed_pex_kernel<<<Bi, std::min(256, ((E + 31) / 32) * 32), 0, s>>>(
              in, gcur, Bi, (int)L.in.d[0], E, V, st);
          nk += mark(s, "embed_pex");
          break;
        }
        default:
          raise(PGB_ERR_UNSUPPORTED,
                std::string("unsupported layer in backward: ") + layer_kind_name(sp.kind));
      }
    }
    if (forked) {
      PGB_CUDA(cudaEventRecord(ev_join, side_stream));
      PGB_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    }
    fork_dw_now = false;
    dim3 sg(bt.n, (unsigned)B);
    sumsq_kernel<<<sg, 128, 0, s>>>(table_for(x_slot, sparse_embed_next), Bi, d_parts);
    nk += mark(s, "sumsq");
    return nk;
  }

  // One full DPSGD step: grads -> [microbatch] -> norms/clip/sum/noise/update.
  int enqueue_step(cudaStream_t s, const float* x_slot, const float* y_slot, int64_t m) {
    int nk = 0;
    // one launch per step: the fused MNIST kernel aggregates in-kernel
    fuse_agg_next = agg_in_kernel && m == 1;
    pairs_next = fused_mnist && mnist_tc && c2_pairs && m == 1 && !fuse_agg_next;
    sparse_embed_next = emb_layer >= 0 && m == 1;
    ghost_next = any_ghost && m == 1;
    try {
      nk += enqueue_grads(s, x_slot, y_slot);
    } catch (...) {
      fuse_agg_next = sparse_embed_next = pairs_next = ghost_next = mlp_noise_next = false;
      throw;
    }
    if (fuse_agg_next) {
      fuse_agg_next = false;
      return nk;
    }
    if (m > 1) {
      const int U = (int)(B / m);
      materialize_kernel<<<grid_for((size_t)P * B), 256, 0, s>>>(table_for(x_slot), (int)B,
                                                                 d_stacks);
      nk += mark(s, "materialize");
      microbatch_kernel<<<grid_for((size_t)P * U), 256, 0, s>>>(d_stacks, bt_stack, (int)B,
                                                                 (int)m, d_units);
      nk += mark(s, "microbatch");
      BlockTable ut = bt_stack;
      for (int p = 0; p < ut.n; ++p) ut.base[p] = d_units + param_off[p] * U;
      dim3 sg(ut.n, (unsigned)U);
      sumsq_kernel<<<sg, 128, 0, s>>>(ut, U, d_parts);
      nk += mark(s, "sumsq");
      nk += enqueue_aggregate(s, ut, ut.n, U);
    } else {
      BlockTable t = table_for(x_slot, sparse_embed_next);
      if (pairs_next) {  // conv2 W: (B+1)/2 clipped pair rows in place of its stack
        t.rows[2] = (int)((B + 1) / 2);
        t.stride[2] = t.size[2];
      }
      if (ghost_next)
        nk += enqueue_ghost_aggregate(s, t);
      else
        nk += enqueue_aggregate(s, t, nparts, (int)B, fused_mnist);
    }
    sparse_embed_next = pairs_next = ghost_next = mlp_noise_next = false;
    return nk;
  }

  // Tile plan of the aggregation kernel for a block table: materialised
  // blocks in kAggCols-column tiles, factored dense blocks in kAggRows x 32
  // tiles. Returns the CTA count.
  static int agg_plan(const BlockTable& t, AggPlan& plan, int rows1 = kAggRowsSep) {
    plan.n = t.n;
    plan.rows1 = rows1;
    int tiles = 0;
    for (int p = 0; p < t.n; ++p) {
      plan.tile_start[p] = tiles;
      if (t.kind[p] == 0) {
        tiles += (int)((t.size[p] + kAggCols - 1) / kAggCols);
      } else if (t.kind[p] == 1) {
        const int64_t out = t.out[p], in = t.size[p] / out;
        tiles += (int)(((in + rows1 - 1) / rows1) * ((out + 31) / 32));
      }
    }
    plan.tile_start[t.n] = tiles;
    return tiles;
  }

  // dynamic shared memory of the aggregation kernel: clip factors + the
  // per-warp staging of factored rows
  static size_t agg_smem(int U) {
    return sizeof(float) * (((U + 3) & ~3) + kAggWarps * kAggChunk * kAggRowsSep);
  }

  // from_fused: the fused MNIST kernel already produced this step's clip
  // factors, norms, clip flags and noise (units == examples).
  AggLaunch agg_launch(const BlockTable& t, int np, int U, int mode, bool from_fused = false) {
    AggLaunch L{};
    if (from_fused) {
      L.scales = d_scale;
      L.clip_flags = d_clipflag;
      L.noise = d_noise;
    } else if (mlp_noise_next && mode == 0) {
      L.noise = d_noise;  // drawn by mlp_kernel's extra CTAs this step
    }
    L.bt = t;
    agg_plan(t, L.plan);
    L.a = cur_args;
    L.parts = d_parts;
    L.params = d_params;
    L.sum_out = d_sum;
    L.norms_out = norms_dst;
    // data-parallel steps count into the all-reduce's fixed buffer; the
    // noise-update kernel copies the reduced count into the result slot
    L.clipped_out = dist && mode == 1 ? d_clipped : clipped_dst;
    L.err = d_err;
    L.U = U;
    L.nparts = np;
    L.mode = mode;
    if (cap_step_base && !L.noise) {
      L.step_base = cap_step_base;
      L.step_off = cap_step_off;
    }
    return L;
  }

  // pdl: launch as a programmatic dependent of the previous kernel on the
  // stream (the fused MNIST kernel), hiding the launch gap between them.
  void launch_agg(const AggLaunch& L, cudaStream_t s, bool pdl = false) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)L.plan.tile_start[L.plan.n]);
    cfg.blockDim = dim3(32 * kAggWarps);
    cfg.dynamicSmemBytes = agg_smem(L.U);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    PGB_CUDA(cudaLaunchKernelEx(&cfg, aggregate_kernel, L));
  }

  // ff: the step's tail inputs come from the fused MNIST kernel that just ran
  // the sparse embedding block of table t (kind 2): its clipped sum (+ noise
  // and update in mode 0) over the rows' example lists
  int enqueue_embed_agg(cudaStream_t s, const BlockTable& t, int np, int mode) {
    const Layer& L = layers[emb_layer];
    EmbAggLaunch A{};
    A.bt = t;
    A.a = cur_args;
    A.parts = d_parts;
    A.u = L.gout;
    A.tok = d_emb_tok;
    A.cnt = d_emb_cnt;
    A.nd = d_emb_nd;
    A.bits = d_emb_bits;
    A.params = d_params;
    A.sum_out = d_sum;
    A.err = d_err;
    A.p = L.pblock;
    A.B = (int)B;
    A.L = (int)L.in.d[0];
    A.E = (int)L.spec.out;
    A.V = (int)L.spec.in;
    A.words = emb_words;
    A.nparts = np;
    A.mode = mode;
    if (cap_step_base) {
      A.step_base = cap_step_base;
      A.step_off = cap_step_off;
    }
    const int rows_per_cta = 8;
    const int grid = std::min<int>((A.V + rows_per_cta - 1) / rows_per_cta, 148 * 8);
    // four elements per lane when the table rows are 16-byte aligned and the
    // block has no shadow copies (PGB_EMB_AGG_SCALAR=1: the scalar kernel);
    // it takes the norms from the fp64 partials itself
    const bool vec4 = A.E % 4 == 0 && t.param_off[A.p] % 4 == 0 && !t.shadow[A.p] &&
                      !t.tcw[A.p] && B <= 1024 && !emb_agg_scalar;
    if (vec4) {  // one wave: six 34-KB CTAs per SM
      embed_agg4_kernel<<<std::min(grid, 148 * 6), 32 * kEmbAggWarps, sizeof(float) * B, s>>>(A);
      return mark(s, mode == 0 ? "embed_agg" : "embed_agg_local");
    }
    finalize_norms_kernel<<<((int)B + 127) / 128, 128, 0, s>>>(d_parts, np, (int)B, d_wts);
    const int nk0 = mark(s, "embed_norms");
    A.norms = d_wts;  // (the weighted-sum weights buffer, free on the step path)
    embed_agg_kernel<<<grid, 256, sizeof(float) * B, s>>>(A);
    return nk0 + mark(s, mode == 0 ? "embed_agg" : "embed_agg_local");
  }

  int enqueue_aggregate(cudaStream_t s, const BlockTable& t, int np, int U, bool ff = false) {
    int nk = 0;
    const bool emb = emb_layer >= 0 && t.kind[layers[emb_layer].pblock] == 2;
    if (!dist && emb && emb_fork && !prof) {  // (per-kernel profiling needs one stream order)
      // the dense head's aggregation (a few latency-bound CTAs) on a side
      // branch beside the embedding table's: independent blocks, both after
      // embed_index (fork / join by events; a captured graph keeps them as
      // parallel branches)
      PGB_CUDA(cudaEventRecord(ev_fork, s));
      PGB_CUDA(cudaStreamWaitEvent(side_stream, ev_fork, 0));
      launch_agg(agg_launch(t, np, U, 0, ff), side_stream);
      nk += mark(side_stream, "aggregate");
      PGB_CUDA(cudaEventRecord(ev_join, side_stream));
      nk += enqueue_embed_agg(s, t, np, 0);
      PGB_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    } else if (!dist) {
      launch_agg(agg_launch(t, np, U, 0, ff), s, (ff || mlp_fused) && pdl_enabled);
      nk += mark(s, "aggregate");
      if (emb) nk += enqueue_embed_agg(s, t, np, 0);
    } else {
      launch_agg(agg_launch(t, np, U, 1, ff), s);
      nk += mark(s, "aggregate_local");
      if (emb) nk += enqueue_embed_agg(s, t, np, 1);
      // one all-reduce of the clipped sum (+ the clip count beside it); NCCL
      // returns identical bytes on every rank, so the replicas stay in step
      auto& N = Nccl::get();
      PGB_NCCL(N.groupStart());
      PGB_NCCL(N.allReduce(d_sum, d_sum, (size_t)P, ncclFloat32, ncclSum, comm, s));
      PGB_NCCL(N.allReduce(d_clipped, d_clipped + 1, 1, ncclInt32, ncclSum, comm, s));
      PGB_NCCL(N.groupEnd());
      // the same noise on every rank (shared seed, counter-based streams):
      // drawn by the fused MNIST kernel already, else here, once per pair
      NoiseLaunch L{};
      L.bt = t;
      L.a = cur_args;
      L.sum = d_sum;
      L.params = d_params;
      L.err = d_err;
      L.noise = ff ? d_noise : nullptr;
      L.step_base = cap_step_base;
      L.step_off = cap_step_off;
      L.cnt_in = d_clipped;
      L.clipped_out = clipped_dst;
      L.only_kind = -1;
      int64_t pairs = 0;
      for (int p = 0; p < t.n; ++p) pairs += (t.size[p] + 1) / 2;
      noise_update_kernel<<<grid_for((size_t)pairs), 256, 0, s>>>(L);
      nk += mark(s, "noise_update");
    }
    return nk;
  }

  // process-wide function attribute: only ever raised (a lower value set for
  // a later layer would make an earlier launch -- or its graph node replayed
  // by a profiler -- exceed it)
  template <class K>
  void gram_attr(K* kern, size_t smem) {
    // (per device: the attribute is a property of the function on each device)
    static std::map<std::pair<int, const void*>, size_t> set;
    size_t& cur = set[{device, (const void*)kern}];
    if (smem > 48 * 1024 && smem > cur) {
      PGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      cur = smem;
    }
  }

  // The clipped sums sum_i s_i dW_i of the ghost conv blocks into d_sum: the
  // input's column-shifted copies and the clip-scaled cotangent as 3xTF32
  // pairs, one GEMM over (example, position) split over the examples, the
  // splits added in order.
  int enqueue_ghost_sums(cudaStream_t s0) {
    int nk = 0;
    // parallel branches (layer k on stream k % 4, per-layer scratch; the
    // kernels' tails and the small copy / reduce launches overlap)
    const bool par = dw_fork && raw_a && !prof && !d_gws.empty();
    if (par) PGB_CUDA(cudaEventRecord(ev_gfork, s0));
    int k = 0, used = 0;
    for (int l = 0; l < desc.n_layers; ++l) {
      const Layer& L = layers[l];
      if (!L.ghost) continue;
      const int br = par ? k % kGhostBranches : 0;
      ++k;
      cudaStream_t s = br ? ghost_streams[br - 1] : s0;
      if (br && !(used & (1 << br))) {
        PGB_CUDA(cudaStreamWaitEvent(s, ev_gfork, 0));
        used |= 1 << br;
      }
      float* cp = par ? d_gcp[l] : d_nhwc;
      float* wt = par ? d_gwt[l] : d_wt;
      float* wt_lo = par ? d_gwt_lo[l] : d_wt_lo;
      float* wsp = par ? d_gws[l] : d_dw_ws;
      const ConvGeom g = conv_geom(L);
      const int Bi = (int)B, HW = g.H * g.W, bn = tg::pick_bn(g.D);
      int Cr, T, big, mtiles;
      tg::dw_tiling(g.C, Cr, T, big, mtiles);
      const long long total = (long long)Bi * g.C * HW;
      const float* in = L.act_in;
      tg::shift3_kernel<<<grid_for((size_t)total), 256, 0, s>>>(
          in, cp, raw_a ? nullptr : d_nhwc_lo, total, g.W);
      const long long gt = (long long)Bi * g.D * HW;
      tg::scale_split_kernel<<<grid_for((size_t)gt), 256, 0, s>>>(L.gout, d_scale,
                                                                  (long long)g.D * HW, gt, wt,
                                                                  wt_lo);
      tg::Params p{};
      const uint64_t da[4] = {(uint64_t)HW, (uint64_t)g.C, (uint64_t)Bi, 3};
      const uint64_t sa[3] = {4ull * HW, 4ull * HW * g.C, 4ull * total};
      const uint32_t ba[4] = {32, (uint32_t)Cr, 1, 1};
      tg::make_map(&p.ta, cp, 4, da, sa, ba);
      tg::make_map(&p.ta_lo, d_nhwc_lo, 4, da, sa, ba);
      const uint64_t db[3] = {(uint64_t)HW, (uint64_t)g.D, (uint64_t)Bi};
      const uint64_t sb[2] = {4ull * HW, 4ull * HW * g.D};
      const uint32_t bb[3] = {32, (uint32_t)bn, 1};
      tg::make_map(&p.tb, wt, 3, db, sb, bb);
      tg::make_map(&p.tb_lo, wt_lo, 3, db, sb, bb);
      p.mode = tg::kConvDwSum;
      p.raw = raw_a ? 1 : 0;
      p.M = mtiles * 128;
      p.N = g.D;
      p.nchunks = (HW + 31) / 32;
      p.C = g.C, p.H = g.H, p.W = g.W, p.D = g.D;
      p.Cr = Cr, p.T = T, p.big_c = big;
      p.bx = g.W, p.dw_by = 32 / g.W;
      const int ntiles = (g.D + bn - 1) / bn;
      p.tiles = ntiles * mtiles;
      const int S = L.ghost_splits;
      p.ex_per = (Bi + S - 1) / S;
      p.nex = Bi;
      p.ws = wsp;
      const int splits = (Bi + p.ex_per - 1) / p.ex_per;
      tg::launch(p, bn, dim3(ntiles, mtiles, splits), s);
      const long long per = (long long)mtiles * ntiles * bn * 128;
      tg::dw_sum_reduce_kernel<<<grid_for((size_t)per), 256, 0, s>>>(
          wsp, splits, mtiles, ntiles * bn, g.C, g.D, Cr, T, big,
          d_sum + param_off[L.pblock]);
      nk += mark(s, "conv_dw_sum") + 3;
    }
    for (int br = 1; br < kGhostBranches; ++br)
      if (used & (1 << br)) {
        PGB_CUDA(cudaEventRecord(ev_gjoin[br - 1], ghost_streams[br - 1]));
        PGB_CUDA(cudaStreamWaitEvent(s0, ev_gjoin[br - 1], 0));
      }
    return nk;
  }

  // The step's tail when ghost conv blocks are present: clip factors once,
  // the ghost blocks' clipped sums by GEMM, the other blocks through the
  // aggregation kernel (with the clip factors given), then noise / mean /
  // update of the ghost blocks (single process) or of everything after the
  // all-reduce (data-parallel).
  int enqueue_ghost_aggregate(cudaStream_t s, const BlockTable& t) {
    int nk = 0;
    ScalesLaunch SL{d_parts, nparts, (int)B, cur_args, d_scale, d_clipflag, norms_dst};
    step_scales_kernel<<<((int)B + 127) / 128, 128, 0, s>>>(SL);
    nk += mark(s, "step_scales");
    BlockTable t2 = t;
    for (const Layer& L : layers)
      if (L.ghost) t2.kind[L.pblock] = 3;  // no aggregation tiles: summed by GEMM
    AggLaunch A = agg_launch(t2, nparts, (int)B, dist ? 1 : 0);
    A.scales = d_scale;
    A.clip_flags = d_clipflag;
    // single process: the aggregation (the other blocks' clipped sums, noise
    // and update) touches none of the ghost blocks' buffers, so it runs on a
    // forked branch beside their GEMMs (PGB_NO_DW_FORK=1: in line)
    const bool fork = !dist && !prof && dw_fork;
    if (fork) {
      PGB_CUDA(cudaEventRecord(ev_fork, s));
      PGB_CUDA(cudaStreamWaitEvent(side_stream, ev_fork, 0));
      launch_agg(A, side_stream);
      nk += mark(side_stream, "aggregate");
      PGB_CUDA(cudaEventRecord(ev_join, side_stream));
    }
    nk += enqueue_ghost_sums(s);
    if (!fork) {
      launch_agg(A, s);
      nk += mark(s, dist ? "aggregate_local" : "aggregate");
    }
    if (dist) {
      auto& N = Nccl::get();
      PGB_NCCL(N.groupStart());
      PGB_NCCL(N.allReduce(d_sum, d_sum, (size_t)P, ncclFloat32, ncclSum, comm, s));
      PGB_NCCL(N.allReduce(d_clipped, d_clipped + 1, 1, ncclInt32, ncclSum, comm, s));
      PGB_NCCL(N.groupEnd());
    }
    NoiseLaunch NL{};
    NL.bt = t2;
    NL.a = cur_args;
    NL.sum = d_sum;
    NL.params = d_params;
    NL.err = d_err;
    NL.noise = nullptr;
    NL.step_base = cap_step_base;
    NL.step_off = cap_step_off;
    NL.cnt_in = d_clipped;
    NL.clipped_out = dist ? clipped_dst : nullptr;
    NL.only_kind = dist ? -1 : 3;
    int64_t pairs = 0;
    for (int p = 0; p < t2.n; ++p) pairs += (t2.size[p] + 1) / 2;
    noise_update_kernel<<<grid_for((size_t)pairs), 256, 0, s>>>(NL);
    nk += mark(s, "noise_update");
    if (fork) PGB_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    return nk;
  }

  // Noise-free clipped sum of the batch into d_sum (no update): the
  // north-star parity probe.
  int enqueue_local_sum(cudaStream_t s, const BlockTable& t, int np, int U) {
    launch_agg(agg_launch(t, np, U, 1), s);
    return 1;
  }

  // dpsgd_step's checks (dpsgd.cpp:36-51) plus the norms-only strategy's
  // microbatch restriction (dpsgd.cpp:194-199)
  void validate_step(const pgb_dp_config& c) const {
    validate_dp_config(c, B);
    if (strategy == PGB_NORMS && c.microbatch != 1)
      raise(PGB_ERR_CONFIG, "dpsgd_step: the norms-only strategy supports microbatch = 1 only");
  }

  // sum_i w_i g_i of the batch into d_sum (GradEngine::weighted_grad_sum,
  // strategies.cpp:432-450): the per-example sources of enqueue_grads summed
  // by the aggregation kernel with the weights in place of clip factors
  void enqueue_weighted_sum(cudaStream_t s, const float* x_slot, const float* y_slot,
                            const float* d_w) {
    enqueue_grads(s, x_slot, y_slot);
    const BlockTable t = table_for(x_slot);
    AggLaunch L = agg_launch(t, nparts, (int)B, 1);
    L.scales = d_w;
    L.clip_flags = d_clipflag;
    L.noise = nullptr;
    L.norms_out = nullptr;
    L.clipped_out = nullptr;
    launch_agg(L, s);
  }

  // ---- step arguments ---------------------------------------------------------
  void push_args(const StepArgs& a) { cur_args = a; }

  StepArgs make_args(const pgb_dp_config& c, int64_t step, const float* x, const float* y) {
    StepArgs a{};
    const int64_t units = (B / c.microbatch) * world;
    a.clip = c.clip_norm;
    a.sigma = c.noise_multiplier;
    a.lr = c.learning_rate;
    a.inv_units = 1.0f / static_cast<float>(units);
    a.seed = c.seed;
    a.step = step;
    a.units = (int)(B / c.microbatch);
    a.add_noise = c.noise_multiplier > 0.0f;
    (void)x;
    (void)y;
    return a;
  }

  // Launch the step for inputs already resident at d_x/d_y slots.
  void launch_step(const float* x_slot, const float* y_slot, int64_t m) {
    const int variant = (m > 1 ? 1 : 0) | (dist ? 2 : 0);
    // the fused MNIST schedule takes its input pointers as updatable node
    // parameters; the layer-wise schedule bakes the input slot into the graph
    int slot_key = 0;
    for (int i = 0; i < kSlots; ++i)
      if (x_slot == d_xb[i]) slot_key = i + 1;
    const int key = variant * (kSlots + 1) + ((fused_mnist || mlp_fused) ? 0 : slot_key);
    if (!graph_enabled) {
      kernels_last = enqueue_step(stream, x_slot, y_slot, m);
      PGB_CUDA(cudaGetLastError());
      return;
    }
    const std::pair<int, int64_t> gkey{key, m};
    auto it = graphs.find(gkey);
    if (it == graphs.end()) {
      StepGraph sg;
      PGB_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      int nk = 0;
      try {
        nk = enqueue_step(stream, x_slot, y_slot, m);
      } catch (...) {
        cudaStreamEndCapture(stream, &sg.graph);
        if (sg.graph) cudaGraphDestroy(sg.graph);
        throw;
      }
      PGB_CUDA(cudaStreamEndCapture(stream, &sg.graph));
      PGB_CUDA(cudaGraphInstantiate(&sg.exec, sg.graph, 0));
      find_step_nodes(sg);
      it = graphs.emplace(gkey, sg).first;
      kernels_last = nk;
    }
    update_step_nodes(it->second, x_slot, y_slot);
    PGB_CUDA(cudaGraphLaunch(it->second.exec, stream));
  }

  // The static graph of C consecutive steps reading chunk slot sl (fused
  // MNIST, one process): step j reads batch j of d_xc[sl], takes its step
  // index from d_step_base[sl] + j and writes its results to result slot
  // sl * C + j. Rebuilt only when C or the DP configuration changes.
  cudaGraphExec_t chunk_graph(int sl, int64_t C, const StepArgs& args) {
    ChunkGraph& cg = chunk_graphs[sl];
    StepArgs a0 = args;
    a0.step = 0;
    if (cg.exec && cg.C == C && std::memcmp(&cg.args, &a0, sizeof(StepArgs)) == 0) return cg.exec;
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
    if (cg.graph) cudaGraphDestroy(cg.graph);
    cg = ChunkGraph{};
    float* nd0 = norms_dst;
    int* cd0 = clipped_dst;
    PGB_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    try {
      for (int64_t j = 0; j < C; ++j) {
        cur_args = a0;
        norms_dst = d_norms_ring + (size_t)(sl * C + j) * B;
        clipped_dst = d_clip_ring + 2 * (sl * C + j);
        cap_step_base = d_step_base + sl;
        cap_step_off = (int)j;
        cap_pdl_tc = j > 0;
        cap_x_next = j + 1 < C ? d_xc[sl] + (j + 1) * B * in_row : nullptr;
        kernels_last = enqueue_step(stream, d_xc[sl] + j * B * in_row, d_yc[sl] + j * B, 1);
      }
    } catch (...) {
      cap_step_base = nullptr;
      cap_pdl_tc = false;
      cap_x_next = nullptr;
      cudaStreamEndCapture(stream, &cg.graph);
      if (cg.graph) cudaGraphDestroy(cg.graph);
      cg.graph = nullptr;
      throw;
    }
    cap_step_base = nullptr;
    cap_step_off = 0;
    cap_pdl_tc = false;
    cap_x_next = nullptr;
    norms_dst = nd0;
    clipped_dst = cd0;
    PGB_CUDA(cudaStreamEndCapture(stream, &cg.graph));
    PGB_CUDA(cudaGraphInstantiate(&cg.exec, cg.graph, 0));
    cg.args = a0;
    cg.C = C;
    return cg.exec;
  }

  // The static graph of C consecutive steps over a device-resident ring of
  // n batches (step s reads batch s mod n; the step index lives in
  // d_step_base[kSlots] and the graph's last node advances it by C).
  cudaGraphExec_t resident_graph(int64_t C, const StepArgs& args, const float* xr,
                                 const float* yr, int n) {
    StepArgs a0 = args;
    a0.step = 0;
    if (resident_x != xr || resident_y != yr || resident_n != n) {
      // another ring: every resident graph bakes the old one
      for (auto& kv : resident) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
      }
      resident.clear();
    }
    ChunkGraph& cg = resident[C];
    if (cg.exec && cg.C == C && std::memcmp(&cg.args, &a0, sizeof(StepArgs)) == 0 &&
        resident_x == xr && resident_y == yr && resident_n == n) {
      kernels_last = cg.nk;
      return cg.exec;
    }
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
    if (cg.graph) cudaGraphDestroy(cg.graph);
    cg = ChunkGraph{};
    PGB_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    try {
      for (int64_t j = 0; j < C; ++j) {
        cur_args = a0;
        cap_step_base = d_step_base + kSlots;
        cap_step_off = (int)j;
        cap_pdl_tc = j > 0;
        cap_xring = xr;
        cap_yring = yr;
        cap_ring_n = n;
        kernels_last = enqueue_step(stream, xr, yr, 1);
      }
      advance_counter_kernel<<<1, 1, 0, stream>>>(d_step_base + kSlots, C);
    } catch (...) {
      cap_step_base = nullptr;
      cap_pdl_tc = false;
      cap_xring = cap_yring = nullptr;
      cudaStreamEndCapture(stream, &cg.graph);
      if (cg.graph) cudaGraphDestroy(cg.graph);
      cg.graph = nullptr;
      throw;
    }
    cap_step_base = nullptr;
    cap_step_off = 0;
    cap_pdl_tc = false;
    cap_xring = cap_yring = nullptr;
    cap_ring_n = 0;
    PGB_CUDA(cudaStreamEndCapture(stream, &cg.graph));
    PGB_CUDA(cudaGraphInstantiate(&cg.exec, cg.graph, 0));
    cg.args = a0;
    cg.C = C;
    cg.nk = kernels_last;
    resident_x = xr;
    resident_y = yr;
    resident_n = n;
    return cg.exec;
  }

  // The kernel nodes whose parameters change from step to step.
  void find_step_nodes(StepGraph& sg) {
    size_t n = 0;
    PGB_CUDA(cudaGraphGetNodes(sg.graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    PGB_CUDA(cudaGraphGetNodes(sg.graph, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      PGB_CUDA(cudaGraphNodeGetType(nd, &ty));
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      PGB_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == (void*)aggregate_kernel && (sg.agg == nullptr || sg.agg_args.mode != 0)) {
        const AggLaunch* L = static_cast<const AggLaunch*>(kp.kernelParams[0]);
        if (sg.agg == nullptr || L->mode == 0) {
          sg.agg = nd;
          sg.agg_args = *L;
        }
      } else if (kp.func == (void*)mlp::mlp_kernel &&
                 static_cast<const mlp::Params*>(kp.kernelParams[0])->gin == nullptr) {
        // (an embedding head reads the pooled activation, not the step input)
        sg.mlp = nd;
        sg.mlp_args = *static_cast<const mlp::Params*>(kp.kernelParams[0]);
      } else if (kp.func == (void*)embed_agg_kernel || kp.func == (void*)embed_agg4_kernel) {
        sg.emb = nd;
        sg.emb_args = *static_cast<const EmbAggLaunch*>(kp.kernelParams[0]);
      } else if (kp.func == (void*)noise_update_kernel) {
        sg.noise = nd;
        sg.noise_args = *static_cast<const NoiseLaunch*>(kp.kernelParams[0]);
      } else if (kp.func == (void*)step_scales_kernel) {
        sg.scales = nd;
        sg.scales_args = *static_cast<const ScalesLaunch*>(kp.kernelParams[0]);
      } else if (kp.func == (void*)mnist::fused_kernel ||
                 kp.func == (void*)mnist::tc_kernel<false> ||
                 kp.func == (void*)mnist::tc_kernel<true>) {
        sg.fused = nd;
        sg.fused_args = *static_cast<const mnist::Params*>(kp.kernelParams[0]);
        if (kp.func != (void*)mnist::fused_kernel) {
          sg.fused_tc = true;
          sg.fused_agg = *static_cast<const AggLaunch*>(kp.kernelParams[1]);
        }
      }
    }
  }

  static bool same_args(const StepArgs& a, const StepArgs& b) {
    return std::memcmp(&a, &b, sizeof(StepArgs)) == 0;
  }

  void set_node(cudaGraphExec_t ex, cudaGraphNode_t nd, void* arg, void* arg2 = nullptr) {
    cudaKernelNodeParams kp{};
    PGB_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
    void* params[2] = {arg, arg2};
    kp.kernelParams = params;
    kp.extra = nullptr;
    PGB_CUDA(cudaGraphExecKernelNodeSetParams(ex, nd, &kp));
  }

  void update_step_nodes(StepGraph& sg, const float* x_slot, const float* y_slot) {
    int* agg_cnt = (dist && sg.agg_args.mode == 1) ? d_clipped : clipped_dst;
    if (sg.agg && (!same_args(sg.agg_args.a, cur_args) || sg.agg_args.norms_out != norms_dst ||
                   sg.agg_args.clipped_out != agg_cnt)) {
      sg.agg_args.a = cur_args;
      sg.agg_args.norms_out = norms_dst;
      sg.agg_args.clipped_out = agg_cnt;
      set_node(sg.exec, sg.agg, &sg.agg_args);
    }
    if (sg.mlp && (sg.mlp_args.x != x_slot || sg.mlp_args.y != y_slot ||
                   (sg.mlp_args.noise && !same_args(sg.mlp_args.a, cur_args)))) {
      sg.mlp_args.x = x_slot;
      sg.mlp_args.y = y_slot;
      if (sg.mlp_args.noise) sg.mlp_args.a = cur_args;
      set_node(sg.exec, sg.mlp, &sg.mlp_args);
    }
    if (sg.emb && !same_args(sg.emb_args.a, cur_args)) {
      sg.emb_args.a = cur_args;
      set_node(sg.exec, sg.emb, &sg.emb_args);
    }
    // (a noise node without a count copy -- the ghost blocks' update -- keeps none)
    if (sg.noise && (!same_args(sg.noise_args.a, cur_args) ||
                     (sg.noise_args.clipped_out && sg.noise_args.clipped_out != clipped_dst))) {
      sg.noise_args.a = cur_args;
      if (sg.noise_args.clipped_out) sg.noise_args.clipped_out = clipped_dst;
      set_node(sg.exec, sg.noise, &sg.noise_args);
    }
    if (sg.scales && (!same_args(sg.scales_args.a, cur_args) || sg.scales_args.norms != norms_dst)) {
      sg.scales_args.a = cur_args;
      sg.scales_args.norms = norms_dst;
      set_node(sg.exec, sg.scales, &sg.scales_args);
    }
    const bool agg_in = sg.fused_tc && sg.fused_args.agg_tiles > 0;
    if (sg.fused && (sg.fused_args.x != x_slot || sg.fused_args.y != y_slot ||
                     sg.fused_args.norms != norms_dst || !same_args(sg.fused_args.a, cur_args) ||
                     (agg_in && (sg.fused_agg.norms_out != norms_dst ||
                                 sg.fused_agg.clipped_out != clipped_dst)))) {
      sg.fused_args.x = x_slot;
      sg.fused_args.y = y_slot;
      sg.fused_args.norms = norms_dst;
      sg.fused_args.a = cur_args;
      if (agg_in) {
        sg.fused_agg.a = cur_args;
        sg.fused_agg.norms_out = norms_dst;
        sg.fused_agg.clipped_out = clipped_dst;
      }
      set_node(sg.exec, sg.fused, &sg.fused_args, sg.fused_tc ? &sg.fused_agg : nullptr);
    }
  }

  // Device errors are sticky (the reference's first one wins and later
  // updates are skipped) until the host reports them here, with the
  // reference's IndexError text (checked_id, kernels.hpp:475-489).
  void check_device_error() {
    if (h_err->code == 0) return;
    const DevError e = *h_err;
    h_err->code = 0;
    PGB_CUDA(cudaMemsetAsync(d_err, 0, sizeof(DevError), stream));
    PGB_CUDA(cudaStreamSynchronize(stream));
    const unsigned long long key = ~e.inv_key;
    const bool label = (key >> 62) & 1;
    const long long pos = (long long)((key >> 32) & ((1ull << 30) - 1));
    const uint32_t bits = (uint32_t)key;
    float v;
    std::memcpy(&v, &bits, sizeof v);
    const std::string what = label ? "softmax_xent label" : "gather_rows";
    const double dv = v;
    const long long id = std::isfinite(dv) ? std::llround(dv) : 0;
    if (!std::isfinite(dv) || (double)id != dv)
      raise(PGB_ERR_INDEX, what + ": non-integral id at position " + std::to_string(pos));
    raise(PGB_ERR_INDEX, what + ": id " + std::to_string(id) + " out of range [0," +
                             std::to_string(label ? e.limit_label : e.limit_id) +
                             ") at position " + std::to_string(pos));
  }

  void read_report(float* norms_out, pgb_step_report* rep, int64_t m, int64_t step) {
    const int U = (int)(B / m);
    PGB_CUDA(cudaMemcpyAsync(h_err, d_err, sizeof(DevError), cudaMemcpyDeviceToHost, stream));
    PGB_CUDA(cudaMemcpyAsync(h_clipped, d_clipped, sizeof(int) * 2, cudaMemcpyDeviceToHost,
                             stream));
    if (norms_out)
      PGB_CUDA(cudaMemcpyAsync(h_norms, d_norms, sizeof(float) * U, cudaMemcpyDeviceToHost,
                               stream));
    PGB_CUDA(cudaStreamSynchronize(stream));
    check_device_error();
    if (norms_out) std::memcpy(norms_out, h_norms, sizeof(float) * U);
    if (rep) {
      rep->clipped_count = dist ? h_clipped[1] : h_clipped[0];
      rep->n_streams = 0;
      if (last_cfg.noise_multiplier > 0.0f) {
        rep->n_streams = bt.n;
        for (int p = 0; p < bt.n; ++p) rep->noise_streams[p] = noise_stream(step, p);
      }
    }
  }

  void step_host(const float* x, const float* y, const pgb_dp_config& c, int64_t step,
                 float* norms_out, pgb_step_report* rep) {
    validate_step(c);
    if (!x || !y) raise(PGB_ERR_CONTRACT, "null input");
    PGB_CUDA(cudaMemcpyAsync(d_x, x, sizeof(float) * B * in_row, cudaMemcpyHostToDevice,
                             stream));
    PGB_CUDA(cudaMemcpyAsync(d_y, y, sizeof(float) * B, cudaMemcpyHostToDevice, stream));
    push_args(make_args(c, step, d_x, d_y));
    last_cfg = c;
    last_step = step;
    launch_step(d_x, d_y, c.microbatch);
    read_report(norms_out, rep, c.microbatch, step);
  }
};

}  // namespace pgb

using namespace pgb;

struct pgb_engine {
  std::unique_ptr<Engine> impl;
};

namespace {
Engine& E(pgb_engine* e) {
  if (!e || !e->impl) raise(PGB_ERR_CONTRACT, "null engine handle");
  PGB_CUDA(cudaSetDevice(e->impl->device));
  return *e->impl;
}
}  // namespace

extern "C" {

pgb_status pgb_engine_create(const pgb_model_desc* desc, int32_t strategy, int64_t batch,
                             int32_t device, pgb_engine** out) {
  return guarded([&] {
    if (!desc || !out) raise(PGB_ERR_CONTRACT, "null argument");
    auto h = std::make_unique<pgb_engine>();
    h->impl = std::make_unique<Engine>();
    h->impl->init(*desc, strategy, batch, device);
    *out = h.release();
  });
}

pgb_status pgb_nccl_unique_id(pgb_unique_id* out) {
  return guarded([&] {
    static_assert(sizeof(pgb_unique_id) == sizeof(ncclUniqueId), "unique id size");
    ncclUniqueId id;
    PGB_NCCL(Nccl::get().getUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
  });
}

pgb_status pgb_engine_create_dist(const pgb_model_desc* desc, int32_t strategy,
                                  int64_t local_batch, int32_t device, int32_t rank,
                                  int32_t world, const pgb_unique_id* id, pgb_engine** out) {
  return guarded([&] {
    if (!desc || !out || !id) raise(PGB_ERR_CONTRACT, "null argument");
    if (world < 1 || rank < 0 || rank >= world) raise(PGB_ERR_CONFIG, "bad rank/world");
    auto h = std::make_unique<pgb_engine>();
    h->impl = std::make_unique<Engine>();
    h->impl->world = world;
    h->impl->rank = rank;
    h->impl->dist = world > 1 || std::getenv("PGB_FORCE_DIST") != nullptr;
    h->impl->init(*desc, strategy, local_batch, device);
    if (h->impl->dist) {
      ncclUniqueId nid;
      std::memcpy(&nid, id, sizeof nid);
      PGB_NCCL(Nccl::get().commInitRank(&h->impl->comm, world, nid, rank));
    }
    *out = h.release();
  });
}

void pgb_engine_destroy(pgb_engine* e) {
  if (!e) return;
  try {
    delete e;
  } catch (...) {
  }
}

pgb_status pgb_engine_info_get(pgb_engine* e, pgb_engine_info* out) {
  return guarded([&] {
    Engine& en = E(e);
    out->batch = en.B;
    out->global_batch = en.B * en.world;
    out->param_count = en.P;
    out->n_params = en.bt.n;
    out->world = en.world;
    out->rank = en.rank;
    out->device = en.device;
    out->workspace_bytes = (int64_t)en.arena_bytes;
    out->kernels_per_step = en.kernels_last;
    out->graph_enabled = en.graph_enabled;
  });
}

pgb_status pgb_engine_set_graph(pgb_engine* e, int32_t enable) {
  return guarded([&] { E(e).graph_enabled = enable != 0; });
}

pgb_status pgb_set_params(pgb_engine* e, const float* flat) {
  return guarded([&] {
    Engine& en = E(e);
    PGB_CUDA(cudaMemcpyAsync(en.d_params, flat, sizeof(float) * en.P, cudaMemcpyHostToDevice,
                             en.stream));
    en.refresh_shadows(en.stream);
    PGB_CUDA(cudaStreamSynchronize(en.stream));
  });
}

pgb_status pgb_get_params(pgb_engine* e, float* flat) {
  return guarded([&] {
    Engine& en = E(e);
    PGB_CUDA(cudaMemcpyAsync(flat, en.d_params, sizeof(float) * en.P, cudaMemcpyDeviceToHost,
                             en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
  });
}

pgb_status pgb_dpsgd_step(pgb_engine* e, const float* x, const float* y,
                          const pgb_dp_config* cfg, int64_t step, float* norms_out,
                          pgb_step_report* rep) {
  return guarded([&] {
    if (!cfg) raise(PGB_ERR_CONTRACT, "null config");
    E(e).step_host(x, y, *cfg, step, norms_out, rep);
  });
}

pgb_status pgb_dpsgd_step_device(pgb_engine* e, const float* d_x, const float* d_y,
                                 const pgb_dp_config* cfg, int64_t step) {
  return guarded([&] {
    Engine& en = E(e);
    if (!cfg) raise(PGB_ERR_CONTRACT, "null config");
    en.validate_step(*cfg);
    if (!d_x || !d_y) raise(PGB_ERR_CONTRACT, "null input");
    en.push_args(en.make_args(*cfg, step, en.d_x, en.d_y));
    en.last_cfg = *cfg;
    en.last_step = step;
    if ((en.fused_mnist || en.mlp_fused) && en.graph_enabled) {
      // read in place: the graph's fused-kernel node is pointed at the batch
      en.launch_step(d_x, d_y, cfg->microbatch);
    } else {
      PGB_CUDA(cudaMemcpyAsync(en.d_x, d_x, sizeof(float) * en.B * en.in_row,
                               cudaMemcpyDeviceToDevice, en.stream));
      PGB_CUDA(cudaMemcpyAsync(en.d_y, d_y, sizeof(float) * en.B, cudaMemcpyDeviceToDevice,
                               en.stream));
      en.launch_step(en.d_x, en.d_y, cfg->microbatch);
    }
  });
}

namespace {
// How pgb_run_steps_device splits n_steps: full multi-step graphs of C steps
// plus one graph of the remainder (every schedule whose inputs the graph can
// read from the device ring by the step counter: fused MNIST and dense-only
// models, one process or data-parallel, microbatch 1); C = 0: per-step graphs.
int64_t resident_chunk(const Engine& en, const pgb_dp_config& cfg, int64_t n_batches,
                       int64_t n_steps) {
  // a run of up to 64 steps is one graph (one launch); longer runs replay
  // graphs of 8 steps (measured: host issue under 0.2 us per step)
  int64_t C = n_steps >= 2 && n_steps <= 64 ? n_steps : 8;
  if (const char* cs = std::getenv("PGB_CHUNK_STEPS")) C = std::max<int64_t>(1, std::atoll(cs));
  const bool ok = (en.fused_mnist || en.mlp_fused) && cfg.microbatch == 1 && en.graph_enabled &&
                  C > 1 && n_batches < (1 << 30);
  return ok ? C : 0;
}
}  // namespace

pgb_status pgb_prepare_steps(pgb_engine* e, const float* d_x, const float* d_y,
                             int64_t n_batches, int64_t n_steps, const pgb_dp_config* cfg) {
  return guarded([&] {
    Engine& en = E(e);
    if (!cfg || !d_x || !d_y) raise(PGB_ERR_CONTRACT, "null argument");
    if (n_batches <= 0 || n_steps < 0) raise(PGB_ERR_CONFIG, "prepare_steps: bad counts");
    en.validate_step(*cfg);
    const int64_t C = resident_chunk(en, *cfg, n_batches, n_steps);
    if (C == 0) return;
    const StepArgs a0 = en.make_args(*cfg, 0, nullptr, nullptr);
    // captured, instantiated and uploaded to the device (the first launch
    // of a graph otherwise pays its upload)
    if (n_steps >= C)
      PGB_CUDA(cudaGraphUpload(en.resident_graph(C, a0, d_x, d_y, (int)n_batches), en.stream));
    if (n_steps % C)
      PGB_CUDA(cudaGraphUpload(en.resident_graph(n_steps % C, a0, d_x, d_y, (int)n_batches),
                               en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
  });
}

pgb_status pgb_run_steps_device(pgb_engine* e, const float* d_x, const float* d_y,
                                int64_t n_batches, int64_t n_steps, const pgb_dp_config* cfg,
                                int64_t step0, int64_t* launches_out) {
  return guarded([&] {
    Engine& en = E(e);
    if (!cfg || !d_x || !d_y) raise(PGB_ERR_CONTRACT, "null argument");
    if (n_batches <= 0 || n_steps < 0) raise(PGB_ERR_CONFIG, "run_steps_device: bad counts");
    en.validate_step(*cfg);
    en.last_cfg = *cfg;
    int64_t launches = 0;
    auto batch = [&](int64_t s) {
      const int64_t bi = ((s % n_batches) + n_batches) % n_batches;
      return std::make_pair(d_x + bi * en.B * en.in_row, d_y + bi * en.B);
    };
    const int64_t C = resident_chunk(en, *cfg, n_batches, n_steps);
    if (C > 0 && n_steps > 0) {
      // full chunks, then the remainder as one more static graph: the host
      // issues one counter write and ceil(n / C) graph launches
      const StepArgs a0 = en.make_args(*cfg, step0, nullptr, nullptr);
      const int64_t full = n_steps / C, rem = n_steps % C;
      cudaGraphExec_t g = full ? en.resident_graph(C, a0, d_x, d_y, (int)n_batches) : nullptr;
      const int kfull = en.kernels_last;
      cudaGraphExec_t gr = rem ? en.resident_graph(rem, a0, d_x, d_y, (int)n_batches) : nullptr;
      const int krem = en.kernels_last;
      set_counter_kernel<<<1, 1, 0, en.stream>>>(en.d_step_base + Engine::kSlots, step0);
      ++launches;
      for (int64_t k = 0; k < full; ++k) {
        PGB_CUDA(cudaGraphLaunch(g, en.stream));
        launches += C * kfull + 1;
      }
      if (gr) {
        PGB_CUDA(cudaGraphLaunch(gr, en.stream));
        launches += rem * krem + 1;
      }
    } else {
      for (int64_t s = 0; s < n_steps; ++s) {
        const auto in = batch(step0 + s);
        en.push_args(en.make_args(*cfg, step0 + s, in.first, in.second));
        if ((en.fused_mnist || en.mlp_fused) && en.graph_enabled) {
          en.launch_step(in.first, in.second, cfg->microbatch);
        } else {
          PGB_CUDA(cudaMemcpyAsync(en.d_x, in.first, sizeof(float) * en.B * en.in_row,
                                   cudaMemcpyDeviceToDevice, en.stream));
          PGB_CUDA(cudaMemcpyAsync(en.d_y, in.second, sizeof(float) * en.B,
                                   cudaMemcpyDeviceToDevice, en.stream));
          en.launch_step(en.d_x, en.d_y, cfg->microbatch);
        }
        launches += en.kernels_last;
      }
    }
    en.last_step = step0 + n_steps - 1;
    PGB_CUDA(cudaGetLastError());
    if (launches_out) *launches_out = launches;
  });
}

pgb_status pgb_synchronize(pgb_engine* e, float* norms_out, pgb_step_report* rep) {
  return guarded([&] {
    Engine& en = E(e);
    en.read_report(norms_out, rep, en.last_cfg.microbatch > 0 ? en.last_cfg.microbatch : 1,
                   en.last_step);
  });
}

pgb_status pgb_sgd_step(pgb_engine* e, const float* x, const float* y, float lr) {
  return guarded([&] {
    Engine& en = E(e);
    PGB_CUDA(cudaMemcpyAsync(en.d_x, x, sizeof(float) * en.B * en.in_row,
                             cudaMemcpyHostToDevice, en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.d_y, y, sizeof(float) * en.B, cudaMemcpyHostToDevice,
                             en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_err, 0, sizeof(DevError), en.stream));
    en.enqueue_grads(en.stream, en.d_x, en.d_y);
    sgd_kernel<<<grid_for((size_t)en.P), 256, 0, en.stream>>>(en.table_for(en.d_x), (int)en.B,
                                                              lr, en.d_params);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaMemcpyAsync(en.h_err, en.d_err, sizeof(DevError), cudaMemcpyDeviceToHost,
                             en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
    en.check_device_error();
  });
}

pgb_status pgb_per_example_grads(pgb_engine* e, const float* x, const float* y,
                                 float* stacks_out, float* norms_out) {
  return guarded([&] {
    Engine& en = E(e);
    PGB_CUDA(cudaMemcpyAsync(en.d_x, x, sizeof(float) * en.B * en.in_row,
                             cudaMemcpyHostToDevice, en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.d_y, y, sizeof(float) * en.B, cudaMemcpyHostToDevice,
                             en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_err, 0, sizeof(DevError), en.stream));
    en.enqueue_grads(en.stream, en.d_x, en.d_y);
    finalize_norms_kernel<<<((int)en.B + 127) / 128, 128, 0, en.stream>>>(
        en.d_parts, en.nparts, (int)en.B, en.d_norms);
    if (stacks_out)
      materialize_kernel<<<grid_for((size_t)en.P * en.B), 256, 0, en.stream>>>(
          en.table_for(en.d_x), (int)en.B, en.d_stacks);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaMemcpyAsync(en.h_err, en.d_err, sizeof(DevError), cudaMemcpyDeviceToHost,
                             en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
    en.check_device_error();
    if (stacks_out)
      PGB_CUDA(cudaMemcpy(stacks_out, en.d_stacks, sizeof(float) * en.B * en.P,
                          cudaMemcpyDeviceToHost));
    if (norms_out)
      PGB_CUDA(cudaMemcpy(norms_out, en.d_norms, sizeof(float) * en.B, cudaMemcpyDeviceToHost));
  });
}

pgb_status pgb_clipped_sum(pgb_engine* e, const float* x, const float* y, float clip_norm,
                           float* sum_out, float* norms_out, int64_t* clipped_out) {
  return guarded([&] {
    Engine& en = E(e);
    if (!(clip_norm > 0.0f)) raise(PGB_ERR_CONFIG, "DpConfig: clip norm must be positive");
    PGB_CUDA(cudaMemcpyAsync(en.d_x, x, sizeof(float) * en.B * en.in_row,
                             cudaMemcpyHostToDevice, en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.d_y, y, sizeof(float) * en.B, cudaMemcpyHostToDevice,
                             en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_err, 0, sizeof(DevError), en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_clipped, 0, sizeof(int) * 2, en.stream));
    pgb_dp_config c{clip_norm, 0.0f, 1.0f, 1, 0};
    en.push_args(en.make_args(c, 0, en.d_x, en.d_y));
    en.enqueue_grads(en.stream, en.d_x, en.d_y);
    en.enqueue_local_sum(en.stream, en.table_for(en.d_x), en.nparts, (int)en.B);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaMemcpyAsync(en.h_err, en.d_err, sizeof(DevError), cudaMemcpyDeviceToHost,
                             en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
    en.check_device_error();
    if (sum_out)
      PGB_CUDA(cudaMemcpy(sum_out, en.d_sum, sizeof(float) * en.P, cudaMemcpyDeviceToHost));
    if (norms_out)
      PGB_CUDA(cudaMemcpy(norms_out, en.d_norms, sizeof(float) * en.B, cudaMemcpyDeviceToHost));
    if (clipped_out) {
      int c0 = 0;
      PGB_CUDA(cudaMemcpy(&c0, en.d_clipped, sizeof(int), cudaMemcpyDeviceToHost));
      *clipped_out = c0;
    }
  });
}

pgb_status pgb_weighted_grad_sum(pgb_engine* e, const float* x, const float* y, const float* w,
                                 float* sum_out) {
  return guarded([&] {
    Engine& en = E(e);
    if (!x || !y || !w || !sum_out) raise(PGB_ERR_CONTRACT, "null argument");
    if (en.dist)
      raise(PGB_ERR_UNSUPPORTED, "weighted_grad_sum: one-process engines only");
    PGB_CUDA(cudaMemcpyAsync(en.d_x, x, sizeof(float) * en.B * en.in_row,
                             cudaMemcpyHostToDevice, en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.d_y, y, sizeof(float) * en.B, cudaMemcpyHostToDevice,
                             en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.d_wts, w, sizeof(float) * en.B, cudaMemcpyHostToDevice,
                             en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_err, 0, sizeof(DevError), en.stream));
    pgb_dp_config c{1.0f, 0.0f, 1.0f, 1, 0};
    en.push_args(en.make_args(c, 0, en.d_x, en.d_y));
    en.enqueue_weighted_sum(en.stream, en.d_x, en.d_y, en.d_wts);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaMemcpyAsync(en.h_err, en.d_err, sizeof(DevError), cudaMemcpyDeviceToHost,
                             en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
    en.check_device_error();
    PGB_CUDA(cudaMemcpy(sum_out, en.d_sum, sizeof(float) * en.P, cudaMemcpyDeviceToHost));
  });
}

pgb_status pgb_batch_grad_sum(pgb_engine* e, const float* x, const float* y, float* sum_out) {
  return guarded([&] {
    Engine& en = E(e);
    std::vector<float> ones((size_t)en.B, 1.0f);
    const pgb_status st = pgb_weighted_grad_sum(e, x, y, ones.data(), sum_out);
    if (st != PGB_OK) raise(st, pgb_last_error());
  });
}

pgb_status pgb_forward(pgb_engine* e, const float* x, const float* y, float* losses_out,
                       float* logits_out) {
  return guarded([&] {
    Engine& en = E(e);
    PGB_CUDA(cudaMemcpyAsync(en.d_x, x, sizeof(float) * en.B * en.in_row,
                             cudaMemcpyHostToDevice, en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.d_y, y, sizeof(float) * en.B, cudaMemcpyHostToDevice,
                             en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_err, 0, sizeof(DevError), en.stream));
    en.enqueue_forward(en.stream, en.d_x, en.d_y);
    PGB_CUDA(cudaGetLastError());
    if (losses_out)
      PGB_CUDA(cudaMemcpyAsync(losses_out, en.d_loss, sizeof(float) * en.B,
                               cudaMemcpyDeviceToHost, en.stream));
    if (logits_out)
      PGB_CUDA(cudaMemcpyAsync(logits_out, en.logits_buffer(),
                               sizeof(float) * en.B * en.desc.classes, cudaMemcpyDeviceToHost,
                               en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.h_err, en.d_err, sizeof(DevError), cudaMemcpyDeviceToHost,
                             en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
    en.check_device_error();
  });
}

pgb_status pgb_aggregate(pgb_engine* e, const float* stacks, const pgb_dp_config* cfg,
                         int64_t step, float* norms_out, pgb_step_report* rep) {
  return guarded([&] {
    Engine& en = E(e);
    if (!cfg || !stacks) raise(PGB_ERR_CONTRACT, "null argument");
    validate_dp_config(*cfg, en.B);
    if (cfg->microbatch != 1) raise(PGB_ERR_CONFIG, "pgb_aggregate: microbatch must be 1");
    PGB_CUDA(cudaMemcpyAsync(en.d_stacks, stacks, sizeof(float) * en.B * en.P,
                             cudaMemcpyHostToDevice, en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_err, 0, sizeof(DevError), en.stream));
    PGB_CUDA(cudaMemsetAsync(en.d_clipped, 0, sizeof(int) * 2, en.stream));
    en.push_args(en.make_args(*cfg, step, en.d_x, en.d_y));
    en.last_cfg = *cfg;
    dim3 sg(en.bt_stack.n, (unsigned)en.B);
    sumsq_kernel<<<sg, 128, 0, en.stream>>>(en.bt_stack, (int)en.B, en.d_parts);
    en.enqueue_aggregate(en.stream, en.bt_stack, en.bt_stack.n, (int)en.B);
    PGB_CUDA(cudaGetLastError());
    en.read_report(norms_out, rep, 1, step);
  });
}

pgb_status pgb_gaussian(int32_t device, uint64_t seed, uint64_t stream, int64_t n, float* out) {
  return guarded([&] {
    if (n <= 0) return;
    PGB_CUDA(cudaSetDevice(device));
    float* d = nullptr;
    PGB_CUDA(cudaMalloc(&d, sizeof(float) * n));
    gaussian_kernel<<<grid_for((size_t)(n + 1) / 2), 256>>>(stream_key(seed, stream), n, d);
    cudaError_t st = cudaMemcpy(out, d, sizeof(float) * n, cudaMemcpyDeviceToHost);
    cudaFree(d);
    PGB_CUDA(st);
  });
}

pgb_status pgb_run_epoch(pgb_engine* e, const float* x, const float* y, int64_t n,
                         const pgb_dp_config* cfg, int64_t step0, float* norms_out,
                         int64_t* clipped_total, double* seconds_out) {
  return guarded([&] {
    Engine& en = E(e);
    if (!cfg || !x || !y) raise(PGB_ERR_CONTRACT, "null argument");
    en.validate_step(*cfg);
    const int64_t steps = n / en.B;
    if (steps <= 0) raise(PGB_ERR_CONFIG, "run_epoch: fewer examples than one batch");
    const int64_t U = en.B / cfg->microbatch;
    const size_t xb = sizeof(float) * en.B * en.in_row, yb = sizeof(float) * en.B;
    constexpr int K = Engine::kSlots;
    // Results go to a ring of K device slots read back on out_stream, so the
    // per-step D2H never sits between two steps on the compute stream (the
    // data-parallel schedule all-reduces each step's clip count inside its
    // own result slot).
    const bool ring = true;
    en.ensure_host_stage(steps, U);
    cudaEvent_t* copied = en.ev_copied;
    cudaEvent_t* consumed = en.ev_consumed;
    cudaEvent_t* done = en.ev_done;
    cudaEvent_t* read = en.ev_read;
    const auto wall0 = std::chrono::steady_clock::now();
    PGB_CUDA(cudaEventRecord(en.ev_t0, en.stream));
    // Inputs arrive in chunks of C steps (one pinned H2D copy per chunk) into
    // a ring of K device chunks. The fused MNIST step takes
    // its input pointers as graph-node parameters, so any offset inside a
    // chunk works; the layer-wise schedule bakes its input slot into the
    // graph and keeps one batch per chunk.
    // Fused MNIST on one GPU: static graphs of C steps per input chunk (one
    // H2D copy of C batches, one graph launch, one read-back of C steps'
    // results), so the host issues ~10 calls per C steps instead of ~10 per
    // step. PGB_CHUNK_STEPS overrides C (1 = the per-step path below).
    int64_t C = 8;  // 4-8 measured best (scripts/e2e_probe.py)
    if (const char* cs = std::getenv("PGB_CHUNK_STEPS")) C = std::max<int64_t>(1, std::atoll(cs));
    // result slots: K chunk slots of C, then the head / remainder slots
    C = std::min<int64_t>(C, Engine::kResSlots / (K + 1));
    // (every one-process schedule: the layer-wise one bakes each step's input
    // pointer into its chunk graph node; noise takes the step from the device)
    const bool chunked = cfg->microbatch == 1 && en.graph_enabled && C > 1 && steps >= C;
    // the fused schedules take input pointers as node parameters: their
    // per-step graphs can read any batch inside a chunk slot; the layer-wise
    // schedule launches those steps directly
    const bool ptr_params = en.fused_mnist || en.mlp_fused;
    if (!chunked) C = 1;
    if (C > 1) en.ensure_chunk_ring(C);
    const int64_t nchunks = (steps + C - 1) / C, nfull = steps / C;
    auto xslot = [&](int sl) { return C > 1 ? en.d_xc[sl] : en.d_xb[sl]; };
    auto yslot = [&](int sl) { return C > 1 ? en.d_yc[sl] : en.d_yb[sl]; };
    auto copy_in = [&](int64_t k) {
      const int sl = (int)(k % K);
      const int64_t cnt = std::min<int64_t>(C, steps - k * C);
      if (k >= K) PGB_CUDA(cudaStreamWaitEvent(en.copy_stream, consumed[sl], 0));
      else PGB_CUDA(cudaStreamWaitEvent(en.copy_stream, en.ev_t0, 0));
      PGB_CUDA(cudaMemcpyAsync(xslot(sl), x + k * C * en.B * en.in_row, xb * cnt,
                               cudaMemcpyHostToDevice, en.copy_stream));
      PGB_CUDA(cudaMemcpyAsync(yslot(sl), y + k * C * en.B, yb * cnt, cudaMemcpyHostToDevice,
                               en.copy_stream));
      if (chunked) {
        en.h_step_base[k] = step0 + k * C;
        PGB_CUDA(cudaMemcpyAsync(en.d_step_base + sl, en.h_step_base + k, sizeof(long long),
                                 cudaMemcpyHostToDevice, en.copy_stream));
      }
      PGB_CUDA(cudaEventRecord(copied[sl], en.copy_stream));
    };
    constexpr int KR = Engine::kResSlots;
    // One step through the per-step graph path: result slot rs_sl, reading
    // batch j of chunk slot sl (the caller made the batch's copy visible).
    auto step_once = [&](int64_t s, int sl, int64_t j, int rs_sl, bool wait_read) {
      if (ring) {
        // result slot rs_sl's previous results must have been read back
        if (wait_read) PGB_CUDA(cudaStreamWaitEvent(en.stream, read[rs_sl], 0));
        en.norms_dst = en.d_norms_ring + (size_t)rs_sl * en.B;
        en.clipped_dst = en.d_clip_ring + 2 * rs_sl;
      }
      const float* xs = xslot(sl) + j * en.B * en.in_row;
      const float* ys = yslot(sl) + j * en.B;
      en.push_args(en.make_args(*cfg, step0 + s, xs, ys));
      if (C > 1 && !ptr_params) {
        en.kernels_last = en.enqueue_step(en.stream, xs, ys, cfg->microbatch);
        PGB_CUDA(cudaGetLastError());
      } else {
        en.launch_step(xs, ys, cfg->microbatch);
      }
      // the step's result read back every step (norms, clipped count)
      cudaStream_t rs = ring ? en.out_stream : en.stream;
      if (ring) {
        PGB_CUDA(cudaEventRecord(done[rs_sl], en.stream));
        PGB_CUDA(cudaStreamWaitEvent(rs, done[rs_sl], 0));
      }
      PGB_CUDA(cudaMemcpyAsync(en.h_clip_stage + 2 * s, en.clipped_dst, sizeof(int) * 2,
                               cudaMemcpyDeviceToHost, rs));
      if (norms_out)
        PGB_CUDA(cudaMemcpyAsync(en.h_norm_stage + s * U, en.norms_dst, sizeof(float) * U,
                                 cudaMemcpyDeviceToHost, rs));
      if (ring) PGB_CUDA(cudaEventRecord(read[rs_sl], rs));
    };
    int64_t k_first = 0;
    if (chunked) {
      // head: chunk 0 as per-batch copies, its steps on the per-step path,
      // each waiting for its own batch (result slots K*C ..)
      PGB_CUDA(cudaStreamWaitEvent(en.copy_stream, en.ev_t0, 0));
      for (int64_t j = 0; j < C; ++j) {
        PGB_CUDA(cudaMemcpyAsync(xslot(0) + j * en.B * en.in_row, x + j * en.B * en.in_row, xb,
                                 cudaMemcpyHostToDevice, en.copy_stream));
        PGB_CUDA(cudaMemcpyAsync(yslot(0) + j * en.B, y + j * en.B, yb, cudaMemcpyHostToDevice,
                                 en.copy_stream));
        PGB_CUDA(cudaEventRecord(en.ev_head[j], en.copy_stream));
      }
      for (int64_t k = 1; k < std::min<int64_t>(K - 1, nchunks); ++k) copy_in(k);
      if (K - 1 < nchunks) copy_in(K - 1);
      for (int64_t j = 0; j < C; ++j) {
        PGB_CUDA(cudaStreamWaitEvent(en.stream, en.ev_head[j], 0));
        step_once(j, 0, j, (int)(K * C + j), false);
      }
      PGB_CUDA(cudaEventRecord(consumed[0], en.stream));
      k_first = 1;
    } else {
      for (int64_t k = 0; k < std::min<int64_t>(K - 1, nchunks); ++k) copy_in(k);
    }
    const StepArgs args0 = en.make_args(*cfg, step0, nullptr, nullptr);
    for (int64_t k = k_first; chunked && k < nfull; ++k) {
      const int sl = (int)(k % K);
      if (k + K - 1 < nchunks && k > 0) copy_in(k + K - 1);
      PGB_CUDA(cudaStreamWaitEvent(en.stream, copied[sl], 0));
      // result slots sl*C .. sl*C+C-1 of chunk k-K must have been read back
      if (k >= K) PGB_CUDA(cudaStreamWaitEvent(en.stream, read[sl], 0));
      PGB_CUDA(cudaGraphLaunch(en.chunk_graph(sl, C, args0), en.stream));
      PGB_CUDA(cudaEventRecord(consumed[sl], en.stream));
      PGB_CUDA(cudaEventRecord(done[sl], en.stream));
      PGB_CUDA(cudaStreamWaitEvent(en.out_stream, done[sl], 0));
      PGB_CUDA(cudaMemcpyAsync(en.h_clip_stage + 2 * k * C, en.d_clip_ring + 2 * sl * C,
                               sizeof(int) * 2 * C, cudaMemcpyDeviceToHost, en.out_stream));
      if (norms_out)
        PGB_CUDA(cudaMemcpyAsync(en.h_norm_stage + k * C * U, en.d_norms_ring + sl * C * en.B,
                                 sizeof(float) * C * U, cudaMemcpyDeviceToHost, en.out_stream));
      PGB_CUDA(cudaEventRecord(read[sl], en.out_stream));
    }
    // per-step path: every step of a non-chunked epoch, or the remainder of a
    // chunked one (result slots from K*C on, clear of the chunk slots; waiting
    // on a slot's read event also covers the head's use of it)
    const int64_t s_begin = chunked ? nfull * C : 0;
    for (int64_t s = s_begin; s < steps; ++s) {
      const int64_t k = s / C, j = s % C;
      const int sl = (int)(k % K);
      const int rs_sl = chunked ? (int)(K * C + (s - s_begin) % (KR - K * C)) : (int)(s % KR);
      if (j == 0) {
        if (!chunked && k + K - 1 < nchunks) copy_in(k + K - 1);
        PGB_CUDA(cudaStreamWaitEvent(en.stream, copied[sl], 0));
      }
      step_once(s, sl, j, rs_sl, chunked || s >= KR);
      if (j == C - 1 || s == steps - 1) PGB_CUDA(cudaEventRecord(consumed[sl], en.stream));
    }
    en.norms_dst = en.d_norms;
    en.clipped_dst = en.d_clipped;
    if (ring) {
      PGB_CUDA(cudaEventRecord(en.ev_t1, en.out_stream));
      PGB_CUDA(cudaStreamWaitEvent(en.stream, en.ev_t1, 0));
    }
    PGB_CUDA(cudaMemcpyAsync(en.h_err, en.d_err, sizeof(DevError), cudaMemcpyDeviceToHost,
                             en.stream));
    PGB_CUDA(cudaEventRecord(en.ev_t1, en.stream));
    PGB_CUDA(cudaEventSynchronize(en.ev_t1));
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    float ms = 0;
    cudaEventElapsedTime(&ms, en.ev_t0, en.ev_t1);
    if (seconds_out) *seconds_out = std::max(wall, ms * 1e-3);
    int64_t tot = 0;
    for (int64_t s = 0; s < steps; ++s)
      tot += en.dist ? en.h_clip_stage[2 * s + 1] : en.h_clip_stage[2 * s];
    if (clipped_total) *clipped_total = tot;
    if (norms_out) std::memcpy(norms_out, en.h_norm_stage, sizeof(float) * steps * U);
    en.last_cfg = *cfg;
    en.last_step = step0 + steps - 1;
    en.check_device_error();
  });
}

#ifdef PGB_TRACE
// Tuning aid (trace builds only): arm the timestamp buffer (out == NULL) or
// copy it out.
pgb_status pgb_debug_trace(long long* out, int n) {
  return guarded([&] {
    static unsigned long long* buf = nullptr;
    if (!buf) {
      PGB_CUDA(cudaMalloc(&buf, 8 * PGB_TRACE_SLOTS));
      PGB_CUDA(cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf)));
    }
    PGB_CUDA(cudaDeviceSynchronize());
    if (!out) {
      PGB_CUDA(cudaMemset(buf, 0, 8 * PGB_TRACE_SLOTS));
      return;
    }
    PGB_CUDA(cudaMemcpy(out, buf, 8 * std::min(n, PGB_TRACE_SLOTS), cudaMemcpyDeviceToHost));
  });
}
#endif

pgb_status pgb_profile_steps(pgb_engine* e, const float* d_x, const float* d_y,
                             const pgb_dp_config* cfg, int64_t step0, int32_t n_steps,
                             int32_t max_kernels, float* ms_out, char* names_out,
                             int32_t* n_kernels_out) {
  return guarded([&] {
    Engine& en = E(e);
    if (!cfg) raise(PGB_ERR_CONTRACT, "null config");
    en.validate_step(*cfg);
    if (n_steps < 1 || n_steps > 32) raise(PGB_ERR_CONFIG, "profile: 1..32 steps");
    PGB_CUDA(cudaMemcpyAsync(en.d_x, d_x, sizeof(float) * en.B * en.in_row,
                             cudaMemcpyDeviceToDevice, en.stream));
    PGB_CUDA(cudaMemcpyAsync(en.d_y, d_y, sizeof(float) * en.B, cudaMemcpyDeviceToDevice,
                             en.stream));
    PGB_CUDA(cudaStreamSynchronize(en.stream));
    // hold the GPU while every instrumented launch is queued, so the events
    // bracket back-to-back kernels rather than host launch gaps
    spin_kernel<<<1, 1, 0, en.stream>>>(2000000LL + 400000LL * n_steps);
    std::vector<std::pair<cudaEvent_t, const char*>> marks;
    std::vector<size_t> step_begin;
    en.prof = &marks;
    try {
      for (int s = 0; s < n_steps; ++s) {
        en.push_args(en.make_args(*cfg, step0 + s, en.d_x, en.d_y));
        step_begin.push_back(marks.size());
        en.mark(en.stream, "begin");
        en.enqueue_step(en.stream, en.d_x, en.d_y, cfg->microbatch);
      }
    } catch (...) {
      en.prof = nullptr;
      throw;
    }
    en.prof = nullptr;
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaStreamSynchronize(en.stream));
    const size_t per = (step_begin.size() > 1 ? step_begin[1] : marks.size()) - 1;
    std::vector<double> acc(per, 0.0);
    for (size_t s = 0; s < step_begin.size(); ++s)
      for (size_t k = 0; k < per; ++k) {
        float ms = 0;
        PGB_CUDA(cudaEventElapsedTime(&ms, marks[step_begin[s] + k].first,
                                      marks[step_begin[s] + k + 1].first));
        acc[k] += ms;
      }
    const int nk = (int)std::min<size_t>(per, (size_t)max_kernels);
    for (int k = 0; k < nk; ++k) {
      if (ms_out) ms_out[k] = (float)(acc[k] / step_begin.size());
      if (names_out) {
        std::strncpy(names_out + 32 * k, marks[k + 1].second, 31);
        names_out[32 * k + 31] = 0;
      }
    }
    if (n_kernels_out) *n_kernels_out = nk;
    for (auto& m : marks) cudaEventDestroy(m.first);
  });
}

pgb_status pgb_debug_tc_gemm(int32_t device, int32_t M, int32_t N, int32_t K, const float* A,
                             const float* Bm, float* Cout) {
  return guarded([&] {
    PGB_CUDA(cudaSetDevice(device));
    float *dA = nullptr, *dB = nullptr, *dC = nullptr;
    PGB_CUDA(cudaMalloc(&dA, sizeof(float) * (size_t)M * K));
    PGB_CUDA(cudaMalloc(&dB, sizeof(float) * (size_t)N * K));
    PGB_CUDA(cudaMalloc(&dC, sizeof(float) * (size_t)M * N));
    PGB_CUDA(cudaMemcpy(dA, A, sizeof(float) * (size_t)M * K, cudaMemcpyHostToDevice));
    PGB_CUDA(cudaMemcpy(dB, Bm, sizeof(float) * (size_t)N * K, cudaMemcpyHostToDevice));
    tc::PlainOp op{M, N, K, dA, dB, dC};
    constexpr int BN = 64;
    const size_t smem = tc::tc_smem_bytes<tc::PlainOp, BN>();
    PGB_CUDA(cudaFuncSetAttribute(tc::tc_gemm_kernel<tc::PlainOp, BN, 128>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((N + BN - 1) / BN, (M + tc::kBM - 1) / tc::kBM, 1);
    tc::tc_gemm_kernel<tc::PlainOp, BN, 128><<<grid, 128, smem>>>(op);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaDeviceSynchronize());
    PGB_CUDA(cudaMemcpy(Cout, dC, sizeof(float) * (size_t)M * N, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
  });
}

pgb_status pgb_debug_tma_box(int32_t device, const float* src, int32_t width, int32_t height,
                             int32_t x0, int32_t y0, float* out) {
  return guarded([&] {
    PGB_CUDA(cudaSetDevice(device));
    float *d_src = nullptr, *d_out = nullptr;
    PGB_CUDA(cudaMalloc(&d_src, sizeof(float) * (size_t)width * height));
    PGB_CUDA(cudaMalloc(&d_out, sizeof(float) * 128));
    PGB_CUDA(cudaMemcpy(d_src, src, sizeof(float) * (size_t)width * height, cudaMemcpyHostToDevice));
    CUtensorMap m;
    const uint64_t dims[2] = {(uint64_t)width, (uint64_t)height};
    const uint64_t st[1] = {sizeof(float) * (uint64_t)width};
    const uint32_t box[2] = {32, 4};
    tg::make_map(&m, d_src, 2, dims, st, box);
    tg::tma_box_probe_kernel<<<1, 128>>>(m, x0, y0, d_out);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaDeviceSynchronize());
    PGB_CUDA(cudaMemcpy(out, d_out, sizeof(float) * 128, cudaMemcpyDeviceToHost));
    cudaFree(d_src);
    cudaFree(d_out);
  });
}

pgb_status pgb_debug_tma_gemm(int32_t device, int32_t M, int32_t N, int32_t K, const float* A,
                              const float* Bm, float* Cout) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || K % 4) raise(PGB_ERR_CONTRACT, "tma gemm: K % 4 == 0");
    PGB_CUDA(cudaSetDevice(device));
    float *dA = nullptr, *dB = nullptr, *dC = nullptr;
    PGB_CUDA(cudaMalloc(&dA, sizeof(float) * (size_t)M * K));
    PGB_CUDA(cudaMalloc(&dB, sizeof(float) * (size_t)N * K));
    PGB_CUDA(cudaMalloc(&dC, sizeof(float) * (size_t)M * N));
    PGB_CUDA(cudaMemcpy(dA, A, sizeof(float) * (size_t)M * K, cudaMemcpyHostToDevice));
    PGB_CUDA(cudaMemcpy(dB, Bm, sizeof(float) * (size_t)N * K, cudaMemcpyHostToDevice));
    float *dAl = nullptr, *dBl = nullptr;
    PGB_CUDA(cudaMalloc(&dAl, sizeof(float) * (size_t)M * K));
    PGB_CUDA(cudaMalloc(&dBl, sizeof(float) * (size_t)N * K));
    tg::split_kernel<<<grid_for((size_t)M * K), 256>>>(dA, dA, dAl, (long long)M * K);
    tg::split_kernel<<<grid_for((size_t)N * K), 256>>>(dB, dB, dBl, (long long)N * K);
    tg::Params p{};
    const int bn = tg::pick_bn(N);
    const uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, db[2] = {(uint64_t)K, (uint64_t)N};
    const uint64_t st[1] = {sizeof(float) * (uint64_t)K};
    const uint32_t ba[2] = {32, 128}, bb[2] = {32, (uint32_t)bn};
    tg::make_map(&p.ta, dA, 2, da, st, ba);
    tg::make_map(&p.tb, dB, 2, db, st, bb);
    tg::make_map(&p.ta_lo, dAl, 2, da, st, ba);
    tg::make_map(&p.tb_lo, dBl, 2, db, st, bb);
    p.mode = tg::kPlain;
    p.M = M;
    p.N = N;
    p.nchunks = (K + 31) / 32;
    p.out = dC;
    p.ldc = N;
    // PGB_DEBUG_KSPLIT=S: the K-split path (raw splits + ordered epilogue)
    const char* ks = std::getenv("PGB_DEBUG_KSPLIT");
    const int S = ks ? std::atoi(ks) : 1;
    const int ntn = (N + bn - 1) / bn, ntm = (M + 127) / 128;
    float* ws = nullptr;
    if (S > 1) {
      PGB_CUDA(cudaMalloc(&ws, sizeof(float) * (size_t)S * ntm * ntn * bn * 128));
      p.ksplit = S;
      p.ws = ws;
      tg::launch(p, bn, dim3(ntn, ntm, S), 0);
      tg::Params q = p;
      q.ntn = ntn;
      q.ntm = ntm;
      tg::splitk_epilogue_kernel<<<grid_for((size_t)ntm * ntn * bn * 32), 256>>>(q);
    } else {
      tg::launch(p, bn, dim3(ntn, ntm, 1), 0);
    }
    PGB_CUDA(cudaGetLastError());
    if (ws) {
      PGB_CUDA(cudaDeviceSynchronize());
      cudaFree(ws);
    }
    PGB_CUDA(cudaDeviceSynchronize());
    PGB_CUDA(cudaMemcpy(Cout, dC, sizeof(float) * (size_t)M * N, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    cudaFree(dAl);
    cudaFree(dBl);
  });
}

pgb_status pgb_debug_umma_probe(int32_t device, int32_t M, int32_t N, int32_t K, int32_t a_mn,
                                int32_t b_mn, const float* A, const float* Bm, float* Draw) {
  return guarded([&] {
    if (!(M == 64 || M == 128) || N < 8 || N > 256 || N % 8 || K < 8 || K > 32 || K % 8)
      raise(PGB_ERR_CONTRACT, "umma probe: M in {64,128}, N in [8,256] step 8, K in {8..32} step 8");
    PGB_CUDA(cudaSetDevice(device));
    float *dA = nullptr, *dB = nullptr, *dD = nullptr;
    PGB_CUDA(cudaMalloc(&dA, sizeof(float) * (size_t)M * K));
    PGB_CUDA(cudaMalloc(&dB, sizeof(float) * (size_t)N * K));
    PGB_CUDA(cudaMalloc(&dD, sizeof(float) * (size_t)128 * N));
    PGB_CUDA(cudaMemcpy(dA, A, sizeof(float) * (size_t)M * K, cudaMemcpyHostToDevice));
    PGB_CUDA(cudaMemcpy(dB, Bm, sizeof(float) * (size_t)N * K, cudaMemcpyHostToDevice));
    const int smem = (int)sizeof(float) * (128 * 32 + 256 * 32);
    PGB_CUDA(cudaFuncSetAttribute(tc::umma_probe_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc::umma_probe_kernel<<<1, 128, smem>>>(dA, dB, dD, M, N, K, a_mn, b_mn);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaDeviceSynchronize());
    PGB_CUDA(cudaMemcpy(Draw, dD, sizeof(float) * (size_t)128 * N, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  });
}

pgb_status pgb_debug_umma_rate(int32_t device, int32_t M, int32_t N, int32_t reps,
                               const uint32_t* strides, int32_t mode, int64_t* cycles) {
  return guarded([&] {
    PGB_CUDA(cudaSetDevice(device));
    long long* d = nullptr;
    PGB_CUDA(cudaMalloc(&d, sizeof(long long)));
    const int smem = 48 * 1024 * 4;
    PGB_CUDA(cudaFuncSetAttribute(tc::umma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
    tc::umma_rate_kernel<<<1, (mode & 8) ? 1024 : 128, smem>>>(M, N, reps, strides[0], strides[1], strides[2],
                                          strides[3], mode, d);
    PGB_CUDA(cudaGetLastError());
    PGB_CUDA(cudaDeviceSynchronize());
    PGB_CUDA(cudaMemcpy(cycles, d, sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(d);
  });
}

pgb_status pgb_load_idx_device(const char* path, int32_t device, float scale_div, float* d_out,
                               int64_t capacity) {
  return guarded([&] {
    if (!path || !d_out) raise(PGB_ERR_CONTRACT, "null argument");
    IdxArray a = read_idx(path);
    const size_t n = a.bytes.size() - a.offset;
    if (capacity < 0 || n > static_cast<size_t>(capacity))
      raise(PGB_ERR_CONTRACT, "load_idx: payload of " + std::to_string(n) +
                                  " elements exceeds the output capacity " +
                                  std::to_string(capacity));
    PGB_CUDA(cudaSetDevice(device));
    // the payload crosses PCIe as bytes (4x fewer than floats) and is decoded
    // on the device with the reference's arithmetic: float(b) / scale
    unsigned char* d_b = nullptr;
    PGB_CUDA(cudaMalloc(&d_b, n ? n : 1));
    cudaError_t st = cudaMemcpy(d_b, a.bytes.data() + a.offset, n, cudaMemcpyHostToDevice);
    if (st == cudaSuccess && n) {
      decode_u8_kernel<<<grid_for(n), 256>>>(d_b, (long long)n, scale_div, d_out);
      st = cudaGetLastError();
      if (st == cudaSuccess) st = cudaDeviceSynchronize();
    }
    cudaFree(d_b);
    PGB_CUDA(st);
  });
}

pgb_status pgb_device_params(pgb_engine* e, float** d) {
  return guarded([&] { *d = E(e).d_params; });
}

pgb_status pgb_device_stream(pgb_engine* e, void** s) {
  return guarded([&] { *s = (void*)E(e).stream; });
}

int32_t pgb_kernels_per_step(pgb_engine* e) { return e && e->impl ? e->impl->kernels_last : 0; }

}  // extern "C"
