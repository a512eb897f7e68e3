// Internal helpers shared by the host (host.cpp) and device (engine.cu) parts
// of libpegrad_b200.so. Not installed; the public surface is
// include/pegrad_b200.h.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pegrad_b200.h"

namespace pgb {

// Carries a pgb_status through C++ code; converted at the C boundary.
struct Failure : std::runtime_error {
  pgb_status code;
  Failure(pgb_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(pgb_status c, const std::string& m) { throw Failure(c, m); }

void set_last_error(const std::string& m);

// Run `f`, translating exceptions into a status + thread-local message.
template <typename F>
pgb_status guarded(F&& f) {
  try {
    f();
    return PGB_OK;
  } catch (const Failure& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return PGB_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PGB_ERR_CONTRACT;
  }
}

// ---- counter-based RNG: bit-identical to proj/core/include/pegrad/rng.hpp:35-62
#if defined(__CUDACC__)
#define PGB_HD __host__ __device__ __forceinline__
#else
#define PGB_HD inline
#endif

PGB_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Stream key hoisted out of the per-element hash: rng_value_at(seed, stream, i)
// = mix64(key + golden*(i+1)) with key = mix64(seed + golden*(stream+1)).
PGB_HD uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed + 0x9E3779B97F4A7C15ull * (stream + 1));
}
PGB_HD uint64_t value_at(uint64_t key, uint64_t i) {
  return mix64(key + 0x9E3779B97F4A7C15ull * (i + 1));
}

// dpsgd.cpp:27-32
PGB_HD uint64_t noise_stream(int64_t step_index, int64_t param_ordinal) {
  return (uint64_t(1) << 32) + uint64_t(step_index) * 4096 + uint64_t(param_ordinal);
}

// Shapes of one example through the layer stack (mirrors trace_forward,
// models.cpp:169-296), computed once per engine.
struct ExShape {
  int rank = 1;
  int64_t d[3] = {0, 0, 0};
  int64_t numel() const {
    int64_t n = 1;
    for (int i = 0; i < rank; ++i) n *= d[i];
    return n;
  }
};

int64_t conv_out_extent(int64_t in, int64_t k, int64_t stride, int64_t pad);
void layer_shapes(const pgb_model_desc& d, ExShape* s /* n_layers+1 */);
void validate_dp_config(const pgb_dp_config& c, int64_t batch);
void check_strategy_support(int32_t strategy, const pgb_model_desc& d);
const char* layer_kind_name(int32_t k);

// An unsigned-byte IDX container read and validated on the host (the
// payload starts at bytes[offset]).
struct IdxArray {
  std::vector<unsigned char> bytes;
  std::vector<int64_t> dims;
  size_t offset = 0;
};
IdxArray read_idx(const std::string& path);

}  // namespace pgb
