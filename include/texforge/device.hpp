#pragma once
// texforge/device.hpp — the runtime beneath the drop-in texforge:: headers.
//
// The reference's headers (R/ = /root/reference/proj/include/texforge/) are
// header-only CPU code. These headers keep every public name and signature,
// but each heavy function forwards to libtexforge_cuda.so through the C ABI
// in ../texforge_cuda.h (sm_100a kernels). This file owns the one piece of
// state that implies: a process-wide engine context on one CUDA device.
//
//   TEXFORGE_DEVICE=<n>   CUDA device of the default context (default 0)
//   TEXFORGE_GPUS=<n>     n > 1: whole-image GLCMs (compute_glcm_serial and the
//                         calls built on it) and compute_glcm_chunked run on a
//                         group of n GPUs with one NCCL communicator
//                         (tfg_group_*: row shards + d-row halo + one ncclReduce)
//   TEXFORGE_GPUS_HOST_REDUCE=1  the group may share GPUs and sums through host
//                         memory (tests of the multi-GPU split on one GPU)
//
// Errors: status codes from the C ABI become the reference's exception types
// with the library's message text (std::invalid_argument for contract
// violations, std::runtime_error for device failures). PipelineError is
// raised by pipeline.hpp, which owns that type.
//
// Link with -ltexforge_cuda (paper_1710_06189_b200/libtexforge_cuda.so).

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../texforge_cuda.h"

namespace texforge::device {

/// The default engine context, created on first use. It is intentionally
/// never destroyed: tearing down CUDA objects from a static destructor races
/// the CUDA runtime's own exit handlers, and process exit frees everything.
inline tfg_ctx* context() {
  static tfg_ctx* ctx = [] {
    int dev = 0;
    if (const char* env = std::getenv("TEXFORGE_DEVICE")) dev = std::atoi(env);
    tfg_ctx* c = nullptr;
    const int rc = tfg_ctx_create(&c, dev, 0);
    if (rc != TFG_OK)
      throw std::runtime_error(std::string("texforge device: cannot create engine context: ") + tfg_last_error());
    return c;
  }();
  return ctx;
}

/// GPUs of the multi-GPU group (TEXFORGE_GPUS, default 1 = no group).
inline int gpus() {
  static const int n = [] {
    const char* env = std::getenv("TEXFORGE_GPUS");
    const int v = env ? std::atoi(env) : 1;
    return v > 1 ? v : 1;
  }();
  return n;
}

/// The multi-GPU group (created on first use when gpus() > 1; never destroyed,
/// like context()).
inline tfg_group* group() {
  static tfg_group* g = [] {
    const char* hr = std::getenv("TEXFORGE_GPUS_HOST_REDUCE");
    const unsigned flags = (hr && std::atoi(hr) != 0) ? TFG_GROUP_HOST_REDUCE : 0u;
    tfg_group* out = nullptr;
    const int rc = tfg_group_create(&out, gpus(), nullptr, flags);
    if (rc != TFG_OK)
      throw std::runtime_error(std::string("texforge device: cannot create the GPU group: ") + tfg_last_error());
    return out;
  }();
  return g;
}

/// Maps a C-ABI status to the reference's exception types.
inline void check(int rc) {
  if (rc == TFG_OK) return;
  const std::string msg = tfg_last_error();
  if (rc == TFG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == TFG_OUT_OF_MEMORY) throw std::bad_alloc();
  throw std::runtime_error("texforge device: " + msg);
}

/// Number of engine kernels the default context has launched (evidence that
/// a call ran on the GPU).
inline std::uint64_t launches() {
  return tfg_launch_count(context()) + (gpus() > 1 ? tfg_group_launch_count(group()) : 0);
}

}  // namespace texforge::device
