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
inline std::uint64_t launches() { return tfg_launch_count(context()); }

}  // namespace texforge::device
