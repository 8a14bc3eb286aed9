#pragma once
// texforge/pipeline.hpp — Scheme 3: row chunks with halos, streamed to the GPU.
// Drop-in for R/include/texforge/pipeline.hpp.
//
//   partition (:48-73)            host arithmetic (tfg_partition), same specs
//   compute_glcm_chunked (:246)   -> tfg_glcm_chunked: the caller's thread
//       pulls chunk i from the ChunkSource into a pinned ring slot while the
//       GPU copies chunk i-1 (copy stream) and votes chunk i-2 (exec stream)
//       into one device accumulator; events hand slots back and forth. The
//       reference's ingest thread + 2-slot mutex/condvar ring becomes CUDA
//       streams + events; results are exact for any K.
//   PgmChunkSource (:104-137)     raw P5 rows are read straight into the
//       pinned slot and quantised inside the vote kernel (no host pass).
//   merge_chunk_glcms (:231-240)  host sum of host matrices.
//
// Failure semantics follow guarded_fetch (:257-265): a std::exception thrown
// by ChunkSource::fetch surfaces as PipelineError{chunk_index}; a
// PipelineError passes through unchanged.

#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "texforge/device.hpp"
#include "texforge/glcm.hpp"
#include "texforge/image.hpp"
#include "texforge/parallel.hpp"
#include "texforge/pgm.hpp"

namespace texforge {

struct PipelineError : std::runtime_error {
  std::size_t chunk_index;
  PipelineError(std::size_t index, const std::string& what)
      : std::runtime_error("chunk " + std::to_string(index) + ": " + what), chunk_index(index) {}
};

/// Owned anchor rows [owned_row_start, owned_row_end) plus read-only halo
/// rows up to buffer_row_end.
struct ChunkSpec {
  std::size_t index = 0;
  std::size_t owned_row_start = 0;
  std::size_t owned_row_end = 0;
  std::size_t buffer_row_end = 0;
  std::size_t chunk_count = 1;

  std::size_t owned_rows() const { return owned_row_end - owned_row_start; }
  std::size_t buffer_rows() const { return buffer_row_end - owned_row_start; }
  bool operator==(const ChunkSpec&) const = default;
};

/// K near-equal owned row ranges (the first H mod K get one more row); a
/// d-row halo for the downward angles, none at 0 degrees or on the last chunk.
inline std::vector<ChunkSpec> partition(std::size_t width, std::size_t height, const GlcmParams& p,
                                        std::size_t chunk_count) {
  std::vector<std::uint64_t> raw(3 * (chunk_count ? chunk_count : 1));
  if (chunk_count >= 1 && chunk_count <= height) raw.resize(3 * chunk_count);
  device::check(tfg_partition(width, height, p.distance, to_degrees(p.angle), chunk_count, raw.data()));
  std::vector<ChunkSpec> out(chunk_count);
  for (std::size_t i = 0; i < chunk_count; ++i)
    out[i] = ChunkSpec{i, raw[3 * i], raw[3 * i + 1], raw[3 * i + 2], chunk_count};
  return out;
}

/// Pull interface: fetch() fills `out` with rows [owned_row_start,
/// buffer_row_end), already quantised to levels().
class ChunkSource {
 public:
  virtual ~ChunkSource() = default;
  virtual std::size_t width() const = 0;
  virtual std::size_t height() const = 0;
  virtual int levels() const = 0;
  virtual void fetch(const ChunkSpec& spec, std::vector<std::uint8_t>& out) = 0;
};

class MemoryChunkSource final : public ChunkSource {
 public:
  explicit MemoryChunkSource(const QuantizedImage& img) : img_(img) {}
  std::size_t width() const override { return img_.width; }
  std::size_t height() const override { return img_.height; }
  int levels() const override { return img_.levels; }
  void fetch(const ChunkSpec& spec, std::vector<std::uint8_t>& out) override {
    const auto* first = img_.pixels.data() + spec.owned_row_start * img_.width;
    out.assign(first, first + spec.buffer_rows() * img_.width);
  }

 private:
  const QuantizedImage& img_;
};

/// Streams a P5 file by rows. fetch() quantises on the host (the reference
/// contract); compute_glcm_chunked instead reads raw rows into the pinned
/// ring with fetch_raw() and lets the vote kernel quantise.
class PgmChunkSource final : public ChunkSource {
 public:
  PgmChunkSource(const std::string& path, int levels) : path_(path), levels_(levels) {
    if (levels < 2 || levels > 256) throw std::invalid_argument("PgmChunkSource: levels must be in [2, 256]");
    std::ifstream f(path, std::ios::binary);
    if (!f) throw PgmError("pgm: cannot open " + path);
    std::vector<std::uint8_t> head(4096);
    f.read(reinterpret_cast<char*>(head.data()), static_cast<std::streamsize>(head.size()));
    head.resize(static_cast<std::size_t>(f.gcount()));
    header_ = parse_pgm_header(head);
  }

  std::size_t width() const override { return header_.width; }
  std::size_t height() const override { return header_.height; }
  int levels() const override { return levels_; }

  void fetch(const ChunkSpec& spec, std::vector<std::uint8_t>& out) override {
    out.resize(spec.buffer_rows() * header_.width);
    fetch_raw(spec, out.data());
    const auto L = static_cast<unsigned>(levels_);
    for (auto& v : out) v = static_cast<std::uint8_t>((v * L) >> 8);
  }

  /// Raw 8-bit rows [owned_row_start, buffer_row_end) into `dst`.
  void fetch_raw(const ChunkSpec& spec, std::uint8_t* dst) {
    if (!in_.is_open()) {
      in_.open(path_, std::ios::binary);
      if (!in_) throw PgmError("pgm: cannot open " + path_);
    }
    const std::size_t n = spec.buffer_rows() * header_.width;
    in_.clear();
    in_.seekg(static_cast<std::streamoff>(header_.data_offset + spec.owned_row_start * header_.width));
    in_.read(reinterpret_cast<char*>(dst), static_cast<std::streamsize>(n));
    if (static_cast<std::size_t>(in_.gcount()) != n) throw PgmError("pgm: truncated pixel data");
  }

 private:
  std::string path_;
  int levels_;
  PgmHeader header_;
  std::ifstream in_;
};

/// Wraps a source with a fixed-rate "link": fetch() returns no earlier than
/// ns_per_byte * bytes after it was entered (pipeline.hpp:143-203). With the
/// device pipeline this models an ingest link slower than PCIe.
class LatencyChunkSource final : public ChunkSource {
 public:
  LatencyChunkSource(ChunkSource& inner, double ns_per_byte) : inner_(inner), ns_per_byte_(ns_per_byte) {}

  std::size_t width() const override { return inner_.width(); }
  std::size_t height() const override { return inner_.height(); }
  int levels() const override { return inner_.levels(); }

  void fetch(const ChunkSpec& spec, std::vector<std::uint8_t>& out) override {
    using clock = std::chrono::steady_clock;
    const auto entered = clock::now();
    inner_.fetch(spec, out);
    if (ns_per_byte_ > 0.0) {
      const auto deadline =
          entered + std::chrono::nanoseconds(std::llround(ns_per_byte_ * static_cast<double>(out.size())));
      // coarse sleep, then yield to the deadline (timed sleeps wake late)
      const auto coarse = deadline - std::chrono::microseconds(500);
      if (clock::now() < coarse) std::this_thread::sleep_until(coarse);
      while (clock::now() < deadline) std::this_thread::yield();
    }
    bytes_served_ += out.size();
  }

  std::uint64_t bytes_served() const { return bytes_served_; }

 private:
  ChunkSource& inner_;
  double ns_per_byte_;
  std::uint64_t bytes_served_ = 0;
};

enum class ChunkExecution {
  pipelined,   // fetch chunk i+1 while the GPU copies/votes chunk i
  sequential,  // fetch, copy, vote, wait — one chunk at a time
};

/// Elementwise sum of per-chunk GLCMs (order-independent).
inline Glcm merge_chunk_glcms(const std::vector<Glcm>& parts) {
  if (parts.empty()) throw std::invalid_argument("merge_chunk_glcms: no parts");
  Glcm out(parts.front().levels);
  for (const Glcm& g : parts) {
    if (g.levels != out.levels) throw std::invalid_argument("merge_chunk_glcms: level mismatch");
    for (std::size_t i = 0; i < g.counts.size(); ++i) out.counts[i] += g.counts[i];
  }
  return out;
}

namespace detail {

// Adapts ChunkSource::fetch to the C ABI's tfg_fetch_fn. Two staging vectors
// alternate (the reference's two-slot ring), then the rows are copied into
// the pinned slot the engine hands us.
struct ChunkPump {
  ChunkSource& source;
  PgmChunkSource* raw_pgm;  // non-null: read raw rows straight into the slot
  std::size_t chunk_count;
  std::vector<std::uint8_t> slot[2];
  std::exception_ptr error;
  std::size_t failed_index = 0;

  static int fetch(void* user, std::size_t index, std::size_t start, std::size_t owned_end, std::size_t buf_end,
                   std::uint8_t* dst, char* err, std::size_t err_len) {
    auto* self = static_cast<ChunkPump*>(user);
    const ChunkSpec spec{index, start, owned_end, buf_end, self->chunk_count};
    try {
      const std::size_t bytes = spec.buffer_rows() * self->source.width();
      if (self->raw_pgm) {
        self->raw_pgm->fetch_raw(spec, dst);
      } else {
        std::vector<std::uint8_t>& buf = self->slot[index % 2];
        self->source.fetch(spec, buf);
        if (buf.size() != bytes)
          throw std::length_error("chunk source returned " + std::to_string(buf.size()) + " bytes, expected " +
                                  std::to_string(bytes));
        std::memcpy(dst, buf.data(), bytes);
      }
      return 0;
    } catch (const std::exception& e) {
      std::snprintf(err, err_len, "%s", e.what());
      self->error = std::current_exception();
    } catch (...) {
      self->error = std::current_exception();
    }
    self->failed_index = index;
    return 1;
  }
};

}  // namespace detail

/// Chunked GLCM through the device stream pipeline; equal to the unchunked
/// result for any K (pipeline.hpp:246-337).
inline Glcm compute_glcm_chunked(ChunkSource& source, const GlcmParams& p, const ExecutionPlan& plan,
                                 std::size_t chunk_count, ChunkExecution mode = ChunkExecution::pipelined) {
  (void)plan;  // the device planner sizes the kernel
  if (source.levels() != p.levels) throw std::invalid_argument("glcm: image levels do not match params levels");
  const std::size_t width = source.width(), height = source.height();
  (void)partition(width, height, p, chunk_count);  // the reference's argument checks and messages

  detail::ChunkPump pump{source, dynamic_cast<PgmChunkSource*>(&source), chunk_count, {}, nullptr, 0};
  const int pixel_levels = pump.raw_pgm ? 256 : p.levels;
  const int d = p.distance, a = to_degrees(p.angle);
  const unsigned flags = mode == ChunkExecution::sequential ? static_cast<unsigned>(TFG_SEQUENTIAL) : 0u;
  Glcm out(p.levels);
  // TEXFORGE_GPUS > 1: the chunks are spread over the GPU group (fetch calls
  // stay serialised) and the partials meet in one ncclReduce
  const int rc =
      device::gpus() > 1
          ? tfg_group_glcm_chunked(device::group(), width, height, pixel_levels, p.levels, &d, &a, 1, chunk_count,
                                   &detail::ChunkPump::fetch, &pump, flags, out.counts.data(), nullptr, nullptr)
          : tfg_glcm_chunked(device::context(), width, height, pixel_levels, p.levels, &d, &a, 1, chunk_count,
                             &detail::ChunkPump::fetch, &pump, flags, out.counts.data(), nullptr, nullptr);
  if (rc == TFG_SOURCE_ERROR && pump.error) {
    try {
      std::rethrow_exception(pump.error);
    } catch (const PipelineError&) {
      throw;
    } catch (const std::exception& e) {
      throw PipelineError(pump.failed_index, e.what());
    }
  }
  device::check(rc);
  return out;
}

}  // namespace texforge
