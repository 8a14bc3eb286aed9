// ref_oracle.cpp — TEST INFRASTRUCTURE ONLY. A C-ABI wrapper around the
// UNMODIFIED reference headers (/root/reference/proj/include/texforge/*.hpp),
// compiled by oracle/Makefile into oracle/_ref/libtexforge_ref.so.
//
// Nothing from the reference is copied: this TU only #includes the headers
// where they lie and forwards to them. It lives in its own shared object so the
// reference's texforge:: names never meet the engine's (ODR).
//
// Used by: tests/golden/make_golden.py (golden vectors), tests/ (parity
// cross-check when the prebuilt .so is present) and bench.py --impl reference /
// the cpu_baseline leg (the reference's own CPU path, timed on the host cores).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "texforge/texforge.hpp"

using namespace texforge;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

QuantizedImage make_img(const uint8_t* px, size_t w, size_t h, int levels) {
  return QuantizedImage(w, h, levels, std::vector<uint8_t>(px, px + w * h));
}

void put(const Glcm& g, uint64_t* out) { std::memcpy(out, g.counts.data(), g.counts.size() * 8); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_quantize(const uint8_t* gray, size_t w, size_t h, int levels, uint8_t* out) {
  return guarded([&] {
    GrayImage img(w, h, std::vector<uint8_t>(gray, gray + w * h));
    auto q = quantize(img, levels);
    std::memcpy(out, q.pixels.data(), w * h);
  });
}

int ref_synth_noise(size_t w, size_t h, uint32_t seed, uint8_t* out) {
  return guarded([&] {
    auto g = synth_noise(w, h, seed);
    std::memcpy(out, g.pixels.data(), w * h);
  });
}

int ref_synth_smooth(size_t w, size_t h, uint32_t seed, uint8_t* out) {
  return guarded([&] {
    auto g = synth_smooth(w, h, seed);
    std::memcpy(out, g.pixels.data(), w * h);
  });
}

int ref_glcm_serial(const uint8_t* px, size_t w, size_t h, int levels, int d, int theta, uint64_t* out) {
  return guarded([&] {
    auto img = make_img(px, w, h, levels);
    put(compute_glcm_serial(img, {d, angle_from_degrees(theta), levels}), out);
  });
}

// Serial GLCM on a QuantizedImage that the caller has already validated; skips
// the defensive copy for timing (the reference's own bench excludes it too).
int ref_glcm_privatized(const uint8_t* px, size_t w, size_t h, int levels, int d, int theta,
                        unsigned workers, unsigned copies, uint64_t* out) {
  return guarded([&] {
    auto img = make_img(px, w, h, levels);
    ExecutionPlan pl = plan(levels, kDefaultScratchBudget, workers);
    if (copies) pl.copies = copies;
    put(compute_glcm_privatized(img, {d, angle_from_degrees(theta), levels}, pl).first, out);
  });
}

int ref_glcm_shared(const uint8_t* px, size_t w, size_t h, int levels, int d, int theta,
                    unsigned workers, uint64_t* out) {
  return guarded([&] {
    auto img = make_img(px, w, h, levels);
    ExecutionPlan pl = plan(levels, kDefaultScratchBudget, workers);
    put(compute_glcm_shared(img, {d, angle_from_degrees(theta), levels}, pl).first, out);
  });
}

int ref_glcm_chunked(const uint8_t* px, size_t w, size_t h, int levels, int d, int theta, size_t k,
                     unsigned workers, int sequential, uint64_t* out) {
  return guarded([&] {
    auto img = make_img(px, w, h, levels);
    ExecutionPlan pl = plan(levels, kDefaultScratchBudget, workers);
    MemoryChunkSource src(img);
    put(compute_glcm_chunked(src, {d, angle_from_degrees(theta), levels}, pl, k,
                             sequential ? ChunkExecution::sequential : ChunkExecution::pipelined),
        out);
  });
}

// Persistent-image timing helpers: build the QuantizedImage once (outside the
// timed region, as R/tools/texforge.cpp:218-236 does) and time only the call.
void* ref_image_new(const uint8_t* px, size_t w, size_t h, int levels) {
  try {
    return new QuantizedImage(make_img(px, w, h, levels));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_image_free(void* img) { delete static_cast<QuantizedImage*>(img); }

int ref_image_glcm(void* img, int d, int theta, unsigned workers, int scheme, uint64_t* out) {
  return guarded([&] {
    const auto& q = *static_cast<QuantizedImage*>(img);
    const GlcmParams p{d, angle_from_degrees(theta), q.levels};
    if (scheme == 0) {
      put(compute_glcm_serial(q, p), out);
    } else {
      put(compute_glcm_privatized(q, p, plan(q.levels, kDefaultScratchBudget, workers)).first, out);
    }
  });
}

int ref_symmetrize(const uint64_t* g, int levels, uint64_t* out) {
  return guarded([&] {
    Glcm in(levels, std::vector<uint64_t>(g, g + (size_t)levels * levels));
    put(symmetrize(in), out);
  });
}

int ref_normalize(const uint64_t* g, int levels, double* out) {
  return guarded([&] {
    Glcm in(levels, std::vector<uint64_t>(g, g + (size_t)levels * levels));
    auto p = normalize(in);
    std::memcpy(out, p.values.data(), p.values.size() * 8);
  });
}

int ref_features(const double* p, int levels, double* out5) {
  return guarded([&] {
    GlcmProbabilities probs;
    probs.levels = levels;
    probs.values.assign(p, p + (size_t)levels * levels);
    auto f = extract_features(probs);
    out5[0] = f.energy;
    out5[1] = f.contrast;
    out5[2] = f.homogeneity;
    out5[3] = f.entropy;
    out5[4] = f.correlation;
  });
}

int ref_partition(size_t w, size_t h, int d, int theta, size_t k, uint64_t* specs) {
  return guarded([&] {
    auto s = partition(w, h, {d, angle_from_degrees(theta), 8}, k);
    for (size_t i = 0; i < s.size(); ++i) {
      specs[3 * i] = s[i].owned_row_start;
      specs[3 * i + 1] = s[i].owned_row_end;
      specs[3 * i + 2] = s[i].buffer_row_end;
    }
  });
}

int ref_plan(int levels, size_t budget, unsigned workers, unsigned* copies, unsigned* gpu, int* degraded) {
  return guarded([&] {
    auto p = plan(levels, budget, workers);
    *copies = p.copies;
    *gpu = p.groups_per_unit;
    *degraded = p.degraded ? 1 : 0;
  });
}

}  // extern "C"
