#pragma once
// texforge/features.hpp — Haralick-5 statistics of a normalised GLCM.
// Drop-in for R/include/texforge/features.hpp (FeatureVector :11-17,
// extract_features :37-69) -> features_kernel on the GPU (one CTA per
// matrix, fp64). The sums run as a fixed parallel tree instead of the
// reference's sequential loop, so results agree to ulps (tests: 1e-10).

#include <stdexcept>

#include "texforge/device.hpp"
#include "texforge/glcm.hpp"

namespace texforge {

struct FeatureVector {
  double energy = 0.0;
  double contrast = 0.0;
  double homogeneity = 0.0;
  double entropy = 0.0;  // bits
  double correlation = 0.0;
};

/// Rejects a matrix whose compensated sum is not 1 within 1e-12; the
/// correlation of a zero-variance distribution is 0.
inline FeatureVector extract_features(const GlcmProbabilities& p) {
  if (p.values.size() != static_cast<std::size_t>(p.levels) * p.levels || p.levels < 1)
    throw std::invalid_argument("extract_features: input is not normalized");
  double f[5];
  device::check(tfg_features(device::context(), p.values.data(), p.levels, f));
  return FeatureVector{f[0], f[1], f[2], f[3], f[4]};
}

}  // namespace texforge
