#pragma once
// texforge/image.hpp — raster types, quantiser and synthetic inputs.
// Drop-in for R/include/texforge/image.hpp (types :13-52, quantize :55-62,
// synth_smooth :76-106, synth_noise :109-116).
//
//   quantize      -> quantize_kernel on the GPU (tfg_quantize). The GLCM entry
//                    points never need it: they fuse q = (v*L)>>8 into the vote.
//   synth_*       -> libtexforge_cuda.so host generators (bit-identical to the
//                    reference's mt19937 / std::sin sequences; synth_smooth
//                    generates rows on every host thread, synth_noise splits
//                    the mt19937 sequence by jump-ahead across them).
//                    tfg_synth_noise_device generates synth_noise in HBM.

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

#include "texforge/device.hpp"

namespace texforge {

/// 8-bit grayscale raster, row-major (image.hpp:13-28).
struct GrayImage {
  std::size_t width = 0;
  std::size_t height = 0;
  std::vector<std::uint8_t> pixels;

  GrayImage() = default;
  GrayImage(std::size_t w, std::size_t h, std::vector<std::uint8_t> px)
      : width(w), height(h), pixels(std::move(px)) {
    if (w == 0 || h == 0) throw std::invalid_argument("GrayImage: dimensions must be positive");
    if (pixels.size() != w * h) throw std::invalid_argument("GrayImage: pixel count does not match dimensions");
  }

  std::uint8_t at(std::size_t row, std::size_t col) const { return pixels[row * width + col]; }
};

/// Raster of gray levels in [0, levels) (image.hpp:31-52). The constructor
/// validates every pixel, exactly like the reference.
struct QuantizedImage {
  std::size_t width = 0;
  std::size_t height = 0;
  int levels = 0;
  std::vector<std::uint8_t> pixels;

  QuantizedImage() = default;
  QuantizedImage(std::size_t w, std::size_t h, int lv, std::vector<std::uint8_t> px)
      : QuantizedImage(trusted{}, w, h, lv, std::move(px)) {
    const auto limit = static_cast<unsigned>(lv);
    for (const std::uint8_t v : pixels)
      if (v >= limit) throw std::invalid_argument("QuantizedImage: pixel value exceeds gray level");
  }

  std::uint8_t at(std::size_t row, std::size_t col) const { return pixels[row * width + col]; }

  // Internal: pixels produced by the device quantiser are < levels by
  // construction, so the O(W*H) host re-scan is skipped.
  struct trusted {};
  QuantizedImage(trusted, std::size_t w, std::size_t h, int lv, std::vector<std::uint8_t> px)
      : width(w), height(h), levels(lv), pixels(std::move(px)) {
    if (w == 0 || h == 0) throw std::invalid_argument("QuantizedImage: dimensions must be positive");
    if (lv < 2 || lv > 256) throw std::invalid_argument("QuantizedImage: levels must be in [2, 256]");
    if (pixels.size() != w * h)
      throw std::invalid_argument("QuantizedImage: pixel count does not match dimensions");
  }
};

/// q = floor(v * levels / 256), computed on the GPU (image.hpp:55-62).
inline QuantizedImage quantize(const GrayImage& img, int levels) {
  if (levels < 2 || levels > 256) throw std::invalid_argument("quantize: levels must be in [2, 256]");
  std::vector<std::uint8_t> out(img.pixels.size());
  if (!out.empty())
    device::check(tfg_quantize(device::context(), img.pixels.data(), img.pixels.size(), levels, out.data(), 0));
  return QuantizedImage(QuantizedImage::trusted{}, img.width, img.height, levels, std::move(out));
}

/// Low-frequency field of four seeded sinusoids (image.hpp:76-106).
inline GrayImage synth_smooth(std::size_t width, std::size_t height, std::uint32_t seed) {
  if (width < 2 || height < 2) throw std::invalid_argument("synth_smooth: dimensions must be >= 2");
  std::vector<std::uint8_t> px(width * height);
  device::check(tfg_synth_smooth(width, height, seed, px.data(), 0));
  return GrayImage(width, height, std::move(px));
}

/// Seeded uniform noise over [0, 255] (image.hpp:109-116).
inline GrayImage synth_noise(std::size_t width, std::size_t height, std::uint32_t seed) {
  if (width < 2 || height < 2) throw std::invalid_argument("synth_noise: dimensions must be >= 2");
  std::vector<std::uint8_t> px(width * height);
  device::check(tfg_synth_noise(width, height, seed, px.data()));
  return GrayImage(width, height, std::move(px));
}

}  // namespace texforge
