// The multi-GPU C ABI (tfg_group_*) called directly from C++: a group of ONE
// GPU with a real NCCL communicator (ncclCommInitAll) and the real
// ncclReduce, checked against a brute-force scan. With TEXFORGE_GPUS > 1 in
// the environment (tests/test_cpp_dropin.py sets 3 + host reduce on a one-GPU
// box) the drop-in texforge:: calls themselves run on the group.
#include <catch2/catch_amalgamated.hpp>

#include <cstdint>
#include <cstring>
#include <random>

#include "texforge/texforge.hpp"

using namespace texforge;

namespace {
Glcm scan(const QuantizedImage& img, const GlcmParams& p) {
  const PixelOffset o = neighbor_offset(p);
  Glcm g(p.levels);
  const auto h = static_cast<std::ptrdiff_t>(img.height), w = static_cast<std::ptrdiff_t>(img.width);
  for (std::ptrdiff_t r = 0; r < h; ++r)
    for (std::ptrdiff_t c = 0; c < w; ++c) {
      const std::ptrdiff_t r2 = r + o.row, c2 = c + o.col;
      if (r2 < 0 || r2 >= h || c2 < 0 || c2 >= w) continue;
      ++g.at(img.at(r2, c2), img.at(r, c));
    }
  return g;
}

QuantizedImage random_image(std::size_t w, std::size_t h, int levels, std::uint32_t seed) {
  std::mt19937 rng(seed);
  std::vector<std::uint8_t> px(w * h);
  for (auto& v : px) v = static_cast<std::uint8_t>(rng() % static_cast<unsigned>(levels));
  return QuantizedImage(w, h, levels, std::move(px));
}

struct VecSource {
  const QuantizedImage* img;
  static int fetch(void* user, std::size_t, std::size_t start, std::size_t, std::size_t buf_end, std::uint8_t* dst,
                   char*, std::size_t) {
    const auto* s = static_cast<VecSource*>(user);
    std::memcpy(dst, s->img->pixels.data() + start * s->img->width, (buf_end - start) * s->img->width);
    return 0;
  }
};
}  // namespace

TEST_CASE("group of one GPU: NCCL communicator, row partition, reduce, chunks") {
  tfg_group* g = nullptr;
  REQUIRE(tfg_group_create(&g, 1, nullptr, 0) == TFG_OK);
  REQUIRE(tfg_group_size(g) == 1);
  for (int levels : {8, 64, 256}) {
    const auto img = random_image(613, 411, levels, 7u + levels);
    const int ds[] = {1, 1, 3, 2}, as[] = {0, 45, 90, 135};
    std::vector<std::uint64_t> counts(4 * levels * levels);
    REQUIRE(tfg_group_glcm(g, img.pixels.data(), img.width, img.height, levels, levels, ds, as, 4, 0,
                           counts.data(), nullptr, nullptr) == TFG_OK);
    std::vector<std::uint64_t> chunked(4 * levels * levels);
    VecSource src{&img};
    REQUIRE(tfg_group_glcm_chunked(g, img.width, img.height, levels, levels, ds, as, 4, 5, &VecSource::fetch, &src, 0,
                                   chunked.data(), nullptr, nullptr) == TFG_OK);
    for (int t = 0; t < 4; ++t) {
      const GlcmParams p{ds[t], angle_from_degrees(as[t]), levels};
      const Glcm want = scan(img, p);
      const std::vector<std::uint64_t> got(counts.begin() + t * levels * levels,
                                           counts.begin() + (t + 1) * levels * levels);
      const std::vector<std::uint64_t> gotc(chunked.begin() + t * levels * levels,
                                            chunked.begin() + (t + 1) * levels * levels);
      CHECK(got == want.counts);
      CHECK(gotc == want.counts);
    }
  }
  CHECK(tfg_group_launch_count(g) > 0);
  tfg_group_destroy(g);
}

TEST_CASE("drop-in calls on the GPU group (TEXFORGE_GPUS)") {
  std::mt19937 rng(11);
  for (int t = 0; t < 12; ++t) {
    const std::size_t w = 40 + rng() % 300, h = 30 + rng() % 200;
    const int levels = 2 + static_cast<int>(rng() % 255);
    const auto img = random_image(w, h, levels, rng());
    const GlcmParams p{1 + static_cast<int>(rng() % 6), angle_from_degrees(45 * (t % 4)), levels};
    CHECK(compute_glcm_serial(img, p) == scan(img, p));
    MemoryChunkSource src(img);
    CHECK(compute_glcm_chunked(src, p, plan(levels), 4) == scan(img, p));
  }
  CHECK(device::gpus() >= 1);
}
