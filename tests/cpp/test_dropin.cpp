// C++ tests of the drop-in texforge:: headers (include/texforge/) on the GPU,
// written against the reference's known answers so they
// run without /root/reference. The reference's own Catch2 suite is built
// separately (tests/cpp/Makefile, target ref).
#include <catch2/catch_amalgamated.hpp>

#include <cstdint>
#include <random>
#include <sstream>

#include "texforge/texforge.hpp"

using namespace texforge;

namespace {
const Angle kAngles[] = {Angle::deg0, Angle::deg45, Angle::deg90, Angle::deg135};

// Brute-force oracle: independent predicate scan, O(L^2 N^2) (test-only).
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

std::uint64_t fnv1a(const std::vector<std::uint64_t>& v) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (std::uint64_t x : v)
    for (int b = 0; b < 8; ++b) {
      h ^= (x >> (8 * b)) & 0xff;
      h *= 0x100000001b3ull;
    }
  return h;
}
}  // namespace

TEST_CASE("device GLCM equals the brute-force scan on random shapes") {
  std::mt19937 rng(5);
  for (int t = 0; t < 60; ++t) {
    const std::size_t w = 2 + rng() % 70, h = 2 + rng() % 50;
    const int levels = 2 + static_cast<int>(rng() % 255);
    const auto img = random_image(w, h, levels, rng());
    const int dmax = static_cast<int>(std::min(w, h)) - 1;
    const GlcmParams p{1 + static_cast<int>(rng() % dmax), kAngles[t % 4], levels};
    const Glcm g = compute_glcm_serial(img, p);
    CHECK(g == scan(img, p));
    CHECK(g.total() == valid_pair_count(w, h, p));
  }
}

TEST_CASE("known answers: 2x2 orientation, checkerboard, pair counts") {
  const QuantizedImage two(2, 2, 2, {0, 1, 1, 0});
  const Glcm g = compute_glcm_serial(two, {1, Angle::deg0, 2});
  CHECK(g.at(1, 0) == 1);
  CHECK(g.at(0, 1) == 1);
  std::vector<std::uint8_t> cb(16);
  for (int i = 0; i < 16; ++i) cb[i] = static_cast<std::uint8_t>(((i / 4) + (i % 4)) % 2);
  const Glcm c = compute_glcm_serial(QuantizedImage(4, 4, 2, cb), {1, Angle::deg0, 2});
  CHECK(c.at(0, 1) == 6);
  CHECK(c.at(1, 0) == 6);
  CHECK(valid_pair_count(1024, 1024, {4, Angle::deg135, 8}) == 1040400);
  CHECK_THROWS_AS(valid_pair_count(4, 4, {4, Angle::deg0, 8}), std::invalid_argument);
}

TEST_CASE("Appendix A hash: 512^2 noise L=8 d=1 0 degrees") {
  const auto img = quantize(synth_noise(512, 512, 1), 8);
  const Glcm g = compute_glcm_serial(img, {1, Angle::deg0, 8});
  CHECK(g.total() == 261632);
  CHECK(fnv1a(g.counts) == 0x94726aef2c9f9fe4ull);
}

TEST_CASE("Appendix A hash: 4096^2 smooth L=32 d=1 all angles") {
  const auto img = quantize(synth_smooth(4096, 4096, 1), 32);
  const std::uint64_t want[] = {0xa3dfa42d5708b8f3ull, 0x5b52858add8ee993ull, 0x8465f23466229a94ull,
                                0x4a4f1beb1c36a831ull};
  for (int a = 0; a < 4; ++a) CHECK(fnv1a(compute_glcm_serial(img, {1, kAngles[a], 32}).counts) == want[a]);
}

TEST_CASE("schemes agree: shared, privatized, chunked, sub-GLCM sums") {
  const auto img = random_image(97, 61, 16, 3);
  for (Angle a : kAngles) {
    const GlcmParams p{2, a, 16};
    const Glcm ref = scan(img, p);
    CHECK(compute_glcm_shared(img, p, plan(16, kDefaultScratchBudget, 4)).first == ref);
    ExecutionPlan pl = plan(16, kDefaultScratchBudget, 3);
    pl.copies = 3;
    const auto [g, st] = compute_glcm_privatized(img, p, pl);
    CHECK(g == ref);
    CHECK(st.per_copy_hottest.size() == 6 * 3);
    CHECK(reduce_subglcms(compute_subglcms(img, p, pl), 16) == ref);
    for (std::size_t k : {1, 2, 5, 9}) {
      MemoryChunkSource src(img);
      CHECK(compute_glcm_chunked(src, p, pl, k) == ref);
    }
  }
}

TEST_CASE("post-processing: symmetrize, normalize bit-exact, features") {
  const Glcm g(2, {3, 0, 1, 2});
  CHECK(symmetrize(g) == Glcm(2, {6, 1, 1, 4}));
  const GlcmProbabilities p = normalize(g);
  const double inv = 1.0 / 6.0;
  CHECK(p.at(0, 0) == 3.0 * inv);
  CHECK(p.at(1, 0) == 1.0 * inv);
  CHECK(p.at(1, 1) == 2.0 * inv);
  CHECK_THROWS_AS(normalize(Glcm(2)), std::invalid_argument);
  GlcmProbabilities u;
  u.levels = 4;
  u.values.assign(16, 1.0 / 16.0);
  const FeatureVector f = extract_features(u);
  CHECK(f.energy == Catch::Approx(1.0 / 16.0).epsilon(1e-12));
  CHECK(f.entropy == Catch::Approx(4.0).epsilon(1e-12));
  u.values[0] = 0.5;
  CHECK_THROWS_AS(extract_features(u), std::invalid_argument);
}

TEST_CASE("PGM source streams raw rows through the fused-quantise path") {
  const GrayImage gray = synth_noise(301, 77, 9);
  std::ostringstream os;
  write_pgm(gray, os);
  const std::string path = "/tmp/texforge_dropin_test.pgm";
  write_pgm_file(gray, path);
  PgmChunkSource src(path, 32);
  const GlcmParams p{3, Angle::deg45, 32};
  CHECK(compute_glcm_chunked(src, p, plan(32), 4) == scan(quantize(gray, 32), p));
  std::remove(path.c_str());
}

TEST_CASE("errors keep the reference's exception types and texts") {
  const auto img = random_image(8, 8, 4, 1);
  CHECK_THROWS_WITH(compute_glcm_serial(img, {1, Angle::deg0, 8}),
                    Catch::Matchers::ContainsSubstring("levels do not match"));
  CHECK_THROWS_WITH(compute_glcm_serial(img, {8, Angle::deg0, 4}),
                    Catch::Matchers::ContainsSubstring("degenerate geometry"));
  CHECK_THROWS_AS(QuantizedImage(2, 1, 4, {1, 4}), std::invalid_argument);
  CHECK_THROWS_AS(partition(8, 8, {1, Angle::deg90, 8}, 9), std::invalid_argument);
  CHECK(device::launches() > 0);
}
