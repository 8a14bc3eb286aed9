#pragma once
// texforge/parallel.hpp — Schemes 1 and 2 and the planner.
// Drop-in for R/include/texforge/parallel.hpp.
//
//   plan (:39-66)                 host arithmetic, unchanged (tests pin it)
//   compute_glcm_shared (:143)    -> Scheme-1 kernel: one global u64 atomic per
//                                    pixel pair (glcm_vote_global_kernel)
//   compute_subglcms (:218)       -> glcm_subglcm_kernel: the reference's exact
//                                    group/lane/copy routing, on the device
//   compute_glcm_privatized (:240)-> glcm_vote_kernel for the counts plus the
//                                    sub-GLCM kernel for per_copy_hottest
//   reduce_subglcms (:228)        host: its inputs and output are host vectors
//   contention_profile (:258)     stats of the device GLCM
//
// The reference's ExecutionPlan described a CPU "launch": worker threads of
// 512-lane groups with R copies in a 48 KiB scratch. It still drives the
// semantics of compute_subglcms / per_copy_hottest exactly; the device
// planner that sizes the real kernel (R copies in up to 227 KB of shared
// memory per CTA, 148 SMs) lives inside libtexforge_cuda.so.

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <thread>
#include <utility>
#include <vector>

#include "texforge/device.hpp"
#include "texforge/glcm.hpp"
#include "texforge/image.hpp"

namespace texforge {

inline constexpr std::size_t kDefaultScratchBudget = 49152;

struct ExecutionPlan {
  unsigned worker_count = 1;
  unsigned group_size = 512;
  unsigned copies = 1;
  std::size_t scratch_budget = kDefaultScratchBudget;
  unsigned groups_per_unit = 2;
  bool degraded = false;
};

struct ContentionStats {
  std::uint64_t total_votes = 0;
  std::uint64_t hottest_cell_votes = 0;
  std::pair<int, int> hottest_cell_index = {0, 0};  // lowest flat index on ties
  std::vector<std::uint64_t> per_copy_hottest;      // privatised: one per sub-GLCM
  double concentration = 0.0;
};

/// R = clamp(floor(budget / (2 * 4L^2)), 1, 8) with two resident groups, or
/// one group ("degraded") when two do not fit (parallel.hpp:39-61).
inline ExecutionPlan plan(int levels, std::size_t scratch_budget, unsigned worker_count) {
  if (levels < 2 || levels > 256) throw std::invalid_argument("plan: levels must be in [2, 256]");
  ExecutionPlan out;
  out.worker_count = worker_count ? worker_count : 1;
  out.scratch_budget = scratch_budget;
  unsigned copies = 0;
  unsigned groups = 0;
  int degraded = 0;
  device::check(tfg_plan(levels, scratch_budget, out.worker_count, &copies, &groups, &degraded));
  out.copies = copies;
  out.groups_per_unit = groups;
  out.degraded = degraded != 0;
  return out;
}

inline ExecutionPlan plan(int levels) {
  const unsigned hw = std::thread::hardware_concurrency();
  return plan(levels, kDefaultScratchBudget, hw ? hw : 1);
}

namespace detail {

inline ContentionStats stats_from_counts(const Glcm& g) {
  ContentionStats s;
  std::size_t best = 0;
  for (std::size_t i = 0; i < g.counts.size(); ++i) {
    s.total_votes += g.counts[i];
    if (g.counts[i] > g.counts[best]) best = i;  // strict: the lowest index wins ties
  }
  s.hottest_cell_votes = g.counts.empty() ? 0 : g.counts[best];
  s.hottest_cell_index = {static_cast<int>(best) / g.levels, static_cast<int>(best) % g.levels};
  if (s.total_votes)
    s.concentration = static_cast<double>(s.hottest_cell_votes) / static_cast<double>(s.total_votes);
  return s;
}

// Group count of the privatised scheme (parallel.hpp:166-181): 0 means
// groups_per_unit * worker_count, raised so no group can exceed 2^32 votes,
// then clamped to [1, rows].
inline std::size_t resolve_group_count(std::size_t requested, const ExecutionPlan& plan, std::size_t width,
                                       std::size_t rows) {
  std::size_t g = requested;
  if (g == 0) {
    g = static_cast<std::size_t>(plan.groups_per_unit ? plan.groups_per_unit : 2) * plan.worker_count;
    const std::uint64_t ceiling = std::uint64_t{1} << 32;
    const std::uint64_t worst = static_cast<std::uint64_t>(rows) * width;
    const auto floor_groups = static_cast<std::size_t>((worst + ceiling - 1) / ceiling);
    if (g < floor_groups) g = floor_groups;
  }
  if (g > rows) g = rows;
  return g ? g : 1;
}

}  // namespace detail

/// Scheme 1: every pair is one atomic on the global matrix (parallel.hpp:143-152).
inline std::pair<Glcm, ContentionStats> compute_glcm_shared(const QuantizedImage& img, const GlcmParams& p,
                                                            const ExecutionPlan& plan) {
  (void)plan;  // the device grid replaces the worker pool
  detail::check_glcm_inputs(img, p);
  Glcm g = detail::device_glcm(img, p, TFG_SCHEME_GLOBAL);
  ContentionStats s = detail::stats_from_counts(g);
  return {std::move(g), std::move(s)};
}

/// Raw (group, copy) sub-GLCMs, group-major (parallel.hpp:218-225).
inline std::vector<std::vector<std::uint32_t>> compute_subglcms(const QuantizedImage& img, const GlcmParams& p,
                                                                const ExecutionPlan& plan,
                                                                std::size_t group_count = 0) {
  detail::check_glcm_inputs(img, p);
  if (plan.copies < 1) throw std::invalid_argument("privatized: plan.copies must be >= 1");
  const std::size_t groups = detail::resolve_group_count(group_count, plan, img.width, img.height);
  const std::size_t cells = static_cast<std::size_t>(p.levels) * p.levels;
  std::vector<std::uint32_t> flat(groups * plan.copies * cells);
  device::check(tfg_subglcms(device::context(), img.pixels.data(), img.width, img.height, img.levels, p.levels,
                             p.distance, to_degrees(p.angle), plan.group_size, plan.copies, groups, 0,
                             flat.data(), nullptr, nullptr));
  std::vector<std::vector<std::uint32_t>> subs(groups * plan.copies);
  for (std::size_t i = 0; i < subs.size(); ++i)
    subs[i].assign(flat.begin() + static_cast<std::ptrdiff_t>(i * cells),
                   flat.begin() + static_cast<std::ptrdiff_t>((i + 1) * cells));
  return subs;
}

/// Elementwise u64 sum of sub-GLCMs (parallel.hpp:228-237).
inline Glcm reduce_subglcms(const std::vector<std::vector<std::uint32_t>>& subs, int levels) {
  Glcm out(levels);
  for (const auto& sub : subs) {
    if (sub.size() != out.counts.size()) throw std::invalid_argument("reduce_subglcms: sub-GLCM length mismatch");
    for (std::size_t i = 0; i < sub.size(); ++i) out.counts[i] += sub[i];
  }
  return out;
}

/// Scheme 2 (parallel.hpp:240-254): counts from the privatised vote kernel,
/// per_copy_hottest from the reference-routed sub-GLCMs.
inline std::pair<Glcm, ContentionStats> compute_glcm_privatized(const QuantizedImage& img, const GlcmParams& p,
                                                                const ExecutionPlan& plan,
                                                                std::size_t group_count = 0) {
  detail::check_glcm_inputs(img, p);
  if (plan.copies < 1) throw std::invalid_argument("privatized: plan.copies must be >= 1");
  const std::size_t groups = detail::resolve_group_count(group_count, plan, img.width, img.height);
  Glcm g(p.levels);
  std::vector<std::uint64_t> hottest(groups * plan.copies);
  device::check(tfg_subglcms(device::context(), img.pixels.data(), img.width, img.height, img.levels, p.levels,
                             p.distance, to_degrees(p.angle), plan.group_size, plan.copies, groups, 0, nullptr,
                             g.counts.data(), hottest.data()));
  ContentionStats s = detail::stats_from_counts(g);
  s.per_copy_hottest = std::move(hottest);
  return {std::move(g), std::move(s)};
}

/// Vote concentration of the exact GLCM (parallel.hpp:258-260).
inline ContentionStats contention_profile(const QuantizedImage& img, const GlcmParams& p) {
  return detail::stats_from_counts(compute_glcm_serial(img, p));
}

}  // namespace texforge
