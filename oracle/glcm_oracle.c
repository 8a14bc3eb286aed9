/*
 * glcm_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference
 * GLCM path (texture-forge, /root/reference/proj/include/texforge/*.hpp).
 *
 * This file is the parity checker for the B200 engine. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product path (paper_1710_06189_b200/) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 * the reference's own known-answer tests (R/tests/test_glcm.cpp, test_image.cpp,
 * test_features.cpp, test_pipeline.cpp) and against golden vectors generated
 * by the reference headers themselves (tests/golden/make_golden.py builds
 * oracle/_ref/libtexforge_ref.so from /root/reference and records its outputs).
 *
 * Citations: R/ = /root/reference/proj/.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

/* R/include/texforge/image.hpp:55-62 — q = (v * L) >> 8 */
int oracle_quantize(const uint8_t* in, size_t n, int levels, uint8_t* out) {
  if (levels < 2 || levels > 256) return 1;
  for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)(((unsigned)in[i] * (unsigned)levels) >> 8);
  return 0;
}

/* R/include/texforge/glcm.hpp:71-80 — (row, col) displacement anchor -> reference */
int oracle_neighbor_offset(int distance, int angle_deg, long* drow, long* dcol) {
  const long d = distance;
  switch (angle_deg) {
    case 0: *drow = 0; *dcol = d; return 0;
    case 45: *drow = d; *dcol = -d; return 0;
    case 90: *drow = d; *dcol = 0; return 0;
    case 135: *drow = d; *dcol = d; return 0;
    default: return 1;
  }
}

/* R/include/texforge/glcm.hpp:83-94 — closed-form in-bounds pair count; 0 on degenerate */
int oracle_valid_pair_count(size_t width, size_t height, int distance, int angle_deg, uint64_t* out) {
  const size_t d = (size_t)distance;
  if (distance < 1 || d >= width || d >= height) return 1;
  switch (angle_deg) {
    case 0: *out = (uint64_t)height * (width - d); return 0;
    case 90: *out = (uint64_t)(height - d) * width; return 0;
    case 45:
    case 135: *out = (uint64_t)(height - d) * (width - d); return 0;
    default: return 1;
  }
}

/*
 * R/include/texforge/glcm.hpp:110-130 (vote_anchor_rows) + :132-139
 * (serial_glcm_rows): anchors in rows [row_begin, min(row_end, H - drow)),
 * cols [d*[dcol<0], W - d*[dcol>0]); pos = ref * L + anchor. Counts are ADDED
 * into `counts` (L*L u64), so chunked callers can accumulate.
 */
int oracle_glcm_rows(const uint8_t* px, size_t width, size_t height, int levels, int distance,
                     int angle_deg, size_t row_begin, size_t row_end, uint64_t* counts) {
  long dr, dc;
  if (levels < 2 || levels > 256) return 1;
  if (oracle_neighbor_offset(distance, angle_deg, &dr, &dc)) return 1;
  const size_t d = (size_t)distance;
  if (distance < 1 || d >= width || d >= height) return 1;
  const size_t col_begin = dc < 0 ? d : 0;
  const size_t col_end = dc > 0 ? width - d : width;
  const size_t row_limit = dr > 0 ? height - d : height;
  if (row_end > row_limit) row_end = row_limit;
  const long shift = dr * (long)width + dc;
  for (size_t r = row_begin; r < row_end; ++r) {
    const uint8_t* anchor = px + r * width;
    const uint8_t* ref = anchor + shift;
    for (size_t c = col_begin; c < col_end; ++c) counts[(size_t)ref[c] * (size_t)levels + anchor[c]] += 1;
  }
  return 0;
}

/* R/include/texforge/glcm.hpp:98-104 + :144-147 — compute_glcm_serial */
int oracle_glcm_serial(const uint8_t* px, size_t width, size_t height, int levels, int distance,
                       int angle_deg, uint64_t* counts) {
  for (size_t i = 0; i < width * height; ++i)
    if ((int)px[i] >= levels) return 1; /* QuantizedImage ctor, image.hpp:46-48 */
  memset(counts, 0, sizeof(uint64_t) * (size_t)levels * (size_t)levels);
  return oracle_glcm_rows(px, width, height, levels, distance, angle_deg, 0, height, counts);
}

/* Fused quantise + vote: quantize(gray, L) then compute_glcm_serial. */
int oracle_glcm_gray(const uint8_t* gray, size_t width, size_t height, int levels, int distance,
                     int angle_deg, uint64_t* counts) {
  long dr, dc;
  if (levels < 2 || levels > 256) return 1;
  if (oracle_neighbor_offset(distance, angle_deg, &dr, &dc)) return 1;
  const size_t d = (size_t)distance;
  if (distance < 1 || d >= width || d >= height) return 1;
  uint8_t lut[256];
  for (int v = 0; v < 256; ++v) lut[v] = (uint8_t)(((unsigned)v * (unsigned)levels) >> 8);
  memset(counts, 0, sizeof(uint64_t) * (size_t)levels * (size_t)levels);
  const size_t col_begin = dc < 0 ? d : 0;
  const size_t col_end = dc > 0 ? width - d : width;
  const size_t row_end = dr > 0 ? height - d : height;
  const long shift = dr * (long)width + dc;
  for (size_t r = 0; r < row_end; ++r) {
    const uint8_t* anchor = gray + r * width;
    const uint8_t* ref = anchor + shift;
    for (size_t c = col_begin; c < col_end; ++c)
      counts[(size_t)lut[ref[c]] * (size_t)levels + lut[anchor[c]]] += 1;
  }
  return 0;
}

/* R/include/texforge/glcm.hpp:150-156 — out(i,j) = g(i,j) + g(j,i) */
void oracle_symmetrize(const uint64_t* g, int levels, uint64_t* out) {
  const size_t n = (size_t)levels;
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j) out[i * n + j] = g[i * n + j] + g[j * n + i];
}

/* R/include/texforge/glcm.hpp:167-177 — inv = 1.0/total; p = (double)c * inv */
int oracle_normalize(const uint64_t* g, int levels, double* out) {
  const size_t n = (size_t)levels * (size_t)levels;
  uint64_t total = 0;
  for (size_t i = 0; i < n; ++i) total += g[i];
  if (total == 0) return 1;
  const double inv = 1.0 / (double)total;
  for (size_t i = 0; i < n; ++i) out[i] = (double)g[i] * inv;
  return 0;
}

/* R/include/texforge/features.hpp:22-31 — compensated sum */
static double kahan_sum(const double* xs, size_t n) {
  double sum = 0.0, carry = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double y = xs[i] - carry;
    double t = sum + y;
    carry = (t - sum) - y;
    sum = t;
  }
  return sum;
}

/*
 * R/include/texforge/features.hpp:37-69 — energy, contrast, homogeneity,
 * entropy (bits), correlation; two fp64 passes in row-major order.
 * out5 = {energy, contrast, homogeneity, entropy, correlation}.
 */
int oracle_features(const double* p, int levels, double* out5) {
  const int n = levels;
  if (fabs(kahan_sum(p, (size_t)n * (size_t)n) - 1.0) > 1e-12) return 1;
  double energy = 0, contrast = 0, homogeneity = 0, entropy = 0;
  double mean_i = 0.0, mean_j = 0.0, cross = 0.0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      const double v = p[(size_t)i * n + j];
      const double diff = (double)(i - j);
      energy += v * v;
      contrast += diff * diff * v;
      homogeneity += v / (1.0 + diff * diff);
      if (v > 0.0) entropy -= v * log2(v);
      mean_i += i * v;
      mean_j += j * v;
      cross += (double)i * j * v;
    }
  }
  double var_i = 0.0, var_j = 0.0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      const double v = p[(size_t)i * n + j];
      var_i += (i - mean_i) * (i - mean_i) * v;
      var_j += (j - mean_j) * (j - mean_j) * v;
    }
  }
  const double sigma = sqrt(var_i) * sqrt(var_j);
  out5[0] = energy;
  out5[1] = contrast;
  out5[2] = homogeneity;
  out5[3] = entropy;
  out5[4] = sigma > 0.0 ? (cross - mean_i * mean_j) / sigma : 0.0;
  return 0;
}

/*
 * R/include/texforge/pipeline.hpp:48-73 — K owned row ranges (first H mod K
 * get +1 row), halo = d rows for theta != 0, none on the last chunk.
 * specs: K x {owned_start, owned_end, buffer_end}.
 */
int oracle_partition(size_t width, size_t height, int distance, int angle_deg, size_t k,
                     uint64_t* specs) {
  const size_t d = (size_t)distance;
  if (distance < 1 || d >= width || d >= height) return 1;
  if (k < 1 || k > height) return 2;
  if (height / k <= d && k > 1) return 3;
  const size_t halo = angle_deg == 0 ? 0 : d;
  const size_t base = height / k, extra = height % k;
  size_t row = 0;
  for (size_t i = 0; i < k; ++i) {
    const size_t end = row + base + (i < extra ? 1 : 0);
    specs[3 * i + 0] = row;
    specs[3 * i + 1] = end;
    specs[3 * i + 2] = i + 1 == k ? end : end + halo;
    row = end;
  }
  return 0;
}

/*
 * R/include/texforge/pipeline.hpp:212-240 — chunked GLCM: each chunk votes its
 * owned anchor rows against a buffer of rows [owned_start, buffer_end); the
 * per-chunk counts are summed (order-independent).
 */
int oracle_glcm_chunked(const uint8_t* px, size_t width, size_t height, int levels, int distance,
                        int angle_deg, size_t k, uint64_t* counts) {
  uint64_t specs[3 * 4096];
  if (k > 4096) return 1;
  int rc = oracle_partition(width, height, distance, angle_deg, k, specs);
  if (rc) return rc;
  memset(counts, 0, sizeof(uint64_t) * (size_t)levels * (size_t)levels);
  for (size_t i = 0; i < k; ++i) {
    const size_t start = specs[3 * i], owned_end = specs[3 * i + 1], buf_end = specs[3 * i + 2];
    rc = oracle_glcm_rows(px + start * width, width, buf_end - start, levels, distance, angle_deg, 0,
                          owned_end - start, counts);
    if (rc) return rc;
  }
  return 0;
}

/* R/include/texforge/parallel.hpp:39-61 — Eq. 4-6 sizing of R against the budget */
int oracle_plan(int levels, size_t scratch_budget, unsigned* copies, unsigned* groups_per_unit,
                int* degraded) {
  if (levels < 2 || levels > 256) return 1;
  const size_t sub = (size_t)levels * (size_t)levels * 4u;
  size_t c = scratch_budget / (2 * sub);
  if (c >= 1) {
    *groups_per_unit = 2;
    *degraded = 0;
  } else {
    *groups_per_unit = 1;
    *degraded = 1;
    c = scratch_budget / sub;
    if (c < 1) c = 1;
  }
  *copies = (unsigned)(c < 8 ? c : 8);
  return 0;
}

/* R/include/texforge/parallel.hpp:91-102 — total, hottest (lowest flat index on ties) */
void oracle_stats(const uint64_t* g, int levels, uint64_t* total, uint64_t* hottest, int* hot_row,
                  int* hot_col) {
  const size_t n = (size_t)levels * (size_t)levels;
  size_t best = 0;
  uint64_t t = 0;
  for (size_t i = 0; i < n; ++i) {
    t += g[i];
    if (g[i] > g[best]) best = i;
  }
  *total = t;
  *hottest = g[best];
  *hot_row = (int)(best / (size_t)levels);
  *hot_col = (int)(best % (size_t)levels);
}

/* FNV-1a-64 over u64 little-endian bytes (SURVEY.md Appendix A hash definition). */
uint64_t oracle_fnv1a64_u64(const uint64_t* v, size_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i)
    for (int b = 0; b < 8; ++b) {
      h ^= (v[i] >> (8 * b)) & 0xffu;
      h *= 0x100000001b3ull;
    }
  return h;
}
