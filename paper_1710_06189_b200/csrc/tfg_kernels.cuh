// tfg_kernels.cuh — sm_100a device code of the B200 GLCM engine.
//
// K1 glcm_vote_kernel: fused quantise + pixel-pair vote + privatised
//    shared-memory sub-GLCMs (the paper's "copies", re-sized
//    for 227 KB/CTA) + in-kernel merge (K2).  Semantics follow
//    R/include/texforge/glcm.hpp:110-130 (vote_anchor_rows) exactly:
//    anchors in rows [0, min(row_end, H - drow)), columns
//    [d*[dcol<0], W - d*[dcol>0]), cell = ref*L + anchor.
// K0 glcm_vote_global_kernel: Scheme 1 (one global atomic per pair,
//    PAPER.md:62-93 / parallel.hpp:121-152) — ablation only.
// K3 symmetrize / normalize, K4 features — post-processing on device.
//
// Work decomposition: the valid-anchor raster is cut into
// 16-pixel "items" (one 16-byte vector per row segment).  A CTA of 1024
// threads owns a contiguous item range and walks it in rounds of 2 items per
// thread; consecutive threads take consecutive 16-byte segments of a row, so
// every LDG.128 of a warp is one coalesced 512-byte access.  The reference
// neighbour of each segment is two aligned 16-byte loads + funnel shifts
// (displacement dcol = 16q + 4k + s: q and the word shift k are template /
// launch constants, s is a byte funnel shift).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tfg {

constexpr int kThreads = 1024;   // threads per vote CTA
constexpr int kRoundItems = 2 * kThreads;

enum Quant : int {
  Q_NONE = 0,   // values used as-is (gray with L=256, or quantised with L=256)
  Q_CLAMP = 1,  // already-quantised input, L<256: clamp to L-1 (validated separately)
  Q_SHIFT = 2,  // gray input, L = 2^k: q = v >> (8-k)       == (v*L)>>8
  Q_MUL = 3     // gray input, any L:   q = (v*L) >> 8       (image.hpp:55-62)
};

enum Strat : int {
  S_COPIES32 = 1,  // 32 u32 copies, interleaved [cell][lane]: bank = lane, conflict-free
  S_COPIES8 = 2,   // 8 u32 copies interleaved [cell][lane%8]
  S_COPY1 = 3,     // one u32 copy
  S_PACKED16 = 4   // one copy of u16 counters, two per word, exact spill at 2^15
};

struct VoteParams {
  const uint8_t* img;               // band 0, 16-byte aligned
  unsigned long long band_stride;   // bytes between bands
  unsigned long long pitch;         // bytes per row, multiple of 16
  int levels;
  int dr;                           // row displacement (>= 0)
  int qoff;                         // 16*floor(dcol/16)
  long long ref_off;                // drow*pitch + qoff: anchor segment -> first reference segment
  int sbits;                        // 8*(dcol mod 4)
  int col_begin, col_end;           // valid anchor columns
  int ch0, nch;                     // first 16-px chunk, chunks per row
  int nrows;                        // anchor rows [0, nrows)
  long long items;                  // nrows*nch (per band)
  long long items_per_cta;
  int step_r, step_j;               // (kThreads / nch, kThreads % nch)
  uint32_t qmask;                   // Q_SHIFT / Q_CLAMP per-byte mask
  int qshift;                       // Q_SHIFT
  int hist_words;                   // shared-memory words
  unsigned long long* glcm;         // band b accumulator at glcm + b*L*L
  uint32_t* partials;               // null -> direct u64 atomics; else [band][grid][L*L]
};

// ---------------------------------------------------------------------------
// quantisation of 4 packed pixels
template <int QUANT>
__device__ __forceinline__ uint32_t quant4(uint32_t w, const VoteParams& p) {
  if constexpr (QUANT == Q_NONE) {
    return w;
  } else if constexpr (QUANT == Q_CLAMP) {
    return __vminu4(w, p.qmask);
  } else if constexpr (QUANT == Q_SHIFT) {
    return (w >> p.qshift) & p.qmask;
  } else {
    const uint32_t L = (uint32_t)p.levels;
    const uint32_t lo = (((w & 0x00FF00FFu) * L) >> 8) & 0x00FF00FFu;  // bytes 0,2
    const uint32_t hi = (((w >> 8) & 0x00FF00FFu) * L) & 0xFF00FF00u;  // bytes 1,3
    return lo | hi;
  }
}

// ---------------------------------------------------------------------------
// one vote of weight n into the privatised sub-GLCMs
template <int STRAT>
__device__ __forceinline__ void emit(uint32_t* h, uint32_t cell, uint32_t n,
                                     unsigned long long* glcm) {
  if constexpr (STRAT == S_COPIES32) {
    atomicAdd(h + cell * 32u, n);
  } else if constexpr (STRAT == S_COPIES8) {
    atomicAdd(h + cell * 8u, n);
  } else if constexpr (STRAT == S_COPY1) {
    atomicAdd(h + cell, n);
  } else {
    // cell c lives in word (c & 0x7fff), half (c >> 15).  A field never
    // wraps: every CTA round adds <= 32768 to the CTA's counters and every
    // field is < 0x8000 at a round boundary, so a field crossing 0x7fff ->
    // 0x8000 is seen by exactly one atomic (its bit 15 flips 0 -> 1), whose
    // thread moves 0x8000 votes to the global u64 cell before the barrier.
    const uint32_t sh = (cell >> 11) & 16u;
    const uint32_t inc = n << sh;
    uint32_t* w = h + (cell & 0x7fffu);
    const uint32_t old = atomicAdd(w, inc);
    if ((~old & (old + inc)) & 0x80008000u) {
      atomicAdd(w, 0u - (0x8000u << sh));
      atomicAdd(glcm + cell, 0x8000ull);
    }
  }
}

// E[i] holds the cells of pixels 4i, 4i+2 (u16 lanes); O[i] of 4i+1, 4i+3.
template <int STRAT>
__device__ __forceinline__ void vote16(uint32_t* h, const uint32_t (&E)[4], const uint32_t (&O)[4],
                                       uint32_t mask, unsigned long long* glcm) {
  if (mask == 0xFFFFu) {
    // run-length shortcut: a segment whose 16 pairs are identical (smooth
    // inputs: 95-99.7% of neighbouring pairs repeat) casts ONE
    // vote of weight 16 instead of 16 colliding atomics.
    const uint32_t c0 = E[0] & 0xFFFFu;
    const uint32_t bc = c0 | (c0 << 16);
    const uint32_t diff = ((E[0] ^ bc) | (O[0] ^ bc)) | ((E[1] ^ bc) | (O[1] ^ bc)) |
                          ((E[2] ^ bc) | (O[2] ^ bc)) | ((E[3] ^ bc) | (O[3] ^ bc));
    if (diff == 0) {
      emit<STRAT>(h, c0, 16u, glcm);
      return;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      emit<STRAT>(h, E[i] & 0xFFFFu, 1u, glcm);
      emit<STRAT>(h, O[i] & 0xFFFFu, 1u, glcm);
      emit<STRAT>(h, E[i] >> 16, 1u, glcm);
      emit<STRAT>(h, O[i] >> 16, 1u, glcm);
    }
  } else if (mask) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (mask & (1u << (4 * i + 0))) emit<STRAT>(h, E[i] & 0xFFFFu, 1u, glcm);
      if (mask & (1u << (4 * i + 1))) emit<STRAT>(h, O[i] & 0xFFFFu, 1u, glcm);
      if (mask & (1u << (4 * i + 2))) emit<STRAT>(h, E[i] >> 16, 1u, glcm);
      if (mask & (1u << (4 * i + 3))) emit<STRAT>(h, O[i] >> 16, 1u, glcm);
    }
  }
}

__device__ __forceinline__ uint4 ldg16(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// The three 16-byte loads of one item (anchor segment + the two aligned
// segments that contain its reference bytes) and its valid-anchor mask.
struct RawItem {
  uint4 a, c0, c1;
  uint32_t mask;
};

// Issues the loads of item (row, j). Interior segments (0 < j < nch-1) need no
// bounds logic: every reference byte of an interior segment lies inside the
// row, so only the two edge segments of a row pay for masks.
template <int KSEL>
__device__ __forceinline__ void issue_item(const VoteParams& p, const uint8_t* band, long long row, int j,
                                           bool live, RawItem& it) {
  it.a = it.c0 = it.c1 = make_uint4(0, 0, 0, 0);
  it.mask = 0;
  if (!live) return;
  const int col0 = (p.ch0 + j) << 4;
  const uint8_t* ap = band + (unsigned long long)row * p.pitch + col0;
  const uint8_t* rp = ap + p.ref_off;
  it.a = ldg16(ap);
  if (j > 0 && j < p.nch - 1) {
    it.mask = 0xFFFFu;
    it.c0 = ldg16(rp);
    if constexpr (KSEL != 4) it.c1 = ldg16(rp + 16);
    return;
  }
  const int lo = p.col_begin - col0;
  const int hi = p.col_end - col0;
  uint32_t m = 0xFFFFu;
  if (lo > 0) m &= 0xFFFFu << lo;
  if (hi < 16) m &= (1u << hi) - 1u;
  it.mask = m;
  const long long cs = (long long)col0 + p.qoff;
  const long long pitch = (long long)p.pitch;
  if (cs >= 0 && cs < pitch) it.c0 = ldg16(rp);
  if constexpr (KSEL != 4) {
    if (cs + 16 >= 0 && cs + 16 < pitch) it.c1 = ldg16(rp + 16);
  }
}

// Reference bytes R[0..3] of an item: bytes [4k+s, 4k+s+16) of c0:c1.
template <int KSEL>
__device__ __forceinline__ void ref_words(const VoteParams& p, const RawItem& it, uint32_t (&A)[4],
                                          uint32_t (&R)[4]) {
  A[0] = it.a.x; A[1] = it.a.y; A[2] = it.a.z; A[3] = it.a.w;
  if constexpr (KSEL == 4) {
    R[0] = it.c0.x; R[1] = it.c0.y; R[2] = it.c0.z; R[3] = it.c0.w;
  } else {
    const uint32_t W[8] = {it.c0.x, it.c0.y, it.c0.z, it.c0.w, it.c1.x, it.c1.y, it.c1.z, it.c1.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) R[i] = __funnelshift_r(W[i + KSEL], W[i + KSEL + 1], p.sbits);
  }
}

template <int QUANT, int STRAT>
__device__ __forceinline__ void cells_of(const VoteParams& p, const uint32_t (&A)[4],
                                         const uint32_t (&R)[4], uint32_t (&E)[4], uint32_t (&O)[4]) {
  const uint32_t L = (uint32_t)p.levels;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = quant4<QUANT>(A[i], p);
    const uint32_t b = quant4<QUANT>(R[i], p);
    // u16 lanes: cell = ref*L + anchor (< 65536 for L <= 256, no lane carry)
    E[i] = (a & 0x00FF00FFu) + (b & 0x00FF00FFu) * L;
    O[i] = ((a >> 8) & 0x00FF00FFu) + ((b >> 8) & 0x00FF00FFu) * L;
  }
}

// ---------------------------------------------------------------------------
// K1 + K2: fused quantise, vote, privatised merge.
// Each thread walks items tid, tid+1024, ... of its CTA's contiguous item
// range, with the NEXT item's loads in flight while the current one votes.
template <int QUANT, int STRAT, int KSEL>
__global__ void __launch_bounds__(kThreads, 1) glcm_vote_kernel(const VoteParams p) {
  extern __shared__ __align__(16) uint32_t hist[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int band_idx = blockIdx.y;
  const uint8_t* band = p.img + (unsigned long long)band_idx * p.band_stride;
  const int cells = p.levels * p.levels;
  unsigned long long* glcm = p.glcm + (size_t)band_idx * cells;

  {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    const int n4 = p.hist_words >> 2;
    for (int i = tid; i < n4; i += kThreads) h4[i] = make_uint4(0, 0, 0, 0);
  }

  uint32_t* h = hist;
  if constexpr (STRAT == S_COPIES32) h += lane;
  if constexpr (STRAT == S_COPIES8) h += (lane & 7);

  const long long start = (long long)blockIdx.x * p.items_per_cta;
  long long end = start + p.items_per_cta;
  if (end > p.items) end = p.items;

  long long row = 0;
  int j = 0;
  RawItem nxt;
  if (start < end) {
    const long long item = start + tid;
    row = item / p.nch;
    j = (int)(item - row * p.nch);
    issue_item<KSEL>(p, band, row, j, item < end, nxt);
  }
  __syncthreads();  // histogram zeroed

  int it = 0;
  for (long long base = start; base < end; base += kThreads, ++it) {
    const RawItem cur = nxt;
    row += p.step_r;
    j += p.step_j;
    if (j >= p.nch) { j -= p.nch; ++row; }
    issue_item<KSEL>(p, band, row, j, base + kThreads + tid < end, nxt);  // prefetch
    uint32_t A[4], R[4], E[4], O[4];
    ref_words<KSEL>(p, cur, A, R);
    cells_of<QUANT, STRAT>(p, A, R, E, O);
    vote16<STRAT>(h, E, O, cur.mask, glcm);
    // PACKED16: <= 2 x 16384 votes per CTA between barriers (spill invariant)
    if constexpr (STRAT == S_PACKED16) {
      if (it & 1) __syncthreads();
    }
  }
  __syncthreads();

  // K2 epilogue: merge the copies of each cell, then one global update per cell.
  uint32_t* part = p.partials
                       ? p.partials + ((size_t)band_idx * gridDim.x + blockIdx.x) * (size_t)cells
                       : nullptr;
  if constexpr (STRAT == S_PACKED16) {
    const int words = p.hist_words;
    for (int w = tid; w < words; w += kThreads) {
      const uint32_t v = hist[w];
      const int c_lo = w, c_hi = w + 32768;
      if (c_lo < cells) {
        const uint32_t s = v & 0xFFFFu;
        if (part) part[c_lo] = s;
        else if (s) atomicAdd(glcm + c_lo, (unsigned long long)s);
      }
      if (c_hi < cells) {
        const uint32_t s = v >> 16;
        if (part) part[c_hi] = s;
        else if (s) atomicAdd(glcm + c_hi, (unsigned long long)s);
      }
    }
  } else {
    constexpr int R = STRAT == S_COPIES32 ? 32 : (STRAT == S_COPIES8 ? 8 : 1);
    for (int c = tid; c < cells; c += kThreads) {
      uint32_t s = 0;
#pragma unroll 8
      for (int k = 0; k < R; ++k) s += hist[c * R + ((k + lane) & (R - 1))];
      if (part) part[c] = s;
      else if (s) atomicAdd(glcm + c, (unsigned long long)s);
    }
  }
}

// Sum of per-CTA partial sub-GLCMs into the u64 accumulator (large L).
__global__ void glcm_reduce_partials_kernel(const uint32_t* __restrict__ partials, int nparts,
                                            int cells, int nbands,
                                            unsigned long long* __restrict__ glcm) {
  const long long total = (long long)cells * nbands;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long band = i / cells;
    const long long c = i - band * cells;
    const uint32_t* src = partials + band * (long long)nparts * cells + c;
    unsigned long long s = 0;
    for (int g = 0; g < nparts; ++g) s += src[(long long)g * cells];
    glcm[i] += s;
  }
}

// K0: Scheme 1, one global atomic per pixel pair (ablation baseline).
template <int QUANT, int KSEL>
__global__ void glcm_vote_global_kernel(const VoteParams p) {
  const int band_idx = blockIdx.y;
  const uint8_t* band = p.img + (unsigned long long)band_idx * p.band_stride;
  unsigned long long* glcm = p.glcm + (size_t)band_idx * p.levels * p.levels;
  for (long long item = blockIdx.x * (long long)blockDim.x + threadIdx.x; item < p.items;
       item += (long long)gridDim.x * blockDim.x) {
    const long long row = item / p.nch;
    const int j = (int)(item - row * p.nch);
    RawItem ri;
    issue_item<KSEL>(p, band, row, j, true, ri);
    uint32_t A[4], R[4], E[4], O[4];
    ref_words<KSEL>(p, ri, A, R);
    cells_of<QUANT, S_COPY1>(p, A, R, E, O);
    const uint32_t m = ri.mask;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (m & (1u << (4 * i + 0))) atomicAdd(glcm + (E[i] & 0xFFFFu), 1ull);
      if (m & (1u << (4 * i + 1))) atomicAdd(glcm + (O[i] & 0xFFFFu), 1ull);
      if (m & (1u << (4 * i + 2))) atomicAdd(glcm + (E[i] >> 16), 1ull);
      if (m & (1u << (4 * i + 3))) atomicAdd(glcm + (O[i] >> 16), 1ull);
    }
  }
}

// Validation of an already-quantised raster (QuantizedImage ctor, image.hpp:46-48).
__global__ void validate_levels_kernel(const uint8_t* img, unsigned long long pitch, int width,
                                       long long rows, unsigned long long band_stride, int levels,
                                       int* err) {
  const int band_idx = blockIdx.y;
  const uint8_t* band = img + (unsigned long long)band_idx * band_stride;
  const int nch = (width + 15) / 16;
  const uint32_t maxv = (uint32_t)(levels - 1) * 0x01010101u;
  uint32_t bad = 0;
  for (long long item = blockIdx.x * (long long)blockDim.x + threadIdx.x; item < rows * nch;
       item += (long long)gridDim.x * blockDim.x) {
    const long long row = item / nch;
    const int j = (int)(item - row * nch);
    const uint4 v = ldg16(band + row * pitch + 16 * j);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const int valid = width - 16 * j;  // bytes of this segment inside the row
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t gt = __vcmpgtu4(w[i], maxv);
      const int vb = valid - 4 * i;
      if (vb <= 0) gt = 0;
      else if (vb < 4) gt &= (1u << (8 * vb)) - 1u;
      bad |= gt;
    }
  }
  if (__any_sync(0xffffffffu, bad != 0) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

// Quantise kernel (standalone texforge::quantize, image.hpp:55-62).
__global__ void quantize_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                long long n, int levels) {
  const long long n16 = n / 16;
  const uint32_t L = (uint32_t)levels;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16;
       i += (long long)gridDim.x * blockDim.x) {
    uint4 v = reinterpret_cast<const uint4*>(in)[i];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lo = (((w[k] & 0x00FF00FFu) * L) >> 8) & 0x00FF00FFu;
      const uint32_t hi = (((w[k] >> 8) & 0x00FF00FFu) * L) & 0xFF00FF00u;
      w[k] = lo | hi;
    }
    reinterpret_cast<uint4*>(out)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  const long long tail = n16 * 16;
  const long long t = tail + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && t < n) out[t] = (uint8_t)(((uint32_t)in[t] * L) >> 8);
}

// ---------------------------------------------------------------------------
// K3: symmetrize (glcm.hpp:150-156), batched over gridDim.y GLCMs.
__global__ void symmetrize_kernel(const unsigned long long* __restrict__ in, int L,
                                  unsigned long long* __restrict__ out) {
  const size_t cells = (size_t)L * L;
  const unsigned long long* g = in + blockIdx.y * cells;
  unsigned long long* o = out + blockIdx.y * cells;
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < cells;
       c += (size_t)gridDim.x * blockDim.x) {
    const size_t i = c / L, j = c - i * L;
    o[c] = g[c] + g[j * L + i];
  }
}

template <typename T, int NT>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  // deterministic fixed-order tree: warp shuffle, then warp 0 over warp sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < NT / 32 ? scratch[lane] : T(0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) scratch[0] = v;
  }
  __syncthreads();
  return scratch[0];
}

// K3: normalize (glcm.hpp:167-177): inv = 1.0/total, p = (double)c * inv,
// the identical IEEE op sequence -> bit-exact with the reference.
// One CTA per GLCM; err[blockIdx.x] = 1 on an all-zero matrix.
__global__ void __launch_bounds__(1024) normalize_kernel(const unsigned long long* __restrict__ in,
                                                         int L, double* __restrict__ out, int* err) {
  __shared__ unsigned long long scratch[32];
  const size_t cells = (size_t)L * L;
  const unsigned long long* g = in + blockIdx.x * cells;
  double* o = out + blockIdx.x * cells;
  unsigned long long t = 0;
  for (size_t c = threadIdx.x; c < cells; c += blockDim.x) t += g[c];
  const unsigned long long total = block_sum<unsigned long long, 1024>(t, scratch);
  if (total == 0) {
    if (threadIdx.x == 0 && err) err[blockIdx.x] = 1;
    return;
  }
  const double inv = __ddiv_rn(1.0, __ull2double_rn(total));
  for (size_t c = threadIdx.x; c < cells; c += blockDim.x) o[c] = __dmul_rn(__ull2double_rn(g[c]), inv);
}

// K4: Haralick-5 (features.hpp:37-69) on a normalised GLCM; one CTA per GLCM.
// Sums run in a fixed parallel order, so results differ from the reference's
// sequential sums by ulps only (tolerance stated in tests: 1e-10).
__global__ void __launch_bounds__(1024) features_kernel(const double* __restrict__ probs, int L,
                                                        double* __restrict__ out5, int* err) {
  __shared__ double scratch[32];
  const size_t cells = (size_t)L * L;
  const double* P = probs + blockIdx.x * cells;
  // normalisation check: compensated per-thread sums, then a fixed tree.
  double s = 0.0, comp = 0.0;
  for (size_t c = threadIdx.x; c < cells; c += blockDim.x) {
    const double y = P[c] - comp;
    const double t = s + y;
    comp = (t - s) - y;
    s = t;
  }
  const double total = block_sum<double, 1024>(s, scratch);
  if (fabs(total - 1.0) > 1e-12) {
    if (threadIdx.x == 0) {
      if (err) err[blockIdx.x] = 1;
      for (int k = 0; k < 5; ++k) out5[blockIdx.x * 5 + k] = __longlong_as_double(0x7ff8000000000000ll);
    }
    return;
  }
  double energy = 0, contrast = 0, homog = 0, entropy = 0, mi = 0, mj = 0, cross = 0;
  for (size_t c = threadIdx.x; c < cells; c += blockDim.x) {
    const int i = (int)(c / L), j = (int)(c - (size_t)i * L);
    const double v = P[c];
    const double diff = (double)(i - j);
    energy += v * v;
    contrast += diff * diff * v;
    homog += v / (1.0 + diff * diff);
    if (v > 0.0) entropy -= v * log2(v);
    mi += i * v;
    mj += j * v;
    cross += (double)i * j * v;
  }
  energy = block_sum<double, 1024>(energy, scratch);
  contrast = block_sum<double, 1024>(contrast, scratch);
  homog = block_sum<double, 1024>(homog, scratch);
  entropy = block_sum<double, 1024>(entropy, scratch);
  mi = block_sum<double, 1024>(mi, scratch);
  mj = block_sum<double, 1024>(mj, scratch);
  cross = block_sum<double, 1024>(cross, scratch);
  double vi = 0, vj = 0;
  for (size_t c = threadIdx.x; c < cells; c += blockDim.x) {
    const int i = (int)(c / L), j = (int)(c - (size_t)i * L);
    const double v = P[c];
    vi += (i - mi) * (i - mi) * v;
    vj += (j - mj) * (j - mj) * v;
  }
  vi = block_sum<double, 1024>(vi, scratch);
  vj = block_sum<double, 1024>(vj, scratch);
  if (threadIdx.x == 0) {
    const double sigma = sqrt(vi) * sqrt(vj);
    double* o = out5 + blockIdx.x * 5;
    o[0] = energy;
    o[1] = contrast;
    o[2] = homog;
    o[3] = entropy;
    o[4] = sigma > 0.0 ? (cross - mi * mj) / sigma : 0.0;
  }
}

}  // namespace tfg
