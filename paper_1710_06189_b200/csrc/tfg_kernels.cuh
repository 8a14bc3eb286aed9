// tfg_kernels.cuh — sm_100a device code of the B200 GLCM engine.
//
// K1 glcm_vote_kernel: fused quantise + pixel-pair vote + privatised
//    shared-memory sub-GLCMs (the paper's "copies", re-sized
//    for 227 KB/CTA) + in-kernel merge (K2).  Semantics follow
//    R/include/texforge/glcm.hpp:110-130 (vote_anchor_rows) exactly:
//    anchors in rows [0, min(row_end, H - drow)), columns
//    [d*[dcol<0], W - d*[dcol>0]), cell = ref*L + anchor.
// K1J glcm_vote_jobs_kernel: up to 8 (L, d, theta) jobs of one image or band
//    batch in one launch (layouts without per-CTA partials, L <= 64); the
//    same vote_cta body, the reference-window variant picked per CTA.
// K0 glcm_vote_global_kernel: Scheme 1 (one global atomic per pair,
//    PAPER.md:62-93 / parallel.hpp:121-152) — ablation only.
// K3 symmetrize / normalize, K4 features — post-processing on device.
//
// Work decomposition: the valid-anchor raster is cut into
// 16-pixel "items" (one 16-byte vector per row segment). A main pass votes the
// interior segments of every row in double batches of 64 consecutive items
// (lanes l and l+32; every LDG.128 of the warp is one coalesced 512-byte
// access), four per grab from a per-CTA ticket counter and then, when the
// launch is cooperative, from the band's shared tail pool; two double batches
// sit in a register ring (one for the PACKED16 variants with two reference
// segments). An edge pass votes the row ends with masks. The reference
// neighbour of each segment is one or two aligned 16-byte loads + funnel
// shifts (displacement dcol = 16q + 4k + s: q and the word shift k are launch
// / template constants, s is a byte funnel shift); a window's one narrow word
// comes from the adjacent lane by shuffle where the L1 data pipe binds
// (nbr_fix). Interior segments start on 128-byte lines when the rows do.
//
// The vote itself is 3 instructions for L <= 128: the quantised anchor and
// reference bytes are pre-scaled so that ONE byte permute (PRMT) of an anchor
// word and a reference word gives a pixel pair's shared-memory offset, then
// one IMAD adds the lane's copy base and one red.shared.add (ATOMS.POPC.INC)
// casts the vote; 5 for the packed-u16 L=256 layout (packed_inc, kPackedDrainBit).
//
// Measured A/B variants kept behind flags: TFG_TMA (TMA-staged
// main pass), S_P16X16 (16 bank-pair copies for L <= 64), TFG_LDG_MODE
// (L2-only loads), TFG_THREADS (CTA size).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tfg {

#ifndef TFG_THREADS
#define TFG_THREADS 1024
#endif
#ifndef TFG_TMA
#define TFG_TMA 0
#endif
constexpr int kThreads = TFG_THREADS;  // threads per vote CTA (32 warps)
// TFG_TMA: per-warp shared stages of the staged main pass behind the histogram
// (2 stages x anchors + reference window, 2 mbarriers per warp)
constexpr size_t kTmaBytes = TFG_TMA ? (size_t)(kThreads / 32) * (2 * 2 * (32 * 16 + 32) + 16) : 0;

enum Quant : int {
  Q_NONE = 0,   // values used as-is (gray with L=256, or quantised with L=256)
  Q_CLAMP = 1,  // already-quantised input, L<256: clamp to L-1 (validated separately)
  Q_SHIFT = 2,  // gray input, L = 2^k: q = v >> (8-k)       == (v*L)>>8
  Q_MUL = 3     // gray input, any L:   q = (v*L) >> 8       (image.hpp:55-62)
};

// Privatised sub-GLCM layouts. x = PRMT(P, Q) = P_byte + 256*Q_byte per pixel.
enum Strat : int {
  S_COPIES32 = 1,  // L <= 32:  32 u32 copies [a + 32b][lane]; P = 8a, Q = b, addr = 16x + 4 lane
  S_COPIES8 = 2,   // L <= 64:  8 u32 copies [b + 64a][lane%8]; P = 4b, Q = a, addr = 8x + 4 (lane%8)
  S_COPY1 = 3,     // L <= 128: 1 u32 copy [a + 128b]; P = 2a, Q = b, addr = 2x
  S_P16X16 = 5,    // L <= 64: 16 copies of u16 counters, copy = lane & 15 owning banks 2k, 2k+1 (p16x16_*)
  S_PACKED16 = 4   // L <= 256: 1 copy of u16 counters, cell a + 256b in word (x & 0x7fff), half b >> 7
                   //           (word = N - 65536 n_hi, packed_inc), drained past 2^15 (kPackedDrainBit)
};

__host__ __device__ constexpr int strat_scale(int s) {  // log2 of the P-byte scale
  return s == S_COPIES32 ? 3 : (s == S_COPIES8 ? 2 : (s == S_COPY1 ? 1 : 0));
}
__host__ __device__ constexpr int strat_copies(int s) {
  return s == S_COPIES32 ? 32 : (s == S_COPIES8 ? 8 : 1);
}

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
  uint32_t div_mul, div_shr;        // fast division by nch (div_mul == 0: nch == 1)
  uint32_t qmask;                   // Q_SHIFT / Q_CLAMP per-byte mask (L-1)*0x01010101
  int qshift;                       // Q_SHIFT: s = 8 - log2 L
  int qshift_scaled;                // Q_SHIFT: s - strat_scale
  int rshift;                       // Q_SHIFT: sbits + the reference side's quantisation shift (item_words)
  uint32_t rmask;                   // Q_SHIFT: the reference side's byte mask
  int hist_words;                   // shared-memory words
  unsigned long long* glcm;         // band b accumulator at glcm + b*L*L
  uint32_t* partials;               // null -> direct u64 atomics; else [band][grid][L*L]
  unsigned long long buf_bytes;     // bytes of one band buffer (rows * pitch): prefetch clamp
  // two-pass decomposition (glcm_vote_kernel): interior segments j in [1, nch-1)
  // of every anchor row (main pass, no masks) and the rest (edge pass)
  int ni;                           // interior segments per row (0: everything is edge work)
  int js;                           // first interior segment (>= 1; 128-B aligned when the rows are)
  uint32_t ni_mul, ni_shr;          // fast division by ni
  long long main_items;             // nrows * ni
  long long main_per_cta;           // multiple of 64; CTA ranges tile [0, pool_beg)
  // shared tail pool (cooperative launches): interior items [pool_beg, main_items)
  // = pool_dbl double batches handed to any CTA of the band from pool_ctr[band]
  long long pool_beg;               // == main_items: no pool
  uint32_t pool_dbl;
  unsigned int* pool_ctr;           // zeroed before the launch; null: no pool
  int ne;                       // edge segments per row (2, or nch when ni == 0)
  uint32_t ne_mul, ne_shr;          // fast division by ne
  long long edge_items;             // nrows * ne
  long long edge_per_cta;
  unsigned int* sync_ctr;           // non-null: cooperative launch, in-kernel partial reduction
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

// Quantised bytes of 4 pixels, times 2^sc (bytes stay < 256: no byte carry).
template <int QUANT, int SC>
__device__ __forceinline__ uint32_t quant4_scaled(uint32_t w, const VoteParams& p) {
  if constexpr (SC == 0) {
    return quant4<QUANT>(w, p);
  } else if constexpr (QUANT == Q_SHIFT) {
    return (w >> p.qshift_scaled) & (p.qmask << SC);  // ((w >> s) & m) << sc in two ops
  } else {
    return quant4<QUANT>(w, p) << SC;
  }
}

// P/Q words of an item: PRMT(P[i], Q[i]) byte j = offset of pixel 4i+j.
template <int QUANT, int STRAT>
__device__ __forceinline__ void prep_words(const VoteParams& p, const uint32_t (&A)[4], const uint32_t (&R)[4],
                                           uint32_t (&P)[4], uint32_t (&Q)[4]) {
  constexpr int sc = strat_scale(STRAT);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (STRAT == S_COPIES8) {  // reference side scaled, anchor-major cells
      P[i] = quant4_scaled<QUANT, sc>(R[i], p);
      Q[i] = quant4<QUANT>(A[i], p);
    } else {
      P[i] = quant4_scaled<QUANT, sc>(A[i], p);
      Q[i] = quant4<QUANT>(R[i], p);
    }
  }
}

// PTX prmt, generic mode: selector nibble bits 2:0 pick a byte of {b, a},
// bit 3 replicates that byte's sign (the __byte_perm intrinsic ignores bit 3).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// byte j of P in bits 0-7, byte j of Q in bits 8-15, bits 16-31 = sign of Q
// byte 0 (zero: every Q byte of a non-packed layout is < 128).
__device__ __forceinline__ uint32_t pair_x(uint32_t P, uint32_t Q, int j) {
  return prmt(P, Q, 0xCC00u | ((4u + j) << 4) | (uint32_t)j);
}

// ---------------------------------------------------------------------------
// shared-memory votes on 32-bit shared addresses
__device__ __forceinline__ void red_smem(uint32_t addr, uint32_t n) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(n) : "memory");
}
__device__ __forceinline__ void red_smem1(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}
__device__ __forceinline__ uint32_t atom_smem(uint32_t addr, uint32_t n) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(n) : "memory");
  return old;
}

template <int STRAT>
__device__ __forceinline__ uint32_t vote_addr(uint32_t hb, uint32_t x) {
  if constexpr (STRAT == S_COPIES32) return x * 16u + hb;
  else if constexpr (STRAT == S_COPIES8) return x * 8u + hb;
  else if constexpr (STRAT == S_COPY1) return x * 2u + hb;
  else return (x & 0x7fffu) * 4u + hb;
}

#ifndef TFG_PACKED_NEG
#define TFG_PACKED_NEG 1
#endif
// PACKED16 increment for pixel j of word Q (b = reference byte).
// TFG_PACKED_NEG (default): ONE PRMT builds 1 (b < 128) or 0xFFFF0001
// (b >= 128; byte 0 from the constant 1, bytes 2-3 the sign of b), so a word
// holds N - 65536 n_hi: low half = N = all votes of its two cells, high half
// = -n_hi mod 2^16 (packed_decode). Otherwise: 1 or 0x10000 (PRMT + add).
__device__ __forceinline__ uint32_t packed_inc(uint32_t Q, int j) {
#if TFG_PACKED_NEG
  return prmt(Q, 1u, 0x0054u | ((8u + j) << 8) | ((8u + j) << 12));
#else
  return prmt(Q, 0u, 0x4400u | ((8u + j) << 4) | (8u + j)) + 1u;
#endif
}
// a PACKED16 word as (n_lo | n_hi << 16)
__device__ __forceinline__ uint32_t packed_decode(uint32_t w) {
#if TFG_PACKED_NEG
  const uint32_t nhi = (0u - (w >> 16)) & 0xFFFFu;
  return ((w & 0xFFFFu) - nhi) | (nhi << 16);
#else
  return w;
#endif
}

// PACKED16 overflow rule (exact, no barriers, no per-vote ownership test).
// Every PACKED16 vote is a returning atomic and its thread ORs the returned
// word into a per-item flag. When a field has reached 2^15 (bit 15 of either
// half set) the thread DRAINS every word it voted in that item: one
// atomicAnd(word, 0x07FF07FF) takes ownership of all whole multiples of 2048
// in both halves at once, and those counts go to the u64 cells. Because the
// AND is atomic, every count is moved exactly once no matter how many
// threads drain the same word. Bound: once a field passes 2^15, every warp
// that votes on it sees bit 15 and drains before its next item, and a warp
// adds <= 512 to one field per item (32 lanes x 16), so before the first
// drain lands the field stays < 2^15 + 32 * 512 + 512 < 2^16.
// TFG_PACKED_NEG: the low half counts both cells, so it alone carries the
// drain bit, and a drain takes the whole word (atom.exch 0) and decodes it;
// the bound is the same (N < 2^15 + 33 * 512).
constexpr uint32_t kDrainBit = 0x80008000u;
constexpr uint32_t kPackedDrainBit = TFG_PACKED_NEG ? 0x00008000u : 0x80008000u;
static_assert(32768u + (kThreads / 32 + 1) * 512u < 65536u, "PACKED16 field bound");

// Drains one PACKED16 word whose cell is x = a + 256 b (b's top bit selects
// the half; the word holds cells (a, b&127) and (a, (b&127)+128)).
__device__ __forceinline__ void packed_drain(uint32_t addr, uint32_t x, unsigned long long* glcm, uint32_t L) {
  uint32_t old;
  const uint32_t a = x & 0xFFu, b = (x >> 8) & 0x7Fu;
#if TFG_PACKED_NEG
  asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(0u) : "memory");
  const uint32_t dec = packed_decode(old);
  const uint32_t lo = dec & 0xFFFFu, hi = dec >> 16;
#else
  asm volatile("atom.shared.and.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(0x07FF07FFu) : "memory");
  const uint32_t lo = old & 0xF800u, hi = (old >> 16) & 0xF800u;
#endif
  if (lo) atomicAdd(glcm + b * L + a, (unsigned long long)lo);
  if (hi) atomicAdd(glcm + (b + 128u) * L + a, (unsigned long long)hi);
}

// Rare path, out of line so the hot loop fits the instruction cache: drain
// the words of the pixels in `mask` of one item.
static __device__ __noinline__ void packed_drain_item(uint32_t hb, uint32_t P0, uint32_t P1, uint32_t P2, uint32_t P3,
                                               uint32_t Q0, uint32_t Q1, uint32_t Q2, uint32_t Q3, uint32_t mask,
                                               unsigned long long* glcm, uint32_t L) {
  const uint32_t P[4] = {P0, P1, P2, P3}, Q[4] = {Q0, Q1, Q2, Q3};
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (mask & (1u << k)) {
      const uint32_t x = pair_x(P[k >> 2], Q[k >> 2], k & 3);
      packed_drain(vote_addr<S_PACKED16>(hb, x), x, glcm, L);
    }
  }
}

// One vote of weight n; returns the old word for PACKED16 (else 0).
template <int STRAT>
__device__ __forceinline__ uint32_t emit(uint32_t hb, uint32_t P, uint32_t Q, int j, uint32_t n) {
  const uint32_t addr = vote_addr<STRAT>(hb, pair_x(P, Q, j));
  if constexpr (STRAT == S_PACKED16) {
    return atom_smem(addr, packed_inc(Q, j) * n);
  } else {
    red_smem(addr, n);
    return 0u;
  }
}

// Edge segments of a row: only the anchors in `mask` vote.
template <int STRAT>
__device__ __noinline__ void vote_masked(uint32_t hb, uint32_t P0, uint32_t P1, uint32_t P2, uint32_t P3,
                                         uint32_t Q0, uint32_t Q1, uint32_t Q2, uint32_t Q3, uint32_t mask,
                                         unsigned long long* glcm, uint32_t L) {
  const uint32_t P[4] = {P0, P1, P2, P3}, Q[4] = {Q0, Q1, Q2, Q3};
  uint32_t flag = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (mask & (1u << k)) flag |= emit<STRAT>(hb, P[k >> 2], Q[k >> 2], k & 3, 1u);
  if constexpr (STRAT == S_PACKED16) {
    if (flag & kPackedDrainBit) packed_drain_item(hb, P0, P1, P2, P3, Q0, Q1, Q2, Q3, mask, glcm, L);
  }
}

// The 16 PACKED16 votes of an unmasked item (returning atomics, then the
// drain rule of kPackedDrainBit). Reference bytes with the half bit cleared: PRMT
// then yields the word index a + 256 (b & 127) directly (no per-vote mask).
__device__ __forceinline__ void packed_vote16(uint32_t hb, const uint32_t (&P)[4], const uint32_t (&Q)[4],
                                              unsigned long long* glcm, uint32_t L) {
  uint32_t flag = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t Qm = Q[i] & 0x7F7F7F7Fu;
#pragma unroll
    for (int j = 0; j < 4; ++j) flag |= atom_smem(hb + pair_x(P[i], Qm, j) * 4u, packed_inc(Q[i], j));
  }
  if (flag & kPackedDrainBit) packed_drain_item(hb, P[0], P[1], P[2], P[3], Q[0], Q[1], Q[2], Q[3], 0xFFFFu, glcm, L);
}

// ---- S_P16X16 (L <= 64): 16 copies of packed u16 counters. Lanes l and
// l+16 share copy k = l & 15, which owns banks 2k and 2k+1, so an ATOMS costs
// ~2 wavefronts instead of COPIES8's 2.93 (random cells, 4 lanes per 4-bank
// group). Cell (ref b, anchor a): half = a & 1; copy k's word
// A1(a) + 256 b + 16384 (a >> 5) + 2k, with A1 = bits {(a>>1)&1 -> 0,
// (a>>2)&7 -> 5..7}: bank = ((a >> 1) & 1) + 2k, so the two lanes of a copy
// share its two banks and no other copy touches them. Per 4-pixel anchor
// word: A1, A2 = (a >> 5) & 1, Ah = (a & 1) << 7. A vote: x = PRMT(A1, B) =
// A1_j + 256 b_j; y = PRMT(A2, hb) = hb with byte 2 := a>>5 (+65536 bytes,
// the address bit a byte cannot hold next to the 4 lane bits); address =
// 4x + y; increment 1 or 0x10000 from Ah's sign; overflow exactly as
// PACKED16 (kDrainBit). Measured: 2.02 wavefronts per ATOMS (COPIES8 2.93),
// but ~2x the instructions per vote (issue-bound) and no POPC.INC
// aggregation for smooth input: slower than COPIES8.
struct P16x16Words {
  uint32_t A1[4], A2[4], Ah[4], B[4];
};
__device__ __forceinline__ void p16x16_prep(const uint32_t (&qa)[4], const uint32_t (&qb)[4], P16x16Words& w) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    w.A1[i] = ((qa[i] >> 1) & 0x01010101u) | ((qa[i] << 3) & 0xE0E0E0E0u);
    w.A2[i] = (qa[i] >> 5) & 0x01010101u;
    w.Ah[i] = (qa[i] << 7) & 0x80808080u;
    w.B[i] = qb[i];
  }
}
__device__ __forceinline__ uint32_t p16x16_addr(uint32_t hb, const P16x16Words& w, int i, int j) {
  const uint32_t x = pair_x(w.A1[i], w.B[i], j);
  const uint32_t y = prmt(w.A2[i], hb, 0x7004u | ((uint32_t)j << 8) | 0x50u);
  return x * 4u + y;
}
// drains word `addr` holding cells (b, a & ~1) [low half] and (b, a | 1) [high half]
__device__ __forceinline__ void p16x16_drain(uint32_t addr, uint32_t a, uint32_t b, unsigned long long* glcm,
                                             uint32_t L) {
  uint32_t old;
  asm volatile("atom.shared.and.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(0x07FF07FFu) : "memory");
  const uint32_t lo = old & 0xF800u, hi = (old >> 16) & 0xF800u;
  if (lo) atomicAdd(glcm + b * L + (a & ~1u), (unsigned long long)lo);
  if (hi) atomicAdd(glcm + b * L + (a | 1u), (unsigned long long)hi);
}
static __device__ __noinline__ void p16x16_drain_item(uint32_t hb, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                      uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3,
                                                      uint32_t mask, unsigned long long* glcm, uint32_t L) {
  const uint32_t a4[4] = {a0, a1, a2, a3}, b4[4] = {b0, b1, b2, b3};
  const uint32_t* qa = a4;
  const uint32_t* qb = b4;
  P16x16Words w;
  p16x16_prep(a4, b4, w);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (mask & (1u << k)) {
      const int i = k >> 2, j = k & 3;
      p16x16_drain(p16x16_addr(hb, w, i, j), (qa[i] >> (8 * j)) & 0xFFu, (qb[i] >> (8 * j)) & 0xFFu, glcm, L);
    }
  }
}
// the pairs in `mask` of one item (qa: quantised anchors, qb: quantised references)
__device__ __forceinline__ void p16x16_vote(uint32_t hb, const uint32_t (&qa)[4], const uint32_t (&qb)[4],
                                            uint32_t mask, unsigned long long* glcm, uint32_t L) {
  P16x16Words w;
  p16x16_prep(qa, qb, w);
  uint32_t flag = 0;
  if (mask == 0xFFFFu) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        flag |= atom_smem(p16x16_addr(hb, w, i, j), prmt(w.Ah[i], 0u, 0x4400u | ((8u + j) << 4) | (8u + j)) + 1u);
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int i = k >> 2, j = k & 3;
      if (mask & (1u << k))
        flag |= atom_smem(p16x16_addr(hb, w, i, j), prmt(w.Ah[i], 0u, 0x4400u | ((8u + j) << 4) | (8u + j)) + 1u);
    }
  }
  if (flag & kDrainBit)
    p16x16_drain_item(hb, qa[0], qa[1], qa[2], qa[3], qb[0], qb[1], qb[2], qb[3], mask, glcm, L);
}

// Votes the 16 pixel pairs of one item. Returns true when the run-length
// shortcut fired (all 16 pairs identical: one vote of weight 16).
template <int STRAT>
__device__ __forceinline__ bool vote16(uint32_t hb, const uint32_t (&P)[4], const uint32_t (&Q)[4],
                                       uint32_t mask, bool rle, unsigned long long* glcm, uint32_t L) {
  if (mask == 0xFFFFu) {
    if (rle) {
      // smooth inputs (95-99.7% of neighbouring pairs repeat)
      const uint32_t bp = __byte_perm(P[0], 0u, 0u), bq = __byte_perm(Q[0], 0u, 0u);
      const uint32_t diff = (P[0] ^ bp) | (P[1] ^ bp) | (P[2] ^ bp) | (P[3] ^ bp) | (Q[0] ^ bq) |
                            (Q[1] ^ bq) | (Q[2] ^ bq) | (Q[3] ^ bq);
      if (diff == 0) {
        const uint32_t old = emit<STRAT>(hb, P[0], Q[0], 0, 16u);
        if constexpr (STRAT == S_PACKED16) {
          if (old & kPackedDrainBit) packed_drain_item(hb, P[0], P[1], P[2], P[3], Q[0], Q[1], Q[2], Q[3], 1u, glcm, L);
        }
        return true;
      }
    }
    if constexpr (STRAT == S_PACKED16) {
      packed_vote16(hb, P, Q, glcm, L);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) red_smem1(vote_addr<STRAT>(hb, pair_x(P[i], Q[i], j)));
    }
  } else if (mask) {
    vote_masked<STRAT>(hb, P[0], P[1], P[2], P[3], Q[0], Q[1], Q[2], Q[3], mask, glcm, L);
  }
  return false;
}

// Layout position (in counters) of real cell (ref b, anchor a).
template <int STRAT>
__device__ __forceinline__ uint32_t cell_pos(uint32_t b, uint32_t a) {
  if constexpr (STRAT == S_COPIES32) return a + 32u * b;
  else if constexpr (STRAT == S_COPIES8) return b + 64u * a;
  else if constexpr (STRAT == S_COPY1) return a + 128u * b;
  else return a + 256u * b;
}

#ifndef TFG_LDG_MODE
#define TFG_LDG_MODE 0
#endif
__device__ __forceinline__ uint4 ldg16(const uint8_t* p) {
#if TFG_LDG_MODE == 1
  uint4 v;  // L2 only (no L1 allocation)
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
#elif TFG_LDG_MODE == 2
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
#else
  return __ldg(reinterpret_cast<const uint4*>(p));
#endif
}

// Bulk prefetch of [a, a+bytes) into L2 (cp.async.bulk.prefetch.L2, sm_90+):
// one instruction moves a whole span of image rows towards the SMs.
__device__ __forceinline__ void prefetch_l2(const void* a, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
}

// mbarrier + bulk-copy (TMA engine) helpers for the staged main pass (TFG_TMA)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TFG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TFG_WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint4 lds16(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// ---------------------------------------------------------------------------
// The three 16-byte loads of one item (anchor segment + the two aligned
// segments that contain its reference bytes) and its valid-anchor mask.
struct RawItem {
  uint4 a, c0, c1;
  uint32_t mask;
};

// KSEL: how the 16 reference bytes sit in the two aligned segments c0:c1 —
// bytes [4k+s, 4k+s+16) with k = KSEL (0..3, c0 loaded), KSEL == 4: c0 alone
// (dcol % 16 == 0), k = KSEL-5 (5..8): same as k but c0 IS the anchor
// segment (theta = 0, d < 16: one load fewer).
template <int KSEL>
__device__ __forceinline__ constexpr bool ksel_c0_is_anchor() { return KSEL >= 5; }
template <int KSEL>
__device__ __forceinline__ constexpr bool ksel_needs_c1() { return KSEL != 4; }


// Issues the loads of item (row, j). Interior segments (0 < j < nch-1) need no
// bounds logic: every reference byte of an interior segment lies inside the
// row, so only the two edge segments of a row pay for masks.
// Nothing here consumes a loaded value, so the loads stay in flight while the
// caller votes the previous batch.
template <int KSEL>
__device__ __forceinline__ void issue_item(const VoteParams& p, const uint8_t* band, uint32_t row, uint32_t j,
                                           bool live, RawItem& it) {
  // No zero-fill: bytes of a dead item or of an out-of-row reference segment
  // only ever feed masked-off anchors (mask bit 0), so they are never voted.
  it.mask = 0;
  if (!live) return;
  const uint32_t col0 = (p.ch0 + j) << 4;
  const uint8_t* ap = band + (unsigned long long)row * (uint32_t)p.pitch + col0;
  const uint8_t* rp = ap + p.ref_off;
  it.a = ldg16(ap);
  if (j > 0 && j + 1 < (uint32_t)p.nch) {
    it.mask = 0xFFFFu;
    if constexpr (!ksel_c0_is_anchor<KSEL>()) it.c0 = ldg16(rp);
    if constexpr (ksel_needs_c1<KSEL>()) it.c1 = ldg16(rp + 16);
    return;
  }
  const int lo = p.col_begin - (int)col0;
  const int hi = p.col_end - (int)col0;
  uint32_t m = 0xFFFFu;
  if (lo > 0) m &= 0xFFFFu << lo;
  if (hi < 16) m &= (1u << hi) - 1u;
  it.mask = m;
  const long long cs = (long long)col0 + p.qoff;
  const long long pitch = (long long)p.pitch;
  if constexpr (!ksel_c0_is_anchor<KSEL>()) {
    if (cs >= 0 && cs < pitch) it.c0 = ldg16(rp);
  }
  if constexpr (ksel_needs_c1<KSEL>()) {
    if (cs + 16 >= 0 && cs + 16 < pitch) it.c1 = ldg16(rp + 16);
  }
}

// Reference bytes R[0..3] of an item.
template <int KSEL>
__device__ __forceinline__ void ref_words(const VoteParams& p, const RawItem& it, uint32_t (&A)[4],
                                          uint32_t (&R)[4]) {
  A[0] = it.a.x; A[1] = it.a.y; A[2] = it.a.z; A[3] = it.a.w;
  const uint4 c0 = ksel_c0_is_anchor<KSEL>() ? it.a : it.c0;
  if constexpr (KSEL == 4) {
    R[0] = c0.x; R[1] = c0.y; R[2] = c0.z; R[3] = c0.w;
  } else {
    constexpr int k = KSEL >= 5 ? KSEL - 5 : KSEL;
    const uint32_t W[8] = {c0.x, c0.y, c0.z, c0.w, it.c1.x, it.c1.y, it.c1.z, it.c1.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) R[i] = __funnelshift_r(W[i + k], W[i + k + 1], p.sbits);
  }
}

// P/Q words of an item with the reference side's power-of-two quantisation
// folded into its funnel shift: (funnel(lo, hi, sbits) >> t) & M ==
// funnel(lo, hi, sbits + t) & M, because the bits the wider shift pulls in
// from the next byte land above the mask (sbits + t <= 31). Saves one shift
// per word; other quantisers and the aligned case (KSEL 4) use the plain path.
template <int QUANT, int STRAT, int KSEL>
__device__ __forceinline__ void item_words(const VoteParams& p, const RawItem& it, uint32_t (&P)[4],
                                           uint32_t (&Q)[4]) {
  if constexpr (QUANT == Q_SHIFT && KSEL != 4) {
    constexpr int sc = strat_scale(STRAT);
    const uint4 c0 = ksel_c0_is_anchor<KSEL>() ? it.a : it.c0;
    constexpr int k = KSEL >= 5 ? KSEL - 5 : KSEL;
    const uint32_t W[8] = {c0.x, c0.y, c0.z, c0.w, it.c1.x, it.c1.y, it.c1.z, it.c1.w};
    const uint32_t A[4] = {it.a.x, it.a.y, it.a.z, it.a.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t rq = __funnelshift_r(W[i + k], W[i + k + 1], p.rshift) & p.rmask;
      if constexpr (STRAT == S_COPIES8) {  // reference side scaled, anchor-major cells
        P[i] = rq;
        Q[i] = quant4<QUANT>(A[i], p);
      } else {
        P[i] = quant4_scaled<QUANT, sc>(A[i], p);
        Q[i] = rq;
      }
    }
  } else {
    uint32_t A[4], R[4];
    ref_words<KSEL>(p, it, A, R);
    prep_words<QUANT, STRAT>(p, A, R, P, Q);
  }
}

// Generic cell words for Scheme 1: u16 lanes cell = ref*L + anchor.
template <int QUANT>
__device__ __forceinline__ void cells_of(const VoteParams& p, const uint32_t (&A)[4],
                                         const uint32_t (&R)[4], uint32_t (&E)[4], uint32_t (&O)[4]) {
  const uint32_t L = (uint32_t)p.levels;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = quant4<QUANT>(A[i], p);
    const uint32_t b = quant4<QUANT>(R[i], p);
    E[i] = (a & 0x00FF00FFu) + (b & 0x00FF00FFu) * L;
    O[i] = ((a >> 8) & 0x00FF00FFu) + ((b >> 8) & 0x00FF00FFu) * L;
  }
}

// q = n / d for n < 2^31 via a precomputed multiplier (d == 1: mul = 0).
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t mul, uint32_t shr) {
  return mul ? (__umulhi(n, mul) >> shr) : n;
}

// ---------------------------------------------------------------------------
// Grid-wide barrier for a cooperative (co-resident) launch: every CTA has
// stored its partial; thread 0 publishes arrival (release) and waits for all
// `n` CTAs (acquire). The counter is zero when the launch starts: the host
// zeroes it once at context creation, and the last CTA to leave each launch
// re-arms it (glcm_vote_kernel epilogue). Launches that share it never
// overlap (tfg_engine.cu ScratchOrder).
// Counter words of a context's cooperative launches: [0] grid barrier,
// [kExitCtr] CTAs done (re-arm), [32..] shared-pool counters per band.
constexpr int kExitCtr = 16;

__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned int v = 0;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= n) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// After the grid barrier: CTA x of a band sums slice x of the band's
// gridDim.x partials (read through L2: __ldcg) and adds it to the u64 GLCM.
// PACKED16 partials are packed u16 pairs (word k = a + 256 b', halves b' and
// b' + 128; residuals < 2^16 each, so u32 sums cannot overflow); the others
// are u32 cells (summed in u64).
template <bool PACKED>
__device__ __forceinline__ void reduce_partials_slice(const VoteParams& p, uint32_t* scratch, int band_idx,
                                                      unsigned long long* glcm) {
  const uint32_t nparts = gridDim.x;
  const uint32_t L = (uint32_t)p.levels;
  const uint32_t words = PACKED ? (uint32_t)p.hist_words : L * L;
  const uint32_t slice = ((words + nparts - 1) / nparts + 3) & ~3u;
  const uint32_t w0 = min(words, blockIdx.x * slice), w1 = min(words, w0 + slice);
  if (w0 >= w1) return;
  const uint32_t* base = p.partials + (size_t)band_idx * nparts * words;
  if constexpr (PACKED) {
    // Thread t sums 4-word column group t % ng of the slice over partials
    // t / ng, t / ng + groups, ...: 16-byte L2 loads, several in flight
    // (the loop is unrolled). Field sums stay < 2^24 (<= 65535 per partial),
    // so they meet in u32 shared-memory counters: [lo fields | hi fields].
    // chunks of <= 4 * blockDim.x words (a grid of few CTAs has wide slices)
    for (uint32_t c0 = w0; c0 < w1; c0 += 4 * blockDim.x) {
      const uint32_t n = min(4 * blockDim.x, w1 - c0), ng = n / 4;  // words and slices are multiples of 4
      uint32_t* acc32 = scratch;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < 2 * n; i += blockDim.x) acc32[i] = 0;
      __syncthreads();
      const uint32_t groups = blockDim.x / ng;
      const uint32_t cg = threadIdx.x % ng, g0 = threadIdx.x / ng;
      if (g0 < groups) {
        uint32_t lo0 = 0, lo1 = 0, lo2 = 0, lo3 = 0, hi0 = 0, hi1 = 0, hi2 = 0, hi3 = 0;
        const uint4* src = reinterpret_cast<const uint4*>(base + c0) + cg;
        const size_t stride4 = words / 4;
#pragma unroll 4
        for (uint32_t q = g0; q < nparts; q += groups) {
          const uint4 v = __ldcg(src + q * stride4);
          lo0 += v.x & 0xFFFFu; hi0 += v.x >> 16;
          lo1 += v.y & 0xFFFFu; hi1 += v.y >> 16;
          lo2 += v.z & 0xFFFFu; hi2 += v.z >> 16;
          lo3 += v.w & 0xFFFFu; hi3 += v.w >> 16;
        }
        uint32_t* a = acc32 + 4 * cg;
        if (lo0) atomicAdd(a + 0, lo0);
        if (lo1) atomicAdd(a + 1, lo1);
        if (lo2) atomicAdd(a + 2, lo2);
        if (lo3) atomicAdd(a + 3, lo3);
        if (hi0) atomicAdd(a + n + 0, hi0);
        if (hi1) atomicAdd(a + n + 1, hi1);
        if (hi2) atomicAdd(a + n + 2, hi2);
        if (hi3) atomicAdd(a + n + 3, hi3);
      }
      __syncthreads();
      for (uint32_t c = threadIdx.x; c < n; c += blockDim.x) {
        const uint32_t w = c0 + c, a = w & 0xFFu, b = w >> 8;
        if (acc32[c]) atomicAdd(glcm + b * L + a, (unsigned long long)acc32[c]);
        if (acc32[n + c]) atomicAdd(glcm + (b + 128u) * L + a, (unsigned long long)acc32[n + c]);
      }
    }
    return;
  }
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(scratch);  // [ncol][2]
  // columns in chunks of at most blockDim.x; thread t: column t % ncol,
  // partials t / ncol, t / ncol + groups, ...
  for (uint32_t c0 = w0; c0 < w1; c0 += blockDim.x) {
    const uint32_t ncol = min((uint32_t)blockDim.x, w1 - c0);
    const uint32_t groups = blockDim.x / ncol;
    const uint32_t col = threadIdx.x % ncol, g0 = threadIdx.x / ncol;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 2 * ncol; i += blockDim.x) acc[i] = 0;
    __syncthreads();
    if (g0 < groups) {
      unsigned long long lo = 0, hi = 0;
      for (uint32_t q = g0; q < nparts; q += groups) {
        const uint32_t v = __ldcg(base + (size_t)q * words + c0 + col);
        if (PACKED) {
          lo += v & 0xFFFFu;
          hi += v >> 16;
        } else {
          lo += v;
        }
      }
      if (lo) atomicAdd(acc + 2 * col, lo);
      if (hi) atomicAdd(acc + 2 * col + 1, hi);
    }
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < ncol; c += blockDim.x) {
      const uint32_t w = c0 + c;
      if (PACKED) {
        const uint32_t a = w & 0xFFu, b = w >> 8;
        if (acc[2 * c]) atomicAdd(glcm + b * L + a, acc[2 * c]);
        if (acc[2 * c + 1]) atomicAdd(glcm + (b + 128u) * L + a, acc[2 * c + 1]);
      } else if (acc[2 * c]) {
        atomicAdd(glcm + w, acc[2 * c]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1 + K2: fused quantise, vote, privatised merge.
//
// Two passes over the CTA's share of the anchor raster:
//  * main pass — the INTERIOR 16-pixel segments of every row (j in [1, nch-1)),
//    flattened. Every reference byte of an interior segment lies inside its
//    row, so these loads need no guards and all 16 pairs vote:
//    no masks, no per-pair branches. A warp takes "double batches" of 64
//    consecutive segments (lane and lane+32; each LDG.128 of the warp is one
//    coalesced 512-byte access) from a per-CTA ticket counter, four per grab,
//    and keeps two double batches in a register ring (one in flight while the
//    other votes). In cooperative launches the last pool_dbl double batches
//    of the band form a shared pool that CTAs drain once their own range is
//    done, so the grid barrier does not wait on the slowest static range. Addresses come from one uniform division per double batch
//    plus a per-lane row-wrap select.
//  * edge pass — the first and last segment of every row (or every segment
//    of a narrow image), with per-lane guarded loads and valid-anchor masks.
// There is no barrier in either loop (PACKED16 included: see kPackedDrainBit).
// vote_cta: the work of CTA `cta` of band `band_idx` (glcm_vote_kernel: the
// block's x and y; glcm_vote_jobs_kernel: one job's share of the grid).
template <int QUANT, int STRAT, int KSEL>
//
// `unit` indexes the launch's scratch (per-CTA partials, pool counters): the
// band for glcm_vote_kernel, the grid row (job x band) for the jobs kernel.
__device__ __forceinline__ void vote_cta(const VoteParams& p, const uint32_t cta, const int band_idx,
                                         const int unit) {
  extern __shared__ __align__(16) uint32_t hist[];
  __shared__ uint32_t s_ticket;
  constexpr uint32_t kWarps = kThreads / 32;
  const int tid = threadIdx.x;
  const uint32_t lane = tid & 31, warp = tid >> 5;
  const uint8_t* band = p.img + (unsigned long long)band_idx * p.band_stride;
  const uint32_t L = (uint32_t)p.levels;
  const int cells = p.levels * p.levels;
  unsigned long long* glcm = p.glcm + (size_t)band_idx * cells;

  {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    const int n4 = p.hist_words >> 2;
    for (int i = tid; i < n4; i += kThreads) h4[i] = make_uint4(0, 0, 0, 0);
  }

  uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(hist));
  if constexpr (STRAT == S_COPIES32) hb += lane * 4u;
  if constexpr (STRAT == S_COPIES8) hb += (lane & 7u) * 4u;
  if constexpr (STRAT == S_P16X16) hb += (lane & 15u) * 8u;  // byte 2 of hb stays 0 (p16x16_addr)

  const uint32_t pitch = (uint32_t)p.pitch;
  const uint32_t nch = (uint32_t)p.nch;
  const uint32_t ni = (uint32_t)p.ni;

#ifndef TFG_RLE_PERIOD
#define TFG_RLE_PERIOD 8  // items between re-samples once the check stops paying (power of 2)
#endif
#ifndef TFG_RLE_MIN
#define TFG_RLE_MIN 4  // uniform lanes of a warp-item for the check to keep paying
#endif
  bool rle = true;  // PACKED16 run-length check; re-sampled every TFG_RLE_PERIOD-th item when it stops paying
  uint32_t nb = 0;
  // Votes one item (16 pairs, or the pairs in `mask`).
  // S_P16X16: quantised anchor / reference words of an item
  auto p16x16_item = [&](const RawItem& cur, uint32_t mask) {
    uint32_t A[4], R[4], qa[4], qb[4];
    ref_words<KSEL>(p, cur, A, R);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      qa[i] = quant4<QUANT>(A[i], p);
      qb[i] = quant4<QUANT>(R[i], p);
    }
    p16x16_vote(hb, qa, qb, mask, glcm, L);
  };
  auto vote_item = [&](const RawItem& cur) {
    if constexpr (STRAT == S_P16X16) {
      if (cur.mask) p16x16_item(cur, cur.mask);
      return;
    }
    uint32_t P[4], Q[4];
    item_words<QUANT, STRAT, KSEL>(p, cur, P, Q);
    if constexpr (STRAT == S_PACKED16) {
      const bool check = rle || (nb & (TFG_RLE_PERIOD - 1)) == 0;
      const bool hit = vote16<STRAT>(hb, P, Q, cur.mask, check, glcm, L);
      if (check) rle = __popc(__ballot_sync(0xffffffffu, hit)) >= TFG_RLE_MIN;
      ++nb;
    } else if (cur.mask == 0xFFFFu) {
      // conflict-free (COPIES*) or hardware-aggregated (COPY1: POPC.INC) layouts
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) red_smem1(vote_addr<STRAT>(hb, pair_x(P[i], Q[i], k)));
    } else if (cur.mask) {
      vote_masked<STRAT>(hb, P[0], P[1], P[2], P[3], Q[0], Q[1], Q[2], Q[3], cur.mask, glcm, L);
    }
  };

  // An unmasked item of the main pass (all 16 pairs vote).
  auto vote_full = [&](const RawItem& cur) {
    if constexpr (STRAT == S_P16X16) {
      p16x16_item(cur, 0xFFFFu);
      return;
    }
    uint32_t P[4], Q[4];
    item_words<QUANT, STRAT, KSEL>(p, cur, P, Q);
    if constexpr (STRAT == S_PACKED16) {
      const bool check = rle || (nb & (TFG_RLE_PERIOD - 1)) == 0;
      const bool hit = vote16<STRAT>(hb, P, Q, 0xFFFFu, check, glcm, L);
      if (check) rle = __popc(__ballot_sync(0xffffffffu, hit)) >= TFG_RLE_MIN;
      ++nb;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) red_smem1(vote_addr<STRAT>(hb, pair_x(P[i], Q[i], k)));
    }
  };

  // ---------------- main pass: interior segments, 64 per double batch -------
  const long long mbeg64 = (long long)cta * p.main_per_cta;
  const long long mend64 = min(mbeg64 + p.main_per_cta, p.pool_beg);
  const uint32_t mbeg = (uint32_t)mbeg64;
  const uint32_t m_items = mend64 > mbeg64 ? (uint32_t)(mend64 - mbeg64) : 0u;
  const uint32_t wrap_off = pitch - ni * 16u;  // next row, back to interior segment 0

  // double batch t -> items lane and lane+32 of [mbeg + 64t, +64). Only
  // whole double batches run here; a CTA's last partial one (< 64 items)
  // joins the edge pass.
  const uint32_t n_full_dbl = m_items / 64;
  const uint32_t lane16 = lane << 4;
  // 64-bit bases are formed once; per double batch one row offset, per item
  // one 32-bit lane offset
  const uint8_t* const abase0 = band + ((p.ch0 + p.js) << 4);
  const uint8_t* const rbase0 = abase0 + p.ref_off;
  // f0: first item of the double batch (warp-uniform)
#ifndef TFG_NBR_SHFL
#define TFG_NBR_SHFL 1
#endif
  // Reference windows with one narrow word (d <= 3 at 0 / 135 degrees: the
  // next segment's first word; 45 degrees: the previous segment's last word):
  // in a double batch that does not wrap a row, that word is the adjacent
  // lane's anchor / reference segment, so it comes by one shuffle per item
  // instead of a 4-byte load per lane (a strided LDG.32 touches the same 4-5
  // L1 lines as a full LDG.128).
  // Enabled for COPIES8 (L <= 64), whose kernel is bound by the L1 data pipe
  // (noise L=64: -3..-6% per call), and for the one-slot PACKED16 variants
  // (KSEL 0 and 3) outside run-length mode (noise warps: theta=45 -3.6%);
  // the issue-bound paths (COPIES32, smooth PACKED16 warps) keep the loads.
  constexpr bool kNbrShfl = TFG_NBR_SHFL && (KSEL == 5 || KSEL == 0 || KSEL == 3) &&
                            (STRAT == S_COPIES8 || (STRAT == S_PACKED16 && KSEL != 5));
  constexpr uint32_t kNbrPending = 0x10000u;  // RawItem.mask of a main-pass x0 (vote_full ignores masks)
  auto nbr_fix = [&](RawItem& x0, RawItem& x1) {
    if constexpr (kNbrShfl) {
      if (x0.mask != kNbrPending) return;  // warp-uniform: the row-wrap path loaded the words
      const uint32_t nxt = (lane + 1) & 31u, prv = (lane + 31) & 31u;
      if constexpr (KSEL == 3) {
        const uint32_t p1 = lane == 31 ? x0.c1.w : x1.c1.w;
        const uint32_t w0 = __shfl_sync(0xffffffffu, x0.c1.w, prv);
        const uint32_t w1 = __shfl_sync(0xffffffffu, p1, prv);
        if (lane != 0) x0.c0.w = w0;
        x1.c0.w = w1;
      } else {
        const uint32_t v0 = KSEL == 5 ? x0.a.x : x0.c0.x, v1 = KSEL == 5 ? x1.a.x : x1.c0.x;
        const uint32_t w0 = __shfl_sync(0xffffffffu, lane == 0 ? v1 : v0, nxt);
        const uint32_t w1 = __shfl_sync(0xffffffffu, v1, nxt);
        x0.c1.x = w0;
        if (lane != 31) x1.c1.x = w1;
      }
    }
  };
  auto issue_dbl = [&](uint32_t f0, RawItem& x0, RawItem& x1) {
    const uint32_t row0 = fast_div(f0, p.ni_mul, p.ni_shr);
    const uint32_t jj0 = f0 - row0 * ni;
    const unsigned long long roff = (unsigned long long)row0 * pitch + (jj0 << 4);
    if (jj0 + 64u <= ni) {
      // warp-uniform common case (~94% at 16384 px rows): no row wrap inside
      // the double batch, so both items of a lane share one pointer and the
      // second sits at a +512 B immediate offset
      const uint8_t* a = abase0 + roff + lane16;
      x0.a = ldg16(a);
      x1.a = ldg16(a + 512);
      // KSEL >= 5 (theta = 0, d < 16): ref_off == 0, the reference row is the anchor row
      const uint8_t* r = ksel_c0_is_anchor<KSEL>() ? a : rbase0 + roff + lane16;
      if (kNbrShfl && !(STRAT == S_PACKED16 && rle)) {
        // the one narrow word of the window comes from the neighbour lane at
        // vote time (nbr_fix); only the batch's boundary lane loads it
        x0.mask = kNbrPending;
        if constexpr (KSEL == 3) {
          x0.c1 = ldg16(r + 16);
          x1.c1 = ldg16(r + 528);
          if (lane == 0) x0.c0.w = __ldg(reinterpret_cast<const uint32_t*>(r + 12));
        } else {
          if constexpr (KSEL == 0) {
            x0.c0 = ldg16(r);
            x1.c0 = ldg16(r + 512);
          }
          if (lane == 31) x1.c1.x = __ldg(reinterpret_cast<const uint32_t*>(r + 528));
        }
        return;
      }
      if constexpr (kNbrShfl) x0.mask = 0;
      if constexpr (!ksel_c0_is_anchor<KSEL>()) {
        x0.c0 = ldg16(r);
        x1.c0 = ldg16(r + 512);
      }
      if constexpr (ksel_needs_c1<KSEL>()) {
        x0.c1 = ldg16(r + 16);
        x1.c1 = ldg16(r + 528);
      }
      return;
    }
    if constexpr (kNbrShfl) x0.mask = 0;
    const uint32_t off0 = lane16 + (jj0 + lane >= ni ? wrap_off : 0u);  // ni >= 64: at most one wrap
    const uint32_t off1 = lane16 + 512u + (jj0 + lane + 32u >= ni ? wrap_off : 0u);
    const uint8_t* a = abase0 + roff;
    x0.a = ldg16(a + off0);
    x1.a = ldg16(a + off1);
    const uint8_t* r = rbase0 + roff;
    if constexpr (!ksel_c0_is_anchor<KSEL>()) {
      x0.c0 = ldg16(r + off0);
      x1.c0 = ldg16(r + off1);
    }
    if constexpr (ksel_needs_c1<KSEL>()) {
      x0.c1 = ldg16(r + off0 + 16);
      x1.c1 = ldg16(r + off1 + 16);
    }
  };

  const uint32_t ticket_addr = static_cast<uint32_t>(__cvta_generic_to_shared(&s_ticket));
  // L2 bulk prefetch of the stream's leading edge (reference bytes of double
  // batches [b0, b0 + nb)), issued by the grab that crosses a multiple of kSpan.
  auto prefetch_span = [&](uint32_t b0, uint32_t nbat) {
    if (b0 >= n_full_dbl) return;
    const uint32_t i0 = mbeg + b0 * 64;
    const uint32_t i1 = mbeg + min(m_items, (b0 + nbat) * 64) - 1;
    const uint32_t r0 = fast_div(i0, p.ni_mul, p.ni_shr), r1 = fast_div(i1, p.ni_mul, p.ni_shr);
    long long a0 = (long long)r0 * pitch + ((p.ch0 + p.js + (i0 - r0 * ni)) << 4) + p.ref_off;
    long long a1 = (long long)r1 * pitch + ((p.ch0 + p.js + (i1 - r1 * ni)) << 4) + p.ref_off + 32;
    a0 = max(a0, 0ll) & ~15ll;
    a1 = min(a1, (long long)p.buf_bytes);
    if (a1 > a0) prefetch_l2(band + a0, (uint32_t)min(a1 - a0, 1ll << 20) & ~15u);
  };
#ifndef TFG_PREFETCH_AHEAD
#define TFG_PREFETCH_AHEAD 48
#endif
#ifndef TFG_PREFETCH_SPAN
#define TFG_PREFETCH_SPAN 16
#endif
  constexpr uint32_t kAhead = TFG_PREFETCH_AHEAD, kSpan = TFG_PREFETCH_SPAN;  // in double batches
  auto grab4 = [&]() -> uint32_t {
    uint32_t tn = 0;
    if (lane == 0) {
      asm volatile("atom.shared.add.u32 %0, [%1], 4;" : "=r"(tn) : "r"(ticket_addr) : "memory");
      if (((tn + 3) & (kSpan - 1)) < 4) prefetch_span(((tn + 3) & ~(kSpan - 1)) + kAhead, kSpan);
    }
    return __shfl_sync(0xffffffffu, tn, 0);
  };

#if TFG_TMA
  // ---- staged main pass: the TMA engine (cp.async.bulk) copies each batch
  // of 32 interior segments (+ its reference window) into the warp's shared
  // stage; two stages per warp, one loading while the other is voted. The
  // register ring of the LDG pass is gone; each lane reads its item with
  // ld.shared. Batches come in pairs from the per-CTA tickets (one double
  // batch per grab), then four double batches per grab from the shared pool.
  {
    constexpr uint32_t kStageA = 32 * 16 + 32;                // anchors + the segment after each row piece
    constexpr bool kRef = !ksel_c0_is_anchor<KSEL>();         // separate reference rows (theta != 0 or d >= 16)
    constexpr uint32_t kStage = kRef ? 2 * kStageA : kStageA;
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(hist + p.hist_words)) + warp * 2 * kStage;
    const uint32_t bars = static_cast<uint32_t>(__cvta_generic_to_shared(hist + p.hist_words)) +
                          kWarps * 2 * kStage + warp * 16;
    if (lane == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 8, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid == 0) s_ticket = kWarps;
    __syncthreads();  // histogram zeroed, ticket counter set, barriers initialised
    // batch generator: single batches of 32 items, two per double batch
    uint32_t q_base = mbeg + warp * 64, q_left = warp < n_full_dbl ? 2u : 0u;
    bool own = true;
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    auto next_batch = [&]() -> uint32_t {
      if (q_left == 0) {
        if (own) {
          uint32_t tn = 0;
          if (lane == 0) {
            asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(tn) : "r"(ticket_addr) : "memory");
            if ((tn & (kSpan - 1)) == 0) prefetch_span(tn + kAhead, kSpan);
          }
          tn = __shfl_sync(0xffffffffu, tn, 0);
          if (tn < n_full_dbl) {
            q_base = mbeg + tn * 64;
            q_left = 2;
          } else {
            own = false;
          }
        }
        if (!own) {
          if constexpr (STRAT == S_PACKED16 || STRAT == S_COPY1) {
            uint32_t g = kNone;
            if (lane == 0 && p.pool_ctr) {
              const uint32_t tp = atomicAdd(p.pool_ctr + unit, 4u);
              if (tp < p.pool_dbl) g = (uint32_t)p.pool_beg + tp * 64;
            }
            g = __shfl_sync(0xffffffffu, g, 0);
            if (g == kNone) return kNone;
            q_base = g;
            q_left = 8;
          } else {
            return kNone;
          }
        }
      }
      const uint32_t b = q_base;
      q_base += 32;
      --q_left;
      return b;
    };
    // items [f0, f0 + 32): n1 of them in row0, the rest at the start of row0 + 1
    auto pieces = [&](uint32_t f0, uint32_t& row0, uint32_t& jj0, uint32_t& n1) {
      row0 = fast_div(f0, p.ni_mul, p.ni_shr);
      jj0 = f0 - row0 * ni;
      n1 = min(32u, ni - jj0);
    };
    auto issue = [&](uint32_t st, uint32_t f0) {  // lane 0
      uint32_t row0, jj0, n1;
      pieces(f0, row0, jj0, n1);
      const uint32_t dstA = sbase + st * kStage, bar = bars + st * 8;
      const uint8_t* a1 = abase0 + (unsigned long long)row0 * pitch + (jj0 << 4);
      const uint32_t b1 = n1 * 16 + 16;
      const uint32_t n2 = 32 - n1;
      const uint32_t b2 = n2 ? n2 * 16 + 16 : 0u;
      constexpr uint32_t kRefLess = ksel_needs_c1<KSEL>() ? 0u : 16u;  // reference pieces skip the extra segment
      mbar_expect_tx(bar, kRef ? 2 * (b1 + b2) - kRefLess * (n2 ? 2u : 1u) : b1 + b2);
      bulk_g2s(dstA, a1, b1, bar);
      if (n2) bulk_g2s(dstA + b1, abase0 + (unsigned long long)(row0 + 1) * pitch, b2, bar);
      if constexpr (kRef) {
        // reference rows: the c0 segments (+ the c1 after the last one when
        // the window is unaligned); the same bytes the LDG pass reads
        constexpr uint32_t kX = ksel_needs_c1<KSEL>() ? 16u : 0u;
        bulk_g2s(dstA + kStageA, a1 + p.ref_off, b1 - 16 + kX, bar);
        if (n2)
          bulk_g2s(dstA + kStageA + b1, abase0 + (unsigned long long)(row0 + 1) * pitch + p.ref_off, b2 - 16 + kX, bar);
      }
    };
    uint32_t fb0 = next_batch();
    uint32_t fb1 = fb0 == kNone ? kNone : next_batch();
    if (lane == 0) {
      if (fb0 != kNone) issue(0, fb0);
      if (fb1 != kNone) issue(1, fb1);
    }
    uint32_t ph0 = 0, ph1 = 0;
    // vote the batch in stage `st`, then refill the stage with the next batch
    auto step = [&](const uint32_t st, uint32_t& fb, uint32_t& ph) {
      mbar_wait(bars + st * 8, ph);
      ph ^= 1u;
      uint32_t row0, jj0, n1;
      pieces(fb, row0, jj0, n1);
      const uint32_t off = sbase + st * kStage + lane * 16 + (lane >= n1 ? 16u : 0u);
      RawItem it;
      it.mask = 0xFFFFu;
      it.a = lds16(off);
      if constexpr (kRef) {
        it.c0 = lds16(off + kStageA);
        if constexpr (ksel_needs_c1<KSEL>()) it.c1 = lds16(off + kStageA + 16);
      } else {
        it.c1 = lds16(off + 16);
      }
      __syncwarp();  // every lane has read the stage before the copy engine refills it
      fb = next_batch();
      if (lane == 0 && fb != kNone) {
        fence_proxy_async();
        issue(st, fb);
      }
      vote_full(it);
    };
    for (;;) {
      if (fb0 == kNone) break;
      step(0, fb0, ph0);
      if (fb1 == kNone) break;
      step(1, fb1, ph1);
    }
    if (lane == 0) {
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bars) : "memory");
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bars + 8) : "memory");
    }
  }
  if (false) {
#else
  {
#endif
  // PACKED16 with the widest reference windows (KSEL 0-3: c0 + c1 loads)
  // keeps ONE double batch in flight per warp: the second ring slot's
  // registers made these variants spill (32-92 bytes); without it they run
  // 1-4% faster (c3 2,089 -> 2,109 Gpairs/s). The other variants keep the
  // two-slot ring, which is faster for them.
  constexpr bool kRing1 = STRAT == S_PACKED16 && KSEL <= 3;
  if constexpr (kRing1) {
  RawItem a0, a1;
  uint32_t q_next = 2 * warp, q_left = 2;
  auto next_dbl = [&]() -> uint32_t {
    if (q_left == 0) {
      q_next = grab4();
      q_left = 4;
    }
    --q_left;
    return q_next++;
  };
  uint32_t ta = next_dbl();
  if (ta < n_full_dbl) issue_dbl(mbeg + ta * 64, a0, a1);
  if (tid == 0) {
    s_ticket = 2 * kWarps;
    for (uint32_t q = 0; q < kAhead + kSpan; q += kSpan) prefetch_span(q + 2 * kWarps, kSpan);
  }
  __syncthreads();  // histogram zeroed, ticket counter set
  while (ta < n_full_dbl) {
    nbr_fix(a0, a1);
    vote_full(a0);
    vote_full(a1);
    ta = next_dbl();
    if (ta < n_full_dbl) issue_dbl(mbeg + ta * 64, a0, a1);
  }
  if constexpr (STRAT == S_PACKED16 || STRAT == S_COPY1) {
    if (p.pool_ctr) {
      constexpr uint32_t kNone = 0xFFFFFFFFu;
      uint32_t gbase = 0, gleft = 0;
      auto grab_pool = [&]() -> uint32_t {
        if (gleft == 0) {
          uint32_t g = kNone;
          if (lane == 0) {
            const uint32_t tp = atomicAdd(p.pool_ctr + unit, 4u);
            if (tp < p.pool_dbl) g = (uint32_t)p.pool_beg + tp * 64;
          }
          g = __shfl_sync(0xffffffffu, g, 0);
          if (g == kNone) return kNone;
          gbase = g;
          gleft = 4;
        }
        const uint32_t r = gbase;
        gbase += 64;
        --gleft;
        return r;
      };
      uint32_t ga = grab_pool();
      if (ga != kNone) issue_dbl(ga, a0, a1);
      while (ga != kNone) {
        nbr_fix(a0, a1);
        vote_full(a0);
        vote_full(a1);
        ga = grab_pool();
        if (ga != kNone) issue_dbl(ga, a0, a1);
      }
    }
  }
  } else {
  RawItem a0, a1, b0i, b1i;
  uint32_t ta = 2 * warp, tb = 2 * warp + 1;
  if (ta < n_full_dbl) issue_dbl(mbeg + ta * 64, a0, a1);
  if (tb < n_full_dbl) issue_dbl(mbeg + tb * 64, b0i, b1i);
  if (tid == 0) {
    s_ticket = 2 * kWarps;
    for (uint32_t q = 0; q < kAhead + kSpan; q += kSpan) prefetch_span(q + 2 * kWarps, kSpan);
  }
  __syncthreads();  // histogram zeroed, ticket counter set

  // one ticket grab (4 double batches) per two revolutions of the ring
  for (;;) {
    if (ta >= n_full_dbl) break;
    nbr_fix(a0, a1);
    vote_full(a0);
    vote_full(a1);
    const uint32_t tn = grab4();
    ta = tn;
    if (ta < n_full_dbl) issue_dbl(mbeg + ta * 64, a0, a1);
    if (tb >= n_full_dbl) break;
    nbr_fix(b0i, b1i);
    vote_full(b0i);
    vote_full(b1i);
    tb = tn + 1;
    if (tb < n_full_dbl) issue_dbl(mbeg + tb * 64, b0i, b1i);
    if (ta >= n_full_dbl) break;
    nbr_fix(a0, a1);
    vote_full(a0);
    vote_full(a1);
    ta = tn + 2;
    if (ta < n_full_dbl) issue_dbl(mbeg + ta * 64, a0, a1);
    if (tb >= n_full_dbl) break;
    nbr_fix(b0i, b1i);
    vote_full(b0i);
    vote_full(b1i);
    tb = tn + 3;
    if (tb < n_full_dbl) issue_dbl(mbeg + tb * 64, b0i, b1i);
  }

  // Shared tail pool (cooperative launches): once its own range is done, a
  // warp takes TFG_POOL_GRAB double batches per grab from the band's global
  // counter (4: grabs of 1 or 2 measured 11% / 1% slower, contention on the
  // one counter). The counter only grows, so an empty grab ends that ring
  // slot. Only the layouts with per-CTA partials (L > 64) end at
  // a grid barrier, so only they carry this loop.
#ifndef TFG_POOL_GRAB
#define TFG_POOL_GRAB 4
#endif
  if constexpr (STRAT == S_PACKED16 || STRAT == S_COPY1) {
    if (p.pool_ctr) {
      constexpr uint32_t kNone = 0xFFFFFFFFu, kGrab = TFG_POOL_GRAB;
      uint32_t gbase = 0, gleft = 0;
      auto grab_pool = [&]() -> uint32_t {  // next pool double batch (warp-uniform) or kNone
        if (gleft == 0) {
          uint32_t g = kNone;
          if (lane == 0) {
            const uint32_t tp = atomicAdd(p.pool_ctr + unit, kGrab);
            if (tp < p.pool_dbl) g = (uint32_t)p.pool_beg + tp * 64;
          }
          g = __shfl_sync(0xffffffffu, g, 0);
          if (g == kNone) return kNone;
          gbase = g;
          gleft = kGrab;
        }
        const uint32_t r = gbase;
        gbase += 64;
        --gleft;
        return r;
      };
      uint32_t ga = grab_pool(), gb = kNone;
      if (ga != kNone) {
        issue_dbl(ga, a0, a1);
        gb = grab_pool();
        if (gb != kNone) issue_dbl(gb, b0i, b1i);
      }
      while (ga != kNone) {
        nbr_fix(a0, a1);
        vote_full(a0);
        vote_full(a1);
        ga = gb == kNone ? kNone : grab_pool();
        if (ga != kNone) issue_dbl(ga, a0, a1);
        if (gb == kNone) break;
        nbr_fix(b0i, b1i);
        vote_full(b0i);
        vote_full(b1i);
        gb = ga == kNone ? kNone : grab_pool();
        if (gb != kNone) issue_dbl(gb, b0i, b1i);
      }
    }
  }

  }  // kRing1
  }  // LDG main pass

  // ---------------- edge pass: first/last segment of each row (or all) -----
  {
    const long long ebeg64 = (long long)cta * p.edge_per_cta;
    const long long eend64 = min(ebeg64 + p.edge_per_cta, p.edge_items);
    const uint32_t ebeg = (uint32_t)ebeg64;
    const uint32_t e_items = eend64 > ebeg64 ? (uint32_t)(eend64 - ebeg64) : 0u;
    const uint32_t ne = (uint32_t)p.ne;
    const uint32_t tail0 = mbeg + n_full_dbl * 64, n_tail = m_items - n_full_dbl * 64;  // main-pass leftovers
    const uint32_t n_work = e_items + n_tail;
    for (uint32_t t = warp; t * 32 < n_work; t += kWarps) {
      const uint32_t local = t * 32 + lane;
      uint32_t row, j;
      if (local < e_items) {
        const uint32_t e = ebeg + local;
        row = fast_div(e, p.ne_mul, p.ne_shr);
        const uint32_t r = e - row * ne;
        // edge segments of a row: [0, js) and [js + ni, nch)
        j = (ni && r >= (uint32_t)p.js) ? r + ni : r;
      } else {
        const uint32_t f = tail0 + (local - e_items);
        row = fast_div(f, p.ni_mul, p.ni_shr);
        j = p.js + (f - row * ni);
      }
      RawItem it;
      issue_item<KSEL>(p, band, row, j, local < n_work, it);
      vote_item(it);
    }
  }
  __syncthreads();

  // K2 epilogue. PACKED16 with partials: the CTA's packed u16-pair words are
  // stored as they are (coalesced 16-byte stores, half the bytes of u32 cells).
  // Otherwise: merge the copies of each real cell (b, a), then one u64 atomic
  // per cell or one plain store into this CTA's u32 partial. With partials and
  // a co-resident (cooperative) grid, the CTAs then meet at a grid barrier and
  // each sums one slice of all its band's partials while they are still in L2
  // (reduce_partials_slice); otherwise glcm_reduce_*_kernel does it.
  if (p.partials) {
    if constexpr (STRAT == S_PACKED16) {
      uint4* dst = reinterpret_cast<uint4*>(p.partials + ((size_t)unit * gridDim.x + blockIdx.x) * (size_t)p.hist_words);
      const uint4* src = reinterpret_cast<const uint4*>(hist);
      for (int i = tid; i < (p.hist_words >> 2); i += kThreads) {
        const uint4 v = src[i];
        dst[i] = make_uint4(packed_decode(v.x), packed_decode(v.y), packed_decode(v.z), packed_decode(v.w));
      }
    } else {
      uint32_t* part = p.partials + ((size_t)unit * gridDim.x + blockIdx.x) * (size_t)cells;
      constexpr int RC = strat_copies(STRAT);
      for (int c = tid; c < cells; c += kThreads) {
        const uint32_t b = (uint32_t)c / L, a = (uint32_t)c - b * L;
        const uint32_t pos = cell_pos<STRAT>(b, a);
        uint32_t sum = 0;
#pragma unroll 8
        for (int k = 0; k < RC; ++k) sum += hist[pos * RC + ((k + lane) & (RC - 1))];
        part[c] = sum;
      }
    }
    if (p.sync_ctr) {
      const unsigned int n = gridDim.x * gridDim.y;
      grid_barrier(p.sync_ctr, n);
      reduce_partials_slice<STRAT == S_PACKED16>(p, hist, unit, glcm);
      // The last CTA out re-arms the counters for the next launch on the
      // stream (every CTA has left the barrier spin and the pool by now), so
      // the host needs no memset per launch.
      if (threadIdx.x == 0) {
        if (atomicAdd(p.sync_ctr + kExitCtr, 1u) == n - 1) {
          *reinterpret_cast<volatile unsigned int*>(p.sync_ctr) = 0u;
          *reinterpret_cast<volatile unsigned int*>(p.sync_ctr + kExitCtr) = 0u;
          if (p.pool_ctr)
            for (unsigned int b = 0; b < gridDim.y; ++b) reinterpret_cast<volatile unsigned int*>(p.pool_ctr)[b] = 0u;
        }
      }
    }
    return;
  }
  if constexpr (STRAT == S_P16X16) {
    // cell (b, a): copy k's field at word A1(a) + 256 b + 16384 (a >> 5) + 2k, half a & 1 (p16x16_addr)
    for (int cc = tid; cc < cells; cc += kThreads) {
      const uint32_t b = (uint32_t)cc / L, a = (uint32_t)cc - b * L;
      const uint32_t a1 = ((a >> 1) & 1u) | (((a >> 2) & 7u) << 5);
      const uint32_t base = a1 + 256u * b + 16384u * (a >> 5), sh = 16u * (a & 1u);
      uint32_t sum = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) sum += (hist[base + 2u * ((k + lane) & 15u)] >> sh) & 0xFFFFu;
      if (sum) atomicAdd(glcm + cc, (unsigned long long)sum);
    }
    return;
  }
  constexpr int RC = strat_copies(STRAT);
  for (int c = tid; c < cells; c += kThreads) {
    const uint32_t b = (uint32_t)c / L, a = (uint32_t)c - b * L;
    const uint32_t pos = cell_pos<STRAT>(b, a);
    uint32_t sum = 0;
#pragma unroll 8
    for (int k = 0; k < RC; ++k) sum += hist[pos * RC + ((k + lane) & (RC - 1))];
    if (sum) atomicAdd(glcm + c, (unsigned long long)sum);
  }
}

template <int QUANT, int STRAT, int KSEL>
__global__ void __launch_bounds__(kThreads, 1) glcm_vote_kernel(const VoteParams p) {
  vote_cta<QUANT, STRAT, KSEL>(p, blockIdx.x, blockIdx.y, blockIdx.y);
}

// Several (d, theta) GLCMs of one image (or band batch) in ONE launch: grid
// row y = band * njobs + job, x = the job's CTAs. Each job keeps its own
// geometry; the reference-window variant (KSEL) is picked per CTA, so all
// of an image's angles share one launch and its fixed costs (SURVEY.md §7
// "small images are latency-bound"). Layouts with per-CTA partials (L > 64)
// run glcm_vote_jobs1_kernel as a cooperative launch: each (job, band) row
// has its own partials, pool counter and reduce slices; one grid barrier for
// the whole launch.
constexpr int kMaxJobs = 8;
struct VoteJobs {
  VoteParams job[kMaxJobs];
  int ksel[kMaxJobs];
  int nbands;
  int njobs;
};

// One KSEL for every job of the launch: the layouts with per-CTA partials
// (COPY1, PACKED16). With the per-job switch below, ptxas spills 100-240
// bytes of the PACKED16 body (its nine inlined variants are allocated as one
// function), which costs the issue-bound smooth path ~2.5%; this form is
// spill-free and the host groups jobs by KSEL.
template <int QUANT, int STRAT, int KSEL>
__global__ void __launch_bounds__(kThreads, 1) glcm_vote_jobs1_kernel(const __grid_constant__ VoteJobs jp) {
  const int band = (int)blockIdx.y / jp.njobs;
  const int j = (int)blockIdx.y - band * jp.njobs;
  vote_cta<QUANT, STRAT, KSEL>(jp.job[j], blockIdx.x, band, blockIdx.y);
}

// PACKED16: two neighbouring KSELs per launch ({0,1}, {2,3}, {5,6}, {7,8};
// e.g. d = 1, 2 and 4 at 0 or 135 degrees), still spill-free with two
// inlined bodies; KSEL 4 uses glcm_vote_jobs1_kernel.
template <int QUANT, int STRAT, int K1, int K2>
__global__ void __launch_bounds__(kThreads, 1) glcm_vote_jobs2_kernel(const __grid_constant__ VoteJobs jp) {
  const int band = (int)blockIdx.y / jp.njobs;
  const int j = (int)blockIdx.y - band * jp.njobs;
  if (jp.ksel[j] == K1)
    vote_cta<QUANT, STRAT, K1>(jp.job[j], blockIdx.x, band, blockIdx.y);
  else
    vote_cta<QUANT, STRAT, K2>(jp.job[j], blockIdx.x, band, blockIdx.y);
}

template <int QUANT, int STRAT>
__global__ void __launch_bounds__(kThreads, 1) glcm_vote_jobs_kernel(const __grid_constant__ VoteJobs jp) {
  // band-major: the jobs of one band run side by side (adjacent blocks, the
  // same wave), so a band is read from DRAM once and from L2 by the other jobs
  const int band = (int)blockIdx.y / jp.njobs;
  const int j = (int)blockIdx.y - band * jp.njobs;
  const VoteParams& p = jp.job[j];
  switch (jp.ksel[j]) {
    case 0: vote_cta<QUANT, STRAT, 0>(p, blockIdx.x, band, blockIdx.y); break;
    case 1: vote_cta<QUANT, STRAT, 1>(p, blockIdx.x, band, blockIdx.y); break;
    case 2: vote_cta<QUANT, STRAT, 2>(p, blockIdx.x, band, blockIdx.y); break;
    case 3: vote_cta<QUANT, STRAT, 3>(p, blockIdx.x, band, blockIdx.y); break;
    case 5: vote_cta<QUANT, STRAT, 5>(p, blockIdx.x, band, blockIdx.y); break;
    case 6: vote_cta<QUANT, STRAT, 6>(p, blockIdx.x, band, blockIdx.y); break;
    case 7: vote_cta<QUANT, STRAT, 7>(p, blockIdx.x, band, blockIdx.y); break;
    case 8: vote_cta<QUANT, STRAT, 8>(p, blockIdx.x, band, blockIdx.y); break;
    default: vote_cta<QUANT, STRAT, 4>(p, blockIdx.x, band, blockIdx.y); break;
  }
}

// Everything below is used by tfg_engine.cu only (tfg_vote_inst.cu defines
// TFG_VOTE_ONLY: its translation units hold just the vote kernels).
#ifndef TFG_VOTE_ONLY
// Sum of per-CTA PACKED16 words into the u64 accumulator. Split-K: CTA
// (x, y) sums partials [y*per, (y+1)*per) of words [4*(x*256+t), +4) with
// 16-byte loads, then adds its 8 cell sums with u64 atomics (spread addresses).
__global__ void __launch_bounds__(256) glcm_reduce_packed_kernel(const uint32_t* __restrict__ partials,
                                                                  int nparts, int words, int levels,
                                                                  int per_split,
                                                                  unsigned long long* __restrict__ glcm) {
  const int band = blockIdx.z;
  const int w4 = blockIdx.x * blockDim.x + threadIdx.x;  // index of a 4-word group
  if (w4 * 4 >= words) return;
  const int g0 = blockIdx.y * per_split, g1 = min(nparts, g0 + per_split);
  const uint4* src = reinterpret_cast<const uint4*>(partials + (size_t)band * nparts * words) + w4;
  const size_t stride4 = (size_t)words / 4;
  uint32_t lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (int g = g0; g < g1; ++g) {
    const uint4 v = __ldg(src + g * stride4);
    lo[0] += v.x & 0xFFFFu; hi[0] += v.x >> 16;
    lo[1] += v.y & 0xFFFFu; hi[1] += v.y >> 16;
    lo[2] += v.z & 0xFFFFu; hi[2] += v.z >> 16;
    lo[3] += v.w & 0xFFFFu; hi[3] += v.w >> 16;
  }
  unsigned long long* out = glcm + (size_t)band * levels * levels;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t x = (uint32_t)(w4 * 4 + k);  // cell a + 256 b, b < 128
    const uint32_t a = x & 0xFFu, b = x >> 8;
    if (lo[k]) atomicAdd(out + b * levels + a, (unsigned long long)lo[k]);
    if (hi[k]) atomicAdd(out + (b + 128) * levels + a, (unsigned long long)hi[k]);
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
    cells_of<QUANT>(p, A, R, E, O);
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

// ---------------------------------------------------------------------------
// Sub-GLCM export (compute_subglcms, parallel.hpp:160-225): the reference's
// exact privatised layout — groups own contiguous row stripes, stripe pixel k
// maps to lane (k - stripe_begin*width) mod group_size, and lane i votes into
// copy (i mod R). One CTA per work item (a row range inside one stripe);
// the R copies of the stripe live in shared memory when they fit, else the
// votes go straight to the global u32 sub-GLCMs. Diagnostic/drop-in path, not
// the throughput path (that is glcm_vote_kernel).
struct SubWork {
  uint32_t group, row0, row1, stripe_begin;
};

struct SubParams {
  const uint8_t* img;
  unsigned long long pitch;
  int width, height, levels, pixel_levels;
  int dr, dc, d;
  uint32_t group_size, copies;
  const SubWork* work;
  uint32_t* subs;  // [group][copy][L*L]
  int use_smem;
};

__global__ void __launch_bounds__(256) glcm_subglcm_kernel(const SubParams p) {
  extern __shared__ uint32_t sh[];
  const SubWork w = p.work[blockIdx.x];
  const uint32_t cells = (uint32_t)p.levels * p.levels;
  const uint32_t words = cells * p.copies;
  if (p.use_smem) {
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  uint32_t* gsub = p.subs + (size_t)w.group * words;
  const int col_begin = p.dc < 0 ? p.d : 0;
  const int col_end = p.dc > 0 ? p.width - p.d : p.width;
  const int row_limit = p.height - p.dr;
  const uint32_t row1 = min(w.row1, (uint32_t)max(row_limit, 0));
  const uint32_t ncols = col_end > col_begin ? (uint32_t)(col_end - col_begin) : 0u;
  const uint32_t L = (uint32_t)p.levels;
  const bool quant = p.pixel_levels != p.levels;
  if (w.row0 < row1 && ncols) {
    const unsigned long long n = (unsigned long long)(row1 - w.row0) * ncols;
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t r = w.row0 + (uint32_t)(i / ncols);
      const uint32_t c = col_begin + (uint32_t)(i % ncols);
      uint32_t a = p.img[(unsigned long long)r * p.pitch + c];
      uint32_t b = p.img[(unsigned long long)(r + p.dr) * p.pitch + (c + p.dc)];
      if (quant) {
        a = (a * L) >> 8;
        b = (b * L) >> 8;
      }
      const unsigned long long k = (unsigned long long)(r - w.stripe_begin) * (unsigned)p.width + c;
      const uint32_t copy = (uint32_t)(k % p.group_size) % p.copies;
      const uint32_t pos = copy * cells + b * L + a;
      if (p.use_smem) atomicAdd(sh + pos, 1u);
      else atomicAdd(gsub + pos, 1u);
    }
  }
  if (p.use_smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x)
      if (sh[i]) atomicAdd(gsub + i, sh[i]);
  }
}

// Hottest cell of each sub-GLCM (ContentionStats::per_copy_hottest,
// parallel.hpp:247-252); one CTA per sub-GLCM.
__global__ void __launch_bounds__(256) subglcm_max_kernel(const uint32_t* __restrict__ subs, int cells,
                                                          unsigned long long* __restrict__ out) {
  __shared__ uint32_t s[8];
  const uint32_t* g = subs + (size_t)blockIdx.x * cells;
  uint32_t m = 0;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) m = max(m, g[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = max(m, s[i]);
    m = max(m, s[0]);
    out[blockIdx.x] = m;
  }
}

// One copy per group (plan.copies == 1, the reference's plan for L >= 128 at
// its default scratch budget): sub-GLCM g is the GLCM of stripe g's anchors,
// voted by glcm_vote_kernel with the stripes as bands. These two kernels turn
// the [groups][cells] u64 stripe GLCMs into the reduce_subglcms sum
// (parallel.hpp:228-237) and the per_copy_hottest maxima (:247-252), and the
// u32 sub-GLCM export (u32 by the reference's 2^32 votes-per-group floor).
__global__ void __launch_bounds__(256) stripe_max_kernel(const unsigned long long* __restrict__ stripes, int cells,
                                                         unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s[8];
  const unsigned long long* g = stripes + (size_t)blockIdx.x * cells;
  unsigned long long m = 0;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) m = max(m, g[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = max(m, s[i]);
    out[blockIdx.x] = m;
  }
}

__global__ void stripe_sum_kernel(const unsigned long long* __restrict__ stripes, int cells, int groups,
                                  unsigned long long* __restrict__ counts, uint32_t* __restrict__ subs32) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x) {
    unsigned long long t = 0;
    for (int g = 0; g < groups; ++g) {
      const unsigned long long v = stripes[(size_t)g * cells + c];
      t += v;
      if (subs32) subs32[(size_t)g * cells + c] = (uint32_t)v;
    }
    if (counts) counts[c] = t;
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

// ---------------------------------------------------------------------------
// Device synth_noise (image.hpp:109-116: pixel k = mt19937(seed)() >> 24, k in
// row-major order). CTA s regenerates outputs [s*seglen, (s+1)*seglen) from
// the generator window the host computed by jump-ahead (tfg_mt19937.cpp):
// each 624-output block is one in-place twist in three dependency phases
// ([0,227) reads only old words, [227,454) and [454,624) read words of the
// previous phase), then tempering. Bit-identical to the sequential generator.
__device__ __forceinline__ uint32_t mt_twist(uint32_t x0, uint32_t x1, uint32_t xm) {
  const uint32_t y = (x0 & 0x80000000u) | (x1 & 0x7FFFFFFFu);
  return xm ^ (y >> 1) ^ ((y & 1u) ? 0x9908B0DFu : 0u);
}

__device__ __forceinline__ uint32_t mt_temper(uint32_t y) {
  y ^= y >> 11;
  y ^= (y << 7) & 0x9D2C5680u;
  y ^= (y << 15) & 0xEFC60000u;
  return y ^ (y >> 18);
}

__global__ void __launch_bounds__(256) synth_noise_kernel(const uint32_t* __restrict__ windows,
                                                          unsigned long long seglen, unsigned long long n,
                                                          unsigned long long width, unsigned long long pitch,
                                                          uint8_t* __restrict__ out) {
  __shared__ uint32_t mt[624];
  const int t = threadIdx.x;
  const unsigned long long k0 = (unsigned long long)blockIdx.x * seglen;
  const unsigned long long k1 = min(k0 + seglen, n);
  for (int i = t; i < 624; i += 256) mt[i] = windows[(size_t)blockIdx.x * 624 + i];
  __syncthreads();
  for (unsigned long long k = k0; k < k1; k += 624) {
    uint32_t v = 0;
    if (t < 227) v = mt_twist(mt[t], mt[t + 1], mt[t + 397]);
    __syncthreads();
    if (t < 227) mt[t] = v;
    __syncthreads();
    if (t < 227) v = mt_twist(mt[227 + t], mt[228 + t], mt[t]);
    __syncthreads();
    if (t < 227) mt[227 + t] = v;
    __syncthreads();
    if (t < 170) v = mt_twist(mt[454 + t], mt[t == 169 ? 0 : 455 + t], mt[227 + t]);
    __syncthreads();
    if (t < 170) mt[454 + t] = v;
    __syncthreads();
    const int cnt = (int)min(624ull, k1 - k);
    for (int i = t; i < cnt; i += 256) {
      const unsigned long long q = k + i, row = q / width;
      out[row * pitch + (q - row * width)] = (uint8_t)(mt_temper(mt[i]) >> 24);
    }
    __syncthreads();  // the next twist overwrites mt
  }
}

#endif  // TFG_VOTE_ONLY

}  // namespace tfg
