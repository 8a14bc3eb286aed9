// Jump-ahead for std::mt19937, so that synth_noise (image.hpp:109-116: pixel
// i = rng() >> 24, i in row-major order, std::mt19937 rng(seed)) can be
// generated on the device by independent segments, bit-identical to the
// reference's single sequential generator.
//
// Sequence model. x[0..623] is the seeded state (std::mt19937's
// initialisation); x[t+624] = x[t+397] ^ twist(x[t] & UPPER | x[t+1] & LOWER)
// for t >= 0, and the reference's output i is temper(x[624+i]). The "window"
// at output k is x[k .. k+623]: a generator holding it as its state array
// emits outputs k, k+1, ... after one in-place twist.
//
// Jump. The recurrence is linear over GF(2) on the 19937-bit state (the top
// bit of x[t] and x[t+1..t+623]); its characteristic polynomial phi has
// degree 19937 and is found once per process by Berlekamp-Massey on the top
// bits of the output sequence. With p(z) = z^J mod phi = sum c_i z^i, the
// window J steps ahead is sum c_i * window(k + i) (Horner-free form: step the
// generator 19937 times, XOR-accumulating the windows where c_i = 1). Only
// the low 31 bits of the first word of a window are outside the linear state;
// the twist never reads them.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/texforge_cuda.h"

namespace {

constexpr int kN = 624, kM = 397, kDeg = 19937;
constexpr uint32_t kMatA = 0x9908B0DFu, kUpper = 0x80000000u, kLower = 0x7FFFFFFFu;
constexpr int kWords = (kDeg + 64) / 64;  // residues mod phi: bits [0, kDeg)

using Poly = std::vector<uint64_t>;

inline uint32_t twist_next(uint32_t x0, uint32_t x1, uint32_t xm) {
  const uint32_t y = (x0 & kUpper) | (x1 & kLower);
  return xm ^ (y >> 1) ^ ((y & 1u) ? kMatA : 0u);
}

void seed_window(uint32_t seed, uint32_t* w) {
  w[0] = seed;
  for (int i = 1; i < kN; ++i) w[i] = 1812433253u * (w[i - 1] ^ (w[i - 1] >> 30)) + (uint32_t)i;
}

inline bool bit(const Poly& p, size_t i) { return (p[i >> 6] >> (i & 63)) & 1u; }
inline void flip(Poly& p, size_t i) { p[i >> 6] ^= 1ull << (i & 63); }

// 64 bits of r starting at bit pos (r padded by one word)
inline uint64_t bits64(const Poly& r, size_t pos) {
  const size_t q = pos >> 6, sh = pos & 63;
  return sh ? (r[q] >> sh) | (r[q + 1] << (64 - sh)) : r[q];
}

// dst ^= src << sh (dst sized to hold the result)
void xor_shifted(Poly& dst, const Poly& src, size_t src_bits, size_t sh) {
  const size_t ws = sh >> 6, bs = sh & 63, nw = (src_bits + 63) / 64;
  for (size_t i = 0; i < nw; ++i) {
    const uint64_t v = src[i];
    if (!v) continue;
    dst[i + ws] ^= v << bs;
    if (bs) dst[i + ws + 1] ^= v >> (64 - bs);
  }
}

// Characteristic polynomial of the MT19937 recurrence (bit i = coefficient
// of z^i, degree kDeg), by Berlekamp-Massey over GF(2).
Poly compute_phi() {
  const size_t n = 2 * kDeg + 64;
  std::vector<uint32_t> x(kN + n + 1);
  seed_window(5489u, x.data());
  for (size_t t = 0; t + kN < x.size(); ++t) x[t + kN] = twist_next(x[t], x[t + 1], x[t + kM]);
  // r = the top-bit sequence reversed: r[j] = s[n-1-j], s[t] = x[kN+t] >> 31
  const size_t nw = n / 64 + 4;
  Poly r(nw, 0);
  for (size_t j = 0; j < n; ++j)
    if (x[kN + (n - 1 - j)] >> 31) flip(r, j);
  Poly C(nw, 0), B(nw, 0), T;
  C[0] = B[0] = 1;
  size_t L = 0, m = 1;
  for (size_t N = 0; N < n; ++N) {
    // d = sum_{i=0..L} C_i s[N-i] = sum_i C_i r[n-1-N+i]
    const size_t off = n - 1 - N;
    uint64_t acc = 0;
    for (size_t w = 0; w * 64 <= L; ++w) acc ^= C[w] & bits64(r, off + 64 * w);
    // bits of C above L are zero, and r is padded with zeros past n
    if (!(__builtin_popcountll(acc) & 1)) {
      ++m;
    } else if (2 * L <= N) {
      T = C;
      xor_shifted(C, B, nw * 64 - 128, m);
      L = N + 1 - L;
      B = T;
      m = 1;
    } else {
      xor_shifted(C, B, nw * 64 - 128, m);
      ++m;
    }
  }
  if (L != (size_t)kDeg) return Poly();
  Poly phi(kWords, 0);  // phi = z^L C(1/z)
  for (size_t i = 0; i <= L; ++i)
    if (bit(C, i)) flip(phi, L - i);
  return phi;
}

const Poly& phi_poly() {
  static Poly phi;
  static std::once_flag once;
  std::call_once(once, [] { phi = compute_phi(); });
  return phi;
}

// t (< 2*kDeg bits) mod phi, in place; leaves the kWords residue words
void reduce(Poly& t, const Poly& phi) {
  for (size_t w = t.size(); w-- > 0;) {
    while (t[w]) {
      const size_t i = w * 64 + 63 - (size_t)__builtin_clzll(t[w]);
      if (i < (size_t)kDeg) {
        t.resize(kWords);
        return;
      }
      xor_shifted(t, phi, kDeg + 1, i - kDeg);  // clears bit i, touches only lower bits
    }
  }
  t.resize(kWords);
}

Poly square_mod(const Poly& a, const Poly& phi) {
  Poly t(2 * kWords + 2, 0);
  for (int w = 0; w < kWords; ++w) {
    uint64_t v = a[w];
    if (!v) continue;
    uint64_t lo = 0, hi = 0;
    for (int b = 0; b < 32; ++b) {
      lo |= ((v >> b) & 1ull) << (2 * b);
      hi |= ((v >> (b + 32)) & 1ull) << (2 * b);
    }
    t[2 * w] = lo;
    t[2 * w + 1] = hi;
  }
  reduce(t, phi);
  return t;
}

Poly mulz_mod(Poly a, const Poly& phi) {
  uint64_t carry = 0;
  for (int w = 0; w < kWords; ++w) {
    const uint64_t v = a[w];
    a[w] = (v << 1) | carry;
    carry = v >> 63;
  }
  if (bit(a, kDeg)) {
    for (int w = 0; w < kWords; ++w) a[w] ^= phi[w];
  }
  return a;
}

// z^J mod phi
Poly pow_z(uint64_t J, const Poly& phi) {
  Poly r(kWords, 0);
  r[0] = 1;
  bool one = true;
  for (int b = 63; b >= 0; --b) {
    if (!one) r = square_mod(r, phi);
    if ((J >> b) & 1u) {
      r = mulz_mod(std::move(r), phi);
      one = false;
    }
  }
  return r;
}

// window <- p(A) window
void jump_window(const Poly& p, uint32_t* window) {
  uint32_t ring[kN], acc[kN];
  std::memcpy(ring, window, sizeof(ring));
  std::memset(acc, 0, sizeof(acc));
  int h = 0;
  for (int i = 0; i < kDeg; ++i) {
    if (bit(p, (size_t)i)) {
      const int n1 = kN - h;
      for (int j = 0; j < n1; ++j) acc[j] ^= ring[h + j];
      for (int j = n1; j < kN; ++j) acc[j] ^= ring[j - n1];
    }
    const int h1 = h + 1 == kN ? 0 : h + 1, hm = h + kM >= kN ? h + kM - kN : h + kM;
    ring[h] = twist_next(ring[h], ring[h1], ring[hm]);
    h = h1;
  }
  std::memcpy(window, acc, sizeof(acc));
}

inline uint32_t temper(uint32_t y) {
  y ^= y >> 11;
  y ^= (y << 7) & 0x9D2C5680u;
  y ^= (y << 15) & 0xEFC60000u;
  return y ^ (y >> 18);
}

// out[i] = output (k + i) >> 24 for a generator holding the window at k
void noise_bytes_from(const uint32_t* window, uint64_t count, uint8_t* out) {
  uint32_t mt[kN];
  std::memcpy(mt, window, sizeof(mt));
  for (uint64_t k = 0; k < count; k += kN) {
    for (int i = 0; i < kN - kM; ++i) mt[i] = twist_next(mt[i], mt[i + 1], mt[i + kM]);
    for (int i = kN - kM; i < kN - 1; ++i) mt[i] = twist_next(mt[i], mt[i + 1], mt[i + kM - kN]);
    mt[kN - 1] = twist_next(mt[kN - 1], mt[0], mt[kM - 1]);
    const int cnt = (int)std::min<uint64_t>(kN, count - k);
    for (int i = 0; i < cnt; ++i) out[k + i] = (uint8_t)(temper(mt[i]) >> 24);
  }
}

}  // namespace

extern "C" {

// Host synth_noise over all hardware threads: segment t starts from its
// jump-ahead window. Used by tfg_synth_noise for large images.
int tfg_synth_noise_parallel(size_t n, uint32_t seed, uint8_t* out, int threads) {
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, 64));
  const uint64_t seglen = ((uint64_t)n + nt - 1) / nt;
  const size_t nseg = (size_t)(((uint64_t)n + seglen - 1) / seglen);
  std::vector<uint32_t> win(nseg * kN);
  const int rc = tfg_mt19937_windows(seed, 0, seglen, nseg, win.data(), nt);
  if (rc != TFG_OK) return rc;
  std::vector<std::thread> pool;
  for (size_t s = 0; s < nseg; ++s) {
    const uint64_t k0 = s * seglen, cnt = std::min<uint64_t>(seglen, n - k0);
    pool.emplace_back(noise_bytes_from, win.data() + s * kN, cnt, out + k0);
  }
  for (auto& th : pool) th.join();
  return TFG_OK;
}

int tfg_mt19937_windows(uint32_t seed, uint64_t first, uint64_t stride, size_t count, uint32_t* out,
                        int threads) {
  if (!out || (count > 1 && stride == 0)) return TFG_INVALID_ARGUMENT;
  if (count == 0) return TFG_OK;
  const Poly& phi = phi_poly();
  if (phi.empty()) return TFG_CUDA_ERROR;  // cannot happen: self-check of the BM degree
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<size_t>((size_t)std::min(nt, 64), count);
  const Poly step = count > 1 ? pow_z(stride, phi) : Poly();
  auto run = [&](size_t s0, size_t s1) {
    uint32_t w[kN];
    seed_window(seed, w);
    const uint64_t k0 = first + s0 * stride;
    if (k0) jump_window(pow_z(k0, phi), w);
    for (size_t s = s0; s < s1; ++s) {
      if (s > s0) jump_window(step, w);
      std::memcpy(out + s * kN, w, sizeof(w));
    }
  };
  const size_t per = (count + nt - 1) / nt;
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) {
    const size_t s0 = t * per, s1 = std::min(count, s0 + per);
    if (s0 < s1) pool.emplace_back(run, s0, s1);
  }
  run(0, std::min(count, per));
  for (auto& th : pool) th.join();
  return TFG_OK;
}

}  // extern "C"
