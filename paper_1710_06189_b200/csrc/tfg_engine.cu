// tfg_engine.cu — host side of libtexforge_cuda.so: context, kernel dispatch,
// the Scheme-3 stream pipeline and the C ABI declared in include/texforge_cuda.h.
//
// Reference mapping (R/ = /root/reference/proj/):
//   tfg_glcm          <- compute_glcm_serial / _privatized / _shared
//                        (glcm.hpp:144, parallel.hpp:240, parallel.hpp:143)
//   tfg_glcm_chunked  <- compute_glcm_chunked (pipeline.hpp:246-337)
//   tfg_glcm_bands    <- a loop of single-image calls in the reference
//   tfg_symmetrize / tfg_normalize / tfg_features <- glcm.hpp:150-177, features.hpp:37-69
//   tfg_quantize      <- quantize (image.hpp:55-62)
//   tfg_synth_noise_device <- synth_noise (image.hpp:109-116), on the device
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/texforge_cuda.h"
#include "tfg_kernels.cuh"

namespace {

thread_local std::string g_error;
thread_local size_t g_error_chunk = 0;

struct Failure {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear a non-sticky error so it is not re-reported by the next launch check
  if (e == cudaErrorMemoryAllocation) fail(TFG_OUT_OF_MEMORY, std::string(what) + ": out of device memory");
  fail(TFG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TFG_OK;
  } catch (const Failure& e) {
    g_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_error = "host out of memory";
    return TFG_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_error = e.what();
    return TFG_CUDA_ERROR;
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes <= cap) return p;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    ck(cudaMalloc(&p, bytes), "cudaMalloc");
    // zeroed once at allocation: the row padding and tail slack of the image
    // buffers are read (never voted) by the 16-byte segment loads, so they
    // must hold defined bytes (compute-sanitizer initcheck)
    ck(cudaMemset(p, 0, bytes), "memset");
    // the memset runs on the legacy stream, which does not order against the
    // context's non-blocking streams: finish it before the buffer is handed out
    ck(cudaStreamSynchronize(nullptr), "memset sync");
    cap = bytes;
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes <= cap) return p;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    ck(cudaMallocHost(&p, bytes), "cudaMallocHost");
    cap = bytes;
    return p;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

struct tfg_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t exec = nullptr, copy = nullptr;
  static constexpr int kAux = 4;
  cudaStream_t aux[kAux]{};              // fork streams of tfg_glcm_multi_async (L <= 64)
  cudaEvent_t fork_ev = nullptr, join_ev[kAux]{};
  cudaEvent_t band_ev = nullptr;         // host pipeline: a band's last votes enqueued (early D2H)
  static constexpr int kSlots = 3;
  DevBuf dslot[kSlots];                  // device chunk ring
  HostBuf hslot[kSlots];                 // pinned chunk ring (chunk sources)
  cudaEvent_t copied[kSlots]{}, consumed[kSlots]{};
  DevBuf img;                            // aligned copy of a device/host image
  DevBuf mtwin;                          // synth_noise_device: generator windows per segment
  DevBuf acc;                            // u64 accumulators
  DevBuf sym, probs, feats;              // post-processing outputs
  DevBuf partials;                       // per-CTA sub-GLCMs (large L)
  DevBuf qbuf;                           // quantize in/out
  DevBuf tmp;                            // per-(d,theta) band scratch
  int* d_err = nullptr;                  // [0] async validation flag, [1]/[2] async post flags, [kSyncErr] sync calls
  unsigned int* sync_ctr = nullptr;      // grid-barrier counter of the cooperative vote launches
  // Launches with per-CTA partials (L > 64) share `partials` and the
  // cooperative counters: each one waits for the previous one (on whatever
  // stream it ran) through this event, so two streams or a sync call plus an
  // async call never overlap on the shared scratch.
  cudaEvent_t scratch_ev = nullptr;
  cudaStream_t scratch_stream = nullptr;
  bool scratch_used = false;
  DevBuf errs;
  HostBuf hout;                          // pinned result staging
  std::atomic<uint64_t> launches{0};
  std::mutex mu;
};

namespace {

constexpr int kSyncErr = 3;  // d_err word of the synchronous calls' validation
int* sync_err(tfg_ctx* ctx) { return ctx->d_err + kSyncErr; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void check_levels(int levels, const char* who) {
  if (levels < 2 || levels > 256) fail(TFG_INVALID_ARGUMENT, std::string(who) + ": levels must be in [2, 256]");
}

// glcm.hpp:71-80
bool offset_of(int distance, int angle, long* dr, long* dc) {
  switch (angle) {
    case 0: *dr = 0; *dc = distance; return true;
    case 45: *dr = distance; *dc = -distance; return true;
    case 90: *dr = distance; *dc = 0; return true;
    case 135: *dr = distance; *dc = distance; return true;
    default: return false;
  }
}

void check_angle(int angle) {
  long a, b;
  if (!offset_of(1, angle, &a, &b)) fail(TFG_INVALID_ARGUMENT, "angle must be one of 0, 45, 90, 135");
}

// glcm.hpp:98-104 (check_glcm_inputs)
void check_geometry(size_t width, size_t height, int distance) {
  const size_t d = (size_t)distance;
  if (distance < 1 || d >= width || d >= height)
    fail(TFG_INVALID_ARGUMENT, "glcm: degenerate geometry (d must be in [1, min(width, height)))");
}


int pick_strategy(int levels, unsigned flags) {
  const int forced = (int)((flags >> TFG_STRATEGY_SHIFT) & 0xF);
  if (forced) {
    const bool ok = (forced == TFG_STRAT_COPIES32 && levels <= 32) || (forced == TFG_STRAT_COPIES8 && levels <= 64) ||
                    (forced == TFG_STRAT_COPY1 && levels <= 128) || (forced == TFG_STRAT_PACKED16) ||
                    (forced == TFG_STRAT_P16X16 && levels <= 64);
    if (!ok) fail(TFG_INVALID_ARGUMENT, "strategy does not support these levels");
    return forced;
  }
  if (levels <= 32) return tfg::S_COPIES32;
  if (levels <= 64) return tfg::S_COPIES8;
  if (levels <= 128) return tfg::S_COPY1;
  return tfg::S_PACKED16;
}

// Shared-memory words of a strategy's layout (tfg_kernels.cuh, enum Strat).
size_t hist_words_of(int strat, int levels) {
  const size_t L = (size_t)levels;
  size_t w = 0;
  switch (strat) {
    case tfg::S_COPIES32: w = L * 32 * 32; break;   // cells a + 32b, 32 copies
    case tfg::S_COPIES8: w = L * 64 * 8; break;     // cells b + 64a, 8 copies
    case tfg::S_COPY1: w = L * 128; break;          // cells a + 128b
    case tfg::S_P16X16: w = 32768; break;           // 16 copies x 2048 words (c = 64b + a)
    default: w = std::min<size_t>(L * 256, 32768); break;  // words (a + 256b) & 0x7fff
  }
  return (w + 3) & ~size_t(3);
}

using VoteKernel = void (*)(const tfg::VoteParams);

// The glcm_vote_kernel instantiations live in tfg_vote_q{0..3}.cu (one
// translation unit per quantiser, compiled in parallel): tfg_vote_inst.cu.
}  // namespace
VoteKernel tfg_pick_vote_q0(int strat, int ksel);
VoteKernel tfg_pick_vote_q1(int strat, int ksel);
VoteKernel tfg_pick_vote_q2(int strat, int ksel);
VoteKernel tfg_pick_vote_q3(int strat, int ksel);
namespace {
using JobsKernel = void (*)(const tfg::VoteJobs);
}  // namespace
JobsKernel tfg_pick_jobs_q0(int strat);
JobsKernel tfg_pick_jobs_q1(int strat);
JobsKernel tfg_pick_jobs_q2(int strat);
JobsKernel tfg_pick_jobs_q3(int strat);
JobsKernel tfg_pick_jobs1_q0(int strat, int ksel);
JobsKernel tfg_pick_jobs1_q1(int strat, int ksel);
JobsKernel tfg_pick_jobs1_q2(int strat, int ksel);
JobsKernel tfg_pick_jobs1_q3(int strat, int ksel);
namespace {
JobsKernel pick_jobs(int quant, int strat) {
  switch (quant) {
    case tfg::Q_NONE: return tfg_pick_jobs_q0(strat);
    case tfg::Q_CLAMP: return tfg_pick_jobs_q1(strat);
    case tfg::Q_SHIFT: return tfg_pick_jobs_q2(strat);
    default: return tfg_pick_jobs_q3(strat);
  }
}
// The KSELs one L > 64 multi-job launch may mix (glcm_vote_jobs2_kernel:
// PACKED16 pairs {0,1} {2,3} {5,6} {7,8}; COPY1: one KSEL).
int ksel_group(int strat, int ksel) {
  if (strat != tfg::S_PACKED16 || ksel == 4) return ksel;
  return ksel < 4 ? (ksel & ~1) : 5 + ((ksel - 5) & ~1);
}
JobsKernel pick_jobs1(int quant, int strat, int ksel) {
  switch (quant) {
    case tfg::Q_NONE: return tfg_pick_jobs1_q0(strat, ksel);
    case tfg::Q_CLAMP: return tfg_pick_jobs1_q1(strat, ksel);
    case tfg::Q_SHIFT: return tfg_pick_jobs1_q2(strat, ksel);
    default: return tfg_pick_jobs1_q3(strat, ksel);
  }
}

VoteKernel pick_vote(int quant, int strat, int ksel) {
  switch (quant) {
    case tfg::Q_NONE: return tfg_pick_vote_q0(strat, ksel);
    case tfg::Q_CLAMP: return tfg_pick_vote_q1(strat, ksel);
    case tfg::Q_SHIFT: return tfg_pick_vote_q2(strat, ksel);
    default: return tfg_pick_vote_q3(strat, ksel);
  }
}
template <int Q>
VoteKernel pick_g(int ksel) {
  switch (ksel >= 5 ? ksel - 5 : ksel) {  // Scheme 1 always loads c0
    case 0: return tfg::glcm_vote_global_kernel<Q, 0>;
    case 1: return tfg::glcm_vote_global_kernel<Q, 1>;
    case 2: return tfg::glcm_vote_global_kernel<Q, 2>;
    case 3: return tfg::glcm_vote_global_kernel<Q, 3>;
    default: return tfg::glcm_vote_global_kernel<Q, 4>;
  }
}
VoteKernel pick_global(int quant, int ksel) {
  switch (quant) {
    case tfg::Q_NONE: return pick_g<tfg::Q_NONE>(ksel);
    case tfg::Q_CLAMP: return pick_g<tfg::Q_CLAMP>(ksel);
    case tfg::Q_SHIFT: return pick_g<tfg::Q_SHIFT>(ksel);
    default: return pick_g<tfg::Q_MUL>(ksel);
  }
}

// Shared tail pool of the cooperative vote launches: per-band counters sit
// 128 bytes past the grid-barrier counter (its own L2 line); all of them are
// zeroed once and re-armed by each launch's last CTA.
constexpr size_t kPoolCtrOffset = 32;
constexpr int kMaxPoolBands = 1024;
#ifndef TFG_POOL_PCT
#define TFG_POOL_PCT 20
#endif
// Percentage of the interior items in the pool (TEXFORGE_POOL_PCT overrides
// it for tuning; 0 disables the pool).
long long pool_pct() {
  static const long long v = [] {
    const char* e = std::getenv("TEXFORGE_POOL_PCT");
    const long long x = e ? std::atoll(e) : (long long)TFG_POOL_PCT;
    return std::min<long long>(std::max<long long>(x, 0), 90);
  }();
  return v;
}

// Line-aligned interior segments (make_geometry); TEXFORGE_ALIGN=0 turns
// them off for A/B timing.
bool align_interior_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("TEXFORGE_ALIGN");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Every vote kernel gets the full 227 KB dynamic shared-memory opt-in once;
// occupancy is then queried per (kernel, smem) pair.
std::mutex g_kinfo_mu;
std::vector<VoteKernel> g_kopted;
std::vector<std::pair<std::pair<VoteKernel, size_t>, int>> g_kocc;

int occupancy_for(const void* fn_ptr, size_t smem) {
  VoteKernel fn = reinterpret_cast<VoteKernel>(const_cast<void*>(fn_ptr));
  std::lock_guard<std::mutex> lk(g_kinfo_mu);
  for (auto& e : g_kocc)
    if (e.first.first == fn && e.first.second == smem) return e.second;
  if (std::find(g_kopted.begin(), g_kopted.end(), fn) == g_kopted.end()) {
    int dev = 0, optin = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr");
    cudaFuncAttributes fa{};
    ck(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(fn)), "cudaFuncGetAttributes");
    ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            optin - (int)fa.sharedSizeBytes),
       "cudaFuncSetAttribute");
    g_kopted.push_back(fn);
  }
  int bps = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, reinterpret_cast<const void*>(fn), tfg::kThreads, smem),
     "occupancy");
  if (bps < 1) fail(TFG_CUDA_ERROR, "vote kernel cannot be resident (shared memory / registers)");
  g_kocc.push_back({{fn, smem}, bps});
  return bps;
}

int floor_div(long a, long b) {
  long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return (int)q;
}

// Geometry of one (d, theta) vote over a buffer of `height` rows of which
// anchor rows [0, row_end) are owned (vote_anchor_rows, glcm.hpp:110-130).
// CUTLASS-style FastDivmod constants: q = umulhi(n, mul) >> shr for n < 2^31
// (d == 1: mul = 0, tfg::fast_div returns n).
void fastdiv_consts(uint32_t dv, uint32_t* mul, uint32_t* shr) {
  if (dv <= 1) {
    *mul = 0;
    *shr = 0;
    return;
  }
  uint32_t l = 0;
  while ((1ull << l) < dv) ++l;  // ceil(log2 d)
  const uint32_t pw = 31 + l;
  *mul = (uint32_t)(((1ull << pw) + dv - 1) / dv);
  *shr = pw - 32;
}

struct VoteGeometry {
  tfg::VoteParams p{};
  int ksel = 4;
  bool empty = false;
};

VoteGeometry make_geometry(size_t width, size_t height, size_t pitch, size_t row_end, int levels,
                           int pixel_levels, int distance, int angle, bool align_interior = false) {
  VoteGeometry g;
  long dr, dc;
  offset_of(distance, angle, &dr, &dc);
  const long d = distance;
  tfg::VoteParams& p = g.p;
  p.pitch = pitch;
  p.buf_bytes = (unsigned long long)pitch * height;
  p.levels = levels;
  p.dr = (int)dr;
  const long qq = floor_div(dc, 16);
  p.qoff = (int)(qq * 16);
  const long rem = dc - qq * 16;  // 0..15
  g.ksel = rem == 0 ? 4 : (int)(rem >> 2);
  if (g.ksel != 4 && dr == 0 && qq == 0) g.ksel += 5;  // theta = 0, d < 16: first ref segment = anchor
  p.sbits = (int)((rem & 3) * 8);
  p.ref_off = (long long)dr * (long long)pitch + p.qoff;
  p.col_begin = dc < 0 ? (int)d : 0;
  p.col_end = dc > 0 ? (int)(width - d) : (int)width;
  const long row_limit = (long)height - dr;
  const long nrows = std::max<long>(0, std::min<long>((long)row_end, row_limit));
  p.nrows = (int)nrows;
  p.ch0 = p.col_begin / 16;
  p.nch = (p.col_end + 15) / 16 - p.ch0;
  p.items = (long long)nrows * p.nch;
  if (p.items >= (1ll << 31))
    fail(TFG_INVALID_ARGUMENT, "glcm: image too large for one launch (>= 2^31 16-pixel segments); split it into chunks");
  g.empty = p.items == 0 || p.col_end <= p.col_begin;
  fastdiv_consts((uint32_t)std::max(p.nch, 1), &p.div_mul, &p.div_shr);
  // two-pass split (glcm_vote_kernel): interior segments [1, nch-1) of every
  // row run unmasked in the main pass; rows too narrow for 64-segment double
  // batches go entirely through the edge pass
  if (p.nch >= 66) {
    p.js = 1;
    p.ni = p.nch - 2;
    if (align_interior && pitch % 128 == 0) {
      // interior segments start on a 128-byte line (the rows do, when the
      // buffer is 128-byte aligned: launch_vote checks the pointer), and
      // ni % 8 == 0 keeps every double batch (64 segments) line-aligned, so
      // a warp's 512-byte LDG.128 touches 4 lines instead of 5. The up to
      // 14 extra edge segments per row go through the masked edge pass.
      const int js = 1 + ((8 - ((p.ch0 + 1) & 7)) & 7);
      const int ni = (p.nch - 1 - js) / 8 * 8;
      if (ni >= 64) {
        p.js = js;
        p.ni = ni;
      }
    }
    p.ne = p.nch - p.ni;
  } else {
    p.js = 1;
    p.ni = 0;
    p.ne = std::max(p.nch, 1);
  }
  p.main_items = (long long)nrows * p.ni;
  p.edge_items = (long long)nrows * p.ne;
  p.pool_beg = p.main_items;  // no shared pool unless launch_vote sets one
  p.pool_dbl = 0;
  p.pool_ctr = nullptr;
  fastdiv_consts((uint32_t)std::max(p.ni, 1), &p.ni_mul, &p.ni_shr);
  fastdiv_consts((uint32_t)p.ne, &p.ne_mul, &p.ne_shr);
  // quantisation mode
  (void)pixel_levels;
  return g;
}

int quant_mode(int pixel_levels, int levels, uint32_t* mask, int* shift, int* lgp = nullptr) {
  *mask = 0;
  *shift = 0;
  if (levels == 256) return tfg::Q_NONE;
  if (pixel_levels == levels) {
    *mask = (uint32_t)(levels - 1) * 0x01010101u;
    return tfg::Q_CLAMP;
  }
  if ((levels & (levels - 1)) == 0) {
    int lg = 0;
    while ((1 << lg) < levels) ++lg;
    *shift = 8 - lg;
    *mask = (uint32_t)(levels - 1) * 0x01010101u;
    if (lgp) *lgp = lg;
    return tfg::Q_SHIFT;
  }
  return tfg::Q_MUL;
}

// Orders the launches that share the context's per-CTA partials and
// cooperative counters (L > 64): the launch on `s` first waits for the
// previous such launch when that ran on another stream, and records the
// event for the next one when it goes out of scope. Skipped while `s` is
// being captured into a CUDA graph (the graph itself fixes the order).
struct ScratchOrder {
  tfg_ctx* ctx;
  cudaStream_t s;
  bool on;
  ScratchOrder(tfg_ctx* c, cudaStream_t st, bool use) : ctx(c), s(st), on(use) {
    if (!on) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      on = false;
      return;
    }
    if (ctx->scratch_used && ctx->scratch_stream != s)
      ck(cudaStreamWaitEvent(s, ctx->scratch_ev, 0), "wait scratch");
  }
  ~ScratchOrder() {
    if (!on) return;
    if (cudaEventRecord(ctx->scratch_ev, s) == cudaSuccess) {
      ctx->scratch_stream = s;
      ctx->scratch_used = true;
    } else {
      cudaGetLastError();
    }
  }
};

// Geometry, quantiser and layout of one (d, theta) vote (launch_vote and
// launch_vote_jobs share it).
struct VotePrep {
  VoteGeometry g;
  int quant = 0;
};
VotePrep prepare_vote(const uint8_t* d_img, size_t width, size_t height, size_t pitch, size_t band_stride,
                      int n_bands, size_t row_end, int pixel_levels, int levels, int distance, int angle,
                      unsigned flags, unsigned long long* d_glcm) {
  const bool aligned = align_interior_enabled() && reinterpret_cast<uintptr_t>(d_img) % 128 == 0 &&
                       (n_bands == 1 || band_stride % 128 == 0);
  VotePrep v;
  v.g = make_geometry(width, height, pitch, row_end, levels, pixel_levels, distance, angle, aligned);
  tfg::VoteParams& p = v.g.p;
  p.img = d_img;
  p.band_stride = band_stride;
  p.glcm = d_glcm;
  int lg = 0;
  v.quant = quant_mode(pixel_levels, levels, &p.qmask, &p.qshift, &lg);
  if (v.quant == tfg::Q_SHIFT && !(flags & TFG_SCHEME_GLOBAL)) {
    // the scaled side of a layout: ((v >> s) & m) << sc == (v >> (s - sc)) & (m << sc); s >= sc
    // holds because each layout is only used for L <= 2^(8 - sc).
    const int strat = pick_strategy(levels, flags);
    p.qshift_scaled = p.qshift - tfg::strat_scale(strat);
    // reference side of item_words: COPIES8 scales it, the others do not
    const bool ref_scaled = strat == tfg::S_COPIES8;
    p.rshift = p.sbits + (ref_scaled ? p.qshift_scaled : p.qshift);
    p.rmask = ref_scaled ? (p.qmask << tfg::strat_scale(strat)) : p.qmask;
  }
  return v;
}

// Fewest 16-pixel items per CTA (caps the grid of small images; a CTA's
// fixed cost is its histogram zeroing and merge). TEXFORGE_MIN_CTA_ITEMS
// overrides it for A/B timing.
long long min_cta_items() {
  static const long long v = [] {
    const char* e = std::getenv("TEXFORGE_MIN_CTA_ITEMS");
    return e ? std::max(32ll, std::atoll(e)) : 512ll;  // c1 (512^2): 21.3 -> 25.5 Gpairs/s vs 2048
  }();
  return v;
}

// Multi-job launches (glcm_vote_jobs_kernel); TEXFORGE_JOBS=0 launches every
// (d, theta) on its own for A/B timing.
bool jobs_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("TEXFORGE_JOBS");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Enqueues n (d, theta) votes of the same image (or band batch) as ONE
// glcm_vote_jobs_kernel launch: job t adds into d_counts + t * per_dt (band
// b at + b * L^2). Layouts with per-CTA partials (L > 64) go out as one
// cooperative launch when the (job, band) rows fit one wave; returns false
// when it does not apply and the caller launches per (d, theta).
bool launch_vote_jobs(tfg_ctx* ctx, const uint8_t* d_img, size_t width, size_t height, size_t pitch,
                      size_t band_stride, int n_bands, size_t row_end, int pixel_levels, const int* levels,
                      const int* distances, const int* angles, unsigned long long* const* outs, int n,
                      unsigned flags, cudaStream_t s) {
  if (n < 2 || n > tfg::kMaxJobs || (flags & TFG_SCHEME_GLOBAL) || !jobs_enabled()) return false;
  // one kernel instantiation: every job needs the same quantiser and layout
  int quant = -1, strat = -1;
  size_t words = 0;
  for (int t = 0; t < n; ++t) {
    uint32_t qm = 0;
    int qs = 0;
    const int q = quant_mode(pixel_levels, levels[t], &qm, &qs);
    const int st = pick_strategy(levels[t], flags);
    if ((quant >= 0 && q != quant) || (strat >= 0 && st != strat)) return false;
    quant = q;
    strat = st;
    words = std::max(words, hist_words_of(st, levels[t]));
  }
  const bool partials = strat == tfg::S_PACKED16 || strat == tfg::S_COPY1;
  const size_t smem = words * 4 + tfg::kTmaBytes;
  tfg::VoteJobs jp{};
  int m = 0;
  long long max_items = 0;
  for (int t = 0; t < n; ++t) {
    VotePrep v = prepare_vote(d_img, width, height, pitch, band_stride, n_bands, row_end, pixel_levels, levels[t],
                              distances[t], angles[t], flags, outs[t]);
    if (v.g.empty) continue;
    v.g.p.hist_words = (int)hist_words_of(strat, levels[t]);
    jp.job[m] = v.g.p;
    jp.ksel[m] = v.g.ksel;
    max_items = std::max(max_items, v.g.p.items);
    ++m;
  }
  if (m == 0) return true;
  // partial layouts: one KSEL group per launch (glcm_vote_jobs1/2_kernel; launch_job_set groups by it)
  for (int j = 1; j < m && partials; ++j)
    if (ksel_group(strat, jp.ksel[j]) != ksel_group(strat, jp.ksel[0])) return false;
  JobsKernel fn = partials ? pick_jobs1(quant, strat, jp.ksel[0]) : pick_jobs(quant, strat);
  if (!fn) return false;
  const int bps = occupancy_for(reinterpret_cast<const void*>(fn), smem);
  // one wave of CTAs split evenly over the (job, band) units (launch_vote's rule per unit)
  const long long units = (long long)m * n_bands;
  const long long slots = (long long)ctx->num_sms * bps;
  // L > 64 layouts (per-CTA partials): one cooperative launch, every unit's
  // partials reduced in-kernel behind one grid barrier; the grid must be
  // co-resident and every unit needs its own pool counter
  if (partials) {
    static const bool coop = [] {
      const char* e = std::getenv("TEXFORGE_COOP");
      const char* j = std::getenv("TEXFORGE_JOBS_COOP");  // A/B knob: 0 = per-(d, theta) launches at L > 64
      return !(e && e[0] == '0') && !(j && j[0] == '0');
    }();
    if (!coop || units > slots || units > kMaxPoolBands) return false;
    const long long per = std::max<long long>(
        1, std::min<long long>(slots / units, (max_items + min_cta_items() - 1) / min_cta_items()));
    const bool packed = strat == tfg::S_PACKED16;
    const size_t per_cta = packed ? words : (size_t)jp.job[0].levels * jp.job[0].levels;
    for (int j = 0; j < m; ++j)  // one partial size per launch
      if (jp.job[j].levels != jp.job[0].levels) return false;
    tfg::VoteParams* ps = jp.job;
    ScratchOrder order(ctx, s, true);
    uint32_t* scratch = static_cast<uint32_t*>(ctx->partials.get((size_t)per * units * per_cta * 4));
    for (int j = 0; j < m; ++j) {
      tfg::VoteParams& p = ps[j];
      const long long pool = p.main_items * pool_pct() / 100 / 256 * 4;  // whole grabs
      p.pool_dbl = (uint32_t)std::min<long long>(pool, 1 << 24);
      p.pool_beg = p.main_items - 64LL * p.pool_dbl;
      p.pool_ctr = ctx->sync_ctr + kPoolCtrOffset;
      p.sync_ctr = ctx->sync_ctr;
      p.partials = scratch;
      p.main_per_cta = ((p.pool_beg + per - 1) / per + 63) / 64 * 64;
      p.edge_per_cta = (p.edge_items + per - 1) / per;
    }
    jp.nbands = n_bands;
    jp.njobs = m;
    void* args[] = {&jp};
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3((unsigned)per, (unsigned)units),
                                                      dim3(tfg::kThreads), args, smem, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      cudaMemsetAsync(ctx->sync_ctr, 0, (kPoolCtrOffset + kMaxPoolBands) * sizeof(unsigned int), s);
      ck(e, "glcm_vote_jobs_kernel cooperative launch");
    }
    ctx->launches++;
    return true;
  }
  static const long long waves = [] {
    const char* e = std::getenv("TEXFORGE_JOBS_WAVES");  // A/B knob: CTA waves when units exceed the SM slots
    return e ? std::max(1ll, std::atoll(e)) : 8ll;
  }();
  long long per = units < slots ? std::max<long long>(1, slots / units)
                                : std::max<long long>(1, (waves * slots + units - 1) / units);
  per = std::max<long long>(1, std::min<long long>(per, (max_items + min_cta_items() - 1) / min_cta_items()));
  if (units > 65535) return false;
  for (int j = 0; j < m; ++j) {
    tfg::VoteParams& p = jp.job[j];
    p.main_per_cta = ((p.pool_beg + per - 1) / per + 63) / 64 * 64;
    p.edge_per_cta = (p.edge_items + per - 1) / per;
  }
  jp.nbands = n_bands;
  jp.njobs = m;
  fn<<<dim3((unsigned)per, (unsigned)units), tfg::kThreads, smem, s>>>(jp);
  ck(cudaGetLastError(), "glcm_vote_jobs_kernel launch");
  ctx->launches++;
  return true;
}

void launch_job_set(tfg_ctx* ctx, const uint8_t* d_img, size_t width, size_t height, size_t pitch,
                    size_t band_stride, int n_bands, size_t row_end, int pixel_levels, const int* levels,
                    const int* distances, const int* angles, unsigned long long* const* outs, int n_jobs,
                    unsigned flags, cudaStream_t s);

// The common case: n (d, theta) at one L, job t adding into d_counts + t * per_dt.
// L > 64: the jobs go out grouped by KSEL (launch_job_set), so this returns true.
bool launch_vote_jobs(tfg_ctx* ctx, const uint8_t* d_img, size_t width, size_t height, size_t pitch,
                      size_t band_stride, int n_bands, size_t row_end, int pixel_levels, int levels,
                      const int* distances, const int* angles, int n, unsigned flags, unsigned long long* d_counts,
                      size_t per_dt, cudaStream_t s) {
  if (n < 2 || n > tfg::kMaxJobs) return false;
  int lv[tfg::kMaxJobs];
  unsigned long long* outs[tfg::kMaxJobs];
  for (int t = 0; t < n; ++t) {
    lv[t] = levels;
    outs[t] = d_counts + (size_t)t * per_dt;
  }
  if ((size_t)levels * levels > 4096 && !(flags & TFG_SCHEME_GLOBAL) && jobs_enabled()) {
    launch_job_set(ctx, d_img, width, height, pitch, band_stride, n_bands, row_end, pixel_levels, lv, distances,
                   angles, outs, n, flags, s);
    return true;
  }
  return launch_vote_jobs(ctx, d_img, width, height, pitch, band_stride, n_bands, row_end, pixel_levels, lv, distances,
                          angles, outs, n, flags, s);
}

// Enqueue the vote of one (d, theta) for n_bands bands into d_glcm (added).
void launch_vote(tfg_ctx* ctx, const uint8_t* d_img, size_t width, size_t height, size_t pitch,
                 size_t band_stride, int n_bands, size_t row_end, int pixel_levels, int levels,
                 int distance, int angle, unsigned flags, unsigned long long* d_glcm, cudaStream_t s) {
  VotePrep v = prepare_vote(d_img, width, height, pitch, band_stride, n_bands, row_end, pixel_levels, levels,
                            distance, angle, flags, d_glcm);
  VoteGeometry& g = v.g;
  if (g.empty) return;
  tfg::VoteParams& p = g.p;
  const int quant = v.quant;
  const size_t cells = (size_t)levels * levels;

  if (flags & TFG_SCHEME_GLOBAL) {
    VoteKernel fn = pick_global(quant, g.ksel);
    const long long blocks = std::min<long long>((p.items + 255) / 256, (long long)ctx->num_sms * 16);
    dim3 grid((unsigned)std::max<long long>(blocks, 1), (unsigned)n_bands);
    fn<<<grid, 256, 0, s>>>(p);
    ck(cudaGetLastError(), "glcm_vote_global_kernel launch");
    ctx->launches++;
    return;
  }

  const int strat = pick_strategy(levels, flags);
  const size_t words = hist_words_of(strat, levels);
  const size_t smem = words * 4 + tfg::kTmaBytes;
  p.hist_words = (int)words;
  VoteKernel fn = pick_vote(quant, strat, g.ksel);
  const int bps = occupancy_for(reinterpret_cast<const void*>(fn), smem);
  // persistent-style grid: at most one wave of CTAs per band set, and no CTA
  // with less than one round of work.
  // One wave of persistent CTAs when the bands fit in it; otherwise ~8 waves,
  // so the last, partial wave costs <= ~1/16 of the time (256 bands on 148
  // SMs at one CTA per band would leave the second wave 27% idle).
  const long long slots = (long long)ctx->num_sms * bps;
  long long per_band = n_bands < slots ? std::max<long long>(1, slots / std::max(n_bands, 1))
                                       : std::max<long long>(1, (8 * slots + n_bands - 1) / n_bands);
  per_band = std::min<long long>(per_band, (p.items + min_cta_items() - 1) / min_cta_items());
  per_band = std::max<long long>(per_band, 1);
  const bool use_partials = cells > 4096;
  // With partials and a grid that is co-resident (one CTA per SM slot), the
  // kernel reduces the partials itself behind a grid barrier (cooperative
  // launch guarantees co-residency); larger grids use the reduce kernels.
  // TEXFORGE_COOP=0: A/B knob for the L > 64 merge, split-K reduce kernels
  // instead of the cooperative launch with the in-kernel reduce (measured:
  // a cooperative launch costs the same as a plain one; the fixed cost of an
  // L=256 launch is ~18 us in-kernel vs ~10 us split-K, but 135 vs 156 us at
  // 16384^2: tools/launch_overhead.py)
  static const int coop_mode = [] {
    const char* e = std::getenv("TEXFORGE_COOP");
    return e ? std::atoi(e) : 1;
  }();
  const bool in_kernel_reduce = coop_mode != 0 && use_partials && per_band * n_bands <= (long long)ctx->num_sms * bps;
  if (in_kernel_reduce && n_bands <= kMaxPoolBands &&
      (strat == tfg::S_PACKED16 || strat == tfg::S_COPY1)) {  // the layouts with the pool loop
    // The grid barrier waits for the slowest CTA, so the last pool_pct % of
    // each band's interior items go to a shared pool that CTAs drain after
    // their own contiguous range (counters zeroed with the barrier's).
    const long long pool = p.main_items * pool_pct() / 100 / 256 * 4;  // whole grabs
    p.pool_dbl = (uint32_t)std::min<long long>(pool, 1 << 24);
    p.pool_beg = p.main_items - 64LL * p.pool_dbl;
    p.pool_ctr = ctx->sync_ctr + kPoolCtrOffset;
  }
  p.main_per_cta = ((p.pool_beg + per_band - 1) / per_band + 63) / 64 * 64;
  p.edge_per_cta = (p.edge_items + per_band - 1) / per_band;
  const bool packed_partials = use_partials && strat == tfg::S_PACKED16;
  ScratchOrder order(ctx, s, use_partials);
  if (use_partials) {
    const size_t per_cta = packed_partials ? words : cells;
    const size_t bytes = (size_t)per_band * n_bands * per_cta * 4;
    p.partials = static_cast<uint32_t*>(ctx->partials.get(bytes));
  }
  dim3 grid((unsigned)per_band, (unsigned)n_bands);
  if (in_kernel_reduce) {
    // counters are zero here: zeroed at context creation, re-armed by the
    // last CTA of every cooperative launch (glcm_vote_kernel epilogue)
    p.sync_ctr = ctx->sync_ctr;
    void* args[] = {&p};
    const cudaError_t e =
        cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), grid, dim3(tfg::kThreads), args, smem, s);
    if (e != cudaSuccess) {
      // a launch that did not run leaves the counters as they were; re-zero
      // them anyway so no later launch can spin on a stale arrival count
      cudaGetLastError();
      cudaMemsetAsync(ctx->sync_ctr, 0, (kPoolCtrOffset + kMaxPoolBands) * sizeof(unsigned int), s);
      ck(e, "glcm_vote_kernel cooperative launch");
    }
    ctx->launches++;
    return;
  }
  fn<<<grid, tfg::kThreads, smem, s>>>(p);
  ck(cudaGetLastError(), "glcm_vote_kernel launch");
  ctx->launches++;
  if (packed_partials) {
    // split-K over the per-CTA partials: ~2 waves of 256-thread CTAs
    const int xblocks = (int)((words / 4 + 255) / 256);
    int splits = std::max(1, (int)std::min<long long>(per_band, (2LL * ctx->num_sms * 8) / std::max(xblocks * n_bands, 1)));
    const int per_split = (int)((per_band + splits - 1) / splits);
    splits = (int)((per_band + per_split - 1) / per_split);
    dim3 rgrid((unsigned)xblocks, (unsigned)splits, (unsigned)n_bands);
    tfg::glcm_reduce_packed_kernel<<<rgrid, 256, 0, s>>>(p.partials, (int)per_band, (int)words, levels, per_split,
                                                          d_glcm);
    ck(cudaGetLastError(), "glcm_reduce_packed_kernel launch");
    ctx->launches++;
  } else if (use_partials) {
    const long long total = (long long)cells * n_bands;
    const int rblocks = (int)std::min<long long>((total + 255) / 256, (long long)ctx->num_sms * 8);
    tfg::glcm_reduce_partials_kernel<<<rblocks, 256, 0, s>>>(p.partials, (int)per_band, (int)cells,
                                                            n_bands, d_glcm);
    ck(cudaGetLastError(), "glcm_reduce_partials_kernel launch");
    ctx->launches++;
  }
}

// Enqueues jobs with per-job (L, d, theta), job t adding into outs[t] (band b
// at + b * L_t^2). Jobs that share a kernel instantiation go out as multi-job
// launches of up to kMaxJobs, in any order: the key is (quantiser, layout)
// and, for the layouts with per-CTA partials, also (L, KSEL group) — one
// partial size and one KSEL group (ksel_group) per launch. Singletons and jobs
// no multi-job launch takes get one launch each (all ordered on `s`).
void launch_job_set(tfg_ctx* ctx, const uint8_t* d_img, size_t width, size_t height, size_t pitch,
                    size_t band_stride, int n_bands, size_t row_end, int pixel_levels, const int* levels,
                    const int* distances, const int* angles, unsigned long long* const* outs, int n_jobs,
                    unsigned flags, cudaStream_t s) {
  std::vector<long long> key(n_jobs);
  for (int t = 0; t < n_jobs; ++t) {
    uint32_t qm = 0;
    int qs = 0;
    const int q = quant_mode(pixel_levels, levels[t], &qm, &qs);
    const int st = pick_strategy(levels[t], flags);
    long long k = q * 16 + st;
    if (st == tfg::S_PACKED16 || st == tfg::S_COPY1) {
      const VoteGeometry g = make_geometry(width, height, pitch, row_end, levels[t], pixel_levels, distances[t],
                                           angles[t]);
      k += 256LL * levels[t] + 65536LL * (ksel_group(st, g.ksel) + 1);
    }
    key[t] = k;
  }
  std::vector<char> done(n_jobs, 0);
  std::vector<int> idx;
  for (int t = 0; t < n_jobs; ++t) {
    if (done[t]) continue;
    idx.clear();
    for (int u = t; u < n_jobs; ++u)
      if (!done[u] && key[u] == key[t]) {
        idx.push_back(u);
        done[u] = 1;
      }
    size_t i = 0;
    while (i < idx.size()) {
      int n = (int)std::min<size_t>(idx.size() - i, tfg::kMaxJobs);
      int lv[tfg::kMaxJobs], dd[tfg::kMaxJobs], aa[tfg::kMaxJobs];
      unsigned long long* oo[tfg::kMaxJobs];
      for (int j = 0; j < n; ++j) {
        const int u = idx[i + j];
        lv[j] = levels[u];
        dd[j] = distances[u];
        aa[j] = angles[u];
        oo[j] = outs[u];
      }
      while (n > 1 && !launch_vote_jobs(ctx, d_img, width, height, pitch, band_stride, n_bands, row_end, pixel_levels,
                                         lv, dd, aa, oo, n, flags, s))
        --n;
      if (n == 1)
        launch_vote(ctx, d_img, width, height, pitch, band_stride, n_bands, row_end, pixel_levels, lv[0], dd[0],
                    aa[0], flags, oo[0], s);
      i += n;
    }
  }
}

void launch_validate(tfg_ctx* ctx, const uint8_t* d_img, size_t width, size_t rows, size_t pitch,
                     size_t band_stride, int n_bands, int levels, int* d_err, cudaStream_t s) {
  if (levels == 256) return;
  const long long items = (long long)rows * ((width + 15) / 16);
  const int blocks = (int)std::min<long long>((items + 255) / 256, (long long)ctx->num_sms * 8);
  dim3 grid(std::max(blocks, 1), n_bands);
  tfg::validate_levels_kernel<<<grid, 256, 0, s>>>(d_img, pitch, (int)width, (long long)rows, band_stride,
                                                   levels, d_err);
  ck(cudaGetLastError(), "validate_levels_kernel launch");
  ctx->launches++;
}

size_t round16(size_t v) { return (v + 15) & ~size_t(15); }

void check_dts(const int* distances, const int* angles, int n_dt, size_t width, size_t height) {
  if (n_dt < 1 || !distances || !angles) fail(TFG_INVALID_ARGUMENT, "glcm: need at least one (distance, angle)");
  for (int i = 0; i < n_dt; ++i) {
    check_angle(angles[i]);
    check_geometry(width, height, distances[i]);
  }
}

void check_pixel_levels(int pixel_levels, int levels) {
  if (pixel_levels != 256 && pixel_levels != levels)
    fail(TFG_INVALID_ARGUMENT, "glcm: image levels do not match params levels");
}

// 0 pageable host, 1 pinned host, 2 device, 3 managed (cudaPointerGetAttributes).
int host_memory_kind(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  switch (a.type) {
    case cudaMemoryTypeHost: return 1;
    case cudaMemoryTypeDevice: return 2;
    case cudaMemoryTypeManaged: return 3;
    default: return 0;
  }
}

// Post-processing of n GLCMs resident at d_counts; results to host buffers.
// counts_done: leading GLCMs whose counts the host pipeline already sent to
// the (pinned) counts_out on ctx->aux[0] (plain counts only).
void finish(tfg_ctx* ctx, unsigned long long* d_counts, int n, int levels, unsigned flags,
            uint64_t* counts_out, double* probs_out, double* feats_out, cudaStream_t s, size_t counts_done = 0) {
  const size_t cells = (size_t)levels * levels;
  unsigned long long* d_final = d_counts;
  if (flags & TFG_SYMMETRIC) {
    d_final = static_cast<unsigned long long*>(ctx->sym.get(n * cells * 8));
    dim3 grid((unsigned)std::min<size_t>((cells + 255) / 256, 1024), (unsigned)n);
    tfg::symmetrize_kernel<<<grid, 256, 0, s>>>(d_counts, levels, d_final);
    ck(cudaGetLastError(), "symmetrize launch");
    ctx->launches++;
  }
  const bool want_probs = (flags & (TFG_NORMALIZE | TFG_FEATURES)) != 0;
  int* d_errs = nullptr;
  double* d_probs = nullptr;
  double* d_feats = nullptr;
  if (want_probs) {
    d_errs = static_cast<int*>(ctx->errs.get(2 * n * sizeof(int)));
    ck(cudaMemsetAsync(d_errs, 0, 2 * n * sizeof(int), s), "memset");
    d_probs = static_cast<double*>(ctx->probs.get(n * cells * 8));
    tfg::normalize_kernel<<<n, 1024, 0, s>>>(d_final, levels, d_probs, d_errs);
    ck(cudaGetLastError(), "normalize launch");
    ctx->launches++;
    if (flags & TFG_FEATURES) {
      d_feats = static_cast<double*>(ctx->feats.get(n * 5 * 8));
      tfg::features_kernel<<<n, 1024, 0, s>>>(d_probs, levels, d_feats, d_errs + n);
      ck(cudaGetLastError(), "features launch");
      ctx->launches++;
    }
  }
  // stage everything through pinned memory, one sync
  const size_t b_counts = n * cells * 8, b_probs = want_probs ? n * cells * 8 : 0;
  const size_t b_feats = d_feats ? n * 5 * 8 : 0, b_err = want_probs ? 2 * n * sizeof(int) : 0;
  char* h = static_cast<char*>(ctx->hout.get(b_counts + b_probs + b_feats + b_err + 64));
  // a pinned caller buffer receives the counts by DMA directly (no staging copy)
  const bool counts_direct = counts_out && host_memory_kind(counts_out) == 1;
  const size_t b_done = counts_direct ? counts_done * cells * 8 : 0;
  ck(cudaMemcpyAsync(counts_direct ? static_cast<void*>(reinterpret_cast<char*>(counts_out) + b_done)
                                   : static_cast<void*>(h),
                     reinterpret_cast<const char*>(d_final) + b_done, b_counts - b_done, cudaMemcpyDeviceToHost, s),
     "D2H counts");
  if (b_probs) ck(cudaMemcpyAsync(h + b_counts, d_probs, b_probs, cudaMemcpyDeviceToHost, s), "D2H probs");
  if (b_feats) ck(cudaMemcpyAsync(h + b_counts + b_probs, d_feats, b_feats, cudaMemcpyDeviceToHost, s), "D2H feats");
  if (b_err) ck(cudaMemcpyAsync(h + b_counts + b_probs + b_feats, d_errs, b_err, cudaMemcpyDeviceToHost, s), "D2H err");
  ck(cudaStreamSynchronize(s), "stream sync");
  if (b_done) ck(cudaStreamSynchronize(ctx->aux[0]), "stream sync");
  if (b_err) {
    const int* e = reinterpret_cast<const int*>(h + b_counts + b_probs + b_feats);
    for (int i = 0; i < n; ++i)
      if (e[i]) fail(TFG_INVALID_ARGUMENT, "normalize: all-zero matrix");
    if (d_feats)
      for (int i = 0; i < n; ++i)
        if (e[n + i]) fail(TFG_INVALID_ARGUMENT, "extract_features: input is not normalized");
  }
  if (counts_out && !counts_direct) std::memcpy(counts_out, h, b_counts);
  if (probs_out && b_probs) std::memcpy(probs_out, h + b_counts, b_probs);
  if (feats_out && b_feats) std::memcpy(feats_out, h + b_counts + b_probs, b_feats);
}

// The synchronous calls validate pre-quantised input into their own error
// word (d_err[kSyncErr], zeroed on the call's stream before its first
// validation); d_err[0] belongs to the *_async API and tfg_check_async_errors.
void clear_sync_flag(tfg_ctx* ctx, cudaStream_t s) {
  ck(cudaMemsetAsync(sync_err(ctx), 0, sizeof(int), s), "memset");
}
void check_sync_flag(tfg_ctx* ctx, cudaStream_t s) {
  int flag = 0;
  ck(cudaMemcpyAsync(&flag, sync_err(ctx), sizeof(int), cudaMemcpyDeviceToHost, s), "D2H err");
  ck(cudaStreamSynchronize(s), "stream sync");
  if (flag) fail(TFG_INVALID_ARGUMENT, "QuantizedImage: pixel value exceeds gray level");
}

// Host copy split over up to 16 host threads (pageable -> pinned staging).
void parallel_memcpy(uint8_t* dst, const uint8_t* src, size_t n) {
  const size_t kMinPerThread = 2u << 20;
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>(std::min<size_t>(hw, 16), std::max<size_t>(1, n / kMinPerThread));
  if (nt <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> pool;
  const size_t per = (n + nt - 1) / nt;
  for (size_t t = 0; t < nt; ++t) {
    const size_t b = t * per, e = std::min(n, b + per);
    if (b < e) pool.emplace_back([=] { std::memcpy(dst + b, src + b, e - b); });
  }
  for (auto& th : pool) th.join();
}

size_t auto_chunks(size_t width, size_t height, int max_d) {
  const size_t bytes = width * height;
  const size_t target = 32u << 20;  // ~32 MiB per chunk (per-launch overhead vs pipeline fill/drain)
  size_t k = (bytes + target - 1) / target;
  const size_t cap = height / (size_t)(max_d + 1);
  if (k > cap) k = cap;
  return std::max<size_t>(k, 1);
}

// Chunk specs, partition() semantics (pipeline.hpp:48-73) with the largest
// halo any requested (d, theta) needs, over the owned anchor rows [0, height)
// of a buffer of `total_rows` >= height rows (a row shard: the rows past
// `height` are the next shard's halo and are read, never voted).
std::vector<uint64_t> chunk_specs(size_t width, size_t height, const int* distances, const int* angles,
                                  int n_dt, size_t k, size_t total_rows = 0) {
  if (total_rows < height) total_rows = height;
  int halo = 0, dmax = 1;
  for (int i = 0; i < n_dt; ++i) {
    dmax = std::max(dmax, distances[i]);
    if (angles[i] != 0) halo = std::max(halo, distances[i]);
  }
  if (k < 1 || k > height) fail(TFG_INVALID_ARGUMENT, "partition: chunk count must be in [1, height]");
  if (height / k <= (size_t)dmax && k > 1)
    fail(TFG_INVALID_ARGUMENT, "partition: too many chunks for this distance (chunk shorter than halo)");
  (void)width;
  std::vector<uint64_t> s(3 * k);
  const size_t base = height / k, extra = height % k;
  size_t row = 0;
  for (size_t i = 0; i < k; ++i) {
    const size_t end = row + base + (i < extra ? 1 : 0);
    s[3 * i] = row;
    s[3 * i + 1] = end;
    s[3 * i + 2] = std::min(total_rows, end + (size_t)halo);
    row = end;
  }
  return s;
}

// Scheme 3 pipeline over host rows. `fetch_rows(i, start, end, dst_host_or_null)`
// either fills a pinned slot (returns that pointer) or returns a pointer to
// the caller's own host rows.
// `specs`: k chunks {owned_row_start, owned_row_end, buffer_row_end} (any
// subset of a partition(): a GPU of a multi-GPU group runs its own chunks).
// Row copies whose rows are contiguous on both sides (pitch == width) go
// out as ONE linear copy instead of a pitched 2D copy (measured the same
// for c2's 4096^2 images, tools/e2e_c2_diag.py; no per-row descriptors).
inline cudaError_t copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                             cudaMemcpyKind kind, cudaStream_t s) {
  if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * rows, kind, s);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, s);
}

template <typename Fetch>
void run_pipeline_specs(tfg_ctx* ctx, size_t width, const std::vector<uint64_t>& specs, int pixel_levels,
                        int levels, const int* distances, const int* angles, int n_dt, unsigned flags,
                        unsigned long long* d_acc, Fetch&& fetch_rows, size_t n_bands = 1,
                        size_t acc_band_stride = 0, const std::function<void(size_t)>& band_done = nullptr,
                        const int* job_levels = nullptr, const size_t* job_off = nullptr) {
  // job_levels / job_off: per-job L and offset inside a band's slice of d_acc
  // (tfg_glcm_shard_jobs); null = every job at `levels`, job t at t * L^2
  // The ring runs continuously over (band, chunk): band b+1's first copy
  // overlaps band b's last votes. Band b's GLCMs go to d_acc + b*acc_band_stride.
  const size_t k = specs.size() / 3;
  const size_t pitch = round16(width);
  size_t max_rows = 0;
  for (size_t i = 0; i < k; ++i) max_rows = std::max<size_t>(max_rows, specs[3 * i + 2] - specs[3 * i]);
  const bool sequential = (flags & TFG_SEQUENTIAL) != 0;
  for (int sl = 0; sl < tfg_ctx::kSlots; ++sl) ctx->dslot[sl].get(max_rows * pitch + 64);
  size_t pending_band = SIZE_MAX;  // band whose band_done waits for the next chunk's H2D
  for (size_t n = 0; n < n_bands * k; ++n) {
    const size_t bnd = n / k, i = n % k;
    const int sl = (int)(n % tfg_ctx::kSlots);
    const size_t start = specs[3 * i], owned_end = specs[3 * i + 1], buf_end = specs[3 * i + 2];
    const size_t rows = buf_end - start;
    // host side: the slot's previous H2D must be done before we refill it
    if (n >= (size_t)tfg_ctx::kSlots) ck(cudaEventSynchronize(ctx->copied[sl]), "event sync");
    const uint8_t* src = fetch_rows(bnd, i, start, owned_end, buf_end, sl);
    uint8_t* dst = static_cast<uint8_t*>(ctx->dslot[sl].p);
    // device side: the slot's previous votes must be done before overwrite
    if (n >= (size_t)tfg_ctx::kSlots) ck(cudaStreamWaitEvent(ctx->copy, ctx->consumed[sl], 0), "wait");
    ck(copy_rows(dst, pitch, src, width, width, rows, cudaMemcpyHostToDevice, ctx->copy), "H2D chunk");
    ck(cudaEventRecord(ctx->copied[sl], ctx->copy), "event record");
    // the previous band's early counts D2H goes out only now, after this
    // chunk's H2D: enqueued before it, its wait on that band's votes held
    // this copy back (c2 e2e: 2 bands 1.06 -> 0.70 ms, tools/e2e_c2_diag.py)
    if (pending_band != SIZE_MAX) {
      band_done(pending_band);
      pending_band = SIZE_MAX;
    }
    ck(cudaStreamWaitEvent(ctx->exec, ctx->copied[sl], 0), "wait");
    if (pixel_levels == levels) launch_validate(ctx, dst, width, rows, pitch, 0, 1, levels, sync_err(ctx), ctx->exec);
    if (job_levels) {
      unsigned long long* outs[64];
      for (int t = 0; t < n_dt; ++t) outs[t] = d_acc + bnd * acc_band_stride + job_off[t];
      launch_job_set(ctx, dst, width, rows, pitch, 0, 1, owned_end - start, pixel_levels, job_levels, distances, angles,
                     outs, n_dt, flags, ctx->exec);
    } else if (!launch_vote_jobs(ctx, dst, width, rows, pitch, 0, 1, owned_end - start, pixel_levels, levels,
                                 distances, angles, n_dt, flags, d_acc + bnd * acc_band_stride,
                                 (size_t)levels * levels, ctx->exec)) {
      for (int t = 0; t < n_dt; ++t)
        launch_vote(ctx, dst, width, rows, pitch, 0, 1, owned_end - start, pixel_levels, levels, distances[t],
                    angles[t], flags, d_acc + bnd * acc_band_stride + (size_t)t * levels * levels, ctx->exec);
    }
    ck(cudaEventRecord(ctx->consumed[sl], ctx->exec), "event record");
    if (band_done && i == k - 1) pending_band = bnd;
    if (sequential) ck(cudaStreamSynchronize(ctx->exec), "stream sync");
  }
  if (pending_band != SIZE_MAX) band_done(pending_band);
}

template <typename Fetch>
void run_pipeline(tfg_ctx* ctx, size_t width, size_t height, int pixel_levels, int levels,
                  const int* distances, const int* angles, int n_dt, size_t k, unsigned flags,
                  unsigned long long* d_acc, Fetch&& fetch_rows, size_t total_rows = 0, size_t n_bands = 1,
                  size_t acc_band_stride = 0, const std::function<void(size_t)>& band_done = nullptr,
                  const int* job_levels = nullptr, const size_t* job_off = nullptr) {
  run_pipeline_specs(ctx, width, chunk_specs(width, height, distances, angles, n_dt, k, total_rows), pixel_levels,
                     levels, distances, angles, n_dt, flags, d_acc, std::forward<Fetch>(fetch_rows), n_bands,
                     acc_band_stride, band_done, job_levels, job_off);
}

// Shared-memory budget of glcm_subglcm_kernel's R sub-GLCM copies.
constexpr size_t kSubSmemBytes = 96 * 1024;

// Host raster -> a pitched device buffer at PCIe speed: pinned caller memory
// goes by DMA; pageable rows are first copied by several host threads into
// the pinned ring slots, each slot's H2D overlapping the next slot's fill.
void stage_host_image(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, uint8_t* d_dst,
                      size_t dpitch) {
  cudaStream_t s = ctx->exec;
  if (host_memory_kind(px) != 0) {
    ck(copy_rows(d_dst, dpitch, px, width, width, height, cudaMemcpyHostToDevice, s), "stage image");
    return;
  }
  const size_t rows_per = std::max<size_t>(1, (size_t)(16u << 20) / std::max<size_t>(width, 1));
  for (int sl = 0; sl < tfg_ctx::kSlots; ++sl) ctx->hslot[sl].get(rows_per * width + 64);
  size_t n = 0;
  for (size_t r = 0; r < height; r += rows_per, ++n) {
    const int sl = (int)(n % tfg_ctx::kSlots);
    const size_t rows = std::min(rows_per, height - r);
    if (n >= (size_t)tfg_ctx::kSlots) ck(cudaEventSynchronize(ctx->copied[sl]), "event sync");
    uint8_t* slot = static_cast<uint8_t*>(ctx->hslot[sl].p);
    parallel_memcpy(slot, px + r * width, rows * width);
    ck(copy_rows(d_dst + r * dpitch, dpitch, slot, width, width, rows, cudaMemcpyHostToDevice, s),
       "stage image");
    ck(cudaEventRecord(ctx->copied[sl], s), "event record");
  }
}

// Host image(s) -> the Scheme-3 stream pipeline over (band, chunk), votes
// added into d_acc ([band][dt][cell]): copy chunk n+1 while voting chunk n,
// across band boundaries. `height` buffer rows of which anchors in rows
// [0, owned_rows) vote. Pinned caller memory is DMA'd in place; pageable
// memory would make every cudaMemcpyAsync a synchronous bounce-buffer copy,
// so its rows are first copied (by several host threads) into the pinned
// ring slot. `band_done(b)`: called once band b's last votes are enqueued.
void host_vote(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, size_t owned_rows, size_t band_stride,
               size_t n_bands, int pixel_levels, int levels, const int* distances, const int* angles_deg, int n_dt,
               unsigned flags, unsigned long long* d_acc,
               const std::function<void(size_t)>& band_done = nullptr, const int* job_levels = nullptr,
               const size_t* job_off = nullptr, size_t job_band_words = 0) {
  int dmax = 1;
  for (int i = 0; i < n_dt; ++i) dmax = std::max(dmax, distances[i]);
  const size_t k = auto_chunks(width, owned_rows, dmax);
  const bool pageable = host_memory_kind(px) == 0;
  if (pageable) {
    const std::vector<uint64_t> sp = chunk_specs(width, owned_rows, distances, angles_deg, n_dt, k, height);
    size_t max_rows = 0;
    for (size_t i = 0; i < k; ++i) max_rows = std::max<size_t>(max_rows, sp[3 * i + 2] - sp[3 * i]);
    for (int sl = 0; sl < tfg_ctx::kSlots; ++sl) ctx->hslot[sl].get(max_rows * width + 64);
  }
  const size_t band_words = job_levels ? job_band_words : (size_t)n_dt * levels * levels;
  run_pipeline(
      ctx, width, owned_rows, pixel_levels, levels, distances, angles_deg, n_dt, k, flags, d_acc,
      [&](size_t b, size_t, size_t start, size_t, size_t buf_end, int sl) -> const uint8_t* {
        const uint8_t* src = px + b * band_stride + start * width;
        if (!pageable) return src;
        uint8_t* dst = static_cast<uint8_t*>(ctx->hslot[sl].p);
        parallel_memcpy(dst, src, (buf_end - start) * width);
        return dst;
      },
      height, n_bands, band_words, band_done, job_levels, job_off);
}

}  // namespace

// ============================================================================
extern "C" {

int tfg_abi_version(void) { return TFG_ABI_VERSION; }
int tfg_memory_kind(const void* p) { return host_memory_kind(p); }
const char* tfg_last_error(void) { return g_error.c_str(); }
size_t tfg_last_error_chunk(void) { return g_error_chunk; }
uint64_t tfg_launch_count(tfg_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int tfg_ctx_create(tfg_ctx** out, int device, unsigned flags) {
  (void)flags;
  if (!out) {
    g_error = "tfg_ctx_create: null output";
    return TFG_INVALID_ARGUMENT;
  }
  *out = nullptr;
  tfg_ctx* ctx = new tfg_ctx();
  const int rc = guarded([&] {
    int n = 0;
    ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) fail(TFG_INVALID_ARGUMENT, "tfg_ctx_create: no such CUDA device");
    ctx->device = device;
    DeviceGuard dg(device);
    ck(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
    ck(cudaStreamCreateWithFlags(&ctx->exec, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking), "stream");
    for (int i = 0; i < tfg_ctx::kSlots; ++i) {
      ck(cudaEventCreateWithFlags(&ctx->copied[i], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&ctx->consumed[i], cudaEventDisableTiming), "event");
    }
    ck(cudaMalloc(&ctx->d_err, 64), "cudaMalloc");
    ck(cudaMemsetAsync(ctx->d_err, 0, 64, ctx->exec), "memset");
    ck(cudaEventCreateWithFlags(&ctx->scratch_ev, cudaEventDisableTiming), "event");
    for (int i = 0; i < tfg_ctx::kAux; ++i) {
      ck(cudaStreamCreateWithFlags(&ctx->aux[i], cudaStreamNonBlocking), "stream");
      ck(cudaEventCreateWithFlags(&ctx->join_ev[i], cudaEventDisableTiming), "event");
    }
    ck(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ctx->band_ev, cudaEventDisableTiming), "event");
    ck(cudaMalloc(&ctx->sync_ctr, (kPoolCtrOffset + kMaxPoolBands) * sizeof(unsigned int)), "cudaMalloc");
    ck(cudaMemsetAsync(ctx->sync_ctr, 0, (kPoolCtrOffset + kMaxPoolBands) * sizeof(unsigned int), ctx->exec),
       "memset");
    // every stream of the context is non-blocking: finish the zeroing before
    // any launch on another stream can read the counters
    ck(cudaStreamSynchronize(ctx->exec), "stream sync");
  });
  if (rc != TFG_OK) {
    tfg_ctx_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return TFG_OK;
}

void tfg_ctx_destroy(tfg_ctx* ctx) {
  if (!ctx) return;
  {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    if (ctx->exec) cudaStreamSynchronize(ctx->exec);
    if (ctx->copy) cudaStreamSynchronize(ctx->copy);
    for (auto& b : ctx->dslot) b.release();
    for (auto& b : ctx->hslot) b.release();
    ctx->img.release();
    ctx->acc.release();
    ctx->sym.release();
    ctx->probs.release();
    ctx->feats.release();
    ctx->partials.release();
    ctx->qbuf.release();
    ctx->tmp.release();
    ctx->errs.release();
    ctx->hout.release();
    for (int i = 0; i < tfg_ctx::kSlots; ++i) {
      if (ctx->copied[i]) cudaEventDestroy(ctx->copied[i]);
      if (ctx->consumed[i]) cudaEventDestroy(ctx->consumed[i]);
    }
    if (ctx->d_err) cudaFree(ctx->d_err);
    if (ctx->sync_ctr) cudaFree(ctx->sync_ctr);
    for (int i = 0; i < tfg_ctx::kAux; ++i) {
      if (ctx->aux[i]) cudaStreamDestroy(ctx->aux[i]);
      if (ctx->join_ev[i]) cudaEventDestroy(ctx->join_ev[i]);
    }
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->scratch_ev) cudaEventDestroy(ctx->scratch_ev);
    if (ctx->band_ev) cudaEventDestroy(ctx->band_ev);
    if (ctx->exec) cudaStreamDestroy(ctx->exec);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete ctx;
}

int tfg_neighbor_offset(int distance, int angle_deg, long* drow, long* dcol) {
  return guarded([&] {
    if (!offset_of(distance, angle_deg, drow, dcol)) fail(TFG_INVALID_ARGUMENT, "neighbor_offset: bad angle");
  });
}

int tfg_valid_pair_count(size_t width, size_t height, int distance, int angle_deg, uint64_t* out) {
  return guarded([&] {
    const size_t d = (size_t)distance;
    if (distance < 1 || d >= width || d >= height)
      fail(TFG_INVALID_ARGUMENT,
           "valid_pair_count: degenerate geometry (d must be in [1, min(width, height)))");
    switch (angle_deg) {
      case 0: *out = (uint64_t)height * (width - d); break;
      case 90: *out = (uint64_t)(height - d) * width; break;
      case 45:
      case 135: *out = (uint64_t)(height - d) * (width - d); break;
      default: fail(TFG_INVALID_ARGUMENT, "valid_pair_count: bad angle");
    }
  });
}

int tfg_partition(size_t width, size_t height, int distance, int angle_deg, size_t chunk_count,
                  uint64_t* specs_out) {
  return guarded([&] {
    const size_t d = (size_t)distance;
    if (distance < 1 || d >= width || d >= height)
      fail(TFG_INVALID_ARGUMENT, "partition: degenerate geometry (d must be in [1, min(width, height)))");
    check_angle(angle_deg);
    if (chunk_count < 1 || chunk_count > height)
      fail(TFG_INVALID_ARGUMENT, "partition: chunk count must be in [1, height]");
    if (height / chunk_count <= d && chunk_count > 1)
      fail(TFG_INVALID_ARGUMENT, "partition: too many chunks for this distance (chunk shorter than halo)");
    auto s = chunk_specs(width, height, &distance, &angle_deg, 1, chunk_count);
    std::memcpy(specs_out, s.data(), s.size() * 8);
  });
}

int tfg_plan(int levels, size_t scratch_budget, unsigned worker_count, unsigned* copies,
             unsigned* groups_per_unit, int* degraded) {
  return guarded([&] {
    check_levels(levels, "plan");
    (void)worker_count;
    const size_t sub = (size_t)levels * levels * 4;  // u32 sub-GLCM (parallel.hpp:48)
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
    *copies = (unsigned)std::min<size_t>(c, 8);
  });
}

int tfg_quantize(tfg_ctx* ctx, const uint8_t* gray, size_t n, int levels, uint8_t* out, unsigned flags) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    check_levels(levels, "quantize");
    if (n == 0) return;
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->exec;
    const size_t n16 = round16(n);
    const uint8_t* d_in = gray;
    uint8_t* d_out = out;
    uint8_t* buf = nullptr;
    const bool dev = (flags & TFG_INPUT_DEVICE) != 0;
    if (!dev) {
      buf = static_cast<uint8_t*>(ctx->qbuf.get(2 * n16));
      ck(cudaMemcpyAsync(buf, gray, n, cudaMemcpyHostToDevice, s), "H2D");
      d_in = buf;
      d_out = buf + n16;
    } else if ((reinterpret_cast<uintptr_t>(gray) | reinterpret_cast<uintptr_t>(out)) & 15) {
      fail(TFG_INVALID_ARGUMENT, "quantize: device buffers must be 16-byte aligned");
    }
    const int blocks = (int)std::min<size_t>((n / 16 + 255) / 256 + 1, (size_t)ctx->num_sms * 8);
    tfg::quantize_kernel<<<blocks, 256, 0, s>>>(d_in, d_out, (long long)n, levels);
    ck(cudaGetLastError(), "quantize launch");
    ctx->launches++;
    if (!dev) ck(cudaMemcpyAsync(out, d_out, n, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
  });
}

namespace {
// One image (or n_bands images) of `height` buffer rows whose anchors in rows
// [0, owned_rows) vote (owned_rows == height: the whole image).
// The caller holds ctx->mu.
int glcm_impl_locked(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, size_t owned_rows, size_t pitch,
                     size_t band_stride, size_t n_bands, int pixel_levels, int levels, const int* distances,
                     const int* angles_deg, int n_dt, unsigned flags, uint64_t* counts_out, double* probs_out,
                     double* feats_out) {
  return guarded([&] {
    check_levels(levels, "glcm");
    check_pixel_levels(pixel_levels, levels);
    if (width == 0 || height == 0) fail(TFG_INVALID_ARGUMENT, "QuantizedImage: dimensions must be positive");
    if (pitch < width) fail(TFG_INVALID_ARGUMENT, "glcm: pitch must be >= width");
    if (n_bands < 1) fail(TFG_INVALID_ARGUMENT, "glcm: need at least one band");
    if (n_bands > 1 && band_stride < pitch * height) fail(TFG_INVALID_ARGUMENT, "glcm: bands overlap");
    check_dts(distances, angles_deg, n_dt, width, height);
    if (!px) fail(TFG_INVALID_ARGUMENT, "glcm: null pixels");
    if (owned_rows > height) fail(TFG_INVALID_ARGUMENT, "glcm: owned rows exceed the buffer rows");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->exec;
    const size_t cells = (size_t)levels * levels;
    const size_t n_out = n_bands * (size_t)n_dt;
    if (owned_rows == 0) {  // a shard that owns no anchors: zero counts
      ck(cudaMemsetAsync(ctx->acc.get(n_out * cells * 8), 0, n_out * cells * 8, s), "memset");
      finish(ctx, static_cast<unsigned long long*>(ctx->acc.p), (int)n_out, levels, flags & ~(TFG_NORMALIZE | TFG_FEATURES),
             counts_out, nullptr, nullptr, s);
      return;
    }
    auto* d_acc = static_cast<unsigned long long*>(ctx->acc.get(n_out * cells * 8));
    ck(cudaMemsetAsync(d_acc, 0, n_out * cells * 8, s), "memset");
    if (pixel_levels == levels) clear_sync_flag(ctx, s);
    const bool dev = (flags & TFG_INPUT_DEVICE) != 0;

    if (!dev) {
      if (pitch != width) fail(TFG_INVALID_ARGUMENT, "glcm: host images must be dense (pitch == width)");
      // PCIe is full duplex: a band's counts go down to a pinned counts_out
      // while later bands are still coming up (plain counts, several bands)
      const bool early = n_bands > 1 && counts_out && host_memory_kind(counts_out) == 1 &&
                         !(flags & (TFG_SYMMETRIC | TFG_NORMALIZE | TFG_FEATURES));
      const size_t band_words = (size_t)n_dt * cells;
      auto band_done = [&](size_t b) {
        if (b + 1 >= n_bands) return;  // the last band goes with finish()
        ck(cudaEventRecord(ctx->band_ev, ctx->exec), "event record");
        ck(cudaStreamWaitEvent(ctx->aux[0], ctx->band_ev, 0), "wait");
        ck(cudaMemcpyAsync(counts_out + b * band_words, d_acc + b * band_words, band_words * 8,
                           cudaMemcpyDeviceToHost, ctx->aux[0]),
           "D2H band counts");
      };
      // every exit (errors included) waits for the early copies into counts_out
      struct AuxDrain {
        cudaStream_t st;
        bool on;
        ~AuxDrain() {
          if (on) cudaStreamSynchronize(st);
        }
      } drain{ctx->aux[0], early};
      host_vote(ctx, px, width, height, owned_rows, band_stride, n_bands, pixel_levels, levels, distances, angles_deg,
                n_dt, flags, d_acc, early ? std::function<void(size_t)>(band_done) : nullptr);
      if (pixel_levels == levels) check_sync_flag(ctx, s);
      finish(ctx, d_acc, (int)n_out, levels, flags, counts_out, probs_out, feats_out, s,
             early ? (n_bands - 1) * (size_t)n_dt : 0);
      return;
    }

    const uint8_t* d_img = px;
    size_t dpitch = pitch, dstride = band_stride;
    const bool aligned = dev && ((reinterpret_cast<uintptr_t>(px) & 15) == 0) && (pitch % 16 == 0) &&
                         (n_bands == 1 || band_stride % 16 == 0);
    if (!aligned) {
      // stage into an aligned, pitched device buffer (one copy per band)
      dpitch = round16(width);
      dstride = dpitch * height;
      uint8_t* buf = static_cast<uint8_t*>(ctx->img.get(dstride * n_bands + 64));
      for (size_t b = 0; b < n_bands; ++b)
        ck(copy_rows(buf + b * dstride, dpitch, px + b * band_stride, pitch, width, height,
                             dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s),
           "stage image");
      d_img = buf;
    }
    if (pixel_levels == levels)
      launch_validate(ctx, d_img, width, height, dpitch, dstride, (int)n_bands, levels, sync_err(ctx), s);
    const bool jobs = n_bands == 1 && launch_vote_jobs(ctx, d_img, width, height, dpitch, dstride, 1, owned_rows,
                                                       pixel_levels, levels, distances, angles_deg, n_dt, flags,
                                                       d_acc, cells, s);
    for (int t = 0; t < n_dt && !jobs; ++t) {
      // bands are batched in one launch (blockIdx.y = band); outputs band-major
      // [band][dt][cell]: launch per dt writing with a band stride of n_dt*cells.
      if (n_dt == 1) {
        launch_vote(ctx, d_img, width, height, dpitch, dstride, (int)n_bands, owned_rows, pixel_levels, levels,
                    distances[t], angles_deg[t], flags, d_acc, s);
      } else {
        // per-dt scratch then scatter into band-major layout
        auto* tmp = static_cast<unsigned long long*>(ctx->tmp.get(n_bands * cells * 8));
        ck(cudaMemsetAsync(tmp, 0, n_bands * cells * 8, s), "memset");
        launch_vote(ctx, d_img, width, height, dpitch, dstride, (int)n_bands, owned_rows, pixel_levels, levels,
                    distances[t], angles_deg[t], flags, tmp, s);
        ck(cudaMemcpy2DAsync(d_acc + (size_t)t * cells, (size_t)n_dt * cells * 8, tmp, cells * 8, cells * 8,
                             n_bands, cudaMemcpyDeviceToDevice, s),
           "scatter");
      }
    }
    if (pixel_levels == levels) check_sync_flag(ctx, s);
    finish(ctx, d_acc, (int)n_out, levels, flags, counts_out, probs_out, feats_out, s);
  });
}

int glcm_impl(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, size_t owned_rows, size_t pitch,
              size_t band_stride, size_t n_bands, int pixel_levels, int levels, const int* distances,
              const int* angles_deg, int n_dt, unsigned flags, uint64_t* counts_out, double* probs_out,
              double* feats_out) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return glcm_impl_locked(ctx, px, width, height, owned_rows, pitch, band_stride, n_bands, pixel_levels, levels,
                          distances, angles_deg, n_dt, flags, counts_out, probs_out, feats_out);
}

}  // namespace

int tfg_glcm_bands(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, size_t pitch,
                   size_t band_stride, size_t n_bands, int pixel_levels, int levels, const int* distances,
                   const int* angles_deg, int n_dt, unsigned flags, uint64_t* counts_out, double* probs_out,
                   double* feats_out) {
  return glcm_impl(ctx, px, width, height, height, pitch, band_stride, n_bands, pixel_levels, levels, distances,
                   angles_deg, n_dt, flags, counts_out, probs_out, feats_out);
}

int tfg_glcm_shard(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t buffer_rows, size_t owned_rows,
                   size_t pitch, size_t band_stride, size_t n_bands, int pixel_levels, int levels,
                   const int* distances, const int* angles_deg, int n_dt, unsigned flags, uint64_t* counts_out) {
  return glcm_impl(ctx, px, width, buffer_rows, owned_rows, pitch, n_bands > 1 ? band_stride : pitch * buffer_rows,
                   n_bands, pixel_levels, levels, distances, angles_deg, n_dt,
                   flags & ~(TFG_SYMMETRIC | TFG_NORMALIZE | TFG_FEATURES), counts_out, nullptr, nullptr);
}

int tfg_glcm_shard_jobs(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t buffer_rows, size_t owned_rows,
                        size_t band_stride, size_t n_bands, int pixel_levels, const int* levels,
                        const int* distances, const int* angles_deg, int n_jobs, unsigned flags,
                        uint64_t* counts_out) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    if (n_jobs < 1 || n_jobs > 64 || !levels) fail(TFG_INVALID_ARGUMENT, "glcm: need 1..64 jobs");
    for (int t = 0; t < n_jobs; ++t) {
      check_levels(levels[t], "glcm");
      check_pixel_levels(pixel_levels, levels[t]);
    }
    if (width == 0 || buffer_rows == 0) fail(TFG_INVALID_ARGUMENT, "QuantizedImage: dimensions must be positive");
    if (flags & TFG_INPUT_DEVICE)
      fail(TFG_INVALID_ARGUMENT, "glcm_shard_jobs: host images only (device images: tfg_glcm_jobs_async)");
    if (n_bands < 1) fail(TFG_INVALID_ARGUMENT, "glcm: need at least one band");
    if (n_bands > 1 && band_stride < width * buffer_rows) fail(TFG_INVALID_ARGUMENT, "glcm: bands overlap");
    check_dts(distances, angles_deg, n_jobs, width, buffer_rows);
    if (!px) fail(TFG_INVALID_ARGUMENT, "glcm: null pixels");
    if (owned_rows > buffer_rows) fail(TFG_INVALID_ARGUMENT, "glcm: owned rows exceed the buffer rows");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->exec;
    std::vector<size_t> off((size_t)n_jobs);
    size_t band_words = 0;
    for (int t = 0; t < n_jobs; ++t) {
      off[t] = band_words;
      band_words += (size_t)levels[t] * levels[t];
    }
    const size_t words = n_bands * band_words;
    if (words > (size_t)INT32_MAX) fail(TFG_INVALID_ARGUMENT, "glcm_shard_jobs: too many output cells for one call");
    auto* d_acc = static_cast<unsigned long long*>(ctx->acc.get(words * 8));
    ck(cudaMemsetAsync(d_acc, 0, words * 8, s), "memset");
    if (owned_rows > 0) {
      if (pixel_levels < 256) clear_sync_flag(ctx, s);
      const bool early = n_bands > 1 && counts_out && host_memory_kind(counts_out) == 1;
      auto band_done = [&](size_t b) {
        if (b + 1 >= n_bands) return;
        ck(cudaEventRecord(ctx->band_ev, ctx->exec), "event record");
        ck(cudaStreamWaitEvent(ctx->aux[0], ctx->band_ev, 0), "wait");
        ck(cudaMemcpyAsync(counts_out + b * band_words, d_acc + b * band_words, band_words * 8,
                           cudaMemcpyDeviceToHost, ctx->aux[0]),
           "D2H band counts");
      };
      struct AuxDrain {
        cudaStream_t st;
        bool on;
        ~AuxDrain() {
          if (on) cudaStreamSynchronize(st);
        }
      } drain{ctx->aux[0], early};
      host_vote(ctx, px, width, buffer_rows, owned_rows, n_bands > 1 ? band_stride : width * buffer_rows, n_bands,
                pixel_levels, levels[0], distances, angles_deg, n_jobs, flags & ~(TFG_SYMMETRIC | TFG_NORMALIZE | TFG_FEATURES),
                d_acc, early ? std::function<void(size_t)>(band_done) : nullptr, levels, off.data(), band_words);
      if (pixel_levels < 256) check_sync_flag(ctx, s);
      // counts only: one u64 "cell" per word
      finish(ctx, d_acc, (int)words, 1, 0, counts_out, nullptr, nullptr, s, early ? (n_bands - 1) * band_words : 0);
    } else {
      finish(ctx, d_acc, (int)words, 1, 0, counts_out, nullptr, nullptr, s);
    }
  });
}

int tfg_glcm(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, size_t pitch, int pixel_levels,
             int levels, const int* distances, const int* angles_deg, int n_dt, unsigned flags,
             uint64_t* counts_out, double* probs_out, double* feats_out) {
  return tfg_glcm_bands(ctx, px, width, height, pitch, pitch * height, 1, pixel_levels, levels, distances,
                        angles_deg, n_dt, flags, counts_out, probs_out, feats_out);
}

int tfg_glcm_chunked(tfg_ctx* ctx, size_t width, size_t height, int pixel_levels, int levels,
                     const int* distances, const int* angles_deg, int n_dt, size_t chunk_count,
                     tfg_fetch_fn fetch, void* user, unsigned flags, uint64_t* counts_out, double* probs_out,
                     double* feats_out) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    check_levels(levels, "glcm");
    check_pixel_levels(pixel_levels, levels);
    if (!fetch) fail(TFG_INVALID_ARGUMENT, "glcm_chunked: null fetch callback");
    check_dts(distances, angles_deg, n_dt, width, height);
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->exec;
    const size_t cells = (size_t)levels * levels;
    auto* d_acc = static_cast<unsigned long long*>(ctx->acc.get((size_t)n_dt * cells * 8));
    ck(cudaMemsetAsync(d_acc, 0, (size_t)n_dt * cells * 8, s), "memset");
    if (pixel_levels == levels) clear_sync_flag(ctx, s);
    const std::vector<uint64_t> specs = chunk_specs(width, height, distances, angles_deg, n_dt, chunk_count);
    size_t max_rows = 0;
    for (size_t i = 0; i < chunk_count; ++i) max_rows = std::max<size_t>(max_rows, specs[3 * i + 2] - specs[3 * i]);
    for (int sl = 0; sl < tfg_ctx::kSlots; ++sl) ctx->hslot[sl].get(max_rows * width + 64);
    try {
      run_pipeline(ctx, width, height, pixel_levels, levels, distances, angles_deg, n_dt, chunk_count, flags, d_acc,
                   [&](size_t, size_t i, size_t start, size_t owned_end, size_t buf_end, int sl) -> const uint8_t* {
                     uint8_t* dst = static_cast<uint8_t*>(ctx->hslot[sl].p);
                     char msg[512] = {0};
                     const int rc = fetch(user, i, start, owned_end, buf_end, dst, msg, sizeof msg);
                     if (rc) {
                       g_error_chunk = i;
                       fail(TFG_SOURCE_ERROR, "chunk " + std::to_string(i) + ": " +
                                                  (msg[0] ? std::string(msg) : std::string("source failure")));
                     }
                     return dst;
                   });
    } catch (...) {
      cudaStreamSynchronize(ctx->exec);
      cudaStreamSynchronize(ctx->copy);
      throw;
    }
    if (pixel_levels == levels) check_sync_flag(ctx, s);
    finish(ctx, d_acc, n_dt, levels, flags, counts_out, probs_out, feats_out, s);
  });
}

int tfg_subglcms(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, int pixel_levels, int levels,
                 int distance, int angle_deg, unsigned group_size, unsigned copies, size_t group_count,
                 unsigned flags, uint32_t* subs_out, uint64_t* counts_out, uint64_t* per_copy_hottest_out) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    check_levels(levels, "glcm");
    check_pixel_levels(pixel_levels, levels);
    if (width == 0 || height == 0) fail(TFG_INVALID_ARGUMENT, "QuantizedImage: dimensions must be positive");
    check_angle(angle_deg);
    check_geometry(width, height, distance);
    if (copies < 1) fail(TFG_INVALID_ARGUMENT, "privatized: plan.copies must be >= 1");
    if (group_size == 0) group_size = 512;
    if (group_count < 1 || group_count > height)
      fail(TFG_INVALID_ARGUMENT, "subglcms: group count must be in [1, height]");
    if (!px) fail(TFG_INVALID_ARGUMENT, "glcm: null pixels");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->exec;
    const size_t cells = (size_t)levels * levels;
    const size_t n_subs = group_count * copies;
    // stage the raster (host or device) into an aligned pitched buffer
    const size_t dpitch = round16(width);
    uint8_t* d_img = static_cast<uint8_t*>(ctx->img.get(dpitch * height + 64));
    const bool dev = (flags & TFG_INPUT_DEVICE) != 0;
    if (dev) {
      ck(cudaMemcpy2DAsync(d_img, dpitch, px, width, width, height, cudaMemcpyDeviceToDevice, s), "stage image");
    } else {
      stage_host_image(ctx, px, width, height, d_img, dpitch);
    }
    if (pixel_levels == levels) {
      clear_sync_flag(ctx, s);
      launch_validate(ctx, d_img, width, height, dpitch, 0, 1, levels, sync_err(ctx), s);
    }
    long sdr, sdc;
    offset_of(distance, angle_deg, &sdr, &sdc);
    if (copies == 1 && cells * 4 > kSubSmemBytes && group_count <= 4 * (size_t)ctx->num_sms &&
        height / group_count >= (size_t)sdr) {
      // One copy per group and a sub-GLCM too large for shared memory: sub-GLCM
      // g is the GLCM of stripe g's anchors (lane routing is moot with one
      // copy), so the stripes vote through the privatised kernel as bands of
      // one launch (band b = stripe b's rows + the halo rows below it, read in
      // place), instead of per-pixel global atomics.
      std::vector<size_t> row0(group_count + 1);
      const size_t base = height / group_count, extra = height % group_count;
      for (size_t g = 0; g < group_count; ++g) row0[g + 1] = row0[g] + base + (g < extra ? 1 : 0);
      auto* d_st = static_cast<unsigned long long*>(ctx->acc.get((group_count + 1) * cells * 8 + n_subs * 8));
      auto* d_cnt = d_st + group_count * cells;
      auto* d_max = d_cnt + cells;
      ck(cudaMemsetAsync(d_st, 0, group_count * cells * 8, s), "memset");
      const long dr = sdr;  // stripes are >= dr rows: every halo lies in the next stripe
      const unsigned vflags = flags & ~TFG_INPUT_DEVICE;
      // bands of equal geometry: [0, extra) (base+1 rows), [extra, G-1) and the
      // last stripe (base rows; the last one has no rows below it)
      auto run = [&](size_t g0, size_t g1) {
        if (g0 >= g1) return;
        const size_t rows = row0[g0 + 1] - row0[g0];
        const size_t below = height - row0[g1 - 1] - rows;  // rows after the group's last stripe
        const size_t halo = std::min<size_t>((size_t)std::max<long>(dr, 0), below);
        launch_vote(ctx, d_img + row0[g0] * dpitch, width, rows + halo, dpitch, rows * dpitch, (int)(g1 - g0), rows,
                    pixel_levels, levels, distance, angle_deg, vflags, d_st + g0 * cells, s);
      };
      const size_t split = std::min(extra, group_count - 1);
      run(0, split);
      run(split, group_count - 1);
      run(group_count - 1, group_count);
      tfg::stripe_sum_kernel<<<(unsigned)std::min<size_t>((cells + 255) / 256, 1024), 256, 0, s>>>(
          d_st, (int)cells, (int)group_count, counts_out ? d_cnt : nullptr, nullptr);
      ck(cudaGetLastError(), "stripe_sum_kernel launch");
      ctx->launches++;
      if (per_copy_hottest_out) {
        tfg::stripe_max_kernel<<<(unsigned)group_count, 256, 0, s>>>(d_st, (int)cells, d_max);
        ck(cudaGetLastError(), "stripe_max_kernel launch");
        ctx->launches++;
        ck(cudaMemcpyAsync(per_copy_hottest_out, d_max, n_subs * 8, cudaMemcpyDeviceToHost, s), "D2H max");
      }
      if (subs_out) {
        uint32_t* d_subs = static_cast<uint32_t*>(ctx->tmp.get(n_subs * cells * 4));
        tfg::stripe_sum_kernel<<<(unsigned)std::min<size_t>((cells + 255) / 256, 1024), 256, 0, s>>>(
            d_st, (int)cells, (int)group_count, nullptr, d_subs);
        ck(cudaGetLastError(), "stripe_sum_kernel launch");
        ctx->launches++;
        ck(cudaMemcpyAsync(subs_out, d_subs, n_subs * cells * 4, cudaMemcpyDeviceToHost, s), "D2H subs");
      }
      if (counts_out) ck(cudaMemcpyAsync(counts_out, d_cnt, cells * 8, cudaMemcpyDeviceToHost, s), "D2H counts");
      ck(cudaStreamSynchronize(s), "stream sync");
      if (pixel_levels == levels) check_sync_flag(ctx, s);
      return;
    }
    // work items: stripe_rows(height, group_count) (parallel.hpp:76-89), cut into <= 64-row pieces
    std::vector<tfg::SubWork> work;
    const size_t base = height / group_count, extra = height % group_count;
    size_t row = 0;
    for (size_t g = 0; g < group_count; ++g) {
      const size_t end = row + base + (g < extra ? 1 : 0);
      for (size_t r = row; r < end; r += 64)
        work.push_back({(uint32_t)g, (uint32_t)r, (uint32_t)std::min(end, r + 64), (uint32_t)row});
      row = end;
    }
    const size_t sub_bytes = n_subs * cells * 4;
    char* scratch = static_cast<char*>(ctx->tmp.get(sub_bytes + work.size() * sizeof(tfg::SubWork) +
                                                         n_subs * 8 + 256));
    uint32_t* d_subs = reinterpret_cast<uint32_t*>(scratch);
    auto* d_work = reinterpret_cast<tfg::SubWork*>(scratch + ((sub_bytes + 15) & ~size_t(15)));
    auto* d_max = reinterpret_cast<unsigned long long*>(
        scratch + ((sub_bytes + 15) & ~size_t(15)) + ((work.size() * sizeof(tfg::SubWork) + 15) & ~size_t(15)));
    ck(cudaMemsetAsync(d_subs, 0, sub_bytes, s), "memset");
    ck(cudaMemcpyAsync(d_work, work.data(), work.size() * sizeof(tfg::SubWork), cudaMemcpyHostToDevice, s),
       "H2D work");
    long dr, dc;
    offset_of(distance, angle_deg, &dr, &dc);
    tfg::SubParams sp{};
    sp.img = d_img;
    sp.pitch = dpitch;
    sp.width = (int)width;
    sp.height = (int)height;
    sp.levels = levels;
    sp.pixel_levels = pixel_levels;
    sp.dr = (int)dr;
    sp.dc = (int)dc;
    sp.d = distance;
    sp.group_size = group_size;
    sp.copies = copies;
    sp.work = d_work;
    sp.subs = d_subs;
    const size_t smem = copies * cells * 4;
    sp.use_smem = smem <= kSubSmemBytes;
    if (sp.use_smem && smem > 48 * 1024)
      ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(tfg::glcm_subglcm_kernel),
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
         "cudaFuncSetAttribute");
    tfg::glcm_subglcm_kernel<<<(unsigned)work.size(), 256, sp.use_smem ? smem : 0, s>>>(sp);
    ck(cudaGetLastError(), "glcm_subglcm_kernel launch");
    ctx->launches++;
    if (per_copy_hottest_out) {
      tfg::subglcm_max_kernel<<<(unsigned)n_subs, 256, 0, s>>>(d_subs, (int)cells, d_max);
      ck(cudaGetLastError(), "subglcm_max_kernel launch");
      ctx->launches++;
      ck(cudaMemcpyAsync(per_copy_hottest_out, d_max, n_subs * 8, cudaMemcpyDeviceToHost, s), "D2H max");
    }
    if (subs_out) ck(cudaMemcpyAsync(subs_out, d_subs, sub_bytes, cudaMemcpyDeviceToHost, s), "D2H subs");
    if (counts_out) {
      auto* d_acc = static_cast<unsigned long long*>(ctx->acc.get(cells * 8));
      ck(cudaMemsetAsync(d_acc, 0, cells * 8, s), "memset");
      launch_vote(ctx, d_img, width, height, dpitch, 0, 1, height, pixel_levels, levels, distance, angle_deg,
                  flags & ~TFG_INPUT_DEVICE, d_acc, s);
      ck(cudaMemcpyAsync(counts_out, d_acc, cells * 8, cudaMemcpyDeviceToHost, s), "D2H counts");
    }
    ck(cudaStreamSynchronize(s), "stream sync");
    if (pixel_levels == levels) check_sync_flag(ctx, s);
  });
}

int tfg_symmetrize(tfg_ctx* ctx, const uint64_t* counts, int levels, uint64_t* out) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    check_levels(levels, "Glcm");
    DeviceGuard dg(ctx->device);
    const size_t cells = (size_t)levels * levels;
    auto* d = static_cast<unsigned long long*>(ctx->acc.get(cells * 8));
    ck(cudaMemcpyAsync(d, counts, cells * 8, cudaMemcpyHostToDevice, ctx->exec), "H2D");
    finish(ctx, d, 1, levels, TFG_SYMMETRIC, out, nullptr, nullptr, ctx->exec);
  });
}

int tfg_normalize(tfg_ctx* ctx, const uint64_t* counts, int levels, double* out) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    check_levels(levels, "Glcm");
    DeviceGuard dg(ctx->device);
    const size_t cells = (size_t)levels * levels;
    auto* d = static_cast<unsigned long long*>(ctx->acc.get(cells * 8));
    ck(cudaMemcpyAsync(d, counts, cells * 8, cudaMemcpyHostToDevice, ctx->exec), "H2D");
    finish(ctx, d, 1, levels, TFG_NORMALIZE, nullptr, out, nullptr, ctx->exec);
  });
}

int tfg_features(tfg_ctx* ctx, const double* probs, int levels, double* out5) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    if (levels < 1 || levels > 256) fail(TFG_INVALID_ARGUMENT, "extract_features: levels must be in [1, 256]");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->exec;
    const size_t cells = (size_t)levels * levels;
    auto* d_p = static_cast<double*>(ctx->probs.get(cells * 8));
    auto* d_f = static_cast<double*>(ctx->feats.get(5 * 8));
    int* d_e = static_cast<int*>(ctx->errs.get(2 * sizeof(int)));
    ck(cudaMemcpyAsync(d_p, probs, cells * 8, cudaMemcpyHostToDevice, s), "H2D");
    ck(cudaMemsetAsync(d_e, 0, 2 * sizeof(int), s), "memset");
    tfg::features_kernel<<<1, 1024, 0, s>>>(d_p, levels, d_f, d_e);
    ck(cudaGetLastError(), "features launch");
    ctx->launches++;
    int e = 0;
    double* h = static_cast<double*>(ctx->hout.get(64));
    ck(cudaMemcpyAsync(h, d_f, 5 * 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaMemcpyAsync(&e, d_e, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    if (e) fail(TFG_INVALID_ARGUMENT, "extract_features: input is not normalized");
    std::memcpy(out5, h, 5 * 8);
  });
}

int tfg_glcm_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch, size_t row_end,
                   int pixel_levels, int levels, int distance, int angle_deg, unsigned flags, uint64_t* d_counts,
                   void* stream) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);  // shared aux streams, events and scratch ordering
  return guarded([&] {
    check_levels(levels, "glcm");
    check_pixel_levels(pixel_levels, levels);
    check_angle(angle_deg);
    if (distance < 1 || (size_t)distance >= width)
      fail(TFG_INVALID_ARGUMENT, "glcm: degenerate geometry (d must be in [1, min(width, height)))");
    if ((reinterpret_cast<uintptr_t>(d_px) & 15) || (pitch % 16) || pitch < width)
      fail(TFG_INVALID_ARGUMENT, "glcm_async: device image must be 16-byte aligned with pitch % 16 == 0");
    if (row_end > height) fail(TFG_INVALID_ARGUMENT, "glcm_async: row_end > height");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
    if (pixel_levels == levels) launch_validate(ctx, d_px, width, height, pitch, 0, 1, levels, ctx->d_err, s);
    launch_vote(ctx, d_px, width, height, pitch, 0, 1, row_end, pixel_levels, levels, distance, angle_deg, flags,
                reinterpret_cast<unsigned long long*>(d_counts), s);
  });
}

int tfg_glcm_bands_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch,
                         size_t band_stride, size_t n_bands, int pixel_levels, int levels, int distance,
                         int angle_deg, unsigned flags, uint64_t* d_counts, void* stream) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);  // shared aux streams, events and scratch ordering
  return guarded([&] {
    check_levels(levels, "glcm");
    check_pixel_levels(pixel_levels, levels);
    check_angle(angle_deg);
    check_geometry(width, height, distance);
    if ((reinterpret_cast<uintptr_t>(d_px) & 15) || (pitch % 16) || pitch < width || (band_stride % 16))
      fail(TFG_INVALID_ARGUMENT, "glcm_async: device image must be 16-byte aligned with pitch % 16 == 0");
    if (n_bands < 1 || n_bands > 65535) fail(TFG_INVALID_ARGUMENT, "glcm: band count must be in [1, 65535]");
    if (n_bands > 1 && band_stride < pitch * height) fail(TFG_INVALID_ARGUMENT, "glcm: bands overlap");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (pixel_levels == levels)
      launch_validate(ctx, d_px, width, height, pitch, band_stride, (int)n_bands, levels, ctx->d_err, s);
    launch_vote(ctx, d_px, width, height, pitch, band_stride, (int)n_bands, height, pixel_levels, levels, distance,
                angle_deg, flags, reinterpret_cast<unsigned long long*>(d_counts), s);
  });
}

int tfg_glcm_multi_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch,
                         size_t band_stride, size_t n_bands, size_t row_end, int pixel_levels, int levels,
                         const int* distances, const int* angles_deg, int n_dt, unsigned flags, uint64_t* d_counts,
                         void* stream) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);  // shared aux streams, events and scratch ordering
  return guarded([&] {
    check_levels(levels, "glcm");
    check_pixel_levels(pixel_levels, levels);
    if (n_dt < 1 || !distances || !angles_deg) fail(TFG_INVALID_ARGUMENT, "glcm: need at least one (distance, angle)");
    for (int t = 0; t < n_dt; ++t) {
      check_angle(angles_deg[t]);
      if (distances[t] < 1 || (size_t)distances[t] >= width)
        fail(TFG_INVALID_ARGUMENT, "glcm: degenerate geometry (d must be in [1, min(width, height)))");
    }
    if ((reinterpret_cast<uintptr_t>(d_px) & 15) || (pitch % 16) || pitch < width || (n_bands > 1 && band_stride % 16))
      fail(TFG_INVALID_ARGUMENT, "glcm_async: device image must be 16-byte aligned with pitch % 16 == 0");
    if (n_bands < 1 || n_bands > 65535) fail(TFG_INVALID_ARGUMENT, "glcm: band count must be in [1, 65535]");
    if (n_bands > 1 && band_stride < pitch * height) fail(TFG_INVALID_ARGUMENT, "glcm: bands overlap");
    if (row_end > height) fail(TFG_INVALID_ARGUMENT, "glcm_async: row_end > height");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (pixel_levels == levels)
      launch_validate(ctx, d_px, width, height, pitch, band_stride, (int)n_bands, levels, ctx->d_err, s);
    const size_t per_dt = n_bands * (size_t)levels * levels;
    // every (d, theta) of an L <= 64 image or band batch in one launch
    if (launch_vote_jobs(ctx, d_px, width, height, pitch, band_stride, (int)n_bands, row_end, pixel_levels, levels,
                         distances, angles_deg, n_dt, flags, reinterpret_cast<unsigned long long*>(d_counts), per_dt,
                         s))
      return;
    // L <= 64 launches share no scratch (direct u64 atomics, per-CTA smem
    // tickets): fork them over the context's aux streams so one GLCM's
    // prologue/epilogue and tail overlap another's votes (small images are
    // launch- and tail-bound); L > 64 launches share the partials and the
    // grid-barrier counter and stay ordered on `s`.
    const bool fork = n_dt > 1 && (size_t)levels * levels <= 4096 && !(flags & TFG_SCHEME_GLOBAL);
    if (fork) ck(cudaEventRecord(ctx->fork_ev, s), "event record");
    for (int t = 0; t < n_dt; ++t) {
      cudaStream_t st = s;
      if (fork) {
        st = ctx->aux[t % tfg_ctx::kAux];
        if (t < tfg_ctx::kAux) ck(cudaStreamWaitEvent(st, ctx->fork_ev, 0), "wait");
      }
      launch_vote(ctx, d_px, width, height, pitch, band_stride, (int)n_bands, row_end, pixel_levels, levels,
                  distances[t], angles_deg[t], flags,
                  reinterpret_cast<unsigned long long*>(d_counts) + (size_t)t * per_dt, st);
    }
    if (fork) {
      for (int i = 0; i < std::min(n_dt, tfg_ctx::kAux); ++i) {
        ck(cudaEventRecord(ctx->join_ev[i], ctx->aux[i]), "event record");
        ck(cudaStreamWaitEvent(s, ctx->join_ev[i], 0), "wait");
      }
    }
  });
}

int tfg_glcm_jobs_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch,
                        size_t band_stride, size_t n_bands, size_t row_end, int pixel_levels, const int* levels,
                        const int* distances, const int* angles_deg, int n_jobs, unsigned flags, uint64_t* d_counts,
                        void* stream) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    if (n_jobs < 1 || !levels || !distances || !angles_deg) fail(TFG_INVALID_ARGUMENT, "glcm: need at least one job");
    for (int t = 0; t < n_jobs; ++t) {
      check_levels(levels[t], "glcm");
      check_pixel_levels(pixel_levels, levels[t]);
      check_angle(angles_deg[t]);
      if (distances[t] < 1 || (size_t)distances[t] >= width)
        fail(TFG_INVALID_ARGUMENT, "glcm: degenerate geometry (d must be in [1, min(width, height)))");
    }
    if ((reinterpret_cast<uintptr_t>(d_px) & 15) || (pitch % 16) || pitch < width || (n_bands > 1 && band_stride % 16))
      fail(TFG_INVALID_ARGUMENT, "glcm_async: device image must be 16-byte aligned with pitch % 16 == 0");
    if (n_bands < 1 || n_bands > 65535) fail(TFG_INVALID_ARGUMENT, "glcm: band count must be in [1, 65535]");
    if (n_bands > 1 && band_stride < pitch * height) fail(TFG_INVALID_ARGUMENT, "glcm: bands overlap");
    if (row_end > height) fail(TFG_INVALID_ARGUMENT, "glcm_async: row_end > height");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (pixel_levels < 256) {
      // pre-quantised input: every job has levels == pixel_levels (check_pixel_levels)
      launch_validate(ctx, d_px, width, height, pitch, band_stride, (int)n_bands, pixel_levels, ctx->d_err, s);
    }
    std::vector<unsigned long long*> outs((size_t)n_jobs);
    size_t off = 0;
    for (int t = 0; t < n_jobs; ++t) {
      outs[t] = reinterpret_cast<unsigned long long*>(d_counts) + off;
      off += n_bands * (size_t)levels[t] * levels[t];
    }
    launch_job_set(ctx, d_px, width, height, pitch, band_stride, (int)n_bands, row_end, pixel_levels, levels,
                   distances, angles_deg, outs.data(), n_jobs, flags, s);
  });
}

int tfg_post_async(tfg_ctx* ctx, const uint64_t* d_counts, int levels, unsigned flags, uint64_t* d_sym_out,
                   double* d_probs_out, double* d_feats_out, void* stream) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);  // shared aux streams, events and scratch ordering
  return guarded([&] {
    check_levels(levels, "Glcm");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
    const size_t cells = (size_t)levels * levels;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(d_counts);
    if ((flags & TFG_SYMMETRIC) && d_sym_out) {
      dim3 grid((unsigned)std::min<size_t>((cells + 255) / 256, 1024), 1);
      tfg::symmetrize_kernel<<<grid, 256, 0, s>>>(src, levels, reinterpret_cast<unsigned long long*>(d_sym_out));
      ck(cudaGetLastError(), "symmetrize launch");
      ctx->launches++;
      src = reinterpret_cast<const unsigned long long*>(d_sym_out);
    }
    if ((flags & (TFG_NORMALIZE | TFG_FEATURES)) && d_probs_out) {
      tfg::normalize_kernel<<<1, 1024, 0, s>>>(src, levels, d_probs_out, ctx->d_err + 1);
      ck(cudaGetLastError(), "normalize launch");
      ctx->launches++;
      if ((flags & TFG_FEATURES) && d_feats_out) {
        tfg::features_kernel<<<1, 1024, 0, s>>>(d_probs_out, levels, d_feats_out, ctx->d_err + 2);
        ck(cudaGetLastError(), "features launch");
        ctx->launches++;
      }
    }
  });
}

int tfg_synth_noise_device(tfg_ctx* ctx, size_t width, size_t height, uint32_t seed, uint8_t* d_out,
                           size_t pitch, void* stream) {
  if (width < 2 || height < 2) {
    g_error = "synth_noise: dimensions must be >= 2";
    return TFG_INVALID_ARGUMENT;
  }
  return tfg_synth_noise_rows_device(ctx, width, 0, height, seed, d_out, pitch, stream);
}

int tfg_synth_noise_rows_device(tfg_ctx* ctx, size_t width, size_t row0, size_t rows, uint32_t seed,
                                uint8_t* d_out, size_t pitch, void* stream) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    if (width < 2 || rows < 1) fail(TFG_INVALID_ARGUMENT, "synth_noise: dimensions must be >= 2");
    if (!d_out || pitch < width) fail(TFG_INVALID_ARGUMENT, "synth_noise_device: null output or pitch < width");
    DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned long long n = (unsigned long long)width * rows;
    const unsigned long long first = (unsigned long long)width * row0;  // generator output of pixel (row0, 0)
    // up to ~4 segments per SM (each a serial chain of 624-output twists) of
    // >= ~1M outputs: each window costs ~4 ms of host jump-ahead per thread
    const unsigned long long per = (n + (unsigned long long)ctx->num_sms * 4 - 1) / ((unsigned long long)ctx->num_sms * 4);
    const unsigned long long seglen = std::max<unsigned long long>(624ull * 1680, (per + 623) / 624 * 624);
    const size_t nseg = (size_t)((n + seglen - 1) / seglen);
    std::vector<uint32_t> win(nseg * 624);
    const int rc = tfg_mt19937_windows(seed, first, seglen, nseg, win.data(), 0);
    if (rc != TFG_OK) fail(rc, "synth_noise_device: generator jump-ahead failed");
    uint32_t* d_win = static_cast<uint32_t*>(ctx->mtwin.get(win.size() * sizeof(uint32_t)));
    ck(cudaMemcpyAsync(d_win, win.data(), win.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s), "H2D");
    tfg::synth_noise_kernel<<<(unsigned)nseg, 256, 0, s>>>(d_win, seglen, n, width, pitch, d_out);
    ck(cudaGetLastError(), "synth_noise_kernel launch");
    ctx->launches++;
    // the window buffer is reused by the next call: finish before returning
    ck(cudaStreamSynchronize(s), "sync");
  });
}

int tfg_check_async_errors(tfg_ctx* ctx) {
  if (!ctx) { g_error = "null context"; return TFG_INVALID_ARGUMENT; }
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded([&] {
    DeviceGuard dg(ctx->device);
    ck(cudaDeviceSynchronize(), "sync");
    int e[3] = {0, 0, 0};
    ck(cudaMemcpy(e, ctx->d_err, sizeof e, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemset(ctx->d_err, 0, sizeof e), "memset");
    if (e[0]) fail(TFG_INVALID_ARGUMENT, "QuantizedImage: pixel value exceeds gray level");
    if (e[1]) fail(TFG_INVALID_ARGUMENT, "normalize: all-zero matrix");
    if (e[2]) fail(TFG_INVALID_ARGUMENT, "extract_features: input is not normalized");
  });
}

}  // extern "C"

#include "tfg_multi_gpu.inc"
