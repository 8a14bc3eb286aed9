/*
 * texforge_cuda.h — C ABI of the B200-native GLCM engine (libtexforge_cuda.so).
 *
 * This is the drop-in boundary beneath the reference's header-only C++ API
 * (R/ = /root/reference/proj/, namespace texforge). Every heavy reference
 * function maps to one entry point here; the C++ shim headers in
 * include/texforge/ and the Python mirror in
 * paper_1710_06189_b200/texforge.py forward to these. Plain pointers and sizes
 * only: no C++ types, no torch types, no exceptions cross this boundary.
 *
 * Conventions (all from the reference):
 *  - images are u8 row-major; `pitch` >= width is the row stride in bytes;
 *  - a GLCM is levels*levels u64, row = reference (displaced) gray, column =
 *    anchor gray (R/include/texforge/glcm.hpp:35-39);
 *  - (distance, angle) -> (drow, dcol): 0:(0,+d) 45:(+d,-d) 90:(+d,0)
 *    135:(+d,+d) (glcm.hpp:71-80);
 *  - `pixel_levels` describes the input pixels: 256 = raw 8-bit gray, quantised
 *    on the fly as q = (v*levels)>>8 (image.hpp:55-62, fused into the vote);
 *    == levels = an already-quantised QuantizedImage whose values must be
 *    < levels (image.hpp:46-48; violation -> TFG_INVALID_ARGUMENT).
 *
 * Return codes: 0 OK; 1 invalid argument (the message text equals the
 * reference's std::invalid_argument text where one exists); 2 CUDA error;
 * 3 NCCL/collective error; 4 out of memory; 5 chunk-source failure (the
 * reference's PipelineError, pipeline.hpp:25-29; tfg_last_error_chunk() holds
 * the failing chunk index). The message is in tfg_last_error() (thread-local).
 *
 * Threading: every synchronous call blocks until its results are on the host.
 * A context serialises its own calls with a mutex; use one context per thread
 * for concurrency. The *_async entry points only enqueue on the caller's stream.
 */
#ifndef TEXFORGE_CUDA_H
#define TEXFORGE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFG_ABI_VERSION 1

enum tfg_status {
  TFG_OK = 0,
  TFG_INVALID_ARGUMENT = 1,
  TFG_CUDA_ERROR = 2,
  TFG_COLLECTIVE_ERROR = 3,
  TFG_OUT_OF_MEMORY = 4,
  TFG_SOURCE_ERROR = 5
};

/* flags for tfg_glcm / tfg_glcm_bands / tfg_glcm_chunked */
enum tfg_flags {
  TFG_INPUT_DEVICE = 1u << 0,   /* px is a device pointer (else host memory) */
  TFG_SYMMETRIC = 1u << 1,      /* counts_out = M + M^T          (glcm.hpp:150-156) */
  TFG_NORMALIZE = 1u << 2,      /* probs_out = normalize(counts) (glcm.hpp:167-177) */
  TFG_FEATURES = 1u << 3,       /* feats_out = extract_features  (features.hpp:37-69) */
  TFG_SCHEME_GLOBAL = 1u << 4,  /* Scheme 1: per-pair global atomics (ablation, parallel.hpp:121-152) */
  TFG_SEQUENTIAL = 1u << 5      /* chunked: no copy/compute overlap (pipeline.hpp:205-208) */
};

/* Vote strategy override (testing / ablation). 0 = automatic by levels. */
#define TFG_STRATEGY_SHIFT 16
#define TFG_STRATEGY(s) ((unsigned)(s) << TFG_STRATEGY_SHIFT)
enum tfg_strategy {
  TFG_STRAT_AUTO = 0,
  TFG_STRAT_COPIES32 = 1, /* 32 lane-interleaved u32 sub-GLCM copies per CTA (L <= 32)  */
  TFG_STRAT_COPIES8 = 2,  /* 8 interleaved u32 copies per CTA (L <= 64)                 */
  TFG_STRAT_COPY1 = 3,    /* one u32 copy per CTA (L <= 238)                            */
  TFG_STRAT_PACKED16 = 4, /* one copy of packed u16 counters + exact spill (L <= 256)   */
  TFG_STRAT_P16X16 = 5    /* 16 bank-pair copies of packed u16 counters (L <= 64)       */
};

typedef struct tfg_ctx tfg_ctx;

/*
 * Chunk source callback (adapts texforge::ChunkSource::fetch,
 * R/include/texforge/pipeline.hpp:77-84). Must fill `dst` (pinned, row stride
 * `width`) with rows [owned_row_start, buffer_row_end) of the image, pixels as
 * described by `pixel_levels`. Return 0 on success; non-zero aborts the
 * pipeline with TFG_SOURCE_ERROR. `err`/`err_len` receive an optional message.
 */
typedef int (*tfg_fetch_fn)(void* user, size_t chunk_index, size_t owned_row_start,
                            size_t owned_row_end, size_t buffer_row_end, uint8_t* dst,
                            char* err, size_t err_len);

/* ---- context ------------------------------------------------------------ */
int tfg_ctx_create(tfg_ctx** out, int device, unsigned flags);
void tfg_ctx_destroy(tfg_ctx* ctx);
const char* tfg_last_error(void);
size_t tfg_last_error_chunk(void);
int tfg_abi_version(void);
/* where `p` lives: 0 pageable host, 1 pinned host, 2 device, 3 managed */
int tfg_memory_kind(const void* p);
/* number of engine kernels this context has launched (evidence counter) */
uint64_t tfg_launch_count(tfg_ctx* ctx);

/* ---- host-side geometry (glcm.hpp:71-104, pipeline.hpp:48-73, parallel.hpp:39-61) */
int tfg_neighbor_offset(int distance, int angle_deg, long* drow, long* dcol);
int tfg_valid_pair_count(size_t width, size_t height, int distance, int angle_deg, uint64_t* out);
/* specs_out: chunk_count x {owned_row_start, owned_row_end, buffer_row_end} */
int tfg_partition(size_t width, size_t height, int distance, int angle_deg, size_t chunk_count,
                  uint64_t* specs_out);
int tfg_plan(int levels, size_t scratch_budget, unsigned worker_count, unsigned* copies,
             unsigned* groups_per_unit, int* degraded);

/* ---- synthetic inputs (image.hpp:76-116), host generators, bit-identical --- */
int tfg_synth_noise(size_t width, size_t height, uint32_t seed, uint8_t* out);
int tfg_synth_smooth(size_t width, size_t height, uint32_t seed, uint8_t* out, int threads);

/* std::mt19937 jump-ahead (replaces stepping the reference's sequential
 * generator, image.hpp:109-116). Writes `count` generator windows of 624
 * words, window s at output index first + s*stride of std::mt19937(seed):
 * a generator whose state array is that window emits outputs k, k+1, ...
 * after one twist. Host only; threads <= 0: all hardware threads. */
int tfg_mt19937_windows(uint32_t seed, uint64_t first, uint64_t stride, size_t count, uint32_t* out,
                        int threads);

/* synth_noise over n pixels on `threads` host threads (<= 0: all), each
 * segment generated from its jump-ahead window; bit-identical to the
 * sequential generator. tfg_synth_noise uses it for images >= 4 Mpixel. */
int tfg_synth_noise_parallel(size_t n, uint32_t seed, uint8_t* out, int threads);

/* synth_noise (image.hpp:109-116) generated ON THE DEVICE, bit-identical:
 * pixel (y, x) of the width x height image -> d_out[y*pitch + x]. Segments of
 * the generator sequence run in parallel from jump-ahead windows. Returns
 * after the kernel has finished on `stream`. */
int tfg_synth_noise_device(tfg_ctx* ctx, size_t width, size_t height, uint32_t seed, uint8_t* d_out,
                           size_t pitch, void* stream);

/* Rows [row0, row0 + rows) of synth_noise(width, <any height>, seed) on the
 * device (pixel (y, x) of those rows -> d_out[(y - row0)*pitch + x]): the
 * generator jumps straight to output row0*width, so a GPU of a row-partitioned
 * image makes only its own shard. Returns after the kernel has finished. */
int tfg_synth_noise_rows_device(tfg_ctx* ctx, size_t width, size_t row0, size_t rows, uint32_t seed,
                                uint8_t* d_out, size_t pitch, void* stream);

/* ---- the hot path ---------------------------------------------------------- */

/* quantize (image.hpp:55-62) on the device; gray/out host or device per flags */
int tfg_quantize(tfg_ctx* ctx, const uint8_t* gray, size_t n, int levels, uint8_t* out,
                 unsigned flags);

/*
 * One image, n_dt (distance, angle) pairs. Replaces compute_glcm_serial
 * (glcm.hpp:144), compute_glcm_privatized (parallel.hpp:240) and, with
 * TFG_SCHEME_GLOBAL, compute_glcm_shared (parallel.hpp:143). Host input is
 * streamed through the K-chunk copy/compute pipeline (Scheme 3).
 * counts_out: n_dt*L*L u64 (host). probs_out: n_dt*L*L f64 or NULL.
 * feats_out: n_dt*5 f64 {energy, contrast, homogeneity, entropy, correlation} or NULL.
 */
int tfg_glcm(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, size_t pitch,
             int pixel_levels, int levels, const int* distances, const int* angles_deg, int n_dt,
             unsigned flags, uint64_t* counts_out, double* probs_out, double* feats_out);

/*
 * Multispectral batch: n_bands images of width x height, band b at
 * px + b*band_stride. counts_out: n_bands*n_dt*L*L (band-major).
 */
int tfg_glcm_bands(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, size_t pitch,
                   size_t band_stride, size_t n_bands, int pixel_levels, int levels,
                   const int* distances, const int* angles_deg, int n_dt, unsigned flags,
                   uint64_t* counts_out, double* probs_out, double* feats_out);

/*
 * One row shard of a larger image (the multi-GPU row partition,
 * partition() semantics, pipeline.hpp:48-73): `px` holds `buffer_rows` rows,
 * of which anchors in rows [0, owned_rows) vote; rows [owned_rows,
 * buffer_rows) are the next shard's read-only halo. Host input streams
 * through the Scheme-3 pipeline, device input (TFG_INPUT_DEVICE) votes in
 * place. n_bands images of the same shape may be passed at band_stride bytes
 * apart (one continuous copy/vote pipeline over all of them).
 * counts_out: n_bands*n_dt*L*L u64 partial counts (host, band-major) for the
 * caller's reduce (merge_chunk_glcms, pipeline.hpp:231-240, or one NCCL reduce).
 */
int tfg_glcm_shard(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t buffer_rows, size_t owned_rows,
                   size_t pitch, size_t band_stride, size_t n_bands, int pixel_levels, int levels,
                   const int* distances, const int* angles_deg, int n_dt, unsigned flags, uint64_t* counts_out);

/*
 * tfg_glcm_shard with per-job levels: job t = (levels[t], distances[t],
 * angles_deg[t]). Replaces a loop of the reference's compute_glcm_chunked /
 * compute_glcm_serial calls over (L, d, theta) on one image
 * (R/include/texforge/pipeline.hpp:246, glcm.hpp:144; R/tools/texforge.cpp:
 * 218-236 loops them): every band of the HOST image is copied up once and all its
 * jobs vote from that copy (jobs that share a kernel instantiation in one
 * launch). counts_out: [band][job][levels[t]^2] u64, jobs back to back.
 * Counts only (no post-processing flags). n_jobs <= 64.
 */
int tfg_glcm_shard_jobs(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t buffer_rows, size_t owned_rows,
                        size_t band_stride, size_t n_bands, int pixel_levels, const int* levels,
                        const int* distances, const int* angles_deg, int n_jobs, unsigned flags,
                        uint64_t* counts_out);

/*
 * Scheme 3 (compute_glcm_chunked, pipeline.hpp:246-337): K row chunks from
 * partition(), fetched by `fetch` into a pinned ring, H2D on a copy stream
 * overlapped with voting on the exec stream into one device accumulator.
 */
int tfg_glcm_chunked(tfg_ctx* ctx, size_t width, size_t height, int pixel_levels, int levels,
                     const int* distances, const int* angles_deg, int n_dt, size_t chunk_count,
                     tfg_fetch_fn fetch, void* user, unsigned flags, uint64_t* counts_out,
                     double* probs_out, double* feats_out);

/*
 * Privatised sub-GLCMs with the reference's exact routing (compute_subglcms,
 * R/include/texforge/parallel.hpp:160-225; per_copy_hottest of
 * compute_glcm_privatized, parallel.hpp:240-254): `group_count` groups own
 * stripe_rows(height, group_count) (parallel.hpp:76-89); stripe pixel k votes
 * into copy ((k - stripe_begin*width) mod group_size) mod copies.
 * group_count must already be resolved by the caller (1 <= group_count <= height).
 * subs_out: group_count*copies*L*L u32 (group-major) or NULL; counts_out: L*L
 * u64 or NULL; per_copy_hottest_out: group_count*copies u64 or NULL.
 */
int tfg_subglcms(tfg_ctx* ctx, const uint8_t* px, size_t width, size_t height, int pixel_levels, int levels,
                 int distance, int angle_deg, unsigned group_size, unsigned copies, size_t group_count,
                 unsigned flags, uint32_t* subs_out, uint64_t* counts_out, uint64_t* per_copy_hottest_out);

/* post-processing on the device (host in/out) */
int tfg_symmetrize(tfg_ctx* ctx, const uint64_t* counts, int levels, uint64_t* out);
int tfg_normalize(tfg_ctx* ctx, const uint64_t* counts, int levels, double* out);
int tfg_features(tfg_ctx* ctx, const double* probs, int levels, double* out5);

/*
 * Device-resident asynchronous entry (no host sync): ADDS the GLCM of one
 * (d, theta) of a device image into d_counts (L*L u64, device) on `stream`
 * (a cudaStream_t; NULL = the legacy default stream, as in CUDA). `row_end` limits the
 * anchor rows (the owned rows of a shard; pass height for the whole image):
 * rows [row_end, height) are read-only halo, exactly like a ChunkSpec.
 * Used by the benchmark, the multi-GPU row shards and the parity tests.
 * A context's async calls share its scratch (per-CTA partials), so they must
 * be ordered on ONE stream (or the caller must serialise them).
 */
int tfg_glcm_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch,
                   size_t row_end, int pixel_levels, int levels, int distance, int angle_deg,
                   unsigned flags, uint64_t* d_counts, void* stream);

/* Multispectral batch on the device, one (d, theta), one launch (blockIdx.y =
 * band): ADDS band b's GLCM into d_counts + b*L*L. Same stream rule as
 * tfg_glcm_async: a context's async calls must be ordered on one stream. */
int tfg_glcm_bands_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch,
                         size_t band_stride, size_t n_bands, int pixel_levels, int levels, int distance,
                         int angle_deg, unsigned flags, uint64_t* d_counts, void* stream);

/* Every (d, theta) of a device image (or band batch) in one call: ADDS the
 * GLCMs into d_counts laid out [n_dt][n_bands][L*L]; anchors in rows
 * [0, row_end) vote (row_end = height for whole images). One validation pass,
 * n_dt vote launches enqueued back to back on `stream` (no host round trip
 * per GLCM). Same stream rule as tfg_glcm_async. */
int tfg_glcm_multi_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch,
                         size_t band_stride, size_t n_bands, size_t row_end, int pixel_levels, int levels,
                         const int* distances, const int* angles_deg, int n_dt, unsigned flags, uint64_t* d_counts,
                         void* stream);

/*
 * Several GLCMs of one device image (or band batch) with per-job levels and
 * (d, theta) — a batch of compute_glcm_serial calls (R/include/texforge/
 * glcm.hpp:144): equivalent to n_jobs tfg_glcm_async calls, job t's counts at
 * d_counts + sum_{u<t} n_bands * levels[u]^2 (band-major). Jobs that share a
 * kernel instantiation (same quantiser and layout; for L > 64 also the same L
 * and reference-window group, as one cooperative launch) run as one launch
 * of up to 8 jobs. Stream-ordered like tfg_glcm_multi_async.
 */
int tfg_glcm_jobs_async(tfg_ctx* ctx, const uint8_t* d_px, size_t width, size_t height, size_t pitch,
                        size_t band_stride, size_t n_bands, size_t row_end, int pixel_levels, const int* levels,
                        const int* distances, const int* angles_deg, int n_jobs, unsigned flags, uint64_t* d_counts,
                        void* stream);

/* Device post-processing on `stream`: symmetrize (in place allowed? no: out != in). */
int tfg_post_async(tfg_ctx* ctx, const uint64_t* d_counts, int levels, unsigned flags,
                   uint64_t* d_sym_out, double* d_probs_out, double* d_feats_out, void* stream);

/* ---- multi-GPU ---------------------------------------------
 * One process, n GPUs: a group of engine contexts plus one NCCL communicator
 * over them (ncclCommInitAll; NVLink/NVSwitch on a B200 box). Failures of a
 * collective return TFG_COLLECTIVE_ERROR. */
typedef struct tfg_group tfg_group;

/* devices: n_gpus CUDA ordinals, or NULL for 0..n_gpus-1. flags:
 * TFG_GROUP_HOST_REDUCE sums the partials through host memory instead of
 * NCCL and lets contexts share a device (testing the multi-GPU split on
 * fewer GPUs; NCCL refuses two ranks on one GPU). */
#define TFG_GROUP_HOST_REDUCE (1u << 0)
int tfg_group_create(tfg_group** out, int n_gpus, const int* devices, unsigned flags);
void tfg_group_destroy(tfg_group* g);
int tfg_group_size(const tfg_group* g);
tfg_ctx* tfg_group_ctx(tfg_group* g, int i);
uint64_t tfg_group_launch_count(tfg_group* g);

/* One host image row-partitioned over the group: partition(W, H, p, G)
 * (R/include/texforge/pipeline.hpp:48-73) gives GPU g its owned rows plus the
 * d-row halo, which it streams through its own Scheme-3 copy/vote pipeline,
 * voting only its owned anchors; the partial GLCMs are summed with ONE
 * ncclReduce into GPU 0 (exact integer sums, like merge_chunk_glcms,
 * pipeline.hpp:231-240), then post-processed there. Same outputs and errors
 * as tfg_glcm (which replaces compute_glcm_serial, glcm.hpp:144). */
int tfg_group_glcm(tfg_group* g, const uint8_t* px, size_t width, size_t height, int pixel_levels, int levels,
                   const int* distances, const int* angles_deg, int n_dt, unsigned flags, uint64_t* counts_out,
                   double* probs_out, double* feats_out);

/* Multispectral batch sharded over the group: contiguous blocks of bands per
 * GPU, no collective (each GPU writes its own bands' results). Same layout as
 * tfg_glcm_bands. */
int tfg_group_glcm_bands(tfg_group* g, const uint8_t* px, size_t width, size_t height, size_t band_stride,
                         size_t n_bands, int pixel_levels, int levels, const int* distances, const int* angles_deg,
                         int n_dt, unsigned flags, uint64_t* counts_out, double* probs_out, double* feats_out);

/* Scheme 3 over the group (compute_glcm_chunked, pipeline.hpp:246-337): chunk i
 * of partition(W, H, p, K) runs on GPU floor(i*G/K); `fetch` calls are
 * serialised (never concurrent); one ncclReduce. A fetch failure returns
 * TFG_SOURCE_ERROR with tfg_last_error_chunk() = the chunk index. */
int tfg_group_glcm_chunked(tfg_group* g, size_t width, size_t height, int pixel_levels, int levels,
                           const int* distances, const int* angles_deg, int n_dt, size_t chunk_count,
                           tfg_fetch_fn fetch, void* user, unsigned flags, uint64_t* counts_out, double* probs_out,
                           double* feats_out);

/* One process per GPU (torchrun-style): a rank's NCCL communicator. */
typedef struct tfg_comm tfg_comm;
#define TFG_COMM_ID_BYTES 128
/* ncclGetUniqueId on the root rank; the caller ships the bytes to every rank. */
int tfg_comm_unique_id(uint8_t* id /* TFG_COMM_ID_BYTES */);
int tfg_comm_init_rank(tfg_comm** out, tfg_ctx* ctx, int nranks, int rank, const uint8_t* id);
void tfg_comm_destroy(tfg_comm* c);
/* In-place SUM of n u64 device counts onto `root` (one ncclReduce on `stream`). */
int tfg_comm_reduce_counts(tfg_comm* c, uint64_t* d_counts, size_t n, int root, void* stream);
/* Row-partition halo (pipeline.hpp:60-61): rank r sends its first `halo` rows
 * of d_slab to rank r-1 and receives rank r+1's first `halo` rows into rows
 * [owned_rows, owned_rows + halo) of its own slab (ncclSend/ncclRecv). */
int tfg_comm_exchange_halo(tfg_comm* c, uint8_t* d_slab, size_t pitch, size_t owned_rows, size_t halo,
                           void* stream);
/* In-place MAX all-reduce of n f64 (timing: the slowest rank defines a step). */
int tfg_comm_allreduce_max_f64(tfg_comm* c, double* d_vals, size_t n, void* stream);

/* Device error flag accumulated by *_async calls (non-zero = a quantised input held a
 * value >= levels); reading it synchronises the context's streams and clears it. */
int tfg_check_async_errors(tfg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TEXFORGE_CUDA_H */
