/*
 * floodstream.h — C ABI of libfloodstream, the B200-native (sm_100a) backend for the
 * flood-ensemble overlap path of arXiv 2104.14667 (reference package `floodstream`).
 *
 * Plain pointers and sizes only; no torch/numpy types.  Every entry point returns an
 * int status (FS_OK on success) and leaves a thread-local message in fs_last_error().
 * All entry points are re-entrant: each calling thread gets its own CUDA stream and
 * scratch buffers on the calling thread's current device (see fs_set_device), and
 * ensemble handles carry their own lock.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/floodstream/):
 *   fs_accumulate_into  <- _kernels_np.py:16-18   accumulate_into(counts, cells)
 *                          _accel.pyx:13-21        (Cython twin)
 *   fs_overlap_counts   <- _kernels_np.py:21-23   overlap_counts(counts, n_inputs)
 *                          _accel.pyx:24-33
 *   fs_pair_counts      <- _kernels_np.py:26-32   pair_counts(a, b)
 *                          _accel.pyx:36-51
 *   fs_composite_fill   <- _kernels_np.py:35-47   composite_fill(counts, n_inputs, out)
 *                          _accel.pyx:54-73
 *   fs_accumulate_many  <- analytics.py:118-120   the per-surface loop of accumulate()
 *   fs_gram_many        <- analytics.py:174-181   the i<j pair_counts loop of similarity_matrix()
 *   fs_ensemble_*       <- streaming.py:134-217 + :394-433 (build_schedule / run_stream) and
 *                          service.py:143-175 (resident recompute of the working set)
 *   fs_cluster_complete_linkage <- analytics.py:184-226 cluster_surfaces() merge loop
 *   fs_outlier_scores   <- analytics.py:229-240   outlier_scores() reduction
 *   fs_similarity_from_gram, fs_similarity_outliers_device
 *                       <- analytics.py:165-181   jaccard() / similarity_matrix() on the
 *                          exact pair counts, and :229-240 (on the device)
 *   fs_time_transform / fs_time_h2d <- device.py:376-401 transform_time / transfer_time
 *                          (the reference's modelled costs, measured)
 *   fs_synth_host / fs_synth_gpu    <- bench.py:472-475 input generation (test/bench input)
 */
#ifndef FLOODSTREAM_H
#define FLOODSTREAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_ABI_VERSION 1

/* status codes */
#define FS_OK 0
#define FS_EINVAL 1  /* bad argument (maps to ValueError)             */
#define FS_ECUDA 2   /* CUDA runtime / device failure (RuntimeError)  */
#define FS_ENOMEM 3  /* device or pinned allocation failed            */
#define FS_ENODEV 4  /* no CUDA device visible                        */

/* streaming variants, same names as streaming.py:54-58 */
#define FS_VARIANT_1B_INITIAL 0
#define FS_VARIANT_2B_INITIAL 1
#define FS_VARIANT_1B_FINAL 2
#define FS_VARIANT_2B_FINAL 3

/* Gram (pairwise intersection) engines */
#define FS_GRAM_AUTO 0
#define FS_GRAM_POPC 1   /* CUDA-core AND+POPC on bit-packed masks           */
#define FS_GRAM_TC_I8 2  /* tcgen05 kind::i8, bits expanded to u8 in SMEM    */
#define FS_GRAM_TC_F4 3  /* tcgen05 kind::mxf4 (bits expanded to e2m1 0/1 in SMEM, block
                            scale 1, f32 exact per <= 2^24-px K chunk): diagonal 256-mask
                            panels on one CTA each, off-diagonal 256 x 256 tiles on CTA
                            pairs (cta_group::2, M = 256, N = 256)                 */

/* ---- housekeeping ------------------------------------------------------ */
const char *fs_last_error(void);
int fs_abi_version(void);
int fs_device_count(int *out);
int fs_set_device(int device);          /* binds the calling thread */
int fs_get_device(int *out);
int fs_synchronize(void);               /* drains the calling thread's stream */

/* ---- reference primitive protocol (host buffers, one mask/pair per call) ---- */
int fs_accumulate_into(uint32_t *counts, const uint8_t *cells, uint64_t n);
int fs_overlap_counts(const uint32_t *counts, uint64_t n, uint64_t n_inputs, int64_t *bins);
int fs_pair_counts(const uint8_t *a, const uint8_t *b, uint64_t n, int64_t *inter,
                   int64_t *uni);
int fs_composite_fill(const uint32_t *counts, uint64_t n, uint64_t n_inputs, uint8_t *out);

/* ---- batched host-level extensions (one upload per mask, fused passes) ---- */
/* counts[p] += #{s < k : cells[s][p] > 0}                                     */
int fs_accumulate_many(uint32_t *counts, const uint8_t *const *cells, uint32_t k, uint64_t n);
/* gram[i*k+j] = |wet(cells[i]) & wet(cells[j])| for all i, j (int64, symmetric) */
int fs_gram_many(const uint8_t *const *cells, uint32_t k, uint64_t n, int64_t *gram);
/* Both calls above keep the stack bit-packed in HBM, in one cache per device keyed by
 * a 128-bit fingerprint of each raster's bytes (hashed on host threads per call): a
 * raster whose content is already resident is not uploaded again, so the drop-in
 * sequence accumulate -> similarity_matrix -> outlier_scores -> cluster_surfaces
 * (analytics.py:106-240) uploads the stack once.  Shared by all threads (one lock per
 * device); at most 4 GiB of packed masks stay cached between calls.                 */
int fs_stack_cache_release(void);  /* free the calling device's cache */
int fs_stack_cache_info(uint32_t *slots_valid, uint32_t *capacity, uint64_t *pixels);

/* ---- resident ensemble: bit-packed masks kept in HBM ---------------------- */
typedef struct fs_ensemble fs_ensemble;

/* Per-item measured timings of one streamed upload (streaming.py:247-261). */
typedef struct fs_stream_item {
  float host_us;   /* hidden host copy (initial variants), else 0 */
  float copy_us;   /* H2D DMA of the raw uint8 raster            */
  float xform_us;  /* binarize + bit-pack transform kernel        */
  float kernel_us; /* per-item accumulate kernel (0 if not run)   */
} fs_stream_item;

typedef struct fs_stream_report {
  double total_us;       /* first op start -> last op end (device clock) */
  uint32_t n_items;
  fs_stream_item *items; /* caller-owned array of n_items, may be NULL */
} fs_stream_report;

int fs_ensemble_create(uint64_t pixels, uint32_t capacity, fs_ensemble **out);
int fs_ensemble_destroy(fs_ensemble *ens);
int fs_ensemble_info(const fs_ensemble *ens, uint64_t *pixels, uint32_t *capacity,
                     uint64_t *words_per_mask, int *device);
/* Device pointer to the packed masks: tile-interleaved, word w of slot s at
 * ((w / 32) * capacity + s) * 32 + w % 32, pixel 32*w + b in bit b (LSB first).     */
int fs_ensemble_packed_ptr(const fs_ensemble *ens, const uint32_t **out);

/* Stream k host rasters (uint8, `pixels` bytes each) through the variant's event
 * DAG (streaming.py:150-215): H2D copy -> pack into slot first + (i % slot_wrap)
 * (slot_wrap == 0: first + i).  with_kernel != 0 also runs the per-item accumulate
 * into the ensemble's running count grid (zeroed first when reset_counts != 0), as
 * run_stream's kernel[i] nodes do.                                                 */
int fs_ensemble_stream(fs_ensemble *ens, uint32_t first, uint32_t slot_wrap,
                       const uint8_t *const *host, uint32_t k, int variant, int with_kernel,
                       int reset_counts, fs_stream_report *rep);
/* Generate synthetic flood-like masks directly into slots (see fs_synth_host). */
int fs_ensemble_synth(fs_ensemble *ens, uint32_t first, uint32_t k, uint64_t seed,
                      uint32_t width, uint32_t height, uint64_t row0, uint32_t members,
                      double eps, uint64_t mask_index0);

/* Fused overlap pass over slots[0..k): counts, histogram and composite in one read
 * of the packed masks.  Surfaces are cycled to n_inputs = cycles*k + remainder
 * (streaming.py:417-425).  Any output pointer may be NULL.  Outputs are HOST
 * pointers unless `device_outputs` is set.  bins has n_inputs+1 entries (int64).  */
int fs_ensemble_overlap(fs_ensemble *ens, const uint32_t *slots, uint32_t k, uint64_t cycles,
                        uint32_t remainder, uint32_t *counts, int64_t *bins, uint8_t *rgba,
                        int device_outputs);
/* Running count grid of fs_ensemble_stream(with_kernel) -> host (or device) */
int fs_ensemble_running_counts(fs_ensemble *ens, uint32_t *counts, int64_t *bins,
                               uint8_t *rgba, uint64_t n_inputs, int device_outputs);
/* Pairwise intersection counts over slots: gram[i*k+j] int64 (host or device). */
int fs_ensemble_gram(fs_ensemble *ens, const uint32_t *slots, uint32_t k, int engine,
                     int64_t *gram, int device_outputs);
/* One full recompute of the working set (service.py:143-175 + the /clusters and
 * /outliers Gram, analytics.py:106-181): counts, histogram (k+1 bins), composite and
 * Gram over slots[0..k), weights 1.  With a tensor-core engine and k <= 256 the
 * overlap products come out of the Gram's diagonal CTAs (one HBM read of the packed
 * masks for everything; *fused = 1), else from the separate overlap kernel.  Any
 * output may be NULL (gram NULL: overlap only).                                     */
int fs_ensemble_recompute(fs_ensemble *ens, const uint32_t *slots, uint32_t k, int engine,
                          uint32_t *counts, int64_t *bins, uint8_t *rgba, int64_t *gram,
                          int device_outputs, int *fused);
/* Duration (ms, CUDA events on the ensemble's compute stream) of the most recent
 * launch of each kernel family: 0 = transform (pack, last item), 1 = fused overlap,
 * 2 = Gram (all launches of the call), 3 = a whole fs_ensemble_recompute call.
 * Blocks until that launch has finished.                                            */
#define FS_KERNEL_PACK 0
#define FS_KERNEL_OVERLAP 1
#define FS_KERNEL_GRAM 2
#define FS_KERNEL_RECOMPUTE 3
int fs_ensemble_kernel_ms(fs_ensemble *ens, int kind, float *ms);
/* The ensemble's compute stream (cudaStream_t) so callers can order collectives and
 * timing events after its work when device_outputs is used.                      */
int fs_ensemble_stream_handle(fs_ensemble *ens, void **stream);
/* Run the ensemble's compute work on a caller-owned stream (e.g. the framework's
 * current stream); NULL restores the ensemble's own stream.  The caller keeps
 * ownership and must keep the stream alive while the ensemble uses it.           */
int fs_ensemble_set_stream(fs_ensemble *ens, void *stream);
/* Blocks until all work queued on the ensemble's streams has finished. */
int fs_ensemble_sync(fs_ensemble *ens);
/* Choose the Gram engine used by FS_GRAM_AUTO (process-wide; default FS_GRAM_TC_F4). */
int fs_set_gram_engine(int engine);
/* Choose the transform kernel: 0 = TMA bulk-staged, 1 = direct vector loads,
 * 2 = 8 coalesced 16-B loads in flight per thread (4 KB per warp, persistent grid),
 * 3 = 2 + next block's loads in flight and an in-kernel tail, 4 (default) = one 4 KB
 * block per warp over a raster-sized grid, 16-B packed stores, in-kernel tail. */
int fs_set_pack_engine(int engine);

/* ---- native interactive-recompute loop (service.py:110-175 without the interpreter) ----
 * A pipeline owns `depth` frame buffers (device outputs, pinned host slots, events) and
 * `depth` host worker threads.  fs_pipeline_run queues n_frames full recomputes of
 * slots[0..k) back to back — fused recompute, Jaccard + outlier kernels, D2H of the
 * [bins | Gram], Jaccard matrix and scores — while the workers run each finished frame's
 * complete-linkage merge (tau, id_rank as in fs_cluster_complete_linkage).  The last
 * frame's products go to the (optional) host outputs; *device_ms = device time of the
 * whole run (CUDA events on the ensemble's compute stream).  One device per pipeline;
 * with an fs_comm attached (below) each rank runs its own band's pipeline and the
 * partials are summed inside the loop.                                                 */
typedef struct fs_pipeline fs_pipeline;
int fs_pipeline_create(fs_ensemble *ens, const uint32_t *slots, uint32_t k, int engine, double tau,
                       const uint32_t *id_rank, uint32_t depth, fs_pipeline **out);
int fs_pipeline_run(fs_pipeline *p, uint32_t n_frames, int64_t *bins, int64_t *gram, double *sim,
                    double *scores, int32_t *labels, double *device_ms);
int fs_pipeline_destroy(fs_pipeline *p);

/* ---- multi-GPU exchange (north_star: "partial Gram matrices are summed with NCCL
 * allreduce"; replaces the reference's single-process analytics.py:174-181 loop when the
 * raster is split into row bands, one band per rank) -------------------------------------
 * An fs_comm is an NCCL communicator on the calling thread's device; libnccl is loaded at
 * run time (the copy torch already mapped, else libnccl.so.2).  Rank 0 creates the id,
 * the caller ships its 128 bytes to every rank (torch.distributed in dist.py), and every
 * rank calls fs_comm_create with it.  fs_pipeline_set_comm makes every frame of
 * fs_pipeline_run sum the [bins | Gram] partials of all ranks (int64, exact) on the
 * ensemble stream before the Jaccard / outlier kernels; NULL detaches.                 */
typedef struct fs_comm fs_comm;
int fs_comm_unique_id(uint8_t *out /* 128 bytes */);
int fs_comm_create(const uint8_t *id /* 128 bytes */, int nranks, int rank, fs_comm **out);
int fs_comm_allreduce_i64(fs_comm *c, int64_t *buf, uint64_t n, void *stream);
int fs_comm_destroy(fs_comm *c);
int fs_pipeline_set_comm(fs_pipeline *p, fs_comm *c);

/* ---- pinned host memory (for zero-staging uploads and fast read-back) ---- */
int fs_host_alloc(uint64_t bytes, void **out);
int fs_host_free(void *p);
/* 1 if p lies in page-locked (pinned or registered) host memory, else 0. */
int fs_host_is_pinned(const void *p, int *out);

/* ---- host-side analytics (exact, deterministic) --------------------------- */
/* Complete-linkage agglomeration of analytics.py:184-226 on a (n,n) float64
 * similarity matrix.  id_rank[i] = rank of surface i's id in lexical order (equal
 * ids share a rank).  Out: label[i] = cluster index in the final cluster list order
 * (before the caller's sort by first id).                                          */
int fs_cluster_complete_linkage(const double *sim, uint32_t n, const uint32_t *id_rank,
                                double tau, int32_t *label);
/* score_i = 1 - (sum_{j != i, ascending} sim[i,j]) / (n-1), float64 left to right. */
int fs_outlier_scores(const double *sim, uint32_t n, double *scores);
/* sim[i,j] = inter/union (1.0 when union == 0), diag 1.0, from an int64 Gram.      */
int fs_similarity_from_gram(const int64_t *gram, uint32_t n, double *sim);

/* The same two products on the device, for the resident recompute: `gram` (n x n
 * int64), `sim` (n x n float64) and `scores` (n float64, may be NULL) are DEVICE
 * pointers; the kernels are queued on `stream` (a cudaStream_t; NULL = the calling
 * thread's stream) and the call returns without waiting.  Bit-identical to
 * fs_similarity_from_gram / fs_outlier_scores (IEEE division, one left-to-right sum
 * per row).                                                                        */
int fs_similarity_outliers_device(const int64_t *gram, uint32_t n, double *sim, double *scores,
                                  void *stream);

/* ---- measured timings: the reference's modelled costs, on the device -----------
 * fs_time_transform: mean / min µs (CUDA events, `reps` back-to-back launches) of the
 * binarize + bit-pack transform of one width x height raster already in HBM (iid
 * p = 0.5 depths) — replaces transform_time (device.py:384-390) in the sweep of
 * bench.py:312-339.  engine -1 = current default, 0 = TMA bulk, 1 = direct, 2 = vector.
 * fs_time_h2d: one host->device copy of `bytes` from pinned (or pageable) memory —
 * replaces transfer_time (device.py:376-382) in the transfer suite (bench.py:193-228). */
int fs_time_transform(uint32_t width, uint32_t height, int reps, int engine, double *us_mean,
                      double *us_min);
int fs_time_h2d(uint64_t bytes, int reps, int pinned, double *us_mean, double *us_min);

/* ---- synthetic input (bench / tests): identical bytes on host and device -------
 * Flood-like prototype+flip generator: mask index i belongs to prototype
 * i / members; a prototype is a 16x16 thresholded low-res field upsampled to
 * width x height; each member flips pixels with probability eps; wet pixels get
 * depth 1..255.  Counter-based (hash of seed, i, pixel), so any row band
 * [row0, row0 + rows) can be generated independently.                           */
int fs_synth_host(uint8_t *out, uint64_t seed, uint32_t width, uint32_t height, uint64_t row0,
                  uint64_t rows, uint64_t mask_index, uint32_t members, double eps,
                  int threads);
/* The same bytes generated on the device: `out` may be device memory (written in
 * place) or host memory, pinned or pageable (generated in device chunks and copied);
 * for producing large inputs (e.g. 64 x 32768^2) at copy speed.                      */
int fs_synth_gpu(uint8_t *out, uint64_t seed, uint32_t width, uint32_t height, uint64_t row0,
                 uint64_t rows, uint64_t mask_index, uint32_t members, double eps);

#ifdef __cplusplus
}
#endif
#endif /* FLOODSTREAM_H */
