// fs_internal.h — launchers shared between the kernel files and the C ABI layer.
#pragma once
#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched at run time)
#include <cuda_runtime.h>

#include "fs_common.cuh"

namespace fs {

constexpr uint32_t kHistSmemBins = 4096;       // overlap classes kept in shared memory
constexpr uint64_t kLutMaxEntries = 1u << 20;  // composite grey LUT (n_inputs + 1)

int num_sms();  // SM count of the calling thread's current device

// Dynamic shared-memory opt-in of one kernel (cudaFuncAttributeMaxDynamicSharedMemorySize).
// Function attributes belong to each device's context, so the granted size is tracked
// per device; concurrent callers serialise on the mutex only until their device is set.
constexpr int kMaxDevices = 64;
struct SmemOptIn {
  std::mutex mu;
  std::atomic<size_t> granted[kMaxDevices] = {};
};
template <typename Kernel>
inline cudaError_t smem_opt_in(SmemOptIn &o, Kernel *fn, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (o.granted[dev].load(std::memory_order_acquire) >= bytes) return cudaSuccess;
  std::lock_guard<std::mutex> lk(o.mu);
  if (o.granted[dev].load(std::memory_order_relaxed) >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) o.granted[dev].store(bytes, std::memory_order_release);
  return e;
}

// 3-D tensor map over the tile-interleaved packed layout, restricted to rows
// [row0, row0 + rows) of `capacity`: dims (32 words, rows, ntiles), box
// (box_words, box_rows, box_tiles), swizzle 0 / 64 / 128 (bytes).  Rows and tiles
// outside the map read as zero.
cudaError_t encode_packed_map(CUtensorMap *out, const uint32_t *packed, uint64_t capacity,
                              uint64_t row0, uint64_t rows, uint64_t ntiles, uint32_t box_words,
                              uint32_t box_rows, uint32_t box_tiles, int swizzle);

// Slot list -> first slot if it is a contiguous ascending run, else -1.
int64_t contiguous_run(const uint32_t *host_slots, uint32_t k);

// ---- transform ---------------------------------------------------------------
// Binarize + bit-pack one raster of `pixels` bytes into slot `slot` of the packed
// buffer (zero padded to wpm words).  engine 0 = TMA bulk-staged, 1 = direct loads.
cudaError_t launch_pack(const uint8_t *src, uint64_t pixels, uint32_t *packed, uint64_t slot,
                        uint64_t capacity, uint64_t wpm, cudaStream_t s, int engine);
void set_pack_engine(int engine);
// iid p = 0.5 depth bytes (transform sweep inputs)
cudaError_t launch_fill_random(uint8_t *dst, uint64_t n, uint64_t seed, cudaStream_t s);
int get_pack_engine();

// ---- reference primitive protocol kernels (flat device arrays) ----------------
cudaError_t launch_accumulate_u8(uint32_t *counts, const uint8_t *cells, uint64_t n,
                                 cudaStream_t s);
cudaError_t launch_histogram(const uint32_t *counts, uint64_t n, uint64_t nbins,
                             unsigned long long *bins, cudaStream_t s);
cudaError_t launch_composite(const uint32_t *counts, uint64_t n, uint64_t n_inputs,
                             const uint8_t *lut, uint32_t *rgba, cudaStream_t s);
cudaError_t launch_pair_counts(const uint8_t *a, const uint8_t *b, uint64_t n,
                               unsigned long long *out2, cudaStream_t s);

// ---- packed-ensemble kernels -------------------------------------------------
struct OverlapArgs {
  const uint32_t *packed;
  uint64_t capacity;
  uint64_t wpm;
  const uint32_t *slots;      // device slot list [k1 | k2] (gather mode)
  const uint32_t *host_slots; // same list on the host (mode selection)
  uint32_t k1, k2;            // first k1 slots count with weight w1, next k2 with w2
  uint32_t w1, w2;
  uint64_t pixels;
  uint32_t *counts;           // may be null
  uint32_t *rgba;             // may be null
  unsigned long long *bins;   // may be null, nbins entries (zeroed by caller)
  uint64_t nbins;             // n_inputs + 1
  uint64_t n_inputs;
  const uint8_t *lut;         // grey LUT of nbins entries, or null (FP64 path)
  int vec;                    // set by launch_overlap: outputs 16-B aligned
  // Multi-panel fused recompute: the diagonal Gram CTAs of panel I write the counts of
  // their <= 256 masks as uint16 to partial16 + I * part_pitch (instead of counts /
  // RGBA / bins); launch_combine_partials then sums the panels into the outputs.
  uint16_t *partial16 = nullptr;
  uint64_t part_pitch = 0;    // pixels per panel slab (multiple of 1024)
};
cudaError_t launch_overlap(const OverlapArgs &a, cudaStream_t s);
// counts / RGBA / bins of `a` from npanels uint16 partial-count slabs
cudaError_t launch_combine_partials(const uint16_t *partial16, uint32_t npanels, uint64_t pitch,
                                    const OverlapArgs &a, cudaStream_t s);

cudaError_t launch_accumulate_packed(const uint32_t *packed, uint64_t slot, uint64_t capacity,
                                     uint64_t pixels, uint32_t *counts, cudaStream_t s);

cudaError_t launch_gram_popc(const uint32_t *packed, uint64_t capacity, uint64_t wpm,
                             const uint32_t *slots, uint32_t k, unsigned long long *gram,
                             cudaStream_t s);
// tcgen05 kind::i8 Gram; partial workspace sized by gram_tc_workspace_bytes().
// fp4: diagonal tiles on kind::mxf4 (off-diagonal tiles stay on kind::i8).
size_t gram_tc_workspace_bytes(uint32_t k, uint64_t wpm, int num_sms, bool fp4,
                               bool fuse = false);
// Non-contiguous slot lists are first gathered into gather_ws (gram_tc_gather_bytes).
size_t gram_tc_gather_bytes(uint32_t k, uint64_t wpm);
cudaError_t launch_gram_tc(const uint32_t *packed, uint64_t capacity, uint64_t wpm,
                           const uint32_t *slots, const uint32_t *host_slots, uint32_t k,
                           unsigned long long *gram, void *workspace, void *gather_ws,
                           int num_sms, bool fp4, const OverlapArgs *fuse, bool *fused,
                           cudaStream_t s);
// The fused recompute of one 129..256-mask FP4 panel (fs_recompute_f4.cu): Gram partial
// tiles (one 256 x 256 int32 tile per CTA chunk of upc units) + the overlap products of
// `ov` (counts / histogram / RGBA, bins zeroed by the caller) from one read of the masks.
// npanels > 1: the diagonal 256-mask tiles of a larger ensemble, panel-major CTAs
// (blockIdx = panel * kchunks + chunk); with ov.partial16 set each panel's counts go to
// its uint16 slab (ov.part_pitch apart) for launch_combine_partials.
// slots != nullptr (device list, npanels == 1): mask m is read from slot slots[m] of the
// ensemble directly, with no gather pass.  rows = 128: a single panel of k <= 128 masks
// (one MMA of N = roundup(k, 16) per K step, 128 x 128 partial tiles for k_gram_reduce<128>).
cudaError_t launch_recompute_f4(const uint32_t *src, uint64_t cap, uint64_t row0, uint32_t k,
                                uint64_t total_units, uint32_t kchunks, uint64_t upc,
                                int32_t *partial, const OverlapArgs &ov, cudaStream_t s,
                                uint32_t npanels = 1, const uint32_t *slots = nullptr,
                                uint32_t rows = 256);
// fuse != nullptr: when all k masks fit one panel (k <= 256) the diagonal CTAs also
// run the overlap pass (counts / histogram / RGBA of `*fuse`, weights 1) and *fused is
// set; bins must be zeroed by the caller.  Otherwise nothing of *fuse is written.
// gram (k x k, upper tiles filled) -> symmetric
cudaError_t launch_gram_mirror(unsigned long long *gram, uint32_t k, uint32_t tile,
                               cudaStream_t s);

cudaError_t launch_synth_packed(uint32_t *packed, uint64_t slot, uint64_t capacity, uint64_t wpm,
                                const SynthParams &sp, uint64_t mask, uint64_t row0,
                                uint64_t pixels, cudaStream_t s);

cudaError_t launch_synth_raw(uint8_t *dst, const SynthParams &sp, uint64_t mask, uint64_t row0,
                             uint64_t pixels, cudaStream_t s);

cudaError_t launch_similarity_outliers(const long long *gram, uint32_t n, double *sim,
                                       double *scores, cudaStream_t s);

// thread-local C-ABI error message + status (fs_capi.cu)
int set_error(int code, const std::string &msg);

// Composite grey LUT in FP64, bit-exact with _kernels_np.py:41-42.
void build_grey_lut(uint64_t n_inputs, uint8_t *lut, uint64_t entries);
uint8_t grey_of(uint64_t c, uint64_t n_inputs);

}  // namespace fs
