// fs_internal.h — launchers shared between the kernel files and the C ABI layer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fs_common.cuh"

namespace fs {

constexpr uint32_t kHistSmemBins = 4096;   // overlap classes kept in shared memory
constexpr uint64_t kLutMaxEntries = 1u << 20;  // composite grey LUT (n_inputs + 1)

// ---- transform ---------------------------------------------------------------
// Binarize + bit-pack one raster of `pixels` bytes into `words_per_mask` words
// (zero padded).  engine 0 = TMA bulk-staged (default), 1 = direct vector loads.
cudaError_t launch_pack(const uint8_t *src, uint64_t pixels, uint32_t *dst, uint64_t wpm,
                        cudaStream_t s, int engine);
void set_pack_engine(int engine);
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
  uint64_t wpm;
  const uint32_t *slots;  // device slot list: [k1 | k2]
  uint32_t k1, k2;        // the first k1 slots count with weight w1, the next k2 with w2
  uint32_t w1, w2;
  uint64_t pixels;
  uint32_t *counts;           // may be null
  uint32_t *rgba;             // may be null
  unsigned long long *bins;   // may be null, nbins entries (zeroed by caller)
  uint64_t nbins;             // n_inputs + 1
  uint64_t n_inputs;
  const uint8_t *lut;         // grey LUT of nbins entries, or null (FP64 path)
};
cudaError_t launch_overlap(const OverlapArgs &a, cudaStream_t s);

cudaError_t launch_accumulate_packed(const uint32_t *packed_mask, uint64_t pixels,
                                     uint32_t *counts, cudaStream_t s);

cudaError_t launch_gram_popc(const uint32_t *packed, uint64_t wpm, const uint32_t *slots,
                             uint32_t k, unsigned long long *gram, cudaStream_t s);
// tcgen05 kind::i8 Gram; partial workspace sized by gram_tc_workspace_bytes().
size_t gram_tc_workspace_bytes(uint32_t k, uint64_t wpm, int num_sms);
cudaError_t launch_gram_tc(const uint32_t *packed, uint64_t wpm, const uint32_t *slots,
                           uint32_t k, unsigned long long *gram, void *workspace,
                           int num_sms, cudaStream_t s);
// gram (k x k, upper tiles filled) -> int64 symmetric
cudaError_t launch_gram_mirror(unsigned long long *gram, uint32_t k, uint32_t tile,
                               cudaStream_t s);

cudaError_t launch_synth_packed(uint32_t *dst, uint64_t wpm, const SynthParams &sp,
                                uint64_t mask, uint64_t row0, uint64_t pixels,
                                cudaStream_t s);

// Composite grey LUT in FP64, bit-exact with _kernels_np.py:41-42.
void build_grey_lut(uint64_t n_inputs, uint8_t *lut, uint64_t entries);
uint8_t grey_of(uint64_t c, uint64_t n_inputs);

}  // namespace fs
