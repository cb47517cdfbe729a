// fs_kernels.cu — per-pixel kernels of the flood-ensemble overlap path (sm_100a).
//
// Reference semantics (all under /root/reference/pkg/src/floodstream/):
//   accumulate_into   _kernels_np.py:16-18   counts[p] += cells[p] > 0
//   overlap_counts    _kernels_np.py:21-23   bins[k] = #{p : counts[p] == k}
//   pair_counts       _kernels_np.py:26-32   (|A & B|, |A | B|) of wet masks
//   composite_fill    _kernels_np.py:35-47   RGBA (g, g, 255, 255), g = floor(255(1-c/n)+0.5)
//   accumulate        analytics.py:106-126   the per-surface loop, fused here
//   transform         device.py:384-390      modelled buffer->image reorganisation; here a
//                                            real binarize + bit-pack kernel
// Every kernel is a streaming HBM pass: 128-bit loads, coalesced stores, persistent
// grids sized to the SM count, shared-memory privatised histograms.
#include <algorithm>
#include <cstdio>
#include <cmath>

#include <cudaTypedefs.h>

#include "fs_bitslice.cuh"

namespace fs {

static std::atomic<int> g_num_sms[kMaxDevices] = {};
int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int n = g_num_sms[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    g_num_sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// ---------------------------------------------------------------------------
// bit helpers
// ---------------------------------------------------------------------------
// 4 bytes -> 4 bits (bit i set iff byte i != 0)
__device__ __forceinline__ uint32_t nz_nibble(uint32_t x) {
  uint32_t t = x | (x >> 4);
  t |= t >> 2;
  t |= t >> 1;
  t &= 0x01010101u;
  return (t * 0x00204081u) >> 21 & 0xFu;
}
__device__ __forceinline__ uint32_t nz_bits16(uint4 v) {
  return nz_nibble(v.x) | (nz_nibble(v.y) << 4) | (nz_nibble(v.z) << 8) |
         (nz_nibble(v.w) << 12);
}

// ---------------------------------------------------------------------------
// Transform: binarize + bit-pack, TMA bulk staged (cp.async.bulk -> SMEM ring)
// ---------------------------------------------------------------------------
constexpr int kPackThreads = 256;
constexpr int kPackChunk = 8192;  // bytes (= pixels) per stage, 256 output words
constexpr int kPackStages = 4;
static int g_pack_engine = 4;  // k_pack_flat: measured fastest (profiles/round2)
void set_pack_engine(int e) { g_pack_engine = e; }
int get_pack_engine() { return g_pack_engine; }

__global__ void __launch_bounds__(kPackThreads)
    k_pack_bulk(const uint8_t *__restrict__ src, uint64_t nchunks, uint32_t *__restrict__ dst,
                uint64_t slot, uint64_t cap) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + kPackStages * kPackChunk);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kPackStages; ++s) ptx::mbar_init(&bar[s], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint64_t nmy =
      nchunks > blockIdx.x ? (nchunks - blockIdx.x - 1) / gridDim.x + 1 : 0;
  if (tid == 0) {
    for (uint64_t j = 0; j < nmy && j < (uint64_t)kPackStages; ++j) {
      uint64_t c = blockIdx.x + j * gridDim.x;
      ptx::mbar_arrive_expect_tx(&bar[j], kPackChunk);
      ptx::bulk_g2s(sm + j * kPackChunk, src + c * kPackChunk, kPackChunk, &bar[j]);
    }
  }
  for (uint64_t j = 0; j < nmy; ++j) {
    const int s = (int)(j % kPackStages);
    const uint32_t parity = (uint32_t)((j / kPackStages) & 1);
    const uint64_t c = blockIdx.x + j * gridDim.x;
    ptx::mbar_wait(&bar[s], parity);
    const uint4 *stage = reinterpret_cast<const uint4 *>(sm + s * kPackChunk);
#pragma unroll
    for (int i = 0; i < kPackChunk / 16 / kPackThreads; ++i) {
      const int q = tid + i * kPackThreads;
      uint32_t h = nz_bits16(stage[q]);
      uint32_t other = __shfl_xor_sync(0xffffffffu, h, 1);
      if ((lane & 1) == 0) dst[pk_off(slot, c * (kPackChunk / 32) + (q >> 1), cap)] = h | (other << 16);
    }
    __syncthreads();
    if (tid == 0 && j + kPackStages < nmy) {
      uint64_t cn = blockIdx.x + (j + kPackStages) * gridDim.x;
      ptx::mbar_arrive_expect_tx(&bar[s], kPackChunk);
      ptx::bulk_g2s(sm + s * kPackChunk, src + cn * kPackChunk, kPackChunk, &bar[s]);
    }
  }
}

// Direct-load variant (no staging): each thread turns 32 bytes into one word.
__global__ void __launch_bounds__(256)
    k_pack_direct(const uint8_t *__restrict__ src, uint64_t nvec, uint32_t *__restrict__ dst,
                  uint64_t slot, uint64_t cap) {
  // nvec = number of full 16-byte vectors; pairs of lanes build one word
  const int lane = threadIdx.x & 31;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       q < ((nvec + 31) / 32) * 32; q += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t h = 0;
    if (q < nvec) h = nz_bits16(ptx::ld_nc_v4(src + q * 16));
    uint32_t other = __shfl_xor_sync(0xffffffffu, h, 1);
    if ((lane & 1) == 0 && q < nvec) dst[pk_off(slot, q >> 1, cap)] = h | (other << 16);
  }
}

// Vector variant: a warp turns one 4 KB block into 128 words; every thread keeps 8
// coalesced 16-B loads in flight (lane t, load i: bytes 512 i + 16 t), lane pairs merge
// their 16-px nibble sets into one 32-px word.
constexpr int kPackVec = 8;
constexpr int kPackBlk = kPackVec * 512;  // bytes (pixels) per warp-block
__global__ void __launch_bounds__(256)
    k_pack_vec(const uint8_t *__restrict__ src, uint64_t nblk, uint32_t *__restrict__ dst,
               uint64_t slot, uint64_t cap) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; b < nblk; b += nw) {
    const uint8_t *base = src + b * kPackBlk + lane * 16;
    uint4 v[kPackVec];
#pragma unroll
    for (int i = 0; i < kPackVec; ++i) v[i] = ptx::ld_nc_v4(base + i * 512);
#pragma unroll
    for (int i = 0; i < kPackVec; ++i) {
      const uint32_t h = nz_bits16(v[i]);
      const uint32_t other = __shfl_xor_sync(0xffffffffu, h, 1);
      if ((lane & 1) == 0)
        dst[pk_off(slot, b * (kPackBlk / 32) + i * 16 + (lane >> 1), cap)] = h | (other << 16);
    }
  }
}

// Pipelined vector variant: like k_pack_vec, but every warp keeps the NEXT 4 KB block's
// eight 16-B loads in flight while it packs the current one, and the same launch packs
// the partial last block and writes the zero padding up to wpm (no separate tail
// launch: a second dependent launch costs several microseconds at any raster size).
__device__ __forceinline__ void pack_block(const uint4 (&v)[kPackVec], uint64_t b, int lane,
                                           uint32_t *__restrict__ dst, uint64_t slot,
                                           uint64_t cap) {
#pragma unroll
  for (int i = 0; i < kPackVec; ++i) {
    const uint32_t h = nz_bits16(v[i]);
    const uint32_t other = __shfl_xor_sync(0xffffffffu, h, 1);
    if ((lane & 1) == 0)
      dst[pk_off(slot, b * (kPackBlk / 32) + i * 16 + (lane >> 1), cap)] = h | (other << 16);
  }
}

__global__ void __launch_bounds__(256)
    k_pack_pipe(const uint8_t *__restrict__ src, uint64_t pixels, uint64_t wpm,
                uint32_t *__restrict__ dst, uint64_t slot, uint64_t cap) {
  const int lane = threadIdx.x & 31;
  const uint64_t nblk = pixels / kPackBlk;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint4 cur[kPackVec], nxt[kPackVec];
  auto load = [&](uint4 (&v)[kPackVec], uint64_t blk) {
    const uint8_t *base = src + blk * kPackBlk + lane * 16;
#pragma unroll
    for (int i = 0; i < kPackVec; ++i) v[i] = ptx::ld_nc_v4(base + i * 512);
  };
  if (b < nblk) load(cur, b);
  while (b < nblk) {
    const uint64_t bn = b + nw;
    if (bn < nblk) load(nxt, bn);
    pack_block(cur, b, lane, dst, slot, cap);
    if (bn >= nblk) break;
    b = bn;
#pragma unroll
    for (int i = 0; i < kPackVec; ++i) cur[i] = nxt[i];
  }
  // partial last block + zero padding: words [nblk * 128, wpm), one word per thread
  const uint64_t w0 = nblk * (kPackBlk / 32);
  for (uint64_t w = w0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < wpm;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
    const uint64_t p0 = w * 32;
    for (int q = 0; q < 32 && p0 + q < pixels; ++q) word |= (uint32_t)(src[p0 + q] != 0) << q;
    dst[pk_off(slot, w, cap)] = word;
  }
}

// Flat variant (the default): one 4 KB block per warp, no loop — the grid is the raster
// (ceil(blocks / 8) CTAs), so the whole read is in flight as soon as the CTAs land, which
// measured best against a cold L2 (profiles/round2/pack_probe.json: "flat").  The warp's
// 128 packed words go through 512 B of shared memory so each lane writes one 16-B vector
// (4 x 128-B tile rows per warp instead of 64-B half-rows); trailing CTAs pack the partial
// last block and the zero padding up to wpm in the same launch.
__global__ void __launch_bounds__(256)
    k_pack_flat(const uint8_t *__restrict__ src, uint64_t pixels, uint64_t wpm,
                uint32_t *__restrict__ dst, uint64_t slot, uint64_t cap) {
  __shared__ __align__(16) uint32_t stage[8][kPackBlk / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t nblk = pixels / kPackBlk;
  const uint64_t body_ctas = (nblk + 7) / 8;
  if (blockIdx.x < body_ctas) {
    const uint64_t b = (uint64_t)blockIdx.x * 8 + wib;
    if (b >= nblk) return;
    const uint8_t *base = src + b * kPackBlk + lane * 16;
    uint4 v[kPackVec];
#pragma unroll
    for (int i = 0; i < kPackVec; ++i) v[i] = ptx::ld_nc_v4(base + i * 512);
#pragma unroll
    for (int i = 0; i < kPackVec; ++i) {
      const uint32_t h = nz_bits16(v[i]);
      const uint32_t other = __shfl_xor_sync(0xffffffffu, h, 1);
      if ((lane & 1) == 0) stage[wib][i * 16 + (lane >> 1)] = h | (other << 16);
    }
    __syncwarp();
    const uint4 q = *reinterpret_cast<const uint4 *>(&stage[wib][4 * lane]);
    // words 4 lane .. 4 lane + 3 of the block: one tile row (pk_off is contiguous within a
    // 32-word tile and 4 lane never crosses one)
    *reinterpret_cast<uint4 *>(dst + pk_off(slot, b * (kPackBlk / 32) + 4 * lane, cap)) = q;
    return;
  }
  // partial last block + zero padding: words [nblk * 128, wpm), one word per thread
  const uint64_t w = nblk * (kPackBlk / 32) + (blockIdx.x - body_ctas) * 256ull + threadIdx.x;
  if (w >= wpm) return;
  uint32_t word = 0;
  const uint64_t p0 = w * 32;
  for (int q = 0; q < 32 && p0 + q < pixels; ++q) word |= (uint32_t)(src[p0 + q] != 0) << q;
  dst[pk_off(slot, w, cap)] = word;
}

// Words [w0, wpm): scalar tail + zero padding.
__global__ void k_pack_tail(const uint8_t *__restrict__ src, uint64_t pixels, uint64_t w0,
                            uint64_t wpm, uint32_t *__restrict__ dst, uint64_t slot,
                            uint64_t cap) {
  uint64_t w = w0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (w >= wpm) return;
  uint32_t word = 0;
  uint64_t p0 = w * 32;
  if (p0 < pixels) {
    for (int b = 0; b < 32; ++b) {
      uint64_t p = p0 + b;
      if (p < pixels && src[p] != 0) word |= 1u << b;
    }
  }
  dst[pk_off(slot, w, cap)] = word;
}

cudaError_t launch_pack(const uint8_t *src, uint64_t pixels, uint32_t *dst, uint64_t slot,
                        uint64_t cap, uint64_t wpm, cudaStream_t s, int engine) {
  if (engine < 0) engine = g_pack_engine;
  uint64_t done_words = 0;
  if (engine == 0) {
    const uint64_t nchunks = pixels / kPackChunk;
    if (nchunks > 0) {
      static SmemOptIn attr;
      const int smem = kPackStages * kPackChunk + kPackStages * 8;
      if (cudaError_t e = smem_opt_in(attr, k_pack_bulk, (size_t)smem); e != cudaSuccess)
        return e;
      uint64_t grid = (uint64_t)num_sms() * 6;
      if (grid > nchunks) grid = nchunks;
      k_pack_bulk<<<(unsigned)grid, kPackThreads, smem, s>>>(src, nchunks, dst, slot, cap);
      done_words = nchunks * (kPackChunk / 32);
    }
  } else if (engine == 4) {
    const uint64_t nblk = pixels / kPackBlk;
    const uint64_t tail = wpm - nblk * (kPackBlk / 32);
    const uint64_t grid = (nblk + 7) / 8 + (tail + 255) / 256;
    if (grid > 0) k_pack_flat<<<(unsigned)grid, 256, 0, s>>>(src, pixels, wpm, dst, slot, cap);
    return cudaGetLastError();
  } else if (engine == 3) {
    const uint64_t nblk = pixels / kPackBlk;
    uint64_t grid = (std::max<uint64_t>(nblk, 1) * 32 + 255) / 256;
    const uint64_t gcap = (uint64_t)num_sms() * 4;
    if (grid > gcap) grid = gcap;
    k_pack_pipe<<<(unsigned)grid, 256, 0, s>>>(src, pixels, wpm, dst, slot, cap);
    return cudaGetLastError();
  } else if (engine == 2) {
    const uint64_t nblk = pixels / kPackBlk;
    if (nblk > 0) {
      uint64_t grid = (nblk * 32 + 255) / 256;
      const uint64_t gcap = (uint64_t)num_sms() * 8;
      if (grid > gcap) grid = gcap;
      k_pack_vec<<<(unsigned)grid, 256, 0, s>>>(src, nblk, dst, slot, cap);
      done_words = nblk * (kPackBlk / 32);
    }
  } else {
    // full 32-byte groups only; the rest goes to the tail kernel
    const uint64_t nvec = (pixels / 32) * 2;
    if (nvec > 0) {
      uint64_t threads = (nvec + 31) / 32 * 32;
      uint64_t grid = (threads + 255) / 256;
      const uint64_t gcap = (uint64_t)num_sms() * 16;
      if (grid > gcap) grid = gcap;
      k_pack_direct<<<(unsigned)grid, 256, 0, s>>>(src, nvec, dst, slot, cap);
      done_words = nvec / 2;
    }
  }
  if (done_words < wpm) {
    uint64_t n = wpm - done_words;
    k_pack_tail<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, pixels, done_words, wpm, dst,
                                                            slot, cap);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Protocol kernels over flat arrays
// ---------------------------------------------------------------------------
__global__ void k_accumulate_u8(uint32_t *__restrict__ counts, const uint8_t *__restrict__ cells,
                                uint64_t n) {
  const uint64_t nvec = n / 16;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nvec; q += stride) {
    uint32_t bits = nz_bits16(ptx::ld_nc_v4(cells + q * 16));
    uint4 *c4 = reinterpret_cast<uint4 *>(counts + q * 16);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      uint4 c = c4[v];
      c.x += (bits >> (4 * v + 0)) & 1u;
      c.y += (bits >> (4 * v + 1)) & 1u;
      c.z += (bits >> (4 * v + 2)) & 1u;
      c.w += (bits >> (4 * v + 3)) & 1u;
      c4[v] = c;
    }
  }
  for (uint64_t p = nvec * 16 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += stride)
    counts[p] += cells[p] != 0;
}

cudaError_t launch_accumulate_u8(uint32_t *counts, const uint8_t *cells, uint64_t n,
                                 cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n / 16 + 255) / 256 + 1;
  uint64_t cap = (uint64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  k_accumulate_u8<<<(unsigned)grid, 256, 0, s>>>(counts, cells, n);
  return cudaGetLastError();
}

// Warp-aggregated histogram increment: lanes holding the same class add once.
__device__ __forceinline__ void hist_add(uint32_t c, bool valid, uint32_t *sh,
                                         unsigned long long *gl) {
  const uint32_t key = valid ? c : 0xFFFFFFFFu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int lane = threadIdx.x & 31;
  if (valid && (__ffs(peers) - 1) == lane) {
    if (sh)
      atomicAdd(sh + c, (uint32_t)__popc(peers));
    else
      atomicAdd(gl + c, (unsigned long long)__popc(peers));
  }
}

__global__ void __launch_bounds__(256)
    k_histogram(const uint32_t *__restrict__ counts, uint64_t n, uint64_t nbins,
                unsigned long long *__restrict__ bins) {
  __shared__ uint32_t sh[kHistSmemBins];
  const bool use_sh = nbins <= kHistSmemBins;
  if (use_sh)
    for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nvec = (n + 3) / 4;
  const uint64_t iters = (nvec + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    uint64_t q = it * stride + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint64_t p = q * 4 + e;
      bool valid = p < n;
      uint32_t c = valid ? __ldg(counts + p) : 0;
      // counts above n_inputs would index past bins; the reference's numpy backend
      // grows the array, the Cython one writes out of bounds.  Callers validate.
      valid = valid && c < nbins;
      hist_add(c, valid, use_sh ? sh : nullptr, bins);
    }
  }
  __syncthreads();
  if (use_sh)
    for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x)
      if (sh[i]) atomicAdd(bins + i, (unsigned long long)sh[i]);
}

cudaError_t launch_histogram(const uint32_t *counts, uint64_t n, uint64_t nbins,
                             unsigned long long *bins, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n / 4 + 255) / 256 + 1;
  uint64_t cap = (uint64_t)num_sms() * 4;
  if (grid > cap) grid = cap;
  k_histogram<<<(unsigned)grid, 256, 0, s>>>(counts, n, nbins, bins);
  return cudaGetLastError();
}

__global__ void k_composite(const uint32_t *__restrict__ counts, uint64_t n, uint64_t n_inputs,
                            const uint8_t *__restrict__ lut, uint32_t *__restrict__ rgba) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += stride) {
    uint32_t c = counts[p];
    const uint8_t *l = (lut != nullptr && c <= n_inputs) ? lut : nullptr;
    rgba[p] = rgba_word(c, n_inputs, l);
  }
}

cudaError_t launch_composite(const uint32_t *counts, uint64_t n, uint64_t n_inputs,
                             const uint8_t *lut, uint32_t *rgba, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n + 255) / 256;
  uint64_t cap = (uint64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  k_composite<<<(unsigned)grid, 256, 0, s>>>(counts, n, n_inputs, lut, rgba);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256)
    k_pair_counts(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, uint64_t n,
                  unsigned long long *__restrict__ out) {
  uint64_t inter = 0, uni = 0;
  const uint64_t nvec = n / 16;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nvec; q += stride) {
    uint32_t wa = nz_bits16(ptx::ld_nc_v4(a + q * 16));
    uint32_t wb = nz_bits16(ptx::ld_nc_v4(b + q * 16));
    inter += __popc(wa & wb);
    uni += __popc(wa | wb);
  }
  for (uint64_t p = nvec * 16 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += stride) {
    bool x = a[p] != 0, y = b[p] != 0;
    inter += x && y;
    uni += x || y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    inter += __shfl_xor_sync(0xffffffffu, inter, o);
    uni += __shfl_xor_sync(0xffffffffu, uni, o);
  }
  __shared__ unsigned long long si[8], su[8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    si[w] = inter;
    su[w] = uni;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ti = 0, tu = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      ti += si[i];
      tu += su[i];
    }
    atomicAdd(out, ti);
    atomicAdd(out + 1, tu);
  }
}

cudaError_t launch_pair_counts(const uint8_t *a, const uint8_t *b, uint64_t n,
                               unsigned long long *out2, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n / 16 + 255) / 256 + 1;
  uint64_t cap = (uint64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  k_pair_counts<<<(unsigned)grid, 256, 0, s>>>(a, b, n, out2);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fused overlap pass over the tile-interleaved packed masks.
//
// A block owns 4 consecutive pixel tiles (4 warps, warp = tile, lane = word: 32 px).
// Lane 0 of warp 0 streams [4 tiles][16 masks][32 words] boxes (8 KB, contiguous in
// HBM) through a 4-stage TMA ring (full/empty mbarriers, so warps drift up to a ring
// apart instead of meeting at a block barrier per box).  Each thread folds its word of
// 16 masks into bit-sliced Harley-Seal counters (ones/twos/fours/eights + NH ripple
// planes): one 32-bit op advances 32 pixels.  After the tile's last mask the per-pixel
// counts are extracted into registers and
//   * the histogram is run-length encoded over the thread's 32 consecutive pixels
//     (flood masks are spatially coherent: ~1-3 shared-memory atomics per word),
//   * the counts are transposed through a padded SMEM tile with 16-B accesses
//     (conflict-free) and written as 16-B streaming stores of counts and RGBA
//     (RGBA from a per-block SMEM table of the exact FP64 grey levels).
// Padding pixels past `pixels` (count 0) are counted once and removed from bin 0.
// ---------------------------------------------------------------------------
constexpr int kOvTiles = 4;
constexpr int kOvThreads = 32 * kOvTiles;
constexpr int kOvGroup = 16;
constexpr int kOvStages = 4;
constexpr int kOvStageWords = kOvTiles * kOvGroup * 32;  // 8 KB

static size_t ov_smem_bytes(uint32_t sbins) {
  return (size_t)kOvStages * kOvStageWords * 4 + (size_t)kOvTiles * 32 * kTileTb * 4 +
         2 * kOvStages * 8 + 2 * (size_t)sbins * 4;
}

template <bool GATHER, int NH>
__global__ void __launch_bounds__(kOvThreads)
    k_overlap(const __grid_constant__ CUtensorMap tm, const OverlapArgs a, uint32_t sbins) {
  constexpr uint32_t kPass = (1u << NH) - 1;  // 16-mask groups per extraction
  extern __shared__ __align__(128) uint8_t sm[];
  uint32_t *stage = reinterpret_cast<uint32_t *>(sm);
  uint32_t *tb = stage + kOvStages * kOvStageWords;
  uint64_t *full = reinterpret_cast<uint64_t *>(tb + kOvTiles * 32 * kTileTb);
  uint64_t *empty = full + kOvStages;
  uint32_t *sh_hist = reinterpret_cast<uint32_t *>(empty + kOvStages);
  uint32_t *sh_lut = sh_hist + sbins;
  const int tid = threadIdx.x;
  const int wi = tid >> 5, lane = tid & 31;
  const bool do_hist = a.bins != nullptr;
  const bool hist_sh = do_hist && a.nbins <= sbins;
  const bool lut_sh = a.rgba != nullptr && a.nbins <= sbins;
  if (hist_sh)
    for (uint32_t i = tid; i < a.nbins; i += kOvThreads) sh_hist[i] = 0;
  if (lut_sh)
    for (uint32_t i = tid; i < a.nbins; i += kOvThreads) sh_lut[i] = rgba_word(i, a.n_inputs, a.lut);
  if (tid == 0) {
    ptx::prefetch_tmap(&tm);
    for (int s = 0; s < kOvStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kOvTiles);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  const uint64_t ntiles = a.wpm / 32;
  const uint64_t ntg = (ntiles + kOvTiles - 1) / kOvTiles;
  const uint32_t G1 = a.w1 ? (a.k1 + kOvGroup - 1) / kOvGroup : 0;
  const uint32_t G2 = a.w2 ? (a.k2 + kOvGroup - 1) / kOvGroup : 0;
  const uint32_t GP = G1 + G2;
  const uint64_t nq = ntg > blockIdx.x ? (ntg - blockIdx.x - 1) / gridDim.x + 1 : 0;
  const uint64_t nitems = nq * GP;

  // group g -> first row (slot-list offset) and row count
  auto group = [&](uint32_t g, uint32_t &off, uint32_t &cnt) {
    if (g < G1) {
      off = g * kOvGroup;
      cnt = min((uint32_t)kOvGroup, a.k1 - off);
    } else {
      const uint32_t gi = g - G1;
      off = a.k1 + gi * kOvGroup;
      cnt = min((uint32_t)kOvGroup, a.k2 - gi * kOvGroup);
    }
  };
  // producer cursor (thread 0 only)
  uint64_t pq = 0;
  uint32_t pg = 0;
  auto issue_next = [&](int s) {
    uint32_t off, cnt;
    group(pg, off, cnt);
    const int tile0 = (int)((blockIdx.x + pq * gridDim.x) * kOvTiles);
    uint32_t *dst = stage + s * kOvStageWords;
    if (!GATHER) {
      ptx::mbar_arrive_expect_tx(&full[s], kOvStageWords * 4);
      ptx::tma_load_3d(dst, &tm, 0, (int)off, tile0, &full[s]);
    } else {
      ptx::mbar_arrive_expect_tx(&full[s], cnt * kOvTiles * 32 * 4);
      for (uint32_t j = 0; j < cnt; ++j)
        ptx::tma_load_3d(dst + j * kOvTiles * 32, &tm, 0, (int)__ldg(a.slots + off + j), tile0,
                         &full[s]);
    }
    if (++pg == GP) {
      pg = 0;
      ++pq;
    }
  };
  if (tid == 0)
    for (int s = 0; s < kOvStages && (uint64_t)s < nitems; ++s) issue_next(s);

  HSCounter<NH> hc;
  hc.reset();
  uint32_t cnt32[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) cnt32[j] = 0;
  uint32_t groups_in_pass = 0;
  uint64_t q = 0;
  uint32_t g = 0;
  int s = 0;
  uint32_t phase = 0;

  for (uint64_t i = 0; i < nitems; ++i) {
    uint32_t off, cnt;
    group(g, off, cnt);
    ptx::mbar_wait(&full[s], phase);
    const uint32_t *st = stage + s * kOvStageWords;
    uint32_t d[16];
    if (cnt == (uint32_t)kOvGroup) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        d[j] = GATHER ? st[(j * kOvTiles + wi) * 32 + lane] : st[(wi * kOvGroup + j) * 32 + lane];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t v =
            GATHER ? st[(j * kOvTiles + wi) * 32 + lane] : st[(wi * kOvGroup + j) * 32 + lane];
        d[j] = (j < (int)cnt) ? v : 0u;
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (tid == 0 && i + kOvStages < nitems) {
      ptx::mbar_wait(&empty[s], phase);
      issue_next(s);
    }
    hc.add16(d);
    ++groups_in_pass;
    const bool range_end = (g == G1 - 1 && G1 > 0) || g == GP - 1;
    if (range_end || groups_in_pass == kPass) {
      hc.extract(cnt32, g < G1 ? a.w1 : a.w2);
      hc.reset();
      groups_in_pass = 0;
    }
    if (g == GP - 1) {
      const uint64_t tile = (blockIdx.x + q * gridDim.x) * kOvTiles + wi;
      if (tile < ntiles)
        emit_tile(cnt32, tile, lane, tb + wi * 32 * kTileTb, a, sh_hist, hist_sh, sh_lut, lut_sh);
#pragma unroll
      for (int j = 0; j < 32; ++j) cnt32[j] = 0;
    }
    if (++s == kOvStages) {
      s = 0;
      phase ^= 1u;
    }
    if (++g == GP) {
      g = 0;
      ++q;
    }
  }
  __syncthreads();
  if (hist_sh)
    for (uint32_t i = tid; i < a.nbins; i += kOvThreads)
      if (sh_hist[i]) atomicAdd(a.bins + i, (unsigned long long)sh_hist[i]);
  if (do_hist && blockIdx.x == 0 && tid == 0) {
    // padding pixels of the last tile were counted in bin 0
    const uint64_t pad = ntiles * 1024 - a.pixels;
    if (pad) atomicAdd(a.bins, (unsigned long long)(0ull - pad));
  }
}

template <bool GATHER, int NH>
static cudaError_t launch_overlap_t(const CUtensorMap &tm, const OverlapArgs &a, uint32_t sbins,
                                    uint64_t ntg, cudaStream_t s) {
  const size_t smem = ov_smem_bytes(sbins);
  static SmemOptIn attr;
  if (cudaError_t e = smem_opt_in(attr, k_overlap<GATHER, NH>, smem); e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_overlap<GATHER, NH>, kOvThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)num_sms() * per_sm;
  if (grid > ntg) grid = ntg;
  k_overlap<GATHER, NH><<<(unsigned)grid, kOvThreads, smem, s>>>(tm, a, sbins);
  return cudaGetLastError();
}

cudaError_t launch_overlap(const OverlapArgs &a_in, cudaStream_t s) {
  if (a_in.pixels == 0) return cudaSuccess;
  OverlapArgs a = a_in;
  a.vec = ((reinterpret_cast<uintptr_t>(a.counts) | reinterpret_cast<uintptr_t>(a.rgba)) & 15) == 0;
  const uint32_t k = a.k1 + a.k2;
  const int64_t first = contiguous_run(a.host_slots, k);
  CUtensorMap tm;
  cudaError_t e;
  const bool gather = first < 0;
  const uint64_t ntiles = a.wpm / 32;
  if (!gather)
    e = encode_packed_map(&tm, a.packed, a.capacity, (uint64_t)first, k, ntiles, 32, kOvGroup,
                          kOvTiles, 0);
  else
    e = encode_packed_map(&tm, a.packed, a.capacity, 0, a.capacity, ntiles, 32, 1, kOvTiles, 0);
  if (e != cudaSuccess) return e;
  // shared-memory histogram / RGBA table sized to the overlap classes
  uint32_t sbins = 0;
  if (a.nbins <= kHistSmemBins) sbins = (uint32_t)((a.nbins + 31) / 32 * 32);
  const uint64_t ntg = (ntiles + kOvTiles - 1) / kOvTiles;
  const uint32_t gmax = std::max((a.k1 + kOvGroup - 1) / kOvGroup, (a.k2 + kOvGroup - 1) / kOvGroup);
  if (gather) {
    if (gmax <= 31) return launch_overlap_t<true, 5>(tm, a, sbins, ntg, s);
    if (gmax <= 255) return launch_overlap_t<true, 8>(tm, a, sbins, ntg, s);
    return launch_overlap_t<true, 12>(tm, a, sbins, ntg, s);
  }
  if (gmax <= 31) return launch_overlap_t<false, 5>(tm, a, sbins, ntg, s);
  if (gmax <= 255) return launch_overlap_t<false, 8>(tm, a, sbins, ntg, s);
  return launch_overlap_t<false, 12>(tm, a, sbins, ntg, s);
}

// ---------------------------------------------------------------------------
// Multi-panel fused recompute, second half: counts = sum of the panels' uint16 partial
// counts; composite from the SMEM grey table; histogram run-length into SMEM bins.
// 24 B/px of traffic (4 panels) instead of the N/8 B/px re-read of the packed masks.
// ---------------------------------------------------------------------------
constexpr int kCombThreads = 256;
__global__ void __launch_bounds__(kCombThreads)
    k_combine_partials(const uint16_t *__restrict__ part, uint32_t npanels, uint64_t pitch,
                       const OverlapArgs a, uint32_t sbins) {
  extern __shared__ uint32_t csm[];
  uint32_t *hist = csm;            // sbins (0 -> global atomics)
  uint32_t *lut = csm + sbins;     // sbins RGBA words
  for (uint32_t i = threadIdx.x; i < sbins; i += blockDim.x) {
    hist[i] = 0;
    lut[i] = (a.rgba != nullptr && i < a.nbins) ? rgba_word(i, a.n_inputs, a.lut) : 0u;
  }
  __syncthreads();
  const uint64_t ngroups = (a.pixels + 7) / 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < ngroups; g += stride) {
    const uint64_t p0 = g * 8;
    uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t q = 0; q < npanels; ++q) {
      const uint4 v = ptx::ld_nc_v4(part + q * pitch + p0);  // pitch is a multiple of 1024
      c[0] += v.x & 0xFFFFu; c[1] += v.x >> 16;
      c[2] += v.y & 0xFFFFu; c[3] += v.y >> 16;
      c[4] += v.z & 0xFFFFu; c[5] += v.z >> 16;
      c[6] += v.w & 0xFFFFu; c[7] += v.w >> 16;
    }
    const int nv = a.pixels - p0 >= 8 ? 8 : (int)(a.pixels - p0);
    if (a.bins != nullptr) {
      uint32_t cur = c[0], run = 1;
      for (int j = 1; j < nv; ++j) {
        if (c[j] != cur) {
          if (sbins) atomicAdd(hist + cur, run);
          else atomicAdd(a.bins + cur, (unsigned long long)run);
          cur = c[j];
          run = 0;
        }
        ++run;
      }
      if (sbins) atomicAdd(hist + cur, run);
      else atomicAdd(a.bins + cur, (unsigned long long)run);
    }
    uint32_t r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      r[j] = a.rgba == nullptr ? 0u : (sbins ? lut[c[j]] : rgba_word(c[j], a.n_inputs, a.lut));
    if (nv == 8 && a.vec) {
      if (a.counts) {
        st_cs_v4(a.counts + p0, make_uint4(c[0], c[1], c[2], c[3]));
        st_cs_v4(a.counts + p0 + 4, make_uint4(c[4], c[5], c[6], c[7]));
      }
      if (a.rgba) {
        st_cs_v4(a.rgba + p0, make_uint4(r[0], r[1], r[2], r[3]));
        st_cs_v4(a.rgba + p0 + 4, make_uint4(r[4], r[5], r[6], r[7]));
      }
    } else {
      for (int j = 0; j < nv; ++j) {
        if (a.counts) a.counts[p0 + j] = c[j];
        if (a.rgba) a.rgba[p0 + j] = r[j];
      }
    }
  }
  if (sbins && a.bins != nullptr) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < sbins && i < a.nbins; i += blockDim.x)
      if (hist[i]) atomicAdd(a.bins + i, (unsigned long long)hist[i]);
  }
}

cudaError_t launch_combine_partials(const uint16_t *partial16, uint32_t npanels, uint64_t pitch,
                                    const OverlapArgs &a_in, cudaStream_t s) {
  if (a_in.pixels == 0) return cudaSuccess;
  OverlapArgs a = a_in;
  a.vec = ((reinterpret_cast<uintptr_t>(a.counts) | reinterpret_cast<uintptr_t>(a.rgba)) & 15) == 0;
  const uint32_t sbins = a.nbins <= 8192 ? (uint32_t)((a.nbins + 31) / 32 * 32) : 0u;
  const size_t smem = (size_t)sbins * 8;
  static SmemOptIn attr;
  if (smem > 48 * 1024)
    if (cudaError_t e = smem_opt_in(attr, k_combine_partials, smem); e != cudaSuccess) return e;
  const uint64_t ngroups = (a.pixels + 7) / 8;
  uint64_t grid = (ngroups + kCombThreads - 1) / kCombThreads;
  const uint64_t gcap = (uint64_t)num_sms() * 8;
  if (grid > gcap) grid = gcap;
  k_combine_partials<<<(unsigned)grid, kCombThreads, smem, s>>>(partial16, npanels, pitch, a, sbins);
  return cudaGetLastError();
}

// Per-item streaming accumulate (run_stream's kernel[i]): counts += bits of one
// mask.  A warp takes one tile: one coalesced 128-B load, then word i is broadcast
// and lane l adds bit l, so the counts stores are lane-contiguous.
__global__ void k_accumulate_packed(const uint32_t *__restrict__ packed, uint64_t slot,
                                    uint64_t cap, uint64_t pixels, uint32_t *__restrict__ counts) {
  const uint64_t nwords = (pixels + 31) / 32;
  const uint64_t ntiles = (nwords + 31) / 32;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = warp; t < ntiles; t += nwarps) {
    const uint32_t mine = ptx::ld_nc_u32(packed + (t * cap + slot) * 32 + lane);
    for (int i = 0; i < 32; ++i) {
      const uint32_t wd = __shfl_sync(0xffffffffu, mine, i);
      const uint64_t px = (t * 32 + i) * 32 + lane;
      if (px < pixels) counts[px] += (wd >> lane) & 1u;
    }
  }
}

cudaError_t launch_accumulate_packed(const uint32_t *packed, uint64_t slot, uint64_t cap,
                                     uint64_t pixels, uint32_t *counts, cudaStream_t s) {
  if (pixels == 0) return cudaSuccess;
  const uint64_t ntiles = ((pixels + 31) / 32 + 31) / 32;
  uint64_t grid = (ntiles + 7) / 8;
  uint64_t cap_grid = (uint64_t)num_sms() * 8;
  if (grid > cap_grid) grid = cap_grid;
  k_accumulate_packed<<<(unsigned)grid, 256, 0, s>>>(packed, slot, cap, pixels, counts);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Gram on CUDA cores: AND + POPC over bit-packed masks (baseline engine)
// ---------------------------------------------------------------------------
constexpr int kGpTile = 64;
constexpr int kGpSlab = 32;

__global__ void __launch_bounds__(256)
    k_gram_popc(const uint32_t *__restrict__ packed, uint64_t cap, uint64_t wpm,
                const uint32_t *__restrict__ slots, uint32_t k, uint32_t nb, uint64_t kchunk,
                unsigned long long *__restrict__ gram) {
  __shared__ uint32_t A[kGpTile][kGpSlab + 1];
  __shared__ uint32_t B[kGpTile][kGpSlab + 1];
  // upper-triangular tile index -> (I, J)
  uint32_t t = blockIdx.x, I = 0;
  while (t >= nb - I) {
    t -= nb - I;
    ++I;
  }
  const uint32_t J = I + t;
  const uint64_t k0 = (uint64_t)blockIdx.y * kchunk;
  const uint64_t k1 = min(k0 + kchunk, wpm);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  uint32_t acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (uint64_t kb = k0; kb < k1; kb += kGpSlab) {
    for (int idx = threadIdx.x; idx < kGpTile * kGpSlab; idx += 256) {
      const int r = idx / kGpSlab, c = idx % kGpSlab;
      const uint32_t ra = I * kGpTile + r, rb = J * kGpTile + r;
      const bool kin = kb + c < k1;
      A[r][c] = (ra < k && kin) ? __ldg(packed + pk_off(__ldg(slots + ra), kb + c, cap)) : 0u;
      B[r][c] = (rb < k && kin) ? __ldg(packed + pk_off(__ldg(slots + rb), kb + c, cap)) : 0u;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < kGpSlab; ++c) {
      uint32_t av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = A[ty * 4 + i][c];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = B[tx * 4 + j][c];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += __popc(av[i] & bv[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t r = I * kGpTile + ty * 4 + i, c = J * kGpTile + tx * 4 + j;
      if (r < k && c < k && acc[i][j]) atomicAdd(gram + (uint64_t)r * k + c, (unsigned long long)acc[i][j]);
    }
}

cudaError_t launch_gram_popc(const uint32_t *packed, uint64_t cap, uint64_t wpm,
                             const uint32_t *slots, uint32_t k, unsigned long long *gram,
                             cudaStream_t s) {
  if (k == 0) return cudaSuccess;
  const uint32_t nb = (k + kGpTile - 1) / kGpTile;
  const uint32_t ntiles = nb * (nb + 1) / 2;
  uint64_t want = (uint64_t)num_sms() * 4;
  uint64_t ksplit = (want + ntiles - 1) / ntiles;
  uint64_t kchunk = (wpm + ksplit - 1) / ksplit;
  kchunk = (kchunk + kGpSlab - 1) / kGpSlab * kGpSlab;
  if (kchunk == 0) kchunk = kGpSlab;
  ksplit = (wpm + kchunk - 1) / kchunk;
  if (ksplit > 65535) {
    ksplit = 65535;
    kchunk = ((wpm + ksplit - 1) / ksplit + kGpSlab - 1) / kGpSlab * kGpSlab;
  }
  dim3 grid(ntiles, (unsigned)ksplit);
  k_gram_popc<<<grid, 256, 0, s>>>(packed, cap, wpm, slots, k, nb, kchunk, gram);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_gram_mirror(gram, k, kGpTile, s);
}

// Fill entries of lower tiles from their mirror (tile size `tile`).
__global__ void k_gram_mirror(unsigned long long *gram, uint32_t k, uint32_t tile) {
  const uint64_t n = (uint64_t)k * k;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(e / k), j = (uint32_t)(e % k);
    if (i / tile > j / tile) gram[e] = gram[(uint64_t)j * k + i];
  }
}

cudaError_t launch_gram_mirror(unsigned long long *gram, uint32_t k, uint32_t tile,
                               cudaStream_t s) {
  if (k <= tile) return cudaSuccess;
  uint64_t n = (uint64_t)k * k;
  uint64_t grid = (n + 255) / 256;
  if (grid > 4096) grid = 4096;
  k_gram_mirror<<<(unsigned)grid, 256, 0, s>>>(gram, k, tile);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Synthetic masks generated straight into the packed layout
// ---------------------------------------------------------------------------
__global__ void k_synth_packed(uint32_t *__restrict__ dst, uint64_t slot, uint64_t cap,
                               uint64_t wpm, SynthParams sp, uint64_t mask, uint64_t row0,
                               uint64_t pixels) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < wpm; w += stride) {
    uint32_t word = 0;
    const uint64_t p0 = w * 32;
    if (p0 < pixels) {
      uint64_t y = row0 + p0 / sp.width;
      uint32_t x = (uint32_t)(p0 % sp.width);
      for (int b = 0; b < 32; ++b) {
        if (p0 + b >= pixels) break;
        if (synth_cell(sp, mask, (uint32_t)y, x) != 0) word |= 1u << b;
        if (++x == sp.width) {
          x = 0;
          ++y;
        }
      }
    }
    dst[pk_off(slot, w, cap)] = word;
  }
}

cudaError_t launch_synth_packed(uint32_t *dst, uint64_t slot, uint64_t cap, uint64_t wpm,
                                const SynthParams &sp, uint64_t mask, uint64_t row0,
                                uint64_t pixels, cudaStream_t s) {
  uint64_t grid = (wpm + 255) / 256;
  const uint64_t gcap = (uint64_t)num_sms() * 16;
  if (grid > gcap) grid = gcap;
  k_synth_packed<<<(unsigned)grid, 256, 0, s>>>(dst, slot, cap, wpm, sp, mask, row0, pixels);
  return cudaGetLastError();
}

// Synthetic masks as raw uint8 rasters (the bytes fs_synth_host writes), 8 px per
// thread-iteration, for generating large host inputs at copy speed.
__global__ void k_synth_raw(uint8_t *__restrict__ dst, SynthParams sp, uint64_t mask,
                            uint64_t row0, uint64_t pixels) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t base = row0 * sp.width;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q * 8 < pixels; q += stride) {
    uint64_t v = 0;
    const uint64_t p0 = q * 8;
    const int nb = (pixels - p0) < 8 ? (int)(pixels - p0) : 8;
    uint64_t y = (base + p0) / sp.width;
    uint32_t x = (uint32_t)((base + p0) % sp.width);
    for (int b = 0; b < nb; ++b) {
      v |= (uint64_t)synth_cell(sp, mask, (uint32_t)y, x) << (8 * b);
      if (++x == sp.width) {
        x = 0;
        ++y;
      }
    }
    if (nb == 8 && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
      reinterpret_cast<uint64_t *>(dst)[q] = v;
    } else {
      for (int b = 0; b < nb; ++b) dst[p0 + b] = (uint8_t)(v >> (8 * b));
    }
  }
}

cudaError_t launch_synth_raw(uint8_t *dst, const SynthParams &sp, uint64_t mask, uint64_t row0,
                             uint64_t pixels, cudaStream_t s) {
  if (pixels == 0) return cudaSuccess;
  uint64_t grid = (pixels / 8 + 255) / 256 + 1;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  k_synth_raw<<<(unsigned)grid, 256, 0, s>>>(dst, sp, mask, row0, pixels);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Jaccard matrix + outlier scores from the exact int64 Gram, on the device
// (analytics.py:165-181 and :229-240 of the reference).  Jaccard = inter / union in
// IEEE double (exact integer operands below 2^53, correctly rounded division = Python's
// int/int true division), 1.0 on the diagonal and for empty unions.  Outlier score of
// row i = 1 - (left-to-right double sum over j != i) / (n - 1): one thread per row keeps
// the reference's summation order, so the result is bit-identical to the host's.
// ---------------------------------------------------------------------------
__global__ void k_similarity(const long long *__restrict__ gram, uint32_t n, double *__restrict__ sim) {
  const uint64_t total = (uint64_t)n * n;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(e / n), j = (uint32_t)(e % n);
    double v = 1.0;
    if (i != j) {
      const long long inter = gram[e];
      const long long uni = gram[(uint64_t)i * n + i] + gram[(uint64_t)j * n + j] - inter;
      if (uni != 0) v = __ddiv_rn((double)inter, (double)uni);
    }
    sim[e] = v;
  }
}

// Row i's sum walks column i instead (sim is exactly symmetric: the Gram is mirrored
// and inter / (g_ii + g_jj - inter) is the same double either way).  A warp owns 32
// consecutive rows: it stages 128 x 32 blocks of the matrix in SMEM with independent,
// coalesced loads (lane l reads column i0 + l of each row j), then every lane adds its
// column in ascending j — the reference's order, so the sums are bit-identical.
constexpr int kOutJ = 128;
__global__ void __launch_bounds__(32)
    k_outliers(const double *__restrict__ sim, uint32_t n, double *__restrict__ scores) {
  __shared__ double tile[kOutJ][33];
  const uint32_t lane = threadIdx.x;
  const uint32_t i = blockIdx.x * 32 + lane;
  double acc = 0.0;
  for (uint32_t j0 = 0; j0 < n; j0 += kOutJ) {
#pragma unroll 8
    for (int r = 0; r < kOutJ; ++r) {
      const uint32_t j = j0 + r;
      tile[r][lane] = (j < n && i < n) ? sim[(uint64_t)j * n + i] : 0.0;
    }
    __syncwarp();
    for (int r = 0; r < kOutJ; ++r) {
      const uint32_t j = j0 + r;
      if (j < n && j != i) acc = __dadd_rn(acc, tile[r][lane]);
    }
    __syncwarp();
  }
  if (i < n) scores[i] = __dsub_rn(1.0, __ddiv_rn(acc, (double)(n - 1)));
}

cudaError_t launch_similarity_outliers(const long long *gram, uint32_t n, double *sim,
                                       double *scores, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t total = (uint64_t)n * n;
  uint64_t grid = (total + 255) / 256;
  const uint64_t gcap = (uint64_t)num_sms() * 8;
  if (grid > gcap) grid = gcap;
  k_similarity<<<(unsigned)grid, 256, 0, s>>>(gram, n, sim);
  if (scores != nullptr && n >= 2) k_outliers<<<(n + 31) / 32, 32, 0, s>>>(sim, n, scores);
  return cudaGetLastError();
}

// iid test rasters for the transform sweep: byte = depth 1..255 with p = 0.5, else 0
__global__ void k_fill_random(uint8_t *__restrict__ dst, uint64_t n, uint64_t seed) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q * 8 < n; q += stride) {
    const uint64_t h = mix64(seed ^ (q * 0x9E3779B97F4A7C15ull));
    uint64_t v = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint64_t byte = (h >> (8 * b)) & 0xFF;
      v |= ((byte & 1) ? (byte | 1) : 0ull) << (8 * b);
    }
    if (q * 8 + 8 <= n) {
      reinterpret_cast<uint64_t *>(dst)[q] = v;
    } else {
      for (uint64_t b = 0; q * 8 + b < n; ++b) dst[q * 8 + b] = (uint8_t)(v >> (8 * b));
    }
  }
}

cudaError_t launch_fill_random(uint8_t *dst, uint64_t n, uint64_t seed, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n / 8 + 255) / 256 + 1;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  k_fill_random<<<(unsigned)grid, 256, 0, s>>>(dst, n, seed);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Host: TMA tensor maps over the packed layout
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

cudaError_t encode_packed_map(CUtensorMap *out, const uint32_t *packed, uint64_t capacity,
                              uint64_t row0, uint64_t rows, uint64_t ntiles, uint32_t box_words,
                              uint32_t box_rows, uint32_t box_tiles, int swizzle) {
  if (g_encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr) return e != cudaSuccess ? e : cudaErrorNotSupported;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[3] = {32, rows > 0 ? rows : 1, ntiles > 0 ? ntiles : 1};
  cuuint64_t strides[2] = {128, capacity * 128};
  cuuint32_t box[3] = {box_words, box_rows, box_tiles};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                          : CU_TENSOR_MAP_SWIZZLE_NONE;
  void *base = const_cast<uint32_t *>(packed) + row0 * 32;
  CUresult r = g_encode(out, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int64_t contiguous_run(const uint32_t *host_slots, uint32_t k) {
  if (k == 0 || host_slots == nullptr) return -1;
  for (uint32_t i = 1; i < k; ++i)
    if (host_slots[i] != host_slots[0] + i) return -1;
  return host_slots[0];
}

// ---------------------------------------------------------------------------
// Host: composite grey LUT, evaluated exactly like _kernels_np.py:41-42 in FP64.
// This translation unit is compiled with -ffp-contract=off for host code.
// ---------------------------------------------------------------------------
uint8_t grey_of(uint64_t c, uint64_t n_inputs) {
  volatile double denom = (double)(n_inputs > 0 ? n_inputs : 1);
  volatile double sat = (double)c / denom;
  volatile double one_minus = 1.0 - sat;
  volatile double scaled = 255.0 * one_minus;
  volatile double shifted = scaled + 0.5;
  double g = std::floor(shifted);
  long long gi = (long long)g;
  return (uint8_t)(gi & 0xFF);
}

void build_grey_lut(uint64_t n_inputs, uint8_t *lut, uint64_t entries) {
  for (uint64_t c = 0; c < entries; ++c) lut[c] = grey_of(c, n_inputs);
}

}  // namespace fs
