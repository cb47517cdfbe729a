// fs_common.cuh — shared definitions for libfloodstream (sm_100a).
//
// Packed-mask layout in HBM (the "transformed", block-tiled layout every kernel
// consumes).  A mask's pixels (flat row-major raster order, so a row band [y0, y1)
// is the contiguous pixel range [y0*W, y1*W)) are bit-packed LSB first: pixel
// p = 32*w + b is bit b of word w.  Words are grouped in TILES of 32 words
// (1024 px, 128 B) and the tiles of all masks are interleaved:
//
//     packed[tile][slot][32 words]        word w of slot s at pk_off(s, w, capacity)
//
// so the same K-range (pixel tile) of every mask in the ensemble is ONE contiguous
// block of capacity x 128 B.  Every consumer streams whole contiguous blocks —
// the overlap pass reads [tile-group][16 masks][32 words] boxes, the Gram reads
// [tile][256 masks][32 words] boxes — through 3-D TMA tensor maps (dims: word,
// slot, tile).  words_per_mask is rounded up to whole tiles; padding is zero.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FS_WORD_ALIGN 32u  // words per mask rounded to 32 words = 1024 px = 128 B

namespace fs {

__host__ __device__ __forceinline__ uint64_t words_for_pixels(uint64_t pixels) {
  uint64_t w = (pixels + 31) / 32;
  return (w + FS_WORD_ALIGN - 1) / FS_WORD_ALIGN * FS_WORD_ALIGN;
}

// word w of slot s in the tile-interleaved layout
__host__ __device__ __forceinline__ uint64_t pk_off(uint64_t slot, uint64_t w, uint64_t capacity) {
  return ((w >> 5) * capacity + slot) * 32u + (w & 31u);
}

// ---- synthetic flood-like masks (counter based; identical on host and device) ----
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct SynthParams {
  uint64_t seed;
  uint32_t width, height;  // full raster dims
  uint32_t members;        // masks per prototype
  uint32_t flip_thr;       // eps * 2^32
};

// Prototype k: 16x16 low-res field thresholded at a per-prototype level in [0.3, 0.6).
__host__ __device__ __forceinline__ bool synth_proto(const SynthParams &sp, uint64_t proto,
                                                     uint32_t by, uint32_t bx) {
  uint64_t lvl = mix64(sp.seed ^ mix64(proto * 0x100000001B3ull + 0xA5A5ull));
  // threshold fraction 0.3 + 0.3*u, as a 32-bit level
  uint32_t thr = (uint32_t)(1288490188ull + (((lvl >> 32) * 1288490189ull) >> 32));
  uint64_t v = mix64(sp.seed ^ mix64((proto << 16) ^ (by << 8) ^ bx ^ 0x5EEDull));
  return (uint32_t)(v >> 32) < thr;
}

// Cell value (depth 0..255) of pixel (y, x) of mask `mask`.
__host__ __device__ __forceinline__ uint8_t synth_cell(const SynthParams &sp, uint64_t mask,
                                                       uint32_t y, uint32_t x) {
  uint64_t proto = mask / sp.members;
  uint32_t by = (uint32_t)((uint64_t)y * 16u / sp.height);
  uint32_t bx = (uint32_t)((uint64_t)x * 16u / sp.width);
  bool wet = synth_proto(sp, proto, by, bx);
  uint64_t p = (uint64_t)y * sp.width + x;
  uint64_t h = mix64(sp.seed * 0x2545F4914F6CDD1Dull ^ (mask << 40) ^ p);
  bool flip = (uint32_t)h < sp.flip_thr;
  wet = wet != flip;
  uint32_t depth = 1u + (uint32_t)((h >> 32) % 255u);
  return wet ? (uint8_t)depth : (uint8_t)0;
}

}  // namespace fs

// ---------------------------------------------------------------------------
// Device-only PTX helpers
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
namespace fs {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint4 ld_nc_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
// Bounded wait: traps (kernel error) instead of hanging the device forever.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  uint64_t spins = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) break;
    if (++spins > (1ull << 26)) __trap();
  }
}

// 1-D bulk async copy global -> shared (TMA bulk engine), completes on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 3-D TMA tile load (coordinates: word, slot, tile) completing on an mbarrier.
__device__ __forceinline__ void tma_load_3d(void *smem_dst, const void *tmap, int c0, int c1,
                                            int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// the same 3-D box into L2 only (no SMEM destination, no barrier)
__device__ __forceinline__ void tma_prefetch_3d(const void *tmap, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tmap),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace ptx
}  // namespace fs
#endif
