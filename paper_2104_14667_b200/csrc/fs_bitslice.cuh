// fs_bitslice.cuh — device building blocks shared by the fused overlap pass and the
// fused Gram+overlap kernel: bit-sliced (Harley-Seal) mask counters, the exact composite
// colour, and the per-tile epilogue (histogram + counts + RGBA) of one warp.
//
// Reference semantics: accumulate_into (_kernels_np.py:16-18), overlap_counts
// (:21-23), composite_fill (:35-47) of /root/reference/pkg/src/floodstream/.
#pragma once
#include "fs_internal.h"

namespace fs {

// grey level g = floor(255 (1 - c / max(n, 1)) + 0.5) in FP64 (or from the host LUT)
__device__ __forceinline__ uint32_t grey_dev(uint64_t c, uint64_t n_inputs, const uint8_t *lut) {
  if (lut != nullptr) return __ldg(lut + c);
  double denom = (double)(n_inputs > 0 ? n_inputs : 1);
  double sat = __ddiv_rn((double)c, denom);
  double g = floor(__dadd_rn(__dmul_rn(255.0, __dsub_rn(1.0, sat)), 0.5));
  long long gi = (long long)g;
  return (uint32_t)(gi & 0xFF);
}
// RGBA (g, g, 255, 255) as one little-endian word; 0 when uncovered
__device__ __forceinline__ uint32_t rgba_word(uint32_t c, uint64_t n_inputs, const uint8_t *lut) {
  if (c == 0) return 0u;
  uint32_t g = grey_dev(c, n_inputs, lut);
  return g | (g << 8) | 0xFFFF0000u;
}

// carry-save adder: (h, l) = a + b + c
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b,
                                    uint32_t c) {
  const uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// Bit-sliced counter of 32 pixels: planes ones/twos/fours/eights plus NH ripple planes
// of sixteens, so one pass counts up to 16 (2^NH - 1) + 15 masks.
template <int NH>
struct HSCounter {
  uint32_t ones, twos, fours, eights;
  uint32_t H[NH];
  __device__ __forceinline__ void reset() {
    ones = twos = fours = eights = 0;
#pragma unroll
    for (int i = 0; i < NH; ++i) H[i] = 0;
  }
  __device__ __forceinline__ void add16(const uint32_t (&d)[16]) {
    uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
    csa(twosA, ones, ones, d[0], d[1]);
    csa(twosB, ones, ones, d[2], d[3]);
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, d[4], d[5]);
    csa(twosB, ones, ones, d[6], d[7]);
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsA, fours, fours, foursA, foursB);
    csa(twosA, ones, ones, d[8], d[9]);
    csa(twosB, ones, ones, d[10], d[11]);
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, d[12], d[13]);
    csa(twosB, ones, ones, d[14], d[15]);
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsB, fours, fours, foursA, foursB);
    csa(sixteens, eights, eights, eightsA, eightsB);
    uint32_t carry = sixteens;
#pragma unroll
    for (int i = 0; i < NH; ++i) {
      const uint32_t t = H[i] & carry;
      H[i] ^= carry;
      carry = t;
    }
  }
  // cnt[j] = count(pixel j): byte g (pixels 8g..8g+7) of planes 0..7 forms an 8 x 8 bit
  // matrix that three delta swaps transpose into byte i = bits 0..7 of the count of pixel
  // 8g + i; planes 8..15 the same for bits 8..15 (a lone plane 8 is read bit by bit).
  // ~7 ops per pixel instead of ~2 per plane per pixel.
  __device__ __forceinline__ void extract1(uint32_t (&cnt)[32]) const {
    constexpr int NP = 4 + NH;  // planes
    static_assert(NP <= 16, "at most 16 planes");
    uint32_t p[16] = {ones, twos, fours, eights};
#pragma unroll
    for (int i = 4; i < 16; ++i) p[i] = i < NP ? H[i < NP ? i - 4 : 0] : 0u;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint64_t x = transpose8x8(p, 0, g);
      uint64_t y = 0;
      if (NP > 9) y = transpose8x8(p, 8, g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 8 * g + i;
        uint32_t c = (uint32_t)((x >> (8 * i)) & 0xFFu);
        if (NP > 9)
          c |= (uint32_t)((y >> (8 * i)) & 0xFFu) << 8;
        else if (NP == 9)
          c |= ((p[8] >> j) & 1u) << 8;
        cnt[j] = c;
      }
    }
  }
  // byte g of planes b0..b0+7 as an 8 x 8 bit matrix (byte b = plane b0 + b), transposed:
  // byte i of the result = bits b0..b0+7 of the count of pixel 8g + i
  __device__ __forceinline__ static uint64_t transpose8x8(const uint32_t (&p)[16], int b0, int g) {
    const uint32_t sel = (uint32_t)g | ((uint32_t)(g + 4) << 4);
    const uint32_t lo = __byte_perm(__byte_perm(p[b0], p[b0 + 1], sel),
                                    __byte_perm(p[b0 + 2], p[b0 + 3], sel), 0x5410);
    const uint32_t hi = __byte_perm(__byte_perm(p[b0 + 4], p[b0 + 5], sel),
                                    __byte_perm(p[b0 + 6], p[b0 + 7], sel), 0x5410);
    uint64_t x = (uint64_t)lo | ((uint64_t)hi << 32);
    uint64_t t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    x = x ^ t ^ (t << 28);
    return x;
  }
  // cnt[j] += wt * count(pixel j)
  __device__ __forceinline__ void extract(uint32_t (&cnt)[32], uint32_t wt) const {
    uint32_t c[32];
    extract1(c);
#pragma unroll
    for (int k = 0; k < 32; ++k) cnt[k] += wt * c[k];
  }
};

__device__ __forceinline__ void st_cs_v4(void *p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

constexpr int kTileTb = 36;  // transpose row stride (words): 16-B aligned, conflict-free v4

// One warp emits one 1024-px tile (tile index `tile`, pixels 1024*tile + 32*w + b):
// cnt32[b] = count of pixel b of word `lane`.  `tb` is this warp's 32 x kTileTb SMEM
// scratch.  Histogram: run-length over the lane's 32 consecutive pixels into the SMEM
// bins (or global bins); padding pixels past a.pixels are counted in bin 0 and must be
// removed once by the caller.  Counts / RGBA: transposed through `tb` and written with
// 16-B streaming stores.
__device__ __forceinline__ void emit_tile(const uint32_t (&cnt32)[32], uint64_t tile, int lane,
                                          uint32_t *tb, const OverlapArgs &a, uint32_t *sh_hist,
                                          bool hist_sh, const uint32_t *sh_lut, bool lut_sh) {
  if (a.bins != nullptr) {
    uint32_t cur = cnt32[0], run = 1;
#pragma unroll
    for (int j = 1; j < 32; ++j) {
      const uint32_t c = cnt32[j];
      if (c != cur) {
        if (hist_sh)
          atomicAdd(sh_hist + cur, run);
        else if (cur < a.nbins)
          atomicAdd(a.bins + cur, (unsigned long long)run);
        cur = c;
        run = 0;
      }
      ++run;
    }
    if (hist_sh)
      atomicAdd(sh_hist + cur, run);
    else if (cur < a.nbins)
      atomicAdd(a.bins + cur, (unsigned long long)run);
  }
  if (a.counts == nullptr && a.rgba == nullptr) return;
  uint32_t *row = tb + lane * kTileTb;
#pragma unroll
  for (int v = 0; v < 8; ++v)
    *reinterpret_cast<uint4 *>(row + 4 * v) =
        make_uint4(cnt32[4 * v], cnt32[4 * v + 1], cnt32[4 * v + 2], cnt32[4 * v + 3]);
  __syncwarp();
  const uint64_t wbase = tile * 32;
#pragma unroll 2
  for (int it = 0; it < 8; ++it) {
    const int w = it * 4 + (lane >> 3), b0 = (lane & 7) * 4;
    const uint4 c = *reinterpret_cast<const uint4 *>(tb + w * kTileTb + b0);
    const uint64_t px0 = (wbase + w) * 32 + b0;
    uint4 r = make_uint4(0, 0, 0, 0);
    if (a.rgba != nullptr) {
      if (lut_sh) {
        r.x = sh_lut[c.x];
        r.y = sh_lut[c.y];
        r.z = sh_lut[c.z];
        r.w = sh_lut[c.w];
      } else {
        r.x = rgba_word(c.x, a.n_inputs, a.lut);
        r.y = rgba_word(c.y, a.n_inputs, a.lut);
        r.z = rgba_word(c.z, a.n_inputs, a.lut);
        r.w = rgba_word(c.w, a.n_inputs, a.lut);
      }
    }
    if (a.vec && px0 + 4 <= a.pixels) {
      if (a.counts) st_cs_v4(a.counts + px0, c);
      if (a.rgba) st_cs_v4(a.rgba + px0, r);
    } else {
      const uint32_t cv[4] = {c.x, c.y, c.z, c.w}, rv[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (px0 + e < a.pixels) {
          if (a.counts) a.counts[px0 + e] = cv[e];
          if (a.rgba) a.rgba[px0 + e] = rv[e];
        }
    }
  }
  __syncwarp();
}

// Partial counts of one 1024-px tile as uint16 (multi-panel fused recompute): the
// same SMEM transpose as emit_tile, then lane l writes 8 consecutive pixels (16 B) of
// word 8 it + l / 4 — a warp stores 512 contiguous bytes per iteration.
__device__ __forceinline__ void emit_partial16(const uint32_t (&cnt32)[32], uint64_t tile,
                                               int lane, uint32_t *tb, uint16_t *dst) {
  uint32_t *row = tb + lane * kTileTb;
#pragma unroll
  for (int v = 0; v < 8; ++v)
    *reinterpret_cast<uint4 *>(row + 4 * v) =
        make_uint4(cnt32[4 * v], cnt32[4 * v + 1], cnt32[4 * v + 2], cnt32[4 * v + 3]);
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int w = it * 8 + (lane >> 2), b0 = (lane & 3) * 8;
    const uint4 c0 = *reinterpret_cast<const uint4 *>(tb + w * kTileTb + b0);
    const uint4 c1 = *reinterpret_cast<const uint4 *>(tb + w * kTileTb + b0 + 4);
    const uint4 o = make_uint4(c0.x | (c0.y << 16), c0.z | (c0.w << 16), c1.x | (c1.y << 16),
                               c1.z | (c1.w << 16));
    st_cs_v4(dst + tile * 1024 + (uint64_t)w * 32 + b0, o);
  }
  __syncwarp();
}

}  // namespace fs
