// fs_tcgen05.cuh — tcgen05 / TMEM / SMEM helpers shared by the tensor-core kernels
// (fs_gram_tc.cu: Gram tiles; fs_recompute_f4.cu: the fused single-panel recompute).
// Descriptor encodings follow cute::UMMA (SmemDescriptor, InstrDescriptor[BlockScaled]).
#pragma once
#include "fs_common.cuh"

namespace fs {
namespace tc {

__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);  // start address
  d |= (uint64_t)1u << 16;                      // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;            // SBO: 8 rows x 128 B
  d |= (uint64_t)1u << 46;                      // descriptor version (sm_100)
  d |= (uint64_t)2u << 61;                      // SWIZZLE_128B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)                      // D format: S32
         | (0u << 7) | (0u << 10)       // A, B: unsigned 8-bit
         | ((uint32_t)(N >> 3) << 17)   // N
         | ((uint32_t)(M >> 4) << 24);  // M
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// block-scaled descriptor (cute::UMMA::InstrDescriptorBlockScaled): a/b format E2M1 (1)
// at bits 7/10, N>>3 at 17, scale format UE8M0 at 23, M>>4 at 24, sf ids 0, K = 64.
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_mxf4(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accum, uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;"
      "\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum), "r"(sfa), "r"(sfb));
}

// 16 columns of this warp's 32 TMEM lanes <- v
__device__ __forceinline__ void tmem_st16(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ptx::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 16 bits -> 16 bytes of 0/1
__device__ __forceinline__ uint4 expand16(uint32_t half) {
  uint4 o;
  o.x = ((half & 0xFu) * 0x00204081u) & 0x01010101u;
  o.y = (((half >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
  o.z = (((half >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
  o.w = (((half >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
  return o;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// Expand one 128-px row slice (4 words) into SW128 operand row `row` at `base`.
__device__ __forceinline__ void expand_row(uint32_t base, uint32_t row, uint4 v) {
  const uint32_t rbase = base + row * 128u;
  const uint32_t sw = row & 7u;
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t half = (w[c >> 1] >> ((c & 1) * 16)) & 0xFFFFu;
    st_shared_v4(rbase + (((uint32_t)c ^ sw) << 4), expand16(half));
  }
}

// FP4: one raw 16-B chunk (4 words, 128 px) of row `row` -> 4 operand chunks (64 B)
// at chunk positions c0..c0+3 of SW128 row `row`.
__device__ __forceinline__ void expand_row_f4(uint32_t base, uint32_t row, uint32_t c0, uint4 v) {
  const uint32_t rbase = base + row * 128u;
  const uint32_t sw = row & 7u;
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t x = w[q];
    uint4 o;
    o.x = (x << 1) & 0x22222222u;
    o.y = x & 0x22222222u;
    o.z = (x >> 1) & 0x22222222u;
    o.w = (x >> 2) & 0x22222222u;
    st_shared_v4(rbase + (((c0 + (uint32_t)q) ^ sw) << 4), o);
  }
}

constexpr uint32_t kSfCol = 448;          // FP4: scale-factor columns [448, 480) of TMEM
constexpr uint32_t kSfOnes = 0x7F7F7F7Fu; // UE8M0 127 = 2^0 in every byte

}  // namespace tc
}  // namespace fs
