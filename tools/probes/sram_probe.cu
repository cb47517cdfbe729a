// sram_probe.cu — does the tensor core's SMEM operand fetch share shared-memory bandwidth
// with st.shared traffic?  (The question behind the fused recompute's per-unit budget.)
//
// One CTA per SM.  Warp 0 (one thread) issues the C2 recompute's MMA pattern — per
// 256-px stage 4 x (M=128 N=256 rows 0-127, M=128 N=128 rows 128-255) kind::mxf4 — over
// a static 4-stage operand ring for `stages` stages, with a commit per stage; warps
// 1..8 store `sts_per_stage` x 512 B per stage-equivalent with st.shared.v4 into a
// separate 64 KB region (no dependency on the MMAs).  Modes: MMA only, STS only, both.
// If the two streams share one SMEM port, "both" ~ "mma" + "sts"; if not, ~ max().
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sram_probe sram_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t a) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc,
                                    uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;"
      "\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}

constexpr int kRing = 4, kStage = 32768, kStsRegion = 65536;
constexpr int kSmem = kRing * kStage + kStsRegion + 1024;

__global__ void __launch_bounds__(288, 1)
    k_probe(int stages, int sts_per_stage, int mode, unsigned long long *cycles,
            const uint4 *gsrc, int fill) {
  extern __shared__ uint8_t sm[];
  __shared__ uint64_t bars[kRing];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tslot;
  __shared__ unsigned long long tend;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  const uint32_t sts_base = base + kRing * kStage;
  // operands: 0 = all zero, 1 = e2m1 1.0 / 0 nibbles from a hash (about half ones)
  for (int i = threadIdx.x; i < (kRing * kStage) / 16; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x5bd1e995u;
    h ^= h >> 15;
    h *= 0x2c1b3c6du;
    h ^= h >> 12;
    const uint32_t v = fill ? (h & 0x22222222u) : 0u;
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(base + 16 * i), "r"(v),
                 "r"(v ^ 0x20202020u), "r"(v ^ 0x02020202u), "r"(v ^ 0x22002200u));
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) mbar_init(&bars[i], 1);
    mbar_init(&done_bar, 1);
    tend = 0;
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x < 128) {
    const uint32_t lanes = (uint32_t)((threadIdx.x >> 5) * 32) << 16;
    const uint32_t v = 0x7F7F7F7Fu;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1};" ::"r"(tmem + lanes + 448u),
        "r"(v));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1};" ::"r"(tmem + lanes + 464u),
        "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const long long t0 = clock64();
  if (threadIdx.x == 0 && (mode & 1)) {
    const uint32_t idA = idesc_mxf4(128, 256), idB = idesc_mxf4(128, 128);
    const uint32_t sfa = tmem + 448u, sfb = tmem + 464u;
    for (int j = 0; j < stages; ++j) {
      const int s = j % kRing;
      if (j >= kRing) mbar_wait(&bars[s], (uint32_t)(((j / kRing) - 1) & 1));
      const uint32_t sb = base + s * kStage;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
        mma(tmem, sw128_desc(sb + ks * 32), sw128_desc(sb + ks * 32), idA, acc, sfa, sfb);
        mma(tmem + 256u, sw128_desc(sb + 16384 + ks * 32), sw128_desc(sb + 16384 + ks * 32), idB,
            acc, sfa, sfb);
      }
      commit(&bars[s]);
    }
    commit(&done_bar);
    mbar_wait(&done_bar, 0);
  } else if (threadIdx.x >= 32 && (mode & 8)) {
    // split: warps 1-4 store sts_per_stage x 512 B per stage with st.shared.v4, warps 5-8
    // stream sts_per_stage / 4 x 512 B per stage of global memory (the expanders' raw
    // units: a quarter of the expanded bytes), 8 x 16-B loads in flight per thread
    const int w = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;
    if (w < 4) {
      const int per_warp = (stages * sts_per_stage) / 4;
      uint32_t x = threadIdx.x * 2654435761u;
      for (int i = 0; i < per_warp; ++i) {
        const uint32_t off = (uint32_t)(((w * 977 + i) * 512) & (kStsRegion - 1)) + lane * 16;
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sts_base + off), "r"(x),
                     "r"(x + 1), "r"(x + 2), "r"(x + 3));
        x += 0x9E3779B9u;
      }
    } else {
      const int per_warp = (stages * sts_per_stage / 4) / 4;
      uint32_t acc = 0;
      const uint4 *p = gsrc + ((size_t)blockIdx.x * 4 + (w - 4)) * 32 + lane;
      for (int i = 0; i < per_warp; i += 8) {
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const size_t off = ((size_t)(i + j) * 148 * 4 * 32) & ((1ull << 26) - 1);
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w)
                       : "l"(p + off));
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].w;
      }
      if (acc == 0x12345678u) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sts_base), "r"(acc));
    }
  } else if (threadIdx.x >= 32 && (mode & 4)) {
    // 8 warps stream global memory (16-B loads, 8 in flight per thread), like the expanders
    const int w = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;
    const int per_warp = (stages * sts_per_stage) / 8;
    uint32_t acc = 0;
    const uint4 *p = gsrc + ((size_t)blockIdx.x * 8 + w) * 32 + lane;
    for (int i = 0; i < per_warp; i += 8) {
      uint4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const size_t off = ((size_t)(i + j) * 148 * 8 * 32) & ((1ull << 26) - 1);
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w)
                     : "l"(p + off));
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].w;
    }
    if (acc == 0x12345678u) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sts_base), "r"(acc));
  } else if (threadIdx.x >= 32 && (mode & 2)) {
    // 8 warps: per stage-equivalent, sts_per_stage warp-wide st.shared.v4 (512 B each)
    const int w = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;
    const int per_warp = (stages * sts_per_stage) / 8;
    uint32_t x = threadIdx.x * 2654435761u;
    for (int i = 0; i < per_warp; ++i) {
      const uint32_t off = (uint32_t)(((w * 977 + i) * 512) & (kStsRegion - 1)) + lane * 16;
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sts_base + off), "r"(x),
                   "r"(x + 1), "r"(x + 2), "r"(x + 3));
      x += 0x9E3779B9u;
    }
  }
  atomicMax(&tend, (unsigned long long)clock64());  // each thread's own finish time
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = tend - (unsigned long long)t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  uint4 *g;
  cudaMalloc(&g, (1ull << 26) * 16 + 4096 * 16);
  cudaMemset(g, 0x5a, (1ull << 26) * 16 + 4096 * 16);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  const int stages = 4096;
  printf("{\"probe\": \"C2 MMA pattern vs concurrent st.shared.v4 traffic, cycles per 256-px stage\","
         " \"ideal_mma\": 768, \"rows\": [\n");
  bool first = true;
  struct Case { int sts, mode, fill; const char *name; };
  // mode bits: 1 MMA, 2 st.shared (sts x 512 B per stage), 4 global loads (sts x 512 B per stage)
  const Case cases[] = {{0, 1, 0, "mma zeros"},        {0, 1, 1, "mma data"},
                        {64, 2, 0, "sts 32KB"},         {64, 3, 1, "mma data + sts 32KB"},
                        {64, 4, 0, "ldg 32KB"},         {64, 5, 1, "mma data + ldg 32KB"},
                        {128, 4, 0, "ldg 64KB"},        {128, 5, 1, "mma data + ldg 64KB"},
                        {64, 8, 0, "sts 32KB + ldg 8KB"}, {64, 9, 1, "mma data + sts 32KB + ldg 8KB"}};
  for (const Case &c : cases) {
    unsigned long long cyc = 0;
    k_probe<<<148, 288, kSmem>>>(stages / 8, c.sts, c.mode, d, g, c.fill);  // warm-up
    k_probe<<<148, 288, kSmem>>>(stages, c.sts, c.mode, d, g, c.fill);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("%s{\"case\": \"%s\", \"cycles_per_stage\": %.1f, \"err\": \"%s\"}", first ? "" : ",\n",
           c.name, (double)cyc / stages, cudaGetErrorString(e));
    first = false;
  }
  printf("\n]}\n");
  return 0;
}
