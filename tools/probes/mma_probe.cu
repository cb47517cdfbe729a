// mma_probe.cu — issue-rate probe for tcgen05.mma.kind::mxf4 (M=128) on one B200.
//
// Every CTA (one per SM) zero-fills 48 KB of SMEM operands, sets all block scales to 1.0
// and lets one thread issue `iters` groups of 4 MMAs (K = 4 x 64) with N = 16 .. 256,
// optionally committing to an mbarrier after every group and waiting for it `lag`
// groups later (the fused kernel's stage ring).  Prints cycles per MMA instruction
// against the ideal M*N*K / (16384 MAC/clk).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
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
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(phase));
}

template <int NACC>
__global__ void __launch_bounds__(128, 1) k_probe(int n, int iters, int lag, int dual,
                                                  unsigned long long *cycles) {
  constexpr int nacc = NACC;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[16];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < (48 * 1024) / 16; i += blockDim.x)
    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 16 * i), "r"(0));
  if (threadIdx.x == 0)
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
  if (threadIdx.x == 0) mbar_init(&done_bar, 1);
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
  {
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
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_mxf4(128, n);
    const uint32_t id2 = idesc_mxf4(128, 128);
    const uint32_t sfa = tmem + 448u, sfb = tmem + 464u;
    const uint32_t a_base = base, b_base = base + 16 * 1024;
    const long long t0 = clock64();
    for (int j = 0; j < iters; ++j) {
      if (lag > 0 && j >= lag) mbar_wait(&bars[(j - lag) % 16], (uint32_t)(((j - lag) / 16) & 1));
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        // rotate over nacc accumulators (compile-time: ks is unrolled)
        mma(tmem + (uint32_t)(ks % nacc) * (nacc > 2 ? 64u : 128u), sw128_desc(a_base + ks * 32),
            sw128_desc(b_base + ks * 32), id, (j > 0 || ks >= nacc) ? 1u : 0u, sfa, sfb);
        if (dual)
          mma(tmem + 256u, sw128_desc(a_base + 128 * 128 + ks * 32),
              sw128_desc(b_base + 128 * 128 + ks * 32), id2, (j > 0 || ks > 0) ? 1u : 0u, sfa, sfb);
      }
      if (lag > 0) commit(&bars[j % 16]);
    }
    commit(&done_bar);
    mbar_wait(&done_bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// The fused C2 kernel's issue pattern: per 256-px stage, 4 x (rows 0-127 x N=256 into
// accumulator 0, rows 128-255 x N=128 into accumulator 256) from a 4-deep stage ring
// (32 KB stages, A = B), descriptors built per MMA from the stage address (mode 0, as in
// k_gram_tc) or precomputed once and offset (mode 1); commit per stage.
__global__ void __launch_bounds__(128, 1) k_probe_ring(int iters, int mode,
                                                       unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[4];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < (128 * 1024) / 16; i += blockDim.x)
    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 16 * i), "r"(0));
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    mbar_init(&done_bar, 1);
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
  {
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
  if (threadIdx.x == 0) {
    const uint32_t idA = idesc_mxf4(128, 256), idB = idesc_mxf4(128, 128);
    const uint32_t sfa = tmem + 448u, sfb = tmem + 464u;
    const uint64_t d0 = sw128_desc(base);
    const long long t0 = clock64();
    for (int j = 0; j < iters; ++j) {
      const int s = j % 4;
      const uint32_t a_base = base + s * 32768;
      if (j >= 4) mbar_wait(&bars[s], (uint32_t)(((j / 4) - 1) & 1));
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
        uint64_t a0, b0, a1, b1;
        if (mode == 0) {
          a0 = sw128_desc(a_base + ks * 32);
          b0 = sw128_desc(a_base + ks * 32);
          a1 = sw128_desc(a_base + 128 * 128 + ks * 32);
          b1 = sw128_desc(a_base + 128 * 128 + ks * 32);
        } else {
          const uint64_t o = (uint64_t)((s * 32768 + ks * 32) >> 4);
          a0 = b0 = d0 + o;
          a1 = b1 = d0 + o + (128 * 128 >> 4);
        }
        mma(tmem, a0, b0, idA, acc, sfa, sfb);
        mma(tmem + 256u, a1, b1, idB, acc, sfa, sfb);
      }
      commit(&bars[s]);
    }
    commit(&done_bar);
    mbar_wait(&done_bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Which M=128, N=128 MMA streams pipeline?  8 MMAs per group (ideal 8 x 64 cycles):
// variant 0: A/B rows 0-127 of two different stage buffers, one accumulator
// variant 1: the same into two accumulators (one per buffer)
// variant 2: rows 0-127 and rows 128-255 of one buffer (A = B), two accumulators
// variant 3: rows 0-127 of one buffer twice, two accumulators (same operands)
__global__ void __launch_bounds__(128, 1) k_probe_pairs(int iters, int variant,
                                                        unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < (64 * 1024) / 16; i += blockDim.x)
    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 16 * i), "r"(0));
  if (threadIdx.x == 0) mbar_init(&done_bar, 1);
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
  {
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
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_mxf4(128, 128);
    const uint32_t sfa = tmem + 448u, sfb = tmem + 464u;
    const uint32_t x0 = base;
    const uint32_t x1 = variant <= 1 ? base + 32768 : variant == 2 ? base + 16384 : base;
    const uint32_t d1 = variant == 0 ? tmem : tmem + 128u;
    const long long t0 = clock64();
    for (int j = 0; j < iters; ++j) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
        mma(tmem, sw128_desc(x0 + ks * 32), sw128_desc(x0 + ks * 32), id, acc, sfa, sfb);
        mma(d1, sw128_desc(x1 + ks * 32), sw128_desc(x1 + ks * 32), id,
            (variant == 0 || j > 0 || ks > 0) ? 1u : 0u, sfa, sfb);
      }
    }
    commit(&done_bar);
    mbar_wait(&done_bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
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
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  printf("{\"probe\": \"tcgen05.mma kind::mxf4 M=128 K=64 issue rate\", \"rows\": [\n");
  bool first = true;
  for (int dual = 0; dual <= 1; ++dual)
   for (int nacc : {1, 2, 4})
    for (int lag : {0, 4})
      for (int n : {16, 64, 128, 256}) {
        if (dual && (n != 256 || nacc != 1)) continue;
        if (nacc > 2 && n > 64) continue;
        if (nacc > 1 && n > 128) continue;
        if (nacc == 1) k_probe<1><<<148, 128, smem>>>(n, iters, lag, dual, d);
        if (nacc == 2) k_probe<2><<<148, 128, smem>>>(n, iters, lag, dual, d);
        if (nacc == 4) k_probe<4><<<148, 128, smem>>>(n, iters, lag, dual, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        const int per = 4 * (dual ? 2 : 1);
        // per-MMA ideal at 16384 FP4 MACs / clk / SM
        const double ideal = 128.0 * n * 64 / 16384.0 + (dual ? 128.0 * 128 * 64 / 16384.0 : 0.0);
        printf("%s{\"n\": %d, \"accumulators\": %d, \"dual_n128\": %d, \"commit_lag\": %d, \"cycles_per_group\": %.1f, "
               "\"ideal_cycles_per_group\": %.1f, \"cycles_per_mma\": %.1f, \"err\": \"%s\"}",
               first ? "" : ",\n", n, nacc, dual, lag, (double)c / iters, ideal * 4,
               (double)c / iters / per, cudaGetErrorString(e));
        first = false;
        if (e != cudaSuccess) return 1;
      }
  printf("\n], \"ring\": [\n");
  cudaFuncSetAttribute(k_probe_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 130 * 1024);
  for (int mode = 0; mode <= 1; ++mode) {
    k_probe_ring<<<148, 128, 130 * 1024>>>(iters, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%s{\"mode\": \"%s\", \"cycles_per_stage\": %.1f, \"ideal\": 768, \"err\": \"%s\"}",
           mode ? ",\n" : "", mode ? "precomputed descriptors" : "descriptors per MMA (k_gram_tc)",
           (double)c / iters, cudaGetErrorString(e));
  }
  printf("\n], \"pairs_n128\": [\n");
  cudaFuncSetAttribute(k_probe_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const char *names[4] = {"two buffers, one accumulator", "two buffers, two accumulators",
                          "rows 0-127 / 128-255, two accumulators",
                          "same operands, two accumulators"};
  for (int v = 0; v < 4; ++v) {
    k_probe_pairs<<<148, 128, 66 * 1024>>>(iters, v, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%s{\"variant\": \"%s\", \"cycles_per_mma\": %.1f, \"ideal\": 64, \"err\": \"%s\"}",
           v ? ",\n" : "", names[v], (double)c / iters / 8, cudaGetErrorString(e));
  }
  printf("\n]}\n");
  return 0;
}
