// tma_probe.cu — raw-ring TMA streaming rate on one B200 (the fused recompute's skeleton).
//
// 148 CTAs (one per SM) stream a 2 GiB buffer laid out like the packed masks of C2
// (tile-interleaved: per 1024-px tile, 256 mask rows x 128 B, contiguous) through an
// SMEM ring of `depth` slots with 3-D TMA boxes {32 words, rows, tiles}; one thread issues,
// the slot is released as soon as it lands (no consumer work).  Prints TB/s per shape.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(phase));
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap *m, int c0, int c1, int c2,
                                     uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// unit = `rows` mask rows x `tiles` tiles; 256 / rows boxes cover one tile's 256 rows
__global__ void __launch_bounds__(32, 1) k_stream(const __grid_constant__ CUtensorMap tm,
                                                  int ntiles, int rows, int tiles, int depth) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[16];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  const uint32_t unit_bytes = (uint32_t)rows * 128u * (uint32_t)tiles;
  const int per_tile = 256 / rows;
  const int units_total = ntiles / tiles * per_tile;
  const int per_cta = (units_total + gridDim.x - 1) / gridDim.x;
  const int u0 = blockIdx.x * per_cta;
  const int u1 = min(u0 + per_cta, units_total);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < depth; ++i) mbar_init(&bars[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int u = u0; u < u1; ++u) {
    const int i = u - u0, slot = i % depth;
    if (i >= depth) mbar_wait(&bars[slot], (uint32_t)(((i / depth) - 1) & 1));
    mbar_expect(&bars[slot], unit_bytes);
    const int tile0 = (u / per_tile) * tiles, row0 = (u % per_tile) * rows;
    tma3(base + slot * unit_bytes, &tm, 0, row0, tile0, &bars[slot]);
  }
  for (int i = max(0, (u1 - u0) - depth); i < u1 - u0; ++i)
    mbar_wait(&bars[i % depth], (uint32_t)((i / depth) & 1));
}

int main() {
  const int ntiles = 65536;  // 2^26 px per mask, 256 masks: 2 GiB
  const size_t bytes = (size_t)ntiles * 256 * 128;
  void *buf = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMemset(buf, 0x5a, bytes);
  CUresult (*encode)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                     const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                     CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                     CUtensorMapFloatOOBfill) = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Shape { int rows, tiles, depth; };
  const Shape shapes[] = {{256, 1, 4}, {256, 1, 2}, {256, 1, 6}, {128, 1, 8}, {64, 1, 16},
                          {256, 2, 2}, {256, 2, 3}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"probe\": \"TMA raw-ring streaming, 148 CTAs, 2 GiB packed tiles\", \"rows\": [\n");
  bool first = true;
  for (const Shape &sh : shapes) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {32, 256, (cuuint64_t)ntiles};
    cuuint64_t strides[2] = {128, 256 * 128};
    cuuint32_t box[3] = {32, (cuuint32_t)sh.rows, (cuuint32_t)sh.tiles};
    cuuint32_t estr[3] = {1, 1, 1};
    if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, buf, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      continue;
    const int smem = sh.rows * 128 * sh.tiles * sh.depth + 1024;
    if (smem > 200 * 1024) continue;
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      k_stream<<<148, 32, smem>>>(tm, ntiles, sh.rows, sh.tiles, sh.depth);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%s{\"box_rows\": %d, \"box_tiles\": %d, \"depth\": %d, \"in_flight_kb\": %d, "
           "\"ms\": %.4f, \"tb_s\": %.2f, \"err\": \"%s\"}",
           first ? "" : ",\n", sh.rows, sh.tiles, sh.depth, sh.rows * 128 * sh.tiles * sh.depth / 1024,
           best, bytes / best / 1e9, cudaGetErrorString(cudaGetLastError()));
    first = false;
  }
  printf("\n]}\n");
  return 0;
}
