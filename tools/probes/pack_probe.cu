// pack_probe.cu — bandwidth probe for the binarize + bit-pack transform (config 5).
//
// Times transform variants on one raster already in HBM, with a cold L2 for every rep
// (256 MiB memset between reps, outside the events), and prints GB/s of raster
// (w*h / t) and the HBM fraction of the 1.125 B/px algorithmic traffic.  Variants:
//   vec      : the library's k_pack_vec (8 x 16-B loads per lane, persistent grid)
//   vec_l2   : same with the .L2::256B prefetch hint on every load
//   wide     : 16 x 16-B loads per lane (8 KB per warp iteration)
//   flat     : one 4 KB block per warp, no loop (grid = blocks / 8)
//   flat_l2  : flat + .L2::256B
//   readonly : the same loads with no packing and one store per warp (read ceiling)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pack_probe pack_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, \
                  __LINE__);                                                   \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

template <bool L2HINT>
__device__ __forceinline__ uint4 ldv(const void *p) {
  uint4 r;
  if (L2HINT)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t nz_nibble(uint32_t x) {
  uint32_t t = ((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x;
  t = (t >> 7) & 0x01010101u;
  return (t * 0x00204081u) >> 21 & 0xFu;
}
__device__ __forceinline__ uint32_t nz16(uint4 v) {
  return nz_nibble(v.x) | (nz_nibble(v.y) << 4) | (nz_nibble(v.z) << 8) | (nz_nibble(v.w) << 12);
}

template <int NV, bool L2HINT, bool READONLY>
__global__ void __launch_bounds__(256) k_loop(const uint8_t *__restrict__ src, uint64_t nblk,
                                              uint32_t *__restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; b < nblk; b += nw) {
    const uint8_t *base = src + b * (NV * 512) + lane * 16;
    uint4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = ldv<L2HINT>(base + i * 512);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (READONLY) {
        acc ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
      } else {
        const uint32_t h = nz16(v[i]);
        const uint32_t o = __shfl_xor_sync(0xffffffffu, h, 1);
        if ((lane & 1) == 0) dst[b * (NV * 16) + i * 16 + (lane >> 1)] = h | (o << 16);
      }
    }
  }
  if (READONLY && acc == 0x12345678u) dst[0] = acc;
}

template <bool L2HINT>
__global__ void __launch_bounds__(256) k_flat(const uint8_t *__restrict__ src, uint64_t nblk,
                                              uint32_t *__restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (b >= nblk) return;
  const uint8_t *base = src + b * 4096 + lane * 16;
  uint4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = ldv<L2HINT>(base + i * 512);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t h = nz16(v[i]);
    const uint32_t o = __shfl_xor_sync(0xffffffffu, h, 1);
    if ((lane & 1) == 0) dst[b * 128 + i * 16 + (lane >> 1)] = h | (o << 16);
  }
}

int main(int argc, char **argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double hbm = argc > 1 ? std::atof(argv[1]) : 6550.4;
  const int sizes[][2] = {{16384, 16384}, {16012, 14512}, {14512, 16012}, {12288, 12288},
                          {10512, 12512}, {8192, 8192}};
  uint8_t *src;
  uint32_t *dst;
  void *flush;
  const size_t maxp = 16384ull * 16384;
  CK(cudaMalloc(&src, maxp));
  CK(cudaMalloc(&dst, maxp / 8 + 4096));
  CK(cudaMalloc(&flush, 256ull << 20));
  CK(cudaMemset(src, 0x01, maxp));
  std::printf("{\"probe\": \"pack\", \"hbm_gbs\": %.1f, \"rows\": [\n", hbm);
  bool first = true;
  for (auto &sz : sizes) {
    const uint64_t P = (uint64_t)sz[0] * sz[1];
    const uint64_t nblk = P / 4096;
    struct V {
      const char *name;
      int kind;
    } vs[] = {{"vec", 0}, {"vec_l2", 1}, {"wide", 2}, {"wide_l2", 3}, {"flat", 4},
              {"flat_l2", 5}, {"readonly", 6}, {"vec_occ", 7}};
    for (auto &v : vs) {
      float best = 1e30f, tot = 0.f;
      const int reps = 6;
      for (int r = 0; r < reps + 1; ++r) {
        CK(cudaMemsetAsync(flush, r, 256ull << 20));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0));
        switch (v.kind) {
          case 0: k_loop<8, false, false><<<sms * 8, 256>>>(src, nblk, dst); break;
          case 1: k_loop<8, true, false><<<sms * 8, 256>>>(src, nblk, dst); break;
          case 2: k_loop<16, false, false><<<sms * 8, 256>>>(src, nblk / 2, dst); break;
          case 3: k_loop<16, true, false><<<sms * 8, 256>>>(src, nblk / 2, dst); break;
          case 4: k_flat<false><<<(unsigned)((nblk + 7) / 8), 256>>>(src, nblk, dst); break;
          case 5: k_flat<true><<<(unsigned)((nblk + 7) / 8), 256>>>(src, nblk, dst); break;
          case 6: k_loop<8, false, true><<<sms * 8, 256>>>(src, nblk, dst); break;
          case 7: k_loop<8, true, false><<<sms * 16, 256>>>(src, nblk, dst); break;
        }
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (r > 0) {
          best = ms < best ? ms : best;
          tot += ms;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
      }
      const double mean_us = tot / reps * 1e3;
      const double rate = P / (mean_us * 1e-6) / 1e9;
      std::printf("%s{\"w\": %d, \"h\": %d, \"variant\": \"%s\", \"us_mean\": %.2f, \"us_best\": %.2f, "
                  "\"raster_gbs\": %.1f, \"hbm_frac\": %.4f}",
                  first ? "" : ",\n", sz[0], sz[1], v.name, mean_us, best * 1e3, rate,
                  rate * 1.125 / hbm);
      first = false;
    }
  }
  std::printf("\n]}\n");
  return 0;
}
