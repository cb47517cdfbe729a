// Throughput probes: POPC, mma.sync b1 and.popc, mma.sync s8, pinned H2D.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void k_popc(const uint32_t* in, uint32_t* out, int iters){
  uint32_t a = in[threadIdx.x & 31] ^ threadIdx.x, b = a*3+1, c=a*7+5, d=a*11+3;
  uint32_t s0=0,s1=0,s2=0,s3=0;
  for(int i=0;i<iters;i++){
    s0 += __popc(a & b); s1 += __popc(b & c); s2 += __popc(c & d); s3 += __popc(d & a);
    a += 1; b ^= s0; c += s1; d ^= s2;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x] = s0+s1+s2+s3;
}
__global__ void k_b1(uint32_t* out, int iters){
  uint32_t a0=threadIdx.x,a1=a0*3,a2=a0*5,a3=a0*7,b0=a0*9,b1=a0*11;
  int c[4][4]={{0}};
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[j][0]),"+r"(c[j][1]),"+r"(c[j][2]),"+r"(c[j][3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));
  }
  int s=0; for(int j=0;j<4;j++) for(int q=0;q<4;q++) s+=c[j][q];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_s8(uint32_t* out, int iters){
  uint32_t a0=threadIdx.x,a1=a0*3,a2=a0*5,a3=a0*7,b0=a0*9,b1=a0*11;
  int c[4][4]={{0}};
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[j][0]),"+r"(c[j][1]),"+r"(c[j][2]),"+r"(c[j][3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));
  }
  int s=0; for(int j=0;j<4;j++) for(int q=0;q<4;q++) s+=c[j][q];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *in,*out; CK(cudaMalloc(&in, 4096)); CK(cudaMemset(in,0x5a,4096)); CK(cudaMalloc(&out, 64<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int blocks = sms*8, threads=256, iters=1<<14;
  k_popc<<<blocks,threads>>>(in,out,16); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); k_popc<<<blocks,threads>>>(in,out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1);
  double n = 4.0*blocks*threads*(double)iters;
  printf("popc: %.3f ms, %.3f Tpopc/s, %.2f popc/clk/SM@1.9GHz\n", ms, n/ms/1e9, n/(ms*1e-3)/sms/1.9e9);
  k_b1<<<blocks,threads>>>(out,16); CK(cudaDeviceSynchronize());
  iters=1<<12;
  cudaEventRecord(e0); k_b1<<<blocks,threads>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1);
  n = 4.0*(blocks*threads/32)*(double)iters*16*8*256*2;
  printf("b1 mma.sync: %.3f ms, %.1f TOPS (and+popc as 2 ops)\n", ms, n/ms/1e9);
  k_s8<<<blocks,threads>>>(out,16); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); k_s8<<<blocks,threads>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1);
  n = 4.0*(blocks*threads/32)*(double)iters*16*8*32*2;
  printf("s8 mma.sync: %.3f ms, %.1f TOPS\n", ms, n/ms/1e9);
  // pinned H2D / D2H sweep
  size_t maxb = (size_t)1<<30; void* h; CK(cudaHostAlloc(&h, maxb, 0)); void* d; CK(cudaMalloc(&d, maxb));
  memset(h, 1, maxb);
  for (size_t b = 1<<16; b <= maxb; b <<= 2){
    cudaMemcpy(d,h,b,cudaMemcpyHostToDevice);
    int reps = b < (1<<24) ? 50 : 5;
    cudaEventRecord(e0); for(int r=0;r<reps;r++) cudaMemcpyAsync(d,h,b,cudaMemcpyHostToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1); double h2d = b*reps/ms/1e6;
    cudaEventRecord(e0); for(int r=0;r<reps;r++) cudaMemcpyAsync(h,d,b,cudaMemcpyDeviceToHost); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1); double d2h = b*reps/ms/1e6;
    printf("pinned %10zu B: H2D %.2f GB/s  D2H %.2f GB/s\n", b, h2d, d2h);
  }
  void* hp = malloc(maxb); memset(hp, 1, maxb);
  cudaEventRecord(e0); cudaMemcpy(d,hp,maxb,cudaMemcpyHostToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms,e0,e1); printf("pageable 1GiB H2D %.2f GB/s\n", maxb/ms/1e6);
  return 0;
}
