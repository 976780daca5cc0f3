// Microbenchmark (design probe): mma.sync m16n8k32 u8*s8->s32 and e4m3 vs
// m16n8k16 f16->f32 issue rate on sm_100a, per SM sub-partition.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_imma scripts/microbench_imma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void hmma(float* c, uint32_t a, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a), "r"(a ^ 1), "r"(a), "r"(a), "r"(b), "r"(b));
}
__device__ __forceinline__ void imma(int* c, uint32_t a, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a), "r"(a ^ 1), "r"(a), "r"(a), "r"(b), "r"(b));
}
__device__ __forceinline__ void qmma(float* c, uint32_t a, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a), "r"(a ^ 1), "r"(a), "r"(a), "r"(b), "r"(b));
}

template <int KIND, int CH>
__global__ void k(int iters, float* out, long long* cyc) {
  float f[CH][4] = {};
  int q[CH][4] = {};
  uint32_t a = threadIdx.x * 0x00010001u + 0x3c003c00u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (KIND == 0) hmma(f[c], a ^ c, a ^ i);
      else if (KIND == 1) imma(q[c], a ^ c, a ^ i);
      else qmma(f[c], a ^ c, a ^ i);
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += f[c][0] + f[c][3] + q[c][0] + q[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  long long h;
  const char* nm[3] = {"hmma m16n8k16 f16", "imma m16n8k32 u8s8", "qmma m16n8k32 e4m3"};
  for (int kind = 0; kind < 3; ++kind)
    for (int warps : {4, 8, 16})
      for (int ch : {1, 4}) {
        auto kern = kind == 0 ? (ch == 1 ? k<0, 1> : k<0, 4>)
                  : kind == 1 ? (ch == 1 ? k<1, 1> : k<1, 4>)
                              : (ch == 1 ? k<2, 1> : k<2, 4>);
        kern<<<148, warps * 32>>>(iters, out, cyc);
        kern<<<148, warps * 32>>>(iters, out, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const double per = double(h) / iters / ch;
        printf("%-20s warps/SM %2d chains %d: %6.2f cyc/mma/warp -> SMSP %.2f cyc/mma\n", nm[kind], warps,
               ch, per, per / ((warps + 3) / 4));
      }
  return 0;
}
