// Microbenchmark (design probe): mma.sync m16n8k16 f16->f32 throughput and
// latency on sm_100a, per SM sub-partition, vs warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_mma scripts/microbench_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                    uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CH>  // CH independent accumulator chains per warp
__global__ void k_mma(int iters, float* out, long long* cyc) {
  float acc[CH][4] = {};
  uint32_t a = threadIdx.x * 0x00010001u + 0x3c003c00u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma(acc[c], a, a ^ c, a, a, a, a ^ i);
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_lop3(int iters, uint32_t* out, long long* cyc) {
  uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * (c + 1);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t r;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(r) : "r"(x[c]), "r"(0x000f000fu), "r"(x[(c + 1) & 7]));
      x[c] = r;
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  uint32_t* outu;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&outu, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  long long h;
  for (int warps : {1, 4, 8, 16}) {
    for (int ch : {1, 2, 4, 8}) {
      auto kern = ch == 1 ? k_mma<1> : ch == 2 ? k_mma<2> : ch == 4 ? k_mma<4> : k_mma<8>;
      kern<<<148, warps * 32>>>(iters, out, cyc);
      kern<<<148, warps * 32>>>(iters, out, cyc);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double per = double(h) / iters / ch;  // cycles per mma per warp
      printf("mma  warps/SM %2d chains %d: %.2f cyc/mma/warp  -> SM-subpartition rate %.2f cyc/mma\n",
             warps, ch, per, per / ((warps + 3) / 4));
    }
    k_lop3<<<148, warps * 32>>>(iters, outu, cyc);
    k_lop3<<<148, warps * 32>>>(iters, outu, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = double(h) / iters / 8;
    printf("lop3 warps/SM %2d (8 chains): %.2f cyc/op/warp -> sub-partition %.2f cyc/op\n", warps, per,
           per / ((warps + 3) / 4));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
