// microbench_ex2.cu -- exp2 throughput per SM on B200: MUFU ex2.approx.f32
// versus ex2.approx.f16x2 (two results per lane per instruction?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_ex2 scripts/microbench_ex2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
__global__ void ex2_f32(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.1f, c = a + 0.2f, d = a + 0.3f;
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void ex2_f16x2(float* out, int iters) {
  uint32_t a = 0x3c003c00u + threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(b));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(c));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(d));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = __half2float(__ushort_as_half((unsigned short)(a ^ b ^ c ^ d)));
}
int main() {
  float* out; cudaMalloc(&out, 148 * 1024 * 4 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int k = 0; k < 2; ++k) {
    auto run = [&](auto kern, const char* name, double per_inst) {
      kern<<<148 * 4, 256>>>(out, iters); cudaDeviceSynchronize();
      cudaEventRecord(e0); kern<<<148 * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double insts = 148.0 * 4 * 256 * iters * 4;  // thread-level instructions
      const double clk = 1.9e9;
      printf("%-10s %.3f ms  %.1f thread-insts/clk/SM  %.1f exp2 results/clk/SM\n", name, ms,
             insts / (ms * 1e-3) / clk / 148, insts * per_inst / (ms * 1e-3) / clk / 148);
    };
    run(ex2_f32, "f32", 1.0);
    run(ex2_f16x2, "f16x2", 2.0);
  }
  cudaFree(out);
}
