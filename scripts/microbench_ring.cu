// microbench_ring.cu -- one producer warp per CTA feeding a shared ring of
// large bulk copies to 8 consumer warps (the K2 structure), no math.
// Sweeps total bytes per launch to separate fixed cost from streaming rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_ring scripts/microbench_ring.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" :: "r"(su(b)), "r"(ph) : "memory");
}
__global__ void ring(const uint8_t* base, const uint32_t* ids, uint32_t n, uint32_t stage, uint32_t ncopy,
                     uint32_t S, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[32], empty[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NC = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(&empty[i])), "r"(NC));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t s0 = (uint64_t)blockIdx.x * n / gridDim.x, s1 = (uint64_t)(blockIdx.x + 1) * n / gridDim.x;
  const uint32_t piece = stage / ncopy;
  if (warp == NC) {
    uint32_t st = 0, ph = 0;
    for (uint32_t k = s0; k < s1; ++k) {
      wait(&empty[st], ph ^ 1);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[st])), "r"(stage) : "memory");
        for (uint32_t c = 0; c < ncopy; ++c) {
          const uint8_t* src = base + ((uint64_t)ids[k] * ncopy + c) * piece;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(su(sm + st * stage + c * piece)), "l"(src), "r"(piece), "r"(su(&full[st])) : "memory");
        }
      }
      if (++st == S) { st = 0; ph ^= 1; }
    }
    return;
  }
  uint32_t acc = 0, st = 0, ph = 0;
  for (uint32_t k = s0; k < s1; ++k) {
    wait(&full[st], ph);
    acc += *reinterpret_cast<const uint32_t*>(sm + st * stage + warp * 64 + lane * 4);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(&empty[st])) : "memory");
    if (++st == S) { st = 0; ph ^= 1; }
  }
  if (acc == 0x1234567) atomicAdd(sink, 1ull);
}
int main() {
  const size_t bytes = 8ull << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  unsigned long long* sink; CK(cudaMalloc(&sink, 8));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  std::mt19937 rng(3);
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (uint32_t stage : {8192u, 17408u, 32768u, 65536u}) {
    for (uint32_t ncopy : {1u, 2u, 4u}) {
      const uint32_t S = (200 * 1024) / stage;
      for (size_t total : {36ull << 20, 68ull << 20, 136ull << 20, 1ull << 30}) {
        const uint32_t n = total / stage;
        std::vector<uint32_t> ids(n);
        for (auto& x : ids) x = rng() % (uint32_t)(bytes / stage);
        uint32_t* d; CK(cudaMalloc(&d, n * 4)); CK(cudaMemcpy(d, ids.data(), n * 4, cudaMemcpyHostToDevice));
        auto go = [&] { ring<<<sms, 9 * 32, S * stage>>>(buf, d, n, stage, ncopy, S, sink); };
        go(); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a)); for (int r = 0; r < 10; ++r) go(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        printf("stage %6u copies %u S %2u total %5zu MB: %7.2f us  %6.0f GB/s\n", stage, ncopy, S, total >> 20,
               ms * 100, (double)n * stage * 10 / (ms / 1e3) / 1e9);
        CK(cudaFree(d));
      }
    }
  }
}
