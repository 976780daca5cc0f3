// microbench_tma.cu -- the K2 ring (one producer warp, S-deep ring of bulk
// copies, 8 consumer warps) with K2's copy details toggled one at a time:
// L2 evict_first cache hint, 32832-byte stages at a 64-byte offset (FP8 layer
// sub-blocks), consumer work per stage (spin), on 111 / 148 CTAs, 67 MB.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_tma scripts/microbench_tma.cu
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
__global__ void ring(const uint8_t* base, const uint32_t* ids, uint32_t n, uint32_t stage, uint32_t slot,
                     uint32_t off, uint32_t S, int hint, uint32_t spin, unsigned long long* sink, uint32_t gstride) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[64], empty[64];
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
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (warp == NC) {
    uint32_t st = 0, ph = 0;
    for (uint32_t k = s0; k < s1; ++k) {
      wait(&empty[st], ph ^ 1);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[st])), "r"(stage) : "memory");
        const uint8_t* src = base + (uint64_t)ids[k] * gstride + off;
        if (hint)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       :: "r"(su(sm + st * slot)), "l"(src), "r"(stage), "r"(su(&full[st])), "l"(pol) : "memory");
        else
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(su(sm + st * slot)), "l"(src), "r"(stage), "r"(su(&full[st])) : "memory");
      }
      if (++st == S) { st = 0; ph ^= 1; }
    }
    return;
  }
  uint32_t acc = 0, st = 0, ph = 0;
  for (uint32_t k = s0; k < s1; ++k) {
    wait(&full[st], ph);
    acc += *reinterpret_cast<const uint32_t*>(sm + st * slot + warp * 64 + lane * 4);
    if (spin) { const long long t = clock64(); while (clock64() - t < spin) {} }
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
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  std::mt19937 rng(3);
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  struct V { const char* name; uint32_t stage, slot, off; int hint; uint32_t spin; int k2 = 0; uint32_t gs = 0; };
  const V vs[] = {{"32768 plain", 32768, 32768, 0, 0, 0},
                  {"32768 evict_first", 32768, 32768, 0, 1, 0},
                  {"32832 @64 (FP8 layer)", 32832, 32896, 64, 0, 0},
                  {"32832 @64 evict_first", 32832, 32896, 64, 1, 0},
                  {"32832 @64 ef spin 800", 32832, 32896, 64, 1, 800},
                  {"32832 @64 ef spin 400", 32832, 32896, 64, 1, 400},
                  // K2's own pattern: block b of 32 layers (1050624 B), layer 5's sub-block
                  {"K2 seq blocks L5", 32832, 32896, 5 * 32832, 1, 0, 1, 1050624},
                  {"K2 rand blocks L5", 32832, 32896, 5 * 32832, 1, 0, 2, 1050624},
                  {"K2 seq blocks L5 spin", 32832, 32896, 5 * 32832, 1, 800, 1, 1050624}};
  for (const V& v : vs)
    for (int grid : {111, 148})
      for (size_t total : {67ull << 20, 1ull << 30}) {
        if (v.k2 && total > (1ull << 30) / 2) continue;
        if (v.k2 && (uint64_t)(total / v.stage) * 1050624 > bytes) continue;
        const uint32_t S = 6;
        const uint32_t n = total / v.stage;
        std::vector<uint32_t> ids(n);
        // random distinct-ish stage slots over 8 GB (>> L2); K2: 16 sequences'
        // consecutive blocks (1), or random blocks (2)
        const uint32_t gs = v.gs ? v.gs : v.slot;
        const uint32_t nslots = (uint32_t)(bytes / gs - 1);
        for (uint32_t i = 0; i < n; ++i)
          ids[i] = v.k2 == 1 ? (i + (uint32_t)(rng() % 4096) * 0) % nslots : rng() % nslots;
        if (v.k2 == 1) { const uint32_t start = rng() % (nslots - n); for (uint32_t i = 0; i < n; ++i) ids[i] = start + i; }
        uint32_t* d; CK(cudaMalloc(&d, n * 4)); CK(cudaMemcpy(d, ids.data(), n * 4, cudaMemcpyHostToDevice));
        auto go = [&] { ring<<<grid, 9 * 32, S * v.slot>>>(buf, d, n, v.stage, v.slot, v.off, S, v.hint, v.spin, sink, gs); };
        go(); CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a)); for (int r = 0; r < 10; ++r) go(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        const double gbs = (double)n * v.stage * 10 / (ms / 1e3) / 1e9;
        printf("%-24s grid %3d total %5zu MB: %8.2f us/launch %6.0f GB/s %5.1f GB/s/SM\n", v.name, grid, total >> 20,
               ms * 100, gbs, gbs / grid);
        CK(cudaFree(d));
      }
}
