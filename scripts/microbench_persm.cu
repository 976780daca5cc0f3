// microbench_persm.cu -- (1) per-SM streaming rate of the K2 ring structure
// (one producer warp, bulk copies into an S-deep ring, 8 consumer warps that
// only touch the data) as a function of the number of SMs streaming and the
// bytes in flight per SM; (2) whether a PDL chain A -> B -> C lets C start
// before A completes (C on SMs A leaves free).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_persm scripts/microbench_persm.cu
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
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void ring(const uint8_t* base, const uint32_t* ids, uint32_t n, uint32_t stage, uint32_t S,
                     unsigned long long* sink) {
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
  if (warp == NC) {
    uint32_t st = 0, ph = 0;
    for (uint32_t k = s0; k < s1; ++k) {
      wait(&empty[st], ph ^ 1);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[st])), "r"(stage) : "memory");
        const uint8_t* src = base + (uint64_t)ids[k] * stage;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su(sm + st * stage)), "l"(src), "r"(stage), "r"(su(&full[st])) : "memory");
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

// PDL chain probe: big CTAs (200 KB smem) spin `spin_ns`, stamp start/end.
__global__ void big(unsigned long long* tr, uint32_t spin_ns, int slot) {
  extern __shared__ uint8_t sm[];
  asm volatile("griddepcontrol.launch_dependents;");
  const uint64_t t0 = gt();
  if (threadIdx.x == 0) tr[slot * 1024 + blockIdx.x * 2] = t0;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  while (gt() - t0 < spin_ns) {}
  if (threadIdx.x == 0) { sm[0] = 1; tr[slot * 1024 + blockIdx.x * 2 + 1] = gt(); }
}
__global__ void small(unsigned long long* tr, int slot) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) tr[slot * 1024 + blockIdx.x * 2] = gt();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) tr[slot * 1024 + blockIdx.x * 2 + 1] = gt();
}

int main() {
  const size_t bytes = 8ull << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  unsigned long long* sink; CK(cudaMalloc(&sink, 8));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  std::mt19937 rng(3);
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (uint32_t stage : {16384u, 32768u, 65536u}) {
    for (uint32_t S : {2u, 3u, 6u, 12u}) {
      if (S * stage > 200 * 1024) continue;
      for (int grid : {18, 37, 74, 111, 148}) {
        const size_t total = 1ull << 30;
        const uint32_t n = total / stage;
        std::vector<uint32_t> ids(n);
        for (auto& x : ids) x = rng() % (uint32_t)(bytes / stage);
        uint32_t* d; CK(cudaMalloc(&d, n * 4)); CK(cudaMemcpy(d, ids.data(), n * 4, cudaMemcpyHostToDevice));
        auto go = [&] { ring<<<grid, 9 * 32, S * stage>>>(buf, d, n, stage, S, sink); };
        go(); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a)); for (int r = 0; r < 5; ++r) go(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        const double gbs = (double)n * stage * 5 / (ms / 1e3) / 1e9;
        printf("stage %6u S %2u inflight %4u KB grid %3d: %7.0f GB/s  %5.1f GB/s per SM\n", stage, S,
               S * stage / 1024, grid, gbs, gbs / grid);
        CK(cudaFree(d));
      }
    }
  }
  // PDL chain
  unsigned long long* tr; CK(cudaMalloc(&tr, 8 * 1024 * 8)); CK(cudaMemset(tr, 0, 8 * 1024 * 8));
  CK(cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  auto launch_big = [&](int grid, int slot, bool pdl) {
    cudaLaunchConfig_t c{}; c.gridDim = dim3(grid); c.blockDim = dim3(288); c.dynamicSmemBytes = 200 * 1024;
    c.stream = s; c.attrs = at; c.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&c, big, tr, 20000u, slot));
  };
  auto launch_small = [&](int slot) {
    cudaLaunchConfig_t c{}; c.gridDim = dim3(128); c.blockDim = dim3(128); c.stream = s; c.attrs = at; c.numAttrs = 1;
    CK(cudaLaunchKernelEx(&c, small, tr, slot));
  };
  for (int variant = 0; variant < 2; ++variant) {
    CK(cudaMemset(tr, 0, 8 * 1024 * 8));
    CK(cudaDeviceSynchronize());
    launch_big(111, 0, false);
    if (variant == 1) launch_small(1);
    launch_big(111, 2, true);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(8 * 1024);
    CK(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long base = ~0ull, a_end = 0, c_min = ~0ull, c_max = 0;
    for (int i = 0; i < 111; ++i) { base = std::min(base, h[i * 2]); a_end = std::max(a_end, h[i * 2 + 1]); }
    for (int i = 0; i < 111; ++i) { c_min = std::min(c_min, h[2048 + i * 2]); c_max = std::max(c_max, h[2048 + i * 2]); }
    printf("PDL %s: A ends %.2f us; C CTAs start %.2f .. %.2f us\n", variant ? "A -> small -> C" : "A -> C",
           (a_end - base) / 1e3, (c_min - base) / 1e3, (c_max - base) / 1e3);
  }
}
