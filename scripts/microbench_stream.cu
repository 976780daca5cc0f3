// microbench_stream.cu -- how fast can one B200 stream scattered KV chunks?
// (design probe for K2; not part of the product)
//   tma: per-warp ring of STAGES cp.async.bulk copies of CHUNK bytes (lane 0
//        issues, mbarrier completion), no compute
//   ldg: each warp reads CHUNK bytes with 16-byte ld.global.nc, UNROLL deep
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_stream.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES>
__global__ void tma_stream(const uint8_t* base, const uint32_t* chunk_ids, uint32_t nchunks,
                           uint32_t chunk, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  uint8_t* ring = sm + (size_t)warp * STAGES * chunk;
  __shared__ uint64_t bars[32 * 16];
  uint64_t* bar = bars + warp * 16;
  const uint32_t W = gridDim.x * wpc, wid = blockIdx.x * wpc + warp;
  const uint32_t s = (uint64_t)wid * nchunks / W, e = (uint64_t)(wid + 1) * nchunks / W;
  const uint32_t n = e - s;
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](uint32_t i) {
    if (lane == 0) {
      const uint32_t st = i % STAGES;
      const uint8_t* src = base + (uint64_t)chunk_ids[s + i] * chunk;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[st])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(ring + st * chunk)), "l"(src), "r"(chunk), "r"(smem_u32(&bar[st])) : "memory");
    }
  };
  for (uint32_t i = 0; i < STAGES && i < n; ++i) issue(i);
  uint32_t acc = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t st = i % STAGES;
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                 :: "r"(smem_u32(&bar[st])), "r"((i / STAGES) & 1) : "memory");
    acc += *reinterpret_cast<const uint32_t*>(ring + st * chunk + lane * 4);
    __syncwarp();
    if (i + STAGES < n) issue(i + STAGES);
  }
  if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

template <int UNROLL>
__global__ void ldg_stream(const uint8_t* base, const uint32_t* chunk_ids, uint32_t nchunks,
                           uint32_t chunk, unsigned long long* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  const uint32_t W = gridDim.x * wpc, wid = blockIdx.x * wpc + warp;
  uint32_t acc = 0;
  const uint32_t per_chunk = chunk / 512;  // 16 B x 32 lanes
  for (uint32_t c = wid; c < nchunks; c += W) {
    const uint4* src = reinterpret_cast<const uint4*>(base + (uint64_t)chunk_ids[c] * chunk) + lane;
    uint4 v[UNROLL];
    for (uint32_t j = 0; j < per_chunk; j += UNROLL) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(src + (j + u) * 32);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc += v[u].x ^ v[u].w;
    }
  }
  if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = 8ull << 30;
  uint8_t* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937 rng(1);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (uint32_t chunk : {1024u, 2048u, 4096u, 8192u}) {
    const uint32_t total_chunks = bytes / chunk;
    const uint32_t n = (uint32_t)((1ull << 30) / chunk);  // 1 GiB per launch
    std::vector<uint32_t> ids(n);
    for (auto& x : ids) x = rng() % total_chunks;
    uint32_t* d_ids;
    CK(cudaMalloc(&d_ids, n * 4));
    CK(cudaMemcpy(d_ids, ids.data(), n * 4, cudaMemcpyHostToDevice));
    auto timeit = [&](auto launch, const char* name, int cfg1, int cfg2) {
      launch();
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a));
      for (int r = 0; r < 5; ++r) launch();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("%-4s chunk %5u  cfg %3d %3d : %7.1f GB/s\n", name, chunk, cfg1, cfg2,
             5.0 * n * chunk / (ms / 1e3) / 1e9);
    };
    for (int warps : {4, 8}) {
      for (int stages : {2, 4, 8}) {
        size_t smem = (size_t)warps * stages * chunk;
        if (smem > 200 * 1024) continue;
        auto run = [&](auto kern) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          int per_sm = 0;
          CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem));
          timeit([&] { kern<<<per_sm * sms, warps * 32, smem>>>(buf, d_ids, n, chunk, sink); }, "tma",
                 per_sm * warps, stages);
        };
        if (stages == 2) run(tma_stream<2>);
        if (stages == 4) run(tma_stream<4>);
        if (stages == 8) run(tma_stream<8>);
      }
    }
    if (chunk >= 512 * 4) {
      for (int blocks_per_sm : {4, 8, 16}) {
        timeit([&] { ldg_stream<4><<<blocks_per_sm * sms, 256>>>(buf, d_ids, n, chunk, sink); }, "ldg",
               blocks_per_sm * 8, 4);
      }
    }
    CK(cudaFree(d_ids));
  }
  return 0;
}
