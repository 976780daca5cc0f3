// Microbenchmark (design probe): the K2 consumer step (attend<FMT,1,BPI>, the
// kernel's own code) on shared-memory-resident blocks, W warps per SM, no
// copies -- cycles per (block, head) per warp vs W.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -Iinclude
//      -Ipaper_2509_06261_b200/csrc --expt-relaxed-constexpr -o scripts/mb_consumer scripts/microbench_consumer.cu
#include <cstdio>
#include "../paper_2509_06261_b200/csrc/decode.cu"
using namespace kvslab;
using namespace kvslab::dev;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int FMT, int BPI>
__global__ void __maxnreg__(128) bench(int iters, float* out, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using Gm = Geo<FMT>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  constexpr uint32_t HG = 8;
  const uint32_t kvq = HG * Gm::kChunk, pq = HG * Gm::kParam;
  const uint32_t stage = (2 * kvq + 2 * pq + 127) / 128 * 128;
  const uint32_t qoff = 2 * stage, total = qoff + HG * 4 * kD * 2;
  for (uint32_t i = threadIdx.x; i < total / 4; i += blockDim.x) {
    uint32_t v = hsh(i * 2654435761u + 17);
    const bool half_data = (FMT == kFP16 && i * 4 < 2 * stage) || i * 4 >= qoff;
    if (half_data) v = (v & 0x83ff83ffu) | 0x30003000u;            // |x| < 1 halves
    else if (FMT == kFP8) v &= 0xbfbfbfbfu;                          // no NaN
    else if (Gm::kParam > 0 && (i * 4) % stage >= 2 * kvq) v = (v & 0x03ff03ffu) | 0x30003000u;
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  __syncthreads();
  const uint32_t base = smem_u32(smem);
  const uint32_t head = warp % HG;
  uint32_t qf[1][8][2];
  load_q_frags<FMT, 1>(base + qoff + head * 4 * kD * 2, g, t, 4, qf);
  float qsb[1][2] = {{0.1f, 0.2f}}, qst[1][2] = {{0.3f, 0.1f}};
  const FragOff fo = make_offsets<FMT>(g, t);
  UnitState<1> us;
  for (int mt = 0; mt < 8; ++mt) us.acc[mt][0][0] = us.acc[mt][0][1] = us.acc[mt][0][2] = us.acc[mt][0][3] = 0.f;
  us.m[0][0] = us.m[0][1] = -INFINITY;
  us.l[0][0] = us.l[0][1] = us.zb[0][0] = us.zb[0][1] = us.zz[0][0] = us.zz[0][1] = 0.f;
  const uint32_t wK = head * Gm::kChunk, wP = 2 * kvq + head * Gm::kParam;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < iters; i += BPI) {
    uint32_t sbs[BPI];
    int valid[BPI];
#pragma unroll
    for (int b = 0; b < BPI; ++b) {
      sbs[b] = base + ((i + b) & 1) * stage;
      valid[b] = 16;
    }
    attend<FMT, 1, BPI>(us, sbs, valid, wK, wP, kvq, pq, fo, qf, qsb, qst, 1.f, 0.125f, g, t);
  }
  const long long t1 = clock64();
  float s = us.l[0][0] + us.zb[0][1] + us.zz[0][0];
  for (int mt = 0; mt < 8; ++mt) s += us.acc[mt][0][0] + us.acc[mt][0][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int FMT, int BPI>
void run(const char* name) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int smem = 200 * 1024, iters = 2048;
  cudaFuncSetAttribute(bench<FMT, BPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    bench<FMT, BPI><<<148, w * 32, smem>>>(iters, out, cyc);
    bench<FMT, BPI><<<148, w * 32, smem>>>(iters, out, cyc);
    long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double m = 0;
    for (long long v : h) m += v;
    m /= 148;
    const double per = m / iters;  // cycles per block per warp
    printf("%-5s BPI %d warps/SM %2d: %7.1f cyc/block/warp  -> %6.1f cyc per block-head per SM  (%s)\n",
           name, BPI, w, per, per / w, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<kFP16, 1>("FP16");
  run<kFP8, 1>("FP8");
  run<kINT8, 1>("INT8");
  run<kINT4, 1>("INT4");
  run<kINT4, 2>("INT4");
  run<kFP8, 2>("FP8");
  return 0;
}
