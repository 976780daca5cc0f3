// microbench_umma.cu -- design probe for a tcgen05 (UMMA) path: one CTA
// computes D[128][N] = A[128][128] . B[N][128]^T with A and B in shared memory
// (K-major, 128-byte swizzle), D in tensor memory, read back with tcgen05.ld,
// and checks it against the host; then times back-to-back MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/mb_umma scripts/microbench_umma.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cmath>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int M = 128, K = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major, 128B-swizzled operand: rows of 64 elements (128 B) per atom column;
// atom column j (elements 64j..64j+63) of all rows is a [rows][128 B] region.
__device__ __forceinline__ uint32_t sw128_off(int row, int k, int rows) {
  const int j = k / 64, kk = k % 64;
  const int gran = kk / 8, within = (kk % 8) * 2;
  return j * rows * 128 + row * 128 + (((gran ^ (row & 7)) * 16) | within);
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);     // start address
  d |= static_cast<uint64_t>(1) << 16;                    // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(sbo >> 4) << 32;             // SBO: 8-row group stride
  d |= static_cast<uint64_t>(1) << 46;                    // version (sm100)
  d |= static_cast<uint64_t>(2) << 61;                    // SWIZZLE_128B
  return d;
}

template <int N>
__global__ void umma_kernel(const __half* A, const __half* B, float* D, int reps, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + M * K * 2;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sA + sw128_off(r, k, M)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + sw128_off(r, k, N)) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(N >= 32 ? N : 32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
  const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
  uint32_t phase = 0;
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (rep == 1) t0 = clock64();
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < K / 16; ++k) {
        const uint32_t aoff = (k / 4) * M * 128 + (k % 4) * 32;
        const uint32_t boff = (k / 4) * N * 128 + (k % 4) * 32;
        const uint64_t ad = make_desc(a0 + aoff, 1024), bd = make_desc(b0 + boff, 1024);
        const uint32_t acc = k > 0 ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&mbar))
                   : "memory");
    }
    // wait for the MMAs
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT;\n\t}\n" ::"r"(smem_u32(&mbar)),
        "r"(phase));
    phase ^= 1;
  }
  if (tid == 0 && reps > 1) *cycles = clock64() - t0;
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // thread t (warp w) reads TMEM lane 32w + lane, columns 0..N-1
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) D[row * N + c0 + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N >= 32 ? N : 32));
}

template <int N>
static void run() {
  std::vector<__half> a(M * K), b(N * K);
  std::vector<float> af(M * K), bf(N * K), ref(M * N), got(M * N);
  srand(1);
  for (int i = 0; i < M * K; ++i) { af[i] = (rand() % 2001 - 1000) / 1000.f; a[i] = __float2half(af[i]); af[i] = __half2float(a[i]); }
  for (int i = 0; i < N * K; ++i) { bf[i] = (rand() % 2001 - 1000) / 1000.f; b[i] = __float2half(bf[i]); bf[i] = __half2float(b[i]); }
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += static_cast<double>(af[m * K + k]) * bf[n * K + k];
      ref[m * N + n] = static_cast<float>(s);
    }
  __half *dA, *dB;
  float* dD;
  long long* dc;
  CK(cudaMalloc(&dA, a.size() * 2));
  CK(cudaMalloc(&dB, b.size() * 2));
  CK(cudaMalloc(&dD, got.size() * 4));
  CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dA, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
  const int smem = (M + N) * K * 2 + 1024;
  CK(cudaFuncSetAttribute(umma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  umma_kernel<N><<<1, 128, smem>>>(dA, dB, dD, 1, dc);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  for (int i = 0; i < M * N; ++i) maxerr = fmax(maxerr, fabs(got[i] - ref[i]));
  printf("N=%d: max |D - ref| = %.3e  (D[0]=%f ref %f, D[last]=%f ref %f)\n", N, maxerr, got[0], ref[0],
         got[M * N - 1], ref[M * N - 1]);
  const int reps = 1001;
  umma_kernel<N><<<1, 128, smem>>>(dA, dB, dD, reps, dc);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  const double flop = 2.0 * M * N * K;
  printf("N=%d: %.1f cycles per 128x%dx128 MMA group (incl. commit+wait), %.0f FLOP/cycle/SM\n", N,
         static_cast<double>(cyc) / (reps - 1), N, flop / (static_cast<double>(cyc) / (reps - 1)));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}

// PV shape: D[128][128] = P[128][64] . V[64][128]; P K-major (one 64-token
// atom column), V token-major = MN-major B: [64-dim column j][token][128 B],
// LBO = 64 tokens * 128 B between the two dim columns, SBO = 1024 B per
// 8-token group; each K=16 step advances V by 16 tokens * 128 B.
__device__ __forceinline__ uint64_t make_desc2(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(lbo >> 4) << 16;
  d |= static_cast<uint64_t>(sbo >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__global__ void pv_kernel(const __half* P, const __half* V, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sP = smem;            // 128 rows x 128 B
  uint8_t* sV = smem + 16384;    // 2 x [64 tokens][128 B]
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<__half*>(sP + sw128_off(r, k, 128)) = P[i];
  }
  for (int i = tid; i < 64 * 128; i += blockDim.x) {
    const int tok = i / 128, d = i % 128;   // V[tok][d]: row = token, 64-dim columns
    *reinterpret_cast<__half*>(sV + sw128_off(tok, d, 64)) = V[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (1u << 16) | (128u >> 3 << 17) | (128u >> 4 << 24);  // b MN-major
  if (tid == 0) {
    for (int k = 0; k < 4; ++k) {
      const uint64_t ad = make_desc2(smem_u32(sP) + k * 32, 16, 1024);
      const uint64_t bd = make_desc2(smem_u32(sV) + k * 2048, 64 * 128, 1024);
      const uint32_t acc = k > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra WAIT2;\n\t}\n" ::"r"(smem_u32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < 128; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) D[row * 128 + c0 + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

static void run_pv() {
  std::vector<__half> p(128 * 64), v(64 * 128);
  std::vector<float> pf(128 * 64), vf(64 * 128), got(128 * 128);
  srand(2);
  for (int i = 0; i < 128 * 64; ++i) { p[i] = __float2half((rand() % 2001 - 1000) / 1000.f); pf[i] = __half2float(p[i]); }
  for (int i = 0; i < 64 * 128; ++i) { v[i] = __float2half((rand() % 2001 - 1000) / 1000.f); vf[i] = __half2float(v[i]); }
  __half *dP, *dV;
  float* dD;
  CK(cudaMalloc(&dP, p.size() * 2));
  CK(cudaMalloc(&dV, v.size() * 2));
  CK(cudaMalloc(&dD, got.size() * 4));
  CK(cudaMemcpy(dP, p.data(), p.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dV, v.data(), v.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(pv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
  pv_kernel<<<1, 128, 40 * 1024>>>(dP, dV, dD);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += static_cast<double>(pf[m * 64 + k]) * vf[k * 128 + n];
      maxerr = fmax(maxerr, fabs(got[m * 128 + n] - s));
    }
  printf("PV (P K-major, V MN-major): max err %.3e  D[0]=%f\n", maxerr, got[0]);
}

int main() {
  run_pv();
  run<128>();
  run<64>();
  run<256>();
  return 0;
}
