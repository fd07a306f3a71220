// tcgen05 2-CTA (cta_group::2) FP8 MMA throughput probe: does a CTA pair issuing
// M256 x N128 x K32 (each SM: 128 rows x 128 columns) reach the full per-SM rate
// that a single CTA only reaches at N = 256?  Garbage operands (rate only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma2_rate.cu -o mma2_rate
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../../paper_2506_04648_b200/csrc/sm100.cuh"

using namespace fpsa::sm100;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t dk(uint32_t a) { return smem_desc_sw128(a, 16, 1024); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_rate(int n, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  long long t0 = clock64();
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 32768;
    const uint32_t idesc = idesc_f8(256, (uint32_t)n, 0, 0, 0);
    for (int it = 0; it < iters; ++it)
      for (int k = 0; k < 4; ++k)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 256),
            "l"(dk(sa + 32 * k)), "l"(dk(sb + 32 * k)), "r"(idesc), "r"(k > 0 ? 1u : 0u)
            : "memory");
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

int main() {
  long long* d_out;
  const int ctas = 148, iters = 2000;
  CK(cudaMalloc(&d_out, ctas * sizeof(long long)));
  const int smem = 2 * 32768 + 1024;
  CK(cudaFuncSetAttribute(mma2_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int n : {64, 128, 256}) {
    mma2_rate<<<ctas, 128, smem>>>(n, 10, d_out);
    CK(cudaDeviceSynchronize());
    mma2_rate<<<ctas, 128, smem>>>(n, iters, d_out);
    CK(cudaDeviceSynchronize());
    long long h[148];
    CK(cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < ctas; i += 2) avg += h[i];
    avg /= (ctas / 2);
    const double per = avg / iters;  // clk per 4 x K32 step of the pair
    const double macs_per_sm = 128.0 * n * 128;  // each SM: 128 rows x n cols x 128 K
    printf("cta_group::2 M256 N%-3d K128 (4 x K32): %8.1f clk/step  %7.0f MAC/clk/SM\n", n, per, macs_per_sm / per);
  }
  return 0;
}
