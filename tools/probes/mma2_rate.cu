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

__device__ __forceinline__ uint64_t dmn64(uint32_t a, uint32_t lbo) {  // MN-major SWIZZLE_64B (V halves)
  const uint64_t d = smem_desc_sw128(a, lbo, 512);
  return (d & ~((uint64_t)7 << 61)) | ((uint64_t)4 << 61);
}

// mode 0: SS, both K-major SW128, N = n
// mode 1: SS, B MN-major SW64 (64-wide atoms, second atom at LBO), N = n
// mode 2: TS, A from TMEM, B MN-major SW64, N = n
// mode 3: the attention step: QK SS K-major N128 into S, then PV TS (A = S's first 32 columns), B MN-major SW64, N = n
// lat != 0: commit and wait after every step (latency instead of throughput)
// ld == 1: warps 4..7 stream tcgen05.ld over 128 TMEM columns (as the softmax warps load S) meanwhile
// ld == 2: warps 4..11 run FMA / MUFU work (two per SM sub-partition, as the softmax warps do)
template <int mode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    mma2_rate(int n, int lat, int iters, int ld, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  __shared__ volatile int s_stop;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    s_stop = 0;
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
  uint32_t phase = 0;
  auto commit_wait = [&]() {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
    mbar_wait(&bar, phase);
    phase ^= 1;
  };
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 32768, sv = sa + 65536;
    const uint32_t id_k = idesc_f8(256, (uint32_t)n, 0, 0, 0), id_mn = idesc_f8(256, (uint32_t)n, 0, 0, 1);
    const uint32_t id_qk = idesc_f8(256, 128, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
      if constexpr (mode == 3) {
        for (int k = 0; k < 4; ++k)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 256),
              "l"(dk(sa + 32 * k)), "l"(dk(sb + 32 * k)), "r"(id_qk), "r"(k > 0 ? 1u : 0u)
              : "memory");
      }
      for (int k = 0; k < 4; ++k) {
        if constexpr (mode == 0)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 256),
              "l"(dk(sa + 32 * k)), "l"(dk(sb + 32 * k)), "r"(id_k), "r"(k > 0 ? 1u : 0u)
              : "memory");
        else if constexpr (mode == 1)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(dk(sa + 32 * k)), "l"(dmn64(sv + 2048 * k, 8192)), "r"(id_mn), "r"(k > 0 ? 1u : 0u)
              : "memory");
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(tmem + 256 + 8 * k), "l"(dmn64(sv + 2048 * k, 8192)), "r"(id_mn), "r"(k > 0 ? 1u : 0u)
              : "memory");
      }
      if (lat) commit_wait();
    }
    if (!lat) commit_wait();
  }
  if (warp >= 4 && ld == 2) {
    float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
    while (!s_stop) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        x0 = fmaf(x0, 0.999f, 0.5f);
        x1 = fmaf(x1, 0.999f, 0.5f);
        x2 = exp2f(-x2 * 1e-3f) + x2 * 0.5f;
        x3 = fmaf(x3, 0.999f, 0.5f);
      }
    }
    if (x0 + x1 + x2 + x3 == 1234.5f) out[0] = 0;
  }
  if (warp >= 4 && warp < 8 && ld == 1) {
    const uint32_t base = tmem + 384 + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    while (!s_stop) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(base + 32 * (c & 1), r);
        tmem_wait_ld();
        acc += r[(c * 7) & 31];
      }
    }
    if (acc == 0x12345678u) out[0] = 0;
  }
  if (threadIdx.x == 0) {
    if (rank != 0) {
      for (int i = 0; i < (lat ? iters : 1); ++i) {
        mbar_wait(&bar, phase);
        phase ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
    s_stop = 1;
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

int main() {
  long long* d_out;
  const int ctas = 148, iters = 2000;
  CK(cudaMalloc(&d_out, ctas * sizeof(long long)));
  const int smem = 3 * 32768 + 1024;
  void (*kern[4])(int, int, int, int, long long*) = {mma2_rate<0>, mma2_rate<1>, mma2_rate<2>, mma2_rate<3>};
  for (auto k : kern) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const char* names[4] = {"SS K-major", "SS B MN-major SW64", "TS B MN-major SW64", "QK N128 + PV TS MN SW64"};
  struct Case { int mode, n; } cases[] = {{0, 64}, {0, 128}, {0, 160}, {0, 256}, {1, 128}, {1, 160}, {2, 128},
                                          {2, 160}, {3, 128}, {3, 160}};
  for (int ld = 0; ld < 3; ld += 2)
  for (auto c : cases)
    for (int lat = 0; lat < 2; ++lat) {
      const int it = lat ? iters / 4 : iters;
      kern[c.mode]<<<ctas, 384, smem>>>(c.n, lat, 10, ld, d_out);
      CK(cudaDeviceSynchronize());
      kern[c.mode]<<<ctas, 384, smem>>>(c.n, lat, it, ld, d_out);
      CK(cudaDeviceSynchronize());
      long long h[148];
      CK(cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int i = 0; i < ctas; i += 2) avg += h[i];
      avg /= (ctas / 2);
      const double per = avg / it;  // clk per step of the pair
      const double macs_per_sm = 128.0 * (c.n + (c.mode == 3 ? 128 : 0)) * 128;
      printf("cta_group::2 M256 %-24s N%-3d K128 %s%s: %8.1f clk/step  %7.0f MAC/clk/SM\n", names[c.mode], c.n,
             lat ? "latency   " : "throughput", ld == 1 ? " +TMEM ld" : ld == 2 ? " +FMA/MUFU warps" : "", per, macs_per_sm / per);
    }
  return 0;
}
