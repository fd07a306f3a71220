// tcgen05 FP8 MMA rate / latency probe for the attention kernel's shapes.
// One CTA per SM, one thread issues; smem / TMEM contents are garbage (rate only).
//   mode 0: QK SS M128 N64 K128 (4 x K32)  + PV TS M128 N128 K64 (2 x K32)    [64-key block]
//   mode 1: QK SS M128 N128 K128 (4 x K32) + PV TS M128 N128 K128 (4 x K32)   [128-key block]
//   mode 2: QK SS M128 N128 only
//   mode 3: PV TS M128 N128 only
//   mode 4: QK SS M128 N256 K128 (4 x K32) only
//   mode 5: PV SS M128 N128 (A = P from smem) only
//   mode 6: PV TS M128 N144 K128 (V + "ones" MN atom through the LBO field) only
//   mode 7: QK N128 + PV TS N144 (the attention kernel's 128-key step)
//   mode 8: PV TS M128 N256 K128 only
//   mode 9: PV TS M128 N160 K128 only
// For each mode: throughput (issue all, commit once) and latency (commit + wait per step).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_rate.cu -o mma_rate
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

__device__ __forceinline__ uint64_t dk(uint32_t a) { return smem_desc_sw128(a, 16, 1024); }
__device__ __forceinline__ uint64_t dmn(uint32_t a) { return smem_desc_sw128(a, 16384, 1024); }
__device__ __forceinline__ uint64_t dones(uint32_t a, uint32_t lbo) { return smem_desc_sw128(a, lbo, 1024); }

__global__ void __launch_bounds__(128, 1) mma_rate(int mode, int iters, int sync_each, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    const uint32_t sq = smem_u32(smem), sk = sq + 32768, sv = sk + 32768, sp = sv + 32768;
    const uint32_t id_qk64 = idesc_f8(128, 64, 0, 0, 0), id_qk128 = idesc_f8(128, 128, 0, 0, 0);
    const uint32_t id_qk256 = idesc_f8(128, 256, 0, 0, 0), id_pv = idesc_f8(128, 128, 0, 0, 1);
    const uint32_t id_pv144 = idesc_f8(128, 144, 0, 0, 1), id_pv256 = idesc_f8(128, 256, 0, 0, 1);
    const uint32_t id_pv160 = idesc_f8(128, 160, 0, 0, 1);
    const uint32_t tS = tmem + 256, tO = tmem;
    long long t0 = clock64();
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      if (mode == 0) {
        for (int k = 0; k < 4; ++k) mma_f8_ss(tS + 64 * (it & 1), dk(sq + 32 * k), dk(sk + 32 * k), id_qk64, k > 0);
        for (int k = 0; k < 2; ++k) mma_f8_ts(tO, tS + 64 * (it & 1) + 8 * k, dmn(sv + k * 4096), id_pv, 1);
      } else if (mode == 1) {
        for (int k = 0; k < 4; ++k) mma_f8_ss(tS, dk(sq + 32 * k), dk(sk + 32 * k), id_qk128, k > 0);
        for (int k = 0; k < 4; ++k) mma_f8_ts(tO, tS + 8 * k, dmn(sv + k * 4096), id_pv, 1);
      } else if (mode == 2) {
        for (int k = 0; k < 4; ++k) mma_f8_ss(tS, dk(sq + 32 * k), dk(sk + 32 * k), id_qk128, k > 0);
      } else if (mode == 3) {
        for (int k = 0; k < 4; ++k) mma_f8_ts(tO, tS + 8 * k, dmn(sv + k * 4096), id_pv, 1);
      } else if (mode == 4) {
        for (int k = 0; k < 4; ++k) mma_f8_ss(tS, dk(sq + 32 * k), dk(sk + 32 * k), id_qk256, k > 0);
      } else if (mode == 5) {
        for (int k = 0; k < 4; ++k) mma_f8_ss(tO, dk(sp + 32 * k), dmn(sv + k * 4096), id_pv, 1);
      } else if (mode == 6) {
        for (int k = 0; k < 4; ++k) mma_f8_ts(tO, tS + 8 * k, dones(sv + k * 4096, sp - sv), id_pv144, 1);
      } else if (mode == 7) {
        for (int k = 0; k < 4; ++k) mma_f8_ss(tS, dk(sq + 32 * k), dk(sk + 32 * k), id_qk128, k > 0);
        for (int k = 0; k < 4; ++k) mma_f8_ts(tO, tS + 128 + 8 * k, dones(sv + k * 4096, sp - sv), id_pv144, 1);
      } else if (mode == 8) {
        for (int k = 0; k < 4; ++k) mma_f8_ts(tO, tS + 8 * k, dmn(sv + k * 4096), id_pv256, 1);
      } else {
        for (int k = 0; k < 4; ++k) mma_f8_ts(tO, tS + 8 * k, dmn(sv + k * 4096), id_pv160, 1);
      }
      if (sync_each) {
        mma_commit(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, phase);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
  long long* d_out;
  const int ctas = 148, iters = 2000;
  CK(cudaMalloc(&d_out, ctas * sizeof(long long)));
  const int smem = 4 * 32768 + 1024;
  CK(cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const char* names[10] = {"QK N64 + PV K64 (64-key step)", "QK N128 + PV K128 (128-key step)", "QK SS N128 only",
                           "PV TS N128 K128 only", "QK SS N256 only", "PV SS N128 K128 only",
                           "PV TS N144 K128 (ones atom) only", "QK N128 + PV TS N144 (kernel step)",
                           "PV TS N256 K128 only", "PV TS N160 K128 only"};
  const double macs[10] = {128.0 * 64 * 128 + 128.0 * 128 * 64, 2 * 128.0 * 128 * 128, 128.0 * 128 * 128,
                           128.0 * 128 * 128, 128.0 * 256 * 128, 128.0 * 128 * 128,
                           128.0 * 128 * 128, 2 * 128.0 * 128 * 128, 128.0 * 256 * 128, 128.0 * 128 * 128};
  const int first = argc > 1 ? atoi(argv[1]) : 0;
  for (int mode = first; mode < 10; ++mode) {
    for (int sync_each = 0; sync_each < 2; ++sync_each) {
      mma_rate<<<ctas, 128, smem>>>(mode, 10, sync_each, d_out);
      CK(cudaDeviceSynchronize());
      mma_rate<<<ctas, 128, smem>>>(mode, iters, sync_each, d_out);
      CK(cudaDeviceSynchronize());
      long long h[148];
      CK(cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int i = 0; i < ctas; ++i) avg += h[i];
      avg /= ctas;
      const double per = avg / iters;
      printf("%-36s %s: %8.1f clk/step  %7.0f MAC/clk/SM\n", names[mode], sync_each ? "latency   " : "throughput",
             per, macs[mode] / per);
    }
  }
  return 0;
}
