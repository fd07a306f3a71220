// Softmax-only throughput probe: the attention kernel's half-row pass
// (softmax.cuh) on synthetic S in TMEM, 8 softmax warps + 2 idle warps per CTA
// (the kernel's shape), one CTA per SM.  Each step: load S (2 x tcgen05.ld.32),
// compute P~ and the row sum, store P~ (tcgen05.st.16), wait.  Variants differ
// in the MUFU / polynomial split and whether the row sum is taken.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 softmax_rate.cu -o softmax_rate
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../../paper_2506_04648_b200/csrc/softmax.cuh"

using namespace fpsa;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

template <int MASK, bool SUM>
__device__ __forceinline__ float pass64(uint32_t s_addr, float c, float boff, uint32_t* w) {
  if (MASK == 1) return (float)softmax_block<64>(s_addr, 64, false, c, boff, w);  // the kernel entry point
  const f2 cc = bcast(c), bb = bcast(boff);
  const float cs = c * (1.0f / 256.0f), bs = (boff + 126.0f) * (1.0f / 256.0f);
  uint32_t sa[32], sb[32];
  tmem_ld32(s_addr, sa);
  tmem_wait_ld();
  softmax_chunk32<0>(sa, cc, bb, cs, bs, w);
  tmem_ld32(s_addr + 32, sb);
  tmem_wait_ld();
  softmax_chunk32<1>(sb, cc, bb, cs, bs, w);
  return __uint_as_float(w[0]);
}

template <int MASK, bool SUM>
__device__ __forceinline__ float pass32(uint32_t s_addr, float c, float boff, uint32_t* w) {
  const f2 cc = bcast(c), bb = bcast(boff);
  const float cs = c * (1.0f / 256.0f), bs = (boff + 126.0f) * (1.0f / 256.0f);
  uint32_t sa[32];
  tmem_ld32(s_addr, sa);
  tmem_wait_ld();
  softmax_chunk32<0>(sa, cc, bb, cs, bs, w);
  return __uint_as_float(w[0]);
}

// 16 softmax warps (4 per lane quarter, 32 columns each) + 2 idle warps
template <int MASK, bool SUM>
__global__ void __launch_bounds__(576, 1) softmax_rate16(int iters, long long* out, float* sink) {
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 16) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  float l = 0.f;
  long long t = 0;
  if (warp < 16) {
    const int quarter = warp & 3, part = warp >> 2;
    const uint32_t base = tmem + 128 + ((uint32_t)(quarter * 32) << 16) + part * 32;
    for (int b2 = 0; b2 < 2; ++b2) {
      uint32_t v[32];
      for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(0.05f * (float)((lane * 7 + i * 13 + part) % 97) - 2.0f);
      tmem_st32(base + 128 * b2, v);
    }
    tmem_wait_st();
    const float c = 0.125f, boff = 8.8f - 3.0f - 8.0f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t s_addr = base + 128 * (it & 1);
      uint32_t w[8];
      l += pass32<MASK, SUM>(s_addr, c, boff, w);
      tmem_st8(s_addr + 16, w);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
    }
    t = clock64() - t0;
  }
  __syncthreads();
  if (warp < 16 && lane == 0) atomicAdd((unsigned long long*)&out[blockIdx.x], (unsigned long long)t);
  if (warp < 16) sink[blockIdx.x * 512 + threadIdx.x] = l;
  tc_fence_before();
  __syncthreads();
  if (warp == 16) tmem_dealloc(tmem, 512);
}

__device__ __forceinline__ uint32_t tmem_base_probe(uint32_t t) { return t; }

template <int MASK, bool SUM, int SPIN = 0>
__global__ void __launch_bounds__(320, 1) softmax_rate(int iters, long long* out, float* sink) {
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t bar_done;
  __shared__ uint64_t hs_full[2], hs_ready[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar_done, 8);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&hs_full[i], 1);
      mbar_init(&hs_ready[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 8) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  if (SPIN == 3 && warp == 9 && lane == 0) {
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
    const uint32_t sq = smem_u32(sm), sk = sq + 16384, sv = sk + 16384;
    const uint32_t id_qk = idesc_f8(128, 128, 0, 0, 0), id_pv = idesc_f8(128, 128, 0, 0, 1);
    const uint32_t addr = smem_u32(&bar_done);
    while (!mbar_try_wait(addr, 0)) {
      for (int k = 0; k < 4; ++k)
        mma_f8_ss(s_tmem, smem_desc_sw128(sq + 32 * k, 16, 1024), smem_desc_sw128(sk + 32 * k, 16, 1024), id_qk, k > 0);
      for (int k = 0; k < 4; ++k)
        mma_f8_ts(s_tmem + 0, s_tmem + 448 + 8 * k, smem_desc_sw128(sv + k * 4096, 16384, 1024), id_pv, 1);
    }
  } else if (SPIN == 3 && warp >= 8) {
    const uint32_t addr = smem_u32(&bar_done);
    while (!mbar_try_wait(addr, 0)) {
    }
  }
  if (SPIN == 6 && warp == 9) {
    // "MMA warp": after softmax step j completes, make S(j + 2) available
    if (lane == 0) {
      mbar_arrive(&hs_full[0]);
      mbar_arrive(&hs_full[1]);
      for (int j = 0; j < iters; ++j) {
        mbar_wait(&hs_ready[j & 1], (j >> 1) & 1);
        if (j + 2 < iters) mbar_arrive(&hs_full[j & 1]);
      }
    }
  }
  if (SPIN && SPIN < 3 && warp >= 8) {
    // the producer / MMA warps of the kernel: poll a barrier the softmax warps complete at the end
    const uint32_t addr = smem_u32(&bar_done);
    if (SPIN == 1) {
      while (!mbar_try_wait(addr, 0)) {
      }
    } else {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(addr), "r"(0), "r"(1000000u) : "memory");
    }
  }
  const uint32_t tmem = s_tmem;
  float l = 0.f;
  long long t = 0;
  if (warp < 8) {
    const int quarter = warp & 3, half = warp >> 2;
    const uint32_t base = tmem + 128 + ((uint32_t)(quarter * 32) << 16) + half * 64;
    // synthetic S: logits around 0 with spread, in both S buffers
    for (int b2 = 0; b2 < 2; ++b2)
      for (int c = 0; c < 64; c += 32) {
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(0.05f * (float)((lane * 7 + i * 13 + c) % 97) - 2.0f);
        tmem_st32(base + 128 * b2 + c, v);
      }
    tmem_wait_st();
    const float c = 0.125f, boff = 8.8f - 3.0f - 8.0f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t s_addr = base + 128 * (it & 1);
      uint32_t w[16];
      if (SPIN == 6) {
        mbar_wait(&hs_full[it & 1], (it >> 1) & 1);
        tc_fence_after();
      }
      if (SPIN == 4) named_bar_sync(1 + quarter, 64);  // the two halves of a row start each step together
      if (SPIN == 5) named_bar_sync(1, 256);           // all softmax warps start each step together
      l += pass64<MASK, SUM>(s_addr, c, boff, w);
      tmem_st16(s_addr + 32, w);  // P into columns that are not read back (keeps S intact)
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (SPIN == 6 && lane == 0) mbar_arrive(&hs_ready[it & 1]);
    }
    t = clock64() - t0;
    if (lane == 0) mbar_arrive(&bar_done);
  }
  __syncthreads();
  if (warp < 8 && lane == 0) atomicAdd((unsigned long long*)&out[blockIdx.x], (unsigned long long)t);
  if (warp < 8) sink[blockIdx.x * 256 + threadIdx.x] = l;
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 512);
}

template <int MASK, bool SUM, int SPIN = 0>
void run(const char* name, long long* d, float* sink) {
  const int iters = 2000;
  CK(cudaMemset(d, 0, 148 * sizeof(long long)));
  const int smem = SPIN == 3 ? 3 * 16384 + 1024 : 0;
  if (smem) CK(cudaFuncSetAttribute(softmax_rate<MASK, SUM, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  softmax_rate<MASK, SUM, SPIN><<<148, 320, smem>>>(iters, d, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(d, 0, 148 * sizeof(long long)));
  softmax_rate<MASK, SUM, SPIN><<<148, 320, smem>>>(iters, d, sink);
  CK(cudaDeviceSynchronize());
  long long h[148];
  CK(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  const double per_warp_step = s / 148.0 / 8.0 / iters;
  // per SMSP: 2 warps x 64 elements per step
  printf("%-40s %7.1f clk per warp-step (64 elem)  %5.2f clk per warp-elem per SMSP\n", name, per_warp_step,
         per_warp_step / 128.0);
}

template <int MASK, bool SUM>
void run16(const char* name, long long* d, float* sink) {
  const int iters = 2000;
  CK(cudaMemset(d, 0, 148 * sizeof(long long)));
  softmax_rate16<MASK, SUM><<<148, 576>>>(iters, d, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(d, 0, 148 * sizeof(long long)));
  softmax_rate16<MASK, SUM><<<148, 576>>>(iters, d, sink);
  CK(cudaDeviceSynchronize());
  long long h[148];
  CK(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  const double per_warp_step = s / 148.0 / 16.0 / iters;
  // per SMSP: 4 warps x 32 elements per step
  printf("%-40s %7.1f clk per warp-step (32 elem)  %5.2f clk per warp-elem per SMSP\n", name, per_warp_step,
         per_warp_step / 128.0);
}

int main() {
  long long* d;
  float* sink;
  CK(cudaMalloc(&d, 148 * sizeof(long long)));
  CK(cudaMalloc(&sink, 148 * 256 * sizeof(float)));
  run<0xAA, true>("poly 1/2 (0xAA), sum", d, sink);
  run<0xAA, false>("poly 1/2 (0xAA), no sum      [kernel]", d, sink);
  run<1, false>("kernel softmax_block (64 cols, sat check)", d, sink);
  run<1, false, 4>("  + pair lockstep (bar.sync 64 per step)", d, sink);
  run<1, false, 5>("  + all-warp lockstep (bar.sync 256 per step)", d, sink);
  run<1, false, 6>("  + kernel-like mbarrier handshake per step", d, sink);
  run<0xAA, false, 1>("  + 2 warps spinning on try_wait", d, sink);
  run<0xAA, false, 2>("  + 2 warps try_wait w/ suspend hint", d, sink);
  run<0xAA, false, 3>("  + tensor core busy (QK SS + PV TS loop)", d, sink);
  run<0x92, true>("poly 3/8 (0x92), sum", d, sink);
  run<0x92, false>("poly 3/8 (0x92), no sum", d, sink);
  run<0x88, true>("poly 1/4 (0x88), sum", d, sink);
  run<0x00, true>("MUFU only, sum", d, sink);
  run<0x00, false>("MUFU only, no sum", d, sink);
  run<0xFF, true>("poly only, sum", d, sink);
  run<0xDA, true>("poly 5/8 (0xDA), sum", d, sink);
  CK(cudaFree(sink));
  CK(cudaMalloc(&sink, 148 * 512 * sizeof(float)));
  run16<0xAA, true>("16 warps: poly 1/2, sum", d, sink);
  run16<0xAA, false>("16 warps: poly 1/2, no sum", d, sink);
  run16<0x92, true>("16 warps: poly 3/8, sum", d, sink);
  run16<0x92, false>("16 warps: poly 3/8, no sum", d, sink);
  return 0;
}
