// Hardware probe for the conventions the attention kernel relies on:
//   A. tcgen05.mma kind::f8f6f4, A and B K-major from SW128 smem (S = Q K^T)
//   B. same, B MN-major (O = P V with V stored [keys][d])
//   C. A operand from TMEM (4 fp8 per 32-bit column), B MN-major
//   D. cvt.rn.satfinite.e4m3x2.f32 vs exact RNE for every f32 bit pattern
//   E. MUFU / FMA-pipe throughput microbenchmarks (ex2 f32, f16x2, ffma2)
//   F. tcgen05.ld throughput
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 probe_sm100.cu -o probe
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

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

static double e4m3_val(uint8_t c) {
  int s = c >> 7, e = (c >> 3) & 15, m = c & 7;
  double v = e == 0 ? m * std::ldexp(1.0, -9) : (8 + m) * std::ldexp(1.0, e - 10);
  return s ? -v : v;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

static CUtensorMap make_map(void* base, uint64_t rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("tensor map encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

// mode 0: SS, B K-major.  mode 1: SS, B MN-major.  mode 2: TS (A from TMEM), B MN-major.
// mode 3: TS, B K-major.
__global__ void __launch_bounds__(128, 1)
    mma_probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
              const uint8_t* a_gmem, float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&tbase, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_tma, 32768);
    tma_load_2d(sA, &ta, 0, 0, &bar_tma);
    tma_load_2d(sB, &tb, 0, 0, &bar_tma);
  }
  mbar_wait(&bar_tma, 0);
  if (mode >= 2) {
    // row r = threadIdx.x holds A[r][0..127], 4 codes per column, columns 128..159
    const uint32_t* row = (const uint32_t*)(a_gmem + threadIdx.x * 128);
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = row[i];
    uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + 128;
    tmem_st32(taddr, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t bmn = (mode == 1 || mode == 2) ? 1 : 0;
    uint32_t idesc = idesc_f8(128, 128, 0, 0, bmn);
    for (int k = 0; k < 4; ++k) {
      uint64_t bdesc = bmn ? smem_desc_sw128(smem_u32(sB) + k * 32 * 128, 16384, 1024)
                           : smem_desc_sw128(smem_u32(sB) + k * 32, 16, 1024);
      if (mode < 2) {
        uint64_t adesc = smem_desc_sw128(smem_u32(sA) + k * 32, 16, 1024);
        mma_f8_ss(tmem, adesc, bdesc, idesc, k > 0);
      } else {
        mma_f8_ts(tmem, tmem + 128 + k * 8, bdesc, idesc, k > 0);
      }
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out[threadIdx.x * 128 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

static int run_mma_probe(int mode) {
  std::vector<uint8_t> A(128 * 128), B(128 * 128);
  srand(1234 + mode);
  auto rnd_code = []() {
    uint8_t c;
    do {
      c = rand() & 0xFF;
    } while ((c & 0x7F) == 0x7F || ((c >> 3) & 15) > 11);  // no NaN, moderate range
    return c;
  };
  for (auto& x : A) x = rnd_code();
  for (auto& x : B) x = rnd_code();
  uint8_t *dA, *dB;
  float* dO;
  CK(cudaMalloc(&dA, 16384));
  CK(cudaMalloc(&dB, 16384));
  CK(cudaMalloc(&dO, 128 * 128 * 4));
  CK(cudaMemcpy(dA, A.data(), 16384, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), 16384, cudaMemcpyHostToDevice));
  CUtensorMap ta = make_map(dA, 128), tb = make_map(dB, 128);
  CK(cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000));
  mma_probe<<<1, 128, 40000>>>(ta, tb, dA, dO, mode);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> O(128 * 128);
  CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
  double maxrel = 0;
  int bad = 0;
  bool bmn = (mode == 1 || mode == 2);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      double ref = 0, mag = 0;
      for (int k = 0; k < 128; ++k) {
        double b = bmn ? e4m3_val(B[k * 128 + n]) : e4m3_val(B[n * 128 + k]);
        ref += e4m3_val(A[m * 128 + k]) * b;
        mag += std::fabs(e4m3_val(A[m * 128 + k]) * b);
      }
      double err = std::fabs(O[m * 128 + n] - ref) / (mag + 1e-30);
      if (err > maxrel) maxrel = err;
      if (err > 1e-5) {
        if (bad < 4) printf("  mode %d mismatch m=%d n=%d got %g ref %g\n", mode, m, n, O[m * 128 + n], ref);
        ++bad;
      }
    }
  printf("MMA probe mode %d (%s): %s  bad=%d maxrel=%.3g\n", mode,
         mode == 0 ? "SS Kmaj/Kmaj" : mode == 1 ? "SS Kmaj/MNmaj" : mode == 2 ? "TS /MNmaj" : "TS /Kmaj",
         bad ? "FAIL" : "PASS", bad, maxrel);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  return bad;
}

// ---------------------------------------------------------------- D. cvt exhaustive
__device__ __forceinline__ uint8_t hw_e4m3(float x) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(0.0f), "f"(x));
  return (uint8_t)(r & 0xFF);
}
__device__ __forceinline__ uint8_t soft_e4m3(float x) {
  uint32_t b = __float_as_uint(x);
  uint8_t sign = (b >> 31) ? 0x80 : 0;
  double v = fabs((double)x);
  double step;
  if (v < 0.015625)
    step = 0.001953125;  // 2^-9
  else {
    int e = ilogb(v);
    step = ldexp(1.0, e - 3);
  }
  double k = rint(v / step);
  double val = k * step;
  if (val > 448.0) val = 448.0;
  uint8_t code;
  if (val < 0.015625)
    code = (uint8_t)(val / 0.001953125);
  else {
    int e = ilogb(val);
    int m = (int)(val / ldexp(1.0, e) * 8.0) - 8;
    code = (uint8_t)(((e + 7) << 3) | m);
  }
  return code | sign;
}
__global__ void cvt_probe(unsigned long long* nbad, unsigned long long* first) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (uint64_t i = tid; i < (1ull << 32); i += stride) {
    uint32_t bits = (uint32_t)i;
    if ((bits & 0x7fffffffu) >= 0x7f800000u) continue;  // inf / nan
    float x = __uint_as_float(bits);
    uint8_t h = hw_e4m3(x), s = soft_e4m3(x);
    if (h != s) {
      ++local;
      atomicCAS(first, 0ull, ((unsigned long long)bits << 16) | ((unsigned long long)h << 8) | s);
    }
  }
  atomicAdd(nbad, local);
}

// ---------------------------------------------------------------- E. pipe throughput
template <int KIND>
__global__ void __launch_bounds__(1024, 1) pipe_bench(float* sink, long long* cycles, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) {  // ex2.approx.f32  (1 exp per op)
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
        x[i] = -y;
      } else if (KIND == 1) {  // ex2.approx.f16x2 (2 exps per op)
        uint32_t v = __float_as_uint(x[i]), y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(v));
        x[i] = __uint_as_float(y ^ 0x80008000u);
      } else if (KIND == 2) {  // ffma (1 fma per op)
        x[i] = fmaf(x[i], 0.999f, 0.0001f);
      } else if (KIND == 3) {  // fma.rn.f32x2 (2 fmas per op), uses x[i] pair with itself
        uint64_t v = ((uint64_t)__float_as_uint(x[i]) << 32) | __float_as_uint(x[i]);
        uint64_t c = ((uint64_t)__float_as_uint(0.999f) << 32) | __float_as_uint(0.999f);
        uint64_t a = ((uint64_t)__float_as_uint(0.0001f) << 32) | __float_as_uint(0.0001f);
        uint64_t y;
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(y) : "l"(v), "l"(c), "l"(a));
        x[i] = __uint_as_float((uint32_t)y);
      } else if (KIND == 4) {  // 3-input max
        float y;
        asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(x[i]), "f"(x[(i + 1) & 7]), "f"(x[(i + 2) & 7]));
        x[i] = y - 1.0f;
      } else if (KIND == 5) {  // cvt e4m3x2 from f32 pair
        uint16_t r;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        x[i] = __uint_as_float(0x3f000000u | r);
      } else if (KIND == 6) {  // cvt e4m3x2 from f16x2
        uint16_t r;
        asm volatile("cvt.rn.satfinite.e4m3x2.f16x2 %0, %1;" : "=h"(r) : "r"(__float_as_uint(x[i])));
        x[i] = __uint_as_float(0x3f000000u | r);
      } else if (KIND == 7) {  // cvt f16x2 from f32 pair
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        x[i] = __uint_as_float(r & 0x3fffffffu);
      } else if (KIND == 8) {  // ex2.approx.ftz.bf16x2
        uint32_t v = __float_as_uint(x[i]), y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(v));
        x[i] = __uint_as_float(y ^ 0x80008000u);
      } else if (KIND == 9) {  // add.f32x2
        uint64_t v = ((uint64_t)__float_as_uint(x[i]) << 32) | __float_as_uint(x[i]);
        uint64_t y;
        asm volatile("add.rn.f32x2 %0, %1, %1;" : "=l"(y) : "l"(v));
        x[i] = __uint_as_float((uint32_t)y) * 0.5f;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// ---------------------------------------------------------------- F. TMEM load throughput
__global__ void __launch_bounds__(512, 1) tmem_ld_bench(float* sink, long long* cycles, int iters, int nwarps) {
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    tmem_alloc(&tbase, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tbase;
  float acc = 0;
  long long t0 = clock64();
  if (warp < nwarps) {
    uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + ((it * 32 + warp / 4 * 128) & 511), r);
      tmem_wait_ld();
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  sink[threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  int bad = 0;
  for (int mode = 0; mode < 4; ++mode) bad += run_mma_probe(mode);

  {
    unsigned long long *dn, *df;
    CK(cudaMalloc(&dn, 8));
    CK(cudaMalloc(&df, 8));
    CK(cudaMemset(dn, 0, 8));
    CK(cudaMemset(df, 0, 8));
    cvt_probe<<<148 * 8, 256>>>(dn, df);
    CK(cudaDeviceSynchronize());
    unsigned long long n, f;
    CK(cudaMemcpy(&n, dn, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&f, df, 8, cudaMemcpyDeviceToHost));
    printf("CVT probe e4m3 (all finite f32): mismatches=%llu first: bits=0x%08llx hw=0x%02llx soft=0x%02llx -> %s\n",
           n, f >> 16, (f >> 8) & 0xff, f & 0xff, n ? "FAIL" : "PASS");
  }

  {
    float* sink;
    long long* cyc;
    CK(cudaMalloc(&sink, 1024 * 4 * 4));
    CK(cudaMalloc(&cyc, 64));
    const char* names[] = {"ex2.f32", "ex2.f16x2", "ffma", "ffma2(f32x2)", "max3", "cvt.e4m3x2.f32",
                           "cvt.e4m3x2.f16x2", "cvt.f16x2.f32", "ex2.bf16x2", "add.f32x2"};
    for (int kind = 0; kind < 10; ++kind) {
      int iters = 2048;
      auto launch = [&](auto kern) {
        kern<<<1, 1024>>>(sink, cyc, 16);
        kern<<<1, 1024>>>(sink, cyc, iters);
      };
      switch (kind) {
        case 0: launch(pipe_bench<0>); break;
        case 1: launch(pipe_bench<1>); break;
        case 2: launch(pipe_bench<2>); break;
        case 3: launch(pipe_bench<3>); break;
        case 4: launch(pipe_bench<4>); break;
        case 5: launch(pipe_bench<5>); break;
        case 6: launch(pipe_bench<6>); break;
        case 7: launch(pipe_bench<7>); break;
        case 8: launch(pipe_bench<8>); break;
        case 9: launch(pipe_bench<9>); break;
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("pipe %s: error %s\n", names[kind], cudaGetErrorString(e));
        return 1;
      }
      long long c;
      CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      double instr_per_clk = 1024.0 * 8 * iters / (double)c;
      printf("PIPE %-18s: %.1f thread-instr/clk/SM\n", names[kind], instr_per_clk);
    }
    for (int nw : {4, 8, 16}) {
      int iters = 4096;
      tmem_ld_bench<<<1, 512>>>(sink, cyc, 16, nw);
      tmem_ld_bench<<<1, 512>>>(sink, cyc, iters, nw);
      CK(cudaDeviceSynchronize());
      long long c;
      CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      double bytes = (double)nw * 32 * 32 * 4 * iters;
      printf("TMEM ld32 %2d warps: %.1f B/clk/SM\n", nw, bytes / c);
    }
  }
  printf("PROBE DONE bad=%d\n", bad);
  return 0;
}
