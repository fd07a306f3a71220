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


// TS MMA with N = 128 + 16: B = [V | ones], V MN-major at sB (128 keys x 128 d,
// SW128), the "ones" MN atom at sB + LBO.  Columns 128..143 of D must be the
// row sums of A.
__global__ void __launch_bounds__(128, 1)
    ones_probe(const __grid_constant__ CUtensorMap tb, const uint8_t* a_gmem, float* out, uint32_t lbo) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = smem;
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&tbase, 256);
    tmem_relinquish();
  }
  // ones atom: 128 rows x 128 bytes of e4m3 1.0
  for (int i = threadIdx.x; i < 16384 / 4; i += 128) reinterpret_cast<uint32_t*>(sB + lbo)[i] = 0x38383838u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_tma, 16384);
    tma_load_2d(sB, &tb, 0, 0, &bar_tma);
  }
  mbar_wait(&bar_tma, 0);
  {
    const uint32_t* row = (const uint32_t*)(a_gmem + threadIdx.x * 128);
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = row[i];
    tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 160, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f8(128, 144, 0, 0, 1);
    for (int k = 0; k < 4; ++k) {
      uint64_t bdesc = smem_desc_sw128(smem_u32(sB) + k * 32 * 128, lbo, 1024);
      mma_f8_ts(tmem, tmem + 160 + k * 8, bdesc, idesc, k > 0);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int c = 0; c < 160; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i)
      if (c + i < 144) out[threadIdx.x * 144 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
  std::vector<uint8_t> A(128 * 128), B(128 * 128);
  srand(99);
  auto rnd_code = []() {
    uint8_t c;
    do {
      c = rand() & 0xFF;
    } while ((c & 0x7F) == 0x7F || ((c >> 3) & 15) > 11);
    return c;
  };
  for (auto& x : A) x = rnd_code() & 0x7F;  // P >= 0
  for (auto& x : B) x = rnd_code();
  uint8_t *dA, *dB;
  float* dO;
  CK(cudaMalloc(&dA, 16384));
  CK(cudaMalloc(&dB, 16384));
  CK(cudaMalloc(&dO, 128 * 144 * 4));
  CK(cudaMemcpy(dA, A.data(), 16384, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), 16384, cudaMemcpyHostToDevice));
  CUtensorMap tb = make_map(dB, 128);
  CK(cudaFuncSetAttribute(ones_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 16384 + 1024));
  int fails = 0;
  for (uint32_t lbo : {16384u, 32768u}) {
    CK(cudaMemset(dO, 0, 128 * 144 * 4));
    ones_probe<<<1, 128, 3 * 16384 + 1024>>>(tb, dA, dO, lbo);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> O(128 * 144);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    int bad_pv = 0, bad_sum = 0;
    for (int m = 0; m < 128; ++m) {
      double rs = 0;
      for (int k = 0; k < 128; ++k) rs += e4m3_val(A[m * 128 + k]);
      for (int n = 0; n < 144; ++n) {
        double ref = 0, mag = 0;
        for (int k = 0; k < 128; ++k) {
          double b = n < 128 ? e4m3_val(B[k * 128 + n]) : 1.0;
          ref += e4m3_val(A[m * 128 + k]) * b;
          mag += std::fabs(e4m3_val(A[m * 128 + k]) * b);
        }
        double err = std::fabs(O[m * 144 + n] - ref) / (mag + 1e-30);
        if (err > 1e-5) {
          if (n < 128) ++bad_pv; else ++bad_sum;
          if (bad_pv + bad_sum < 4) printf("  lbo %u m=%d n=%d got %g ref %g\n", lbo, m, n, O[m * 144 + n], ref);
        }
      }
    }
    printf("N=144 ones-atom probe, LBO=%u: PV %s (bad %d), row sums %s (bad %d)\n", lbo, bad_pv ? "FAIL" : "PASS",
           bad_pv, bad_sum ? "FAIL" : "PASS", bad_sum);
    fails += bad_pv + bad_sum;
  }
  return fails ? 1 : 0;
}
