// TMA gather throughput vs row width: natural-order [L][H][128] bf16 tiles (3,5,16) of the Wan2.1-14B
// 720p grid, loaded with 5D boxes of 1, 2 or 4 heads (rows of 256, 512, 1024 contiguous bytes), one CTA per
// SM streaming boxes through a ring of stages with no consumer work.  Prints GB/s per configuration.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_rows.cu -o tma_rows -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "../../paper_2506_04648_b200/csrc/sm100.cuh"
using namespace fpsa::sm100;

constexpr int kGT = 21, kGH = 45, kGW = 80, kH = 40, kD = 128, kST = 3, kSH = 5, kSW = 16;

template <int HB, int STAGES>
__global__ void __launch_bounds__(32, 1) stream(const __grid_constant__ CUtensorMap tm, int n_items, long long* clk) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[STAGES];
  constexpr uint32_t kBytes = kST * kSH * kSW * kD * 2 * HB;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncwarp();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    const int dh = kGH / kSH, dw = kGW / kSW, M = (kGT / kST) * dh * dw, groups = kH / HB;
    int k = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++k) {
      const int st = k % STAGES;
      if (k >= STAGES) mbar_wait(&full[st], ((k / STAGES) - 1) & 1);
      const int hg = it / M, u = it % M;
      const int ut = u / (dh * dw), uh = (u / dw) % dh, uw = u % dw;
      mbar_arrive_expect_tx(&full[st], kBytes);
      tma_load_5d(smem + st * kBytes, &tm, 0, hg * HB, uw * kSW, uh * kSH, ut * kST, &full[st]);
      (void)groups;
    }
    for (int j = k - STAGES < 0 ? 0 : k - STAGES; j < k; ++j) mbar_wait(&full[j % STAGES], (j / STAGES) & 1);
  }
  __syncwarp();
  if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
}

template <int HB, int STAGES>
void run(void* x, PFN_cuTensorMapEncodeTiled_v12000 enc) {
  CUtensorMap tm;
  cuuint64_t dims[5] = {kD, kH, kGW, kGH, kGT};
  cuuint64_t strides[4] = {kD * 2, (cuuint64_t)kH * kD * 2, (cuuint64_t)kH * kD * 2 * kGW,
                           (cuuint64_t)kH * kD * 2 * kGW * kGH};
  cuuint32_t box[5] = {kD, HB, kSW, kSH, kST};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed\n");
    return;
  }
  const int M = (kGT / kST) * (kGH / kSH) * (kGW / kSW), n_items = M * (kH / HB);
  const int smem = STAGES * kST * kSH * kSW * kD * 2 * HB;
  cudaFuncSetAttribute(stream<HB, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* clk;
  cudaMalloc(&clk, 148 * sizeof(long long));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    stream<HB, STAGES><<<148, 32, smem>>>(tm, n_items, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)kGT * kGH * kGW * kH * kD * 2;
  printf("heads per box %d, stages %d, box %6d B: %.3f ms  %.0f GB/s  (%s)\n", HB, STAGES,
         kST * kSH * kSW * kD * 2 * HB, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  void* x;
  const size_t n = (size_t)kGT * kGH * kGW * kH * kD;
  cudaMalloc(&x, n * 2);
  cudaMemset(x, 0, n * 2);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  run<1, 1>(x, enc);
  run<1, 2>(x, enc);
  run<1, 3>(x, enc);
  run<2, 1>(x, enc);
  run<4, 1>(x, enc);  // 245 KB box does not fit: expect a launch error
  return 0;
}
