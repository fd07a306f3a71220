// Fidelity sums on the device, per head: the inputs of the reference's
// cosine_similarity / mse / snr_db (/root/reference/pkg/src/fp8sta/metrics.py:41-88)
// so full-scale schedule sweeps can report fidelity without a host copy.
//
// out[h*6 + 0..5] (f64) = sum(r a), sum(r r), sum(a a), sum((r - a)^2), max|r|, max|a|
// over the tokens x d elements of head h; r = reference, a = approximation.
// The host finishes the metrics (paper_2506_04648_b200/metrics.py).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"

namespace fpsa {
namespace {

template <typename T>
__device__ __forceinline__ double ld(const T* p) {
  if constexpr (sizeof(T) == 4) return (double)*p;
  else return (double)__bfloat162float(*p);
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

template <typename TR, typename TA>
__global__ void __launch_bounds__(256) fidelity_kernel(const TR* __restrict__ r, const TA* __restrict__ a,
                                                       int64_t tokens, int32_t d, int64_t ts, int64_t hs,
                                                       double* __restrict__ out) {
  const int32_t h = blockIdx.y;
  double s[6] = {0, 0, 0, 0, 0, 0};
  const int64_t n = tokens * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / d, c = i % d;
    const int64_t off = t * ts + h * hs + c;
    const double x = ld(r + off), y = ld(a + off), e = x - y;
    s[0] += x * y;
    s[1] += x * x;
    s[2] += y * y;
    s[3] += e * e;
    s[4] = fmax(s[4], fabs(x));
    s[5] = fmax(s[5], fabs(y));
  }
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v = __shfl_xor_sync(0xffffffffu, s[k], o);
      s[k] = k < 4 ? s[k] + v : fmax(s[k], v);
    }
  __shared__ double part[8][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) part[warp][k] = s[k];
  __syncthreads();
  if (threadIdx.x < 6) {
    const int k = threadIdx.x;
    double v = part[0][k];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = k < 4 ? v + part[w][k] : fmax(v, part[w][k]);
    if (k < 4) atomicAdd(out + h * 6 + k, v);
    else atomic_max_nonneg(out + h * 6 + k, v);
  }
}

template <typename TR, typename TA>
void run(const void* r, const void* a, int64_t tokens, int32_t heads, int32_t d, int64_t ts, int64_t hs, double* out,
         cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n = tokens * d;
  const int bx = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8 / heads + 1));
  fidelity_kernel<TR, TA><<<dim3(bx, heads), 256, 0, st>>>(static_cast<const TR*>(r), static_cast<const TA*>(a), tokens,
                                                           d, ts, hs, out);
}

}  // namespace
}  // namespace fpsa

extern "C" int fpsa_fidelity(const void* ref, int ref_dtype, const void* approx, int approx_dtype, int64_t tokens,
                             int32_t heads, int32_t d, int64_t token_stride, int64_t head_stride, double* out,
                             void* stream) {
  fpsa::clear_error();
  if (!ref || !approx || !out) return fpsa::fail(FPSA_EINVAL, "null buffer");
  if (tokens < 1 || heads < 1 || d < 1) return fpsa::fail(FPSA_EINVAL, "empty problem");
  if ((ref_dtype != FPSA_F32 && ref_dtype != FPSA_BF16) || (approx_dtype != FPSA_F32 && approx_dtype != FPSA_BF16))
    return fpsa::fail(FPSA_EUNSUPPORTED, "fidelity inputs must be f32 or bf16");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(out, 0, sizeof(double) * 6 * heads, st) != cudaSuccess)
    return fpsa::fail(FPSA_ECUDA, std::string("fpsa_fidelity reset: ") + cudaGetErrorString(cudaGetLastError()));
  if (ref_dtype == FPSA_F32) {
    if (approx_dtype == FPSA_F32) fpsa::run<float, float>(ref, approx, tokens, heads, d, token_stride, head_stride, out, st);
    else fpsa::run<float, __nv_bfloat16>(ref, approx, tokens, heads, d, token_stride, head_stride, out, st);
  } else {
    if (approx_dtype == FPSA_F32) fpsa::run<__nv_bfloat16, float>(ref, approx, tokens, heads, d, token_stride, head_stride, out, st);
    else fpsa::run<__nv_bfloat16, __nv_bfloat16>(ref, approx, tokens, heads, d, token_stride, head_stride, out, st);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fpsa::fail(FPSA_ECUDA, std::string("fpsa_fidelity launch: ") + cudaGetErrorString(e));
  return FPSA_OK;
}
