// Tile-major FP8 quantisation kernels (K1: per-3D-tile Q/K, K2: per-channel V).
//
// Reference semantics (/root/reference/pkg/src/fp8sta):
//   quantize.py:102-108  scale = max(peak/max_value, f64 tiny); 1.0 if peak == 0
//   quantize.py:111-124  one scale per 3D tile over all tv*d entries (Q, K)
//   quantize.py:127-134  one scale per column over all L rows (V)
//   fp8.py:153-188       codes = RNE(x_f64 / scale) onto the fp8 grid, saturating,
//                        sign bit kept for values that round to zero
//   grid.py:132-154      tile-major row order (tiles row-major, tokens row-major inside)
//
// Bit-exactness: the reference divides in float64 and rounds the f64 quotient
// to fp8.  Here every element first takes a fast f32 path: a = x * f32(1/s)
// is within 2^-22 relative of the quotient, so if the two f32 values
// a*(1 -+ 2^-20) convert to the same fp8 code (hardware cvt.rn.satfinite,
// exact RNE, verified exhaustively on the device), that code is the RNE of
// the exact f64 quotient.  Otherwise (about 1 element in 30k) the element is
// recomputed exactly: q = x / s in f64, rounded to f32 with round-to-odd,
// then converted (round-to-odd to 24 bits followed by RNE to <= 4 bits equals
// direct RNE).  Compile without FTZ: signed zeros and f32 subnormals matter.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"

namespace fpsa {
namespace {

constexpr int kQuantThreads = 256;
constexpr int kQuantWarps = kQuantThreads / 32;

struct Geometry {
  int32_t gt, gh, gw;  // token grid
  int32_t st, sh, sw;  // tile extents
  int32_t dt, dh, dw;  // tiles per axis
  int32_t tv;          // tile volume
  int32_t M;           // tiles
  int32_t pitch;       // rows per tile slot in the code matrix
  int32_t natural;     // input in natural (t,h,w) order; else tile-contiguous
};

// Token index of local row r of flat tile u.
__device__ __forceinline__ int64_t token_of(const Geometry& g, int32_t u, int32_t r) {
  if (!g.natural) return (int64_t)u * g.tv + r;
  const int32_t ut = u / (g.dh * g.dw), uh = (u / g.dw) % g.dh, uw = u % g.dw;
  const int32_t lt = r / (g.sh * g.sw), lh = (r / g.sw) % g.sh, lw = r % g.sw;
  const int64_t t = (int64_t)ut * g.st + lt, h = (int64_t)uh * g.sh + lh, w = (int64_t)uw * g.sw + lw;
  return (t * g.gh + h) * g.gw + w;
}

template <typename T, int VEC>
struct Loader;
template <int VEC>
struct Loader<float, VEC> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[VEC]) {
    if constexpr (VEC == 4) {
      float4 a = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
      float2 a = __ldg(reinterpret_cast<const float2*>(p));
      v[0] = a.x; v[1] = a.y;
    }
  }
};
template <int VEC>
struct Loader<__nv_bfloat16, VEC> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&v)[VEC]) {
    if constexpr (VEC == 4) {
      uint2 a = __ldg(reinterpret_cast<const uint2*>(p));
      v[0] = __uint_as_float(a.x << 16); v[1] = __uint_as_float(a.x & 0xFFFF0000u);
      v[2] = __uint_as_float(a.y << 16); v[3] = __uint_as_float(a.y & 0xFFFF0000u);
    } else {
      uint32_t a = __ldg(reinterpret_cast<const unsigned int*>(p));
      v[0] = __uint_as_float(a << 16); v[1] = __uint_as_float(a & 0xFFFF0000u);
    }
  }
};

// cvt.rn.satfinite of a pair; `hi` lands in the upper byte.
template <int FMT>
__device__ __forceinline__ uint32_t cvt_pair(float hi, float lo) {
  uint16_t r;
  if constexpr (FMT == FPSA_E4M3)
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  else
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

// Exact code of the f64 quotient x / s (slow path).
template <int FMT>
__device__ __noinline__ uint32_t encode_exact(float x, double s) {
  const double q = __ddiv_rn((double)x, s);
  float f = __double2float_rz(q);
  if ((double)f != q) f = __uint_as_float(__float_as_uint(f) | 1u);  // round to odd
  return cvt_pair<FMT>(0.0f, f) & 0xFFu;
}

// Codes of two elements sharing (or not) a scale.
template <int FMT>
__device__ __forceinline__ uint32_t encode2(float x0, float x1, double s0, double s1, float r0, float r1,
                                            bool fast_ok) {
  const float a0 = x0 * r0, a1 = x1 * r1;
  const float kLo = 0.99999904632568359375f, kHi = 1.00000095367431640625f;  // 1 -+ 2^-20
  const uint32_t clo = cvt_pair<FMT>(a1 * kLo, a0 * kLo);
  const uint32_t chi = cvt_pair<FMT>(a1 * kHi, a0 * kHi);
  if (fast_ok && clo == chi) return clo;
  uint32_t c0 = clo & 0xFFu, c1 = clo >> 8;
  if (!fast_ok || c0 != (chi & 0xFFu)) c0 = encode_exact<FMT>(x0, s0);
  if (!fast_ok || c1 != (chi >> 8)) c1 = encode_exact<FMT>(x1, s1);
  return c0 | (c1 << 8);
}

__device__ __forceinline__ bool finite_f(float v) { return fabsf(v) <= FLT_MAX; }

__device__ __forceinline__ double scale_of(float peak, double maxv) {
  if (peak == 0.0f) return 1.0;
  const double s = __ddiv_rn((double)peak, maxv);
  return s > DBL_MIN ? s : DBL_MIN;
}
__device__ __forceinline__ bool rcp_ok(float r) { return r >= FLT_MIN && r <= FLT_MAX; }

template <typename T, int D, int FMT>
__global__ void __launch_bounds__(kQuantThreads)
    quant_tile_kernel(const T* __restrict__ x, int64_t token_stride, int64_t head_stride, Geometry g,
                      uint8_t* __restrict__ codes, double* __restrict__ scales, int32_t* err) {
  constexpr int VEC = D / 32;
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  const int32_t u = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* xh = x + (int64_t)h * head_stride + lane * VEC;

  // pass 1: tile amax (exact: max of |x| over the tile)
  float peak = 0.0f;
  bool bad = false;
#pragma unroll 4
  for (int32_t r = warp; r < g.tv; r += kQuantWarps) {
    float v[VEC];
    Loader<T, VEC>::load(xh + token_of(g, u, r) * token_stride, v);
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      bad |= !finite_f(v[i]);
      peak = fmaxf(peak, fabsf(v[i]));
    }
  }
  __shared__ float s_peak[kQuantWarps];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, o));
  __syncthreads();
  if (bad) s_bad = 1;
  if (lane == 0) s_peak[warp] = peak;
  __syncthreads();
  peak = s_peak[0];
#pragma unroll
  for (int i = 1; i < kQuantWarps; ++i) peak = fmaxf(peak, s_peak[i]);
  if (s_bad && err) {
    if (threadIdx.x == 0) atomicOr(err, 1);
  }
  const double s = scale_of(peak, kMax);
  const float r = (float)(1.0 / s);
  const bool fast = rcp_ok(r);

  // pass 2: codes (re-read hits L2)
  uint8_t* out = codes + ((int64_t)h * g.M + u) * g.pitch * D + lane * VEC;
#pragma unroll 4
  for (int32_t row = warp; row < g.tv; row += kQuantWarps) {
    float v[VEC];
    Loader<T, VEC>::load(xh + token_of(g, u, row) * token_stride, v);
    if constexpr (VEC == 4) {
      const uint32_t lo = encode2<FMT>(v[0], v[1], s, s, r, r, fast);
      const uint32_t hi = encode2<FMT>(v[2], v[3], s, s, r, r, fast);
      *reinterpret_cast<uint32_t*>(out + (int64_t)row * D) = lo | (hi << 16);
    } else {
      *reinterpret_cast<uint16_t*>(out + (int64_t)row * D) = (uint16_t)encode2<FMT>(v[0], v[1], s, s, r, r, fast);
    }
  }
  for (int32_t row = g.tv + warp; row < g.pitch; row += kQuantWarps) {
    if constexpr (VEC == 4)
      *reinterpret_cast<uint32_t*>(out + (int64_t)row * D) = 0u;
    else
      *reinterpret_cast<uint16_t*>(out + (int64_t)row * D) = 0;
  }
  if (threadIdx.x == 0) scales[(int64_t)h * g.M + u] = s;
}

// V pass A: per-(head, channel) amax over all tokens, as uint bits of |x|.
template <typename T, int D>
__global__ void __launch_bounds__(kQuantThreads)
    chan_amax_kernel(const T* __restrict__ x, int64_t token_stride, int64_t head_stride, int64_t L,
                     int32_t rows_per_block, uint32_t* __restrict__ amax, int32_t* err) {
  constexpr int VEC = D / 32;
  const int32_t h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t t1 = min(L, t0 + rows_per_block);
  const T* xh = x + (int64_t)h * head_stride + lane * VEC;
  float m[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) m[i] = 0.0f;
  bool bad = false;
#pragma unroll 4
  for (int64_t t = t0 + warp; t < t1; t += kQuantWarps) {
    float v[VEC];
    Loader<T, VEC>::load(xh + t * token_stride, v);
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      bad |= !finite_f(v[i]);
      m[i] = fmaxf(m[i], fabsf(v[i]));
    }
  }
  __shared__ float s_m[kQuantWarps][D];
#pragma unroll
  for (int i = 0; i < VEC; ++i) s_m[warp][lane * VEC + i] = m[i];
  if (bad && err) atomicOr(err, 1);
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += kQuantThreads) {
    float mm = s_m[0][c];
#pragma unroll
    for (int w = 1; w < kQuantWarps; ++w) mm = fmaxf(mm, s_m[w][c]);
    atomicMax(amax + (int64_t)h * D + c, __float_as_uint(mm));
  }
}

// V pass B: codes with per-channel scales, tile-major padded layout.
template <typename T, int D, int FMT>
__global__ void __launch_bounds__(kQuantThreads)
    quant_chan_kernel(const T* __restrict__ x, int64_t token_stride, int64_t head_stride, Geometry g,
                      const uint32_t* __restrict__ amax, uint8_t* __restrict__ codes, double* __restrict__ scales) {
  constexpr int VEC = D / 32;
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  const int32_t u = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s[VEC];
  float r[VEC];
  bool fast = true;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const float peak = __uint_as_float(amax[(int64_t)h * D + lane * VEC + i]);
    s[i] = scale_of(peak, kMax);
    r[i] = (float)(1.0 / s[i]);
    fast &= rcp_ok(r[i]);
  }
  if (u == 0 && warp == 0) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) scales[(int64_t)h * D + lane * VEC + i] = s[i];
  }
  const T* xh = x + (int64_t)h * head_stride + lane * VEC;
  uint8_t* out = codes + ((int64_t)h * g.M + u) * g.pitch * D + lane * VEC;
#pragma unroll 4
  for (int32_t row = warp; row < g.tv; row += kQuantWarps) {
    float v[VEC];
    Loader<T, VEC>::load(xh + token_of(g, u, row) * token_stride, v);
    if constexpr (VEC == 4) {
      const uint32_t lo = encode2<FMT>(v[0], v[1], s[0], s[1], r[0], r[1], fast);
      const uint32_t hi = encode2<FMT>(v[2], v[3], s[2], s[3], r[2], r[3], fast);
      *reinterpret_cast<uint32_t*>(out + (int64_t)row * D) = lo | (hi << 16);
    } else {
      *reinterpret_cast<uint16_t*>(out + (int64_t)row * D) =
          (uint16_t)encode2<FMT>(v[0], v[1], s[0], s[1], r[0], r[1], fast);
    }
  }
  for (int32_t row = g.tv + warp; row < g.pitch; row += kQuantWarps) {
    if constexpr (VEC == 4)
      *reinterpret_cast<uint32_t*>(out + (int64_t)row * D) = 0u;
    else
      *reinterpret_cast<uint16_t*>(out + (int64_t)row * D) = 0;
  }
}

int make_geometry(fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t pitch, int in_order, Geometry* g) {
  fpsa_dims3 td;
  if (int st = fpsa_tile_grid(grid, tile, &td)) return st;
  if (d != 64 && d != 128) return fail(FPSA_EUNSUPPORTED, "head dim must be 64 or 128, got " + std::to_string(d));
  const int32_t tv = tile.t * tile.h * tile.w;
  if (pitch < tv) return fail(FPSA_EINVAL, "tile_pitch smaller than the tile volume");
  if (in_order != FPSA_ORDER_TILE && in_order != FPSA_ORDER_NATURAL) return fail(FPSA_EINVAL, "bad token order");
  *g = Geometry{grid.t, grid.h, grid.w, tile.t, tile.h, tile.w, td.t, td.h, td.w,
                tv,     td.t * td.h * td.w, pitch, in_order == FPSA_ORDER_NATURAL};
  return FPSA_OK;
}

int check_common(const void* x, int dtype, int32_t heads, int fmt, const void* codes, const void* scales) {
  if (!x || !codes || !scales) return fail(FPSA_EINVAL, "null buffer");
  if (heads < 1) return fail(FPSA_EINVAL, "heads must be >= 1");
  if (dtype != FPSA_F32 && dtype != FPSA_BF16) return fail(FPSA_EUNSUPPORTED, "input dtype must be f32 or bf16");
  if (fmt != FPSA_E4M3 && fmt != FPSA_E5M2) return fail(FPSA_EINVAL, "fmt must be e4m3 or e5m2");
  return FPSA_OK;
}

int cuda_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FPSA_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return FPSA_OK;
}

template <typename T, int D, int FMT>
void launch_qk(const void* x, int64_t ts, int64_t hs, int32_t heads, const Geometry& g, uint8_t* codes,
               double* scales, int32_t* err, cudaStream_t st) {
  dim3 grid(g.M, heads);
  quant_tile_kernel<T, D, FMT><<<grid, kQuantThreads, 0, st>>>(static_cast<const T*>(x), ts, hs, g, codes, scales, err);
}

template <typename T, int D, int FMT>
void launch_v(const void* x, int64_t ts, int64_t hs, int32_t heads, const Geometry& g, uint8_t* codes,
              double* scales, uint32_t* amax, int32_t* err, cudaStream_t st) {
  const int64_t L = (int64_t)g.gt * g.gh * g.gw;
  const int32_t rows_per_block = 256;
  dim3 ga((unsigned)((L + rows_per_block - 1) / rows_per_block), heads);
  chan_amax_kernel<T, D><<<ga, kQuantThreads, 0, st>>>(static_cast<const T*>(x), ts, hs, L, rows_per_block, amax, err);
  dim3 gb(g.M, heads);
  quant_chan_kernel<T, D, FMT><<<gb, kQuantThreads, 0, st>>>(static_cast<const T*>(x), ts, hs, g, amax, codes, scales);
}

template <template <typename, int, int> class F, typename... Args>
void dispatch(int dtype, int32_t d, int fmt, Args&&... args) {
  if (dtype == FPSA_F32) {
    if (d == 128) {
      if (fmt == FPSA_E4M3) F<float, 128, FPSA_E4M3>::run(args...); else F<float, 128, FPSA_E5M2>::run(args...);
    } else {
      if (fmt == FPSA_E4M3) F<float, 64, FPSA_E4M3>::run(args...); else F<float, 64, FPSA_E5M2>::run(args...);
    }
  } else {
    if (d == 128) {
      if (fmt == FPSA_E4M3) F<__nv_bfloat16, 128, FPSA_E4M3>::run(args...); else F<__nv_bfloat16, 128, FPSA_E5M2>::run(args...);
    } else {
      if (fmt == FPSA_E4M3) F<__nv_bfloat16, 64, FPSA_E4M3>::run(args...); else F<__nv_bfloat16, 64, FPSA_E5M2>::run(args...);
    }
  }
}

template <typename T, int D, int FMT>
struct RunQK {
  template <typename... A>
  static void run(A... a) { launch_qk<T, D, FMT>(a...); }
};
template <typename T, int D, int FMT>
struct RunV {
  template <typename... A>
  static void run(A... a) { launch_v<T, D, FMT>(a...); }
};

}  // namespace
}  // namespace fpsa

using namespace fpsa;

extern "C" int fpsa_quantize_qk(const void* x, int dtype, int64_t token_stride, int64_t head_stride, int32_t heads,
                                fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, int in_order,
                                int fmt, uint8_t* codes, double* scales, int32_t* err_flag, void* stream) {
  clear_error();
  if (int s = check_common(x, dtype, heads, fmt, codes, scales)) return s;
  Geometry g;
  if (int s = make_geometry(grid, tile, d, tile_pitch, in_order, &g)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dispatch<RunQK>(dtype, d, fmt, x, token_stride, head_stride, heads, g, codes, scales, err_flag, st);
  return cuda_status("fpsa_quantize_qk");
}

extern "C" int fpsa_quantize_v(const void* x, int dtype, int64_t token_stride, int64_t head_stride, int32_t heads,
                               fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, int in_order, int fmt,
                               uint8_t* codes, double* scales, void* workspace, int32_t* err_flag, void* stream) {
  clear_error();
  if (int s = check_common(x, dtype, heads, fmt, codes, scales)) return s;
  if (!workspace) return fail(FPSA_EINVAL, "workspace is NULL");
  Geometry g;
  if (int s = make_geometry(grid, tile, d, tile_pitch, in_order, &g)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* amax = static_cast<uint32_t*>(workspace);
  if (cudaMemsetAsync(amax, 0, (size_t)heads * d * sizeof(uint32_t), st) != cudaSuccess)
    return cuda_status("fpsa_quantize_v memset");
  dispatch<RunV>(dtype, d, fmt, x, token_stride, head_stride, heads, g, codes, scales, amax, err_flag, st);
  return cuda_status("fpsa_quantize_v");
}
