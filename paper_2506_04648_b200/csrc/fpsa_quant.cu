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
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include <cfloat>
#include <cstdint>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"
#include "sm100.cuh"

namespace fpsa {
namespace {

constexpr int kQuantThreads = 512;
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

// First token of flat tile u (natural order) or of its tile-contiguous row block.
__device__ __forceinline__ int32_t tile_base(const Geometry& g, int32_t u) {
  if (!g.natural) return u * g.tv;
  const int32_t ut = u / (g.dh * g.dw), uh = (u / g.dw) % g.dh, uw = u % g.dw;
  return ((ut * g.st) * g.gh + uh * g.sh) * g.gw + uw * g.sw;
}
// Token offset of local row r from the tile base (identical for every tile).
__device__ __forceinline__ int32_t local_offset(const Geometry& g, int32_t r) {
  if (!g.natural) return r;
  const int32_t lt = r / (g.sh * g.sw), lh = (r / g.sw) % g.sh, lw = r % g.sw;
  return (lt * g.gh + lh) * g.gw + lw;
}

// Per-CTA table of row offsets (in elements), built once with one division
// chain per row instead of per row per pass.
constexpr int kMaxTableRows = 2048;
__device__ __forceinline__ void build_row_table(const Geometry& g, int64_t token_stride, int64_t* table) {
  if (g.natural)
    for (int32_t r = threadIdx.x; r < min(g.tv, kMaxTableRows); r += blockDim.x)
      table[r] = (int64_t)local_offset(g, r) * token_stride;
  __syncthreads();
}
// Element offset of local row r from the tile's first token (tiles above kMaxTableRows tokens: computed).
__device__ __forceinline__ int64_t row_offset(const Geometry& g, const int64_t* table, int32_t r, int64_t ts) {
  if (!g.natural) return (int64_t)r * ts;
  return r < kMaxTableRows ? table[r] : (int64_t)local_offset(g, r) * ts;
}

// Raw vector of VEC consecutive channels (16-bit inputs stay packed in registers).
template <typename T, int VEC>
struct Vec;
template <>
struct Vec<float, 4> {
  using raw = float4;
  static __device__ __forceinline__ raw load(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ void unpack(const raw& a, float (&v)[4]) { v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; }
};
template <>
struct Vec<float, 2> {
  using raw = float2;
  static __device__ __forceinline__ raw load(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
  static __device__ __forceinline__ void unpack(const raw& a, float (&v)[2]) { v[0] = a.x; v[1] = a.y; }
};
template <>
struct Vec<__nv_bfloat16, 4> {
  using raw = uint2;
  static __device__ __forceinline__ raw load(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }
  static __device__ __forceinline__ void unpack(const raw& a, float (&v)[4]) {
    v[0] = __uint_as_float(a.x << 16); v[1] = __uint_as_float(a.x & 0xFFFF0000u);
    v[2] = __uint_as_float(a.y << 16); v[3] = __uint_as_float(a.y & 0xFFFF0000u);
  }
};
template <>
struct Vec<__nv_bfloat16, 2> {
  using raw = uint32_t;
  static __device__ __forceinline__ raw load(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const unsigned int*>(p)); }
  static __device__ __forceinline__ void unpack(const raw& a, float (&v)[2]) {
    v[0] = __uint_as_float(a << 16); v[1] = __uint_as_float(a & 0xFFFF0000u);
  }
};
template <typename T, int VEC>
struct Loader {
  static __device__ __forceinline__ void load(const T* p, float (&v)[VEC]) { Vec<T, VEC>::unpack(Vec<T, VEC>::load(p), v); }
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
__device__ __forceinline__ uint32_t encode_exact_inl(float x, double s) {
  const double q = __ddiv_rn((double)x, s);
  float f = __double2float_rz(q);
  if ((double)f != q) f = __uint_as_float(__float_as_uint(f) | 1u);  // round to odd
  return cvt_pair<FMT>(0.0f, f) & 0xFFu;
}
template <int FMT>
__device__ __noinline__ uint32_t encode_exact(float x, double s) {
  return encode_exact_inl<FMT>(x, s);
}

__device__ __forceinline__ double scale_of(float peak, double maxv) {
  if (peak == 0.0f) return 1.0;
  const double s = __ddiv_rn((double)peak, maxv);
  return s > DBL_MIN ? s : DBL_MIN;
}

// Per-scale constants of the fast path: f32(1/s) * (1 -+ 2^-20).
struct Bracket {
  float lo, hi;
  bool ok;
};
__device__ __forceinline__ Bracket bracket_of(double s) {
  const float r = (float)(1.0 / s);
  const bool ok = r >= FLT_MIN && r <= FLT_MAX / 2;
  return Bracket{r * 0.99999904632568359375f, r * 1.00000095367431640625f, ok};
}

// Same bracket from the f32 peak without f64 arithmetic: r = f32(max_value/peak)
// is within one f32 ulp of f32(1/s) with s = f64(peak/max_value), and the
// bracket margin (2^-20) covers that ulp plus the two roundings below.
template <int FMT>
__device__ __forceinline__ Bracket bracket_f32(float peak) {
  constexpr float kMaxF = FMT == FPSA_E4M3 ? 448.0f : 57344.0f;
  if (peak == 0.0f) return Bracket{0.99999904632568359375f, 1.00000095367431640625f, true};
  const float r = __fdiv_rn(kMaxF, peak);
  const bool ok = r >= FLT_MIN && r <= FLT_MAX / 2 && peak >= FLT_MIN;
  return Bracket{r * 0.99999904632568359375f, r * 1.00000095367431640625f, ok};
}

__device__ __forceinline__ void mul2(float a0, float a1, float b0, float b1, float& d0, float& d1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// Fast codes of VEC elements: the two bracket values x*lo and x*hi round to
// the same fp8 code iff that code is the RNE of the exact f64 quotient (see
// header).  `slow` is raised when any element needs the exact path.
template <int FMT, int VEC>
__device__ __forceinline__ uint32_t encode_fast(const float (&v)[VEC], const Bracket (&b)[VEC], bool& slow) {
  uint32_t clo = 0, chi = 0;
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    float l0, l1, h0, h1;
    mul2(v[e], v[e + 1], b[e].lo, b[e + 1].lo, l0, l1);
    mul2(v[e], v[e + 1], b[e].hi, b[e + 1].hi, h0, h1);
    clo |= cvt_pair<FMT>(l1, l0) << (8 * e);
    chi |= cvt_pair<FMT>(h1, h0) << (8 * e);
  }
  slow |= clo != chi;
  return clo;
}

// Scalar arguments, not array references: a reference to a register array forces
// the caller to keep that array in local memory around every call site.
template <int FMT, int VEC>
__device__ __noinline__ uint32_t encode_slow4(float v0, float v1, float v2, float v3, float p0, float p1, float p2,
                                              float p3) {
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  const float v[4] = {v0, v1, v2, v3}, peak[4] = {p0, p1, p2, p3};
  uint32_t c = 0;
#pragma unroll
  for (int e = 0; e < VEC; ++e) c |= encode_exact<FMT>(v[e], scale_of(peak[e], kMax)) << (8 * e);
  return c;
}
template <int FMT, int VEC>
__device__ __forceinline__ uint32_t encode_slow(const float (&v)[VEC], const float (&peak)[VEC]) {
  if constexpr (VEC == 4)
    return encode_slow4<FMT, 4>(v[0], v[1], v[2], v[3], peak[0], peak[1], peak[2], peak[3]);
  else
    return encode_slow4<FMT, 2>(v[0], v[1], 0.0f, 0.0f, peak[0], peak[1], 0.0f, 0.0f);
}

#ifndef FPSA_QUANT_STORE
#define FPSA_QUANT_STORE 0  // measurement switch: 0 st.global, 1 st.global.cs (streaming), 2 no code stores
#endif
template <int VEC>
__device__ __forceinline__ void store_codes(uint8_t* p, uint32_t c) {
  if constexpr (VEC == 4) {
    if constexpr (FPSA_QUANT_STORE == 1)
      asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(c) : "memory");
    else if constexpr (FPSA_QUANT_STORE == 2)
      asm volatile("" ::"l"(p), "r"(c));
    else
      *reinterpret_cast<uint32_t*>(p) = c;
  } else {
    *reinterpret_cast<uint16_t*>(p) = (uint16_t)c;
  }
}

// |x| max in the bit domain (exact for floats; NaN/inf bit patterns sort above
// every finite value, so one compare at the end detects non-finite input).
template <typename T, int VEC>
__device__ __forceinline__ uint32_t absmax_bits(const typename Vec<T, VEC>::raw& a, uint32_t m);
template <>
__device__ __forceinline__ uint32_t absmax_bits<__nv_bfloat16, 4>(const uint2& a, uint32_t m) {
  return __vmaxu2(__vmaxu2(m, a.x & 0x7FFF7FFFu), a.y & 0x7FFF7FFFu);
}
template <>
__device__ __forceinline__ uint32_t absmax_bits<__nv_bfloat16, 2>(const uint32_t& a, uint32_t m) {
  return __vmaxu2(m, a & 0x7FFF7FFFu);
}
template <>
__device__ __forceinline__ uint32_t absmax_bits<float, 4>(const float4& a, uint32_t m) {
  m = max(m, __float_as_uint(a.x) & 0x7FFFFFFFu);
  m = max(m, __float_as_uint(a.y) & 0x7FFFFFFFu);
  m = max(m, __float_as_uint(a.z) & 0x7FFFFFFFu);
  return max(m, __float_as_uint(a.w) & 0x7FFFFFFFu);
}
template <>
__device__ __forceinline__ uint32_t absmax_bits<float, 2>(const float2& a, uint32_t m) {
  m = max(m, __float_as_uint(a.x) & 0x7FFFFFFFu);
  return max(m, __float_as_uint(a.y) & 0x7FFFFFFFu);
}
// Reduce the packed accumulator to a float |x| max.
template <typename T>
__device__ __forceinline__ float bits_to_peak(uint32_t m) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t hi = max(m & 0xFFFFu, m >> 16);
    return __uint_as_float(hi << 16);
  } else {
    return __uint_as_float(m);
  }
}

constexpr int kRegRows = 16;  // rows per warp kept in registers (16-bit inputs, tv <= 256)

// One tensor of a fused quantisation launch.
struct QuantJob {
  const void* x;
  int64_t ts, hs;    // token / head strides (elements)
  uint8_t* codes;    // tile-major padded [heads*M*pitch][D]
  double* scales;    // per-tile [heads*M] or per-channel [heads*D]
  int32_t channel;   // 0: one scale per 3D tile, 1: per-channel scale from `amax`
};
struct QuantArgs {
  QuantJob job[3];
  const uint32_t* amax;  // per-(head, channel) |x| max bits for channel jobs
  int32_t* err;
};

// blockIdx = (tile u, head h, job z).  Q/K: tile amax -> f64 scale -> codes;
// V: codes with the per-channel scales of a preceding chan_amax_kernel.
template <typename T, int D, int FMT>
__global__ void __launch_bounds__(kQuantThreads, 1)
    quant_kernel(Geometry g, QuantArgs a) {
  constexpr int VEC = D / 32;
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  constexpr bool kRegCapable = sizeof(T) == 2;
  using V = Vec<T, VEC>;
  __shared__ int64_t s_row[kMaxTableRows];
  __shared__ uint32_t s_peak[kQuantWarps];
  const QuantJob job = a.job[blockIdx.z];
  const int32_t u = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  build_row_table(g, job.ts, s_row);
  const T* xt = static_cast<const T*>(job.x) + (int64_t)h * job.hs + (int64_t)tile_base(g, u) * job.ts + lane * VEC;
  uint8_t* out = job.codes + ((int64_t)h * g.M + u) * g.pitch * D + lane * VEC;
  const bool in_regs = kRegCapable && g.tv <= kQuantWarps * kRegRows;
  typename V::raw raw[kRegCapable ? kRegRows : 1];
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < (kRegCapable ? kRegRows : 1); ++i) {
      const int32_t r = min(warp + i * kQuantWarps, g.tv - 1);  // clamped: no branch around the load
      raw[i] = V::load(xt + row_offset(g, s_row, r, job.ts));
    }
  }
  float pk[VEC];  // |x| max behind each element's scale (0 for non-finite input)
  Bracket b[VEC];
  if (!job.channel) {
    uint32_t m = 0;
    if (in_regs) {
#pragma unroll
      for (int i = 0; i < (kRegCapable ? kRegRows : 1); ++i)
        if (warp + i * kQuantWarps < g.tv) m = absmax_bits<T, VEC>(raw[i], m);
    } else {
#pragma unroll 4
      for (int32_t r = warp; r < g.tv; r += kQuantWarps) m = absmax_bits<T, VEC>(V::load(xt + row_offset(g, s_row, r, job.ts)), m);
    }
    // fold the packed lanes to f32 bit patterns first: those compare as integers
    m = __float_as_uint(bits_to_peak<T>(m));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_peak[warp] = m;
    __syncthreads();
    m = s_peak[0];
#pragma unroll
    for (int i = 1; i < kQuantWarps; ++i) m = max(m, s_peak[i]);
    float peak = __uint_as_float(m);
    if (!(peak <= FLT_MAX)) {
      if (threadIdx.x == 0 && a.err) atomicOr(a.err, 1);
      peak = 0.0f;
    }
    const double sc = scale_of(peak, kMax);
    const Bracket bb = bracket_of(sc);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      pk[e] = peak;
      b[e] = bb;
    }
    if (threadIdx.x == 0) job.scales[(int64_t)h * g.M + u] = sc;
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float peak = __uint_as_float(a.amax[(int64_t)h * D + lane * VEC + e]);
      pk[e] = peak <= FLT_MAX ? peak : 0.0f;
      const double sc = scale_of(pk[e], kMax);
      b[e] = bracket_of(sc);
      if (u == 0 && warp == 0) job.scales[(int64_t)h * D + lane * VEC + e] = sc;
    }
  }
  bool fast_ok = true;
#pragma unroll
  for (int e = 0; e < VEC; ++e) fast_ok &= b[e].ok;

  // Fast codes for every row; the rare rows whose bracket straddles a rounding
  // boundary are redone exactly afterwards, outside the streaming loop.
  bool any_slow = !fast_ok;
  auto emit = [&](int32_t row, const typename V::raw& rw) {
    float v[VEC];
    V::unpack(rw, v);
    bool slow = false;
    const uint32_t c = encode_fast<FMT, VEC>(v, b, slow);
    any_slow |= slow;
    store_codes<VEC>(out + (int64_t)row * D, c);
  };
  auto fixup = [&](int32_t row, const typename V::raw& rw) {
    float v[VEC];
    V::unpack(rw, v);
    bool slow = !fast_ok;
    encode_fast<FMT, VEC>(v, b, slow);
    if (slow) store_codes<VEC>(out + (int64_t)row * D, encode_slow<FMT, VEC>(v, pk));
  };
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < (kRegCapable ? kRegRows : 1); ++i) {
      const int32_t row = warp + i * kQuantWarps;
      if (row < g.tv) emit(row, raw[i]);
    }
    if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
      for (int i = 0; i < (kRegCapable ? kRegRows : 1); ++i) {
        const int32_t row = warp + i * kQuantWarps;
        if (row < g.tv) fixup(row, raw[i]);
      }
    }
  } else {
#pragma unroll 4
    for (int32_t row = warp; row < g.tv; row += kQuantWarps) emit(row, V::load(xt + row_offset(g, s_row, row, job.ts)));
    if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll 1
      for (int32_t row = warp; row < g.tv; row += kQuantWarps) fixup(row, V::load(xt + row_offset(g, s_row, row, job.ts)));
    }
  }
  for (int32_t row = g.tv + warp; row < g.pitch; row += kQuantWarps) store_codes<VEC>(out + (int64_t)row * D, 0u);
}

// ---------------------------------------------------------------------------
// Chunked two-pass quantiser for tiles the TMA kernel cannot stage (more than
// 256 tokens, e.g. the C4 early / late regimes' 1680- and 504-token tiles):
// every CTA takes 128 rows of one tile, pass 1 reduces the chunk's |x| max
// into the tile's slot (atomicMax on the f32 bits), pass 2 -- a second
// launch -- encodes the chunk with the tile's scale, pass 3 turns the slots
// into the f64 scales.  The slot of tile (h, u) is the low word of its own
// (zeroed) f64 scale, so no workspace is needed.  Streaming grids of many
// small CTAs instead of one CTA walking a whole tile twice.
constexpr int kChunkRows = 128;
constexpr int kChunkThreads = 256;
constexpr int kChunkWarps = kChunkThreads / 32;

// element offset of local row r of tile u (natural or tile order)
__device__ __forceinline__ int64_t chunk_row_offset(const Geometry& g, int32_t r, int64_t ts) {
  return (g.natural ? (int64_t)local_offset(g, r) : (int64_t)r) * ts;
}

__device__ __forceinline__ uint32_t* amax_slot(const QuantJob& job, int32_t h, int32_t u, int32_t M) {
  return reinterpret_cast<uint32_t*>(job.scales + (int64_t)h * M + u);
}

// pass 3: f64 scales from the tile max slots, in place
template <int FMT>
__global__ void scales_from_amax_kernel(double* scales, int64_t n, int32_t* err) {
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float peak = __uint_as_float(*reinterpret_cast<const uint32_t*>(scales + i));
    if (!(peak <= FLT_MAX)) {
      if (err) atomicOr(err, 1);
      peak = 0.0f;
    }
    scales[i] = scale_of(peak, kMax);
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(kChunkThreads) tile_amax_chunk_kernel(Geometry g, QuantArgs a, int32_t chunks) {
  constexpr int VEC = D / 32;
  using V = Vec<T, VEC>;
  __shared__ int64_t s_off[kChunkRows];
  __shared__ uint32_t s_m;
  const int32_t u = blockIdx.x / chunks, c = blockIdx.x % chunks, h = blockIdx.y, z = blockIdx.z;
  const QuantJob job = a.job[z];
  if (job.channel) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t r0 = c * kChunkRows, nr = min(kChunkRows, g.tv - r0);
  if (threadIdx.x < nr) s_off[threadIdx.x] = chunk_row_offset(g, r0 + threadIdx.x, job.ts);
  if (threadIdx.x == 0) s_m = 0u;
  __syncthreads();
  const T* xt = static_cast<const T*>(job.x) + (int64_t)h * job.hs + (int64_t)tile_base(g, u) * job.ts + lane * VEC;
  uint32_t m = 0;
#pragma unroll 4
  for (int32_t r = warp; r < nr; r += kChunkWarps) m = absmax_bits<T, VEC>(V::load(xt + s_off[r]), m);
  m = __float_as_uint(bits_to_peak<T>(m));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMax(&s_m, m);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(amax_slot(job, h, u, g.M), s_m);
}

template <typename T, int D, int FMT>
__global__ void __launch_bounds__(kChunkThreads) encode_chunk_kernel(Geometry g, QuantArgs a, int32_t chunks) {
  constexpr int VEC = D / 32;
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  using V = Vec<T, VEC>;
  __shared__ int64_t s_off[kChunkRows];
  const int32_t u = blockIdx.x / chunks, c = blockIdx.x % chunks, h = blockIdx.y, z = blockIdx.z;
  const QuantJob job = a.job[z];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t r0 = c * kChunkRows, nr = min(kChunkRows, g.tv - r0);
  if (threadIdx.x < nr) s_off[threadIdx.x] = chunk_row_offset(g, r0 + threadIdx.x, job.ts);
  __syncthreads();
  float pk[VEC];
  Bracket b[VEC];
  if (!job.channel) {
    float peak = __uint_as_float(*amax_slot(job, h, u, g.M));
    if (!(peak <= FLT_MAX)) peak = 0.0f;  // reported by scales_from_amax_kernel
    const Bracket bb = bracket_f32<FMT>(peak);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      pk[e] = peak;
      b[e] = bb;
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float peak = __uint_as_float(a.amax[(int64_t)h * D + lane * VEC + e]);
      pk[e] = peak <= FLT_MAX ? peak : 0.0f;
      b[e] = bracket_f32<FMT>(pk[e]);
      if (u == 0 && c == 0 && warp == 0) job.scales[(int64_t)h * D + lane * VEC + e] = scale_of(pk[e], kMax);
    }
  }
  bool fast_ok = true;
#pragma unroll
  for (int e = 0; e < VEC; ++e) fast_ok &= b[e].ok;
  const T* xt = static_cast<const T*>(job.x) + (int64_t)h * job.hs + (int64_t)tile_base(g, u) * job.ts + lane * VEC;
  uint8_t* out = job.codes + ((int64_t)h * g.M + u) * g.pitch * D + lane * VEC;
#pragma unroll 4
  for (int32_t r = warp; r < nr; r += kChunkWarps) {
    float v[VEC];
    V::unpack(V::load(xt + s_off[r]), v);
    bool slow = !fast_ok;
    uint32_t code = encode_fast<FMT, VEC>(v, b, slow);
    if (slow) code = encode_slow<FMT, VEC>(v, pk);  // rare: exact f64 path (ties of bf16 data)
    store_codes<VEC>(out + (int64_t)(r0 + r) * D, code);
  }
  if (c == chunks - 1)  // the tile slot's padding rows
    for (int32_t r = g.tv + warp; r < g.pitch; r += kChunkWarps) store_codes<VEC>(out + (int64_t)r * D, 0u);
}

// V pass A: per-(head, channel) |x| max over all tokens (bit domain, atomicMax).
template <typename T, int D>
__global__ void __launch_bounds__(kQuantThreads)
    chan_amax_kernel(const T* __restrict__ x, int64_t token_stride, int64_t head_stride, int64_t L,
                     int32_t rows_per_block, uint32_t* __restrict__ amax, int32_t* err) {
  constexpr int VEC = D / 32;
  using V = Vec<T, VEC>;
  const int32_t h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t t1 = min(L, t0 + rows_per_block);
  const T* xh = x + (int64_t)h * head_stride + lane * VEC;
  uint32_t m[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) m[e] = 0;
#pragma unroll 8
  for (int64_t t = t0 + warp; t < t1; t += kQuantWarps) {
    float v[VEC];
    V::unpack(V::load(xh + t * token_stride), v);
#pragma unroll
    for (int e = 0; e < VEC; ++e) m[e] = max(m[e], __float_as_uint(v[e]) & 0x7FFFFFFFu);
  }
  __shared__ uint32_t s_m[kQuantWarps][D];
#pragma unroll
  for (int e = 0; e < VEC; ++e) s_m[warp][lane * VEC + e] = m[e];
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += kQuantThreads) {
    uint32_t mm = s_m[0][c];
#pragma unroll
    for (int w = 1; w < kQuantWarps; ++w) mm = max(mm, s_m[w][c]);
    if (mm > 0x7F7FFFFFu && err) atomicOr(err, 1);
    atomicMax(amax + (int64_t)h * D + c, mm);
  }
}

// ---------------------------------------------------------------------------
// General quantisers: any head dim, f32 / bf16 / f64 input, every element
// through the exact path (f64 quotient -> round-to-odd f32 -> RNE cvt), f64
// maxima.  The reference's standalone quantize_qk_tilewise /
// quantize_v_channelwise accept any L x d float64 matrix (quantize.py:111-134);
// these kernels serve the requests the fast kernels do not (d not in {64,128},
// f64 data), off the attention hot path.
template <typename T>
__device__ __forceinline__ double load_elem(const T* p) {
  if constexpr (sizeof(T) == 2) return (double)__uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p)) << 16);
  else return (double)__ldg(p);
}
template <int FMT>
__device__ __forceinline__ uint32_t encode_exact_d(double x, double s) {
  const double q = __ddiv_rn(x, s);
  float f = __double2float_rz(q);
  if ((double)f != q) f = __uint_as_float(__float_as_uint(f) | 1u);  // round to odd
  return cvt_pair<FMT>(0.0f, f) & 0xFFu;
}
__device__ __forceinline__ double scale_of_d(double peak, double maxv) {
  if (peak == 0.0) return 1.0;
  const double s = __ddiv_rn(peak, maxv);
  return s > DBL_MIN ? s : DBL_MIN;
}
constexpr int kGenThreads = 256;

// one CTA per (tile, head): f64 tile max -> scale -> exact codes; padding rows zero
template <typename T, int FMT>
__global__ void __launch_bounds__(kGenThreads) quant_tile_generic_kernel(const T* x, int64_t ts, int64_t hs, Geometry g,
                                                                          int32_t d, uint8_t* codes, double* scales,
                                                                          int32_t* err) {
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  __shared__ unsigned long long s_max;
  const int32_t u = blockIdx.x, h = blockIdx.y;
  const T* xt = x + (int64_t)h * hs + (int64_t)tile_base(g, u) * ts;
  auto off = [&](int32_t r) { return g.natural ? (int64_t)local_offset(g, r) * ts : (int64_t)r * ts; };
  if (threadIdx.x == 0) s_max = 0ull;
  __syncthreads();
  unsigned long long m = 0ull;  // |x| bits: non-negative doubles order as integers, NaN / inf above all
  const int64_t n = (int64_t)g.tv * d;
  for (int64_t i = threadIdx.x; i < n; i += kGenThreads) {
    const double v = load_elem(xt + off((int32_t)(i / d)) + i % d);
    m = max(m, (unsigned long long)__double_as_longlong(fabs(v)));
  }
  atomicMax(&s_max, m);
  __syncthreads();
  double peak = __longlong_as_double((long long)s_max);
  if (!(peak <= DBL_MAX)) {
    if (threadIdx.x == 0 && err) atomicOr(err, 1);
    peak = 0.0;
  }
  const double sc = scale_of_d(peak, kMax);
  if (threadIdx.x == 0) scales[(int64_t)h * g.M + u] = sc;
  uint8_t* out = codes + ((int64_t)h * g.M + u) * g.pitch * d;
  for (int64_t i = threadIdx.x; i < (int64_t)g.pitch * d; i += kGenThreads) {
    const int32_t r = (int32_t)(i / d);
    out[i] = r < g.tv ? (uint8_t)encode_exact_d<FMT>(load_elem(xt + off(r) + i % d), sc) : (uint8_t)0;
  }
}

// v: per-(head, channel) f64 |x| max over all tokens (atomicMax on the bits)
template <typename T>
__global__ void __launch_bounds__(kGenThreads) chan_amax_generic_kernel(const T* x, int64_t ts, int64_t hs, int64_t L,
                                                                         int32_t d, unsigned long long* amax) {
  const int32_t h = blockIdx.y;
  const int64_t n = L * d;
  for (int64_t i = (int64_t)blockIdx.x * kGenThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kGenThreads) {
    const double v = load_elem(x + (int64_t)h * hs + (i / d) * ts + i % d);
    atomicMax(amax + (int64_t)h * d + i % d, (unsigned long long)__double_as_longlong(fabs(v)));
  }
}

// v codes with the channel scales, in the tile-major padded layout; one CTA per (tile, head)
template <typename T, int FMT>
__global__ void __launch_bounds__(kGenThreads) quant_chan_generic_kernel(const T* x, int64_t ts, int64_t hs, Geometry g,
                                                                          int32_t d, const unsigned long long* amax,
                                                                          uint8_t* codes, double* scales,
                                                                          int32_t* err) {
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  const int32_t u = blockIdx.x, h = blockIdx.y;
  const T* xt = x + (int64_t)h * hs + (int64_t)tile_base(g, u) * ts;
  auto off = [&](int32_t r) { return g.natural ? (int64_t)local_offset(g, r) * ts : (int64_t)r * ts; };
  auto scale_c = [&](int32_t c) {
    double peak = __longlong_as_double((long long)amax[(int64_t)h * d + c]);
    return scale_of_d(peak <= DBL_MAX ? peak : 0.0, kMax);
  };
  if (u == 0)
    for (int32_t c = threadIdx.x; c < d; c += kGenThreads) {
      const double peak = __longlong_as_double((long long)amax[(int64_t)h * d + c]);
      if (!(peak <= DBL_MAX) && err) atomicOr(err, 1);
      scales[(int64_t)h * d + c] = scale_c(c);
    }
  uint8_t* out = codes + ((int64_t)h * g.M + u) * g.pitch * d;
  for (int64_t i = threadIdx.x; i < (int64_t)g.pitch * d; i += kGenThreads) {
    const int32_t r = (int32_t)(i / d), c = (int32_t)(i % d);
    out[i] = r < g.tv ? (uint8_t)encode_exact_d<FMT>(load_elem(xt + off(r) + c), scale_c(c)) : (uint8_t)0;
  }
}

// ---------------------------------------------------------------------------
// TMA-fed persistent quantiser (bf16 input, d = 128, tile volume <= 256).
//
// One CTA per SM loops over (tensor, head, tile) items.  A producer warp
// streams each tile into shared memory with 3D TMA loads (one box per run
// of tile_w consecutive tokens, strided by the token stride, so the gather
// to tile-major order is done by the copy engine), kTmaStages tiles ahead;
// 24 consumer warps reduce the tile amax from shared memory and write the
// codes.  HBM traffic is one read of q/k/v and one write of the codes.
#ifndef FPSA_QUANT_WARPS
#define FPSA_QUANT_WARPS 20  // round 2 (one barrier, tie table): 1.113 ms vs 1.137 (24), 1.131 (16), 1.269 (28); round 1 (two barriers): 24 best
#endif
constexpr int kTmaConsumerWarps = FPSA_QUANT_WARPS;
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;
constexpr int kTmaStages = 3;
constexpr int kTmaMaxRows = 256;
constexpr int kTmaD = 128;
constexpr int kTmaStageBytes = kTmaMaxRows * kTmaD * 2;

struct TmaQuantArgs {
  int32_t whole_tile;  // one TMA box per tile (5D natural-order view / tv-row box) instead of one per w-run
  uint8_t* codes[3];
  double* scales[3];
  int32_t channel[3];
  int32_t njobs, heads;
  const uint32_t* amax;
  int32_t* err;
};

#ifndef FPSA_QUANT_ORDER
#define FPSA_QUANT_ORDER 0  // 0: (tensor, head, tile) with tiles fastest; 1: (tensor, tile, head), heads fastest
#endif
#ifndef FPSA_QUANT_LOADONLY
#define FPSA_QUANT_LOADONLY 0
#endif
__device__ __forceinline__ void item_of(int32_t it, int32_t per_job, int32_t heads, int32_t M, int32_t& z,
                                        int32_t& h, int32_t& u) {
  z = it / per_job;
  const int32_t rem = it - z * per_job;
  if (FPSA_QUANT_ORDER) {
    u = rem / heads;
    h = rem - u * heads;
  } else {
    h = rem / M;
    u = rem - h * M;
  }
}

// Exact ties of bf16 data without f64 arithmetic per element.  With x and the block peak P both bf16, the
// quotient Q = x * maxv / P (maxv = 448 = 7 * 2^6, or 57344 = 7 * 2^13) lies either exactly on a rounding
// midpoint B = o * 2^f of the fp8 grid (o odd, o <= 31) or at least 2^-13 (relative) away from it, far
// outside the fast path's 2^-19 bracket; so an ambiguous element is an exact tie.  Its code then depends
// only on how the reference's f64 quotient q64 = RN64(x / RN64(P / maxv)) compares with B: q64 == B rounds
// to the even code, q64 < B down, q64 > B up.  That comparison depends only on P's 8-bit significand and on
// B's odd significand o (powers of two scale out), so one table per format, indexed by the peak's mantissa
// bits and the tie class (the lower code's mantissa, normal or subnormal), decides every tie: bit k of .x
// "up", of .y "even", of .z "the class can occur at all" (o * P_m divisible by 7); otherwise the element
// takes the exact f64 path.  Built per CTA at kernel start from the same IEEE f64 operations.
constexpr int kTieEntries = 128;  // bf16 mantissa bits of the peak
template <int FMT>
__device__ __forceinline__ int32_t tie_odd(int k) {  // odd significand o of tie class k
  constexpr int kM = FMT == FPSA_E4M3 ? 8 : 4;     // mantissa codes per binade
  return k < kM ? 2 * kM + 1 + 2 * k : 2 * (k - kM) + 1;  // normal: (2 kM + 2m + 1); subnormal: 2m + 1
}
template <int FMT>
__device__ __forceinline__ int tie_class(uint32_t code) {  // class of the midpoint above code (magnitude)
  constexpr int kMB = FMT == FPSA_E4M3 ? 3 : 2, kM = 1 << kMB;
  const uint32_t mag = code & 0x7Fu, m = mag & (kM - 1u);
  return (mag >> kMB) ? (int)m : kM + (int)m;
}
template <int FMT>
__device__ void build_tie_table(uint3* table, int tid, int nthreads) {
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  constexpr int kClasses = FMT == FPSA_E4M3 ? 16 : 8;
  for (int i = tid; i < kTieEntries * kClasses; i += nthreads) {
    const int e = i / kClasses, k = i % kClasses;
    const double pm = (double)(128 + e);                  // the peak's significand, scaled to an integer
    const double s = __ddiv_rn(pm, kMax);                 // scale_of: RN64(P / maxv), up to a power of two
    const double xo = (double)(tie_odd<FMT>(k) * (128 + e));  // o * P_m, exact
    const double x = __ddiv_rn(xo, kMax);                 // the tying input, if representable
    const bool ok = __fma_rn(x, kMax, -xo) == 0.0;
    const double q = __ddiv_rn(x, s);                     // the reference's f64 quotient
    const double o = (double)tie_odd<FMT>(k);
    if (ok) {
      atomicOr(&table[e].z, 1u << k);
      if (q > o) atomicOr(&table[e].x, 1u << k);
      if (q == o) atomicOr(&table[e].y, 1u << k);
    }
  }
}
// The code of an ambiguous element (clo / chi: the codes of the bracket ends, chi one step above in
// magnitude) from the tie table; the exact f64 path when the peak is not a normal bf16 value or the class
// cannot tie.
template <int FMT>
__device__ __forceinline__ uint32_t resolve_tie(const uint3* table, uint32_t clo, uint32_t chi, float x,
                                                float peak, bool use_table) {
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  const uint32_t pb = __float_as_uint(peak);
  const uint32_t exp = (pb >> 23) & 0xFFu;
  if (use_table && (pb & 0xFFFFu) == 0u && exp != 0u && exp != 0xFFu) {
    const uint3 t = table[(pb >> 16) & 0x7Fu];
    const uint32_t bit = 1u << tie_class<FMT>(clo);
    if (t.z & bit) return (t.x & bit) ? chi : ((t.y & bit) ? ((clo & 1u) ? chi : clo) : clo);
  }
  // inlined: a call here would constrain the register allocation of the whole kernel (1.30 vs 1.08 ms)
  return encode_exact_inl<FMT>(x, scale_of(peak, kMax));
}

#ifdef FPSA_QTRACE
// measurement builds only: per-tile timeline of CTA 0 (clock64): [0] load issued, [1] warp 0 saw it full,
// [2] warp 0 past the tile-max barrier, [3] warp 0 released the stage, [4] warp 23 released the stage
__device__ long long g_qtl[128][5];
__device__ unsigned long long g_qcount[4];  // fix-up loop trips (warp), ambiguous bytes (lane), tiles
#define FPSA_QTL(k, ev)                                                            \
  do {                                                                            \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (k) < 128) g_qtl[(k)][(ev)] = clock64(); \
  } while (0)
#else
#define FPSA_QTL(k, ev) \
  do {                  \
  } while (0)
#endif

template <int FMT>
__global__ void __launch_bounds__(kTmaThreads, 1)
    quant_tma_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
                     const __grid_constant__ CUtensorMap tm2, Geometry g, TmaQuantArgs a) {
  using namespace sm100;
  constexpr int VEC = 4;
  constexpr double kMax = FMT == FPSA_E4M3 ? 448.0 : 57344.0;
  using V = Vec<__nv_bfloat16, VEC>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kTmaStages], empty[kTmaStages];
  __shared__ uint32_t s_peak[3];  // tile |x| max bits by tile index mod 3 (shared-memory atomicMax of the warps)
  __shared__ uint3 s_tie[kTieEntries];  // exact-tie decisions by the peak's mantissa bits (build_tie_table)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t per_job = a.heads * g.M;
  const int32_t n_items = a.njobs * per_job;
  const int32_t runs = g.tv / g.sw;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTmaStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTmaConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kTmaConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      prefetch_tmap(&tm0);
      prefetch_tmap(&tm1);
      prefetch_tmap(&tm2);
      int k = 0;
      for (int32_t it = blockIdx.x; it < n_items; it += gridDim.x, ++k) {
        const int st = k % kTmaStages;
        if (k >= kTmaStages) mbar_wait(&empty[st], ((k / kTmaStages) - 1) & 1);
        int32_t z, h, u;
        item_of(it, per_job, a.heads, g.M, z, h, u);
        const void* tm = z == 0 ? (const void*)&tm0 : (z == 1 ? (const void*)&tm1 : (const void*)&tm2);
        uint8_t* dst = smem + st * kTmaStageBytes;
        FPSA_QTL(k, 0);
        mbar_arrive_expect_tx(&full[st], (uint32_t)g.tv * kTmaD * 2);
        if (a.whole_tile) {
          // one box per tile: natural order through the 5D view (c, head, w, h, t) with box
          // (128, 1, sw, sh, st), which lands the tile in its local (t, h, w) row order; tile order
          // through the 3D view with a box of tv rows
          if (g.natural) {
            const int32_t ut = u / (g.dh * g.dw), uh = (u / g.dw) % g.dh, uw = u % g.dw;
            tma_load_5d(dst, tm, 0, h, uw * g.sw, uh * g.sh, ut * g.st, &full[st]);
          } else {
            tma_load_3d(dst, tm, 0, u * g.tv, h, &full[st]);
          }
        } else {
          const int32_t base = tile_base(g, u);
          for (int32_t r = 0; r < runs; ++r) {
            // run r = (lt, lh) of the tile; in tile order runs are consecutive rows
            const int32_t lt = r / g.sh, lh = r - lt * g.sh;
            const int32_t tok = g.natural ? base + (lt * g.gh + lh) * g.gw : base + r * g.sw;
            tma_load_3d(dst + r * g.sw * kTmaD * 2, tm, 0, tok, h, &full[st]);
          }
        }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  // One CTA-wide barrier per tile (the tile max); each warp then encodes its rows and releases the stage
  // itself.  Ambiguous elements (the bracket straddles a rounding boundary: exact ties of bf16 data, ~0.4%
  // of elements) are flagged per row in a register mask and re-encoded exactly by their own lane after
  // the row loop, while the tile is still in shared memory (no queue, no atomics).  Holding the stage
  // until then is deliberate: copying the rows to registers and releasing the stage first keeps three
  // loads in flight per SM and measured 1.78 ms against 1.16 (profiles/r02_quant_early_release_rejected.txt).
  static_assert(kTmaMaxRows <= 32 * kTmaConsumerWarps, "row mask holds one bit per row of a warp");
  if (threadIdx.x == 0) s_peak[0] = s_peak[1] = s_peak[2] = 0;
  for (int i = threadIdx.x; i < kTieEntries; i += kTmaConsumerWarps * 32) s_tie[i] = make_uint3(0u, 0u, 0u);
  named_bar_sync(1, kTmaConsumerWarps * 32);
  build_tie_table<FMT>(s_tie, threadIdx.x, kTmaConsumerWarps * 32);  // overlaps the first tile loads
  named_bar_sync(1, kTmaConsumerWarps * 32);
  int k = 0;
  for (int32_t it = blockIdx.x; it < n_items; it += gridDim.x, ++k) {
    const int st = k % kTmaStages;
    int32_t z, h, u;
    item_of(it, per_job, a.heads, g.M, z, h, u);
#if FPSA_QUANT_LOADONLY
    mbar_wait(&full[st], (k / kTmaStages) & 1);  // measurement build: the loads alone (codes not written)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    continue;
#endif
    // select, do not index: a dynamically indexed parameter array is copied to local memory
    const bool channel = (z == 0 ? a.channel[0] : z == 1 ? a.channel[1] : a.channel[2]) != 0;
    uint8_t* const codes = z == 0 ? a.codes[0] : z == 1 ? a.codes[1] : a.codes[2];
    double* const scales = z == 0 ? a.scales[0] : z == 1 ? a.scales[1] : a.scales[2];
    uint8_t* out = codes + ((int64_t)h * g.M + u) * g.pitch * kTmaD + lane * VEC;
    const uint2* tile = reinterpret_cast<const uint2*>(smem + st * kTmaStageBytes) + lane;
    uint32_t* const peak_slot = &s_peak[k % 3];
    mbar_wait(&full[st], (k / kTmaStages) & 1);
    if (warp == 0) FPSA_QTL(k, 1);
    if (!channel) {
      uint32_t m = 0;
#pragma unroll 8
      for (int32_t r = warp; r < g.tv; r += kTmaConsumerWarps) m = absmax_bits<__nv_bfloat16, VEC>(tile[r * 32], m);
      m = __float_as_uint(bits_to_peak<__nv_bfloat16>(m));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) atomicMax(peak_slot, m);
    }
    named_bar_sync(1, kTmaConsumerWarps * 32);
    // slot (k + 2) % 3 was last read after the previous barrier and is next written after the following one
    if (threadIdx.x == 0) s_peak[(k + 2) % 3] = 0;
    if (warp == 0) FPSA_QTL(k, 2);
    float pk[VEC];
    Bracket b[VEC];
    if (!channel) {
      float peak = __uint_as_float(*peak_slot);
      if (!(peak <= FLT_MAX)) {
        if (warp == 0 && lane == 0 && a.err) atomicOr(a.err, 1);
        peak = 0.0f;
      }
      const Bracket bb = bracket_f32<FMT>(peak);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        pk[e] = peak;
        b[e] = bb;
      }
      if (warp == 0 && lane == 0) scales[(int64_t)h * g.M + u] = scale_of(peak, kMax);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const float peak = __uint_as_float(a.amax[(int64_t)h * kTmaD + lane * VEC + e]);
        pk[e] = peak <= FLT_MAX ? peak : 0.0f;
        b[e] = bracket_f32<FMT>(pk[e]);
        if (u == 0 && warp == 0) scales[(int64_t)h * kTmaD + lane * VEC + e] = scale_of(pk[e], kMax);
      }
    }
    bool fast_ok = true;
#pragma unroll
    for (int e = 0; e < VEC; ++e) fast_ok &= b[e].ok;
    const uint32_t force = fast_ok ? 0u : 0xFFFFFFFFu;  // a bracket out of range: every element exact
    uint32_t amb = 0;  // bit i: row warp + i * kTmaConsumerWarps has an ambiguous element in this lane
    int32_t i = 0;
#pragma unroll 4
    for (int32_t r = warp; r < g.tv; r += kTmaConsumerWarps, ++i) {
      float v[VEC];
      V::unpack(tile[r * 32], v);
      uint32_t clo = 0, chi = 0;
#pragma unroll
      for (int e = 0; e < VEC; e += 2) {
        float l0, l1, h0, h1;
        mul2(v[e], v[e + 1], b[e].lo, b[e + 1].lo, l0, l1);
        mul2(v[e], v[e + 1], b[e].hi, b[e + 1].hi, h0, h1);
        clo |= cvt_pair<FMT>(l1, l0) << (8 * e);
        chi |= cvt_pair<FMT>(h1, h0) << (8 * e);
      }
      store_codes<VEC>(out + (int64_t)r * kTmaD, clo);
      amb |= ((clo ^ chi) | force) != 0u ? 1u << i : 0u;
    }
#ifdef FPSA_QTRACE
    {
      const unsigned trips = __reduce_max_sync(0xffffffffu, (unsigned)__popc(amb));
      if (lane == 0) atomicAdd(&g_qcount[0], (unsigned long long)trips);
      if (lane == 0 && warp == 0) atomicAdd(&g_qcount[2], 1ull);
    }
#endif
    while (amb) {  // rare: this lane's rows with ambiguous bytes, re-encoded from the f64 quotient
      const int32_t ri = __ffs(amb) - 1;
      amb &= amb - 1;
      const int32_t r = warp + ri * kTmaConsumerWarps;
      float v[VEC];
      V::unpack(tile[r * 32], v);
      uint32_t clo = 0, chi = 0;
#pragma unroll
      for (int e = 0; e < VEC; e += 2) {
        float l0, l1, h0, h1;
        mul2(v[e], v[e + 1], b[e].lo, b[e + 1].lo, l0, l1);
        mul2(v[e], v[e + 1], b[e].hi, b[e + 1].hi, h0, h1);
        clo |= cvt_pair<FMT>(l1, l0) << (8 * e);
        chi |= cvt_pair<FMT>(h1, h0) << (8 * e);
      }
      const uint32_t diff = clo ^ chi;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        if (!(((diff | force) >> (8 * e)) & 0xFFu)) continue;
#ifdef FPSA_QTRACE
        atomicAdd(&g_qcount[1], 1ull);
#endif
        const uint32_t lo = (clo >> (8 * e)) & 0xFFu, hi = (chi >> (8 * e)) & 0xFFu;
        // a bracket out of range (force): every element takes the exact path
        const uint32_t c = resolve_tie<FMT>(s_tie, lo, hi, v[e], pk[e], force == 0u);
        clo = (clo & ~(0xFFu << (8 * e))) | (c << (8 * e));
      }
      store_codes<VEC>(out + (int64_t)r * kTmaD, clo);
    }
    __syncwarp();
    if (warp == 0) FPSA_QTL(k, 3);
    if (warp == kTmaConsumerWarps - 1) FPSA_QTL(k, 4);
    if (lane == 0) mbar_arrive(&empty[st]);
    for (int32_t r = g.tv + warp; r < g.pitch; r += kTmaConsumerWarps) store_codes<VEC>(out + (int64_t)r * kTmaD, 0u);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// [heads][L][d] view of a bf16 input with token / head strides (elements).
// One box per tile.  Natural order: 5D view (c, head, w, h, t) of a [t][h][w] token grid with box
// (128, 1, sw, sh, st); tile order: 3D view [heads][L][d] with a box of tv rows.
bool make_tile_map(CUtensorMap* m, const void* x, const Geometry& g, int32_t heads, int64_t ts, int64_t hs) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int64_t hstride = (hs > 0 ? hs : ts) * 2;
  if (g.natural) {
    cuuint64_t dims[5] = {(cuuint64_t)kTmaD, (cuuint64_t)heads, (cuuint64_t)g.gw, (cuuint64_t)g.gh, (cuuint64_t)g.gt};
    cuuint64_t strides[4] = {(cuuint64_t)hstride, (cuuint64_t)ts * 2, (cuuint64_t)ts * 2 * g.gw,
                             (cuuint64_t)ts * 2 * g.gw * g.gh};
    cuuint32_t box[5] = {(cuuint32_t)kTmaD, 1, (cuuint32_t)g.sw, (cuuint32_t)g.sh, (cuuint32_t)g.st};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(x), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const int64_t L = (int64_t)g.gt * g.gh * g.gw;
  cuuint64_t dims[3] = {(cuuint64_t)kTmaD, (cuuint64_t)L, (cuuint64_t)heads};
  cuuint64_t strides[2] = {(cuuint64_t)ts * 2, (cuuint64_t)hstride};
  cuuint32_t box[3] = {(cuuint32_t)kTmaD, (cuuint32_t)g.tv, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_input_map(CUtensorMap* m, const void* x, int64_t L, int32_t heads, int64_t ts, int64_t hs, int32_t sw) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kTmaD, (cuuint64_t)L, (cuuint64_t)heads};
  cuuint64_t strides[2] = {(cuuint64_t)ts * 2, (cuuint64_t)(hs > 0 ? hs : ts) * 2};
  cuuint32_t box[3] = {(cuuint32_t)kTmaD, (cuuint32_t)sw, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// Launch the TMA quantiser if the request fits it; returns false to fall back.
bool try_tma_quant(const void* const* xs, int njobs, int dtype, int64_t ts, int64_t hs, int32_t heads,
                   const Geometry& g, int32_t d, int fmt, const TmaQuantArgs& a, cudaStream_t st) {
  if (dtype != FPSA_BF16 || d != kTmaD || g.tv > kTmaMaxRows || g.sw > 256 || (ts * 2) % 16 || (hs * 2) % 16)
    return false;
  if (heads > 1 && hs == 0) return false;
  const int64_t L = (int64_t)g.gt * g.gh * g.gw;
  CUtensorMap tm[3];
  static const bool runs_only = getenv("FPSA_QUANT_RUNS") != nullptr;  // measurement switch: one box per w-run
  TmaQuantArgs aa = a;
  aa.whole_tile = !runs_only && g.st <= 256 && g.sh <= 256 && g.sw <= 256;
  for (int i = 0; i < 3; ++i) {
    const void* x = xs[i < njobs ? i : 0];
    if (aa.whole_tile && !make_tile_map(&tm[i], x, g, heads, ts, hs)) aa.whole_tile = 0;
  }
  if (!aa.whole_tile)
    for (int i = 0; i < 3; ++i)
      if (!make_input_map(&tm[i], xs[i < njobs ? i : 0], L, heads, ts, hs, g.sw)) return false;
  const int smem = kTmaStages * kTmaStageBytes;
  auto kern = fmt == FPSA_E4M3 ? quant_tma_kernel<FPSA_E4M3> : quant_tma_kernel<FPSA_E5M2>;
  if (ensure_smem_attr(reinterpret_cast<const void*>(kern), smem, "quant_tma_kernel") != FPSA_OK) return false;
  const int64_t items = (int64_t)njobs * heads * g.M;
  const int grid = (int)std::min<int64_t>(items, device_sm_count());
  kern<<<grid, kTmaThreads, smem, st>>>(tm[0], tm[1], tm[2], g, aa);
  return true;
}

int make_geometry(fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t pitch, int in_order, Geometry* g) {
  fpsa_dims3 td;
  if (int st = fpsa_tile_grid(grid, tile, &td)) return st;
  if (d < 1) return fail(FPSA_EINVAL, "head dim must be >= 1, got " + std::to_string(d));
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
  if (dtype != FPSA_F32 && dtype != FPSA_BF16 && dtype != FPSA_F64)
    return fail(FPSA_EUNSUPPORTED, "input dtype must be f32, bf16 or f64");
  if (fmt != FPSA_E4M3 && fmt != FPSA_E5M2) return fail(FPSA_EINVAL, "fmt must be e4m3 or e5m2");
  return FPSA_OK;
}

int cuda_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FPSA_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return FPSA_OK;
}

template <typename T, int D, int FMT>
void launch_jobs(const Geometry& g, int32_t heads, const QuantArgs& a, int njobs, cudaStream_t st) {
  dim3 grid(g.M, heads, njobs);
  quant_kernel<T, D, FMT><<<grid, kQuantThreads, 0, st>>>(g, a);
}

template <typename T, int D>
void launch_amax(const void* x, int64_t ts, int64_t hs, int32_t heads, const Geometry& g, uint32_t* amax,
                 int32_t* err, cudaStream_t st) {
  const int64_t L = (int64_t)g.gt * g.gh * g.gw;
  const int32_t rows_per_block = 512;
  dim3 ga((unsigned)((L + rows_per_block - 1) / rows_per_block), heads);
  chan_amax_kernel<T, D><<<ga, kQuantThreads, 0, st>>>(static_cast<const T*>(x), ts, hs, L, rows_per_block, amax, err);
}

// dtype x d x fmt dispatch of a callable template F<T, D, FMT>::run(args...)
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
struct RunChunked {
  // jobs with channel == 0 must have zeroed scale arrays (their words hold the tile maxima until pass 3)
  static void run(const Geometry& g, int32_t heads, const QuantArgs& a, int njobs, cudaStream_t st) {
    const int32_t chunks = (g.tv + kChunkRows - 1) / kChunkRows;
    dim3 grid(g.M * chunks, heads, njobs);
    tile_amax_chunk_kernel<T, D><<<grid, kChunkThreads, 0, st>>>(g, a, chunks);
    encode_chunk_kernel<T, D, FMT><<<grid, kChunkThreads, 0, st>>>(g, a, chunks);
    const int64_t n = (int64_t)heads * g.M;
    for (int z = 0; z < njobs; ++z)
      if (!a.job[z].channel)
        scales_from_amax_kernel<FMT><<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(a.job[z].scales,
                                                                                                  n, a.err);
  }
};
template <typename T, int D, int FMT>
struct RunJobs {
  static void run(const Geometry& g, int32_t heads, const QuantArgs& a, int njobs, cudaStream_t st) {
    launch_jobs<T, D, FMT>(g, heads, a, njobs, st);
  }
};
template <typename T, int D, int FMT>
struct RunAmax {
  static void run(const void* x, int64_t ts, int64_t hs, int32_t heads, const Geometry& g, uint32_t* amax,
                  int32_t* err, cudaStream_t st) {
    launch_amax<T, D>(x, ts, hs, heads, g, amax, err, st);
  }
};

// the general (exact, any d, f64) quantisers; true when the request needs them
bool needs_general(int dtype, int32_t d) { return dtype == FPSA_F64 || (d != 64 && d != 128); }

template <typename T, int FMT>
void launch_general_tile(const void* x, int64_t ts, int64_t hs, int32_t heads, const Geometry& g, int32_t d,
                         uint8_t* codes, double* scales, int32_t* err, cudaStream_t st) {
  quant_tile_generic_kernel<T, FMT><<<dim3(g.M, heads), kGenThreads, 0, st>>>(static_cast<const T*>(x), ts, hs, g, d,
                                                                              codes, scales, err);
}
template <typename T, int FMT>
void launch_general_chan(const void* x, int64_t ts, int64_t hs, int32_t heads, const Geometry& g, int32_t d,
                         unsigned long long* amax, uint8_t* codes, double* scales, int32_t* err, cudaStream_t st) {
  const int64_t L = (int64_t)g.gt * g.gh * g.gw;
  const int64_t blocks = std::min<int64_t>((L * d + kGenThreads - 1) / kGenThreads, 4096);
  chan_amax_generic_kernel<T><<<dim3((unsigned)blocks, heads), kGenThreads, 0, st>>>(static_cast<const T*>(x), ts, hs, L,
                                                                                      d, amax);
  quant_chan_generic_kernel<T, FMT><<<dim3(g.M, heads), kGenThreads, 0, st>>>(static_cast<const T*>(x), ts, hs, g, d,
                                                                              amax, codes, scales, err);
}
template <template <typename, int> class F, typename... Args>
void dispatch_general(int dtype, int fmt, Args&&... args) {
  if (dtype == FPSA_F64) {
    if (fmt == FPSA_E4M3) F<double, FPSA_E4M3>::run(args...); else F<double, FPSA_E5M2>::run(args...);
  } else if (dtype == FPSA_F32) {
    if (fmt == FPSA_E4M3) F<float, FPSA_E4M3>::run(args...); else F<float, FPSA_E5M2>::run(args...);
  } else {
    if (fmt == FPSA_E4M3) F<__nv_bfloat16, FPSA_E4M3>::run(args...); else F<__nv_bfloat16, FPSA_E5M2>::run(args...);
  }
}
template <typename T, int FMT>
struct RunGeneralTile {
  template <typename... A>
  static void run(A... a) { launch_general_tile<T, FMT>(a...); }
};
template <typename T, int FMT>
struct RunGeneralChan {
  template <typename... A>
  static void run(A... a) { launch_general_chan<T, FMT>(a...); }
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
  if (needs_general(dtype, d)) {
    dispatch_general<RunGeneralTile>(dtype, fmt, x, token_stride, head_stride, heads, g, d, codes, scales, err_flag,
                                     static_cast<cudaStream_t>(stream));
    return cuda_status("fpsa_quantize_qk");
  }
  QuantArgs a{};
  a.job[0] = QuantJob{x, token_stride, head_stride, codes, scales, 0};
  a.err = err_flag;
  dispatch<RunJobs>(dtype, d, fmt, g, heads, a, 1, static_cast<cudaStream_t>(stream));
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
  if (needs_general(dtype, d)) {  // f64 channel maxima: workspace >= heads*d*8 bytes
    auto* amax64 = static_cast<unsigned long long*>(workspace);
    if (cudaMemsetAsync(amax64, 0, (size_t)heads * d * 8, st) != cudaSuccess) return cuda_status("fpsa_quantize_v memset");
    dispatch_general<RunGeneralChan>(dtype, fmt, x, token_stride, head_stride, heads, g, d, amax64, codes, scales,
                                     err_flag, st);
    return cuda_status("fpsa_quantize_v");
  }
  uint32_t* amax = static_cast<uint32_t*>(workspace);
  if (cudaMemsetAsync(amax, 0, (size_t)heads * d * sizeof(uint32_t), st) != cudaSuccess)
    return cuda_status("fpsa_quantize_v memset");
  dispatch<RunAmax>(dtype, d, fmt, x, token_stride, head_stride, heads, g, amax, err_flag, st);
  QuantArgs a{};
  a.job[0] = QuantJob{x, token_stride, head_stride, codes, scales, 1};
  a.amax = amax;
  a.err = err_flag;
  dispatch<RunJobs>(dtype, d, fmt, g, heads, a, 1, st);
  return cuda_status("fpsa_quantize_v");
}

namespace fpsa {
namespace {
// v channel maxima: 4-byte words on the fast paths, 8-byte on the general (f64 / any d) path
int64_t qkv_workspace_words(int32_t heads, int32_t d) { return 2 * (int64_t)heads * d + heads + 1; }

int quantize_qkv(const void* q, const void* k, const void* v, int dtype, int64_t token_stride, int64_t head_stride,
                 int32_t heads, fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, int in_order,
                 int fmt, uint8_t* q_codes, uint8_t* k_codes, uint8_t* v_codes, double* q_scales, double* k_scales,
                 double* v_scales, const float* q_amax, const float* k_amax, const float* v_amax, void* workspace,
                 int32_t* err_flag, void* stream, const char* name) {
  if (int s = check_common(q, dtype, heads, fmt, q_codes, q_scales)) return s;
  if (int s = check_common(k, dtype, heads, fmt, k_codes, k_scales)) return s;
  if (int s = check_common(v, dtype, heads, fmt, v_codes, v_scales)) return s;
  if (!workspace) return fail(FPSA_EINVAL, "workspace is NULL");
  Geometry g;
  if (int s = make_geometry(grid, tile, d, tile_pitch, in_order, &g)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (needs_general(dtype, d)) {
    auto* amax64 = static_cast<unsigned long long*>(workspace);
    if (cudaMemsetAsync(amax64, 0, (size_t)heads * d * 8, st) != cudaSuccess) return cuda_status(name);
    dispatch_general<RunGeneralTile>(dtype, fmt, q, token_stride, head_stride, heads, g, d, q_codes, q_scales,
                                     err_flag, st);
    dispatch_general<RunGeneralTile>(dtype, fmt, k, token_stride, head_stride, heads, g, d, k_codes, k_scales,
                                     err_flag, st);
    dispatch_general<RunGeneralChan>(dtype, fmt, v, token_stride, head_stride, heads, g, d, amax64, v_codes, v_scales,
                                     err_flag, st);
    return cuda_status(name);
  }
  // workspace: v channel amax bits [heads*d] (+ spare words)
  uint32_t* amax = static_cast<uint32_t*>(workspace);
  if (cudaMemsetAsync(workspace, 0, (size_t)qkv_workspace_words(heads, d) * 4, st) != cudaSuccess)
    return cuda_status(name);
  // v channel maxima: the caller's (f32 |x| max bits compare as u32), else one pass over v
  const uint32_t* vmax = reinterpret_cast<const uint32_t*>(v_amax);
  if (!v_amax) {
    dispatch<RunAmax>(dtype, d, fmt, v, token_stride, head_stride, heads, g, amax, err_flag, st);
    vmax = amax;
  }
  (void)q_amax;  // tile maxima are reduced from the tile in shared memory anyway (the caller's must equal them)
  (void)k_amax;
  {
    TmaQuantArgs ta{};
    ta.codes[0] = q_codes; ta.codes[1] = k_codes; ta.codes[2] = v_codes;
    ta.scales[0] = q_scales; ta.scales[1] = k_scales; ta.scales[2] = v_scales;
    ta.channel[2] = 1;
    ta.njobs = 3;
    ta.heads = heads;
    ta.amax = vmax;
    ta.err = err_flag;
    const void* xs[3] = {q, k, v};
    static const bool no_tma = getenv("FPSA_QUANT_NO_TMA") != nullptr;  // measurement switch
    if (!no_tma && try_tma_quant(xs, 3, dtype, token_stride, head_stride, heads, g, d, fmt, ta, st))
      return cuda_status(name);
  }
  QuantArgs a{};
  a.job[0] = QuantJob{q, token_stride, head_stride, q_codes, q_scales, 0};
  a.job[1] = QuantJob{k, token_stride, head_stride, k_codes, k_scales, 0};
  a.job[2] = QuantJob{v, token_stride, head_stride, v_codes, v_scales, 1};
  a.amax = vmax;
  a.err = err_flag;
  static const bool per_tile_cta = getenv("FPSA_QUANT_TILE_CTA") != nullptr;  // measurement switch
  if (per_tile_cta) {
    dispatch<RunJobs>(dtype, d, fmt, g, heads, a, 3, st);
    return cuda_status(name);
  }
  // chunked passes: the q / k scale arrays hold the tile maxima until the last pass
  if (cudaMemsetAsync(q_scales, 0, (size_t)heads * g.M * 8, st) != cudaSuccess ||
      cudaMemsetAsync(k_scales, 0, (size_t)heads * g.M * 8, st) != cudaSuccess)
    return cuda_status(name);
  dispatch<RunChunked>(dtype, d, fmt, g, heads, a, 3, st);
  return cuda_status(name);
}
}  // namespace
}  // namespace fpsa

extern "C" int fpsa_quantize_workspace_bytes(int32_t heads, int32_t d, int64_t* bytes) {
  clear_error();
  if (!bytes || heads < 1 || d < 1) return fail(FPSA_EINVAL, "bad arguments");
  *bytes = qkv_workspace_words(heads, d) * 4;
  return FPSA_OK;
}

extern "C" int fpsa_quantize_qkv(const void* q, const void* k, const void* v, int dtype, int64_t token_stride,
                                 int64_t head_stride, int32_t heads, fpsa_dims3 grid, fpsa_dims3 tile, int32_t d,
                                 int32_t tile_pitch, int in_order, int fmt, uint8_t* q_codes, uint8_t* k_codes,
                                 uint8_t* v_codes, double* q_scales, double* k_scales, double* v_scales,
                                 void* workspace, int32_t* err_flag, void* stream) {
  clear_error();
  return quantize_qkv(q, k, v, dtype, token_stride, head_stride, heads, grid, tile, d, tile_pitch, in_order, fmt,
                      q_codes, k_codes, v_codes, q_scales, k_scales, v_scales, nullptr, nullptr, nullptr, workspace,
                      err_flag, stream, "fpsa_quantize_qkv");
}

extern "C" int fpsa_quantize_qkv_amax(const void* q, const void* k, const void* v, int dtype, int64_t token_stride,
                                      int64_t head_stride, int32_t heads, fpsa_dims3 grid, fpsa_dims3 tile, int32_t d,
                                      int32_t tile_pitch, int in_order, int fmt, const float* q_tile_amax,
                                      const float* k_tile_amax, const float* v_channel_amax, uint8_t* q_codes,
                                      uint8_t* k_codes, uint8_t* v_codes, double* q_scales, double* k_scales,
                                      double* v_scales, void* workspace, int32_t* err_flag, void* stream) {
  clear_error();
  return quantize_qkv(q, k, v, dtype, token_stride, head_stride, heads, grid, tile, d, tile_pitch, in_order, fmt,
                      q_codes, k_codes, v_codes, q_scales, k_scales, v_scales, q_tile_amax, k_tile_amax,
                      v_channel_amax, workspace, err_flag, stream, "fpsa_quantize_qkv_amax");
}

// ---------------------------------------------------------------------------
// Element codec (fp8.encode / fp8.decode / quantize_dequantize, fp8.py:153-234)
namespace fpsa {
namespace {
constexpr int kCodecThreads = 256;

// RNE of x (or of the f64 quotient x / scale) onto the format: f32 without a scale rounds the f32 value
// directly (the reference's bounds32 path), everything else goes through f64 (bounds64).  NaN -> err bit 0;
// infinity -> the inf code (E5M2) or err bit 1 (E4M3); finite magnitudes above max_value saturate.
template <typename T, int FMT>
__global__ void __launch_bounds__(kCodecThreads) encode_kernel(const T* x, const double* scale, int64_t n,
                                                               uint8_t* codes, int32_t* err) {
  for (int64_t i = (int64_t)blockIdx.x * kCodecThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCodecThreads) {
    const double v = load_elem(x + i);
    uint32_t c;
    if (isnan(v)) {
      atomicOr(err, 1);
      c = 0;
    } else if (isinf(v)) {
      if (FMT == FPSA_E5M2) c = signbit(v) ? 0xFCu : 0x7Cu;
      else {
        atomicOr(err, 2);
        c = 0;
      }
    } else if (scale) {
      c = encode_exact_d<FMT>(v, scale[i]);
    } else if (sizeof(T) <= 4) {
      c = cvt_pair<FMT>(0.0f, (float)v) & 0xFFu;  // f32 / bf16 value: exactly an f32
    } else {
      c = encode_exact_d<FMT>(v, 1.0);
    }
    codes[i] = (uint8_t)c;
  }
}

// value(code) [* scale in f64]; a NaN pattern sets err bit 0 (the reference raises)
template <int FMT, typename O>
__global__ void __launch_bounds__(kCodecThreads) decode_kernel(const uint8_t* codes, const double* scale, int64_t n,
                                                               O* out, int32_t* err) {
  for (int64_t i = (int64_t)blockIdx.x * kCodecThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCodecThreads) {
    const uint32_t c = codes[i];
    const uint32_t e = FMT == FPSA_E4M3 ? (c >> 3) & 0xF : (c >> 2) & 0x1F;
    const uint32_t m = FMT == FPSA_E4M3 ? c & 7 : c & 3;
    constexpr int kMb = FMT == FPSA_E4M3 ? 3 : 2, kBias = FMT == FPSA_E4M3 ? 7 : 15, kTop = FMT == FPSA_E4M3 ? 15 : 31;
    double mag;
    bool nan = false;
    if (e == 0) mag = ldexp((double)m, 1 - kBias - kMb);
    else mag = ldexp((double)(m + (1u << kMb)), (int)e - kBias - kMb);
    if (FMT == FPSA_E4M3 && e == kTop && m == 7) nan = true;
    if (FMT == FPSA_E5M2 && e == kTop) {
      if (m == 0) mag = INFINITY;
      else nan = true;
    }
    if (nan) {
      atomicOr(err, 1);
      mag = NAN;
    }
    double val = (c & 0x80) ? -mag : mag;
    if (scale) val *= scale[i];
    out[i] = (O)val;
  }
}

template <typename T>
void launch_encode(const void* x, const double* scale, int64_t n, int fmt, uint8_t* codes, int32_t* err,
                   cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>((n + kCodecThreads - 1) / kCodecThreads, device_sm_count() * 8);
  if (fmt == FPSA_E4M3)
    encode_kernel<T, FPSA_E4M3><<<blocks, kCodecThreads, 0, st>>>(static_cast<const T*>(x), scale, n, codes, err);
  else
    encode_kernel<T, FPSA_E5M2><<<blocks, kCodecThreads, 0, st>>>(static_cast<const T*>(x), scale, n, codes, err);
}
}  // namespace
}  // namespace fpsa

extern "C" int fpsa_encode(const void* x, int dtype, const double* scale, int64_t n, int fmt, uint8_t* codes,
                           int32_t* err_flag, void* stream) {
  clear_error();
  if (n < 0) return fail(FPSA_EINVAL, "n must be >= 0");
  if (n == 0) return FPSA_OK;
  if (!x || !codes || !err_flag) return fail(FPSA_EINVAL, "null buffer");
  if (fmt != FPSA_E4M3 && fmt != FPSA_E5M2) return fail(FPSA_EINVAL, "fmt must be e4m3 or e5m2");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == FPSA_F32) launch_encode<float>(x, scale, n, fmt, codes, err_flag, st);
  else if (dtype == FPSA_F64) launch_encode<double>(x, scale, n, fmt, codes, err_flag, st);
  else if (dtype == FPSA_BF16) launch_encode<__nv_bfloat16>(x, scale, n, fmt, codes, err_flag, st);
  else return fail(FPSA_EUNSUPPORTED, "input dtype must be f32, bf16 or f64");
  return cuda_status("fpsa_encode");
}

extern "C" int fpsa_decode(const uint8_t* codes, int64_t n, int fmt, const double* scale, void* out, int out_dtype,
                           int32_t* err_flag, void* stream) {
  clear_error();
  if (n < 0) return fail(FPSA_EINVAL, "n must be >= 0");
  if (n == 0) return FPSA_OK;
  if (!codes || !out || !err_flag) return fail(FPSA_EINVAL, "null buffer");
  if (fmt != FPSA_E4M3 && fmt != FPSA_E5M2) return fail(FPSA_EINVAL, "fmt must be e4m3 or e5m2");
  if (out_dtype != FPSA_F32 && out_dtype != FPSA_F64) return fail(FPSA_EUNSUPPORTED, "out dtype must be f32 or f64");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = (int)std::min<int64_t>((n + kCodecThreads - 1) / kCodecThreads, device_sm_count() * 8);
#define FPSA_DEC(F_, O_) decode_kernel<F_, O_><<<blocks, kCodecThreads, 0, st>>>(codes, scale, n, static_cast<O_*>(out), err_flag)
  if (fmt == FPSA_E4M3) {
    if (out_dtype == FPSA_F32) FPSA_DEC(FPSA_E4M3, float); else FPSA_DEC(FPSA_E4M3, double);
  } else {
    if (out_dtype == FPSA_F32) FPSA_DEC(FPSA_E5M2, float); else FPSA_DEC(FPSA_E5M2, double);
  }
#undef FPSA_DEC
  return cuda_status("fpsa_decode");
}

#ifdef FPSA_QTRACE
extern "C" int fpsa_qtrace_counts(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, fpsa::g_qcount, sizeof(fpsa::g_qcount)) == cudaSuccess ? 0 : 1;
}
extern "C" int fpsa_qtrace_timeline(long long* out) {
  cudaMemcpyFromSymbol(out, fpsa::g_qtl, sizeof(fpsa::g_qtl));
  return (int)(sizeof(fpsa::g_qtl) / sizeof(long long));
}
#endif
