// K4: sliding-tile sparse FP8 attention forward, sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces fp8sta.attention.fp8_sparse_forward / _engine
// (/root/reference/pkg/src/fp8sta/attention.py:91-149, :179-208).
//
// One CTA = (head h, query tile u, two 128-row query blocks of u).  The key
// sequence of u is the concatenation of its admissible key tiles in
// ascending id order (sparsity.py:63-67, the reference's reduction order),
// each key tile cut into 64-key blocks; a tile's last block has
// n_tail = tv - 64 (nb - 1) keys (rounded up to 16), so no padding key of a
// 240-token tile is multiplied or exponentiated.  Per key block j and query
// block q:
//
//   S(q,j) = Q_q K_j^T               tcgen05.mma kind::f8f6f4 M128 N64, A/B from
//                                    smem, fp32 accumulator in TMEM buffer (q, j % 2)
//   x      = S * (sq[u] * sk[v] * softmax_scale * log2 e)     per-tile factors
//   m      = reference row max, raised lazily (only when a block overflows the
//            e4m3 range above it)
//   P~     = e4m3(448 * 2^-tau * 2^(x - m))   re-quantised per key block,
//            written back to TMEM over S(q,j) (4 codes per column)
//   O_q   += P~ V_j                  tcgen05.mma, A = P~ from TMEM, B = V from
//                                    smem (MN-major, V stored [keys][d])
//   l      += sum of the unrounded P~ (fp32)
// and finally out = O * v_scale[c] / l.
//
// TMEM (512 columns): O_0, O_1 (128 each), S(0, even/odd), S(1, even/odd)
// (64 each).  With S double-buffered, QK(q, j+1) runs while the softmax
// works on S(q, j), and the MMA issue order PV(q, j), QK(q, j+2) never makes
// the softmax wait on its own P.
//
// Warp roles (320 threads): warps 0-3 own the 128 rows (TMEM lanes) of query
// block 0, warps 4-7 those of query block 1, one thread per row; warp 8 is
// the TMA producer (and TMEM allocator), warp 9 the MMA issuer.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <mutex>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"
#include "sm100.cuh"

namespace fpsa {
namespace {

using namespace sm100;

constexpr int kSoftmaxWarps = 8;
constexpr int kTmaWarp = kSoftmaxWarps;
constexpr int kMmaWarp = kSoftmaxWarps + 1;
constexpr int kThreads = (kSoftmaxWarps + 2) * 32;

constexpr int kStages = 8;    // K/V ring depth (64-key blocks)
constexpr int kBlk = 128;     // rows per query block
constexpr int kKeys = 64;     // keys per key block = S columns per softmax thread
constexpr int kFacCap = 2048;  // key-tile scale factors cached in shared memory per CTA
constexpr float kLog2_448 = 8.807354922057604f;
constexpr uint32_t kNegInf = 0xFF800000u;

struct AttnParams {
  const double* q_scales;
  const double* k_scales;
  const double* v_scales;
  const int32_t* offs;
  const int32_t* ids;
  const int32_t* items;
  int32_t M, tv, pitch, nb, nqb;  // nb: 64-key blocks per tile; nqb: 128-row query blocks per tile
  int32_t n_tail;     // S columns of the last key block of a tile (tv - 64 (nb-1), rounded up to 16)
  int32_t tail_pad8;  // 1 if the last 8 of those columns are zero padding (tv % 16 == 8)
  float softmax_log2;  // f32(softmax_scale * log2 e)
  float tau;
  void* out;
  int64_t out_ts, out_hs;
  int32_t natural;
  int32_t gh, gw, st, sh, sw, dh, dw;
};

template <int D>
struct Smem {
  static constexpr int kQTile = kBlk * D;   // bytes of one 128-row fp8 query block
  static constexpr int kKTile = kKeys * D;  // bytes of one 64-key fp8 K or V block
  static constexpr int kQ = 0;
  static constexpr int kK = 2 * kQTile;
  static constexpr int kV = kK + kStages * kKTile;
  static constexpr int kBytes = kV + kStages * kKTile;
  static constexpr uint32_t kSBO = 8 * D;  // 8 rows of D bytes
};

template <int D>
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t addr) {
  uint64_t d = smem_desc_sw128(addr, 16, Smem<D>::kSBO);
  if constexpr (D == 64) d = (d & ~((uint64_t)7 << 61)) | ((uint64_t)4 << 61);  // SWIZZLE_64B
  return d;
}
template <int D>
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t addr) {
  uint64_t d = smem_desc_sw128(addr, 16384, Smem<D>::kSBO);
  if constexpr (D == 64) d = (d & ~((uint64_t)7 << 61)) | ((uint64_t)4 << 61);
  return d;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float y;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
  return y;
}
// ---- packed f32x2 arithmetic (sm_100 FFMA2 / FADD2): two lanes per instruction
struct f2 {
  float x, y;
};
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ f2 bcast(float v) { return f2{v, v}; }

// Scalar saturating FMA (there is no .sat for f32x2): clamps to [0, 1].
__device__ __forceinline__ float fma_sat(float a, float b, float c) {
  float d;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x on the FMA pipe for a pair, x = s * c + noff given as
//   xs = sat(s * c/256 + (noff + 126)/256)  in [0, 1]   (x clamped to [-126, 130],
//   so the exponent add below never leaves the float range)
// Cody-Waite split x = j + f (j = round(x), |f| <= 1/2) with the rounding
// done by the magic-number add, then a degree-2 minimax for 2^f (rel. err
// 1.7e-3, far below the 2^-4 step of the e4m3 P it feeds) and j added to the
// exponent field.  Used for half of the columns so that MUFU ex2 (16/clk/SM)
// is not the only exp source.
__device__ __forceinline__ f2 exp2_poly_sat(f2 xs) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  const f2 t = fma2(xs, bcast(256.0f), bcast(kMagic - 126.0f));  // kMagic + round(x), x = 256 xs - 126
  const f2 g = add2(t, bcast(126.0f - kMagic));                   // round(x) + 126
  const f2 f = fma2(xs, bcast(256.0f), f2{-g.x, -g.y});           // x - round(x)
  f2 y = fma2(bcast(0.238487109541893f), f, bcast(0.703453540802002f));
  y = fma2(y, f, bcast(1.0004364252090454f));
  return f2{__uint_as_float(__float_as_uint(y.x) + (__float_as_uint(t.x) << 23)),
            __uint_as_float(__float_as_uint(y.y) + (__float_as_uint(t.y) << 23))};
}

// Four e4m3 codes in one word (a.x lowest byte).
__device__ __forceinline__ uint32_t e4m3x4(f2 a, f2 b) {
  uint32_t r;
  asm("{\n\t.reg .b16 lo, hi;\n\t"
      "cvt.rn.satfinite.e4m3x2.f32 lo, %2, %1;\n\t"
      "cvt.rn.satfinite.e4m3x2.f32 hi, %4, %3;\n\t"
      "mov.b32 %0, {lo, hi};\n\t}"
      : "=r"(r)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// P~ for 16 S columns [16U, 16U + 16) of a thread's half row, read from the
// 32-column chunk `s` that holds columns [32 (U/2), 32 (U/2) + 32): 4 groups
// of 4 keys, the odd groups (columns with bit 2 set) on the FMA-pipe
// polynomial, the even groups on MUFU ex2.  Writes 4 packed P words
// w[4U..4U+3] and accumulates the unrounded weights into acc.
template <int U>
__device__ __forceinline__ void softmax_unit(const uint32_t* s, f2 cc, f2 bb, float cs, float bs, f2* acc,
                                             uint32_t* w) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int c0 = 16 * (U & 1) + 4 * g;
    const f2 a{__uint_as_float(s[c0]), __uint_as_float(s[c0 + 1])};
    const f2 b{__uint_as_float(s[c0 + 2]), __uint_as_float(s[c0 + 3])};
    f2 pa, pb;
    if (g & 1) {
      pa = exp2_poly_sat(f2{fma_sat(a.x, cs, bs), fma_sat(a.y, cs, bs)});
      pb = exp2_poly_sat(f2{fma_sat(b.x, cs, bs), fma_sat(b.y, cs, bs)});
    } else {
      pa = fma2(a, cc, bb);
      pb = fma2(b, cc, bb);
      pa = f2{ex2(pa.x), ex2(pa.y)};
      pb = f2{ex2(pb.x), ex2(pb.y)};
    }
    acc[g & 1] = add2(acc[g & 1], pa);
    acc[2 + (g & 1)] = add2(acc[2 + (g & 1)], pb);
    w[4 * U + g] = e4m3x4(pa, pb);
  }
}

// The last 8 of the ncol valid columns are zero K rows (tv % 16 == 8): -inf
// drops them from max, sum and P.  `s` holds columns [base, base + 32).
__device__ __forceinline__ void mask_pad8(uint32_t* s, int base, int ncol) {
#pragma unroll
  for (int i = 8; i < 32; i += 16)
    if (base + i + 8 == ncol) {
#pragma unroll
      for (int k = i; k < i + 8; ++k) s[k] = kNegInf;
    }
}

template <int C>
__device__ __forceinline__ void softmax_chunk(uint32_t* s, int ncol, bool pad8, f2 cc, f2 bb, float cs, float bs,
                                              f2* acc, uint32_t* w) {
  if (pad8) mask_pad8(s, 32 * C, ncol);
  if (ncol > 32 * C) softmax_unit<2 * C>(s, cc, bb, cs, bs, acc, w);
  else w[8 * C] = w[8 * C + 1] = w[8 * C + 2] = w[8 * C + 3] = 0u;
  if (ncol > 32 * C + 16) softmax_unit<2 * C + 1>(s, cc, bb, cs, bs, acc, w);
  else w[8 * C + 4] = w[8 * C + 5] = w[8 * C + 6] = w[8 * C + 7] = 0u;
}

// One row of one key block: 64 S columns streamed from TMEM in two 32-column
// chunks (the second tcgen05.ld is in flight while the first chunk is
// processed), ncol (multiple of 16, 16..64) valid.  P words of absent
// columns are zero.  Returns the row sum of the unrounded weights.
__device__ __forceinline__ float softmax_block(uint32_t s_addr, int ncol, bool pad8, float c, float boff, uint32_t* w) {
  const f2 cc = bcast(c), bb = bcast(boff);
  const float cs = c * (1.0f / 256.0f), bs = (boff + 126.0f) * (1.0f / 256.0f);
  f2 acc[4] = {bcast(0.f), bcast(0.f), bcast(0.f), bcast(0.f)};
  uint32_t sa[32], sb[32];
  if (ncol > 0) {
    tmem_ld32(s_addr, sa);
    tmem_wait_ld();
  }
  if (ncol > 32) tmem_ld32(s_addr + 32, sb);
  softmax_chunk<0>(sa, ncol, pad8, cc, bb, cs, bs, acc, w);
  if (ncol > 32) tmem_wait_ld();
  softmax_chunk<1>(sb, ncol, pad8, cc, bb, cs, bs, acc, w);
  const f2 t = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
  return t.x + t.y;
}

// Max of the first ncol (16..64) raw S values of a row.
__device__ __forceinline__ float block_max(uint32_t s_addr, int ncol, bool pad8) {
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int base = 0; base < kKeys; base += 32) {
    if (base < ncol) {
      uint32_t s[32];
      tmem_ld32(s_addr + base, s);
      tmem_wait_ld();
      if (pad8) mask_pad8(s, base, ncol);
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        if (base + i < ncol) {
          m0 = max3(m0, __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
          m1 = max3(m1, __uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
        }
      }
    }
  }
  return fmaxf(m0, m1);
}

#ifdef FPSA_TRACE
// Debug builds only: counters accumulated over all CTAs.
//   [0] softmax: cycles waiting for S   [1] softmax: loop cycles   [2] softmax: first-pass compute
//   [3] MMA: cycles waiting for P~      [5] rescales   [6] steps   [7] MMA: cycles waiting for K/V
__device__ unsigned long long g_trace[8];
#endif

template <int D, int FMT, int OUT>
__global__ void __launch_bounds__(kThreads, 1)
    fpsa_attn_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using S = Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_o;
  __shared__ uint64_t bar_kv_full[kStages], bar_kv_empty[kStages];
  __shared__ uint64_t bar_s_full[2][2];   // [query block][S buffer]
  __shared__ uint64_t bar_p_ready[2][2];  // [query block][step parity]: a block's warps may run one step apart
  __shared__ uint64_t bar_pv[2];          // [query block]: PV(q, j) complete
  __shared__ uint32_t s_tmem;
  __shared__ float s_vscale[D];
  __shared__ float s_kfac[kFacCap];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t h = p.items[3 * blockIdx.x + 0];
  const int32_t u = p.items[3 * blockIdx.x + 1];
  const int32_t qb0 = p.items[3 * blockIdx.x + 2];
  const int nqb = min(2, p.nqb - qb0);
  const int32_t kt0 = p.offs[u];
  const int32_t n_kt = p.offs[u + 1] - kt0;
  const int32_t n_kv = n_kt * p.nb;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    mbar_init(&bar_o, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&bar_kv_full[i], 1);
      mbar_init(&bar_kv_empty[i], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&bar_s_full[q][0], 1);
      mbar_init(&bar_s_full[q][1], 1);
      mbar_init(&bar_p_ready[q][0], 4);  // one arrival per softmax warp of the block
      mbar_init(&bar_p_ready[q][1], 4);
      mbar_init(&bar_pv[q], 1);
    }
    fence_barrier_init();
  }
  if (warp == kTmaWarp) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  if (warp == kMmaWarp) {
    // per-CTA tables: V channel factors and the k-scale of every in-window key tile
    for (int i = lane; i < D; i += 32) s_vscale[i] = (float)p.v_scales[(int64_t)h * D + i];
    for (int i = lane; i < min(n_kt, kFacCap); i += 32)
      s_kfac[i] = (float)p.k_scales[(int64_t)h * p.M + p.ids[kt0 + i]];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  // O_q at column 128 q; S(q, buffer) at 256 + 128 q + 64 buffer (computed, not
  // indexed: a local array would live in memory)
  auto tm_o = [tmem](int q) { return tmem + 128u * (uint32_t)q; };
  auto tm_s = [tmem](int q, int32_t j) { return tmem + 256u + 128u * (uint32_t)q + 64u * (uint32_t)(j & 1); };

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer (warp-uniform, one elected lane issues)
    if (lane == 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
    }
    __syncwarp();
    const int32_t qrow = (h * p.M + u) * p.pitch + qb0 * kBlk;
    mbar_arrive_expect_tx_w(&bar_q, nqb * S::kQTile);
    for (int q = 0; q < nqb; ++q) tma_load_2d_w(smem + S::kQ + q * S::kQTile, &tm_q, 0, qrow + q * kBlk, &bar_q);
    int32_t kt = 0, b = 0, st = 0;
    uint32_t ph = 0;
    int32_t krow = (h * p.M + p.ids[kt0]) * p.pitch;
    for (int32_t j = 0; j < n_kv; ++j) {
      if (j >= kStages) mbar_wait(&bar_kv_empty[st], ph ^ 1);
      mbar_arrive_expect_tx_w(&bar_kv_full[st], 2 * S::kKTile);
      tma_load_2d_w(smem + S::kK + st * S::kKTile, &tm_k, 0, krow + b * kKeys, &bar_kv_full[st]);
      tma_load_2d_w(smem + S::kV + st * S::kKTile, &tm_v, 0, krow + b * kKeys, &bar_kv_full[st]);
      if (++b == p.nb) {
        b = 0;
        if (++kt < n_kt) krow = (h * p.M + __ldg(p.ids + kt0 + kt)) * p.pitch;
      }
      if (++st == kStages) {
        st = 0;
        ph ^= 1;
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (warp-uniform, one elected lane issues)
    constexpr uint32_t idesc_qk = idesc_f8(128, kKeys, FMT, FMT, 0);
    const uint32_t idesc_qk_tail = idesc_f8(128, (uint32_t)p.n_tail, FMT, FMT, 0);
    constexpr uint32_t idesc_pv = idesc_f8(128, D, FPSA_E4M3, FMT, 1);
    const uint32_t sq = smem_u32(smem + S::kQ);
    const uint32_t sk0 = smem_u32(smem + S::kK), sv0 = smem_u32(smem + S::kV);
    mbar_wait(&bar_q, 0);
    tc_fence_after();
    // S(q, j) = Q_q K_j^T into TMEM buffer (q, j % 2); (st, b) = stage and in-tile block of j
    auto issue_qk = [&](int q, int32_t j, int st, bool tail) {
      const uint32_t sk = sk0 + st * S::kKTile;
      const uint32_t idq = tail ? idesc_qk_tail : idesc_qk;
      const uint32_t sqq = sq + q * S::kQTile;
#pragma unroll
      for (int k = 0; k < D / 32; ++k)
        mma_f8_ss_w(tm_s(q, j), desc_kmajor<D>(sqq + 32 * k), desc_kmajor<D>(sk + 32 * k), idq, k > 0 ? 1u : 0u);
      mma_commit_w(&bar_s_full[q][j & 1]);
    };
    // (st2, b2): stage / in-tile block of step j + 2, with the full-barrier phase
    int st2 = 0, b2 = 0;
    uint32_t ph2 = 0;
    auto advance2 = [&]() {
      if (++b2 == p.nb) b2 = 0;
      if (++st2 == kStages) {
        st2 = 0;
        ph2 ^= 1;
      }
    };
    for (int32_t j = 0; j < min(n_kv, 2); ++j) {
      mbar_wait(&bar_kv_full[st2], ph2);
      tc_fence_after();
      for (int q = 0; q < nqb; ++q) issue_qk(q, j, st2, b2 == p.nb - 1);
      advance2();
    }
    int st = 0;
    for (int32_t j = 0; j < n_kv; ++j) {
      const uint32_t sv = sv0 + st * S::kKTile;
      const bool more = j + 2 < n_kv;
      if (more) {
#ifdef FPSA_TRACE
        const long long tk0 = clock64();
#endif
        mbar_wait(&bar_kv_full[st2], ph2);
#ifdef FPSA_TRACE
        if (lane == 0) atomicAdd(&g_trace[7], (unsigned long long)(clock64() - tk0));
#endif
        tc_fence_after();
      }
      for (int q = 0; q < nqb; ++q) {
        // O_q += P~(q, j) V_j once the softmax has written P~ over S(q, j)
#ifdef FPSA_TRACE
        const long long tp0 = clock64();
#endif
        mbar_wait(&bar_p_ready[q][j & 1], (j >> 1) & 1);
#ifdef FPSA_TRACE
        if (lane == 0) atomicAdd(&g_trace[3], (unsigned long long)(clock64() - tp0));
#endif
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kKeys / 32; ++k)
          mma_f8_ts_w(tm_o(q), tm_s(q, j) + 8 * k, desc_mnmajor<D>(sv + k * 32 * D), idesc_pv,
                      (j > 0 || k > 0) ? 1u : 0u);
        mma_commit_w(&bar_pv[q]);
        if (more) issue_qk(q, j + 2, st2, b2 == p.nb - 1);
      }
      mma_commit_w(&bar_kv_empty[st]);
      if (more) advance2();
      if (++st == kStages) st = 0;
    }
    mma_commit_w(&bar_o);
  } else if (warp / 4 < nqb) {
    // ------------------------------------------------------------ softmax: one thread per row
    const int q = warp / 4;                     // query block
    const int row = (warp & 3) * 32 + lane;     // TMEM lane = row of the query block
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t o_addr = tm_o(q) + lane_off;
    const float qs = (float)p.q_scales[h * p.M + u];
    const float sl = p.softmax_log2;
    const float tau = p.tau;
    // Rows keep a reference max m_ref (log2 units); P~ = e4m3(448 * 2^(x - m_ref - tau)).
    // No per-block max is taken: if the row sum of P~ stays <= 448 no element
    // can have saturated and the block is accepted as computed.  The first
    // block and blocks with a larger sum (a logit above m_ref + tau, or a
    // false alarm) take the exact path, which lazily raises m_ref for the
    // warp and rescales the TMEM accumulator (oracle.onepass_forward).
    float m_ref = 0.0f, l = 0.0f;
    int32_t kt = 0, b = 0;
#ifdef FPSA_TRACE
    long long w_s = 0, w_c = 0, n_resc = 0;
    const long long t_loop = clock64();
#endif
    for (int32_t j = 0; j < n_kv; ++j) {
      const float kf = kt < kFacCap ? s_kfac[kt] : (float)__ldg(p.k_scales + h * p.M + __ldg(p.ids + kt0 + kt));
      const float c = (qs * kf) * sl;
      const bool tail = b == p.nb - 1;
      const int ncol = tail ? p.n_tail : kKeys;
      const bool pad8 = tail && p.tail_pad8;
      const uint32_t s_addr = tm_s(q, j) + lane_off;
#ifdef FPSA_TRACE
      const long long ts0 = clock64();
#endif
      mbar_wait(&bar_s_full[q][j & 1], (j >> 1) & 1);
#ifdef FPSA_TRACE
      w_s += clock64() - ts0;
      const long long tc0 = clock64();
#endif
      tc_fence_after();
      if (j == 0) m_ref = block_max(s_addr, ncol, pad8) * c;
      uint32_t w[kKeys / 4];
      float lb;
      bool redo = false;
#pragma unroll 1
      for (;;) {  // one pass; a second one only after the exact path raised m_ref
        lb = softmax_block(s_addr, ncol, pad8, c, kLog2_448 - m_ref - tau, w);
#ifdef FPSA_TRACE
        if (!redo) w_c += clock64() - tc0;
#endif
        // a row sum <= 448 bounds every element
        if (redo || !__any_sync(0xffffffffu, lb > 448.0f)) break;
        const float mb = block_max(s_addr, ncol, pad8) * c;
        if (!__any_sync(0xffffffffu, mb > m_ref + tau)) break;
        const float m_new = fmaxf(m_ref, mb);
        const float alpha = ex2(m_ref - m_new);
        l *= alpha;
        m_ref = m_new;
#ifdef FPSA_TRACE
        ++n_resc;
#endif
        if (j > 0) mbar_wait(&bar_pv[q], (j - 1) & 1);  // O complete up to block j-1
        tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t o[32];
          tmem_ld32(o_addr + cc, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(o_addr + cc, o);
        }
        tmem_wait_st();
        redo = true;
      }
      l += lb;
      tmem_st16(s_addr, w);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p_ready[q][j & 1]);
      if (++b == p.nb) {
        b = 0;
        ++kt;
      }
    }
#ifdef FPSA_TRACE
    if (lane == 0) {
      atomicAdd(&g_trace[0], (unsigned long long)w_s);
      atomicAdd(&g_trace[1], (unsigned long long)(clock64() - t_loop));
      atomicAdd(&g_trace[2], (unsigned long long)w_c);
      atomicAdd(&g_trace[5], (unsigned long long)n_resc);
      atomicAdd(&g_trace[6], (unsigned long long)n_kv);
    }
#endif
    // ------------------------------------------------------------ epilogue
    mbar_wait(&bar_o, 0);
    tc_fence_after();
    const float inv_l = 1.0f / l;
    const int32_t r = (qb0 + q) * kBlk + row;  // row inside the tile
    int64_t token;
    if (p.natural) {
      const int32_t ut = u / (p.dh * p.dw), uh = (u / p.dw) % p.dh, uw = u % p.dw;
      const int32_t lt = r / (p.sh * p.sw), lh = (r / p.sw) % p.sh, lw = r % p.sw;
      token = ((int64_t)(ut * p.st + lt) * p.gh + (uh * p.sh + lh)) * p.gw + (uw * p.sw + lw);
    } else {
      token = (int64_t)u * p.tv + r;
    }
#pragma unroll 1
    for (int col = 0; col < D; col += 32) {
      uint32_t o[32];
      tmem_ld32(o_addr + col, o);
      tmem_wait_ld();
      if (r < p.tv) {
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(o[i]) * inv_l * s_vscale[col + i];
        if constexpr (OUT == FPSA_F32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + token * p.out_ts + h * p.out_hs + col);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + token * p.out_ts + h * p.out_hs + col);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint32_t wv[4];
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) {
              __nv_bfloat162 b2 = __floats2bfloat162_rn(f[8 * i + 2 * k2], f[8 * i + 2 * k2 + 1]);
              wv[k2] = *reinterpret_cast<uint32_t*>(&b2);
            }
            dst[i] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kTmaWarp) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- host side
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

int make_code_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int32_t d, int32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(FPSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d};
  cuuint32_t box[2] = {(cuuint32_t)d, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, d == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FPSA_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return FPSA_OK;
}

template <int D, int FMT, int OUT>
int launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p, int32_t n_items,
           cudaStream_t st) {
  auto kern = fpsa_attn_kernel<D, FMT, OUT>;
  constexpr int smem = Smem<D>::kBytes + 1024;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return fail(FPSA_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(cudaGetLastError()));
    configured = true;
  }
  kern<<<n_items, kThreads, smem, st>>>(tq, tk, tv, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FPSA_ECUDA, std::string("fpsa_attn_fwd launch: ") + cudaGetErrorString(e));
  return FPSA_OK;
}

}  // namespace
}  // namespace fpsa

using namespace fpsa;

extern "C" int fpsa_attn_fwd(const uint8_t* q_codes, const uint8_t* k_codes, const uint8_t* v_codes,
                             const double* q_scales, const double* k_scales, const double* v_scales, int32_t heads,
                             fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, const int32_t* offs,
                             const int32_t* ids, const int32_t* items, int32_t n_items, float softmax_scale, int fmt,
                             float tau_log2, void* out, int out_dtype, int64_t out_token_stride,
                             int64_t out_head_stride, int out_order, void* stream) {
  clear_error();
  fpsa_dims3 td;
  if (int s = fpsa_tile_grid(grid, tile, &td)) return s;
  if (!q_codes || !k_codes || !v_codes || !q_scales || !k_scales || !v_scales || !offs || !ids || !items || !out)
    return fail(FPSA_EINVAL, "null buffer");
  if (d != 64 && d != 128) return fail(FPSA_EUNSUPPORTED, "head dim must be 64 or 128, got " + std::to_string(d));
  const int32_t tv = tile.t * tile.h * tile.w;
  if (tile_pitch < tv || tile_pitch % kBlk) return fail(FPSA_EINVAL, "tile_pitch must be a multiple of 128 >= tile volume");
  if (tv % 8) return fail(FPSA_EUNSUPPORTED, "tile volume must be a multiple of 8, got " + std::to_string(tv));
  if (!(softmax_scale > 0.0f)) return fail(FPSA_EINVAL, "softmax_scale must be > 0");
  if (fmt != FPSA_E4M3 && fmt != FPSA_E5M2) return fail(FPSA_EINVAL, "fmt must be e4m3 or e5m2");
  if (out_dtype != FPSA_F32 && out_dtype != FPSA_BF16) return fail(FPSA_EUNSUPPORTED, "out dtype must be f32 or bf16");
  if (!(tau_log2 >= 0.0f && tau_log2 <= 8.0f)) return fail(FPSA_EINVAL, "tau_log2 must be in [0, 8]");
  if (heads < 1 || n_items < 1) return fail(FPSA_EINVAL, "empty problem");
  const int32_t M = td.t * td.h * td.w;
  const int64_t rows = (int64_t)heads * M * tile_pitch;
  CUtensorMap tq, tk, tvm;
  if (int s = make_code_map(&tq, q_codes, rows, d, kBlk)) return s;
  if (int s = make_code_map(&tk, k_codes, rows, d, kKeys)) return s;
  if (int s = make_code_map(&tvm, v_codes, rows, d, kKeys)) return s;
  AttnParams p{};
  p.q_scales = q_scales;
  p.k_scales = k_scales;
  p.v_scales = v_scales;
  p.offs = offs;
  p.ids = ids;
  p.items = items;
  p.M = M;
  p.tv = tv;
  p.pitch = tile_pitch;
  p.nb = (tv + kKeys - 1) / kKeys;
  p.nqb = (tv + kBlk - 1) / kBlk;
  {
    const int32_t tail = tv - kKeys * (p.nb - 1);  // valid keys of a tile's last 64-key block
    p.n_tail = (tail + 15) / 16 * 16;
    p.tail_pad8 = p.n_tail != tail;
  }
  p.softmax_log2 = softmax_scale * 1.4426950408889634f;
  p.tau = tau_log2;
  p.out = out;
  p.out_ts = out_token_stride;
  p.out_hs = out_head_stride;
  p.natural = out_order == FPSA_ORDER_NATURAL;
  p.gh = grid.h;
  p.gw = grid.w;
  p.st = tile.t;
  p.sh = tile.h;
  p.sw = tile.w;
  p.dh = td.h;
  p.dw = td.w;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define FPSA_LAUNCH(D_, F_, O_) return launch<D_, F_, O_>(tq, tk, tvm, p, n_items, st)
  if (d == 128) {
    if (fmt == FPSA_E4M3) {
      if (out_dtype == FPSA_F32) FPSA_LAUNCH(128, FPSA_E4M3, FPSA_F32); else FPSA_LAUNCH(128, FPSA_E4M3, FPSA_BF16);
    } else {
      if (out_dtype == FPSA_F32) FPSA_LAUNCH(128, FPSA_E5M2, FPSA_F32); else FPSA_LAUNCH(128, FPSA_E5M2, FPSA_BF16);
    }
  } else {
    if (fmt == FPSA_E4M3) {
      if (out_dtype == FPSA_F32) FPSA_LAUNCH(64, FPSA_E4M3, FPSA_F32); else FPSA_LAUNCH(64, FPSA_E4M3, FPSA_BF16);
    } else {
      if (out_dtype == FPSA_F32) FPSA_LAUNCH(64, FPSA_E5M2, FPSA_F32); else FPSA_LAUNCH(64, FPSA_E5M2, FPSA_BF16);
    }
  }
#undef FPSA_LAUNCH
}

#ifdef FPSA_TRACE
extern "C" int fpsa_trace_read(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, fpsa::g_trace, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(fpsa::g_trace, z, sizeof z);
  }
  return 0;
}
#endif
