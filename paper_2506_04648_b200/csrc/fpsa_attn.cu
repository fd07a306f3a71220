// K4: sliding-tile sparse FP8 attention forward, sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces fp8sta.attention.fp8_sparse_forward / _engine
// (/root/reference/pkg/src/fp8sta/attention.py:91-149, :179-208).
//
// One CTA = (head h, query tile u, up to two 128-row query blocks of u).
// The key sequence of u is the concatenation of its admissible key tiles in
// ascending id order (sparsity.py:63-67, the reference's reduction order),
// each key tile cut into 128-key blocks (tiles are stored padded to a
// multiple of 128 rows, pad rows zero and masked).  Per key block j:
//
//   S_q(j)  = Q_q K_j^T              tcgen05.mma kind::f8f6f4, A/B from smem,
//                                    fp32 accumulator in TMEM (128 lanes x 128 cols)
//   x       = S * (sq[u] * sk[v] * softmax_scale * log2 e)     per-tile factors
//   m       = running row max, rescaled lazily (only when a block max exceeds
//             the reference max by more than tau)
//   P~      = e4m3(448 * 2^-tau * 2^(x - m))  re-quantised per tile, written
//             back to TMEM (4 codes per column, aliasing S_q)
//   O_q    += P~ V_j                  tcgen05.mma, A = P~ from TMEM, B = V from
//                                    smem (MN-major, V stored [keys][d])
//   l      += sum of the unrounded P~ (fp32)
// and finally out = O * v_scale[c] / l.
//
// Warp roles (320 threads): warps 0-3 softmax for query block 0, warps 4-7
// for query block 1 (one thread per row = TMEM lane), warp 8 TMA producer
// (and TMEM allocator), warp 9 MMA issuer.  The two query blocks ping-pong so
// that the tensor core works on one block while the other is in softmax.
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

// 16 softmax warps: for each 128-row query block, warps w and w+4 share the
// TMEM lane quarter w and split the 128 S columns in two halves (a "pair"),
// plus a TMA warp and an MMA warp.
constexpr int kSoftmaxWarps = 16;
constexpr int kHalf = 64;  // S columns per softmax thread
constexpr int kTmaWarp = kSoftmaxWarps;
constexpr int kMmaWarp = kSoftmaxWarps + 1;
constexpr int kThreads = (kSoftmaxWarps + 2) * 32;

constexpr int kStages = 4;
constexpr int kBlk = 128;  // rows per query block and keys per key block
constexpr float kLog2_448 = 8.807354922057604f;
// Groups of 4 columns whose exp2 runs on the FMA pipe (polynomial) instead of
// MUFU ex2: every other group, so both pipes stay busy in the same instruction
// window (MUFU ex2 alone would bound the kernel at 16 exp/clk/SM).
__device__ __forceinline__ constexpr bool kPolyGroup(int g) { return (g & 1) == 1; }

struct AttnParams {
  const double* q_scales;
  const double* k_scales;
  const double* v_scales;
  const int32_t* offs;
  const int32_t* ids;
  const int32_t* items;
  int32_t M, tv, pitch, nb;
  float scale_log2;  // softmax_scale * log2(e)
  float tau;
  void* out;
  int64_t out_ts, out_hs;
  int32_t natural;
  int32_t gh, gw, st, sh, sw, dh, dw;
};

template <int D>
struct Smem {
  static constexpr int kTile = kBlk * D;  // bytes of one 128-row fp8 tile
  static constexpr int kQ = 0;
  static constexpr int kK = 2 * kTile;
  static constexpr int kV = kK + kStages * kTile;
  static constexpr int kBytes = kV + kStages * kTile;
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
__device__ __forceinline__ f2 fma_sat_pair(f2 a, float b, float c) {
  f2 d;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d.x) : "f"(a.x), "f"(b), "f"(c));
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d.y) : "f"(a.y), "f"(b), "f"(c));
  return d;
}

// 2^x on the FMA pipe for a pair, x = s * c + noff given as
//   xs = sat(s * c/256 + (noff + 126)/256)  in [0, 1]   (x clamped to [-126, 130],
//   so the exponent add below never leaves the float range)
// Cody-Waite split x = j + f (j = round(x), |f| <= 1/2) with the rounding
// done by the magic-number add, then a degree-2 minimax for 2^f (rel. err
// 1.7e-3, far below the 2^-4 step of the e4m3 P it feeds) and j added to the
// exponent field.  Used for a fraction of the columns so that MUFU ex2 is not
// the only exp source.
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

__device__ __forceinline__ uint32_t e4m3x2(float hi, float lo) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

#ifdef FPSA_TRACE
// Debug builds only: cycle counters accumulated over all CTAs.
//   [0] softmax: waiting for S   [1] softmax: total loop   [2] MMA: waiting for K/V
//   [3] MMA: waiting for P       [4] MMA: total loop        [5] softmax: rescale count
__device__ unsigned long long g_trace[8];
#define TRACE_T0() const long long _t0 = clock64()
#define TRACE_ADD(i, v) atomicAdd(&g_trace[i], (unsigned long long)(v))
#else
#define TRACE_T0()
#define TRACE_ADD(i, v)
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
  __shared__ uint64_t bar_s_full[2], bar_p_ready[2];
  __shared__ uint32_t s_tmem;
  __shared__ float s_vscale[D];
  __shared__ float s_xchg[2][2][kBlk];       // [query block][half][row] pair exchange
  __shared__ uint32_t s_flag[2][8][2];       // [j parity][pair][half] overflow verdicts

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t h = p.items[3 * blockIdx.x + 0];
  const int32_t u = p.items[3 * blockIdx.x + 1];
  const int32_t qb0 = p.items[3 * blockIdx.x + 2];
  const int nqb = min(2, p.nb - qb0);
  const int32_t kt0 = p.offs[u];
  const int32_t n_kv = (p.offs[u + 1] - kt0) * p.nb;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    mbar_init(&bar_o, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&bar_kv_full[i], 1);
      mbar_init(&bar_kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_s_full[i], 1);
      mbar_init(&bar_p_ready[i], 256);
    }
    fence_barrier_init();
  }
  if (warp == kTmaWarp) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  if (warp == kMmaWarp) {
    for (int i = lane; i < D; i += 32) s_vscale[i] = (float)p.v_scales[(int64_t)h * D + i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tm_s[2] = {tmem, tmem + 128};
  const uint32_t tm_o[2] = {tmem + 256, tmem + 256 + D};

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
      const int32_t qrow = (h * p.M + u) * p.pitch + qb0 * kBlk;
      mbar_arrive_expect_tx(&bar_q, nqb * S::kTile);
      for (int q = 0; q < nqb; ++q) tma_load_2d(smem + S::kQ + q * S::kTile, &tm_q, 0, qrow + q * kBlk, &bar_q);
      for (int32_t j = 0; j < n_kv; ++j) {
        const int st = j % kStages;
        if (j >= kStages) mbar_wait(&bar_kv_empty[st], ((j / kStages) - 1) & 1);
        const int32_t kt = j / p.nb, b = j - kt * p.nb;
        const int32_t v = p.ids[kt0 + kt];
        const int32_t krow = (h * p.M + v) * p.pitch + b * kBlk;
        mbar_arrive_expect_tx(&bar_kv_full[st], 2 * S::kTile);
        tma_load_2d(smem + S::kK + st * S::kTile, &tm_k, 0, krow, &bar_kv_full[st]);
        tma_load_2d(smem + S::kV + st * S::kTile, &tm_v, 0, krow, &bar_kv_full[st]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_f8(128, 128, FMT, FMT, 0);
      constexpr uint32_t idesc_pv = idesc_f8(128, D, FPSA_E4M3, FMT, 1);
      const uint32_t sq = smem_u32(smem + S::kQ);
      mbar_wait(&bar_q, 0);
      tc_fence_after();
#ifdef FPSA_TRACE
      long long w_kv = 0, w_p = 0;
      const long long t_loop = clock64();
#endif
      for (int32_t j = 0; j <= n_kv; ++j) {
        const int st = j % kStages;
        if (j < n_kv) {
#ifdef FPSA_TRACE
          const long long ta = clock64();
#endif
          mbar_wait(&bar_kv_full[st], (j / kStages) & 1);
#ifdef FPSA_TRACE
          w_kv += clock64() - ta;
#endif
          tc_fence_after();
        }
        const int pst = (j + kStages - 1) % kStages;  // stage of block j-1
        const uint32_t sk = smem_u32(smem + S::kK + st * S::kTile);
        const uint32_t sv_prev = smem_u32(smem + S::kV + pst * S::kTile);
        for (int q = 0; q < nqb; ++q) {
          if (j > 0) {
#ifdef FPSA_TRACE
            const long long tb = clock64();
#endif
            mbar_wait(&bar_p_ready[q], (j - 1) & 1);
#ifdef FPSA_TRACE
            w_p += clock64() - tb;
#endif
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < kBlk / 32; ++k)
              mma_f8_ts(tm_o[q], tm_s[q] + 8 * k, desc_mnmajor<D>(sv_prev + k * 32 * D), idesc_pv,
                        (j > 1 || k > 0) ? 1u : 0u);
          }
          if (j < n_kv) {
            const uint32_t sqq = sq + q * S::kTile;
#pragma unroll
            for (int k = 0; k < D / 32; ++k)
              mma_f8_ss(tm_s[q], desc_kmajor<D>(sqq + 32 * k), desc_kmajor<D>(sk + 32 * k), idesc_qk, k > 0 ? 1u : 0u);
            mma_commit(&bar_s_full[q]);
          }
        }
        if (j > 0) mma_commit(&bar_kv_empty[pst]);
      }
      mma_commit(&bar_o);
#ifdef FPSA_TRACE
      TRACE_ADD(2, w_kv);
      TRACE_ADD(3, w_p);
      TRACE_ADD(4, clock64() - t_loop);
#endif
    }
  } else if (warp / 8 < nqb) {
    // ------------------------------------------------------------ softmax: row x column half
    const int q = warp / 8;               // query block
    const int c = (warp / 4) & 1;         // column half of S and O owned by this thread
    const int pair = warp & 7 & 3 | (q << 2);  // warps (w, w+4) of a query block share TMEM lanes
    const int row = threadIdx.x & 127;    // TMEM lane = row of the query block
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t s_half = tm_s[q] + lane_off + c * kHalf;
    const uint32_t p_half = tm_s[q] + lane_off + c * (kHalf / 4);
    const uint32_t o_half = tm_o[q] + lane_off + c * (D / 2);
    const float cq = (float)p.q_scales[h * p.M + u] * p.scale_log2;
    const float tau = p.tau;
    auto pair_sync = [&]() { named_bar_sync(1 + pair, 64); };
    // Rows keep a reference max m_ref; P~ = e4m3(448 * 2^(x - m_ref - tau)).
    // No per-block max is taken: if both half-row sums of P~ stay <= 448 no
    // element can have saturated and the block is accepted as computed.  The
    // first block and blocks with a larger sum (a logit above m_ref + tau, or
    // a false alarm) take the exact path, which lazily raises m_ref and
    // rescales the TMEM accumulator; the two halves of a row decide together.
    float m_ref = 0.0f, l = 0.0f;
#ifdef FPSA_TRACE
    long long w_s = 0, n_resc = 0;
    const long long t_loop = clock64();
#endif
    for (int32_t j = 0; j < n_kv; ++j) {
      const int32_t kt = j / p.nb, b = j - kt * p.nb;
      const int32_t v = __ldg(p.ids + kt0 + kt);
      const float cj = cq * (float)__ldg(p.k_scales + h * p.M + v);
      const int valid = min(kBlk, p.tv - b * kBlk) - c * kHalf;  // valid columns of this half (may be <= 0)
#ifdef FPSA_TRACE
      const long long ts0 = clock64();
#endif
      mbar_wait(&bar_s_full[q], j & 1);
#ifdef FPSA_TRACE
      w_s += clock64() - ts0;
#endif
      tc_fence_after();
      float sv[kHalf];
      // S stays intact in TMEM until P is written over it: the exact path reloads it.
      auto load_s = [&]() {
        tmem_ld32(s_half + 0, reinterpret_cast<uint32_t*>(sv + 0));
        tmem_ld32(s_half + 32, reinterpret_cast<uint32_t*>(sv + 32));
        tmem_wait_ld();
        // key columns >= valid are padding (zero K/V rows of a key tile's last
        // block): -inf drops them from max, sum and P (valid % 8 == 0, host-checked)
        if (valid < kHalf) {
#pragma unroll
          for (int i = 0; i < kHalf; i += 8) {
            const bool ok = i < valid;
#pragma unroll
            for (int k2 = i; k2 < i + 8; ++k2) sv[k2] = ok ? sv[k2] : -INFINITY;
          }
        }
      };
      // exact row max over both halves (pair exchange through shared memory)
      auto row_max = [&]() {
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int i = 0; i < kHalf; i += 4) {
          mx0 = max3(mx0, sv[i], sv[i + 1]);
          mx1 = max3(mx1, sv[i + 2], sv[i + 3]);
        }
        s_xchg[q][c][row] = fmaxf(mx0, mx1);
        pair_sync();
        const float m = fmaxf(s_xchg[q][0][row], s_xchg[q][1][row]) * cj;
        pair_sync();  // the exchange slots are reused
        return m;
      };
      uint32_t w[kHalf / 4];
      auto exp_half = [&](float mref) {
        const f2 cc2 = bcast(cj), noff = bcast(kLog2_448 - mref - tau);
        const float cs = cj * (1.0f / 256.0f), ns = (kLog2_448 - mref - tau + 126.0f) * (1.0f / 256.0f);
        f2 lsum0 = bcast(0.0f), lsum1 = bcast(0.0f);
#pragma unroll
        for (int k2 = 0; k2 < kHalf; k2 += 4) {
          f2 pa, pb;
          if (kPolyGroup(k2 / 4)) {
            pa = exp2_poly_sat(fma_sat_pair(f2{sv[k2], sv[k2 + 1]}, cs, ns));
            pb = exp2_poly_sat(fma_sat_pair(f2{sv[k2 + 2], sv[k2 + 3]}, cs, ns));
          } else {
            pa = fma2(f2{sv[k2], sv[k2 + 1]}, cc2, noff);
            pb = fma2(f2{sv[k2 + 2], sv[k2 + 3]}, cc2, noff);
            pa = f2{ex2(pa.x), ex2(pa.y)};
            pb = f2{ex2(pb.x), ex2(pb.y)};
          }
          lsum0 = add2(lsum0, pa);
          lsum1 = add2(lsum1, pb);
          w[k2 / 4] = e4m3x4(pa, pb);
        }
        const f2 ls = add2(lsum0, lsum1);
        return ls.x + ls.y;
      };
      load_s();
      if (j == 0) m_ref = row_max();
      float lb = exp_half(m_ref);
      // half-row sums <= 448 bound every element; the pair agrees on the verdict
      const uint32_t over = __any_sync(0xffffffffu, lb > 448.0f) ? 1u : 0u;
      if (lane == 0) s_flag[j & 1][pair][c] = over;
      pair_sync();
      if (s_flag[j & 1][pair][0] | s_flag[j & 1][pair][1]) {
        load_s();
        const float mb = row_max();
        if (__any_sync(0xffffffffu, mb > m_ref + tau)) {  // identical in both warps of the pair
          const float m_new = fmaxf(m_ref, mb);
          const float alpha = ex2(m_ref - m_new);
          l *= alpha;
          m_ref = m_new;
#ifdef FPSA_TRACE
          ++n_resc;
#endif
#pragma unroll 1
          for (int cc = 0; cc < D / 2; cc += 16) {
            uint32_t o[16];
            tmem_ld16(o_half + cc, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(o_half + cc, o);
          }
          tmem_wait_st();
          lb = exp_half(m_ref);
        }
      }
      l += lb;
      tmem_st16(p_half, w);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar_p_ready[q]);
    }
#ifdef FPSA_TRACE
    if (lane == 0) {
      TRACE_ADD(0, w_s);
      TRACE_ADD(1, clock64() - t_loop);
      TRACE_ADD(5, n_resc);
      TRACE_ADD(6, n_kv);
    }
#endif
    // ------------------------------------------------------------ epilogue
    s_xchg[q][c][row] = l;
    mbar_wait(&bar_o, 0);
    tc_fence_after();
    pair_sync();
    const float inv_l = 1.0f / (s_xchg[q][0][row] + s_xchg[q][1][row]);
    const int32_t r = (qb0 + q) * kBlk + row;  // row inside the tile
    int64_t token;
    if (p.natural) {
      const int32_t ut = u / (p.dh * p.dw), uh = (u / p.dw) % p.dh, uw = u % p.dw;
      const int32_t lt = r / (p.sh * p.sw), lh = (r / p.sw) % p.sh, lw = r % p.sw;
      token = ((int64_t)(ut * p.st + lt) * p.gh + (uh * p.sh + lh)) * p.gw + (uw * p.sw + lw);
    } else {
      token = (int64_t)u * p.tv + r;
    }
#pragma unroll
    for (int cc = 0; cc < D / 2; cc += 32) {
      const int col = c * (D / 2) + cc;
      uint32_t o[32];
      tmem_ld32(o_half + cc, o);
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

int make_code_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int32_t d) {
  auto fn = encode_fn();
  if (!fn) return fail(FPSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d};
  cuuint32_t box[2] = {(cuuint32_t)d, (cuuint32_t)kBlk};
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
  if (int s = make_code_map(&tq, q_codes, rows, d)) return s;
  if (int s = make_code_map(&tk, k_codes, rows, d)) return s;
  if (int s = make_code_map(&tvm, v_codes, rows, d)) return s;
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
  p.nb = tile_pitch / kBlk;
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
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
