// Per-row softmax building blocks of the attention kernel (fpsa_attn.cu):
// packed f32x2 arithmetic, the FMA-pipe exp2 polynomial, e4m3 packing, and
// the 64-column half-row pass that turns S (TMEM) into P~ words.
// Shared with tools/probes/softmax_rate.cu, which times them in isolation.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

namespace fpsa {
namespace {

using namespace sm100;

constexpr int kHalf = 64;  // S columns per softmax thread

#ifdef FPSA_TRACE
__device__ unsigned long long g_trace[8];  // debug builds only, see fpsa_attn.cu
// per-step timeline of CTA 0 (clock64): softmax warps 0..7 x 4 events, MMA warp 4 events
constexpr int kTlSteps = 256;
__device__ long long g_tl[kTlSteps][10][4];
#define FPSA_TL(slot, ev, step)                                                        \
  do {                                                                                 \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (step) < kTlSteps && (slot) < 10) \
      g_tl[(step)][(slot)][(ev)] = clock64();                                          \
  } while (0)
#else
#define FPSA_TL(slot, ev, step) \
  do {                          \
  } while (0)
#endif
constexpr uint32_t kNegInf = 0xFF800000u;

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

// y + (t << 23): adds the rounded exponent to y's exponent field.  Written as
// a clamped funnel shift so ptxas emits LEA.HI on the ALU pipe instead of an
// IMAD on the (busier) FMA pipe.
__device__ __forceinline__ uint32_t exp_insert(uint32_t y, uint32_t t) {
  uint32_t r;
  asm("{\n\t.reg .b32 e;\n\tshf.l.clamp.b32 e, 0, %1, 23;\n\tadd.u32 %0, e, %2;\n\t}" : "=r"(r) : "r"(t), "r"(y));
  return r;
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
  return f2{__uint_as_float(exp_insert(__float_as_uint(y.x), __float_as_uint(t.x))),
            __uint_as_float(exp_insert(__float_as_uint(y.y), __float_as_uint(t.y)))};
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
// 32-column chunk `s` that holds columns [32 (U/2), 32 (U/2) + 32): in each
// group of 4 keys, columns 0 and 1 on MUFU ex2 and columns 2 and 3 on the
// FMA-pipe polynomial (the same split as softmax_chunk32).  Writes 4 packed
// P words w[4U..4U+3].
template <int U>
__device__ __forceinline__ void softmax_unit(const uint32_t* s, f2 cc, f2 bb, float cs, float bs, uint32_t* w) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const float* v = reinterpret_cast<const float*>(s + 16 * (U & 1) + 4 * g);
    f2 m = fma2(f2{v[0], v[1]}, cc, bb);
    m = f2{ex2(m.x), ex2(m.y)};
    const f2 pp = exp2_poly_sat(f2{fma_sat(v[2], cs, bs), fma_sat(v[3], cs, bs)});
    w[4 * U + g] = e4m3x4(m, pp);
  }
}

// All 32 columns of chunk C (P words w[8C..8C+7]), in groups of 4 keys:
// columns 0 and 1 always on MUFU ex2 (one FFMA2 forms both arguments from an
// adjacent register pair); columns 2 and 3 on the FMA-pipe polynomial in every
// group (FPSA_POLY_PER8 == 4, the default: measured best with the ping-pong
// softmax), in every other group (2: columns 6 and 7 of each 8), or never (0).  oracle.fpsa_oracle._poly_columns mirrors it.
#ifndef FPSA_POLY_PER8
#define FPSA_POLY_PER8 4
#endif
template <int C>
__device__ __forceinline__ void softmax_chunk32(const uint32_t* s, f2 cc, f2 bb, float cs, float bs, uint32_t* w) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float* v = reinterpret_cast<const float*>(s + 4 * q);
    constexpr int kPer8 = FPSA_POLY_PER8;
    f2 m;
    if (kPer8 == 8 || (kPer8 == 6 && (q & 1))) {  // columns 0 and 1 on the polynomial too
      m = exp2_poly_sat(f2{fma_sat(v[0], cs, bs), fma_sat(v[1], cs, bs)});
    } else {
      m = fma2(f2{v[0], v[1]}, cc, bb);
      m = f2{ex2(m.x), ex2(m.y)};
    }
    const bool poly = kPer8 >= 4 || (kPer8 == 2 && (q & 1));
    f2 pp;
    if (poly) {
      pp = exp2_poly_sat(f2{fma_sat(v[2], cs, bs), fma_sat(v[3], cs, bs)});
    } else {
      pp = fma2(f2{v[2], v[3]}, cc, bb);
      pp = f2{ex2(pp.x), ex2(pp.y)};
    }
    w[8 * C + q] = e4m3x4(m, pp);
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
                                              uint32_t* w) {
  if (pad8) mask_pad8(s, 32 * C, ncol);
  if (ncol > 32 * C) softmax_unit<2 * C>(s, cc, bb, cs, bs, w);
  else w[8 * C] = w[8 * C + 1] = w[8 * C + 2] = w[8 * C + 3] = 0u;
  if (ncol > 32 * C + 16) softmax_unit<2 * C + 1>(s, cc, bb, cs, bs, w);
  else w[8 * C + 4] = w[8 * C + 5] = w[8 * C + 6] = w[8 * C + 7] = 0u;
}

// Nonzero iff some packed e4m3 code is 0x7E (448, the saturation value): P~ >= 0
// so codes are <= 0x7E, and adding 2 to each byte sets its top bit only for 0x7E.
template <int NC>
__device__ __forceinline__ uint32_t saturated(const uint32_t* w) {
  uint32_t a = 0u;
#pragma unroll
  for (int i = 0; i < NC / 4; i += 2) a |= (w[i] + 0x02020202u) | (w[i + 1] + 0x02020202u);
  return a & 0x80808080u;
}

// One row part of one key block: NC (64 or 32) S columns from TMEM, ncol
// (multiple of 16, 0..NC) valid, P~ words of absent columns zero.  The row
// sum of P~ is not taken here: the PV MMA accumulates it in the "ones"
// columns of O.  Returns nonzero if some P~ reached the e4m3 saturation value.
template <int NC>
__device__ __forceinline__ uint32_t softmax_block(uint32_t s_addr, int ncol, bool pad8, float c, float boff,
                                                  uint32_t* w) {
  const f2 cc = bcast(c), bb = bcast(boff);
  const float cs = c * (1.0f / 256.0f), bs = (boff + 126.0f) * (1.0f / 256.0f);
  uint32_t sa[32], sb[32];
  if (ncol == NC && !pad8) {
    // common case: all columns valid, no guards around the 32-column chunks
#ifdef FPSA_TRACE
    const long long tl0 = clock64();
#endif
    tmem_ld32(s_addr, sa);
    tmem_wait_ld();
#ifdef FPSA_TRACE
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_trace[4], (unsigned long long)(clock64() - tl0));
#endif
    softmax_chunk32<0>(sa, cc, bb, cs, bs, w);
    if constexpr (NC == 64) {
      tmem_ld32(s_addr + 32, sb);
      tmem_wait_ld();
      softmax_chunk32<1>(sb, cc, bb, cs, bs, w);
    }
  } else {
    if (ncol > 0) {
      tmem_ld32(s_addr, sa);
      tmem_wait_ld();
    }
    if constexpr (NC == 64) {
      if (ncol > 32) tmem_ld32(s_addr + 32, sb);
    }
    softmax_chunk<0>(sa, ncol, pad8, cc, bb, cs, bs, w);
    if constexpr (NC == 64) {
      if (ncol > 32) tmem_wait_ld();
      softmax_chunk<1>(sb, ncol, pad8, cc, bb, cs, bs, w);
    }
  }
  return saturated<NC>(w);
}

// Software-pipelined form: the row part's S is already in registers (s[0..NC)),
// loaded while the previous block's P~ store was in flight.  Same math as
// softmax_block_full.
template <int NC>
__device__ __forceinline__ void load_s_all(uint32_t s_addr, uint32_t* s) {
  tmem_ld32(s_addr, s);
  if constexpr (NC == 64) tmem_ld32(s_addr + 32, s + 32);
}
template <int NC>
__device__ __forceinline__ uint32_t compute_p_regs(const uint32_t* s, int ncol, float c, float boff, uint32_t* w) {
  const f2 cc = bcast(c), bb = bcast(boff);
  const float cs = c * (1.0f / 256.0f), bs = (boff + 126.0f) * (1.0f / 256.0f);
  softmax_chunk32<0>(s, cc, bb, cs, bs, w);
  if constexpr (NC == 64) softmax_chunk32<1>(s + 32, cc, bb, cs, bs, w);
  // Columns >= ncol (the zero padding keys of a tile's last block) are left as computed: their V rows
  // and their rows of the kernel's tail "ones" atom are zero, so they add nothing to O or to l.  (A
  // padding code can only look saturated when the reference max is below -tau, which just triggers a
  // redundant exact-mode redo.)
  (void)ncol;
  return saturated<NC>(w);
}

// softmax_chunk32 with two key tiles in the block (packed key blocks): columns < split take factor a, the
// others factor b.  split is a multiple of 16, so the factor is chosen once per 16-column unit.
template <int C>
__device__ __forceinline__ void softmax_chunk32_split(const uint32_t* s, int split, f2 cca, f2 ccb, float csa,
                                                      float csb, f2 bb, float bs, uint32_t* w) {
  const bool s0 = 32 * C >= split, s1 = 32 * C + 16 >= split;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const bool sb = q < 4 ? s0 : s1;
    const f2 cc = sb ? ccb : cca;
    const float cs = sb ? csb : csa;
    const float* v = reinterpret_cast<const float*>(s + 4 * q);
    constexpr int kPer8 = FPSA_POLY_PER8;
    f2 m;
    if (kPer8 == 8 || (kPer8 == 6 && (q & 1))) {
      m = exp2_poly_sat(f2{fma_sat(v[0], cs, bs), fma_sat(v[1], cs, bs)});
    } else {
      m = fma2(f2{v[0], v[1]}, cc, bb);
      m = f2{ex2(m.x), ex2(m.y)};
    }
    const bool poly = kPer8 >= 4 || (kPer8 == 2 && (q & 1));
    f2 pp;
    if (poly) {
      pp = exp2_poly_sat(f2{fma_sat(v[2], cs, bs), fma_sat(v[3], cs, bs)});
    } else {
      pp = fma2(f2{v[2], v[3]}, cc, bb);
      pp = f2{ex2(pp.x), ex2(pp.y)};
    }
    w[8 * C + q] = e4m3x4(m, pp);
  }
}

// compute_p_regs for a block whose columns < split belong to one key tile (factor ca) and the rest to the
// next (cb); columns >= ncol (padding keys, or past the end of a packed key stream) get P~ = 0.  split and
// ncol are relative to this NC-column part (may be <= 0 or >= NC).
template <int NC>
__device__ __forceinline__ uint32_t compute_p_regs2(const uint32_t* s, int split, int ncol, float ca, float cb,
                                                    float boff, uint32_t* w) {
  const f2 cca = bcast(ca), ccb = bcast(cb), bb = bcast(boff);
  const float csa = ca * (1.0f / 256.0f), csb = cb * (1.0f / 256.0f), bs = (boff + 126.0f) * (1.0f / 256.0f);
  softmax_chunk32_split<0>(s, split, cca, ccb, csa, csb, bb, bs, w);
  if constexpr (NC == 64) softmax_chunk32_split<1>(s + 32, split, cca, ccb, csa, csb, bb, bs, w);
  if (ncol < NC) {
#pragma unroll
    for (int i = 0; i < NC / 4; ++i)
      if (4 * i >= ncol) w[i] = 0u;
  }
  return saturated<NC>(w);
}

// max over the first ncol (<= 128) columns of S * c, c = ca for columns < split and cb above (-inf if none)
template <int NC>
__device__ __forceinline__ float block_max(uint32_t s_addr, int ncol, bool pad8);
__device__ __forceinline__ float block_max_split(uint32_t s_addr, int split, int ncol, float ca, float cb) {
  if (split >= ncol) return block_max<128>(s_addr, ncol, false) * ca;  // one key tile (the common case)
  float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
  for (int base = 0; base < 128; base += 32) {
    if (base < ncol) {
      uint32_t s[32];
      tmem_ld32(s_addr + base, s);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float x = __uint_as_float(s[i]);
        if (base + i < ncol) {
          if (base + i < split) ma = fmaxf(ma, x);
          else mb = fmaxf(mb, x);
        }
      }
    }
  }
  // c > 0: max(S) * c == max(S * c) under round-to-nearest (monotone)
  return fmaxf(ma * ca, mb * cb);
}

// Max of the first ncol (0..NC) raw S values of a row part (-inf if none).
template <int NC>
__device__ __forceinline__ float block_max(uint32_t s_addr, int ncol, bool pad8) {
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int base = 0; base < NC; base += 32) {
    if (base < ncol) {
      uint32_t s[32];
      tmem_ld32(s_addr + base, s);
      tmem_wait_ld();
      if (pad8) mask_pad8(s, base, ncol);
      if (base + 32 > ncol) {  // tail: drop the columns >= ncol (any ncol)
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (base + i >= ncol) s[i] = kNegInf;
      }
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        m0 = max3(m0, __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
        m1 = max3(m1, __uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
      }
    }
  }
  return fmaxf(m0, m1);
}

}  // namespace
}  // namespace fpsa
