// Passthrough path: full-precision sliding-tile sparse attention on bf16
// operands, sm_100a (tcgen05 kind::f16 + TMEM + TMA).
//
// Replaces the reference's passthrough branch of fp8_sparse_forward and its
// sparse_reference (/root/reference/pkg/src/fp8sta/attention.py:152-154,
// :165-176, :192-194): _engine with unit factors and no P rounding, i.e. f32
// softmax attention restricted to the window's key tiles.  On the GPU the
// operands are bf16 (exact for bf16 inputs, RNE-rounded from f32 inputs) and
// P is held in TMEM as bf16 for the PV MMA; accumulation is f32 throughout.
//
// Two kernels:
//   tile_gather_bf16   [tokens, heads, d] (natural or tile order, f32/bf16)
//                      -> tile-major padded bf16 [heads][M][pitch][d], pad rows 0
//   attn_bf16_kernel   persistent, same work list / CSR / warp roles as the FP8
//                      kernel (fpsa_attn.cu):
//     S(j)  = Q K_j^T                       kind::f16 M128 N128, 8 x K16, SS
//     P     = 2^(S * scale log2 e - m)      m = row max of the first key block
//     l    += sum P                         CUDA cores (f32, unrounded P)
//     O    += bf16(P) V_j                   kind::f16 M128 N=D, A = P from TMEM,
//                                           B = V MN-major ([keys][d] as stored)
//   out = O / l.  P is never saturated (bf16 has the f32 exponent range); a
//   row whose sum overflowed (a logit > 127 above m, in log2 units) sends its
//   item to the same exact-max redo launch the FP8 kernel uses.
//
// Shared memory (d = 128): Q 32 KB, K ring 2 x 32 KB (a K stage is released as
// soon as its QK completes), V ring 3 x 32 KB = 192 KB.  bf16 rows of d = 128
// are 256 B, so each tile is stored as two 128-byte-wide SWIZZLE_128B slabs
// (d 0-63, d 64-127), loaded by one 3D TMA box.
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
#include "softmax.cuh"

namespace fpsa {
namespace {

using namespace sm100;

namespace pt {
constexpr int kBlk = 128;
constexpr int kParts = 2, kPartCols = 64;
constexpr int kSoftmaxWarps = 8, kTmaWarp = 8, kMmaWarp = 9;
constexpr int kThreads = 12 * 32;
constexpr uint32_t kRegsSoftmax = 216, kRegsProducer = 64;
constexpr int kKStages = 2, kVStages = 3;
constexpr int kRedoHeader = 4;  // same workspace layout as fpsa_attn_fwd

struct Params {
  const int32_t* offs;
  const int32_t* ids;
  const int32_t* items;
  int32_t n_items;
  int32_t* redo;
  int32_t exact;
  int32_t M, tv, pitch, nb, n_tail;  // n_tail: valid keys of a tile's last block
  float softmax_log2;
  void* out;
  int64_t out_ts, out_hs;
  int32_t natural;
  int32_t gh, gw, st, sh, sw, dh, dw;
};

template <int D>
struct Smem {
  static constexpr int kSlab = kBlk * 128;       // 128 rows x 64 bf16
  static constexpr int kTile = kSlab * (D / 64);  // one 128-row block
  static constexpr int kQ = 0;
  static constexpr int kK = kTile;
  static constexpr int kV = kK + kKStages * kTile;
  static constexpr int kBytes = kV + kVStages * kTile;
};

__device__ __forceinline__ void mma_bf16_ss_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_w(void* smem_dst, const void* tmap, int32_t c0, int32_t c1, int32_t c2,
                                              uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n\t}" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// kind::f16 instruction descriptor: bf16 A and B, f32 accumulate (same field layout as idesc_f8).
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t b_mn_major) { return idesc_f8(M, N, 1, 1, b_mn_major); }

// One 64-key row part: P = 2^(s c - m) for ncol valid columns,
// packed bf16 pairs into w[32]; returns the f32 sum of the (unrounded) P.
__device__ __forceinline__ float softmax_part_bf16(uint32_t* s, int ncol, float c, float neg_m, uint32_t* w) {
  if (ncol < kPartCols) {  // tail block: columns >= ncol (any ncol) drop out of P and of the sum
#pragma unroll
    for (int k = 0; k < kPartCols; ++k)
      if (k >= ncol) s[k] = kNegInf;
  }
  const f2 cc = bcast(c), bb = bcast(neg_m);
  f2 acc[4] = {bcast(0.0f), bcast(0.0f), bcast(0.0f), bcast(0.0f)};
#pragma unroll
  for (int i = 0; i < kPartCols / 2; ++i) {
    f2 x = fma2(f2{__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])}, cc, bb);
    x = f2{ex2(x.x), ex2(x.y)};
    acc[i & 3] = add2(acc[i & 3], x);
    w[i] = bf16x2(x.x, x.y);
  }
  const f2 a = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
  return a.x + a.y;
}

template <int D, int OUT>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bf16_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using S = Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_qfree, bar_o, bar_ofree;
  __shared__ uint64_t bar_k_full[kKStages], bar_k_empty[kKStages], bar_v_full[kVStages], bar_v_empty[kVStages];
  __shared__ uint64_t bar_s_full[2], bar_p_ready[2];
  __shared__ uint32_t s_tmem;
  __shared__ float s_xchg[kParts][kBlk];
  __shared__ uint32_t s_ovf;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* items = p.exact ? p.redo + kRedoHeader : p.items;
  const int32_t count = p.exact ? *reinterpret_cast<volatile int32_t*>(p.redo) : p.n_items;
  if ((int32_t)blockIdx.x >= count) return;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    mbar_init(&bar_qfree, 1);
    mbar_init(&bar_o, 1);
    mbar_init(&bar_ofree, kSoftmaxWarps);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_s_full[i], 1);
      mbar_init(&bar_p_ready[i], kSoftmaxWarps);
    }
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&bar_k_full[i], 1);
      mbar_init(&bar_k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&bar_v_full[i], 1);
      mbar_init(&bar_v_empty[i], 1);
    }
    s_ovf = 0;
    fence_barrier_init();
  }
  if (warp == kTmaWarp) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tm_o = tmem;  // O: columns 0..D-1
  auto tm_s = [tmem](uint32_t g) { return tmem + 256u + 128u * (g & 1u); };

  if (warp >= kSoftmaxWarps) regs_dec<kRegsProducer>();
  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
    }
    __syncwarp();
    uint32_t gk = 0, gv = 0;  // K / V block counters over all items of this CTA
    int32_t iter = 0;
    for (int32_t it = blockIdx.x; it < count; it += gridDim.x, ++iter) {
      const int32_t h = items[3 * it], u = items[3 * it + 1], qb = items[3 * it + 2];
      const int32_t kt0 = __ldg(p.offs + u), n_kt = __ldg(p.offs + u + 1) - kt0;
      const int32_t n_kv = n_kt * p.nb, steps = p.exact ? 2 * n_kv : n_kv;
      const int32_t pv0 = p.exact ? n_kv : 0;
      if (iter >= 1) mbar_wait(&bar_qfree, (iter - 1) & 1);
      mbar_arrive_expect_tx_w(&bar_q, S::kTile);
      tma_load_3d_w(smem + S::kQ, &tm_q, 0, (h * p.M + u) * p.pitch + qb * kBlk, 0, &bar_q);
      int32_t kt = 0, b = 0;
      int32_t krow = (h * p.M + __ldg(p.ids + kt0)) * p.pitch;
      for (int32_t s = 0; s < steps; ++s) {
        {
          const uint32_t st = gk % kKStages;
          if (gk >= (uint32_t)kKStages) mbar_wait(&bar_k_empty[st], ((gk / kKStages) - 1) & 1);
          mbar_arrive_expect_tx_w(&bar_k_full[st], S::kTile);
          tma_load_3d_w(smem + S::kK + st * S::kTile, &tm_k, 0, krow + b * kBlk, 0, &bar_k_full[st]);
          ++gk;
        }
        if (s >= pv0) {  // exact mode: the max pass needs no V
          const uint32_t st = gv % kVStages;
          if (gv >= (uint32_t)kVStages) mbar_wait(&bar_v_empty[st], ((gv / kVStages) - 1) & 1);
          mbar_arrive_expect_tx_w(&bar_v_full[st], S::kTile);
          tma_load_3d_w(smem + S::kV + st * S::kTile, &tm_v, 0, krow + b * kBlk, 0, &bar_v_full[st]);
          ++gv;
        }
        if (++b == p.nb) {
          b = 0;
          if (++kt == n_kt) kt = 0;
          krow = (h * p.M + __ldg(p.ids + kt0 + kt)) * p.pitch;
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_qk = idesc_bf16(128, 128, 0);
    constexpr uint32_t idesc_pv = idesc_bf16(128, D, 1);
    constexpr uint64_t kTileU = S::kTile >> 4, kSlabU = S::kSlab >> 4;
    const uint64_t dq = smem_desc_sw128(smem_u32(smem + S::kQ), 16, 1024);
    const uint64_t dk0 = smem_desc_sw128(smem_u32(smem + S::kK), 16, 1024);
    const uint64_t dv0 = smem_desc_sw128(smem_u32(smem + S::kV), S::kSlab, 1024);  // MN atoms = slabs
    uint32_t g = 0, gk = 0, gv = 0;
    int32_t iter = 0;
    for (int32_t it = blockIdx.x; it < count; it += gridDim.x, ++iter) {
      const int32_t u = items[3 * it + 1];
      const int32_t n_kt = __ldg(p.offs + u + 1) - __ldg(p.offs + u);
      const int32_t n_kv = n_kt * p.nb, steps = p.exact ? 2 * n_kv : n_kv;
      const int32_t pv0 = p.exact ? n_kv : 0;
      mbar_wait(&bar_q, iter & 1);
      tc_fence_after();
      auto issue_qk = [&](uint32_t gg) {
        const uint32_t st = gk % kKStages;
        mbar_wait(&bar_k_full[st], (gk / kKStages) & 1);
        tc_fence_after();
        const uint64_t dk = dk0 + st * kTileU;
        const uint32_t ts = tm_s(gg);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {  // K16 steps: 32 B within a slab, then the next slab
          const uint64_t off = (uint64_t)(k / 4) * kSlabU + 2 * (k % 4);
          mma_bf16_ss_w(ts, dq + off, dk + off, idesc_qk, k > 0 ? 1u : 0u);
        }
        mma_commit_w(&bar_k_empty[st]);
        mma_commit_w(&bar_s_full[gg & 1]);
        ++gk;
      };
      for (int32_t s = 0; s < min(steps, 2); ++s) issue_qk(g + s);
      if (steps <= 2) mma_commit_w(&bar_qfree);
      for (int32_t s = 0; s < steps; ++s) {
        const uint32_t gs = g + s;
        mbar_wait(&bar_p_ready[gs & 1], (gs >> 1) & 1);
        tc_fence_after();
        if (s >= pv0) {
          if (s == pv0 && iter > 0) {
            mbar_wait(&bar_ofree, (iter - 1) & 1);
            tc_fence_after();
          }
          const uint32_t st = gv % kVStages;
          mbar_wait(&bar_v_full[st], (gv / kVStages) & 1);
          tc_fence_after();
          const uint64_t dv = dv0 + st * kTileU;
          const uint32_t ts = tm_s(gs);
#pragma unroll
          for (int k = 0; k < kBlk / 16; ++k)  // keys 16k..16k+15: P columns of part k/4, 16 keys x 128 B of V
            mma_bf16_ts_w(tm_o, ts + kPartCols * (k / 4) + 8 * (k % 4), dv + (uint64_t)k * (16 * 128 / 16),
                          idesc_pv, (s > pv0 || k > 0) ? 1u : 0u);
          mma_commit_w(&bar_v_empty[st]);
          ++gv;
        }
        if (s + 2 < steps) {
          issue_qk(gs + 2);
          if (s + 3 == steps) mma_commit_w(&bar_qfree);
        }
      }
      mma_commit_w(&bar_o);
      g += steps;
    }
  } else if (warp < kSoftmaxWarps) {
    regs_inc<kRegsSoftmax>();
    // ------------------------------------------------------------ softmax: (row, column part)
    const int quarter = warp & 3, part = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float c = p.softmax_log2;
    auto row_sync = [&]() { named_bar_sync(1 + quarter, 32 * kParts); };
    auto row_combine = [&](float v, bool is_max) {
      s_xchg[part][row] = v;
      row_sync();
      const float a = s_xchg[0][row], b = s_xchg[1][row];
      row_sync();
      return is_max ? fmaxf(a, b) : a + b;
    };
    auto ncol_of = [&](int32_t bb) {
      return min(max((bb == p.nb - 1 ? p.n_tail : kBlk) - kPartCols * part, 0), kPartCols);
    };
    uint32_t g = 0;
    int32_t iter = 0;
    for (int32_t it = blockIdx.x; it < count; it += gridDim.x, ++iter) {
      const int32_t h = items[3 * it], u = items[3 * it + 1], qb = items[3 * it + 2];
      const int32_t n_kt = __ldg(p.offs + u + 1) - __ldg(p.offs + u);
      const int32_t n_kv = n_kt * p.nb;
      float m_ref = 0.0f;
      if (p.exact) {
        float m_acc = -INFINITY;
        int32_t b = 0;
        for (int32_t j = 0; j < n_kv; ++j, ++g) {
          mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
          tc_fence_after();
          m_acc = fmaxf(m_acc, block_max<kPartCols>(tm_s(g) + lane_off + part * kPartCols, ncol_of(b), false));
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_p_ready[g & 1]);
          if (++b == p.nb) b = 0;
        }
        m_ref = row_combine(m_acc, true) * c;
      }
      float l = 0.0f;
      {
        int32_t b = 0;
        uint32_t sreg[kPartCols];
        mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        if (!p.exact)
          m_ref = row_combine(block_max<kPartCols>(tm_s(g) + lane_off + part * kPartCols, ncol_of(0), false), true) * c;
        load_s_all<kPartCols>(tm_s(g) + lane_off + part * kPartCols, sreg);
        tmem_wait_ld();
        for (int32_t j = 0; j < n_kv; ++j, ++g) {
          uint32_t w[kPartCols / 2];
          l += softmax_part_bf16(sreg, ncol_of(b), c, -m_ref, w);
          tmem_st32(tm_s(g) + lane_off + part * kPartCols, w);
          if (++b == p.nb) b = 0;
          const bool more = j + 1 < n_kv;
          if (more) {
            mbar_wait(&bar_s_full[(g + 1) & 1], ((g + 1) >> 1) & 1);
            tc_fence_after();
            load_s_all<kPartCols>(tm_s(g + 1) + lane_off + part * kPartCols, sreg);
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_p_ready[g & 1]);
          if (more) tmem_wait_ld();
        }
      }
      // ---------------------------------------------------------- epilogue
      l = row_combine(l, false);
      const bool ovf = !(l < INFINITY);  // inf or nan: some logit beyond the f32 range above m
      mbar_wait(&bar_o, iter & 1);
      tc_fence_after();
      const float inv_l = 1.0f / l;
      const int32_t r = qb * kBlk + row;
      int64_t token;
      if (p.natural) {
        const int32_t ut = u / (p.dh * p.dw), uh = (u / p.dw) % p.dh, uw = u % p.dw;
        const int32_t lt = r / (p.sh * p.sw), lh = (r / p.sw) % p.sh, lw = r % p.sw;
        token = ((int64_t)(ut * p.st + lt) * p.gh + (uh * p.sh + lh)) * p.gw + (uw * p.sw + lw);
      } else {
        token = (int64_t)u * p.tv + r;
      }
#pragma unroll
      for (int cc = 0; cc < D / kParts; cc += 32) {
        const int col = part * (D / kParts) + cc;
        uint32_t o[32];
        tmem_ld32(tm_o + lane_off + col, o);
        tmem_wait_ld();
        if (r < p.tv) {
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(o[i]) * inv_l;
          if constexpr (OUT == FPSA_F32) {
            float4* dst =
                reinterpret_cast<float4*>(static_cast<float*>(p.out) + token * p.out_ts + h * p.out_hs + col);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + token * p.out_ts +
                                                  h * p.out_hs + col);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(bf16x2(f[8 * i], f[8 * i + 1]), bf16x2(f[8 * i + 2], f[8 * i + 3]),
                                  bf16x2(f[8 * i + 4], f[8 * i + 5]), bf16x2(f[8 * i + 6], f[8 * i + 7]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_ofree);
      if (!p.exact) {
        if (__any_sync(0xffffffffu, ovf && r < p.tv) && lane == 0) atomicOr(&s_ovf, 1u);
        named_bar_sync(5, kSoftmaxWarps * 32);
        if (threadIdx.x == 0 && s_ovf) {
          s_ovf = 0;
          const int32_t slot = atomicAdd(p.redo, 1);
          p.redo[kRedoHeader + 3 * slot] = h;
          p.redo[kRedoHeader + 3 * slot + 1] = u;
          p.redo[kRedoHeader + 3 * slot + 2] = qb;
        }
        named_bar_sync(5, kSoftmaxWarps * 32);  // s_ovf is reused by the next item
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kTmaWarp) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- gather
// 16 B (8 bf16 channels) per thread, d/8 threads per padded tile-major row
// (h, u, r): r < tv copied from its source token, r >= tv zero.  32-bit index
// math (rows < 2^31), one row per d/8 lanes, coalesced 16 B stores.
template <typename T>
__global__ void __launch_bounds__(256) tile_gather_bf16(const T* __restrict__ x, int64_t ts, int64_t hs, int32_t M,
                                                        int32_t pitch, int32_t tv, int32_t d, int32_t n_rows,
                                                        int32_t natural, int32_t gh, int32_t gw, int32_t st,
                                                        int32_t sh, int32_t sw, int32_t dh, int32_t dw,
                                                        __nv_bfloat16* __restrict__ out) {
  const int32_t per_row = d / 8;
  const int32_t rows_per_block = blockDim.x / per_row;
  const int32_t c8 = threadIdx.x % per_row;
  for (int32_t row = blockIdx.x * rows_per_block + threadIdx.x / per_row; row < n_rows;
       row += gridDim.x * rows_per_block) {
    const int32_t r = row % pitch, hu = row / pitch;
    const int32_t u = hu % M, h = hu / M;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (r < tv) {
      int32_t token;
      if (natural) {
        const int32_t ut = u / (dh * dw), uh = (u / dw) % dh, uw = u % dw;
        const int32_t lt = r / (sh * sw), lh = (r / sw) % sh, lw = r % sw;
        token = ((ut * st + lt) * gh + (uh * sh + lh)) * gw + (uw * sw + lw);
      } else {
        token = u * tv + r;
      }
      const T* src = x + (int64_t)token * ts + (int64_t)h * hs + 8 * c8;
      if constexpr (sizeof(T) == 4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(src));
        const float4 b = __ldg(reinterpret_cast<const float4*>(src) + 1);
        v = make_uint4(bf16x2(a.x, a.y), bf16x2(a.z, a.w), bf16x2(b.x, b.y), bf16x2(b.z, b.w));
      } else {
        v = __ldg(reinterpret_cast<const uint4*>(src));
      }
    }
    reinterpret_cast<uint4*>(out)[(int64_t)row * per_row + c8] = v;
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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

// [rows][d] bf16 seen as (64 channels, rows, d/64 slabs): one box = 128 rows x d,
// landing in shared memory as d/64 consecutive 16 KB SWIZZLE_128B slabs.
int make_bf16_map(CUtensorMap* m, const void* base, int64_t rows, int32_t d) {
  auto fn = encoder();
  if (!fn) return fail(FPSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(d / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)kBlk, (cuuint32_t)(d / 64)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FPSA_ECUDA, "cuTensorMapEncodeTiled (bf16) failed: " + std::to_string((int)r));
  return FPSA_OK;
}


template <int D, int OUT>
int launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, Params p, cudaStream_t st) {
  auto kern = attn_bf16_kernel<D, OUT>;
  constexpr int smem = Smem<D>::kBytes + 1024;
  if (int s = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem, "fpsa_attn_bf16_fwd")) return s;
  if (cudaMemsetAsync(p.redo, 0, sizeof(int32_t), st) != cudaSuccess)
    return fail(FPSA_ECUDA, std::string("fpsa_attn_bf16_fwd redo reset: ") + cudaGetErrorString(cudaGetLastError()));
  const int grid = std::min(p.n_items, device_sm_count());
  p.exact = 0;
  kern<<<grid, kThreads, smem, st>>>(tq, tk, tv, p);
  p.exact = 1;
  kern<<<grid, kThreads, smem, st>>>(tq, tk, tv, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FPSA_ECUDA, std::string("fpsa_attn_bf16_fwd launch: ") + cudaGetErrorString(e));
  return FPSA_OK;
}

}  // namespace pt
}  // namespace
}  // namespace fpsa

using namespace fpsa;

extern "C" int fpsa_tile_gather_bf16(const void* x, int dtype, int64_t token_stride, int64_t head_stride,
                                     int32_t heads, fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch,
                                     int in_order, void* out, void* stream) {
  clear_error();
  fpsa_dims3 td;
  if (int s = fpsa_tile_grid(grid, tile, &td)) return s;
  if (!x || !out) return fail(FPSA_EINVAL, "null buffer");
  if (d % 64) return fail(FPSA_EUNSUPPORTED, "head dim must be a multiple of 64, got " + std::to_string(d));
  if (token_stride % 8 || head_stride % 8 || reinterpret_cast<uintptr_t>(x) % 16)
    return fail(FPSA_EINVAL, "input strides must be multiples of 8 elements and the base 16-byte aligned");
  const int32_t tv = tile.t * tile.h * tile.w;
  if (tile_pitch < tv || tile_pitch % pt::kBlk) return fail(FPSA_EINVAL, "tile_pitch must be a multiple of 128 >= tile volume");
  if (heads < 1) return fail(FPSA_EINVAL, "heads must be >= 1");
  if (dtype != FPSA_F32 && dtype != FPSA_BF16) return fail(FPSA_EUNSUPPORTED, "input dtype must be f32 or bf16");
  const int32_t M = td.t * td.h * td.w;
  const int64_t rows = (int64_t)heads * M * tile_pitch;
  if (rows >= (int64_t)1 << 31) return fail(FPSA_EUNSUPPORTED, "too many rows for one gather");
  const int32_t rows_per_block = 256 / (d / 8);
  const int blocks = (int)std::min<int64_t>((rows + rows_per_block - 1) / rows_per_block, (int64_t)device_sm_count() * 16);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nat = in_order == FPSA_ORDER_NATURAL;
  auto* o = static_cast<__nv_bfloat16*>(out);
  if (dtype == FPSA_F32)
    pt::tile_gather_bf16<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(x), token_stride, head_stride, M,
                                                        tile_pitch, tv, d, (int32_t)rows, nat, grid.h, grid.w, tile.t,
                                                        tile.h, tile.w, td.h, td.w, o);
  else
    pt::tile_gather_bf16<__nv_bfloat16><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), token_stride,
                                                                head_stride, M, tile_pitch, tv, d, (int32_t)rows, nat,
                                                                grid.h, grid.w, tile.t, tile.h, tile.w, td.h, td.w, o);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FPSA_ECUDA, std::string("fpsa_tile_gather_bf16 launch: ") + cudaGetErrorString(e));
  return FPSA_OK;
}

extern "C" int fpsa_attn_bf16_fwd(const void* q_tiles, const void* k_tiles, const void* v_tiles, int32_t heads,
                                  fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, const int32_t* offs,
                                  const int32_t* ids, const int32_t* items, int32_t n_items, float softmax_scale,
                                  void* out, int out_dtype, int64_t out_token_stride, int64_t out_head_stride,
                                  int out_order, void* workspace, int64_t workspace_bytes, void* stream) {
  clear_error();
  fpsa_dims3 td;
  if (int s = fpsa_tile_grid(grid, tile, &td)) return s;
  if (!q_tiles || !k_tiles || !v_tiles || !offs || !ids || !items || !out) return fail(FPSA_EINVAL, "null buffer");
  if (d != 64 && d != 128) return fail(FPSA_EUNSUPPORTED, "head dim must be 64 or 128, got " + std::to_string(d));
  const int32_t tv = tile.t * tile.h * tile.w;
  if (tile_pitch < tv || tile_pitch % pt::kBlk) return fail(FPSA_EINVAL, "tile_pitch must be a multiple of 128 >= tile volume");
  if (!(softmax_scale > 0.0f)) return fail(FPSA_EINVAL, "softmax_scale must be > 0");
  if (out_dtype != FPSA_F32 && out_dtype != FPSA_BF16) return fail(FPSA_EUNSUPPORTED, "out dtype must be f32 or bf16");
  if (heads < 1 || n_items < 1) return fail(FPSA_EINVAL, "empty problem");
  int64_t need = 0;
  fpsa_attn_workspace_bytes(n_items, &need);
  if (!workspace || workspace_bytes < need)
    return fail(FPSA_ECAPACITY, "attention workspace must hold " + std::to_string(need) + " bytes");
  const int32_t M = td.t * td.h * td.w;
  const int64_t rows = (int64_t)heads * M * tile_pitch;
  CUtensorMap tq, tk, tvm;
  if (int s = pt::make_bf16_map(&tq, q_tiles, rows, d)) return s;
  if (int s = pt::make_bf16_map(&tk, k_tiles, rows, d)) return s;
  if (int s = pt::make_bf16_map(&tvm, v_tiles, rows, d)) return s;
  pt::Params p{};
  p.offs = offs;
  p.ids = ids;
  p.items = items;
  p.n_items = n_items;
  p.redo = static_cast<int32_t*>(workspace);
  p.M = M;
  p.tv = tv;
  p.pitch = tile_pitch;
  p.nb = (tv + pt::kBlk - 1) / pt::kBlk;
  p.n_tail = tv - pt::kBlk * (p.nb - 1);
  p.softmax_log2 = softmax_scale * 1.4426950408889634f;
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
  if (d == 128) {
    if (out_dtype == FPSA_F32) return pt::launch<128, FPSA_F32>(tq, tk, tvm, p, st);
    return pt::launch<128, FPSA_BF16>(tq, tk, tvm, p, st);
  }
  if (out_dtype == FPSA_F32) return pt::launch<64, FPSA_F32>(tq, tk, tvm, p, st);
  return pt::launch<64, FPSA_BF16>(tq, tk, tvm, p, st);
}
