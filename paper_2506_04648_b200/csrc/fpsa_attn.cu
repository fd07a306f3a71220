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

constexpr int kThreads = 320;
constexpr int kStages = 4;
constexpr int kBlk = 128;  // rows per query block and keys per key block
constexpr float kLog2_448 = 8.807354922057604f;
// Columns [kPolyFrom, 128) of every key block take the FMA-pipe exp2; the rest MUFU ex2.
constexpr int kPolyFrom = 96;

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

// 2^x for a pair on the FMA pipe (Cody-Waite split + degree-3 minimax, rel. err 7.5e-5),
// used for a fraction of the columns so that the MUFU pipe is not the only exp source.
__device__ __forceinline__ f2 exp2_poly(f2 x) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds x to an integer
  x.x = fmaxf(x.x, -126.0f);  // keeps the exponent add below in range; 2^-126 -> code 0
  x.y = fmaxf(x.y, -126.0f);
  const f2 t = add2(x, bcast(kMagic));
  const f2 j = add2(t, bcast(-kMagic));
  const f2 f = add2(x, f2{-j.x, -j.y});
  f2 y = fma2(bcast(0.055180370807647705f), f, bcast(0.24261191487312317f));
  y = fma2(y, f, bcast(0.6932594180107117f));
  y = fma2(y, f, bcast(0.9999279975891113f));
  // scale by 2^j: add j to the exponent field (t's low mantissa bits hold j)
  return f2{__uint_as_float(__float_as_uint(y.x) + (__float_as_uint(t.x) << 23)),
            __uint_as_float(__float_as_uint(y.y) + (__float_as_uint(t.y) << 23))};
}

__device__ __forceinline__ uint32_t e4m3x2(float hi, float lo) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

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
      mbar_init(&bar_p_ready[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 8) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  if (warp == 9) {
    for (int i = lane; i < D; i += 32) s_vscale[i] = (float)p.v_scales[(int64_t)h * D + i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tm_s[2] = {tmem, tmem + 128};
  const uint32_t tm_o[2] = {tmem + 256, tmem + 256 + D};

  if (warp == 8) {
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
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_f8(128, 128, FMT, FMT, 0);
      constexpr uint32_t idesc_pv = idesc_f8(128, D, FPSA_E4M3, FMT, 1);
      const uint32_t sq = smem_u32(smem + S::kQ);
      mbar_wait(&bar_q, 0);
      tc_fence_after();
      for (int32_t j = 0; j <= n_kv; ++j) {
        const int st = j % kStages;
        if (j < n_kv) {
          mbar_wait(&bar_kv_full[st], (j / kStages) & 1);
          tc_fence_after();
        }
        const int pst = (j + kStages - 1) % kStages;  // stage of block j-1
        const uint32_t sk = smem_u32(smem + S::kK + st * S::kTile);
        const uint32_t sv_prev = smem_u32(smem + S::kV + pst * S::kTile);
        for (int q = 0; q < nqb; ++q) {
          if (j > 0) {
            mbar_wait(&bar_p_ready[q], (j - 1) & 1);
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
    }
  } else if (warp / 4 < nqb) {
    // ------------------------------------------------------------ softmax (one row per thread)
    const int q = warp / 4;
    const int row = threadIdx.x & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float cq = (float)p.q_scales[h * p.M + u] * p.scale_log2;
    const float tau = p.tau;
    float m_ref = -INFINITY, l = 0.0f;
    for (int32_t j = 0; j < n_kv; ++j) {
      const int32_t kt = j / p.nb, b = j - kt * p.nb;
      const int32_t v = __ldg(p.ids + kt0 + kt);
      const float c = cq * (float)__ldg(p.k_scales + h * p.M + v);
      const int valid = min(kBlk, p.tv - b * kBlk);
      mbar_wait(&bar_s_full[q], j & 1);
      tc_fence_after();
      float s[kBlk];
      tmem_ld32(tm_s[q] + lane_off + 0, reinterpret_cast<uint32_t*>(s + 0));
      tmem_ld32(tm_s[q] + lane_off + 32, reinterpret_cast<uint32_t*>(s + 32));
      tmem_ld32(tm_s[q] + lane_off + 64, reinterpret_cast<uint32_t*>(s + 64));
      tmem_ld32(tm_s[q] + lane_off + 96, reinterpret_cast<uint32_t*>(s + 96));
      tmem_wait_ld();
      // Key columns >= valid are padding (zero K/V rows of a key tile's last
      // block): set to -inf so they drop out of the max, the sum and P
      // (valid is a multiple of 8, checked on the host).
      if (valid < kBlk) {
#pragma unroll
        for (int i = 0; i < kBlk; i += 8) {
          const bool ok = i < valid;
#pragma unroll
          for (int k = i; k < i + 8; ++k) s[k] = ok ? s[k] : -INFINITY;
        }
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int i = 0; i < kBlk; i += 4) {
        mx0 = max3(mx0, s[i], s[i + 1]);
        mx1 = max3(mx1, s[i + 2], s[i + 3]);
      }
      const float mb = fmaxf(mx0, mx1) * c;
      if (j == 0) {
        m_ref = mb;
      } else if (__any_sync(0xffffffffu, mb > m_ref + tau)) {
        const float m_new = fmaxf(m_ref, mb);
        const float alpha = ex2(m_ref - m_new);
        l *= alpha;
        m_ref = m_new;
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 16) {
          uint32_t o[16];
          tmem_ld16(tm_o[q] + lane_off + cc, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16(tm_o[q] + lane_off + cc, o);
        }
        tmem_wait_st();
      }
      const f2 cc2 = bcast(c), noff = bcast(kLog2_448 - m_ref - tau);
      f2 lsum0 = bcast(0.0f), lsum1 = bcast(0.0f);
#pragma unroll
      for (int i0 = 0; i0 < kBlk; i0 += 32) {
        uint32_t w[8];
#pragma unroll
        for (int k = i0; k < i0 + 32; k += 4) {
          f2 pa = fma2(f2{s[k], s[k + 1]}, cc2, noff);
          f2 pb = fma2(f2{s[k + 2], s[k + 3]}, cc2, noff);
          if (k >= kPolyFrom) {
            pa = exp2_poly(pa);
            pb = exp2_poly(pb);
          } else {
            pa = f2{ex2(pa.x), ex2(pa.y)};
            pb = f2{ex2(pb.x), ex2(pb.y)};
          }
          lsum0 = add2(lsum0, pa);
          lsum1 = add2(lsum1, pb);
          w[(k - i0) / 4] = e4m3x2(pa.y, pa.x) | (e4m3x2(pb.y, pb.x) << 16);
        }
        tmem_st8(tm_s[q] + lane_off + i0 / 4, w);
      }
      const f2 lsum = add2(lsum0, lsum1);
      l += lsum.x + lsum.y;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar_p_ready[q]);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(&bar_o, 0);
    tc_fence_after();
    const int32_t r = (qb0 + q) * kBlk + row;  // row inside the tile
    const float inv_l = 1.0f / l;
    int64_t token;
    if (p.natural) {
      const int32_t ut = u / (p.dh * p.dw), uh = (u / p.dw) % p.dh, uw = u % p.dw;
      const int32_t lt = r / (p.sh * p.sw), lh = (r / p.sw) % p.sh, lw = r % p.sw;
      token = ((int64_t)(ut * p.st + lt) * p.gh + (uh * p.sh + lh)) * p.gw + (uw * p.sw + lw);
    } else {
      token = (int64_t)u * p.tv + r;
    }
    const float* vs = s_vscale;
#pragma unroll
    for (int cc = 0; cc < D; cc += 32) {
      uint32_t o[32];
      tmem_ld32(tm_o[q] + lane_off + cc, o);
      tmem_wait_ld();
      if (r < p.tv) {
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(o[i]) * inv_l * vs[cc + i];
        if constexpr (OUT == FPSA_F32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + token * p.out_ts + h * p.out_hs + cc);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + token * p.out_ts + h * p.out_hs + cc);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint32_t wv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              __nv_bfloat162 b2 = __floats2bfloat162_rn(f[8 * i + 2 * k], f[8 * i + 2 * k + 1]);
              wv[k] = *reinterpret_cast<uint32_t*>(&b2);
            }
            dst[i] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 512);
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
