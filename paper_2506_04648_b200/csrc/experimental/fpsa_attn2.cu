// EXPERIMENTAL, not part of the default build (DESIGN.md §6 item 1).
//
// K4, 2-CTA form: the two 128-row query blocks of a tile run as a CTA pair
// (cluster of 2) whose MMAs are tcgen05 cta_group::2 (M = 256), which the
// probe tools/probes/mma2_rate.cu measures at the full per-SM tensor rate.
// Per key block j, in each CTA of the pair (rows = its query block):
//   S(j)  = Q K_j^T     M256 N128, K half (64 keys) in each CTA's smem
//   P~    = e4m3(448 2^-tau 2^(x - m))
//   [O|l] += P~ [V_j|1] M256 N160, A = P~ from each CTA's TMEM; each CTA's B half is [64 V channels | 16
//                       ones] (SWIZZLE_64B MN-major, the ones tile reached through the descriptor's LBO as in
//                       the single-CTA kernel, a zero-row tail variant for a tile's last block), so O columns
//                       0-63 / 80-143 hold the channels and 64-79 / 144-159 the row sum of the rounded P~
// The leader CTA issues all MMAs; the peer's relay warp forwards its TMA completions, its softmax warps
// arrive remotely on the leader's p_ready / ofree barriers; commits multicast to both CTAs.
// -DA2_PBUF: P~ in its own TMEM columns (160..223) and an s_free barrier, so QK(j+2) is issued as soon as
// the owners hold S(j) in registers instead of after PV(j).
//
// Status (round 1): passes tests/test_gpu_attention.py (28 cases incl. E5M2, odd tile volumes, exact
// mode). C2 attention, same box, interleaved (profiles/r01_ab_a2_r3x.txt): single-CTA 11.7 ms, this
// kernel 12.4-12.6 ms (14.2 before the ones split), -DA2_PBUF 12.8 ms.
// What the measurements say (profiles/r01_probe_mma2_rate.txt, r01_trace_a2_n160.txt, r01_trace_a2_pbuf.txt):
// the pair's QK + PV step takes 576 clk back to back and 974 clk issue-to-completion in isolation, and
// neither concurrent tcgen05.ld traffic nor FMA/MUFU-saturated warps on the same SM change that by more
// than 5 %; in the kernel one MMA-warp iteration takes ~1450 clk, ~650 of them between p_ready and the last
// PV issue. ncu's source counters for the single-CTA kernel point the same way (tools/mma_warp_share.py):
// the MMA warp spends about half of the launch executing its ~140-instruction step body (descriptor
// arithmetic, R2UR moves, elect / divergence checks, barrier address math) at a few cycles per dependent
// instruction ('wait', 'selected', 'not_selected' against the softmax warps) and ~20 % waiting for p_ready. Halving the MMA
// work per SM therefore does not shorten the step; the issue path does. Tried without gain: in-asm
// descriptor steps (ptxas adds SELs), issuing from one lane (ptxas wraps each MMA in an elect loop), more
// producer registers (same SASS).  Build and A/B:
//   cd paper_2506_04648_b200 && nvcc -shared -Xcompiler -fPIC -std=c++17 -O3 -lineinfo \
//     -gencode arch=compute_100a,code=sm_100a -DFPSA_ATTN2 csrc/fpsa_attn.cu csrc/experimental/fpsa_attn2.cu \
//     csrc/fpsa_attn_bf16.cu csrc/fpsa_quant.cu csrc/fpsa_metrics.cu csrc/fpsa_io.cu csrc/fpsa_host.cpp \
//     -o libfpsa_a2.so
//   FPSA_LIB=libfpsa_a2.so python bench.py   (FPSA_ATTN_1CTA=1 falls back to the single-CTA kernel)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../../../include/fpsa.h"
#include "../fpsa_internal.h"
#include "../sm100.cuh"
#include "../softmax.cuh"

namespace fpsa {
namespace {

using namespace sm100;

namespace a2 {
#ifdef A2_TRACE
__device__ long long g_a2[3][128][4];  // [leader MMA, leader softmax warp 0, peer softmax warp 0][step][event]
#define A2_TL(who, step, ev)                                                            \
  do {                                                                                  \
    if ((blockIdx.x >> 1) == 0 && (threadIdx.x & 31) == 0 && (step) < 128) g_a2[who][step][ev] = clock64(); \
  } while (0)
#else
#define A2_TL(who, step, ev) \
  do {                       \
  } while (0)
#endif
constexpr int D = 128;
constexpr int kSoftmaxWarps = 8;
constexpr int kTmaWarp = 8, kMmaWarp = 9, kHelperWarp = 10, kRelayWarp = 11;
constexpr int kThreads = 12 * 32;
constexpr uint32_t kRegsSoftmax = 216, kRegsProducer = 64;
constexpr int kStages = 4;
constexpr int kBlk = 128;
constexpr float kLog2_448 = 8.807354922057604f;
constexpr int kRedoHeader = 4;
constexpr int kFacCap = 512;

struct Params {
  const double* q_scales;
  const double* k_scales;
  const double* v_scales;
  const int32_t* offs;
  const int32_t* ids;
  const int32_t* items;
  int32_t n_items;
  int32_t* redo;
  int32_t exact;
  int32_t M, tv, pitch, nb, n_tail;
  float softmax_log2;
  float tau;
  void* out;
  int64_t out_ts, out_hs;
  int32_t natural;
  int32_t gh, gw, st, sh, sw, dh, dw;
};

struct Smem {
  static constexpr int kQTile = kBlk * D;        // 16 KB: this CTA's query block
  static constexpr int kKHalf = 64 * D;          // 8 KB: 64 keys x 128 B
  static constexpr int kVHalf = kBlk * 64;       // 8 KB: 128 keys x 64 channels
  static constexpr int kQ = 0;
  static constexpr int kK = 2 * kQTile;
  static constexpr int kV = kK + kStages * kKHalf;
  static constexpr int kOnes = kV + kStages * kVHalf;  // 128 keys x 64 B of e4m3 1.0: the ones MN atom
  static constexpr int kOnesTail = kOnes + kVHalf;      // the same with rows >= n_tail (padding keys) zero
  static constexpr int kBytes = kOnesTail + kVHalf;
};

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same shared offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// four MMAs of one step under one elect; `acc` predicates only the first; the descriptors advance by
// ak / bk (16-byte units) per K32 step
__device__ __forceinline__ void mma2_ss_x4_w(uint32_t d, uint64_t a, uint64_t ak, uint64_t b, uint64_t bk,
                                             uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.u32 t, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %5, %6, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %7, %8, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %9, %10, %3, t;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "l"(a + ak), "l"(b + bk), "l"(a + 2 * ak), "l"(b + 2 * bk),
      "l"(a + 3 * ak), "l"(b + 3 * bk)
      : "memory");
}
__device__ __forceinline__ void mma2_ts_x4_w(uint32_t d, uint32_t a, uint64_t b, uint64_t bk, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.eq.u32 t, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%5], %6, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%7], %8, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%9], %10, %3, t;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(a + 8), "l"(b + bk), "r"(a + 16), "l"(b + 2 * bk), "r"(a + 24),
      "l"(b + 3 * bk)
      : "memory");
}
__device__ __forceinline__ void commit2_w(uint64_t* bar) {  // arrives on `bar` in both CTAs of the pair
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int FMT, int OUT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using S = Smem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q[2], bar_qpeer[2], bar_qfree[2];
  __shared__ uint64_t bar_o, bar_ofree;
  __shared__ uint64_t bar_kv_full[kStages], bar_kv_peer[kStages], bar_kv_empty[kStages];
  __shared__ uint64_t bar_s_full[2], bar_p_ready[2];
#ifdef A2_PBUF
  __shared__ uint64_t bar_s_free[2], bar_p_free[2];
#endif
  __shared__ uint32_t s_tmem;
  __shared__ float s_xchg[2][kBlk];
  __shared__ float s_fac[2][kFacCap];
  __shared__ float s_vsc[2][D];
  __shared__ int32_t s_hdr[2][4];
  __shared__ uint64_t bar_meta_full[2], bar_meta_empty[2];
  __shared__ uint32_t s_ovf[2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int32_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int32_t* items = p.exact ? p.redo + kRedoHeader : p.items;
  const int32_t count = p.exact ? *reinterpret_cast<volatile int32_t*>(p.redo) : p.n_items;
  if ((p.exact ? cid : 2 * cid) >= count) return;  // both CTAs of the pair leave together
  auto skip = [&](int32_t it) { return !p.exact && (items[3 * it + 2] & 1); };  // odd blocks ride with the pair
  // The main list holds (tile, query block) items with the blocks of a tile adjacent; clusters walk it two
  // items at a time so that every cluster meets the even blocks (TODO: a compacted pair list for tiles with
  // an odd number of query blocks, which shift the parity).
  const int32_t stride = p.exact ? ncl : 2 * ncl;
  auto first_item = [&](int32_t c) { return p.exact ? c : 2 * c; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_q[i], 1);
      mbar_init(&bar_qpeer[i], 1);
      mbar_init(&bar_qfree[i], 1);
      mbar_init(&bar_s_full[i], 1);
      mbar_init(&bar_p_ready[i], 8);  // the step owner's 4 warps in each CTA (leader only)
#ifdef A2_PBUF
      mbar_init(&bar_s_free[i], 8);  // S(j) is in the owners' registers (leader only)
      mbar_init(&bar_p_free[i], 1);  // PV(j) has read P~(j) (multicast commit)
#endif
    }
    mbar_init(&bar_o, 1);
    mbar_init(&bar_ofree, 2 * kSoftmaxWarps);  // leader only: both CTAs' softmax warps
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_meta_full[i], 32);
      mbar_init(&bar_meta_empty[i], kSoftmaxWarps * 32);
    }
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&bar_kv_full[i], 1);
      mbar_init(&bar_kv_peer[i], 1);
      mbar_init(&bar_kv_empty[i], 1);
    }
    s_ovf[0] = s_ovf[1] = 0;
    fence_barrier_init();
  }
  {
    const uint32_t one = FMT == FPSA_E4M3 ? 0x38383838u : 0x3C3C3C3Cu;  // 1.0 in V's format
    for (int i = threadIdx.x; i < S::kVHalf / 4; i += kThreads) {
      reinterpret_cast<uint32_t*>(smem + S::kOnes)[i] = one;
      reinterpret_cast<uint32_t*>(smem + S::kOnesTail)[i] = (4 * i) / 64 < p.n_tail ? one : 0u;
    }
    fence_proxy_async_smem();  // generic-proxy writes read by the tensor core
  }
  if (warp == kTmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive or multicast commit
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tm_o = tmem;  // O: columns 0..159 (channels 0-63, row sum, channels 64-127, row sum)
  auto tm_s = [tmem](uint32_t g) { return tmem + 256u + 128u * (g & 1u); };
#ifdef A2_PBUF
  // P~ of each step parity in its own 32 columns (160..223) so QK(j+2) may overwrite S(j) before P~(j) exists
  auto tm_p = [tmem](uint32_t g) { return tmem + 160u + 32u * (g & 1u); };
#else
  auto tm_p = [tm_s](uint32_t g) { return tm_s(g); };  // P~ over the first 32 columns of S(j)
#endif
  const float tau = p.exact ? 0.0f : p.tau;

  if (warp >= kSoftmaxWarps) regs_dec<kRegsProducer>();
  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA: this CTA's Q block, K / V halves
    if (lane == 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
    }
    __syncwarp();
    uint32_t g = 0;
    int32_t iter = 0;
    for (int32_t it = first_item(cid); it < count; it += stride) {
      if (skip(it)) continue;
      const int32_t h = items[3 * it], u = items[3 * it + 1], qb = items[3 * it + 2] + (int32_t)rank;
      const int32_t kt0 = __ldg(p.offs + u), n_kt = __ldg(p.offs + u + 1) - kt0;
      const int32_t n_kv = n_kt * p.nb, steps = p.exact ? 2 * n_kv : n_kv;
      const int qbuf = iter & 1;
      if (iter >= 2) mbar_wait(&bar_qfree[qbuf], ((iter >> 1) - 1) & 1);
      mbar_arrive_expect_tx_w(&bar_q[qbuf], S::kQTile);
      tma_load_2d_w(smem + S::kQ + qbuf * S::kQTile, &tm_q, 0, (h * p.M + u) * p.pitch + qb * kBlk, &bar_q[qbuf]);
      int32_t kt = 0, b = 0;
      int32_t krow = (h * p.M + __ldg(p.ids + kt0)) * p.pitch;
      for (int32_t s = 0; s < steps; ++s, ++g) {
        const uint32_t st = g % kStages;
        if (g >= (uint32_t)kStages) mbar_wait(&bar_kv_empty[st], ((g / kStages) - 1) & 1);
        mbar_arrive_expect_tx_w(&bar_kv_full[st], S::kKHalf + S::kVHalf);
        tma_load_2d_w(smem + S::kK + st * S::kKHalf, &tm_k, 0, krow + b * kBlk + 64 * (int32_t)rank, &bar_kv_full[st]);
        tma_load_2d_w(smem + S::kV + st * S::kVHalf, &tm_v, 64 * (int32_t)rank, krow + b * kBlk, &bar_kv_full[st]);
        if (++b == p.nb) {
          b = 0;
          if (++kt == n_kt) kt = 0;
          krow = (h * p.M + __ldg(p.ids + kt0 + kt)) * p.pitch;
        }
      }
      ++iter;
    }
  } else if (warp == kMmaWarp) {
    if (rank == 0) {
      // ------------------------------------------------------------ MMA issuer (leader CTA only)
      constexpr uint32_t idesc_qk = idesc_f8(256, 128, FMT, FMT, 0);
      // PV: N = 160, each CTA's B half is [64 V channels | 16 ones]: O columns 0-63 and 80-143 hold the
      // channels, 64-79 and 144-159 the row sum of P~ (the tensor core sums the rounded weights)
      constexpr uint32_t idesc_pv = idesc_f8(256, 160, FPSA_E4M3, FMT, 1);
      const uint64_t dq0 = smem_desc_sw128(smem_u32(smem + S::kQ), 16, 1024);
      const uint64_t dk0 = smem_desc_sw128(smem_u32(smem + S::kK), 16, 1024);
      // SWIZZLE_64B MN-major V halves; the second MN atom (LBO) is the ones tile, the tail ones tile for a
      // tile's last key block. Each stage step moves the start and shortens LBO by the same amount.
      const uint32_t sv0 = smem_u32(smem + S::kV);
      auto sw64 = [](uint64_t d) { return (d & ~((uint64_t)7 << 61)) | ((uint64_t)4 << 61); };
      const uint64_t dv0 = sw64(smem_desc_sw128(sv0, smem_u32(smem + S::kOnes) - sv0, 512));
      const uint64_t dvt0 = sw64(smem_desc_sw128(sv0, smem_u32(smem + S::kOnesTail) - sv0, 512));
      constexpr uint64_t kVStageStep = (uint64_t)(S::kVHalf >> 4) - ((uint64_t)(S::kVHalf >> 4) << 16);
      uint32_t g = 0;
      int32_t iter = 0;
      uint32_t qk_st = 0, qk_ph = 0, pv_st = 0;
      for (int32_t it = first_item(cid); it < count; it += stride) {
        if (skip(it)) continue;
        const int32_t u = items[3 * it + 1];
        const int32_t n_kt = __ldg(p.offs + u + 1) - __ldg(p.offs + u);
        const int32_t n_kv = n_kt * p.nb, steps = p.exact ? 2 * n_kv : n_kv;
        const int32_t pv0 = p.exact ? n_kv : 0;
        const int qbuf = iter & 1;
        const uint64_t dq = dq0 + (uint64_t)qbuf * (S::kQTile >> 4);
        mbar_wait(&bar_q[qbuf], (iter >> 1) & 1);
        mbar_wait(&bar_qpeer[qbuf], (iter >> 1) & 1);
        tc_fence_after();
        auto issue_qk = [&](uint32_t gg) {
          mbar_wait(&bar_kv_full[qk_st], qk_ph);
          mbar_wait(&bar_kv_peer[qk_st], qk_ph);
          tc_fence_after();
          const uint64_t dk = dk0 + qk_st * (S::kKHalf >> 4);
          mma2_ss_x4_w(tm_s(gg), dq, 2, dk, 2, idesc_qk, 0u);
          commit2_w(&bar_s_full[gg & 1]);
          if (++qk_st == kStages) {
            qk_st = 0;
            qk_ph ^= 1;
          }
        };
#ifdef A2_PBUF
        auto wait_sfree = [&](uint32_t gg) {  // QK(gg) overwrites S(gg - 2): its owners must have loaded it
          if (gg >= 2) mbar_wait(&bar_s_free[gg & 1], ((gg >> 1) - 1) & 1);
        };
#else
        auto wait_sfree = [](uint32_t) {};  // PV(gg - 2), issued before QK(gg), has read P~ from S(gg - 2)
#endif
        for (int32_t s = 0; s < min(steps, 2); ++s) {
          wait_sfree(g + s);
          issue_qk(g + s);
        }
        if (steps <= 2) commit2_w(&bar_qfree[qbuf]);
        for (int32_t s = 0; s < steps; ++s) {
          const uint32_t gs = g + s;
#ifdef A2_PBUF
          if (s + 2 < steps) {  // QK(j+2) as soon as S(j) is in registers, ahead of PV(j)
            wait_sfree(gs + 2);
            issue_qk(gs + 2);
            if (s + 3 == steps) commit2_w(&bar_qfree[qbuf]);
          }
#endif
          A2_TL(0, gs, 0);
          mbar_wait(&bar_p_ready[gs & 1], (gs >> 1) & 1);
          A2_TL(0, gs, 1);
          tc_fence_after();
          if (s >= pv0) {
            if (s == pv0 && iter > 0) {
              mbar_wait(&bar_ofree, (iter - 1) & 1);
              tc_fence_after();
            }
            const uint64_t dv = ((s - pv0) % p.nb == p.nb - 1 ? dvt0 : dv0) + pv_st * kVStageStep;
            // keys 32k..: P~ columns 8k.., V rows 32k.. (32 x 64 B)
            mma2_ts_x4_w(tm_o, tm_p(gs), dv, 32 * 64 / 16, idesc_pv, s > pv0 ? 1u : 0u);
          }
          A2_TL(0, gs, 2);
#ifdef A2_PBUF
          commit2_w(&bar_p_free[gs & 1]);
#endif
          commit2_w(&bar_kv_empty[pv_st]);
          if (++pv_st == kStages) pv_st = 0;
#ifndef A2_PBUF
          if (s + 2 < steps) {
            issue_qk(gs + 2);
            if (s + 3 == steps) commit2_w(&bar_qfree[qbuf]);
          }
#endif
          A2_TL(0, gs, 3);
        }
        commit2_w(&bar_o);
        g += steps;
        ++iter;
      }
    }
  } else if (warp == kRelayWarp) {
    if (rank == 1) {
      // ------------------------------------------------------------ relay (peer CTA): forward the completion
      // of this CTA's Q and K/V loads to the leader, whose MMAs read both CTAs' shared memory
      uint32_t g = 0;
      int32_t iter = 0;
      for (int32_t it = first_item(cid); it < count; it += stride) {
        if (skip(it)) continue;
        const int32_t u = items[3 * it + 1];
        const int32_t n_kt = __ldg(p.offs + u + 1) - __ldg(p.offs + u);
        const int32_t n_kv = n_kt * p.nb, steps = p.exact ? 2 * n_kv : n_kv;
        const int qbuf = iter & 1;
        mbar_wait(&bar_q[qbuf], (iter >> 1) & 1);
        if (lane == 0) mbar_arrive_remote(&bar_qpeer[qbuf], 0);
        for (int32_t s = 0; s < steps; ++s, ++g) {
          const uint32_t st = g % kStages;
          mbar_wait(&bar_kv_full[st], (g / kStages) & 1);
          if (lane == 0) mbar_arrive_remote(&bar_kv_peer[st], 0);
        }
        ++iter;
      }
    }
  } else if (warp == kHelperWarp) {
    const float sl = p.softmax_log2;
    int32_t iter = 0;
    for (int32_t it = first_item(cid); it < count; it += stride) {
      if (skip(it)) continue;
      const int slot = iter & 1;
      if (iter >= 2) mbar_wait(&bar_meta_empty[slot], ((iter >> 1) - 1) & 1);
      const int32_t h = items[3 * it], u = items[3 * it + 1];
      const int32_t kt0 = __ldg(p.offs + u), n_kt = __ldg(p.offs + u + 1) - kt0;
      const float qs = (float)__ldg(p.q_scales + h * p.M + u);
      const double* ks = p.k_scales + (int64_t)h * p.M;
      for (int32_t i = lane; i < min(n_kt, kFacCap); i += 32)
        s_fac[slot][i] = (qs * (float)__ldg(ks + __ldg(p.ids + kt0 + i))) * sl;
      for (int i = lane; i < D; i += 32) s_vsc[slot][i] = (float)__ldg(p.v_scales + (int64_t)h * D + i);
      if (lane == 0) {
        s_hdr[slot][0] = kt0;
        s_hdr[slot][1] = n_kt;
      }
      mbar_arrive(&bar_meta_full[slot]);
      ++iter;
    }
  } else if (warp < kSoftmaxWarps) {
    regs_inc<kRegsSoftmax>();
    const int quarter = warp & 3, part = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl = p.softmax_log2;
    auto row_sync = [&]() { named_bar_sync(1 + quarter, 64); };
    auto row_comb = [&](float m, bool is_max) {
      s_xchg[part][row] = m;
      row_sync();
      const float a = s_xchg[0][row], b2 = s_xchg[1][row];
      row_sync();
      return is_max ? fmaxf(a, b2) : a + b2;
    };
    auto signal = [&](uint64_t* bar) {  // this warp's tcgen05 traffic of the step is complete: tell the leader
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(bar);
        else mbar_arrive_remote(bar, 0);
      }
    };
    auto owned = [&](uint32_t gg) { return (int)(gg & 1u) == part; };
    auto ncol_blk = [&](int32_t bb) { return bb == p.nb - 1 ? p.n_tail : kBlk; };
    uint32_t g = 0;
    int32_t iter = 0;
    for (int32_t it = first_item(cid); it < count; it += stride) {
      if (skip(it)) continue;
      const int32_t h = items[3 * it], u = items[3 * it + 1], qb = items[3 * it + 2] + (int32_t)rank;
      const bool live = qb * kBlk < p.tv;  // a tile with an odd number of blocks pairs its last with nothing
      const int slot = iter & 1;
      mbar_wait(&bar_meta_full[slot], (iter >> 1) & 1);
      const int32_t kt0 = s_hdr[slot][0], n_kt = s_hdr[slot][1];
      const int32_t n_kv = n_kt * p.nb;
      const float* fac = s_fac[slot];
      auto factor_at = [&](int32_t kt) {
        if (kt < kFacCap) return fac[kt];
        const float qs = (float)__ldg(p.q_scales + h * p.M + u);
        return (qs * (float)__ldg(p.k_scales + (int64_t)h * p.M + __ldg(p.ids + kt0 + kt))) * sl;
      };
      float m_ref = 0.0f;
      uint32_t sat = 0u;
      if (p.exact) {
        float m_acc = -INFINITY;
        int32_t kt = 0, b = 0;
        for (int32_t j = 0; j < n_kv; ++j, ++g) {
          if (owned(g)) {
            const float c = factor_at(kt);
            mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
            tc_fence_after();
            m_acc = fmaxf(m_acc, block_max<kBlk>(tm_s(g) + lane_off, ncol_blk(b), false) * c);
#ifdef A2_PBUF
            signal(&bar_s_free[g & 1]);
            if (g >= 2) mbar_wait(&bar_p_free[g & 1], ((g >> 1) - 1) & 1);  // keeps the phases in step
#endif
            signal(&bar_p_ready[g & 1]);
          }
          if (b == p.nb - 1) {
            b = 0;
            ++kt;
          } else {
            ++b;
          }
        }
        m_ref = row_comb(m_acc, true);
      } else {
        float m0 = -INFINITY;
        if (owned(g)) {
          mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
          tc_fence_after();
          m0 = block_max<kBlk>(tm_s(g) + lane_off, ncol_blk(0), false) * factor_at(0);
        }
        m_ref = row_comb(m0, true);
      }
      {
        int32_t kt = 0, b = 0;
        float c = factor_at(0);
        const float bias = kLog2_448 - m_ref - tau;
        for (int32_t j = 0; j < n_kv; ++j, ++g) {
          if (owned(g)) {
            if (warp == 0 || warp == 4) A2_TL(1 + rank, g, 0);
            mbar_wait(&bar_s_full[g & 1], (g >> 1) & 1);
            if (warp == 0 || warp == 4) A2_TL(1 + rank, g, 1);
            tc_fence_after();
            const uint32_t s_row = tm_s(g) + lane_off;
            const int n = ncol_blk(b);
            uint32_t w[kBlk / 4];
            {
              uint32_t sreg[64];
              load_s_all<64>(s_row, sreg);
              tmem_wait_ld();
              sat |= compute_p_regs<64>(sreg, min(n, 64), c, bias, w);
            }
            {
              uint32_t sreg[64];
              load_s_all<64>(s_row + 64, sreg);
              tmem_wait_ld();
#ifdef A2_PBUF
              signal(&bar_s_free[g & 1]);
#endif
              sat |= compute_p_regs<64>(sreg, max(n - 64, 0), c, bias, w + 16);
            }
            if (warp == 0 || warp == 4) A2_TL(1 + rank, g, 2);
#ifdef A2_PBUF
            if (g >= 2) {
              mbar_wait(&bar_p_free[g & 1], ((g >> 1) - 1) & 1);  // PV(j-2) has read this P~ buffer
              tc_fence_after();
            }
#endif
            tmem_st32(tm_p(g) + lane_off, w);
            tmem_wait_st();
            signal(&bar_p_ready[g & 1]);
            if (warp == 0 || warp == 4) A2_TL(1 + rank, g, 3);
          }
          if (b == p.nb - 1) {
            b = 0;
            if (++kt < n_kt) c = factor_at(kt);
          } else {
            ++b;
          }
        }
      }
      // ---------------------------------------------------------- epilogue
      mbar_wait(&bar_o, iter & 1);
      tc_fence_after();
      float inv_l;
      {
        uint32_t lw[16];
        tmem_ld16(tm_o + lane_off + 64, lw);  // row sum of P~ (the ones columns of CTA 0's half)
        tmem_wait_ld();
        inv_l = 1.0f / __uint_as_float(lw[0]);
      }
      const int32_t r = qb * kBlk + row;
      int64_t token;
      if (p.natural) {
        const int32_t ut = u / (p.dh * p.dw), uh = (u / p.dw) % p.dh, uw = u % p.dw;
        const int32_t lt = r / (p.sh * p.sw), lh = (r / p.sw) % p.sh, lw = r % p.sw;
        token = ((int64_t)(ut * p.st + lt) * p.gh + (uh * p.sh + lh)) * p.gw + (uw * p.sw + lw);
      } else {
        token = (int64_t)u * p.tv + r;
      }
      const float* vs = s_vsc[slot];
#pragma unroll
      for (int cc = 0; cc < D / 2; cc += 32) {
        const int col = part * (D / 2) + cc;
        uint32_t o[32];
        tmem_ld32(tm_o + lane_off + col + (col >= 64 ? 16 : 0), o);
        tmem_wait_ld();
        if (r < p.tv) {
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(o[i]) * inv_l * vs[col + i];
          if constexpr (OUT == FPSA_F32) {
            float4* dst =
                reinterpret_cast<float4*>(static_cast<float*>(p.out) + token * p.out_ts + h * p.out_hs + col);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + token * p.out_ts +
                                                  h * p.out_hs + col);
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
      signal(&bar_ofree);
      mbar_arrive(&bar_meta_empty[slot]);
      if (!p.exact) {
        if (__any_sync(0xffffffffu, live && sat != 0u) && lane == 0) atomicOr(&s_ovf[iter & 1], 1u);
        named_bar_sync(5, kSoftmaxWarps * 32);
        if (threadIdx.x == 0 && s_ovf[iter & 1]) {  // either CTA may append its pair (duplicates are harmless)
          s_ovf[iter & 1] = 0;
          const int32_t slot2 = atomicAdd(p.redo, 1);
          p.redo[kRedoHeader + 3 * slot2] = h;
          p.redo[kRedoHeader + 3 * slot2 + 1] = u;
          p.redo[kRedoHeader + 3 * slot2 + 2] = qb - (int32_t)rank;
        }
      }
      ++iter;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == kTmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

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

int make_map(CUtensorMap* m, const uint8_t* base, int64_t rows, uint32_t box_cols, uint32_t box_rows,
             CUtensorMapSwizzle swz) {
  auto fn = encoder();
  if (!fn) return fail(FPSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FPSA_ECUDA, "cuTensorMapEncodeTiled (2-CTA) failed: " + std::to_string((int)r));
  return FPSA_OK;
}

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int FMT, int OUT>
int launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, Params p, cudaStream_t st) {
  auto kern = attn2_kernel<FMT, OUT>;
  constexpr int smem = Smem::kBytes + 1024;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return fail(FPSA_ECUDA, std::string("cudaFuncSetAttribute (2-CTA): ") + cudaGetErrorString(cudaGetLastError()));
    configured = true;
  }
  if (cudaMemsetAsync(p.redo, 0, sizeof(int32_t), st) != cudaSuccess)
    return fail(FPSA_ECUDA, std::string("redo reset: ") + cudaGetErrorString(cudaGetLastError()));
  // persistent: as many pairs as can be co-resident (pairs need two free SMs of one TPC; not all 74 fit)
  static int max_pairs = 0;
  if (!max_pairs) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms(), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&max_pairs, (void*)kern, &cfg) != cudaSuccess || max_pairs <= 0) {
      cudaGetLastError();
      max_pairs = sms() / 2;
    }
    if (getenv("FPSA_ATTN2_VERBOSE")) printf("attn2: %d co-resident CTA pairs\n", max_pairs);
  }
  const int grid = 2 * std::min(p.n_items, max_pairs);
  p.exact = 0;
  kern<<<grid, kThreads, smem, st>>>(tq, tk, tv, p);
  p.exact = 1;
  kern<<<grid, kThreads, smem, st>>>(tq, tk, tv, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FPSA_ECUDA, std::string("attn2 launch: ") + cudaGetErrorString(e));
  return FPSA_OK;
}

}  // namespace a2
}  // namespace
}  // namespace fpsa

using namespace fpsa;

// Same contract as fpsa_attn_fwd for d = 128 and tiles of more than 128 tokens (fpsa_attn_fwd dispatches).
extern "C" int fpsa_attn2_fwd(const uint8_t* q_codes, const uint8_t* k_codes, const uint8_t* v_codes,
                              const double* q_scales, const double* k_scales, const double* v_scales, int32_t heads,
                              fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, const int32_t* offs,
                              const int32_t* ids, const int32_t* items, int32_t n_items, float softmax_scale,
                              int fmt, float tau_log2, void* out, int out_dtype, int64_t out_token_stride,
                              int64_t out_head_stride, int out_order, void* workspace, int64_t workspace_bytes,
                              void* stream) {
  fpsa_dims3 td;
  if (int s = fpsa_tile_grid(grid, tile, &td)) return s;
  const int32_t tv = tile.t * tile.h * tile.w;
  const int32_t M = td.t * td.h * td.w;
  const int64_t rows = (int64_t)heads * M * tile_pitch;
  CUtensorMap tq, tk, tvm;
  if (int s = a2::make_map(&tq, q_codes, rows, 128, 128, CU_TENSOR_MAP_SWIZZLE_128B)) return s;
  if (int s = a2::make_map(&tk, k_codes, rows, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return s;
  if (int s = a2::make_map(&tvm, v_codes, rows, 64, 128, CU_TENSOR_MAP_SWIZZLE_64B)) return s;
  a2::Params p{};
  p.q_scales = q_scales;
  p.k_scales = k_scales;
  p.v_scales = v_scales;
  p.offs = offs;
  p.ids = ids;
  p.items = items;
  p.n_items = n_items;
  p.redo = static_cast<int32_t*>(workspace);
  p.M = M;
  p.tv = tv;
  p.pitch = tile_pitch;
  p.nb = (tv + 127) / 128;
  p.n_tail = tv - 128 * (p.nb - 1);
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
  (void)d;
  (void)workspace_bytes;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fmt == FPSA_E4M3) {
    if (out_dtype == FPSA_F32) return a2::launch<FPSA_E4M3, FPSA_F32>(tq, tk, tvm, p, st);
    return a2::launch<FPSA_E4M3, FPSA_BF16>(tq, tk, tvm, p, st);
  }
  if (out_dtype == FPSA_F32) return a2::launch<FPSA_E5M2, FPSA_F32>(tq, tk, tvm, p, st);
  return a2::launch<FPSA_E5M2, FPSA_BF16>(tq, tk, tvm, p, st);
}

#ifdef A2_TRACE
extern "C" int fpsa_a2_trace(long long* out) {
  cudaMemcpyFromSymbol(out, fpsa::a2::g_a2, sizeof(fpsa::a2::g_a2));
  return 0;
}
#endif
