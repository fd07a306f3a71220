// K4: sliding-tile sparse FP8 attention forward, sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces fp8sta.attention.fp8_sparse_forward / _engine
// (/root/reference/pkg/src/fp8sta/attention.py:91-149, :179-208).
//
// Persistent kernel: one CTA per SM walks a list of work items, one item =
// (head h, query tile u, one 128-row query block of u).  The key sequence of
// u is the concatenation of its admissible key tiles in ascending id order
// (sparsity.py:63-67, the reference's reduction order), each key tile cut
// into 128-key blocks; a tile's last block has n_tail = tv - 128 (nb - 1)
// valid keys.  The zero padding keys past them have zero V rows, and the PV of
// a last block uses a "ones" atom whose rows past n_tail are zero, so their P~
// codes add nothing to O or to the row sum l (no per-step masking).  Per key block j:
//
//   S(j)  = Q K_j^T                  tcgen05.mma kind::f8f6f4 M128 N128, A/B from
//                                    smem, fp32 accumulator in TMEM buffer j % 2
//   x     = S * (sq[u] * sk[v] * softmax_scale * log2 e)     per-tile factors
//   m     = row max of the first key block (fixed for the item)
//   P~    = e4m3(448 * 2^-tau * 2^(x - m))   re-quantised per key block,
//           written to TMEM P~ buffer j % 2 (4 codes per column)
//   [O|l] += P~ [V_j | 1]             tcgen05.mma N = D + 16, A = P~ from TMEM,
//                                    B = V from smem (MN-major, V stored [keys][d])
//                                    plus a constant "ones" MN atom: the extra
//                                    columns accumulate the row sum l of P~
// and finally out = O * v_scale[c] / l.
//
// Overflow: a P~ code equal to 0x7E (448) may be a saturated weight (a logit
// more than tau above m).  Its item is appended to a redo list and recomputed
// by a second launch of the same kernel in exact mode: a first pass over the
// keys takes the exact row max, a second pass uses it with tau = 0
// (DESIGN.md).
//
// TMEM: [O|l] (D + 16 columns), P~ buffers at columns 160 / 192, S(even) at
// column 256, S(odd) at 384.  S(j+2) is computed as soon as the owners of S(j)
// have it in registers; PV(j) reads P~(j) from its own buffer.
//
// Warp roles (384 threads): warps w and w+4 (w < 4) share TMEM lane quarter w
// (rows 32w..32w+31) and take alternate key blocks (ping-pong): warp w the
// even steps, warp w+4 the odd ones, each computing whole 128-key rows.  Warp
// 8 is the TMA producer (and TMEM allocator), warp 9 issues the QKs, warp 11
// the PVs (split issue: QK and PV touch disjoint TMEM, and every PV comes from
// the one PV warp in order), warp 10 claims work items (a global atomic
// counter: CTAs take the next item of the longest-first list when they are
// ready for it, so no CTA is left with a longer share) and prefetches their
// metadata.  The claimed (head, tile, block) triples reach the other roles
// through a 4-deep ring in shared memory.  Step barriers are reused every
// second step, so none may run two phases ahead of its waiter (DESIGN.md,
// "Phase discipline of the split issue").
//
// Normalised-P mode (template NORM, the reference's exact semantics,
// attention.py:133-145): three passes over the keys of an item -- exact row
// max m, row sum l = sum exp(s - m) in f64, then P~ = e4m3(448 * exp(s - m) / f32(l))
// with s = S * f32(k_scale * f32(q_scale * softmax_scale)) and exp correctly
// rounded to f32 -- and out = O * f32(v_scale / 448), no division by l.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <mutex>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"
#include "sm100.cuh"
#include "softmax.cuh"

#ifndef FPSA_GEOM_PREFETCH
#define FPSA_GEOM_PREFETCH 1  // next block's geometry / factors computed during the current S load
#endif
#ifndef FPSA_PACK_FASTPATH
#define FPSA_PACK_FASTPATH 1  // packed blocks inside one key tile take the per-tile softmax code
#endif


namespace fpsa {
namespace {

using namespace sm100;

#ifndef FPSA_MBAR_SUSPEND_NS
#define FPSA_MBAR_SUSPEND_NS 100000
#endif
#ifdef FPSA_WATCH
// debug builds only: per (CTA, warp) the shared address and parity of the barrier it waits on (0: none),
// written to mapped host memory so a hung launch can be inspected (tools/watch_attn.py)
__device__ int* g_watch;
#endif
// every wait of this kernel carries the suspend-time hint (sm100.cuh mbar_try_wait)
__device__ __forceinline__ void attn_wait(uint64_t* bar, uint32_t parity) {
#ifdef FPSA_WATCH
  volatile int* w = g_watch + (blockIdx.x * 16 + (threadIdx.x >> 5)) * 4;
  if ((threadIdx.x & 31) == 0) {
    w[0] = (int)smem_u32(bar);
    w[1] = (int)parity;
    w[2] = w[2] + 1;
    __threadfence_system();
  }
#endif
  mbar_wait<FPSA_MBAR_SUSPEND_NS>(bar, parity);
#ifdef FPSA_WATCH
  if ((threadIdx.x & 31) == 0) {
    w[0] = 0;
    __threadfence_system();
  }
#endif
}

// Ping-pong softmax: the two warps of an SMSP (one TMEM lane quarter) take alternate key blocks, each
// computing whole 128-key rows (both warps on the two halves of every block measured 12.65 vs 12.1 ms;
// three warps per SMSP at 144 registers 11.4 vs 11.05 ms, profiles/r02_ab_three_parts_rejected.txt).
constexpr int kParts = 2;                       // softmax warps sharing one TMEM lane quarter (row)
constexpr int kEpiParts = 2;                    // parts that read O in the epilogue (D / 2 channels each)
constexpr int kSoftmaxWarps = 4 * kParts;
constexpr int kTmaWarp = kSoftmaxWarps;
constexpr int kMmaWarp = kSoftmaxWarps + 1;     // issues the QKs
constexpr int kHelperWarp = kSoftmaxWarps + 2;  // claims items, prefetches their metadata
constexpr int kPvWarp = kSoftmaxWarps + 3;      // issues the PVs
constexpr int kThreads = (kSoftmaxWarps + 4) * 32;  // two softmax warpgroups + the producer warpgroup
// setmaxnreg split of the 64K-register file: per SMSP one warp of each warpgroup
// (4 warps per quarter at 104 registers was measured slower: 13.4 vs 12.8 ms at C2; 112/64 deadlocks)
constexpr uint32_t kRegsSoftmax = 216, kRegsProducer = 64;

constexpr int kStages = 4;     // K/V ring depth (128-key blocks)
constexpr int kBlk = 128;      // rows per query block = keys per key block
constexpr float kLog2_448 = 8.807354922057604f;
constexpr int kRedoHeader = 4;  // int32 words before the redo items in the workspace
constexpr int kFacCap = 512;    // key-tile factors per item kept in shared memory (more: read from L2)
constexpr int kItemRing = 4;                    // claimed items in flight between the helper and the other roles
constexpr int kItemReaders = 3 + kSoftmaxWarps;  // TMA, QK and PV warps, softmax warps
struct AttnParams {
  const double* q_scales;
  const double* k_scales;
  const double* v_scales;
  const int32_t* offs;
  const int32_t* ids;
  const int32_t* items;  // (head, tile, query block) triples
  int32_t n_items;
  int32_t* redo;         // [0]: count, [kRedoHeader..]: triples of items to recompute exactly
  int32_t* claim;        // work-item counter of this launch (zeroed before the launch)
  int32_t exact;         // 1: this launch recomputes the redo list with the exact row max
  int32_t M, tv, pitch, nb;  // nb: 128-key blocks per tile
  int32_t n_tail;     // valid keys of the last key block of a tile: tv - 128 (nb-1); the
                      // QK MMA still runs N = 128 over zero K rows, whose S = 0 the softmax drops
  float softmax_log2;  // f32(softmax_scale * log2 e)
  float softmax_scale;  // f32 softmax scale (normalised-P factors)
  float tau;
  void* out;
  int64_t out_ts, out_hs;
  int32_t natural;
  int32_t gh, gw, st, sh, sw, dh, dw;
  int32_t packed;  // key blocks run over the concatenated valid keys of the window's tiles (no padding keys)
  uint32_t div_tv, div_nb;  // ceil(2^32 / tv), ceil(2^32 / nb): exact quotients of the block geometry
};

// floor(x / d) for the magic m = ceil(2^32 / d), exact while x < 2^32 / d (key positions here are < 2^21)
__device__ __forceinline__ uint32_t div_magic(uint32_t x, uint32_t m) { return __umulhi(x, m); }

// TMA maps of the packed key blocks' segments: box heights 16, 32, ..., 128 rows (index n / 16 - 1), so a
// block split between two key tiles costs two loads per operand.
struct SegMaps {
  CUtensorMap k[kBlk / 16];
  CUtensorMap v[kBlk / 16];
};

// Position in an item's key stream during one pass.  Unpacked: every tile is cut into nb 128-key blocks (the
// last has n_tail valid keys); packed (tile volume a multiple of 16 and >= 128): blocks of 128 consecutive
// keys of the concatenated tiles, so a block holds the tail of tile kt and the head of tile kt + 1.
struct KeyWalk {
  int32_t kt = 0;  // tile (index into the item's window list)
  int32_t r = 0;   // packed: first row of the next block in tile kt; unpacked: block index in tile kt
};
// The next block: keys [0, split) come from tile kt_a (from row `row0` on), keys [split, nvalid) from tile
// kt_a + 1 (from row 0), keys >= nvalid are absent (padding or past the stream end).
template <bool PACKED>
__device__ __forceinline__ void next_block(const AttnParams& p, int32_t n_kt, KeyWalk& w, int32_t& kt_a,
                                           int32_t& row0, int32_t& split, int32_t& nvalid) {
  kt_a = w.kt;
  if constexpr (PACKED) {
    row0 = w.r;
    const int32_t n1 = min(kBlk, p.tv - w.r);
    split = nvalid = n1;
    w.r += n1;
    if (w.r == p.tv) {
      ++w.kt;
      w.r = 0;
      if (n1 < kBlk && w.kt < n_kt) {
        w.r = kBlk - n1;
        nvalid = kBlk;
      }
    }
  } else {
    row0 = w.r * kBlk;
    nvalid = w.r == p.nb - 1 ? p.n_tail : kBlk;
    split = kBlk;
    if (++w.r == p.nb) {
      w.r = 0;
      ++w.kt;
    }
  }
}
// Geometry of block j of a pass in closed form (the softmax warps visit only the blocks they own).
template <bool PACKED>
__device__ __forceinline__ void block_at(const AttnParams& p, int32_t n_kt, int32_t j, int32_t& kt_a, int32_t& split,
                                         int32_t& nvalid) {
  if constexpr (PACKED) {
    const int32_t pos = j * kBlk;
    kt_a = p.div_tv ? (int32_t)div_magic((uint32_t)pos, p.div_tv) : pos / p.tv;
    split = min(kBlk, p.tv - (pos - kt_a * p.tv));
    nvalid = min(kBlk, n_kt * p.tv - pos);
  } else {
    kt_a = p.div_nb ? (int32_t)div_magic((uint32_t)j, p.div_nb) : j / p.nb;
    nvalid = j - kt_a * p.nb == p.nb - 1 ? p.n_tail : kBlk;
    split = kBlk;
  }
}

// 128-key blocks of one pass over an item's n_kt key tiles
template <bool PACKED>
__device__ __forceinline__ int32_t blocks_per_pass(const AttnParams& p, int32_t n_kt) {
  return PACKED ? (n_kt * p.tv + kBlk - 1) / kBlk : n_kt * p.nb;
}

// S = Q K^T: K = D in K32 steps (one elect for the four MMAs of D = 128)
template <int D>
__device__ __forceinline__ void qk_mma(uint32_t ts, uint64_t dq, uint64_t dk, uint32_t idesc) {
  if constexpr (D == 128) {
    mma_f8_ss_x4_w(ts, dq, dq + 2, dq + 4, dq + 6, dk, dk + 2, dk + 4, dk + 6, idesc, 0u);
  } else {
#pragma unroll
    for (int k = 0; k < D / 32; ++k) mma_f8_ss_w(ts, dq + 2 * k, dk + 2 * k, idesc, k > 0 ? 1u : 0u);
  }
}

template <int D>
struct Smem {
  static constexpr int kTile = kBlk * D;  // bytes of one 128-row fp8 tile
  static constexpr int kQ = 0;            // two query-block buffers (next item prefetched)
  static constexpr int kK = 2 * kTile;
  static constexpr int kV = kK + kStages * kTile;
  static constexpr int kOnes = kV + kStages * kTile;  // 128 rows x D bytes of e4m3 1.0 (the "ones" MN atom)
  static constexpr int kOnesTail = kOnes + kTile;      // the same with rows >= n_tail (padding keys) zero
  static constexpr int kBytes = kOnesTail + kTile;
  static constexpr uint32_t kSBO = 8 * D;  // 8 rows of D bytes
};

template <int D>
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t addr) {
  uint64_t d = smem_desc_sw128(addr, 16, Smem<D>::kSBO);
  if constexpr (D == 64) d = (d & ~((uint64_t)7 << 61)) | ((uint64_t)4 << 61);  // SWIZZLE_64B
  return d;
}
// MN-major V block whose second MN atom (columns D..D+15 of B) is the ones
// region at byte offset `lbo` (leading byte offset field, 16-byte units).
template <int D>
__device__ __forceinline__ uint64_t desc_mnmajor_ones(uint32_t addr, uint32_t lbo) {
  uint64_t d = smem_desc_sw128(addr, lbo, Smem<D>::kSBO);
  if constexpr (D == 64) d = (d & ~((uint64_t)7 << 61)) | ((uint64_t)4 << 61);
  return d;
}
template <int D>
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t addr) {
  uint64_t d = smem_desc_sw128(addr, 16384, Smem<D>::kSBO);
  if constexpr (D == 64) d = (d & ~((uint64_t)7 << 61)) | ((uint64_t)4 << 61);
  return d;
}

#ifdef FPSA_TRACE
// Debug builds only: counters accumulated over all CTAs.
//   [0] softmax: cycles waiting for S   [1] softmax: step-loop cycles   [2] softmax: first-pass compute
//   [3] MMA: cycles waiting for P~      [5] redo items                  [6] softmax warp-steps
//   [4] softmax: S load (tcgen05.ld + wait) cycles   [7] MMA: cycles waiting for K/V
#endif

// The normalised-P mode's exp: CUDA's accurate expf (<= 2 ulp, like numpy's own f32 exp against the
// correctly rounded value; an f64 exp rounded to f32 measured 34x slower for the same parity).
// Not inlined: it is called per element of a fully unrolled row and would otherwise multiply the code size.
#ifndef FPSA_NORM_EXP_F64
__device__ __noinline__ float exp_f32_cr(float x) { return expf(x); }
#else
__device__ __noinline__ float exp_f32_cr(float x) { return __double2float_rn(exp((double)x)); }
#endif

// Normalised-P pass 2: f64 sum of exp(S * c - m) over the first ncol of NC S columns; columns < split use
// factor ca, the others cb (a packed block's two key tiles).
template <int NC>
__device__ __forceinline__ double expsum_norm(const uint32_t* s, int split, int ncol, float ca, float cb, float m) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < NC; ++i)
    if (i < ncol) acc += (double)exp_f32_cr(__fsub_rn(__fmul_rn(__uint_as_float(s[i]), i < split ? ca : cb), m));
  return acc;
}
// Normalised-P pass 3: P~ = e4m3(448 * (exp(S * c - m) / l)), packed 4 per word; columns >= ncol are 0.
template <int NC>
__device__ __forceinline__ void compute_p_norm(const uint32_t* s, int split, int ncol, float ca, float cb, float m,
                                               float l, uint32_t* w) {
#pragma unroll
  for (int i = 0; i < NC; i += 4) {
    float pv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float c = i + k < split ? ca : cb;
      const float e = exp_f32_cr(__fsub_rn(__fmul_rn(__uint_as_float(s[i + k]), c), m));
      pv[k] = i + k < ncol ? __fmul_rn(__fdiv_rn(e, l), 448.0f) : 0.0f;
    }
    w[i / 4] = e4m3x4(f2{pv[0], pv[1]}, f2{pv[2], pv[3]});
  }
}

template <int D, int FMT, int OUT, bool NORM, bool PACKED>
__global__ void __launch_bounds__(kThreads, 1)
    fpsa_attn_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ SegMaps seg,
                     const AttnParams p) {
  using S = Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q[2], bar_qfree[2];  // query-block buffer (item parity): loaded / no longer read
  __shared__ uint64_t bar_o, bar_ofree;        // O complete for the item / epilogue has read O
  __shared__ uint64_t bar_kv_full[kStages], bar_kv_empty[kStages];
  // S(j) full: by j mod kSF (a waiter is never two phases ahead); P~(j) ready / its buffer free: by j mod
  // kParts (the owning part); S buffer j mod 2 loaded by its owners (early QK)
  constexpr int kSF = 2;
  __shared__ uint64_t bar_s_full[kSF], bar_p_ready[kParts];
  __shared__ uint64_t bar_s_free[2], bar_p_free[kParts];
  __shared__ uint32_t s_tmem;
  __shared__ float s_xchg[kParts][kBlk];  // [part][row] exchange between the warps of a row
  // per-item metadata, prefetched by the helper warp one item ahead (slot = item parity)
  __shared__ float s_fac[2][kFacCap];  // key-tile factors c(kt) = (sq * sk) * scale log2 e
  __shared__ float s_vsc[2][D];        // V channel scales
  __shared__ int32_t s_hdr[2][4];      // kt0, n_kt, unused, unused
  __shared__ uint64_t bar_meta_full[2], bar_meta_empty[2];
  __shared__ uint32_t s_ovf[2];      // per item parity: some row overflowed
  // claimed work items (helper warp -> TMA, MMA, softmax): head (-1: no more items), tile, query block
  __shared__ int32_t s_item[kItemRing][4];
  __shared__ uint64_t bar_item_full[kItemRing], bar_item_empty[kItemRing];
  __shared__ double s_xchg_d[NORM ? kParts : 1][kBlk];  // normalised-P row-sum exchange

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // re-read from the parameter bank at each use (a long-lived pointer is spilled across the role switch)
  auto item_at = [&p](int32_t i) { return (p.exact ? p.redo + kRedoHeader : p.items)[i]; };
  const int32_t count = p.exact ? *reinterpret_cast<volatile int32_t*>(p.redo) : p.n_items;
  if ((int32_t)blockIdx.x >= count) return;  // at most `count` CTAs can claim an item
  constexpr int32_t kNormPasses = 3;
  const int32_t passes = NORM ? kNormPasses : (p.exact ? 2 : 1);  // key sweeps per item; the last one runs PV
  // next claimed item of this role's `iter`-th loop trip; false when the list is exhausted
  auto next_item = [&](int32_t iter, int32_t& h, int32_t& u, int32_t& qb) {
    const int r = iter % kItemRing;
    attn_wait(&bar_item_full[r], (iter / kItemRing) & 1);
    h = s_item[r][0];
    u = s_item[r][1];
    qb = s_item[r][2];
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar_item_empty[r]);
    return h >= 0;
  };

  // P~(gg) ready (or S(gg) consumed): one arrival per owning warp; the PV warp waits for all of them
  constexpr uint32_t kPArrivals = kSoftmaxWarps / kParts;
  // barrier slot and phase of step gg: S full (kSF slots), P~ ready / P~ buffer free (kParts slots)
  auto sf_wait = [&](uint32_t gg) { attn_wait(&bar_s_full[gg % kSF], (gg / kSF) & 1); };
  // Split issue: before P~(gg) ready (or S(gg) consumed) is signalled, PV(gg - kParts) must have been
  // handled, so that p_ready[gg % kParts] never runs two phases ahead of the PV warp.  The main pass gets this
  // from waiting for its P~ buffer; the max / sum passes of the exact and normalised modes, which store no
  // P~, wait here (without it the softmax could signal two phases of one barrier before the PV warp
  // observed the first, and the PV warp would then wait for a phase that needs its own K/V release).
  auto p_free_wait = [&](uint32_t gg) {
    if (gg >= (uint32_t)kParts) attn_wait(&bar_p_free[gg % kParts], ((gg / kParts) - 1) & 1);
  };
  // (a shared-memory counter instead of the p_ready mbarrier measured slower: 11.5-11.65 vs 11.26-11.33 ms)
  auto p_arrive = [&](uint32_t gg) { mbar_arrive(&bar_p_ready[gg % kParts]); };  // lane 0, after its fence
  auto p_wait = [&](uint32_t gg) { attn_wait(&bar_p_ready[gg % kParts], (gg / kParts) & 1); };

  if (threadIdx.x == 0) {
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(&bar_item_full[i], 1);
      mbar_init(&bar_item_empty[i], kItemReaders);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_q[i], 1);
      mbar_init(&bar_qfree[i], 1);
      mbar_init(&bar_s_free[i], kSoftmaxWarps / kParts);
    }
    for (int i = 0; i < kSF; ++i) mbar_init(&bar_s_full[i], 1);
    for (int i = 0; i < kParts; ++i) {
      mbar_init(&bar_p_ready[i], kPArrivals);  // one arrival per writing warp
      mbar_init(&bar_p_free[i], 1);
    }
    mbar_init(&bar_o, 1);
    mbar_init(&bar_ofree, kSoftmaxWarps);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_meta_full[i], 32);                 // every helper lane releases its own writes
      mbar_init(&bar_meta_empty[i], kSoftmaxWarps * 32);  // every softmax thread releases its reads
    }
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&bar_kv_full[i], 1);
      mbar_init(&bar_kv_empty[i], 1);
    }
    s_ovf[0] = s_ovf[1] = 0;
#ifdef FPSA_WATCH
    if (blockIdx.x == 0) {
      volatile int* a = g_watch + 148 * 16 * 4;
      int n = 0;
      auto put = [&](uint64_t* b, int cnt) { for (int i = 0; i < cnt; ++i) a[n++] = (int)smem_u32(b + i); };
      put(bar_q, 2); put(bar_qfree, 2); put(&bar_o, 1); put(&bar_ofree, 1); put(bar_kv_full, kStages);
      put(bar_kv_empty, kStages); put(bar_s_full, kSF); put(bar_p_ready, kParts); put(bar_s_free, 2);
      put(bar_p_free, kParts); put(bar_meta_full, 2); put(bar_meta_empty, 2); put(bar_item_full, kItemRing);
      put(bar_item_empty, kItemRing);
      __threadfence_system();
    }
#endif
    fence_barrier_init();
  }
  if (warp == kTmaWarp) {
    tmem_alloc(&s_tmem, 512);
    tmem_relinquish();
  }
  for (int i = threadIdx.x; i < S::kTile / 4; i += kThreads) {  // 1.0 in V's format; row = key of the block
    const uint32_t one = FMT == FPSA_E4M3 ? 0x38383838u : 0x3C3C3C3Cu;
    reinterpret_cast<uint32_t*>(smem + S::kOnes)[i] = one;
    reinterpret_cast<uint32_t*>(smem + S::kOnesTail)[i] = (4 * i) / D < p.n_tail ? one : 0u;
  }
  if constexpr (PACKED) {
    // a stream's last block leaves stage rows unloaded: their P~ codes are zeroed, and zero-initialised
    // stages guarantee that what those codes multiply is a finite e4m3 value, never a NaN pattern
    for (int i = threadIdx.x; i < 2 * kStages * S::kTile / 16; i += kThreads)
      reinterpret_cast<uint4*>(smem + S::kK)[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_proxy_async_smem();  // generic-proxy writes read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tm_o = tmem;  // O: columns 0..D-1, row sums of P~: D..D+15
  // S buffers at columns 256 and 384 (computed, not indexed: a local array would live in memory)
  auto tm_s = [tmem](uint32_t g) { return tmem + 256u + 128u * (g & 1u); };
  // P~(j) in its own 32 columns (160 / 192), so S(j)'s buffer is free once loaded.  Split issue: warp 9
  // issues the QKs (on S(j - 2) loaded), warp 11 the PVs (on P~(j) stored); QK and PV touch disjoint TMEM
  // (S buffers / P~ buffers and O), and every PV comes from the one PV warp, in order
  auto tm_p = [tmem](uint32_t g) { return tmem + 160u + 32u * (g % (uint32_t)kParts); };
  static_assert(D + 16 <= 160 && 160 + 32 * kParts <= 256, "TMEM: O | P~ buffers | S buffers at 256 and 384");
  const float tau = p.exact ? 0.0f : p.tau;

  if (warp >= kSoftmaxWarps) regs_dec<kRegsProducer>();  // producer warpgroup: TMA, QK, helper, PV warps
  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer (warp-uniform, one elected lane issues)
    if (lane == 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
      if constexpr (PACKED)
        for (int i = 0; i < kBlk / 16; ++i) {
          prefetch_tmap(&seg.k[i]);
          prefetch_tmap(&seg.v[i]);
        }
    }
    __syncwarp();
    uint32_t g = 0;  // K/V block counter over all items of this CTA
    int32_t h, u, qb;
    for (int32_t iter = 0; next_item(iter, h, u, qb); ++iter) {
      const int32_t kt0 = __ldg(p.offs + u), n_kt = __ldg(p.offs + u + 1) - kt0;
      const int32_t n_kv = blocks_per_pass<PACKED>(p, n_kt), steps = passes * n_kv;
      const int qbuf = iter & 1;
      if (iter >= 2) attn_wait(&bar_qfree[qbuf], ((iter >> 1) - 1) & 1);
      mbar_arrive_expect_tx_w(&bar_q[qbuf], S::kTile);
      tma_load_2d_w(smem + S::kQ + qbuf * S::kTile, &tm_q, 0, (h * p.M + u) * p.pitch + qb * kBlk, &bar_q[qbuf]);
      KeyWalk w;
      for (int32_t s = 0, j = 0; s < steps; ++s, ++g) {
        if (j == n_kv) {  // exact / normalised modes stream the keys 2 / 3 times
          j = 0;
          w = KeyWalk{};
        }
        ++j;
        int32_t kt_a, row0, split, nvalid;
        next_block<PACKED>(p, n_kt, w, kt_a, row0, split, nvalid);
        const int32_t krow = (h * p.M + __ldg(p.ids + kt0 + kt_a)) * p.pitch + row0;
        const uint32_t st = g % kStages;
        uint8_t* const ks = smem + S::kK + st * S::kTile;
        uint8_t* const vs = smem + S::kV + st * S::kTile;
        if (g >= (uint32_t)kStages) attn_wait(&bar_kv_empty[st], ((g / kStages) - 1) & 1);
        if (!PACKED || split == kBlk) {
          mbar_arrive_expect_tx_w(&bar_kv_full[st], 2 * S::kTile);
          tma_load_2d_w(ks, &tm_k, 0, krow, &bar_kv_full[st]);
          tma_load_2d_w(vs, &tm_v, 0, krow, &bar_kv_full[st]);
        } else {
          // two segments: rows [row0, tv) of tile kt_a, rows [0, nvalid - split) of tile kt_a + 1
          mbar_arrive_expect_tx_w(&bar_kv_full[st], 2 * nvalid * D);
          tma_load_2d_w(ks, &seg.k[split / 16 - 1], 0, krow, &bar_kv_full[st]);
          tma_load_2d_w(vs, &seg.v[split / 16 - 1], 0, krow, &bar_kv_full[st]);
          if (nvalid > split) {
            const int32_t krow2 = (h * p.M + __ldg(p.ids + kt0 + kt_a + 1)) * p.pitch;
            const int n2 = nvalid - split;
            tma_load_2d_w(ks + split * D, &seg.k[n2 / 16 - 1], 0, krow2, &bar_kv_full[st]);
            tma_load_2d_w(vs + split * D, &seg.v[n2 / 16 - 1], 0, krow2, &bar_kv_full[st]);
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ QK issuer (warp-uniform, one elected lane issues)
    // S(j) = Q K^T into TMEM buffer j % 2, issued as soon as the owners of S(j - 2) have it in registers
    // (s_free); the PVs come from the PV warp.  Descriptors are built once; a K-chunk / stage step only
    // moves the 14-bit start-address field (16-byte units), which never carries out.
    constexpr uint32_t idesc_qk = idesc_f8(128, 128, FMT, FMT, 0);
    constexpr uint64_t kTileU = S::kTile >> 4;
    const uint64_t dq0 = desc_kmajor<D>(smem_u32(smem + S::kQ));
    const uint64_t dk0 = desc_kmajor<D>(smem_u32(smem + S::kK));
    uint32_t g = 0;
    uint32_t qk_st = 0, qk_ph = 0;  // K/V stage + full-barrier phase of the next QK
    int32_t h, u, qb;
    for (int32_t iter = 0; next_item(iter, h, u, qb); ++iter) {
      const int32_t n_kt = __ldg(p.offs + u + 1) - __ldg(p.offs + u);
      const int32_t steps = passes * blocks_per_pass<PACKED>(p, n_kt);
      const int qbuf = iter & 1;
      const uint64_t dq = dq0 + (uint64_t)qbuf * kTileU;
      attn_wait(&bar_q[qbuf], (iter >> 1) & 1);
      tc_fence_after();
      for (int32_t s = 0; s < steps; ++s) {
        const uint32_t gs = g + s;
        attn_wait(&bar_kv_full[qk_st], qk_ph);
        if (gs >= 2) attn_wait(&bar_s_free[gs & 1], ((gs - 2) >> 1) & 1);  // S(gs - 2) is in registers
        tc_fence_after();
        // N = 128 for every block: a tile's last block reads zero K rows past tv (S = 0 there, finite),
        // which the softmax drops; below N = 256 an MMA costs the same at any N
#ifndef FPSA_NO_MMA
        qk_mma<D>(tm_s(gs), dq, dk0 + qk_st * kTileU, idesc_qk);
#endif
        mma_commit_w(&bar_s_full[gs % kSF]);
        if (s + 1 == steps) mma_commit_w(&bar_qfree[qbuf]);  // the item's last QK has read Q
        if (++qk_st == kStages) {
          qk_st = 0;
          qk_ph ^= 1;
        }
      }
      g += steps;
    }
  } else if (warp == kPvWarp) {
    // ------------------------------------------------------------ PV issuer (split issue)
    constexpr uint32_t idesc_pv = idesc_f8(128, D + 16, FPSA_E4M3, FMT, 1);
    constexpr uint64_t kTileU = S::kTile >> 4;
    constexpr uint64_t kVStageStep = kTileU - (kTileU << 16);
    constexpr uint64_t kVk = 32 * D / 16;
    const uint32_t sv0 = smem_u32(smem + S::kV);
    const uint64_t dv0 = desc_mnmajor_ones<D>(sv0, smem_u32(smem + S::kOnes) - sv0);
    const uint64_t dvt0 = desc_mnmajor_ones<D>(sv0, smem_u32(smem + S::kOnesTail) - sv0);
    uint32_t g = 0, pv_st = 0;
    int32_t h, u, qb;
    for (int32_t iter = 0; next_item(iter, h, u, qb); ++iter) {
      const int32_t n_kt = __ldg(p.offs + u + 1) - __ldg(p.offs + u);
      const int32_t n_kv = blocks_per_pass<PACKED>(p, n_kt), steps = passes * n_kv;
      const int32_t pv0 = (passes - 1) * n_kv;
      int32_t bp = 0;
      for (int32_t s = 0; s < steps; ++s) {
        const uint32_t gs = g + s;
        const uint64_t dv = (!PACKED && bp == p.nb - 1 ? dvt0 : dv0) + pv_st * kVStageStep;
        if (s == pv0 && iter > 0) attn_wait(&bar_ofree, (iter - 1) & 1);  // the previous item's epilogue read O
        FPSA_TL(9, 0, gs);
        p_wait(gs);
        FPSA_TL(9, 1, gs);
        tc_fence_after();
        const uint32_t tp = tm_p(gs);
#ifndef FPSA_NO_MMA
        if (s >= pv0)
          mma_f8_ts_x4_w(tm_o, tp, tp + 8, tp + 16, tp + 24, dv, dv + kVk, dv + 2 * kVk, dv + 3 * kVk, idesc_pv,
                         s > pv0 ? 1u : 0u);
#endif
        FPSA_TL(9, 2, gs);
        mma_commit_w(&bar_kv_empty[pv_st]);  // K(j) was read by QK(j), complete before S(j) was seen full
        mma_commit_w(&bar_p_free[gs % kParts]);
        FPSA_TL(9, 3, gs);
        if (++pv_st == kStages) pv_st = 0;
        if (++bp == p.nb) bp = 0;
      }
      mma_commit_w(&bar_o);
      g += steps;
    }
  } else if (warp == kHelperWarp) {
    // ------------------------------------------------------------ metadata prefetch (one item ahead)
    const float sl = p.softmax_log2;
    for (int32_t iter = 0;; ++iter) {
      // claim the next item and post it to the ring (the claim's latency is hidden: the ring runs ahead)
      const int r = iter % kItemRing;
      if (iter >= kItemRing) attn_wait(&bar_item_empty[r], ((iter / kItemRing) - 1) & 1);
      int32_t idx = 0;
      if (lane == 0) idx = atomicAdd(p.claim, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      const bool more = idx < count;
      const int32_t h = more ? item_at(3 * idx) : -1;
      const int32_t u = more ? item_at(3 * idx + 1) : 0;
      if (lane == 0) {
        s_item[r][0] = h;
        s_item[r][1] = u;
        s_item[r][2] = more ? item_at(3 * idx + 2) : 0;
        mbar_arrive(&bar_item_full[r]);  // release: the item words above are visible to waiters
      }
      if (!more) break;
      const int slot = iter & 1;
      if (iter >= 2) attn_wait(&bar_meta_empty[slot], ((iter >> 1) - 1) & 1);
      const int32_t kt0 = __ldg(p.offs + u), n_kt = __ldg(p.offs + u + 1) - kt0;
      const float qs = (float)__ldg(p.q_scales + h * p.M + u);
      const double* ks = p.k_scales + (int64_t)h * p.M;
      // c(kt) = f32(f32(sq) * f32(sk)) * f32(scale log2 e), the oracle's factor order; normalised-P mode:
      // the reference's f32(f32(sk) * f32(f32(sq) * scale)) (attention.py:122)
      const float qsc = qs * p.softmax_scale;
      for (int32_t i = lane; i < min(n_kt, kFacCap); i += 32) {
        const float kf = (float)__ldg(ks + __ldg(p.ids + kt0 + i));
        s_fac[slot][i] = NORM ? kf * qsc : (qs * kf) * sl;
      }
      // v factors: f32(sv), or f32(sv / 448) in normalised-P mode (attention.py:206-207)
      for (int i = lane; i < D; i += 32) {
        const double sv = __ldg(p.v_scales + (int64_t)h * D + i);
        s_vsc[slot][i] = NORM ? (float)(sv * (1.0 / 448.0)) : (float)sv;
      }
      if (lane == 0) {
        s_hdr[slot][0] = kt0;
        s_hdr[slot][1] = n_kt;
      }
      mbar_arrive(&bar_meta_full[slot]);  // release: this lane's writes above are visible to waiters
    }
  } else if (warp < kSoftmaxWarps) {
    regs_inc<kRegsSoftmax>();
    // ------------------------------------------------------------ softmax: (row, column part)
    const int quarter = warp & 3;
    const int part = warp >> 2;              // owns the steps j with j % 2 == part
    const int row = quarter * 32 + lane;     // TMEM lane = row of the query block
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t o_addr = tm_o + lane_off + part * (D / kEpiParts);
    const float sl = p.softmax_log2;
    auto row_sync = [&]() {
#ifdef FPSA_WATCH
      volatile int* w = g_watch + (blockIdx.x * 16 + warp) * 4;
      if (lane == 0) { w[0] = -1; __threadfence_system(); }
#endif
      named_bar_sync(1 + quarter, 32 * kParts);
#ifdef FPSA_WATCH
      if (lane == 0) { w[0] = 0; __threadfence_system(); }
#endif
    };
    auto row_max = [&](float m) {  // max over all parts of the row
      s_xchg[part][row] = m;
      row_sync();
      float r = s_xchg[0][row];
#pragma unroll
      for (int i = 1; i < kParts; ++i) r = fmaxf(r, s_xchg[i][row]);
      row_sync();  // the exchange slots are reused
      return r;
    };
    uint32_t g = 0;
#ifdef FPSA_TRACE
    long long w_s = 0, w_c = 0, t_loop = 0;
    int64_t n_steps = 0;
#endif
    int32_t h, u, qb;
    for (int32_t iter = 0; next_item(iter, h, u, qb); ++iter) {
      const int slot = iter & 1;
      attn_wait(&bar_meta_full[slot], (iter >> 1) & 1);
      const int32_t kt0 = s_hdr[slot][0], n_kt = s_hdr[slot][1];
      const int32_t n_kv = blocks_per_pass<PACKED>(p, n_kt);
      const float* fac = s_fac[slot];
      auto factor_at = [&](int32_t kt) {
        if (kt < kFacCap) return fac[kt];
        const float qs = (float)__ldg(p.q_scales + h * p.M + u);  // windows beyond kFacCap tiles: from L2
        const float kf = (float)__ldg(p.k_scales + (int64_t)h * p.M + __ldg(p.ids + kt0 + kt));
        return NORM ? kf * (qs * p.softmax_scale) : (qs * kf) * sl;
      };
      float m_ref = 0.0f;
      uint32_t sat = 0u;
#ifdef FPSA_TRACE
      const long long tl0 = clock64();
#endif
      {
        // ping-pong: this warp computes the whole 128-key rows of its lane quarter for the steps with
        // g % 2 == part (S buffer g % 2 == part), the other warp of the SMSP the other steps, so one
        // warp's TMEM load / store and hand-off latency overlaps the other's exp work
        const uint32_t s_row = tm_s((uint32_t)part) + lane_off;
        auto owned = [&](uint32_t gg) { return (int)(gg % (uint32_t)kParts) == part; };
        // first block of a pass starting at step counter gg that this warp owns (then every second one)
        auto first_owned = [&](uint32_t gg) {
          return (int32_t)(((uint32_t)part + (uint32_t)kParts - gg % (uint32_t)kParts) % (uint32_t)kParts);
        };
        // factors of a block's two key tiles: keys < split from tile kt_a, the rest from kt_a + 1
        auto factors = [&](int32_t kt_a, int32_t split, int32_t nvalid, float& ca, float& cb) {
          ca = factor_at(kt_a);
          cb = nvalid > split ? factor_at(kt_a + 1) : ca;
        };
        float l_norm = 1.0f;  // normalised-P mode: f32 of the f64 row sum
        if (NORM || p.exact) {
          // pass 0 (exact and normalised modes): running max over this warp's key blocks, then over the pair
          float m_acc = -INFINITY;
          for (int32_t j = first_owned(g); j < n_kv; j += kParts) {
            const uint32_t gj = g + j;
            int32_t kt_a, split, nvalid;
            block_at<PACKED>(p, n_kt, j, kt_a, split, nvalid);
            float ca, cb;
            factors(kt_a, split, nvalid, ca, cb);
            sf_wait(gj);
            tc_fence_after();
            m_acc = fmaxf(m_acc, block_max_split(s_row, split, nvalid, ca, cb));
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(&bar_s_free[gj & 1]);
              p_free_wait(gj);
              p_arrive(gj);  // S consumed
            }
          }
          g += n_kv;
          m_ref = row_max(m_acc);
          if constexpr (NORM) {
            // pass 1: l = sum exp(s - m) in f64 over this warp's blocks, then over the pair
            double l_acc = 0.0;
            for (int32_t j = first_owned(g); j < n_kv; j += kParts) {
              const uint32_t gj = g + j;
              int32_t kt_a, split, nvalid;
              block_at<PACKED>(p, n_kt, j, kt_a, split, nvalid);
              float ca, cb;
              factors(kt_a, split, nvalid, ca, cb);
              sf_wait(gj);
              tc_fence_after();
#pragma unroll
              for (int hb = 0; hb < 2; ++hb) {
                uint32_t sreg[64];
                load_s_all<64>(s_row + 64 * hb, sreg);
                tmem_wait_ld();
                l_acc += expsum_norm<64>(sreg, split - 64 * hb, nvalid - 64 * hb, ca, cb, m_ref);
              }
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                mbar_arrive(&bar_s_free[gj & 1]);
                p_free_wait(gj);
                p_arrive(gj);  // S consumed
              }
            }
            g += n_kv;
            s_xchg_d[part][row] = l_acc;
            row_sync();
            double l_row = s_xchg_d[0][row];
#pragma unroll
            for (int i = 1; i < kParts; ++i) l_row += s_xchg_d[i][row];
            row_sync();
            l_norm = (float)l_row;  // f32(denominator), attention.py:137-138
          }
        } else {
          // reference max = row max of the item's first key block, taken by the warp that owns it
          float m0 = -INFINITY;
          if (owned(g)) {
            int32_t kt_a, split, nvalid;
            block_at<PACKED>(p, n_kt, 0, kt_a, split, nvalid);
            float ca, cb;
            factors(kt_a, split, nvalid, ca, cb);
            sf_wait(g);
            tc_fence_after();
            m0 = block_max_split(s_row, split, nvalid, ca, cb);
          }
          m_ref = row_max(m0);
        }
        // block geometry and key-tile factors of this warp's next block, computed while the current
        // block's S is loaded (FPSA_GEOM_PREFETCH) instead of between its P~ signal and the next S wait
        int32_t nx_kt = 0, nx_split = 0, nx_nvalid = 0;
        float nx_ca = 0.0f, nx_cb = 0.0f;
        auto geom = [&](int32_t jj) {
          block_at<PACKED>(p, n_kt, jj, nx_kt, nx_split, nx_nvalid);
          factors(nx_kt, nx_split, nx_nvalid, nx_ca, nx_cb);
        };
        if (FPSA_GEOM_PREFETCH && first_owned(g) < n_kv) geom(first_owned(g));
        for (int32_t j = first_owned(g); j < n_kv; j += kParts) {
          const uint32_t g_own = g + j;
          {
            if (!FPSA_GEOM_PREFETCH) geom(j);
            const int32_t kt_a = nx_kt, split = nx_split, nvalid = nx_nvalid;
            const float ca = nx_ca, cb = nx_cb;
            (void)kt_a;
#ifdef FPSA_TRACE
            const long long ts0 = clock64();
#endif
            FPSA_TL(warp, 0, g_own);
            sf_wait(g_own);
            FPSA_TL(warp, 1, g_own);
#ifdef FPSA_TRACE
            w_s += clock64() - ts0;
            const long long tc0 = clock64();
            ++n_steps;
#endif
            tc_fence_after();
            const float bias = kLog2_448 - m_ref - tau;
            uint32_t w[kBlk / 4];
            const bool fast = FPSA_PACK_FASTPATH && PACKED && split == kBlk && nvalid == kBlk;
            // P~ words of one 64-column half (hb) from its S registers
            auto half = [&](int hb, const uint32_t* sreg) {
              if constexpr (NORM) {
                compute_p_norm<64>(sreg, split - 64 * hb, nvalid - 64 * hb, ca, cb, m_ref, l_norm, w + 16 * hb);
              } else if constexpr (!PACKED) {
                // one key tile per block; padding keys need no mask (zero V rows, zero rows of the tail ones atom)
                sat |= compute_p_regs<64>(sreg, hb ? max(nvalid - 64, 0) : min(nvalid, 64), ca, bias, w + 16 * hb);
              } else {
                if (fast)  // a packed block inside one key tile: the per-tile code (no selects, no mask)
                  sat |= compute_p_regs<64>(sreg, 64, ca, bias, w + 16 * hb);
                else
                  sat |= compute_p_regs2<64>(sreg, split - 64 * hb, nvalid - 64 * hb, ca, cb, bias, w + 16 * hb);
              }
            };
            {
              uint32_t sreg[64];
              load_s_all<64>(s_row, sreg);
              if (FPSA_GEOM_PREFETCH && j + kParts < n_kv) geom(j + kParts);
              tmem_wait_ld();
              half(0, sreg);
            }
            {
              // P~(j) goes into P~ buffer j % 2 once PV(j - 2) has read it; the first 64 keys' codes go out
              // while the second half is computed (11.07 -> 11.00 ms)
              if (g_own >= (uint32_t)kParts) attn_wait(&bar_p_free[g_own % kParts], ((g_own / kParts) - 1) & 1);
              tc_fence_after();
              tmem_st16(tm_p(g_own) + lane_off, w);
            }
            {
              uint32_t sreg[64];
              load_s_all<64>(s_row + 64, sreg);
              tmem_wait_ld();
              // S(j) is in registers: its buffer may take S(j+2)
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&bar_s_free[g_own & 1]);
              half(1, sreg);
            }
            tmem_st16(tm_p(g_own) + 16 + lane_off, w + 16);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) p_arrive(g_own);
            FPSA_TL(warp, 3, g_own);
          }
        }
        g += n_kv;
      }
#ifdef FPSA_TRACE
      t_loop += clock64() - tl0;
#endif
      // ---------------------------------------------------------- epilogue
      // parts 0 and 1 read O (D / 2 channels each); a third part has nothing to read
      if (part < kEpiParts) {
      attn_wait(&bar_o, iter & 1);
      tc_fence_after();
      float inv_l = 1.0f;  // normalised-P mode: P~ is already normalised (out = O * v_fac)
      if constexpr (!NORM) {
        uint32_t lw[16];
        tmem_ld16(tm_o + lane_off + D, lw);  // row sum of P~ (the ones columns, all equal)
        tmem_wait_ld();
        inv_l = 1.0f / __uint_as_float(lw[0]);
      }
      const int32_t r = qb * kBlk + row;  // row inside the tile
      int64_t token;
      if (p.natural) {
        const int32_t ut = u / (p.dh * p.dw), uh = (u / p.dw) % p.dh, uw = u % p.dw;
        const int32_t lt = r / (p.sh * p.sw), lh = (r / p.sw) % p.sh, lw = r % p.sw;
        token = ((int64_t)(ut * p.st + lt) * p.gh + (uh * p.sh + lh)) * p.gw + (uw * p.sw + lw);
      } else {
        token = (int64_t)u * p.tv + r;
      }
      const float* vs = s_vsc[slot];
      static_assert(D / kEpiParts >= 16, "each softmax thread stores at least 16 output channels");
#pragma unroll
      for (int cc = 0; cc < D / kEpiParts; cc += 32) {
        const int col = part * (D / kEpiParts) + cc;
        uint32_t o[32];
        if constexpr (D / kEpiParts >= 32) tmem_ld32(o_addr + cc, o);
        else tmem_ld16(o_addr + cc, *reinterpret_cast<uint32_t(*)[16]>(o));
        tmem_wait_ld();
        constexpr int kN = D / kEpiParts >= 32 ? 32 : 16;
        if (r < p.tv) {
          float f[32];
#pragma unroll
          for (int i = 0; i < kN; ++i) f[i] = __uint_as_float(o[i]) * inv_l * vs[col + i];
          if constexpr (OUT == FPSA_F32) {
            float4* dst =
                reinterpret_cast<float4*>(static_cast<float*>(p.out) + token * p.out_ts + h * p.out_hs + col);
#pragma unroll
            for (int i = 0; i < kN / 4; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + token * p.out_ts +
                                                  h * p.out_hs + col);
#pragma unroll
            for (int i = 0; i < kN / 8; ++i) {
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_ofree);
      mbar_arrive(&bar_meta_empty[slot]);  // this item's metadata slot may be refilled
      if (!NORM && !p.exact) {
        // items with a possibly saturated P~ are recomputed exactly by the redo launch
        if (__any_sync(0xffffffffu, sat != 0u) && lane == 0) atomicOr(&s_ovf[iter & 1], 1u);
        named_bar_sync(5, kSoftmaxWarps * 32);
        if (threadIdx.x == 0 && s_ovf[iter & 1]) {
          s_ovf[iter & 1] = 0;
          const int32_t slot = atomicAdd(p.redo, 1);
          p.redo[kRedoHeader + 3 * slot] = h;
          p.redo[kRedoHeader + 3 * slot + 1] = u;
          p.redo[kRedoHeader + 3 * slot + 2] = qb;
#ifdef FPSA_TRACE
          atomicAdd(&g_trace[5], 1ull);
#endif
        }
      }
    }
#ifdef FPSA_TRACE
    if (lane == 0) {
      atomicAdd(&g_trace[0], (unsigned long long)w_s);
      atomicAdd(&g_trace[1], (unsigned long long)t_loop);
      atomicAdd(&g_trace[2], (unsigned long long)w_c);
      atomicAdd(&g_trace[6], (unsigned long long)n_steps);
    }
#endif
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

// Main persistent launch, then the exact-mode launch over the redo list (its CTAs exit at once when the list
// is empty).  Normalised-P mode: one three-pass launch, nothing to redo.  Workspace words 0..2 (redo count,
// the two launches' claim counters) are zeroed first.
template <int D, int FMT, int OUT, bool NORM, bool PACKED>
int launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const SegMaps& seg, AttnParams p,
           cudaStream_t st) {
  auto kern = fpsa_attn_kernel<D, FMT, OUT, NORM, PACKED>;
  constexpr int smem = Smem<D>::kBytes + 1024;
  if (int s = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem, "fpsa_attn_fwd")) return s;
  if (cudaMemsetAsync(p.redo, 0, kRedoHeader * sizeof(int32_t), st) != cudaSuccess)
    return fail(FPSA_ECUDA, std::string("fpsa_attn_fwd workspace reset: ") + cudaGetErrorString(cudaGetLastError()));
  const int grid = std::min(p.n_items, device_sm_count());
  p.exact = 0;
  p.claim = p.redo + 1;
  kern<<<grid, kThreads, smem, st>>>(tq, tk, tv, seg, p);
  if constexpr (!NORM) {
    p.exact = 1;
    p.claim = p.redo + 2;
    kern<<<grid, kThreads, smem, st>>>(tq, tk, tv, seg, p);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FPSA_ECUDA, std::string("fpsa_attn_fwd launch: ") + cudaGetErrorString(e));
  return FPSA_OK;
}

// packed or per-tile key blocks (p.packed, chosen by the host)
template <int D, int FMT, int OUT, bool NORM>
int launch_p(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const SegMaps& seg, AttnParams p,
             cudaStream_t st) {
  if (p.packed) return launch<D, FMT, OUT, NORM, true>(tq, tk, tv, seg, p, st);
  return launch<D, FMT, OUT, NORM, false>(tq, tk, tv, seg, p, st);
}

}  // namespace
}  // namespace fpsa

using namespace fpsa;

extern "C" int fpsa_attn_fwd(const uint8_t* q_codes, const uint8_t* k_codes, const uint8_t* v_codes,
                             const double* q_scales, const double* k_scales, const double* v_scales, int32_t heads,
                             fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, const int32_t* offs,
                             const int32_t* ids, const int32_t* items, int32_t n_items, float softmax_scale, int fmt,
                             float tau_log2, int p_mode, void* out, int out_dtype, int64_t out_token_stride,
                             int64_t out_head_stride, int out_order, void* workspace, int64_t workspace_bytes,
                             void* stream) {
  clear_error();
  if (p_mode != FPSA_P_ONEPASS && p_mode != FPSA_P_NORMALIZED) return fail(FPSA_EINVAL, "p_mode must be 0 or 1");
  const bool norm = p_mode == FPSA_P_NORMALIZED;
  if (norm && out_dtype != FPSA_F32)
    return fail(FPSA_EUNSUPPORTED, "the normalised-P mode writes f32 output (the reference's dtype)");
  fpsa_dims3 td;
  if (int s = fpsa_tile_grid(grid, tile, &td)) return s;
  if (!q_codes || !k_codes || !v_codes || !q_scales || !k_scales || !v_scales || !offs || !ids || !items || !out)
    return fail(FPSA_EINVAL, "null buffer");
  if (d != 64 && d != 128) return fail(FPSA_EUNSUPPORTED, "head dim must be 64 or 128, got " + std::to_string(d));
  const int32_t tv = tile.t * tile.h * tile.w;
  if (tile_pitch < tv || tile_pitch % kBlk) return fail(FPSA_EINVAL, "tile_pitch must be a multiple of 128 >= tile volume");
  if (!(softmax_scale > 0.0f)) return fail(FPSA_EINVAL, "softmax_scale must be > 0");
  if (fmt != FPSA_E4M3 && fmt != FPSA_E5M2) return fail(FPSA_EINVAL, "fmt must be e4m3 or e5m2");
  if (out_dtype != FPSA_F32 && out_dtype != FPSA_BF16) return fail(FPSA_EUNSUPPORTED, "out dtype must be f32 or bf16");
  if (!(tau_log2 >= 0.0f && tau_log2 <= 8.0f)) return fail(FPSA_EINVAL, "tau_log2 must be in [0, 8]");
  if (heads < 1 || n_items < 1) return fail(FPSA_EINVAL, "empty problem");
  int64_t need = 0;
  fpsa_attn_workspace_bytes(n_items, &need);
  if (!workspace || workspace_bytes < need)
    return fail(FPSA_ECAPACITY, "attention workspace must hold " + std::to_string(need) + " bytes");
  const int32_t M = td.t * td.h * td.w;
  const int64_t rows = (int64_t)heads * M * tile_pitch;
  CUtensorMap tq, tk, tvm;
  if (int s = make_code_map(&tq, q_codes, rows, d, kBlk)) return s;
  if (int s = make_code_map(&tk, k_codes, rows, d, kBlk)) return s;
  if (int s = make_code_map(&tvm, v_codes, rows, d, kBlk)) return s;
  SegMaps seg;  // packed key blocks' segments, 16..128 rows
  for (int i = 0; i < kBlk / 16; ++i) {
    if (int s = make_code_map(&seg.k[i], k_codes, rows, d, 16 * (i + 1))) return s;
    if (int s = make_code_map(&seg.v[i], v_codes, rows, d, 16 * (i + 1))) return s;
  }
  AttnParams p{};
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
  p.nb = (tv + kBlk - 1) / kBlk;
  p.n_tail = tv - kBlk * (p.nb - 1);  // valid keys of a tile's last 128-key block
  p.softmax_log2 = softmax_scale * 1.4426950408889634f;
  p.softmax_scale = softmax_scale;
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
  // packed key blocks: needs 16-row segment boundaries and at most two key tiles per 128-key block
  static const bool no_pack = getenv("FPSA_ATTN_NO_PACK") != nullptr;  // measurement switch
  p.packed = !no_pack && tv % 16 == 0 && tv > kBlk && tv % kBlk != 0;
  // magic divisors of the softmax warps' block geometry: exact while (key position) * divisor < 2^32
  // (positions stay below M * tv); 0 selects a plain division
  auto magic = [](uint64_t d, uint64_t bound) -> uint32_t {
    if (d < 2 || bound * d >= (1ull << 32)) return 0u;
    return (uint32_t)(((1ull << 32) + d - 1) / d);
  };
  p.div_tv = magic((uint64_t)tv, (uint64_t)M * tv + kBlk);
  p.div_nb = magic((uint64_t)p.nb, (uint64_t)M * p.nb + 1);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define FPSA_LAUNCH(D_, F_, O_) return launch_p<D_, F_, O_, false>(tq, tk, tvm, seg, p, st)
  if (norm) {  // f32 output only
    if (d == 128) {
      if (fmt == FPSA_E4M3) return launch_p<128, FPSA_E4M3, FPSA_F32, true>(tq, tk, tvm, seg, p, st);
      return launch_p<128, FPSA_E5M2, FPSA_F32, true>(tq, tk, tvm, seg, p, st);
    }
    if (fmt == FPSA_E4M3) return launch_p<64, FPSA_E4M3, FPSA_F32, true>(tq, tk, tvm, seg, p, st);
    return launch_p<64, FPSA_E5M2, FPSA_F32, true>(tq, tk, tvm, seg, p, st);
  }
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

extern "C" int fpsa_attn_workspace_bytes(int32_t n_items, int64_t* bytes) {
  if (!bytes || n_items < 0) return fail(FPSA_EINVAL, "bad arguments");
  *bytes = (int64_t)(kRedoHeader + 3 * (int64_t)n_items) * (int64_t)sizeof(int32_t);
  return FPSA_OK;
}

#ifdef FPSA_TRACE
extern "C" int fpsa_trace_timeline(long long* out) {
  cudaMemcpyFromSymbol(out, fpsa::g_tl, sizeof(fpsa::g_tl));
  return (int)(sizeof(fpsa::g_tl) / sizeof(long long));
}
extern "C" int fpsa_trace_read(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, fpsa::g_trace, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(fpsa::g_trace, z, sizeof z);
  }
  return 0;
}
#endif

#ifdef FPSA_WATCH
extern "C" int fpsa_debug_set_watch(void* p) {
  int* q = static_cast<int*>(p);
  return cudaMemcpyToSymbol(fpsa::g_watch, &q, sizeof(q)) == cudaSuccess ? 0 : 1;
}
#endif
