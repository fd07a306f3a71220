// Issue-throughput probe of the softmax instruction mix, alone and in pairs, to
// learn which instructions share a pipe on sm_100a.  asm volatile ops on fixed
// inputs (no dependency chains), 32 warps per SM, 148 CTAs.
//   t(mix of A and B) ~ max(tA, tB) -> different pipes;  ~ tA + tB -> same pipe.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 pipe_mix.cu -o pipe_mix
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

enum { EX2, EX2H, FFMA, FFMA2, FADD2, MAX3, CVT8, CVT8H, CVTH, IMAD, FMASAT, HFMA2, LOP3, NKIND };
static const char* kNames[NKIND] = {"ex2.f32",   "ex2.f16x2",       "ffma",          "ffma2 (f32x2)", "fadd2 (f32x2)",
                                    "max3.f32",  "cvt.e4m3x2.f32",  "cvt.e4m3x2.f16x2", "cvt.f16x2.f32", "imad",
                                    "fma.sat",   "hfma2",           "lop3"};

// One op of kind K on chain register r (each op consumes the chain's previous value).
template <int K>
__device__ __forceinline__ void op(uint64_t& r, float a, float b) {
  uint32_t lo = (uint32_t)r, hi = (uint32_t)(r >> 32);
  if constexpr (K == EX2) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(lo));
  } else if constexpr (K == EX2H) {
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(lo));
  } else if constexpr (K == FFMA) {
    asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(lo) : "f"(a), "f"(b));
  } else if constexpr (K == FFMA2) {
    const uint64_t c = ((uint64_t)__float_as_uint(a) << 32) | __float_as_uint(b);
    asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(r) : "l"(c));
    return;
  } else if constexpr (K == FADD2) {
    const uint64_t c = ((uint64_t)__float_as_uint(a) << 32) | __float_as_uint(b);
    asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(r) : "l"(c));
    return;
  } else if constexpr (K == MAX3) {
    asm volatile("max.f32 %0, %0, %1, %2;" : "+r"(lo) : "f"(a), "f"(b));
  } else if constexpr (K == CVT8) {
    // new low half = e4m3x2(a, lo as float), high half kept (F2FP ... PACK_AB_MERGE_C)
    asm volatile("{\n\t.reg .b16 t, l16, h16;\n\t.reg .f32 x;\n\tmov.b32 x, %0;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %1, x;\n\tmov.b32 {l16, h16}, %0;\n\tmov.b32 %0, {t, h16};\n\t}"
                 : "+r"(lo) : "f"(a));
  } else if constexpr (K == CVT8H) {
    asm volatile("{\n\t.reg .b16 t, l16, h16;\n\tcvt.rn.satfinite.e4m3x2.f16x2 t, %0;\n\tmov.b32 {l16, h16}, %0;\n\tmov.b32 %0, {t, h16};\n\t}" : "+r"(lo));
  } else if constexpr (K == CVTH) {
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %0;" : "+r"(lo) : "f"(a));
  } else if constexpr (K == IMAD) {
    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(lo) : "r"(hi | 1u), "r"(__float_as_uint(a)));
  } else if constexpr (K == FMASAT) {
    asm volatile("fma.rn.sat.f32 %0, %0, %1, %2;" : "+r"(lo) : "f"(a), "f"(b));
  } else if constexpr (K == HFMA2) {
    asm volatile("fma.rn.f16x2 %0, %0, %0, %1;" : "+r"(lo) : "r"(hi));
  } else {
    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(lo) : "r"(hi), "r"(__float_as_uint(a)));
  }
  r = ((uint64_t)hi << 32) | lo;
}

template <int A, int B>
__global__ void __launch_bounds__(1024, 1) mix(long long* cycles, uint64_t* sink, int iters) {
  const float a = 0.001f * threadIdx.x, b = 0.5f;
  uint64_t ra[8], rb[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ra[i] = 0x3c003c003f000000ull + threadIdx.x + i;
    rb[i] = 0x3c003c003e000000ull + threadIdx.x + 3 * i;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      op<A>(ra[i], a, b);
      if constexpr (B >= 0) op<B>(rb[i], a, b);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= ra[i] ^ rb[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int A, int B>
double run(long long* d, int iters) {
  static uint64_t* sink = nullptr;
  if (!sink) CK(cudaMalloc(&sink, 148 * 1024 * sizeof(uint64_t)));
  mix<A, B><<<148, 1024>>>(d, sink, 10);
  CK(cudaDeviceSynchronize());
  mix<A, B><<<148, 1024>>>(d, sink, iters);
  CK(cudaDeviceSynchronize());
  long long h[148];
  CK(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  return s / 148.0;
}

template <int K>
double single(long long* d, int iters) {
  const double cyc = run<K, -1>(d, iters);
  const double rate = 1024.0 * 8 * iters / cyc;  // thread-instr per clk per SM
  printf("%-18s %7.1f thread-instr/clk/SM  (%5.2f clk per warp-instr per SMSP)\n", kNames[K], rate, 128.0 / rate);
  return cyc;
}

template <int A, int B>
void pair(long long* d, int iters, double ta, double tb) {
  const double t = run<A, B>(d, iters);
  printf("mix %-16s + %-16s: %6.2f x max, %5.2f x sum  -> %s\n", kNames[A], kNames[B], t / (ta > tb ? ta : tb),
         t / (ta + tb), t / (ta + tb) > 0.85 ? "SAME pipe" : (t / (ta > tb ? ta : tb) < 1.15 ? "separate" : "partial"));
}

int main() {
  long long* d;
  CK(cudaMalloc(&d, 148 * sizeof(long long)));
  const int it = 400;
  double t[NKIND];
  t[EX2] = single<EX2>(d, it);
  t[EX2H] = single<EX2H>(d, it);
  t[FFMA] = single<FFMA>(d, it);
  t[FFMA2] = single<FFMA2>(d, it);
  t[FADD2] = single<FADD2>(d, it);
  t[MAX3] = single<MAX3>(d, it);
  t[CVT8] = single<CVT8>(d, it);
  t[CVT8H] = single<CVT8H>(d, it);
  t[CVTH] = single<CVTH>(d, it);
  t[IMAD] = single<IMAD>(d, it);
  t[FMASAT] = single<FMASAT>(d, it);
  t[HFMA2] = single<HFMA2>(d, it);
  t[LOP3] = single<LOP3>(d, it);
  pair<EX2, CVT8>(d, it, t[EX2], t[CVT8]);
  pair<FFMA2, CVT8>(d, it, t[FFMA2], t[CVT8]);
  pair<EX2, FFMA2>(d, it, t[EX2], t[FFMA2]);
  pair<MAX3, CVT8>(d, it, t[MAX3], t[CVT8]);
  pair<MAX3, FFMA2>(d, it, t[MAX3], t[FFMA2]);
  pair<IMAD, FFMA2>(d, it, t[IMAD], t[FFMA2]);
  pair<IMAD, CVT8>(d, it, t[IMAD], t[CVT8]);
  pair<FADD2, FFMA2>(d, it, t[FADD2], t[FFMA2]);
  pair<FMASAT, FFMA2>(d, it, t[FMASAT], t[FFMA2]);
  pair<FFMA, FFMA2>(d, it, t[FFMA], t[FFMA2]);
  pair<LOP3, FFMA2>(d, it, t[LOP3], t[FFMA2]);
  pair<LOP3, CVT8>(d, it, t[LOP3], t[CVT8]);
  pair<HFMA2, FFMA2>(d, it, t[HFMA2], t[FFMA2]);
  pair<EX2H, CVT8H>(d, it, t[EX2H], t[CVT8H]);
  pair<CVTH, CVT8>(d, it, t[CVTH], t[CVT8]);
  pair<EX2, IMAD>(d, it, t[EX2], t[IMAD]);
  return 0;
}
