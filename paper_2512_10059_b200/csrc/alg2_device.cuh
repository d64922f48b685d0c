// alg2_device.cuh -- Algorithm 2 of arXiv 2512.10059 (PAPER.md:353-390,
// SPEC.md:494-502): the fused Boys-and-contraction benchmark
//     z_i = sum_{l=0..k} c_l sum_j F_l(x_i + x_j) y_j
// evaluated on the B200 without storing a single Boys value.
//
// The O(N^2) pair sweep is FP64-bound, so the design goal is zero wasted FP64
// work:
//   * x is sorted once (CUB radix sort, with y carried along); a warp then
//     holds 32 neighbouring x_i, and for one x_j the 32 sums x_i + x_j almost
//     always fall in the same region -- the A/B/C branches are warp-uniform
//     without any per-pair binning;
//   * blocks stage tiles of (x_j, e^{-x_j}, y_j) in shared memory (broadcast
//     reads); each thread owns one x_i and accumulates z_i in a register;
//   * per pair, F_0..F_k are produced by the same recurrences as the bulk kernel
//     (boys_device.cuh) but folded into w = sum_l c_l F_l on the fly, so F never
//     exists as an array; e^{-(x_i+x_j)} = e^{-x_i} e^{-x_j} replaces one exp
//     per pair by one multiply, and the B/C seeds use Newton-refined
//     reciprocal / inverse square root instead of IEEE division and sqrt (a few
//     ulp instead of correctly rounded; the benchmark's contract is agreement
//     with the direct sum within N k 1e-12 relative).
#pragma once

#include "boys_device.cuh"

namespace boysfn_dev {

constexpr int kAlg2Threads = 128;  // x_i per block
constexpr int kAlg2TileJ = 256;    // x_j per shared-memory tile

struct Alg2Coef {
  double c[kMaxCoef + 16];  // c_0..c_k, k <= 32
};

#ifdef __CUDACC__

// 1/b for a normal positive b: rcp.approx (MUFU.RCP64H) + two Newton steps.
__device__ __forceinline__ double rcp_normal(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = __fma_rn(-b, r, 1.0);
  e = __fma_rn(e, e, e);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-b, r, 1.0);
  return __fma_rn(r, e, r);
}

// 1/sqrt(s) for a normal positive s: rsqrt.approx (MUFU.RSQ64H, ~2^-22) + two
// Newton steps (error ~1.5 e^2 per step).
__device__ __forceinline__ double rsqrt_normal(double s) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double h = 0.5 * s;
  y = __fma_rn(y, __fma_rn(-h * y, y, 0.5), y);
  y = __fma_rn(y, __fma_rn(-h * y, y, 0.5), y);
  return y;
}

// w = sum_l c_l F_l(s) for one argument s, given e = e^{-s}.
template <int K, int NA, int MA, int NB, int MB>
__device__ __forceinline__ double boys_dot(const EvalParams& P, const Alg2Coef& C, double s, double e) {
  if (s < P.x0) {  // region A: seed F_K, downward (eval.cpp:38-47)
    double F = rational<NA, MA>(P.numA, P.denA, s);
    double w = C.c[K] * F;
    const double twos = s + s;
#pragma unroll
    for (int l = K - 1; l >= 0; --l) {
      const double t = __fma_rn(twos, F, e);
      F = (l == 0) ? t : __dmul_rn(t, recip_odd(l));
      w = __fma_rn(C.c[l], F, w);
    }
    return w;
  }
  // regions B and C: seed F_0, upward (eval.cpp:49-57, 73-77).  The pair sum is
  // a normal positive double here, so the branch-free reciprocal / inverse
  // square root (<= 2 ulp) replace the IEEE division and square root.
  double F, tail, inv2s;
  if (s < P.x1) {
    inv2s = 0.5 * rcp_normal(s);
    F = rational<NB, MB>(P.numB, P.denB, s);
    tail = -__dmul_rn(e, inv2s);
  } else {
    const double y = rsqrt_normal(s);
    F = kHalfSqrtPi * y;
    inv2s = 0.5 * (y * y);
    tail = -0.0;
  }
  double w = C.c[0] * F;
#pragma unroll
  for (int l = 0; l < K; ++l) {
    F = __fma_rn(__dmul_rn(static_cast<double>(2 * l + 1), inv2s), F, tail);
    w = __fma_rn(C.c[l + 1], F, w);
  }
  return w;
}

// Persistent pair kernel.  Work items are (i-block of kAlg2Threads sorted x_i,
// j-segment of seg_len x_j); blocks claim items from a counter until none are
// left, so the last wave is item-sized, not block-sized (a grid of one block
// per i-block left 3.46 waves at N = 2^19: the last 46% full).  Each thread
// owns one x_i, streams its segment's x_j through shared memory in tiles of
// kAlg2TileJ, and writes its partial sum to partial[seg * n + i]; the segments
// are added in order by the scatter kernel (deterministic).
// xs sorted ascending, es = e^{-xs}, ys carried along.
template <int K, int NA, int MA, int NB, int MB>
__global__ void __launch_bounds__(kAlg2Threads)
    boys_alg2_kernel(const __grid_constant__ EvalParams P, const __grid_constant__ Alg2Coef C,
                     const double* __restrict__ xs, const double* __restrict__ es,
                     const double* __restrict__ ys, size_t n, int nseg, size_t seg_len,
                     unsigned long long* __restrict__ counter, double* __restrict__ partial) {
  __shared__ double sx[kAlg2TileJ], se[kAlg2TileJ], sy[kAlg2TileJ];
  __shared__ unsigned long long s_item;
  const int tid = threadIdx.x;
  const size_t nib = (n + kAlg2Threads - 1) / kAlg2Threads;
  const unsigned long long items = static_cast<unsigned long long>(nib) * nseg;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(counter, 1ull);
    __syncthreads();
    const unsigned long long item = s_item;
    __syncthreads();  // everyone has read s_item before the next claim overwrites it
    if (item >= items) break;
    const size_t ib = static_cast<size_t>(item / nseg);
    const int seg = static_cast<int>(item % nseg);
    const size_t i = ib * kAlg2Threads + tid;
    const double xi = i < n ? xs[i] : 0.0;
    const double ei = i < n ? es[i] : 1.0;
    const size_t jb = static_cast<size_t>(seg) * seg_len;
    const size_t je = jb + seg_len < n ? jb + seg_len : n;
    double acc0 = 0.0, acc1 = 0.0;
    for (size_t j0 = jb; j0 < je; j0 += kAlg2TileJ) {
#pragma unroll
      for (int r = 0; r < kAlg2TileJ / kAlg2Threads; ++r) {
        const size_t j = j0 + r * kAlg2Threads + tid;
        const bool ok = j < je;
        sx[r * kAlg2Threads + tid] = ok ? xs[j] : 0.0;
        se[r * kAlg2Threads + tid] = ok ? es[j] : 1.0;
        sy[r * kAlg2Threads + tid] = ok ? ys[j] : 0.0;  // padding contributes y = 0
      }
      __syncthreads();
#pragma unroll 2
      for (int jj = 0; jj < kAlg2TileJ; jj += 2) {  // two independent pair chains per step
        const double w0 = boys_dot<K, NA, MA, NB, MB>(P, C, xi + sx[jj], __dmul_rn(ei, se[jj]));
        const double w1 = boys_dot<K, NA, MA, NB, MB>(P, C, xi + sx[jj + 1], __dmul_rn(ei, se[jj + 1]));
        acc0 = __fma_rn(sy[jj], w0, acc0);
        acc1 = __fma_rn(sy[jj + 1], w1, acc1);
      }
      __syncthreads();
    }
    if (i < n) partial[static_cast<size_t>(seg) * n + i] = acc0 + acc1;
  }
}

#endif  // __CUDACC__

}  // namespace boysfn_dev
