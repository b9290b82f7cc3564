// Warp-parallel certified evaluation of one output of the reference's SciPy
// fold (blur.cuh contract):
//     acc_{h+1} = RN(x_i w_0),  acc_j = RN(acc_{j+1} + t_j),  R = acc_1,
//     t_j = RN(RN(x_{i-j} + x_{i+j}) w_j)                       (j = h .. 1)
// The blur tiers call this for the outputs whose fast value could not be
// certified (their error bounds include the FFT's norm-wise bound, large
// against outputs near zero).  Instead of the sequential chain of h dependent
// fp64 adds (~10 us at h ~ 800 on one lane):
//   * the lanes form the terms t_j, bit-identical to SciPy's (lane L takes
//     j = h - L, h - L - 32, ...: consecutive lanes read consecutive samples);
//   * their exact-real sum S = acc_{h+1} + sum t_j is accumulated in
//     double-double (cascaded two-sum per lane, double-double butterfly),
//     error E_dd <= 8 (h + 96)^2 u^2 A, A = |acc_{h+1}| + sum |t_j|;
//   * SciPy's own result R differs from S by its h rounded additions, each off
//     by at most u |acc_j| <= u (A + |R - S|), so |R - S| <= h u A / (1 - h u)
//     (u = 2^-53);
//   * R lies in [S - E, S + E]; if both ends (directed rounding) round to the
//     same fp32 value, that value is fp32(R).
// The bound is ~h u A -- free of the FFT error and of the max|x| proxy of the
// tiers' certificates; the few outputs it leaves uncertain get the tighter
// u sum_j |S_j| bound from a second pass over the partial sums, and only what
// that leaves (outputs within ~1e-15 of an fp32 rounding boundary) takes the
// caller's sequential fold.  Returns whether *out holds fp32(R).
#pragma once
#include "common.cuh"

namespace plas {

__device__ __forceinline__ void two_sum(double a, double b, double* s, double* e) {
  const double ss = __dadd_rn(a, b);
  const double bb = __dsub_rn(ss, a);
  *e = __dadd_rn(__dsub_rn(a, __dsub_rn(ss, bb)), __dsub_rn(b, bb));
  *s = ss;
}
// (hi, lo) += (bh, bl), double-double
__device__ __forceinline__ void dd_add(double* hi, double* lo, double bh, double bl) {
  double s, e;
  two_sum(*hi, bh, &s, &e);
  e = __dadd_rn(e, __dadd_rn(*lo, bl));
  two_sum(s, e, hi, lo);
}

// X(k): sample k of the line, 0 outside it (the caller's padding rule).
// All 32 lanes call it with the same (i, h, w); the result is valid in every lane.
template <typename Load>
__device__ __forceinline__ bool fold_certified_warp(const Load& X, int i, int h, const double* __restrict__ w,
                                                    float* out) {
  const int lane = threadIdx.x & 31;
  const double u = 1.1102230246251565e-16;  // 2^-53
  const double acc0 = __dmul_rn((double)X(i), __ldg(w));
  // U taps per batch with every load issued first (the samples may come from
  // global memory: one round trip per batch, not per tap)
  constexpr int U = 4;
  double ch = 0.0, cl = 0.0, ca = 0.0;
  for (int j0 = h - lane; j0 >= 1; j0 -= 32 * U) {
    float a[U], b[U];
    double wj[U];
#pragma unroll
    for (int v = 0; v < U; v++) {
      const int j = j0 - 32 * v;
      const bool ok = j >= 1;
      a[v] = ok ? X(i - j) : 0.f;
      b[v] = ok ? X(i + j) : 0.f;
      wj[v] = ok ? __ldg(w + j) : 0.0;
    }
#pragma unroll
    for (int v = 0; v < U; v++) {
      const double t = __dmul_rn(__dadd_rn((double)a[v], (double)b[v]), wj[v]);
      double s, e;
      two_sum(ch, t, &s, &e);
      ch = s;
      cl = __dadd_rn(cl, e);
      ca = __dadd_rn(ca, fabs(t));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ph = __shfl_xor_sync(PLAS_FULL_MASK, ch, o), pl = __shfl_xor_sync(PLAS_FULL_MASK, cl, o);
    dd_add(&ch, &cl, ph, pl);
    ca += __shfl_xor_sync(PLAS_FULL_MASK, ca, o);
  }
  // every lane holds an accurate total; lane 0's decides for the warp
  double th = __shfl_sync(PLAS_FULL_MASK, ch, 0), tl = __shfl_sync(PLAS_FULL_MASK, cl, 0);
  ca = __shfl_sync(PLAS_FULL_MASK, ca, 0);
  dd_add(&th, &tl, acc0, 0.0);  // S = acc0 + all terms
  const double hd = (double)h;
  const double A = fabs(acc0) + ca * (1.0 + 4.0 * (hd + 64.0) * u);  // >= |acc0| + sum |t|
  const double delta = (hd * u * A + hd * 4.9406564584124654e-324) * (1.0 + 4.0 * hd * u);
  const double edd = 8.0 * (hd + 96.0) * (hd + 96.0) * u * u * A;
  const double E = (delta + edd) * 1.001 + 1e-300;
  {
    const double lo_end = __dsub_rd(__dadd_rd(th, tl), E);
    const double hi_end = __dadd_ru(__dadd_ru(th, tl), E);
    const float fa = __double2float_rn(lo_end), fb = __double2float_rn(hi_end);
    *out = fa;
    if (fa == fb) return true;
  }
  // Tighter bound on demand: |R - S| <= u sum_j |S_j| / (1 - h u) with S_j the
  // exact partial sums in SciPy's order (cancellation keeps them far below A).
  // Rows of 32 consecutive taps (lane L: j = h - 32 m - L); a warp scan per row
  // gives S_j in fp64 (each within g A of exact), then sum |S_j| over the warp.
  double base = acc0, sa = 0.0;
  for (int j0 = h - lane; j0 + lane >= 1; j0 -= 32) {  // warp-uniform trip count: rows while j0 + lane >= 1
    const bool ok = j0 >= 1;
    const double t = ok ? __dmul_rn(__dadd_rn((double)X(i - j0), (double)X(i + j0)), __ldg(w + j0)) : 0.0;
    double sc = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double p = __shfl_up_sync(PLAS_FULL_MASK, sc, o);
      if (lane >= o) sc = __dadd_rn(sc, p);
    }
    if (ok) sa = __dadd_rn(sa, fabs(__dadd_rn(base, sc)));
    base = __dadd_rn(base, __shfl_sync(PLAS_FULL_MASK, sc, 31));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sa += __shfl_xor_sync(PLAS_FULL_MASK, sa, o);
  sa = __shfl_sync(PLAS_FULL_MASK, sa, 0);
  const double g = (hd + 96.0) * u;  // error of every fp64 partial sum here, relative to A
  const double SA = sa * (1.0 + 2.0 * g) + hd * g * A * 1.01;  // >= sum_j |S_j|
  const double delta2 = (u * SA + hd * 4.9406564584124654e-324) * (1.0 + 4.0 * hd * u);
  const double E2 = (delta2 + edd) * 1.001 + 1e-300;
  const double lo_end = __dsub_rd(__dadd_rd(th, tl), E2);
  const double hi_end = __dadd_ru(__dadd_ru(th, tl), E2);
  const float fa = __double2float_rn(lo_end), fb = __double2float_rn(hi_end);
  *out = fa;
  return fa == fb;
}

// The sequential fold itself (SciPy's order), one lane: the rare fallback.
// (terms in batches of 8 with their loads issued first, then the ordered adds)
template <typename Load>
__device__ __forceinline__ float fold_sequential(const Load& X, int i, int h, const double* __restrict__ w) {
  double acc = __dmul_rn((double)X(i), __ldg(w));
  int j = h;
  for (; j >= 8; j -= 8) {
    float a[8], b[8];
    double wj[8];
#pragma unroll
    for (int v = 0; v < 8; v++) {
      a[v] = X(i - (j - v));
      b[v] = X(i + (j - v));
      wj[v] = __ldg(w + j - v);
    }
#pragma unroll
    for (int v = 0; v < 8; v++) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn((double)a[v], (double)b[v]), wj[v]));
  }
  for (; j >= 1; j--) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn((double)X(i - j), (double)X(i + j)), __ldg(w + j)));
  return __double2float_rn(acc);
}

}  // namespace plas
