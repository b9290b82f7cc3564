// K1 / K1b: renormalized separable Gaussian blur (plas.py:64-68, blur.py:7-30).
//
// Arithmetic contract: the reference runs
// SciPy's correlate1d symmetric-kernel loop per line position,
//     acc = in[0] * w0;  for j = h .. 1:  acc += (in[-j] + in[+j]) * w_j
// in fp64 with zero padding, rounding to the array dtype after each axis.
// Every add and multiply below is an explicit __dadd_rn/__dmul_rn so no FMA
// contraction changes the rounding; the result is bit-identical to SciPy.
//
// Layout: grids are (H, W, S) row-major with S >= C channels (rows padded to a
// float4 multiple for the sort).  A "line" is one (column, channel) for the
// axis-0 pass and one (row, channel) for the axis-1 pass.  Each thread owns R
// consecutive outputs of one line and keeps two rolling register windows of
// fp64 inputs (lo = in[i-j], hi = in[i+j]) so every tap costs 2 loads per R
// outputs; the j loop is unrolled by R so the ring indices are static.
#pragma once
#include "common.cuh"

namespace plas {

constexpr int BLUR_R = 8;

struct BlurLevelRef {
  // either a fixed (h, w) or a schedule lookup through ctrl->level
  const Ctrl* ctrl;
  const int* hs;
  const double* weights;
  const long long* woff;
  int h_direct;
  const double* w_direct;
  __device__ __forceinline__ void get(int* h, const double** w) const {
    if (ctrl) {
      int lv = ctrl->level;
      *h = hs[lv];
      *w = weights + woff[lv];
    } else {
      *h = h_direct;
      *w = w_direct;
    }
  }
};

template <typename T>
__device__ __forceinline__ double ld_as_double(const T* p) {
  return (double)__ldg(p);
}

// EPI: 0 = store rounded to Tout; 1 = f32 parity target: fp32(acc) / den32[y, x];
//      2 = fp64 renormalized: acc / den64[y, x]
template <typename Tin, typename Tout, int EPI, int AXIS>
__global__ void __launch_bounds__(256) blur_axis_kernel(const Tin* __restrict__ in,
                                                         Tout* __restrict__ out, int H, int W,
                                                         int C, int S, BlurLevelRef lvl,
                                                         const void* __restrict__ den) {
  constexpr int R = BLUR_R;
  int h;
  const double* w;
  lvl.get(&h, &w);
  const int n = AXIS == 0 ? H : W;
  const long long stride = AXIS == 0 ? (long long)W * S : (long long)S;
  const int nchunks = (n + R - 1) / R;
  const long long inner = AXIS == 0 ? (long long)W * S : (long long)S;
  const long long nouter = AXIS == 0 ? 1 : H;
  const long long total = inner * nchunks * nouter;
  const double w0 = __ldg(w);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long in_idx = t % inner;
    long long rest = t / inner;
    int chunk = (int)(rest % nchunks);
    long long outer = rest / nchunks;
    int c = (int)(in_idx % S);
    if (c >= C) continue;
    long long base = AXIS == 0 ? in_idx : outer * (long long)W * S + in_idx;
    const Tin* line = in + base;
    const int i0 = chunk * R;
    auto v = [&](int i) -> double {
      return (i >= 0 && i < n) ? ld_as_double(line + (long long)i * stride) : 0.0;
    };
    double acc[R], lo[R], hi[R];
#pragma unroll
    for (int k = 0; k < R; k++) {
      acc[k] = __dmul_rn(v(i0 + k), w0);
      lo[k] = v(i0 + k - h);
      hi[k] = v(i0 + k + h);
    }
    // step t: lo value for output k is in[i0+k-h+t] at slot (k+t)%R,
    //         hi value is in[i0+k+h-t] at slot (k-t)%R.
    const int nblk = h / R, rem = h % R;
    for (int b = 0; b < nblk; b++) {
#pragma unroll
      for (int u = 0; u < R; u++) {
        const int tt = b * R + u;
        const double wj = __ldg(w + (h - tt));
#pragma unroll
        for (int k = 0; k < R; k++)
          acc[k] = __dadd_rn(acc[k], __dmul_rn(__dadd_rn(lo[(k + u) % R], hi[(k - u + R) % R]), wj));
        lo[u % R] = v(i0 + R - h + tt);
        hi[(R - 1 - u) % R] = v(i0 + h - tt - 1);
      }
    }
#pragma unroll
    for (int u = 0; u < R; u++) {
      if (u < rem) {
        const int tt = nblk * R + u;
        const double wj = __ldg(w + (h - tt));
#pragma unroll
        for (int k = 0; k < R; k++)
          acc[k] = __dadd_rn(acc[k], __dmul_rn(__dadd_rn(lo[(k + u) % R], hi[(k - u + R) % R]), wj));
        lo[u % R] = v(i0 + R - h + tt);
        hi[(R - 1 - u) % R] = v(i0 + h - tt - 1);
      }
    }
    Tout* oline = out + base;
#pragma unroll
    for (int k = 0; k < R; k++) {
      const int i = i0 + k;
      if (i < n) {
        Tout r;
        if (EPI == 0) {
          r = (Tout)acc[k];
        } else if (EPI == 1) {
          long long cell = AXIS == 0 ? (long long)i * W + in_idx / S : outer * W + i;
          r = (Tout)__fdiv_rn(__double2float_rn(acc[k]), ((const float*)den)[cell]);
        } else {
          long long cell = AXIS == 0 ? (long long)i * W + in_idx / S : outer * W + i;
          r = (Tout)__ddiv_rn(acc[k], ((const double*)den)[cell]);
        }
        oline[(long long)i * stride] = r;
      }
    }
  }
}

// border_weight (blur.py:13-15) of an (H, W) ones plane, exact fp64 fold.
// row_weight[y] = axis-0 fold of the ones column (identical for every x).
__device__ __forceinline__ double border_row_value(int y, int H, int h, const double* __restrict__ w) {
  double a = __dmul_rn(1.0, __ldg(w));
  for (int j = h; j >= 1; j--) {
    double p = __dadd_rn((y - j >= 0) ? 1.0 : 0.0, (y + j < H) ? 1.0 : 0.0);
    a = __dadd_rn(a, __dmul_rn(p, __ldg(w + j)));
  }
  return a;
}

__global__ void border_rows_kernel(double* __restrict__ row_weight, int H, BlurLevelRef lvl) {
  int h;
  const double* w;
  lvl.get(&h, &w);
  for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < H; y += gridDim.x * blockDim.x)
    row_weight[y] = border_row_value(y, H, h, w);
}

// den[y, x] = axis-1 fold of the plane A[y, :] = row_weight[y]; den(y, x) ==
// den(y, W-1-x) so only the left half is folded and mirrored.
__global__ void border_weight_kernel(const double* __restrict__ row_weight, float* __restrict__ den32,
                                     double* __restrict__ den64, int H, int W, BlurLevelRef lvl) {
  int h;
  const double* w;
  lvl.get(&h, &w);
  const int half = (W + 1) / 2;
  const long long total = (long long)H * half;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int y = (int)(t / half), x = (int)(t % half);
    double a = row_weight[y];
    double acc = __dmul_rn(a, __ldg(w));
    for (int j = h; j >= 1; j--) {
      double p = __dadd_rn((x - j >= 0) ? a : 0.0, (x + j < W) ? a : 0.0);
      acc = __dadd_rn(acc, __dmul_rn(p, __ldg(w + j)));
    }
    long long c0 = (long long)y * W + x, c1 = (long long)y * W + (W - 1 - x);
    if (den32) {
      float f = __double2float_rn(acc);
      den32[c0] = f;
      den32[c1] = f;
    }
    if (den64) {
      den64[c0] = acc;
      den64[c1] = acc;
    }
  }
}

// The sort only needs den32 = fp32(den).  den(y, x) is A(y) folded along x
// over the in-range taps, which in exact arithmetic is A(y) * B(x) with
// B(x) = sum of the in-range weights.  Both SciPy's fp64 fold and this
// product lie within (2h + 4) 2^-53 A(y) of the exact product (weights sum to
// 1, non-negative terms), so when fp32(p - bound) == fp32(p + bound) the fp32
// value equals fp32 of the reference fold; otherwise the cell is folded
// exactly.  O(H W) instead of O(H W h) -- the border plane is data-independent
// but per level.
// row_weight[y] = A(y) (border_rows_kernel); col_weight[x] = B(x) -- on the
// sort's square grid the same array (B(x) = A(x) up to the fold's rounding,
// which the bound covers).
__global__ void border_weight32_kernel(const double* __restrict__ row_weight, const double* __restrict__ col_weight,
                                       float* __restrict__ den32, int H, int W, BlurLevelRef lvl) {
  int h;
  const double* w;
  lvl.get(&h, &w);
  const double scale = (2.0 * h + 8.0) * 1.1102230246251565e-16 * 2.0;  // x2 safety
  // one row per CTA iteration: no per-element division
  for (int y = blockIdx.x; y < H; y += gridDim.x)
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    const long long t = (long long)y * W + x;
    const double a = row_weight[y];
    const double p = a * col_weight[x];
    const double bnd = scale * a;
    float r = __double2float_rn(p);
    if (__double2float_rn(p - bnd) != __double2float_rn(p + bnd)) {  // exact fold (blur.py:13-15)
      double acc = __dmul_rn(a, __ldg(w));
      for (int j = h; j >= 1; j--)
        acc = __dadd_rn(acc, __dmul_rn(__dadd_rn((x - j >= 0) ? a : 0.0, (x + j < W) ? a : 0.0), __ldg(w + j)));
      r = __double2float_rn(acc);
    }
    den32[t] = r;
  }
}

}  // namespace plas
