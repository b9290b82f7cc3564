// K5: smoothness loss forward/backward (smoothness.py:57-97), fp64 like the
// reference (its tests compare at rtol 1e-12).  The blur passes reuse
// blur_axis_kernel<double, double, ...>; these are the elementwise stages.
#pragma once
#include "common.cuh"

namespace plas {

// centered = plane - plane[0, 0, :]   (smoothness.py:85-86)
__global__ void anchor_center_kernel(const double* __restrict__ plane, double* __restrict__ out,
                                     long long cells, int C) {
  const long long total = cells * C;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int c = (int)(t % C);
    out[t] = __dsub_rn(plane[t], plane[c]);
  }
}

// residual = centered - blurred/den (blurred/den already divided by the blur
// epilogue); per-element Huber values (summed in NumPy's order); upstream u = scale * clip(residual, +-delta)
// (smoothness.py:87-89, huber 41-47, huber_grad 50-54)
__global__ void __launch_bounds__(256) huber_kernel(const double* __restrict__ centered,
                                                   const double* __restrict__ blurred,
                                                   double* __restrict__ u, long long total,
                                                   double delta, double scale, int zero_residual,
                                                   double* __restrict__ hval) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    double r = zero_residual ? 0.0 : __dsub_rn(centered[t], blurred[t]);
    double a = fabs(r);
    double hub = a <= delta ? __dmul_rn(__dmul_rn(0.5, r), r)
                            : __dmul_rn(delta, __dsub_rn(a, __dmul_rn(0.5, delta)));
    hval[t] = hub;
    double cl = r < -delta ? -delta : (r > delta ? delta : r);
    u[t] = __dmul_rn(scale, cl);
  }
}

// v = u / den[cell]  (the transpose of the renormalized blur, smoothness.py:95)
__global__ void div_den_kernel(const double* __restrict__ u, const double* __restrict__ den,
                               double* __restrict__ v, long long cells, int C) {
  const long long total = cells * C;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    v[t] = __ddiv_rn(u[t], den[t / C]);
}

// grad = u - back  (smoothness.py:96)
__global__ void sub_kernel(const double* __restrict__ u, const double* __restrict__ back,
                           double* __restrict__ grad, long long total) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    grad[t] = __dsub_rn(u[t], back[t]);
}

}  // namespace plas

namespace plas {

// ---------------------------------------------------------------------------
// Fused smoothness fwd+bwd for one plane (smoothness.py:57-97) in one kernel:
// a CTA owns a TS x TS tile of cells and, channel group by channel group,
//   c    = plane - plane[0, 0]                on the tile + 2R halo (0 outside)
//   B    = axis1(axis0(c))                    on the tile + R halo
//   Rsd  = c - B / den                        (den = border weight, exact fold)
//   hval = huber(Rsd) on the tile            (summed after in NumPy's order)
//   u    = scale * clip(Rsd), v = u / den     on the tile + R halo (v = 0 outside)
//   grad = u - axis1(axis0(v))                on the tile (grad = u if detached)
// with the same SciPy fold (acc = x0 w0; acc += (x-j + x+j) w_j, j = R..1,
// separate fp64 roundings) and the same divisions / clips as the unfused
// kernels, so the results are identical; one read of the plane and one write
// of the gradient instead of ~10 passes over it.
constexpr int SM_TS = 16;     // tile side (cells)
constexpr int SM_CG = 4;      // channels per group

template <int R>
struct SmoothTile {
  static constexpr int NC = SM_TS + 4 * R;  // c region side
  static constexpr int NB = SM_TS + 2 * R;  // B / v region side
  static constexpr size_t smem_doubles =
      (size_t)NC * NC * SM_CG + (size_t)NB * NC * SM_CG + (size_t)NB * NB * SM_CG + (size_t)NB * NB;
};

template <int R>
__device__ __forceinline__ double fold5(const double* x, int stride, const double* w) {
  // x points at the centre; taps at +-j*stride
  double acc = __dmul_rn(x[0], w[0]);
#pragma unroll
  for (int j = R; j >= 1; j--) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(x[-j * stride], x[j * stride]), w[j]));
  return acc;
}

template <int R>
__global__ void __launch_bounds__(256) smooth_fused_kernel(const double* __restrict__ plane, double* __restrict__ grad,
                                                           int H, int W, int C, const double* __restrict__ wts,
                                                           double delta, double scale, int detach,
                                                           double* __restrict__ hval) {
  using T = SmoothTile<R>;
  constexpr int NC = T::NC, NB = T::NB;
  extern __shared__ double sm[];
  double* cbuf = sm;                                  // [NC][NC][CG]
  double* a0 = cbuf + (size_t)NC * NC * SM_CG;        // [NB][NC][CG] axis0(c); later axis0(v) rows [R, R+TS)
  double* vbuf = a0 + (size_t)NB * NC * SM_CG;        // [NB][NB][CG] u (later v)
  double* den = vbuf + (size_t)NB * NB * SM_CG;       // [NB][NB]
  __shared__ double w[R + 1];
  const int tid = threadIdx.x;
  if (tid <= R) w[tid] = wts[tid];
  const int y0 = blockIdx.y * SM_TS, x0 = blockIdx.x * SM_TS;
  __syncthreads();
  // border weight on the B region (exact fold of a ones plane, blur.py:13-15)
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int by = e / NB, bx = e - by * NB;
    const int y = y0 - R + by, x = x0 - R + bx;
    double d = 1.0;
    if (y >= 0 && y < H && x >= 0 && x < W && R > 0) {
      double a = __dmul_rn(1.0, w[0]);
#pragma unroll
      for (int j = R; j >= 1; j--)
        a = __dadd_rn(a, __dmul_rn(__dadd_rn(y - j >= 0 ? 1.0 : 0.0, y + j < H ? 1.0 : 0.0), w[j]));
      double acc = __dmul_rn(a, w[0]);
#pragma unroll
      for (int j = R; j >= 1; j--)
        acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(x - j >= 0 ? a : 0.0, x + j < W ? a : 0.0), w[j]));
      d = acc;
    }
    den[e] = d;
  }
  for (int c0 = 0; c0 < C; c0 += SM_CG) {
    const int cg = min(SM_CG, C - c0);  // loops cover cg channels; buffers keep the SM_CG stride
    // c on the NC x NC region
    for (int e = tid; e < NC * NC * cg; e += blockDim.x) {
      const int cell = e / cg, ch = e - cell * cg;
      const int cy = cell / NC, cx = cell - cy * NC;
      const int y = y0 - 2 * R + cy, x = x0 - 2 * R + cx;
      double v = 0.0;
      if (y >= 0 && y < H && x >= 0 && x < W)
        v = __dsub_rn(plane[((long long)y * W + x) * C + c0 + ch], plane[c0 + ch]);
      cbuf[cell * SM_CG + ch] = v;
    }
    __syncthreads();
    // axis 0 of c: rows [R, R + NB) of the c region, all NC columns
    for (int e = tid; e < NB * NC * cg; e += blockDim.x) {
      const int cell = e / cg, ch = e - cell * cg;
      const int ry = cell / NC, cx = cell - ry * NC;
      a0[cell * SM_CG + ch] = fold5<R>(cbuf + ((size_t)(ry + R) * NC + cx) * SM_CG + ch, NC * SM_CG, w);
    }
    __syncthreads();
    // axis 1 -> residual, Huber (tile only), u on the NB region
    for (int e = tid; e < NB * NB * cg; e += blockDim.x) {
      const int cell = e / cg, ch = e - cell * cg;
      const int by = cell / NB, bx = cell - by * NB;
      const int y = y0 - R + by, x = x0 - R + bx;
      double u = 0.0;
      if (y >= 0 && y < H && x >= 0 && x < W) {
        const double blurred = __ddiv_rn(fold5<R>(a0 + ((size_t)by * NC + bx + R) * SM_CG + ch, SM_CG, w), den[cell]);
        const double r = R > 0 ? __dsub_rn(cbuf[((size_t)(by + R) * NC + bx + R) * SM_CG + ch], blurred) : 0.0;
        if (by >= R && by < R + SM_TS && bx >= R && bx < R + SM_TS) {
          const double a = fabs(r);
          hval[((long long)y * W + x) * C + c0 + ch] =
              a <= delta ? __dmul_rn(__dmul_rn(0.5, r), r) : __dmul_rn(delta, __dsub_rn(a, __dmul_rn(0.5, delta)));
        }
        const double cl = r < -delta ? -delta : (r > delta ? delta : r);
        u = __dmul_rn(scale, cl);
      }
      vbuf[cell * SM_CG + ch] = u;
    }
    __syncthreads();
    if (detach || R == 0) {
      for (int e = tid; e < SM_TS * SM_TS * cg; e += blockDim.x) {
        const int cell = e / cg, ch = e - cell * cg;
        const int ty = cell / SM_TS, tx = cell - ty * SM_TS;
        const int y = y0 + ty, x = x0 + tx;
        if (y < H && x < W)
          grad[((long long)y * W + x) * C + c0 + ch] = vbuf[((size_t)(ty + R) * NB + tx + R) * SM_CG + ch];
      }
    } else {
      // v = u / den on the NB region (0 outside the grid) into the c buffer (c is dead)
      for (int e = tid; e < NB * NB * cg; e += blockDim.x) {
        const int cell = e / cg, ch = e - cell * cg;
        const int by = cell / NB, bx = cell - by * NB;
        const int y = y0 - R + by, x = x0 - R + bx;
        cbuf[cell * SM_CG + ch] = (y < 0 || y >= H || x < 0 || x >= W)
                                      ? 0.0 : __ddiv_rn(vbuf[cell * SM_CG + ch], den[cell]);
      }
      __syncthreads();
      // axis 0 of v for the tile rows, all NB columns -> a0 [TS][NB][CG]
      for (int e = tid; e < SM_TS * NB * cg; e += blockDim.x) {
        const int cell = e / cg, ch = e - cell * cg;
        const int ty = cell / NB, bx = cell - ty * NB;
        a0[cell * SM_CG + ch] = fold5<R>(cbuf + ((size_t)(ty + R) * NB + bx) * SM_CG + ch, NB * SM_CG, w);
      }
      __syncthreads();
      for (int e = tid; e < SM_TS * SM_TS * cg; e += blockDim.x) {
        const int cell = e / cg, ch = e - cell * cg;
        const int ty = cell / SM_TS, tx = cell - ty * SM_TS;
        const int y = y0 + ty, x = x0 + tx;
        if (y < H && x < W) {
          const double back = fold5<R>(a0 + ((size_t)ty * NB + tx + R) * SM_CG + ch, SM_CG, w);
          grad[((long long)y * W + x) * C + c0 + ch] =
              __dsub_rn(vbuf[((size_t)(ty + R) * NB + tx + R) * SM_CG + ch], back);
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace plas
