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
// epilogue); partial Huber sums; upstream u = scale * clip(residual, +-delta)
// (smoothness.py:87-89, huber 41-47, huber_grad 50-54)
__global__ void __launch_bounds__(256) huber_kernel(const double* __restrict__ centered,
                                                   const double* __restrict__ blurred,
                                                   double* __restrict__ u, long long total,
                                                   double delta, double scale, int zero_residual,
                                                   double* __restrict__ partials) {
  __shared__ double sh[32];
  double sum = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    double r = zero_residual ? 0.0 : __dsub_rn(centered[t], blurred[t]);
    double a = fabs(r);
    double hub = a <= delta ? __dmul_rn(__dmul_rn(0.5, r), r)
                            : __dmul_rn(delta, __dsub_rn(a, __dmul_rn(0.5, delta)));
    sum += hub;
    double cl = r < -delta ? -delta : (r > delta ? delta : r);
    u[t] = __dmul_rn(scale, cl);
  }
  double tot = block_sum<256>(sum, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
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
