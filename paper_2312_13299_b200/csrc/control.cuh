// K4 (device-resident convergence / schedule controller, plas.py:251-274),
// K6 (VAD, metrics.py:25-40), K7 (init gather, plas.py:241-242) and the
// fp64 grid_distance statistic (plas.py:71-84).
#pragma once
#include "common.cuh"

namespace plas {

constexpr int RED_THREADS = 256;

// ---------------------------------------------------------------- init
// feat[i] = fp32(features[idx[i]]) with RN fp64->fp32 rounding; pad channels
// are zeroed; any non-finite feature raises a flag (plas.py:236-237).
template <typename Tin>
__global__ void gather_init_kernel(const Tin* __restrict__ features, const int* __restrict__ idx,
                                   float* __restrict__ feat, long long n, int D, int S,
                                   int* __restrict__ nonfinite) {
  const long long total = n * S;
  int bad = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long i = t / S;
    int d = (int)(t - i * S);
    float v = 0.f;
    if (d < D) {
      Tin x = features[(long long)idx[i] * D + d];
      bad |= !isfinite((double)x);
      v = (float)x;
    }
    feat[t] = v;
  }
  if (__any_sync(PLAS_FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// DEVICE-mode initial permutation: keyed bijection on [0, n)
__global__ void init_perm_device_kernel(int* __restrict__ idx, long long n, unsigned long long key0,
                                        unsigned long long key1) {
  Feistel fe;
  fe.init(key0 ^ (key1 * 0x9E3779B97F4A7C15ull) ^ 0x1417ull, (unsigned)n);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    idx[i] = (int)fe((unsigned)i);
}

__global__ void perm_i64_to_i32_kernel(const long long* __restrict__ in, int* __restrict__ out,
                                       long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (int)in[i];
}

__global__ void perm_i32_to_i64_kernel(const int* __restrict__ in, long long* __restrict__ out,
                                       long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (long long)in[i];
}

// ---------------------------------------------------------------- distance
// partial sums of per-cell fp64 Euclidean distances between feat and target
__global__ void __launch_bounds__(RED_THREADS) distance_kernel(const float* __restrict__ a,
                                                               const float* __restrict__ b,
                                                               long long n, int D, int S,
                                                               double* __restrict__ partials) {
  __shared__ double sh[32];
  double sum = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    const float* pa = a + i * S;
    const float* pb = b + i * S;
    for (int c = 0; c < S; c += 4) {
      float4 x = *reinterpret_cast<const float4*>(pa + c);
      float4 y = *reinterpret_cast<const float4*>(pb + c);
      float xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int e = 0; e < 4; e++)
        if (c + e < D) {
          double df = (double)xs[e] - (double)ys[e];
          s = fma(df, df, s);
        }
    }
    sum += sqrt(s);
  }
  double tot = block_sum<RED_THREADS>(sum, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// fixed-order fp64 reduction of `nparts` partials by one CTA (thread 0 result)
__device__ __forceinline__ double reduce_partials(const double* partials, int nparts, double* sh) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
  return block_sum<RED_THREADS>(s, sh);
}

// ---------------------------------------------------------------- controller
struct Sched {
  const double* radii;
  const int* betas;
  const int* hs;
  long long* level_counts;  // device, per level
  double* trace;            // device, trace_cap
};

__device__ __forceinline__ void set_cond(unsigned long long handle, unsigned v) {
  if (handle) cudaGraphSetConditional((cudaGraphConditionalHandle)handle, v);
}

// prepare the pass about to run (DEVICE mode draws its own offsets)
__device__ __forceinline__ void prepare_device_pass(Ctrl* c) {
  int dy, dx;
  unsigned long long gk;
  device_pass_draws(c, &dy, &dx, &gk);
  set_pass_geometry(c, dy, dx);
}

__global__ void level_begin_kernel(Ctrl* c, Sched s) {
  if (threadIdx.x) return;
  const int lv = c->level;
  c->beta = s.betas[lv];
  c->h = s.hs[lv];
  c->pass = 0;
  c->strikes = 0;
  c->level_done = 0;
}

// level-start distance -> previous (plas.py:256-258); opens the pass loop
__global__ void __launch_bounds__(RED_THREADS) level_start_finalize_kernel(
    Ctrl* c, Sched s, const double* partials, int nparts, long long n, unsigned long long inner) {
  __shared__ double sh[32];
  double tot = reduce_partials(partials, nparts, sh);
  if (threadIdx.x) return;
  double d = tot / (double)n;
  c->previous = d;
  if (c->trace_pos >= c->trace_cap) {
    c->status = 1;
    c->level_done = 1;
    set_cond(inner, 0);
    return;
  }
  s.trace[c->trace_pos++] = d;
  if (c->rng_mode == 1) prepare_device_pass(c);
  set_cond(inner, 1);
}

// after a pass: current, strike logic (plas.py:266-272), next pass geometry
__global__ void __launch_bounds__(RED_THREADS) pass_finalize_kernel(
    Ctrl* c, Sched s, const double* partials, int nparts, long long n, unsigned long long inner) {
  __shared__ double sh[32];
  double tot = reduce_partials(partials, nparts, sh);
  if (threadIdx.x) return;
  const double current = tot / (double)n;
  const double previous = c->previous;
  c->current = current;
  c->reorders++;
  c->pass++;
  if (c->trace_pos >= c->trace_cap) {
    c->status = 1;
    c->level_done = 1;
    set_cond(inner, 0);
    return;
  }
  s.trace[c->trace_pos++] = current;
  if (previous <= 0.0 || (previous - current) / previous < c->threshold)
    c->strikes++;
  else
    c->strikes = 0;
  c->previous = current;
  if (c->strikes >= 2) {
    c->level_done = 1;
    set_cond(inner, 0);
  } else if (c->rng_mode == 1) {
    prepare_device_pass(c);
  }
}

// level bookkeeping (plas.py:273-274); radius decay is the schedule table
__global__ void level_end_kernel(Ctrl* c, Sched s, unsigned long long outer) {
  if (threadIdx.x) return;
  s.level_counts[c->level] = c->pass + 1;
  c->levels_done = c->level + 1;
  c->level++;
  if (c->level >= c->num_levels || c->status) set_cond(outer, 0);
}

// parity mode: host-drawn offsets for the next pass
__global__ void set_pass_kernel(Ctrl* c, int dy, int dx) {
  if (threadIdx.x) return;
  set_pass_geometry(c, dy, dx);
}

// ---------------------------------------------------------------- VAD
// pass 0: sum |g[p,c] - g[q,c]|; pass 1: sum (|.| - mean)^2  (two-pass variance)
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) vad_kernel(const T* __restrict__ g, int H, int W,
                                                          int C, int S, const double* mean_ptr,
                                                          double* __restrict__ partials) {
  __shared__ double sh[32];
  const double mean = mean_ptr ? *mean_ptr : 0.0;
  const bool second = mean_ptr != nullptr;
  double sum = 0.0;
  const long long total = (long long)H * W * C;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long cellc = t / C;
    int c = (int)(t - cellc * C);
    int y = (int)(cellc / W), x = (int)(cellc - (long long)y * W);
    double v = (double)g[cellc * S + c];
    if (y + 1 < H) {
      double e = fabs((double)g[(cellc + W) * S + c] - v);
      if (second) {
        e -= mean;
        e *= e;
      }
      sum += e;
    }
    if (x + 1 < W) {
      double e = fabs((double)g[(cellc + 1) * S + c] - v);
      if (second) {
        e -= mean;
        e *= e;
      }
      sum += e;
    }
  }
  double tot = block_sum<RED_THREADS>(sum, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// out = sum(partials) / count
__global__ void __launch_bounds__(RED_THREADS) mean_finalize_kernel(const double* partials,
                                                                    int nparts, double count,
                                                                    double* out) {
  __shared__ double sh[32];
  double tot = reduce_partials(partials, nparts, sh);
  if (threadIdx.x == 0) *out = tot / count;
}

// ---------------------------------------------------------------- API grid_distance
// fp64 inputs, optional per-channel weights (plas.py:71-84)
__global__ void __launch_bounds__(RED_THREADS) grid_distance_f64_kernel(
    const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ w,
    long long n, int D, double* __restrict__ partials) {
  __shared__ double sh[32];
  double sum = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int d = 0; d < D; d++) {
      double df = a[i * D + d] - b[i * D + d];
      if (w) df = df * w[d];
      s += df * df;
    }
    sum += sqrt(s);
  }
  double tot = block_sum<RED_THREADS>(sum, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

}  // namespace plas
