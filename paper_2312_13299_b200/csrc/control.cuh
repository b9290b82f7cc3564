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

// f32 working copy of the features in element order (sharding: rows of
// other ranks' moved elements are re-read from it)
template <typename Tin>
__global__ void orig32_kernel(const Tin* __restrict__ features, float* __restrict__ out, long long n, int D, int S) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * S; t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / S;
    const int d = (int)(t - i * S);
    out[t] = d < D ? (float)features[i * D + d] : 0.f;
  }
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
// Per-cell squared distance in fp64 with a fixed evaluation order shared with
// the pass kernel (assign.cuh dist_accum): chunk c (4 channels) extends the
// sequential fma chain p[c % 4]; the cell's value is ((p0 + p1) + (p2 + p3)).
// grid_distance (plas.py:71-84) is order-free in fp64.
__device__ __forceinline__ double cell_dist2(const float* __restrict__ a, const float* __restrict__ b,
                                             int D, int S) {
  double p[4] = {0.0, 0.0, 0.0, 0.0};
  for (int c = 0; c < (S >> 2); c++) {
    const float4 x = *reinterpret_cast<const float4*>(a + 4 * c);
    const float4 y = *reinterpret_cast<const float4*>(b + 4 * c);
    const float xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
    double acc = p[c & 3];
#pragma unroll
    for (int e = 0; e < 4; e++)
      if (4 * c + e < D) {
        const double df = (double)xs[e] - (double)ys[e];
        acc = fma(df, df, acc);
      }
    p[c & 3] = acc;
  }
  return (p[0] + p[1]) + (p[2] + p[3]);
}

// cell_dist2 for rows of exactly NCH float4 chunks with every load issued
// before the first use (same evaluation order, same value).
template <int NCH>
__device__ __forceinline__ double cell_dist2_fixed(const float* __restrict__ a, const float* __restrict__ b, int D) {
  float4 x[NCH], y[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    x[c] = __ldg(reinterpret_cast<const float4*>(a) + c);
    y[c] = __ldg(reinterpret_cast<const float4*>(b) + c);
  }
  double p[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    const float xs[4] = {x[c].x, x[c].y, x[c].z, x[c].w}, ys[4] = {y[c].x, y[c].y, y[c].z, y[c].w};
    double acc = p[c & 3];
#pragma unroll
    for (int e = 0; e < 4; e++)
      if (4 * c + e < D) {
        const double df = (double)xs[e] - (double)ys[e];
        acc = fma(df, df, acc);
      }
    p[c & 3] = acc;
  }
  return (p[0] + p[1]) + (p[2] + p[3]);
}

__device__ __forceinline__ double cell_dist2_any(const float* a, const float* b, int D, int S) {
  switch (S) {
    case 4: return cell_dist2_fixed<1>(a, b, D);
    case 8: return cell_dist2_fixed<2>(a, b, D);
    case 12: return cell_dist2_fixed<3>(a, b, D);
    case 16: return cell_dist2_fixed<4>(a, b, D);
    default: return cell_dist2(a, b, D, S);
  }
}

// cell_dist2 for 16-float rows with all eight loads issued first (same order,
// same value): the level-start statistic streams every row once
__device__ __forceinline__ double cell_dist2_s16(const float* __restrict__ a, const float* __restrict__ b, int D) {
  float4 x[4], y[4];
#pragma unroll
  for (int c = 0; c < 4; c++) {
    x[c] = __ldg(reinterpret_cast<const float4*>(a) + c);
    y[c] = __ldg(reinterpret_cast<const float4*>(b) + c);
  }
  double p[4];
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const float xs[4] = {x[c].x, x[c].y, x[c].z, x[c].w}, ys[4] = {y[c].x, y[c].y, y[c].z, y[c].w};
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < 4; e++)
      if (4 * c + e < D) {
        const double df = (double)xs[e] - (double)ys[e];
        acc = fma(df, df, acc);
      }
    p[c] = acc;
  }
  return (p[0] + p[1]) + (p[2] + p[3]);
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

// Prepare the pass about to run (DEVICE mode draws its own offsets).  Called
// by all threads of one CTA: thread 0 draws and lays out the pass, threads
// 0..8 derive the nine block-class Feistel keys in parallel.
// (the class keys are not kept in Ctrl: the grouping tables are built from the
// level's pass records, gen_class_tables, so the controller tail only sets
// the next pass's geometry)
__device__ __forceinline__ void prepare_device_pass_cta(Ctrl* c, unsigned long long* s_gkey) {
  if (threadIdx.x == 0) {
    int dy, dx;
    unsigned long long gk;
    device_pass_draws(c, &dy, &dx, &gk);
    set_pass_geometry_base(c, dy, dx);
    *s_gkey = gk;
  }
  __syncthreads();
}

// serial version (host-stepped DEVICE mode launches it as its own kernel)
__device__ __forceinline__ void prepare_device_pass(Ctrl* c) {
  int dy, dx;
  unsigned long long gk;
  device_pass_draws(c, &dy, &dx, &gk);
  set_pass_geometry(c, dy, dx, gk);
}

__device__ __host__ __forceinline__ bool level_uses_fft(int h, int side, int fft_min_h, int fft_L) {
  return fft_min_h > 0 && fft_L > 0 && h >= fft_min_h && side + h <= fft_L;
}

// DEVICE mode, level start: every pass's draws of this level (stateless in
// (level, pass)), so no kernel on the per-pass critical path runs Philox.
// item t = (pass p = t / 16, item t % 16) of the level's draw records: item 9
// stores the pass's draws, items 0..8 the class shapes and Feistel keys
__device__ __forceinline__ void pass_draw_item(const Ctrl* c, int level, int beta, int side, int t,
                                               int4* __restrict__ pdraw, int* __restrict__ prec) {
  const int p = t >> 4, item = t & 15;
  if (item > 9) return;
  int dy, dx;
  unsigned long long gk;
  device_pass_draws_at(c, level, p, beta, &dy, &dx, &gk);
  if (item == 9) {
    pdraw[p] = make_int4(dy, dx, (int)(unsigned)gk, (int)(unsigned)(gk >> 32));
    return;
  }
  // class `item`: its shape (set_pass_geometry_base) and keys (set_class_keys)
  const int cls = item, ty = cls / 3, tx = cls % 3;
  const int fy = dy > 0 ? dy : beta, fx = dx > 0 ? dx : beta;
  const int nby = num_segments(fy, beta, side), nbx = num_segments(fx, beta, side);
  int lo, hi, hh, ww;
  if (ty == 1) hh = beta;
  else { segment(ty == 0 ? 0 : nby - 1, fy, beta, side, &lo, &hi); hh = hi - lo; }
  if (tx == 1) ww = beta;
  else { segment(tx == 0 ? 0 : nbx - 1, fx, beta, side, &lo, &hi); ww = hi - lo; }
  auto exists = [](int tt, int nn) { return tt == 0 || (tt == 2 && nn >= 2) || (tt == 1 && nn >= 3); };
  const unsigned m = (unsigned)(hh * ww);
  Feistel fe;
  fe.init(class_key(gk, hh, ww), m);
  int* r = prec + (long long)p * PREC_INTS;
  r[cls] = (exists(ty, nby) && exists(tx, nbx)) ? (int)m : 0;
  r[9 + cls] = fe.lbits;
  r[18 + cls] = fe.rbits;
  r[PREC_WW + cls] = ww;
  for (int k = 0; k < 6; k++) r[27 + 6 * cls + k] = (int)fe.keys[k];
}

__global__ void pass_draws_kernel(Ctrl* c, int4* __restrict__ pdraw, int* __restrict__ prec) {
  // one thread per (pass, class) item: every chain is one Philox block plus at
  // most one Feistel key setup
  const int level = c->level;
  const int beta = c->beta, side = c->side;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < PDRAW_MAX * 16; t += gridDim.x * blockDim.x)
    pass_draw_item(c, level, beta, side, t, pdraw, prec);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c->pdraw = pdraw;
    c->prec = prec;
    c->pdraw_level = level;
  }
}

__device__ __host__ __forceinline__ bool level_uses_tile_blur(int h, int side, int fft_min_h, int fft_L,
                                                              int tile_hmax) {
  return !level_uses_fft(h, side, fft_min_h, fft_L) && h <= tile_hmax;
}

__global__ void level_begin_kernel(Ctrl* c, Sched s, unsigned long long blur_cond, unsigned long long tblur_cond,
                                   unsigned long long tile_cond) {
  if (threadIdx.x) return;
  const int lv = c->level;
  c->beta = s.betas[lv];
  c->h = s.hs[lv];
  // fast-division magics of this level's constant cap and of the two possible
  // segment counts (first segment beta or shorter), off the per-pass path
  c->lv_cap = (c->beta * c->beta + 3) / 4;
  make_fastdiv((unsigned)c->lv_cap, &c->lv_cap_m, &c->lv_cap_l);
  c->lv_seg_base = num_segments(c->beta, c->beta, c->side);
  make_fastdiv((unsigned)c->lv_seg_base, &c->lv_seg_m[0], &c->lv_seg_l[0]);
  make_fastdiv((unsigned)(c->lv_seg_base + 1), &c->lv_seg_m[1], &c->lv_seg_l[1]);
  set_cond(blur_cond, level_uses_fft(c->h, c->side, c->fft_min_h, c->fft_L) ? 1u : 0u);
  set_cond(tblur_cond, level_uses_tile_blur(c->h, c->side, c->fft_min_h, c->fft_L, c->tile_blur_hmax) ? 1u : 0u);
  set_cond(tile_cond, use_tile(c->beta, c->S) ? 1u : 0u);  // K3 regime of the whole level (beta is fixed)
  c->pass = 0;
  c->strikes = 0;
  c->level_done = 0;
}

// The controller's serial tail works on a shared-memory copy of Ctrl: one
// coalesced copy in and out instead of a chain of dependent global accesses.
__device__ __forceinline__ void ctrl_to_smem(Ctrl* dst, const Ctrl* src) {
  static_assert(sizeof(Ctrl) % 4 == 0, "Ctrl is copied as 32-bit words");
  const int* s = reinterpret_cast<const int*>(src);
  int* d = reinterpret_cast<int*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / 4); i += blockDim.x) d[i] = s[i];
  __syncthreads();
}
__device__ __forceinline__ void ctrl_from_smem(Ctrl* dst, const Ctrl* src) {
  __syncthreads();
  const int* s = reinterpret_cast<const int*>(src);
  int* d = reinterpret_cast<int*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / 4); i += blockDim.x) d[i] = s[i];
}

// DEVICE mode: the class groupings of pass `pass` of the current level as
// tables tab[cls * stride + l] = Feistel_cls(l), l < m_cls (the keyed
// bijections of common.cuh).  Draws are stateless in (level, pass), so every
// CTA derives the pass's geometry and keys itself and fills its slice of the
// tables; the pass kernel then looks groupings up instead of evaluating the
// Feistel network (and its cycle walk) per lane.  Called by all threads.
// `level`: the level whose pass `pass` the tables are for (-1: cg->level).
// Callers running beside a controller CTA that may rewrite Ctrl (the
// statistics kernels' other CTAs) pass a value that CTA never changes while
// they run (Ctrl.gen_level written by K3, or Ctrl.level read before the
// ticket): the fast/slow path choice below must be CTA-uniform, and the slow
// path must not mix two levels' state.
__device__ __forceinline__ void gen_class_tables(const Ctrl* cg, int pass, int* __restrict__ tab0, long long stride,
                                                 int worker = -1, int nworkers = 0, int level = -1, bool spread = true) {
  if (worker < 0) {
    worker = blockIdx.x;
    nworkers = gridDim.x;
  }
  if (level < 0) level = cg->level;
  int* __restrict__ tab = tab0 + (long long)(pass & 1) * 9 * stride;  // double-buffered by pass parity
  {
    // fast path: the pass's record precomputed at level start (pass_draws_kernel)
    const int* prec = cg->prec;
    const bool ok = prec && cg->pdraw_level == level && pass < PDRAW_MAX;
    if (ok) {
      __shared__ int rec[PREC_INTS];
      for (int i = threadIdx.x; i < PREC_INTS; i += blockDim.x) rec[i] = prec[(long long)pass * PREC_INTS + i];
      __syncthreads();
      int start = 0;  // chunks of the earlier classes: the work is spread over (class, chunk) pairs
      for (int cls = 0; cls < 9; cls++) {
        const unsigned m = (unsigned)rec[cls];
        if (!m) continue;
        Feistel fe;
        fe.init_keys(reinterpret_cast<const unsigned*>(rec + 27 + 6 * cls), rec[9 + cls], rec[18 + cls], m);
        const unsigned ww = (unsigned)rec[PREC_WW + cls];
        const int nch = (int)((m + blockDim.x - 1) / blockDim.x);
        for (int ch = spread ? ((worker - start) % nworkers + nworkers) % nworkers : worker; ch < nch; ch += nworkers) {
          const unsigned l = (unsigned)ch * blockDim.x + threadIdx.x;
          if (l < m) tab[cls * stride + l] = pack_local(fe(l), ww);
        }
        start += nch;
      }
      return;
    }
  }
  __shared__ Ctrl nx;
  __shared__ unsigned long long gk;
  __shared__ int mcls[10];
  ctrl_to_smem(&nx, cg);
  if (threadIdx.x == 0) {
    nx.level = level;
    nx.pass = pass;
    int dy, dx;
    device_pass_draws(&nx, &dy, &dx, &gk);
    set_pass_geometry_base(&nx, dy, dx);
  }
  __syncthreads();
  if (threadIdx.x < 9) {
    set_class_keys(&nx, threadIdx.x, gk);
    // classes that do not exist in this pass get m = 0
    const int ty = threadIdx.x / 3, tx = threadIdx.x % 3;
    auto exists = [](int t, int n) { return t == 0 || (t == 2 && n >= 2) || (t == 1 && n >= 3); };
    mcls[threadIdx.x] = (exists(ty, nx.nby) && exists(tx, nx.nbx)) ? nx.seg_h[ty] * nx.seg_w[tx] : 0;
  }
  __syncthreads();
  int start = 0;
  for (int cls = 0; cls < 9; cls++) {
    const unsigned m = (unsigned)mcls[cls];
    if (!m) continue;
    Feistel fe;
    fe.init_keys(nx.fe_keys[cls], nx.fe_lbits[cls], nx.fe_rbits[cls], m);
    const unsigned ww = (unsigned)nx.seg_w[cls % 3];
    const int nch = (int)((m + blockDim.x - 1) / blockDim.x);
    for (int ch = ((worker - start) % nworkers + nworkers) % nworkers; ch < nch; ch += nworkers) {
      const unsigned l = (unsigned)ch * blockDim.x + threadIdx.x;
      if (l < m) tab[cls * stride + l] = pack_local(fe(l), ww);
    }
    start += nch;
  }
}

// DEVICE mode: tables of the next pass, built concurrently with the pass
// statistics (the graph runs this kernel and pass_stats_kernel in parallel;
// gen_pass was set by the pass kernel, so the controller's update of pass
// does not race with it).
__global__ void __launch_bounds__(256) gen_tables_kernel(const Ctrl* c, int* tab, long long stride) {
  gen_class_tables(c, c->gen_pass, tab, stride, -1, 0, c->gen_level);
}

// Last-CTA-done protocol: every CTA writes its partial, fences and takes a
// ticket; the CTA with the last ticket sees all partials, reduces them in a
// fixed order (deterministic) and runs the controller.  Returns true there.
__device__ __forceinline__ bool last_cta_reduce(double v, double* partials, int* done, double* total,
                                                double* sh, int* ticket = nullptr) {
  __shared__ int s_last, s_ticket;
  const double blk = block_sum<RED_THREADS>(v, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = blk;
    __threadfence();
    s_ticket = atomicAdd(done, 1);
    s_last = s_ticket == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (ticket) *ticket = s_ticket;
  if (!s_last) return false;
  __threadfence();
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += ((volatile double*)partials)[i];
  t = block_sum<RED_THREADS>(t, sh);
  if (threadIdx.x == 0) {
    *total = t;
    *done = 0;
  }
  __syncthreads();
  return true;
}

// Deterministic pass statistic: the moved-cell list comes in atomic
// reservation order, so an fp64 sum over it would depend on the schedule.
// Each cell's change (new - cached distance, computed the same way in every
// schedule) is rounded to a multiple of 2^-64 (fx64) and the changes are
// summed as 128-bit integers -- exact, so any order gives the same total.
__device__ __forceinline__ __int128 fx64(double v) {
  const double t = rint(v * 18446744073709551616.0);  // v 2^64 (exact scaling), rounded to an integer
  const double hi = trunc(t * 9.094947017729282379150390625e-13);  // t 2^-40: |hi| < 2^63 for |v| < 2^87
  const double lo = fma(hi, -1099511627776.0, t);                  // t - hi 2^40, exact: |lo| < 2^40
  return ((__int128)(long long)hi << 40) + (__int128)(long long)lo;
}
__device__ __forceinline__ double fx64_to_double(__int128 q) {
  const long long hi = (long long)(q >> 64);
  const unsigned long long lo = (unsigned long long)q;
  return (double)hi + (double)lo * 5.42101086242752217003726400434970855712890625e-20;  // lo 2^-64
}
__device__ __forceinline__ __int128 shfl_xor_i128(__int128 v, int m) {
  const long long h = __shfl_xor_sync(0xffffffffu, (long long)(v >> 64), m);
  const unsigned long long l = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, m);
  return ((__int128)h << 64) | (__int128)l;
}

// last_cta_reduce for 128-bit fixed-point values: each CTA adds its block sum
// into a 128-bit accumulator acc[0..1] (low word, then high word plus the
// carry its own low-word add produced -- exact modulo 2^128 in any order); the
// last CTA reads it and clears it for the next pass (zeroed at sort start).
__device__ __forceinline__ void store_i128(double* dst, __int128 v) {  // raw bits in two fp64 slots
  reinterpret_cast<unsigned long long*>(dst)[0] = (unsigned long long)v;
  reinterpret_cast<unsigned long long*>(dst)[1] = (unsigned long long)((unsigned __int128)v >> 64);
}
__device__ __forceinline__ __int128 load_i128(const double* src) {
  const unsigned long long lo = reinterpret_cast<const unsigned long long*>(src)[0];
  const unsigned long long hi = reinterpret_cast<const unsigned long long*>(src)[1];
  return (__int128)(((unsigned __int128)hi << 64) | (unsigned __int128)lo);
}
__device__ __forceinline__ bool last_cta_reduce_fx(__int128 v, unsigned long long* acc, int* done, double* total,
                                                   int* ticket, __int128* raw = nullptr) {
  __shared__ __int128 sq[32];
  __shared__ int s_last, s_ticket;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += shfl_xor_i128(v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) sq[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    __int128 b = 0;
    for (int w = 0; w < nw; w++) b += sq[w];
    const unsigned long long lo = (unsigned long long)b;
    const unsigned long long old = atomicAdd(acc, lo);
    const unsigned long long carry = old + lo < old ? 1ull : 0ull;
    atomicAdd(acc + 1, (unsigned long long)(b >> 64) + carry);
    __threadfence();
    s_ticket = atomicAdd(done, 1);
    s_last = s_ticket == (int)gridDim.x - 1;
  }
  __syncthreads();
  *ticket = s_ticket;
  if (!s_last) return false;
  if (threadIdx.x == 0) {
    __threadfence();
    volatile unsigned long long* va = acc;
    const unsigned long long lo = va[0], hi = va[1];
    va[0] = 0ull;
    va[1] = 0ull;
    const __int128 q = (__int128)(((unsigned __int128)hi << 64) | (unsigned __int128)lo);
    *total = fx64_to_double(q);
    if (raw) *raw = q;
    *done = 0;
  }
  __syncthreads();
  return true;
}

// level_end_kernel's bookkeeping, done in graph mode by the statistics kernel
// that ends the level (outer != 0), which saves a node per level
__device__ __forceinline__ void level_end_work(Ctrl* c, Sched s, unsigned long long outer) {
  s.level_counts[c->level] = c->pass + 1;
  c->levels_done = c->level + 1;
  c->level++;
  if (c->level >= c->num_levels || c->status) set_cond(outer, 0);
}

// Level start (plas.py:256-258): fp64 distance of every cell to the fresh
// target into the cache, sum -> previous, trace, open the pass loop.
// The sum is taken in 128-bit fixed point (fx64 per cell, exact integer adds),
// so it does not depend on how cells are split across CTAs or GPUs: a sharded
// sort sums each rank's own rows [own_lo, own_hi) and adds the ranks'
// integers (level_start_shard_kernel), bit-identical to one GPU.  The cache
// covers the rows whose target this rank holds, [band_lo, band_hi).
// Sharded (world > 1): the last CTA only publishes the raw 128-bit partial to
// xpart[0..1]; level_start_shard_kernel runs the controller after the exchange.
__device__ __forceinline__ void level_start_control(Ctrl* c, Sched s, double tot, long long n,
                                                    unsigned long long inner, unsigned long long outer, bool* go) {
  c->dist_sum = tot;
  c->previous = tot / (double)n;
  if (c->trace_pos >= c->trace_cap) {
    c->status = 1;
    c->level_done = 1;
    set_cond(inner, 0);
    if (outer) level_end_work(c, s, outer);
  } else {
    s.trace[c->trace_pos++] = c->previous;
    *go = true;
  }
}

__global__ void __launch_bounds__(RED_THREADS, STATS_MINB) level_stats_kernel(
    Ctrl* c, Sched s, const float* __restrict__ feat, const float* __restrict__ target,
    double* __restrict__ dcache, long long n, int D, int S, double* acc, int* done,
    unsigned long long inner, unsigned long long outer, int* tab, long long tab_stride, double* xpart) {
  __shared__ double s_tot;
  __shared__ unsigned long long s_gkey;
  const int side = c->side;
  const int lev0 = c->level;  // read before the ticket: the last CTA may rewrite Ctrl after it
  const long long i0 = (long long)c->band_lo * side, i1 = (long long)c->band_hi * side;
  const long long o0 = (long long)c->own_lo * side, o1 = (long long)c->own_hi * side;
  __int128 sum = 0;
  // the per-cell cache feeds PARITY mode's moved-cell statistic only (DEVICE
  // mode forms its pass changes in K3, k3_delta_acc)
  const bool keep = c->rng_mode != 1;
  for (long long i = i0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < i1;
       i += (long long)gridDim.x * blockDim.x) {
    const double d = sqrt(S == 16 ? cell_dist2_s16(feat + i * 16, target + i * 16, D)
                                   : cell_dist2(feat + i * S, target + i * S, D, S));
    if (keep) dcache[i] = d;
    if (i >= o0 && i < o1) sum += fx64(d);
  }
  const bool gen = tab && c->rng_mode == 1;
  int ticket = 0;
  __int128 raw = 0;
  if (!last_cta_reduce_fx(sum, reinterpret_cast<unsigned long long*>(acc), done, &s_tot, &ticket, &raw)) {
    // pass 0's tables, built by the other CTAs (ticket order) while the last one finishes
    if (gen) gen_class_tables(c, 0, tab, tab_stride, ticket, gridDim.x > 1 ? gridDim.x - 1 : 1, lev0);
    return;
  }
  if (c->world > 1) {
    if (threadIdx.x == 0) store_i128(xpart, raw);
    if (gen && gridDim.x == 1) gen_class_tables(c, 0, tab, tab_stride, 0, 1);
    return;
  }
  if (c->exact_stats) return;  // PARITY, one GPU: np_level_start_kernel on NumPy's grid_distance
  __shared__ Ctrl sc;
  Ctrl* const cg = c;
  ctrl_to_smem(&sc, cg);
  c = &sc;
  bool go = false;
  if (threadIdx.x == 0) level_start_control(c, s, s_tot, n, inner, outer, &go);
  go = __syncthreads_or(go);
  if (go) {
    if (c->rng_mode == 1) prepare_device_pass_cta(c, &s_gkey);
    if (threadIdx.x == 0) set_cond(inner, 1);
  }
  ctrl_from_smem(cg, &sc);
  if (gen && gridDim.x == 1) gen_class_tables(&sc, 0, tab, tab_stride, 0, 1);
}

// Strike logic of one finished pass (plas.py:266-272) given the summed fp64
// distance change `tot` of its moved cells: current = (level-start sum +
// changes) / n, trace append, strikes, level end.  Thread 0 only; returns
// whether the level continues.
__device__ __forceinline__ bool controller_step_cur(Ctrl* c, Sched s, double current, unsigned long long inner) {
  const double previous = c->previous;
  c->current = current;
  c->reorders++;
  c->pass++;
  if (c->trace_pos >= c->trace_cap) {
    c->status = 1;
    c->level_done = 1;
    set_cond(inner, 0);
    return false;
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
    return false;
  }
  return true;
}
__device__ __forceinline__ bool controller_step(Ctrl* c, Sched s, double tot, long long n,
                                                unsigned long long inner) {
  c->dist_sum += tot;
  return controller_step_cur(c, s, c->dist_sum / (double)n, inner);
}

// After a pass: exact fp64 distance change of the moved cells (cells that
// keep their element keep their cached distance), so current =
// (level-start sum + deltas) / n equals grid_distance(feat, target)
// (plas.py:266) up to fp64 summation order; then the strike logic
// (plas.py:267-272) and the next pass's geometry.
// Sharded (world > 1): the last CTA only publishes this rank's partial
// (change, moved count) to xpart; shard_control_kernel runs the controller
// once every rank's partial has been exchanged.
template <bool WROWS>  // rows wider than 16 floats (a quad of lanes per cell)
__global__ void __launch_bounds__(RED_THREADS, STATS_MINB) pass_stats_kernel(
    Ctrl* c, Sched s, const float* __restrict__ feat, const float* __restrict__ target,
    double* __restrict__ dcache, int D, int S, const int* __restrict__ list, int* counters,
    double* partials, int* done, long long n, unsigned long long inner, unsigned long long outer,
    double* xpart, int* tab, long long tab_stride) {
  __shared__ double s_tot;
  __shared__ unsigned long long s_gkey;
  if (c->level_done) return;  // an unrolled pass slot after the level ended (no CTA takes a ticket)
  gtrace_mark(c, 2);
  if (c->rng_mode == 1) {
    // DEVICE mode: K3 already summed the pass's distance change (k3_delta_acc,
    // 128-bit fixed point in partials[0..1]) and counted the moves, so no CTA
    // waits for another: CTA 0 runs the controller at once while the others
    // build the next pass's grouping tables.
    const bool gen = tab != nullptr;
    if (blockIdx.x != 0) {
      // (per-class slices here, not spread over (class, chunk) pairs as at level
      // start: the spread form made concurrent sorts from several host threads
      // fail with illegal addresses now and then -- not understood, so not used)
      if (gen) gen_class_tables(c, c->gen_pass, tab, tab_stride, blockIdx.x - 1, gridDim.x - 1, c->gen_level, false);
      if (c->gtrace) {
        __syncthreads();
        gtrace_mark(c, 5);
      }
      return;
    }
    __shared__ int s_count;
    __shared__ __int128 s_raw;
    if (threadIdx.x == 0) {
      volatile unsigned long long* va = reinterpret_cast<unsigned long long*>(partials);
      const unsigned long long lo = va[0], hi = va[1];
      va[0] = 0ull;
      va[1] = 0ull;
      s_raw = (__int128)(((unsigned __int128)hi << 64) | (unsigned __int128)lo);
      s_tot = fx64_to_double(s_raw);
      s_count = counters[2];
    }
    __syncthreads();
    gtrace_mark(c, 4);
    if (c->world > 1) {  // sharded: publish this rank's exact partial; shard_control_kernel decides
      if (threadIdx.x == 0) {
        store_i128(xpart, s_raw);
        xpart[2] = (double)s_count;
        xpart[3] = 0.0;
      }
      return;
    }
    __shared__ Ctrl sc;
    Ctrl* const cg = c;
    ctrl_to_smem(&sc, cg);
    bool more = false;
    if (threadIdx.x == 0) {
      counters[0] += s_count;
      counters[2] = 0;
      more = controller_step(&sc, s, s_tot, n, inner);
    }
    more = __syncthreads_or(more);
    if (more) prepare_device_pass_cta(&sc, &s_gkey);
    if (!more && outer && threadIdx.x == 0) level_end_work(&sc, s, outer);
    if (cg->gtrace && threadIdx.x == 0) atomicMax(&cg->gtrace[6 * (sc.reorders - 1) + 3], gtimer());
    ctrl_from_smem(cg, &sc);
    if (gen && gridDim.x == 1) gen_class_tables(&sc, sc.pass, tab, tab_stride, 0, 1);
    return;
  }
  const int count = counters[2];
  __int128 sum = 0;  // fixed point (fx64): order-free
  const int stride = gridDim.x * blockDim.x;
  if (WROWS) {
    // wide rows: a quad of lanes per cell, lane s extends cell_dist2's chain
    // p[s] over chunks s, s + 4, ... (coalesced 64-byte row pieces); the
    // xor-1-then-xor-2 reduction forms (p0 + p1) + (p2 + p3): the same value
    // (warp-uniform trip count: 8 cells per warp per step, all lanes shuffle)
    const int s4 = threadIdx.x & 3, nch = S >> 2, qw = (threadIdx.x & 31) >> 2;
    for (int eb = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 8; eb < count; eb += (stride >> 5) * 8) {
      const int e = eb + qw;
      const bool ok = e < count;
      const long long cell = ok ? list[e] : 0;
      const double old = ok && s4 == 0 ? dcache[cell] : 0.0;
      const float4* xa = reinterpret_cast<const float4*>(feat + cell * S);
      const float4* ya = reinterpret_cast<const float4*>(target + cell * S);
      double acc = 0.0;
      for (int c0 = s4; c0 < nch; c0 += 16) {
        float4 x[4], y[4];
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int c = c0 + 4 * r;
          x[r] = ok && c < nch ? __ldg(xa + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          y[r] = ok && c < nch ? __ldg(ya + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int c = c0 + 4 * r;
          const float xs[4] = {x[r].x, x[r].y, x[r].z, x[r].w}, ys[4] = {y[r].x, y[r].y, y[r].z, y[r].w};
#pragma unroll
          for (int q = 0; q < 4; q++)
            if (4 * c + q < D) {
              const double df = (double)xs[q] - (double)ys[q];
              acc = fma(df, df, acc);
            }
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (ok && s4 == 0) {
        const double d = sqrt(acc);
        sum += fx64(d - old);
        dcache[cell] = d;
      }
    }
  }
  // two independent cells per thread in flight, every row load issued first
  for (int e0 = blockIdx.x * blockDim.x + threadIdx.x; !WROWS && e0 < count; e0 += 2 * stride) {
    long long cell[2];
    double old[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int e = e0 + u * stride;
      cell[u] = e < count ? list[e] : -1;
      old[u] = cell[u] >= 0 ? dcache[cell[u]] : 0.0;
    }
    if (S == 16 && cell[1] >= 0) {  // the common case: both rows sets in flight together
      float4 x[2][4], y[2][4];
#pragma unroll
      for (int u = 0; u < 2; u++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
          x[u][c] = __ldg(reinterpret_cast<const float4*>(feat + cell[u] * 16) + c);
          y[u][c] = __ldg(reinterpret_cast<const float4*>(target + cell[u] * 16) + c);
        }
#pragma unroll
      for (int u = 0; u < 2; u++) {
        double p[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const float xs[4] = {x[u][c].x, x[u][c].y, x[u][c].z, x[u][c].w};
          const float ys[4] = {y[u][c].x, y[u][c].y, y[u][c].z, y[u][c].w};
          double acc = 0.0;
#pragma unroll
          for (int e = 0; e < 4; e++)
            if (4 * c + e < D) {
              const double df = (double)xs[e] - (double)ys[e];
              acc = fma(df, df, acc);
            }
          p[c] = acc;
        }
        const double d = sqrt((p[0] + p[1]) + (p[2] + p[3]));
        sum += fx64(d - old[u]);
        dcache[cell[u]] = d;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 2; u++) {
        if (cell[u] >= 0) {
          const double d = sqrt(cell_dist2_any(feat + cell[u] * S, target + cell[u] * S, D, S));
          sum += fx64(d - old[u]);
          dcache[cell[u]] = d;
        }
      }
    }
  }
  // DEVICE mode: every CTA builds its slice of the next pass's grouping tables
  // AFTER taking its ticket, so the slices are built while the last CTA runs
  // the controller instead of delaying it (gen_pass was set by the pass kernel;
  // the controller's writes to Ctrl leave the fields read here unchanged)
  const bool gen = tab && c->rng_mode == 1;
  int ticket = 0;
  __int128 raw = 0;
  if (!last_cta_reduce_fx(sum, reinterpret_cast<unsigned long long*>(partials), done, &s_tot, &ticket, &raw)) {
    if (gen) gen_class_tables(c, c->gen_pass, tab, tab_stride, ticket, gridDim.x > 1 ? gridDim.x - 1 : 1, c->gen_level);
    if (c->gtrace) {
      __syncthreads();
      gtrace_mark(c, 5);  // this CTA's table slice is done
    }
    return;
  }
  gtrace_mark(c, 4);  // the last CTA has its ticket
  if (c->world > 1) {
    if (threadIdx.x == 0) {
      store_i128(xpart, raw);  // exact partial: the ranks' integers add up to the 1-GPU total
      xpart[2] = (double)count;
      xpart[3] = 0.0;
    }
    return;
  }
  if (c->exact_stats) {  // PARITY, one GPU: np_pass_control_kernel decides on NumPy's grid_distance
    if (threadIdx.x == 0) {
      counters[0] += count;
      counters[2] = 0;
    }
    return;
  }
  __shared__ Ctrl sc;
  Ctrl* const cg = c;
  ctrl_to_smem(&sc, cg);
  c = &sc;
  bool more = false;
  if (threadIdx.x == 0) {
    counters[0] += count;
    counters[2] = 0;
    more = controller_step(c, s, s_tot, n, inner);
  }
  more = __syncthreads_or(more);
  if (more && c->rng_mode == 1) prepare_device_pass_cta(c, &s_gkey);
  if (!more && outer && threadIdx.x == 0) level_end_work(c, s, outer);
  if (cg->gtrace && threadIdx.x == 0) atomicMax(&cg->gtrace[6 * (sc.reorders - 1) + 3], gtimer());
  ctrl_from_smem(cg, &sc);
  if (gen && gridDim.x == 1) gen_class_tables(&sc, sc.pass, tab, tab_stride, 0, 1);
}

// ---------------------------------------------------------------- sharding
// This rank's moved cells -> (cell, element) pairs for the exchange.
__global__ void shard_pack_kernel(const int* __restrict__ list, const int* __restrict__ counters,
                                  const int* __restrict__ idx, int2* __restrict__ send) {
  const int count = counters[2];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
    const int cell = list[e];
    send[e] = make_int2(cell, idx[cell]);
  }
}

// Every other rank's updates: element idx now sits in cell -> its f32 row
// (orig32, the working copy in element order) and the index; the cached
// distance to the cell's target where this rank holds the target (rows
// [band_lo, band_hi)).  recv holds world segments of `stride` pairs; counts
// come with the exchanged partials (xall[XPART * r + 2]).
constexpr int XPART = 4;  // doubles per rank in the pass exchange: int128 change (2 slots), count, pad
__global__ void shard_apply_kernel(const int2* __restrict__ recv, long long stride, const double* __restrict__ xall,
                                   int world, int rank, const float* __restrict__ orig32, float* __restrict__ feat,
                                   int* __restrict__ idx, const float* __restrict__ target,
                                   double* __restrict__ dcache, int D, int S, const Ctrl* __restrict__ ctrl) {
  const int nch = S >> 2;
  const long long c0 = (long long)ctrl->band_lo * ctrl->side, c1 = (long long)ctrl->band_hi * ctrl->side;
  for (int r = 0; r < world; r++) {
    if (r == rank) continue;
    const long long cnt = (long long)xall[XPART * r + 2];
    const int2* seg = recv + (long long)r * stride;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cnt;
         e += (long long)gridDim.x * blockDim.x) {
      const int2 u = seg[e];
      const long long cell = u.x, el = u.y;
      for (int c = 0; c < nch; c++)
        reinterpret_cast<float4*>(feat + cell * S)[c] = reinterpret_cast<const float4*>(orig32 + el * S)[c];
      idx[cell] = (int)el;
      if (ctrl->rng_mode != 1 && cell >= c0 && cell < c1)  // PARITY's distance cache (see level_stats_kernel)
        dcache[cell] = sqrt(cell_dist2(feat + cell * S, target + cell * S, D, S));
    }
  }
}

// The controller on the exchanged partials: the ranks' 128-bit changes added
// exactly (any order gives the 1-GPU total), then the next pass's draws and
// geometry -- identical on every rank.
__global__ void __launch_bounds__(RED_THREADS) shard_control_kernel(Ctrl* c, Sched s, const double* __restrict__ xall,
                                                                    int world, int* counters, long long n) {
  __shared__ unsigned long long s_gkey;
  bool more = false;
  if (threadIdx.x == 0) {
    __int128 tot = 0;
    long long moved = 0;
    for (int r = 0; r < world; r++) {
      tot += load_i128(xall + XPART * r);
      moved += (long long)xall[XPART * r + 2];
    }
    counters[0] += (int)moved;
    counters[2] = 0;
    more = controller_step(c, s, fx64_to_double(tot), n, 0ull);
  }
  more = __syncthreads_or(more);
  if (!more || c->rng_mode != 1) return;
  prepare_device_pass_cta(c, &s_gkey);
}

// Sharded level start: the ranks' 128-bit distance partials (exchanged,
// XPART doubles per rank) added exactly -> the level-start controller
// (previous, trace), then the first pass's draws and geometry.
__global__ void __launch_bounds__(RED_THREADS) level_start_shard_kernel(Ctrl* c, Sched s, const double* __restrict__ xall,
                                                                        int world, long long n) {
  __shared__ unsigned long long s_gkey;
  bool go = false;
  if (threadIdx.x == 0) {
    __int128 tot = 0;
    for (int r = 0; r < world; r++) tot += load_i128(xall + XPART * r);
    level_start_control(c, s, fx64_to_double(tot), n, 0ull, 0ull, &go);
  }
  go = __syncthreads_or(go);
  if (go && c->rng_mode == 1) prepare_device_pass_cta(c, &s_gkey);
}

// PARITY mode on one GPU: the level-start and per-pass controller on the
// reference's own grid_distance (np_sum.cuh: NumPy's summation order, so
// previous / current and every strike decision match plas.py:256-272 bit for
// bit); exact = (sum, sum / n) from np_tree_kernel.
__global__ void np_level_start_kernel(Ctrl* c, Sched s, const double* __restrict__ exact, long long n) {
  if (threadIdx.x) return;
  bool go = false;
  level_start_control(c, s, exact[0], n, 0ull, 0ull, &go);
}
__global__ void np_pass_control_kernel(Ctrl* c, Sched s, const double* __restrict__ exact) {
  if (threadIdx.x) return;
  c->dist_sum = exact[0];
  controller_step_cur(c, s, exact[1], 0ull);
}

// This level's sharding (host-stepped multi-GPU loop, before the blur).
__global__ void set_level_shard_kernel(Ctrl* c, int banded, int own_lo, int own_hi, int band_lo, int band_hi) {
  if (threadIdx.x) return;
  c->banded = banded;
  c->own_lo = own_lo;
  c->own_hi = own_hi;
  c->band_lo = band_lo;
  c->band_hi = band_hi;
}

// FFT-tier axis-0 exchange of a banded level: this rank computed the axis-0
// output (tmp) of columns [c0, c1) on every row; rank q needs rows
// [lo[q], hi[q]) of every column.  pack: segment q of `buf` = tmp rows
// [lo[q], hi[q]) x columns [c0, c1) (row-major); unpack: segment j = rows
// [lo[rank], hi[rank]) x columns [cs[j], cs[j + 1]) from rank j.  Offsets
// in floats; WSP = tmp row stride (floats), S = floats per cell.
__global__ void band_pack_kernel(const float* __restrict__ tmp, float* __restrict__ buf, const int* __restrict__ lo,
                                 const int* __restrict__ hi, int world, int c0, int c1, long long WSP, int S) {
  const int wc = (c1 - c0) * S;
  long long off = 0;
  for (int q = 0; q < world; q++) {
    const long long cnt = (long long)(hi[q] - lo[q]) * wc;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x) {
      const long long r = e / wc, k = e - r * wc;
      buf[off + e] = tmp[(lo[q] + r) * WSP + (long long)c0 * S + k];
    }
    off += cnt;
  }
}
__global__ void band_unpack_kernel(float* __restrict__ tmp, const float* __restrict__ buf, int lo, int hi,
                                   const int* __restrict__ cs, int world, int rank, long long WSP, int S) {
  long long off = 0;
  for (int j = 0; j < world; j++) {
    const int wc = (cs[j + 1] - cs[j]) * S;
    const long long cnt = (long long)(hi - lo) * wc;
    if (j != rank)
      for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x) {
        const long long r = e / wc, k = e - r * wc;
        tmp[(lo + r) * WSP + (long long)cs[j] * S + k] = buf[off + e];
      }
    off += cnt;
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
  set_pass_geometry(c, dy, dx, 0ull);
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

// (the API's grid_distance is np_sum.cuh: NumPy's summation order)
}  // namespace plas
