// Shared device helpers for the PLAS sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PLAS_FULL_MASK 0xffffffffu
#ifndef STATS_MINB
#define STATS_MINB 4
#endif
#ifndef BPAD_MINB
#define BPAD_MINB 3
#endif

namespace plas {

// ------------------------------------------------------------------
// Device-resident sort controller: every pass/level decision of
// plas.py:251-274 is taken on the device from these fields.
// ------------------------------------------------------------------
struct Ctrl {
  // level state
  int level;          // current level index into the schedule
  int num_levels;
  int pass;           // passes executed in this level
  int strikes;        // consecutive sub-threshold passes (plas.py:268-271)
  int beta;           // block side of this level (plas.py:60-61)
  int h;              // blur half-width ceil(r) of this level
  // geometry of the pass about to run / running (plas.py:87-110)
  int dy, dx;
  int first_y, first_x;  // first segment end (dy if dy > 0 else beta)
  int nby, nbx;          // number of block rows / columns
  int cap;               // groups per block slot = ceil(beta^2 / 4)
  int level_done;        // 1 when strikes reached 2 (host-visible in parity mode)
  long long total_groups;  // nby * nbx * cap
  double previous;     // last mean distance (plas.py:256, 272)
  double current;
  long long reorders;  // total passes (plas.py:265)
  long long trace_pos; // next free slot of the trace buffer
  long long trace_cap;
  int status;          // 0 ok, 1 trace overflow
  int levels_done;
  int side;
  int rng_mode;        // 0 parity (host draws), 1 device
  unsigned long long key0, key1;  // Philox4x64 key (numpy SeedSequence state)
  double threshold;
  int min_block;
  int pad_;
  // derived per-pass geometry (set_pass_geometry)
  int seg_h[3], seg_w[3];          // first / interior / last segment extents
  unsigned cap_m, nbx_m;           // fast-division magics for cap and nbx
  int cap_l, nbx_l;
  unsigned fe_keys[9][6];          // DEVICE mode: Feistel round keys per block class
  int fe_lbits[9], fe_rbits[9];
  // running sum of per-cell distances (level-start sum + exact per-pass deltas)
  double dist_sum;
  long long fallbacks;             // warps that took the exact fp64 decision path
  int S;                           // row stride (floats)
  int tile;                        // this pass runs the shared-memory tile kernel
  int fft_min_h;                   // levels with h >= fft_min_h (> 0) blur by FFT
  int fft_L;                       // FFT length (0 = no FFT tier)
  int tile_blur_hmax;              // levels with h <= this (and not FFT) blur in one tile kernel
  // multi-GPU sharding (world > 1): this rank's share of the pass
  int rank, world;
  long long g_lo, g_hi;            // gather kernel: groups [g_lo, g_hi)
  int b_lo, b_hi;                  // tile kernel: blocks [b_lo, b_hi)
  // DEVICE mode: this level's per-pass draws (dy, dx, grouping key), filled by
  // pass_draws_kernel at level start for passes < PDRAW_MAX
  const int4* pdraw;
  const int* prec;                 // per-pass grouping records (PREC_INTS each), same level
  int pdraw_level;                 // level the table holds (-1: none)
  // fast-division magics precomputed at level start (the per-pass geometry
  // update is on the serial critical path): cap, and nbx for its two values
  unsigned lv_cap_m, lv_seg_m[2];
  int lv_cap_l, lv_seg_l[2], lv_seg_base, lv_cap;
  int gen_pass;                    // pass whose grouping tables gen_tables_kernel builds
  int gen_level;                   // its level (written with gen_pass by K3; the controller never touches it)
  // multi-GPU, per level (set_level_shard_kernel): banded = this level's
  // passes split by block rows whose first row lies in [own_lo, own_hi) (the
  // rank's share of rows); the rank keeps target / distance cache valid on
  // rows [band_lo, band_hi) (its blocks' rows for any offset of the level)
  int banded;
  int own_lo, own_hi, band_lo, band_hi;
  int lazy_idx;                    // pass kernels read element indices of moving cells only (large grids)
  int exact_stats;                 // PARITY on one GPU: strike decisions on NumPy-order grid_distance (np_sum.cuh)
  unsigned long long* gtrace;      // diagnostics (PLAS_GTRACE): per pass ~K3 start, K3 end, ~stats start, stats end
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// record the first start (slot 0/2, stored complemented) or the last time (other slots)
__device__ __forceinline__ void gtrace_mark(const Ctrl* c, int slot) {
  if (c->gtrace && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    atomicMax(&c->gtrace[6 * c->reorders + slot], (slot == 0 || slot == 2) ? ~t : t);
  }
}

constexpr int PDRAW_MAX = 1024;  // passes per level with precomputed draws (beyond: computed on the fly)
// per-pass grouping record: m[9], lbits[9], rbits[9], keys[9][6], ww[9]
constexpr int PREC_INTS = 96;
constexpr int PREC_WW = 81;

// Grouping-table entry of local block index l (row-major in a block of width
// ww): (ly << 16) | lx, so the pass kernels get the cell's offset from the
// block origin (ly * side + lx) and its staged row (ly * ww + lx) without a
// division per group.  side < 2^16 (n < 2^31).
__host__ __device__ __forceinline__ int pack_local(unsigned l, unsigned ww) {
  const unsigned ly = l / ww;
  return (int)((ly << 16) | (l - ly * ww));
}

// Blocks whose feature + target rows fit in TILE_SMEM_MAX bytes of shared
// memory are processed by the tile kernel (coalesced staging), larger blocks
// by the gather kernel.
// measured at C2: 24 KB 114.2 ms, 32 KB 113.1 ms, 40 KB 114.9 ms, 48 KB 115.3-117.0 ms (C4: 32 KB
// 2.610 s, 48 KB 2.635 s)
#ifndef TILE_ROWS_KB
#define TILE_ROWS_KB 32
#endif
constexpr int TILE_ROWS_MAX = TILE_ROWS_KB * 1024;  // F + T rows of one block
__host__ __device__ __forceinline__ bool use_tile(int beta, int S) {
  return 2ll * beta * beta * S * 4 <= TILE_ROWS_MAX;
}

// ------------------------------------------------------------------
// Division by a runtime-invariant 32-bit divisor (round-up method):
// q = (umulhi(n, m) + n) >> l with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1.
// ------------------------------------------------------------------
__host__ __device__ __forceinline__ void make_fastdiv(unsigned d, unsigned* m, int* l) {
  int s = 0;
  while ((1ull << s) < d) s++;
  *l = s;
  *m = (unsigned)((((1ull << 32) * ((1ull << s) - d)) / d) + 1ull);
}
__host__ __device__ __forceinline__ unsigned fastdiv(unsigned n, unsigned m, int l) {
#ifdef __CUDA_ARCH__
  unsigned hi = __umulhi(n, m);
#else
  unsigned hi = (unsigned)(((unsigned long long)n * m) >> 32);
#endif
  return (unsigned)(((unsigned long long)hi + n) >> l);
}

// ------------------------------------------------------------------
// Philox4x64-10 (Random123 constants; same generator NumPy's Philox uses)
// ------------------------------------------------------------------
__host__ __device__ __forceinline__ void philox4x64_10(const unsigned long long in[4],
                                                       unsigned long long k0,
                                                       unsigned long long k1,
                                                       unsigned long long out[4]) {
  unsigned long long c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
#ifdef __CUDA_ARCH__
    unsigned long long hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    unsigned long long hi1 = __umul64hi(0xCA5A826395121157ull, c2);
#else
    unsigned long long hi0 = (unsigned long long)(((unsigned __int128)0xD2E7470EE14C6C93ull * c0) >> 64);
    unsigned long long hi1 = (unsigned long long)(((unsigned __int128)0xCA5A826395121157ull * c2) >> 64);
#endif
    unsigned long long lo0 = 0xD2E7470EE14C6C93ull * c0;
    unsigned long long lo1 = 0xCA5A826395121157ull * c2;
    unsigned long long n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Unbiased bounded draw in [0, n) from a stream of 32-bit words (Lemire).
// `words` supplies 8 32-bit values; with n <= 2^31 a rejection beyond 8 words
// has probability < 2^-8 per word ... the loop falls back to a fresh block.
struct DeviceDraw {
  unsigned long long key0, key1;
  unsigned long long ctr[4];
  unsigned long long buf[4];
  int used;  // 32-bit halves consumed from buf (0..8)
  __host__ __device__ void init(unsigned long long k0, unsigned long long k1, unsigned long long a,
                                unsigned long long b, unsigned long long c) {
    key0 = k0;
    key1 = k1;
    ctr[0] = 0;
    ctr[1] = a;
    ctr[2] = b;
    ctr[3] = c;
    used = 8;
  }
  __host__ __device__ unsigned int next32() {
    if (used == 8) {
      ctr[0]++;
      philox4x64_10(ctr, key0, key1, buf);
      used = 0;
    }
    unsigned long long w = buf[used >> 1];
    unsigned int v = (used & 1) ? (unsigned int)(w >> 32) : (unsigned int)w;
    used++;
    return v;
  }
  __host__ __device__ unsigned int bounded(unsigned int n) {
    if (n <= 1) return 0;
    unsigned long long m = (unsigned long long)next32() * n;
    unsigned int left = (unsigned int)m;
    if (left < n) {
      unsigned int thresh = (0u - n) % n;
      while (left < thresh) {
        m = (unsigned long long)next32() * n;
        left = (unsigned int)m;
      }
    }
    return (unsigned int)(m >> 32);
  }
  __host__ __device__ unsigned long long next64() {
    unsigned long long lo = next32();
    unsigned long long hi = next32();
    return lo | (hi << 32);
  }
};

// ------------------------------------------------------------------
// Keyed bijection on [0, m): unbalanced Feistel network on the smallest
// power-of-two domain >= m with cycle walking (DEVICE-mode grouping law,
// SURVEY Appendix A.1 option (b)).
// ------------------------------------------------------------------
__host__ __device__ __forceinline__ unsigned int mix32(unsigned int x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

struct Feistel {
  unsigned int keys[6];
  int lbits, rbits;  // domain bits = lbits + rbits
  unsigned int m;
  __host__ __device__ void init(unsigned long long k, unsigned int m_) {
    m = m_;
    int bits = 0;
    while ((1u << bits) < m_ && bits < 31) bits++;
    if (bits < 2) bits = 2;
    lbits = bits >> 1;
    rbits = bits - lbits;
#pragma unroll
    for (int r = 0; r < 6; r++) {
      k = k * 6364136223846793005ull + 1442695040888963407ull;
      keys[r] = (unsigned int)(k >> 32);
    }
  }
  __host__ __device__ void init_keys(const unsigned* k, int lb, int rb, unsigned m_) {
#pragma unroll
    for (int r = 0; r < 6; r++) keys[r] = k[r];
    lbits = lb;
    rbits = rb;
    m = m_;
  }
  __host__ __device__ __forceinline__ unsigned int once(unsigned int x) const {
    // state (L: a bits, R: b bits) -> (R, L ^ F(R)); shapes alternate, 4 rounds
    // (Luby-Rackoff: 4 rounds of a keyed mixing function give a strong PRP)
    unsigned int a = lbits, b = rbits;
    unsigned int L = x >> b, R = x & ((1u << b) - 1u);
#pragma unroll
    for (int r = 0; r < 4; r++) {
      unsigned int f = mix32(R ^ keys[r]) & ((1u << a) - 1u);
      unsigned int nL = R, nR = L ^ f;
      // new shape: L has b bits, R has a bits
      unsigned int t = a;
      a = b;
      b = t;
      L = nL;
      R = nR;
    }
    return (L << b) | R;
  }
  __host__ __device__ __forceinline__ unsigned int operator()(unsigned int i) const {
    if (m <= 1) return 0;
    unsigned int x = once(i);
    while (x >= m) x = once(x);
    return x;
  }
};

// ------------------------------------------------------------------
// Pass geometry (plas.py:87-110): segment bounds of block row/col b.
// ------------------------------------------------------------------
__host__ __device__ __forceinline__ void segment(int b, int first, int beta, int side, int* lo,
                                                 int* hi) {
  int s = (b == 0) ? 0 : first + (b - 1) * beta;
  int e = first + b * beta;
  if (e > side) e = side;
  *lo = s;
  *hi = e;
}

__host__ __device__ __forceinline__ int num_segments(int first, int beta, int side) {
  return first < side ? 1 + (side - first + beta - 1) / beta : 1;
}

__host__ __device__ __forceinline__ unsigned long long class_key(unsigned long long gkey, int h,
                                                                 int w) {
  unsigned long long k = gkey ^ ((unsigned long long)(unsigned)h << 32) ^ (unsigned)w;
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// Geometry of the pass about to run (everything but the DEVICE-mode keys).
__host__ __device__ __forceinline__ void set_pass_geometry_base(Ctrl* c, int dy, int dx) {
  c->dy = dy;
  c->dx = dx;
  c->first_y = dy > 0 ? dy : c->beta;
  c->first_x = dx > 0 ? dx : c->beta;
  c->nby = num_segments(c->first_y, c->beta, c->side);
  c->nbx = num_segments(c->first_x, c->beta, c->side);
  c->cap = (c->beta * c->beta + 3) / 4;
  c->total_groups = (long long)c->nby * c->nbx * c->cap;
  int lo, hi;
  segment(0, c->first_y, c->beta, c->side, &lo, &hi);
  c->seg_h[0] = hi - lo;
  c->seg_h[1] = c->beta;
  segment(c->nby - 1, c->first_y, c->beta, c->side, &lo, &hi);
  c->seg_h[2] = hi - lo;
  segment(0, c->first_x, c->beta, c->side, &lo, &hi);
  c->seg_w[0] = hi - lo;
  c->seg_w[1] = c->beta;
  segment(c->nbx - 1, c->first_x, c->beta, c->side, &lo, &hi);
  c->seg_w[2] = hi - lo;
  c->tile = use_tile(c->beta, c->S) ? 1 : 0;
  // contiguous, balanced shares of the pass's groups / blocks (whole pass when world == 1)
  const long long nb = (long long)c->nby * c->nbx;
  const int W = c->world > 0 ? c->world : 1;
  if (W == 1) {
    c->g_lo = 0;
    c->g_hi = c->total_groups;
    c->b_lo = 0;
    c->b_hi = (int)nb;
  } else if (c->banded) {
    // row bands aligned to this pass's block tiling: the block rows whose
    // first row y0(by) lies in [own_lo, own_hi) (y0(0) = 0, y0(by) = first_y +
    // (by - 1) beta), so a rank's cells are rows [own_lo, own_hi + beta)
    auto first_by = [&](int Y) {
      if (Y <= 0) return 0;
      int by = Y <= c->first_y ? 1 : 1 + (Y - c->first_y + c->beta - 1) / c->beta;
      return by < c->nby ? by : c->nby;
    };
    const int by_lo = first_by(c->own_lo), by_hi = c->own_hi >= c->side ? c->nby : first_by(c->own_hi);
    c->b_lo = by_lo * c->nbx;
    c->b_hi = by_hi * c->nbx;
    c->g_lo = (long long)c->b_lo * c->cap;
    c->g_hi = (long long)c->b_hi * c->cap;
  } else {
    c->g_lo = c->total_groups * c->rank / W;
    c->g_hi = c->total_groups * (c->rank + 1) / W;
    c->b_lo = (int)(nb * c->rank / W);
    c->b_hi = (int)(nb * (c->rank + 1) / W);
  }
  if (c->lv_cap == c->cap) {  // level-start magics (level_begin_kernel)
    c->cap_m = c->lv_cap_m;
    c->cap_l = c->lv_cap_l;
  } else {
    make_fastdiv((unsigned)c->cap, &c->cap_m, &c->cap_l);
  }
  const int si = c->nbx - c->lv_seg_base;
  if (si == 0 || si == 1) {
    c->nbx_m = c->lv_seg_m[si];
    c->nbx_l = c->lv_seg_l[si];
  } else {
    make_fastdiv((unsigned)c->nbx, &c->nbx_m, &c->nbx_l);
  }
}

// DEVICE-mode Feistel keys of block class cls.  gkey keys the per-class
// groupings; classes with equal (h, w) get identical keys, so all blocks of
// one shape share one grouping (plas.py:209).
__host__ __device__ __forceinline__ void set_class_keys(Ctrl* c, int cls, unsigned long long gkey) {
  const int hh = c->seg_h[cls / 3], ww = c->seg_w[cls % 3];
  Feistel fe;
  fe.init(class_key(gkey, hh, ww), (unsigned)(hh * ww));
  for (int r = 0; r < 6; r++) c->fe_keys[cls][r] = fe.keys[r];
  c->fe_lbits[cls] = fe.lbits;
  c->fe_rbits[cls] = fe.rbits;
}

__host__ __device__ __forceinline__ void set_pass_geometry(Ctrl* c, int dy, int dx,
                                                           unsigned long long gkey) {
  set_pass_geometry_base(c, dy, dx);
  if (c->rng_mode == 1)
    for (int cls = 0; cls < 9; cls++) set_class_keys(c, cls, gkey);
}

// DEVICE-mode per-pass draws: dy, dx and the grouping key come from the
// Philox4x64-10 stream keyed like NumPy's (SeedSequence state), at counter
// (block, pass, level, purpose) -- stateless, identical on every GPU.
__host__ __device__ __forceinline__ void device_pass_draws_at(const Ctrl* c, int level, int pass, int beta, int* dy,
                                                              int* dx, unsigned long long* gkey) {
  DeviceDraw d;
  d.init(c->key0, c->key1, (unsigned long long)pass, (unsigned long long)level, 0x504153535ull /* "PASS" */);
  *dy = (int)d.bounded((unsigned)beta);
  *dx = (int)d.bounded((unsigned)beta);
  *gkey = d.next64();
}

__host__ __device__ __forceinline__ void device_pass_draws(const Ctrl* c, int* dy, int* dx,
                                                           unsigned long long* gkey) {
#ifdef __CUDA_ARCH__
  if (c->pdraw && c->pdraw_level == c->level && c->pass < PDRAW_MAX) {  // precomputed at level start
    const int4 v = c->pdraw[c->pass];
    *dy = v.x;
    *dx = v.y;
    *gkey = ((unsigned long long)(unsigned)v.w << 32) | (unsigned)v.z;
    return;
  }
#endif
  DeviceDraw d;
  d.init(c->key0, c->key1, (unsigned long long)c->pass, (unsigned long long)c->level,
         0x504153535ull /* "PASS" */);
  *dy = (int)d.bounded((unsigned)c->beta);
  *dx = (int)d.bounded((unsigned)c->beta);
  *gkey = d.next64();
}

// warp / block reductions in fp64 with a fixed order (deterministic)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(PLAS_FULL_MASK, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < NT / 32 ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

}  // namespace plas
