// K3: fused group assignment (plas.py:113-156 _assign_groups, driven by
// plas.py:196-223 _reassign_pass) + the per-pass distance statistic
// (plas.py:266 grid_distance) in one kernel.
//
// Four lanes cooperate on one group of k <= 4 cells (8 groups per warp):
//   lane s loads its own feature row F_s and every target row T_j of the
//   group (the 4 lanes load the same T_j address, which the LSU merges), and
//   computes cost[s][j] with the reference's arithmetic:
//      c = fp32( sqrt_fp64( sum_d fp64( fp32(F_s[d] - T_j[d])^2 ) ) )
//   sequential in d, no FMA.  The 16 costs are exchanged with shuffles; lane s
//   evaluates the (k-1)! lexicographic arrangements that start with s
//   (cost summed in fp64 in slot order, strict '<' keeps the first minimum),
//   the four lane minima are reduced on (cost, index) so the lexicographically
//   first strict minimum wins exactly as in the reference.  The element in slot
//   i then moves to slot P[i]; identity arrangements and fixed points write
//   nothing (~3.6% of cells move per pass).
//   Finally each lane adds the fp64 distance of its element to the target of
//   its new cell, so the pass statistic needs no second sweep over HBM.
#pragma once
#include "common.cuh"

namespace plas {

// slot destination of slot s under arrangement p of k elements (k = 2, 3, 4)
__device__ __forceinline__ int perm_dest(int k, int p, int s) {
  if (k == 4) {
    int first = p / 6, local = p % 6;
    int o0 = first == 0 ? 1 : 0;
    int o1 = first <= 1 ? 2 : 1;
    int o2 = first <= 2 ? 3 : 2;
    // local order: (o0,o1,o2),(o0,o2,o1),(o1,o0,o2),(o1,o2,o0),(o2,o0,o1),(o2,o1,o0)
    int a = local < 2 ? o0 : (local < 4 ? o1 : o2);
    int b, c;
    switch (local) {
      case 0: b = o1; c = o2; break;
      case 1: b = o2; c = o1; break;
      case 2: b = o0; c = o2; break;
      case 3: b = o2; c = o0; break;
      case 4: b = o0; c = o1; break;
      default: b = o1; c = o0; break;
    }
    return s == 0 ? first : (s == 1 ? a : (s == 2 ? b : c));
  } else if (k == 3) {
    int first = p / 2, local = p % 2;
    int o0 = first == 0 ? 1 : 0;
    int o1 = first == 2 ? 1 : 2;
    int a = local == 0 ? o0 : o1, b = local == 0 ? o1 : o0;
    return s == 0 ? first : (s == 1 ? a : b);
  } else if (k == 2) {
    return s == 0 ? p : 1 - p;
  }
  return s;
}

// C[i][j] for the group lives in lane (base + i) as c[j]; fetch by (i, j)
struct CostMat {
  float v[4][4];
};

__device__ __forceinline__ float sel4(const float* r, int i) {
  return i == 0 ? r[0] : (i == 1 ? r[1] : (i == 2 ? r[2] : r[3]));
}

// Evaluate the arrangements starting with slot s; return (best cost, best p).
// All register indices are static (runtime choices go through selects) so the
// cost matrix never spills to local memory.
__device__ __forceinline__ void lane_best(const CostMat& C, int k, int s, double* best_cost,
                                          int* best_p) {
  double bc = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int bp = 0x7fffffff;
  if (s < k) {
    const double c0 = (double)sel4(C.v[0], s);
    if (k == 4) {
      const int o0 = s == 0 ? 1 : 0, o1 = s <= 1 ? 2 : 1, o2 = s <= 2 ? 3 : 2;
      double x[4][3];
#pragma unroll
      for (int i = 1; i < 4; i++) {
        x[i][0] = (double)sel4(C.v[i], o0);
        x[i][1] = (double)sel4(C.v[i], o1);
        x[i][2] = (double)sel4(C.v[i], o2);
      }
      // lexicographic arrangements (s, a, b, d) over the remaining {o0 < o1 < o2}
      const int A[6] = {0, 0, 1, 1, 2, 2};
      const int B[6] = {1, 2, 0, 2, 0, 1};
      const int E[6] = {2, 1, 2, 0, 1, 0};
#pragma unroll
      for (int l = 0; l < 6; l++) {
        double c = __dadd_rn(0.0, c0);
        c = __dadd_rn(c, x[1][A[l]]);
        c = __dadd_rn(c, x[2][B[l]]);
        c = __dadd_rn(c, x[3][E[l]]);
        if (c < bc) {
          bc = c;
          bp = 6 * s + l;
        }
      }
    } else if (k == 3) {
      const int o0 = s == 0 ? 1 : 0, o1 = s == 2 ? 1 : 2;
      const double a0 = (double)sel4(C.v[1], o0), a1 = (double)sel4(C.v[1], o1);
      const double b0 = (double)sel4(C.v[2], o0), b1 = (double)sel4(C.v[2], o1);
      double c = __dadd_rn(__dadd_rn(__dadd_rn(0.0, c0), a0), b1);
      bc = c;
      bp = 2 * s;
      c = __dadd_rn(__dadd_rn(__dadd_rn(0.0, c0), a1), b0);
      if (c < bc) {
        bc = c;
        bp = 2 * s + 1;
      }
    } else if (k == 2) {
      bc = __dadd_rn(__dadd_rn(0.0, c0), (double)sel4(C.v[1], 1 - s));
      bp = s;
    }
  }
  *best_cost = bc;
  *best_p = bp;
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4v(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float f4get(const float4& v, int e) {
  return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}

// Process one group per 4 lanes.  All 32 lanes of the warp must call this
// together.  `cell` is this lane's cell (valid when s < k); k may differ
// between the 8 groups of a warp.  Rows have stride S (multiple of 4).
// REG: feature/target rows of up to FCAP floats are kept in registers; the
// generic path (FCAP == 0) streams rows and moves them chunk by chunk.
// Returns this lane's fp64 distance contribution (0 when !want_dist).
template <int FCAP, typename IdxT>
__device__ __forceinline__ double group_assign(float* __restrict__ feat, IdxT* __restrict__ idx,
                                               const float* __restrict__ target, int D, int S,
                                               long long cell, int k, bool want_dist,
                                               int* moved) {
  const int lane = threadIdx.x & 31;
  const int s = lane & 3;
  const int gbase = lane & ~3;
  const bool act = s < k;
  const int nch = S >> 2;
  long long cj[4];
#pragma unroll
  for (int j = 0; j < 4; j++) cj[j] = __shfl_sync(PLAS_FULL_MASK, cell, gbase + j);

  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  constexpr int NC = FCAP > 0 ? FCAP / 4 : 1;
  float4 F[NC];
  float4 T[FCAP > 0 && FCAP <= 16 ? 4 : 1][FCAP > 0 && FCAP <= 16 ? NC : 1];
  if (FCAP > 0) {
#pragma unroll
    for (int c = 0; c < NC; c++) {
      if (c < nch) {
        F[c] = act ? ld4v(feat + cell * S + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          float4 t = (act && j < k) ? ld4(target + cj[j] * S + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
          if (FCAP <= 16) T[j][c] = t;
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int d = 4 * c + e;
            if (d < D) {
              float df = __fsub_rn(f4get(F[c], e), f4get(t, e));
              acc[j] = __dadd_rn(acc[j], (double)__fmul_rn(df, df));
            }
          }
        }
      }
    }
  } else {
    for (int c = 0; c < nch; c++) {
      float4 f = act ? ld4v(feat + cell * S + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        float4 t = (act && j < k) ? ld4(target + cj[j] * S + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int d = 4 * c + e;
          if (d < D) {
            float df = __fsub_rn(f4get(f, e), f4get(t, e));
            acc[j] = __dadd_rn(acc[j], (double)__fmul_rn(df, df));
          }
        }
      }
    }
  }
  float cst[4];
#pragma unroll
  for (int j = 0; j < 4; j++) cst[j] = __double2float_rn(__dsqrt_rn(acc[j]));
  CostMat C;
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) C.v[i][j] = __shfl_sync(PLAS_FULL_MASK, cst[j], gbase + i);

  double bc;
  int bp;
  lane_best(C, k, s, &bc, &bp);
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    double oc = __shfl_xor_sync(PLAS_FULL_MASK, bc, o);
    int op = __shfl_xor_sync(PLAS_FULL_MASK, bp, o);
    if (oc < bc || (oc == bc && op < bp)) {
      bc = oc;
      bp = op;
    }
  }
  if (k < 2) bp = 0;
  const int dst = act ? perm_dest(k, bp, s) : s;
  const long long cdst = dst == 0 ? cj[0] : (dst == 1 ? cj[1] : (dst == 2 ? cj[2] : cj[3]));
  const bool move = act && bp != 0 && dst != s;
  IdxT my_idx = 0;
  if (move) my_idx = idx[cell];
  double dist = 0.0;
  if (FCAP > 0) {
    __syncwarp();
    if (move) {
#pragma unroll
      for (int c = 0; c < NC; c++)
        if (c < nch) *reinterpret_cast<float4*>(feat + cdst * S + 4 * c) = F[c];
      idx[cdst] = my_idx;
    }
    if (want_dist && act) {
#pragma unroll
      for (int c = 0; c < NC; c++) {
        if (c < nch) {
          float4 t;
          if (FCAP <= 16) {
            t = dst == 0 ? T[0][c] : (dst == 1 ? T[1][c] : (dst == 2 ? T[2][c] : T[3][c]));
          } else {
            t = ld4(target + cdst * S + 4 * c);
          }
#pragma unroll
          for (int e = 0; e < 4; e++) {
            if (4 * c + e < D) {
              double df = (double)f4get(F[c], e) - (double)f4get(t, e);
              dist = fma(df, df, dist);
            }
          }
        }
      }
      dist = sqrt(dist);
    }
  } else {
    // generic rows: read chunk c of every slot, then write it to the
    // destination; reads of a chunk complete warp-wide before its writes.
    for (int c = 0; c < nch; c++) {
      float4 f = act ? ld4v(feat + cell * S + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
      if (move) *reinterpret_cast<float4*>(feat + cdst * S + 4 * c) = f;
      __syncwarp();
      if (want_dist && act) {
        float4 t = ld4(target + cdst * S + 4 * c);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          if (4 * c + e < D) {
            double df = (double)f4get(f, e) - (double)f4get(t, e);
            dist = fma(df, df, dist);
          }
        }
      }
    }
    if (move) idx[cdst] = my_idx;
    if (want_dist && act) dist = sqrt(dist);
  }
  if (move) *moved += 1;
  return dist;
}

// Per-pass kernel: group g of the pass -> (block, quad) -> 4 cells.
// PARITY: the class grouping is the filtered master permutation
//   sel[cls][...] (plas.py:209, built by class_select_kernel).
// DEVICE: the class grouping is a keyed bijection on [0, m).
template <int FCAP, bool PARITY>
__global__ void __launch_bounds__(256) pass_kernel(float* __restrict__ feat, int* __restrict__ idx,
                                                    const float* __restrict__ target, int D, int S,
                                                    const Ctrl* __restrict__ ctrl,
                                                    const int* __restrict__ sel, long long sel_stride,
                                                    double* __restrict__ partials,
                                                    int* __restrict__ moved_out) {
  __shared__ double sh[32];
  const int side = ctrl->side;
  const int beta = ctrl->beta;
  const int fy = ctrl->first_y, fx = ctrl->first_x;
  const int nby = ctrl->nby, nbx = ctrl->nbx;
  const long long cap = ctrl->cap;
  const long long total = ctrl->total_groups;
  unsigned long long gkey = 0;
  if (!PARITY) {
    int ddy, ddx;
    device_pass_draws(ctrl, &ddy, &ddx, &gkey);
  }
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double dsum = 0.0;
  int moved = 0;
  for (long long gb = warp * 8; gb < total; gb += nwarps * 8) {
    const long long g = gb + (lane >> 2);
    const int s = lane & 3;
    int k = 0;
    long long cell = 0;
    if (g < total) {
      const long long b = g / cap;
      const long long q = g - b * cap;
      const int by = (int)(b / nbx), bx = (int)(b - (long long)by * nbx);
      int y0, y1, x0, x1;
      segment(by, fy, beta, side, &y0, &y1);
      segment(bx, fx, beta, side, &x0, &x1);
      const int hh = y1 - y0, ww = x1 - x0;
      const long long m = (long long)hh * ww;
      const long long rem = m - 4 * q;
      k = rem >= 4 ? 4 : (rem > 0 ? (int)rem : 0);
      if (s < k) {
        long long l;
        if (PARITY) {
          const int ty = by == 0 ? 0 : (by == nby - 1 ? 2 : 1);
          const int tx = bx == 0 ? 0 : (bx == nbx - 1 ? 2 : 1);
          l = sel[(long long)(ty * 3 + tx) * sel_stride + 4 * q + s];
        } else {
          Feistel fe;
          fe.init(class_key(gkey, hh, ww), (unsigned)m);
          l = fe((unsigned)(4 * q + s));
        }
        cell = (long long)(y0 + l / ww) * side + x0 + l % ww;
      }
    }
    dsum += group_assign<FCAP, int>(feat, idx, target, D, S, cell, k, true, &moved);
  }
  double tot = block_sum<256>(dsum, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
  if (moved_out) {
    int mv = __reduce_add_sync(PLAS_FULL_MASK, moved);
    if (lane == 0 && mv) atomicAdd(moved_out, mv);
  }
}

// Parity mode: per class (ty, tx) the stable filter master_perm[master_perm < m]
// (plas.py:209).  One CTA per class; master perm of beta^2 entries.
__global__ void __launch_bounds__(1024) class_select_kernel(const int* __restrict__ mp,
                                                             const Ctrl* __restrict__ ctrl,
                                                             int* __restrict__ sel,
                                                             long long sel_stride) {
  __shared__ int counts[1024];
  const int cls = blockIdx.x;
  const int ty = cls / 3, tx = cls % 3;
  const int side = ctrl->side, beta = ctrl->beta;
  const int nby = ctrl->nby, nbx = ctrl->nbx;
  // class exists?  type 0 = first segment, 2 = last (needs >= 2 segments), 1 = interior (>= 3)
  auto exists = [](int t, int n) { return t == 0 || (t == 2 && n >= 2) || (t == 1 && n >= 3); };
  if (!exists(ty, nby) || !exists(tx, nbx)) return;
  int y0, y1, x0, x1;
  segment(ty == 0 ? 0 : (ty == 2 ? nby - 1 : 1), ctrl->first_y, beta, side, &y0, &y1);
  segment(tx == 0 ? 0 : (tx == 2 ? nbx - 1 : 1), ctrl->first_x, beta, side, &x0, &x1);
  const long long m = (long long)(y1 - y0) * (x1 - x0);
  const long long n = (long long)beta * beta;
  const long long per = (n + blockDim.x - 1) / blockDim.x;
  const long long s0 = threadIdx.x * per, s1 = min(n, s0 + per);
  int cnt = 0;
  for (long long i = s0; i < s1; i++) cnt += mp[i] < m;
  counts[threadIdx.x] = cnt;
  __syncthreads();
  // exclusive scan (Hillis-Steele on 1024 entries)
  for (int off = 1; off < 1024; off <<= 1) {
    int v = threadIdx.x >= off ? counts[threadIdx.x - off] : 0;
    __syncthreads();
    counts[threadIdx.x] += v;
    __syncthreads();
  }
  long long pos = threadIdx.x ? counts[threadIdx.x - 1] : 0;
  int* out = sel + (long long)cls * sel_stride;
  for (long long i = s0; i < s1; i++) {
    int v = mp[i];
    if (v < m) out[pos++] = v;
  }
}

// ABI kernel for _assign_groups on an explicit (G, k) group list (plas.py:113-156).
template <int FCAP>
__global__ void __launch_bounds__(256) groups_kernel(float* __restrict__ feat,
                                                     long long* __restrict__ idx,
                                                     const float* __restrict__ target, int D, int S,
                                                     const long long* __restrict__ groups,
                                                     long long G, int k) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  int moved = 0;
  for (long long gb = warp * 8; gb < G; gb += nwarps * 8) {
    const long long g = gb + (lane >> 2);
    const int s = lane & 3;
    const int kk = g < G ? k : 0;
    const long long cell = (s < kk) ? groups[g * k + s] : 0;
    group_assign<FCAP, long long>(feat, idx, target, D, S, cell, kk, false, &moved);
  }
}

}  // namespace plas
