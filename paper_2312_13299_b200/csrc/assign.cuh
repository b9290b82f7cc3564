// K3: fused group assignment (plas.py:113-156 _assign_groups, driven by
// plas.py:196-223 _reassign_pass), one kernel per pass.
//
// Four lanes cooperate on one group of k <= 4 cells (8 groups per warp).
// Lane s of a group loads float4 chunk s (s+4, s+8, ... for rows wider than
// 16 floats) of all 4 feature rows and all 4 target rows of the group, so one
// load instruction moves whole 64-byte rows of 8 groups (8 L1 wavefronts
// instead of 32 for a thread-per-group layout).  The lanes accumulate the
// partial squared distances of the 16 (element, target) pairs over their
// chunk, reduce-scatter them (lane s ends with row s of the cost matrix) and
// exchange the costs with shuffles.
//
// Decision = the reference's first strict minimum over the k! lexicographic
// arrangements of sum_i c[i][p(i)] with
//     c = fp32( sqrt_f64( sum_d f64( fp32(F_d - T_d)^2 ) ) )
// (sequential fp64 sums, no FMA), taken in two tiers:
//   fast:  costs and arrangement sums in fp32 (FFMA partial sums in any order,
//          sqrt.approx).  Every fast cost is within (D/2 + 7) 2^-24 (relative)
//          of the reference cost and every fast arrangement sum within
//          (D/2 + 10) 2^-24 of the reference sum (non-negative terms), so if
//          the second-best fast sum exceeds the best by more than
//          2 (D+24) 2^-24 of itself, the reference's strict minimum is the same
//          arrangement and is unique.
//   exact: otherwise (near-ties, exact ties, overflow, tiny costs) the warp
//          recomputes the costs with the reference arithmetic in fp64
//          (__fsub_rn / __fmul_rn / __dadd_rn / __dsqrt_rn) and applies the
//          lexicographic first-minimum rule.  Such groups are counted.
// The element in slot i moves to slot P[i]; identity arrangements and fixed
// points write nothing (~3.6% of cells move per pass).
// The destination cells of all moves go to a moved-cell list (per-CTA shared
// staging, one global reservation per flush); the statistic kernel
// (control.cuh pass_stats_kernel) then updates the per-cell fp64 distance
// cache and the running sum for exactly those cells.
#pragma once
#include "common.cuh"
#include "control.cuh"

namespace plas {

__device__ __forceinline__ float4 ld4g(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4v(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, const float4& v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float f4get(const float4& v, int e) {
  return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}
__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// packed f32x2 arithmetic (sm_100: FADD2 / FFMA2, two fp32 lanes per instruction)
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long sqacc2(unsigned long long d, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(d), "l"(c));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sel4(const float* r, int i) {
  return i == 0 ? r[0] : (i == 1 ? r[1] : (i == 2 ? r[2] : r[3]));
}
template <typename T>
__device__ __forceinline__ T pick4(const T (&a)[4], int i) {
  return i == 0 ? a[0] : (i == 1 ? a[1] : (i == 2 ? a[2] : a[3]));
}

// destination slot of slot i under lexicographic arrangement p of k elements
// (itertools.permutations order, plas.py:31-34), packed 2 bits per slot
__device__ __forceinline__ int perm_dest(int k, int p, int i) {
  if (k == 4) {
    const unsigned long long w =
        p < 8 ? 0xb1e16c9c78d8b4e4ull : (p < 16 ? 0x36c672d22d8d39c9ull : 0x1b4b278763931e4eull);
    return (int)((w >> (8 * (p & 7) + 2 * i)) & 3ull);
  }
  if (k == 3) return (int)((0x61209211824ull >> (8 * p + 2 * i)) & 3ull);
  if (k == 2) return p == 0 ? i : 1 - i;
  return i;
}
// all four destinations of arrangement p of k slots, 2 bits per slot
__device__ __forceinline__ unsigned perm_dest_code(int k, int p) {
  unsigned long long w;
  int sh;
  if (k == 4) {
    w = p < 8 ? 0xb1e16c9c78d8b4e4ull : (p < 16 ? 0x36c672d22d8d39c9ull : 0x1b4b278763931e4eull);
    sh = 8 * (p & 7);
  } else if (k == 3) {
    w = 0x61209211824ull | 0xc0c0c0c0c0c0ull;  // slot 3 stays
    sh = 8 * p;
  } else if (k == 2) {
    w = 0xe1e4ull;
    sh = 8 * p;
  } else {
    w = 0xe4ull;
    sh = 0;
  }
  return (unsigned)((w >> sh) & 0xffull);
}

struct CostMat {
  float v[4][4];  // v[i][j] = cost of slot i's element in slot j's target
};

// Arrangements that start with slot s, lexicographic: k=4 -> (s, a, b, e) over
// the remaining {o0 < o1 < o2}, p = 6s + l; k=3 -> p = 2s + l; k=2 -> p = s.
// exact tier: reference arithmetic in fp64 (first strict minimum)
__device__ __forceinline__ void lane_best_exact(const CostMat& C, int k, int s, double* best_cost,
                                                int* best_p) {
  double bc = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int bp = 0x7fffffff;
  if (s < k) {
    const double c0 = (double)sel4(C.v[0], s);
    if (k == 4) {
      const int o[3] = {s == 0 ? 1 : 0, s <= 1 ? 2 : 1, s <= 2 ? 3 : 2};
      double x[4][3];
#pragma unroll
      for (int i = 1; i < 4; i++)
#pragma unroll
        for (int q = 0; q < 3; q++) x[i][q] = (double)sel4(C.v[i], o[q]);
      const int A[6] = {0, 0, 1, 1, 2, 2}, B[6] = {1, 2, 0, 2, 0, 1}, E[6] = {2, 1, 2, 0, 1, 0};
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

// fast tier from the lane's column view: c0 = C[0][s], x[i][q] = C[i][o_q]
// (o = the other targets in increasing order); same sums as lane_best_fast
__device__ __forceinline__ void lane_best_fast_cols(float c0, const float (&x)[4][3], int k, int s, float* b1,
                                                    int* p1, float* b2) {
  const float INF = __int_as_float(0x7f800000);
  float v1 = INF, v2 = INF;
  int q1 = 0x7fffffff;
  bool ovf = false;  // an arrangement sum overflowed (see below)
  if (s < k) {
    if (k == 4) {
      const int A[6] = {0, 0, 1, 1, 2, 2}, B[6] = {1, 2, 0, 2, 0, 1}, E[6] = {2, 1, 2, 0, 1, 0};
#pragma unroll
      for (int l = 0; l < 6; l++) {
        const float c = ((c0 + x[1][A[l]]) + x[2][B[l]]) + x[3][E[l]];
        ovf |= c == INF;
        if (c < v1) {
          v2 = v1;
          v1 = c;
          q1 = 6 * s + l;
        } else if (c < v2) {
          v2 = c;
        }
      }
    } else if (k == 3) {  // the other targets of {0, 1, 2} are o_0 < o_1
      const float ca = (c0 + x[1][0]) + x[2][1];
      const float cb = (c0 + x[1][1]) + x[2][0];
      ovf = ca == INF || cb == INF;
      if (cb < ca) {
        v1 = cb;
        q1 = 2 * s + 1;
        v2 = ca;
      } else {
        v1 = ca;
        q1 = 2 * s;
        v2 = cb;
      }
    } else if (k == 2) {
      v1 = c0 + x[1][0];
      q1 = s;
      ovf = v1 == INF;
    }
  }
  // The fast costs sum fp32 squares in fp32: a sum can overflow to +inf where
  // the reference's fp64 sum of the same squares stays finite (plas.py:129-137),
  // so an infinite arrangement says nothing about the reference's order.  A
  // lane that saw one reports b2 = -inf, which fails the certificate for the
  // whole group after the min-reduction (decide_from_acc).
  *b1 = v1;
  *p1 = q1;
  *b2 = ovf ? -INF : v2;
}

// Decide one group (all 32 lanes call together; k may differ between the 8
// groups of a warp).  rowj[j] = row index (cell or staged local index) of slot
// j, Fb/Tb the row bases.  With WIDE == false (S <= 16) Fc[i] returns chunk s
// of feature row i for the move.  Returns the arrangement index (0 = identity).
//
// Lane s keeps its partial sums in *rotated* target order: acc[i][jj] is the
// pair (slot i, target jj ^ s) -- the target rows are fetched through
// rowt[jj] = rowj[jj ^ s], which the caller gets for free from its shuffles.
// Then the column reduce-scatter over the group's 4 lanes needs no selects:
// lane s keeps jj in {0, 1} and receives jj ^ 2 from lane s ^ 2 (the same
// target, jj ^ s), then keeps jj = 0 (target s) and receives jj = 1 from lane
// s ^ 1 (target 1 ^ s ^ 1 = s).
// acc[i][jj] += the packed squared differences of chunk pair (Fc[i], Tc[jj])
__device__ __forceinline__ void accum_chunks(unsigned long long (&acc)[4][4], const float4 (&Fc)[4],
                                             const float4 (&Tc)[4]) {
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      acc[i][j] = sqacc2(sub2(pk2(Fc[i].x, Fc[i].y), pk2(Tc[j].x, Tc[j].y)), acc[i][j]);
      acc[i][j] = sqacc2(sub2(pk2(Fc[i].z, Fc[i].w), pk2(Tc[j].z, Tc[j].w)), acc[i][j]);
    }
}

// chunk c of the 4 feature rows (slot order) and the 4 target rows (rotated
// order) of a group.  No data selects: slots >= k read row rowj = 0 (their
// pairs are never used); a lane past the row (c >= nch) reads chunk 0 of the
// quad's first feature row as every operand, so all its differences are
// exactly zero.
template <bool TNC>
__device__ __forceinline__ void load_chunks(const float* Fb, const float* Tb, const int (&rowj)[4],
                                            const int (&rowt)[4], int S, int c, bool valid, float4 (&Fc)[4],
                                            float4 (&Tc)[4]) {
  const float* Tv = valid ? Tb : Fb;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const unsigned fo = valid ? (unsigned)rowj[i] * (unsigned)S + 4u * c : (unsigned)rowj[0] * (unsigned)S;
    const unsigned to = valid ? (unsigned)rowt[i] * (unsigned)S + 4u * c : (unsigned)rowj[0] * (unsigned)S;
    Fc[i] = ld4v(Fb + fo);
    Tc[i] = (TNC && valid) ? ld4g(Tv + to) : ld4v(Tv + to);
  }
}

template <bool OOL>  // exact tier out of line (wide rows)
__device__ __forceinline__ int decide_from_acc(const unsigned long long (&acc)[4][4], const float* Fb,
                                               const float* Tb, const int (&rowj)[4], int D, int S, int k,
                                               int* exact, float (&col)[4]);

// Exact tier for the whole warp (same decision wherever the fast one was
// certain): lane s recomputes row s of the cost matrix with the reference
// arithmetic, then the first strict minimum over the lexicographic
// arrangements (~1.7 % of warps take it at C2).
__device__ __forceinline__ int decide_exact_body(const float* Fb, const float* Tb, const int (&rowj)[4], int D,
                                                 int S, int k) {
  const int lane = threadIdx.x & 31;
  const int s = lane & 3;
  const int gbase = lane & ~3;
  const int nch = S >> 2;
  double dacc[4] = {0.0, 0.0, 0.0, 0.0};
  float cst[4];
  const long long fo = (long long)pick4(rowj, s) * S;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    if (s < k && j < k) {
      const long long to = (long long)rowj[j] * S;
      for (int c = 0; c < nch; c++) {
        const float4 f = ld4v(Fb + fo + 4 * c);
        const float4 t = ld4v(Tb + to + 4 * c);
#pragma unroll
        for (int e = 0; e < 4; e++)
          if (4 * c + e < D) {
            const float df = __fsub_rn(f4get(f, e), f4get(t, e));
            dacc[j] = __dadd_rn(dacc[j], (double)__fmul_rn(df, df));
          }
      }
    }
    cst[j] = __double2float_rn(__dsqrt_rn(dacc[j]));
  }
  CostMat C;
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) C.v[i][j] = __shfl_sync(PLAS_FULL_MASK, cst[j], gbase + i);
  double bc;
  int bp;
  lane_best_exact(C, k, s, &bc, &bp);
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    const double oc = __shfl_xor_sync(PLAS_FULL_MASK, bc, o);
    const int op = __shfl_xor_sync(PLAS_FULL_MASK, bp, o);
    if (oc < bc || (oc == bc && op < bp)) {
      bc = oc;
      bp = op;
    }
  }
  // every arrangement sum +inf (fp32 costs overflowed): the reference keeps
  // best = 0, the identity (plas.py:138-146, strict < against best_cost = inf)
  return bp == 0x7fffffff ? 0 : bp;
}
// Out of line for the wide-row kernels (C3: 1.687 -> 1.664 s); inlined in the
// 16-float kernels, where the call's register save cost more (C2 110.7 ->
// 111.6 ms, C4 2.204 -> 2.248 s).
__device__ __noinline__ int decide_exact_call(const float* Fb, const float* Tb, const int (&rowj)[4], int D, int S,
                                              int k) {
  return decide_exact_body(Fb, Tb, rowj, D, S, k);
}

template <bool WIDE, bool TNC>
__device__ __forceinline__ int decide4(const float* Fb, const float* Tb, const int (&rowj)[4],
                                       const int (&rowt)[4], int D, int S, int k, float4 (&Fc)[4], int* exact,
                                       float (&col)[4]) {
  const int s = threadIdx.x & 3;
  const int nch = S >> 2;
  // fast-tier partial squared distances: acc[i][jj] holds the (even, odd)
  // channel halves as one f32x2 register, fed straight from the 8-byte halves
  // of the loaded chunks; pad channels (>= D) are zero in both rows
  unsigned long long acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0ull;
  const int rounds = WIDE ? (nch + 3) >> 2 : 1;
  for (int r = 0; r < rounds; r++) {
    const int c = 4 * r + s;
    float4 Tc[4];
    load_chunks<TNC>(Fb, Tb, rowj, rowt, S, c, c < nch, Fc, Tc);
    accum_chunks(acc, Fc, Tc);
  }
  return decide_from_acc<WIDE>(acc, Fb, Tb, rowj, D, S, k, exact, col);
}

// col[i] = the fast cost C[i][s] of slot i's element in target s (lane s of
// the group), returned for the DEVICE-mode pass statistic (k3_delta_acc).
template <bool OOL>  // exact tier out of line (wide rows)
__device__ __forceinline__ int decide_from_acc(const unsigned long long (&acc)[4][4], const float* Fb,
                                               const float* Tb, const int (&rowj)[4], int D, int S, int k,
                                               int* exact, float (&col)[4]) {
  const int lane = threadIdx.x & 31;
  const int s = lane & 3;
  const int gbase = lane & ~3;
  float part[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const float2 h = upk2(acc[i][j]);
      part[i][j] = h.x + h.y;
    }
  // reduce-scatter over the 4 lanes by column (rotated order, no selects):
  // lane s ends with column s of the cost matrix, col[i] = C[i][s]
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const float h0 = part[i][0] + __shfl_xor_sync(PLAS_FULL_MASK, part[i][2], 2);
    const float h1 = part[i][1] + __shfl_xor_sync(PLAS_FULL_MASK, part[i][3], 2);
    col[i] = sqrt_approx(h0 + __shfl_xor_sync(PLAS_FULL_MASK, h1, 1));
  }
  // lane s takes the arrangements that put slot 0's element in target s: it
  // needs C[i][o_q] for the other targets o_0 < o_1 < o_2, i.e. column o_q's
  // entry i, shuffled from lane o_q (a per-lane source, no selects)
  const int o3[3] = {s == 0 ? 1 : 0, s <= 1 ? 2 : 1, s <= 2 ? 3 : 2};
  float x[4][3];
#pragma unroll
  for (int i = 1; i < 4; i++)
#pragma unroll
    for (int q = 0; q < 3; q++) x[i][q] = __shfl_sync(PLAS_FULL_MASK, col[i], gbase + o3[q]);
  float b1, b2;
  int bp;
  lane_best_fast_cols(col[0], x, k, s, &b1, &bp, &b2);
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    const float ob1 = __shfl_xor_sync(PLAS_FULL_MASK, b1, o);
    const int op = __shfl_xor_sync(PLAS_FULL_MASK, bp, o);
    const float ob2 = __shfl_xor_sync(PLAS_FULL_MASK, b2, o);
    const bool take = ob1 < b1 || (ob1 == b1 && op < bp);
    const float lose = take ? b1 : ob1;  // the loser's best is a candidate for second
    b2 = fminf(fminf(b2, ob2), lose);
    if (take) {
      b1 = ob1;
      bp = op;
    }
  }
  // relative: 2 (D+24) 2^-24 for the fp32 roundings; absolute: a cost whose
  // sum of squares lies below the normal fp32 range (2^-126) carries an error
  // up to its own size, < 1.1e-19, in both the fast and the reference
  // arithmetic -- 4e-18 covers four of them on each side.  b2 = -inf: an
  // overflowed fast sum (lane_best_fast_cols).
  const float margin = 2.0f * (float)(D + 24) * 5.9604645e-08f;
  const bool certain =
      k < 2 || (b2 < __int_as_float(0x7f800000) && b2 > 1e-30f && (b2 - b1) > margin * b2 + 4e-18f);
  if (__any_sync(PLAS_FULL_MASK, !certain)) {
    bp = OOL ? decide_exact_call(Fb, Tb, rowj, D, S, k) : decide_exact_body(Fb, Tb, rowj, D, S, k);
    if (s == 0 && k >= 2 && !certain) *exact += 1;
  }
  return k < 2 ? 0 : bp;
}

// Grouping-table entry (pack_local: (ly << 16) | lx) of slot s of quad q of a
// block of class cls.  PARITY: the filtered master permutation
// (plas.py:209, class_select_kernel); DEVICE: the keyed bijection tabulated by
// gen_class_tables (the caller passes the buffer of this pass's parity).
__device__ __forceinline__ unsigned group_entry(const int* __restrict__ sel, long long sel_stride, int cls,
                                                unsigned q, int s) {
  return (unsigned)__ldg(sel + (long long)cls * sel_stride + 4 * q + s);
}
#ifdef PLAS_DEBUG_BOUNDS
#define PLAS_DBG_E(e) e_
#else
#define PLAS_DBG_E(e) e
#endif
__device__ __forceinline__ int entry_cell_off(unsigned e, int side) { return (int)(e >> 16) * side + (int)(e & 0xffffu); }
__device__ __forceinline__ int entry_row(unsigned e, int ww) { return (int)(e >> 16) * ww + (int)(e & 0xffffu); }

// Element indices follow their rows.  Lazy (Ctrl.lazy_idx, large grids): a
// lane reads its cell's index only when its element moves (after the
// decision, ~4-6 % of cells per pass) instead of gathering every cell's index
// with the rows -- a random 4-byte read costs a 32-byte sector, ~130 MB per
// C4 pass from DRAM (C4 2.245 -> 2.205 s); on small grids the index array
// stays in L2 and the early read hides its latency (C2 110.4 vs 111.6 ms
// lazy).  The warp reads all moving indices before any lane writes.
__device__ __forceinline__ void move_index(int* __restrict__ idx, bool my_mv, int cell, int dcell, int eager,
                                           bool lazy) {
  int v = eager;
  if (lazy && my_mv) v = idx[cell];
  __syncwarp();
  if (my_mv) idx[dcell] = v;
}

// Moved-cell list: CTAs stage the destination cells of their moves in shared
// memory and append them to list[] with one reservation on *count per flush.
struct MoveOut {
  int* list;
  int* count;                // moved cells of the pass (the list length when the list is staged)
  unsigned long long* acc;   // DEVICE mode: the pass's 128-bit fixed-point distance change
};

constexpr int WARP_LIST = 512;  // shared staging entries per warp
#ifndef K3_MINB
#define K3_MINB 4
#endif

// Append this lane's moved cell (if mv) to its warp's staging segment; the
// warp-uniform fill level lives in *wcnt (a register in every lane).  A full
// segment is flushed by the warp with one global reservation.
template <int CAP = WARP_LIST>
__device__ __forceinline__ void stage_move(bool mv, int cell, int* wlist, int* wcnt, const MoveOut& mo) {
  const unsigned bal = __ballot_sync(PLAS_FULL_MASK, mv);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  if (mv) wlist[*wcnt + __popc(bal & ((1u << lane) - 1u))] = cell;
  *wcnt += __popc(bal);
  if (*wcnt > CAP - 32) {
    __syncwarp();
    int base = 0;
    if (lane == 0) base = atomicAdd(mo.count, *wcnt);
    base = __shfl_sync(PLAS_FULL_MASK, base, 0);
    for (int i = lane; i < *wcnt; i += 32) mo.list[base + i] = wlist[i];
    __syncwarp();
    *wcnt = 0;
  }
}

// CTA-wide: append every warp's remaining entries with one reservation
template <int CAP = WARP_LIST>
__device__ __forceinline__ void flush_moves(const MoveOut& mo, int* s_list, int wcnt, int* s_wcnt,
                                            int* s_base) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) s_wcnt[wid] = wcnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < nw; w++) tot += s_wcnt[w];
    *s_base = tot ? atomicAdd(mo.count, tot) : 0;
  }
  __syncthreads();
  int off = *s_base;
  for (int w = 0; w < wid; w++) off += s_wcnt[w];
  for (int i = lane; i < wcnt; i += 32) mo.list[off + i] = s_list[wid * CAP + i];
}

// DEVICE-mode pass statistic, formed in K3 (no moved-cell list, no per-cell
// distance recomputation).  Lane s of a group holds column s of the fast cost
// matrix (col[i] = C[i][s], decide_from_acc); when the decision brings slot
// src's element into target s, that cell's distance changes by
// C[src][s] - C[s][s].  Each change is rounded to a multiple of 2^-64 (fx64)
// and summed as a 128-bit integer, so the pass total does not depend on which
// lane, CTA or rank handled the group: DEVICE sorts repeat bit for bit and a
// sharded sort sums to the 1-GPU total.  The fast costs are within
// (D/2 + 7) 2^-24 (relative) of the reference's, so the running mean drifts
// from grid_distance by < 1e-6 of the moved cells' distance per pass and is
// re-anchored exactly at every level start (level_stats_kernel); changes that
// are not finite or beyond fx64's range (|change| >= 2^86: fp32 costs that
// overflowed) are dropped.  PARITY mode keeps the exact per-cell fp64 changes
// (pass_stats_kernel over the moved-cell list): its strike decisions must be
// the reference's.
__device__ __forceinline__ void k3_delta_acc(const float (&col)[4], unsigned code, int s, __int128* q) {
  int src = s;
#pragma unroll
  for (int i = 0; i < 4; i++)
    if (((code >> (2 * i)) & 3u) == (unsigned)s) src = i;
  if (src != s) {
    const double dd = (double)pick4(col, src) - (double)pick4(col, s);
    if (fabs(dd) < 7.7371252455336267e25) *q += fx64(dd);  // 2^86
  }
}

// End of a pass kernel: the CTA's moved-cell count and (DEVICE) its 128-bit
// distance change, one atomic each per CTA.  Called by every thread.
template <bool KD>
__device__ __forceinline__ void k3_cta_epilogue(const MoveOut& mo, int nmv, __int128 q) {
  __shared__ __int128 sq[32];
  __shared__ int sn[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  nmv = __reduce_add_sync(PLAS_FULL_MASK, nmv);
  if (KD) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += shfl_xor_i128(q, o);
  }
  if (lane == 0) {
    sn[wid] = nmv;
    if (KD) sq[wid] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    __int128 b = 0;
    for (int w = 0; w < nw; w++) {
      t += sn[w];
      if (KD) b += sq[w];
    }
    if (t) atomicAdd(mo.count, t);
    if (KD && b != 0) {
      const unsigned long long lo = (unsigned long long)b;
      const unsigned long long old = atomicAdd(mo.acc, lo);
      const unsigned long long carry = old + lo < old ? 1ull : 0ull;
      atomicAdd(mo.acc + 1, (unsigned long long)((unsigned __int128)b >> 64) + carry);
    }
  }
}

// per-pass class tables in shared memory
struct PassShared {
  int seg[6];
  int wcnt[32];
  int base;
};

__device__ __forceinline__ void load_pass_shared(PassShared& ps, const Ctrl* __restrict__ ctrl) {
  if (threadIdx.x < 3) {
    ps.seg[threadIdx.x] = ctrl->seg_h[threadIdx.x];
    ps.seg[3 + threadIdx.x] = ctrl->seg_w[threadIdx.x];
  }
  __syncthreads();
}

// Per-pass kernel (gather regime): CTA iteration = 64 consecutive groups of
// the pass (8 warps x 8 groups); group g -> (block, quad) -> 4 cells.
// PARITY: the class grouping is the filtered master permutation
//   sel[cls][...] (plas.py:209, built by class_select_kernel).
// DEVICE: the class grouping is a keyed bijection on [0, m) (Ctrl.fe_*).
template <bool WIDE, bool PARITY>
__global__ void __launch_bounds__(256, WIDE ? 2 : K3_MINB) pass_kernel(float* __restrict__ feat, int* __restrict__ idx,
                                                       const float* __restrict__ target, int D, int S,
                                                       const Ctrl* __restrict__ ctrl,
                                                       const int* __restrict__ sel, long long sel_stride,
                                                       MoveOut mo, int* __restrict__ counters) {
  __shared__ PassShared ps;
  __shared__ int s_list[8 * WARP_LIST];
  if (ctrl->level_done) return;  // an unrolled pass slot after the level ended
  gtrace_mark(ctrl, 0);
  load_pass_shared(ps, ctrl);
  // DEVICE: the grouping tables of this pass's parity (gen_class_tables)
  const int* selp = PARITY ? sel : sel + (long long)(ctrl->pass & 1) * 9 * sel_stride;
  if (!PARITY && blockIdx.x == 0 && threadIdx.x == 0) {
    const_cast<Ctrl*>(ctrl)->gen_pass = ctrl->pass + 1;
    const_cast<Ctrl*>(ctrl)->gen_level = ctrl->level;
  }
  int* wlist = s_list + (threadIdx.x >> 5) * WARP_LIST;
  int wcnt = 0;
  const int side = ctrl->side;
  const int beta = ctrl->beta;
  const bool lazy = ctrl->lazy_idx != 0;
  const int fy = ctrl->first_y, fx = ctrl->first_x;
  const int nby = ctrl->nby, nbx = ctrl->nbx;
  const unsigned cap = (unsigned)ctrl->cap;
  const unsigned g_lo = (unsigned)ctrl->g_lo, total = (unsigned)ctrl->g_hi;  // this rank's groups
  const unsigned cap_m = ctrl->cap_m, nbx_m = ctrl->nbx_m;
  const int cap_l = ctrl->cap_l, nbx_l = ctrl->nbx_l;
  const int nch = S >> 2;
  const int lane = threadIdx.x & 31, s = lane & 3, gl = threadIdx.x >> 2;
  int exact = 0;
  // the moved-cell list: PARITY (the statistics kernel recomputes the moved
  // cells' exact distances) and sharded sorts (the exchange); DEVICE mode on
  // one GPU only counts the moves
  const bool stage = PARITY || ctrl->world > 1;
  int nmv = 0;
  __int128 dq = 0;  // DEVICE: this lane's fixed-point distance change (k3_delta_acc)
  // geometry of group g for lane slot s; the table entry load is issued here
  // and consumed one iteration later (prefetch)
  struct Geo {
    int k, base;  // slot count, block origin cell
    unsigned e;   // this lane's table entry (pack_local)
  };
  auto geo = [&](unsigned g) {
    Geo o{0, 0, 0u};
    if (g < total) {
      const unsigned b = fastdiv(g, cap_m, cap_l);
      const unsigned q = g - b * cap;
      const unsigned by = fastdiv(b, nbx_m, nbx_l);
      const unsigned bx = b - by * (unsigned)nbx;
      const int ty = by == 0 ? 0 : (by == (unsigned)nby - 1 ? 2 : 1);
      const int tx = bx == 0 ? 0 : (bx == (unsigned)nbx - 1 ? 2 : 1);
      const int hh = ps.seg[ty], ww = ps.seg[3 + tx];
      const int rem = hh * ww - 4 * (int)q;
      if (rem >= 2) {  // a single leftover cell never moves
        o.k = rem >= 4 ? 4 : rem;
        const int y0 = by == 0 ? 0 : fy + ((int)by - 1) * beta;
        const int x0 = bx == 0 ? 0 : fx + ((int)bx - 1) * beta;
        o.base = y0 * side + x0;
        if (s < o.k) o.e = group_entry(selp, sel_stride, ty * 3 + tx, q, s);
      }
    }
    return o;
  };
  Geo gnext = geo(g_lo + blockIdx.x * 64u + gl);
  for (unsigned base = g_lo + blockIdx.x * 64u; base < total; base += gridDim.x * 64u) {
    const Geo gc = gnext;
    gnext = geo(base + gridDim.x * 64u + gl);
    const int k = gc.k;
    const int cell = s < k ? gc.base + entry_cell_off(gc.e, side) : 0;
    // this lane's element index, needed only if its cell moves (loaded with the rows)
    const int my_idx0 = (!lazy && s < k) ? idx[cell] : 0;
    int rowj[4], rowt[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      rowj[j] = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + j);
      rowt[j] = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + (j ^ s));
    }
    float4 Fc[4];
    float col[4];
    const int bp = decide4<WIDE, true>(feat, target, rowj, rowt, D, S, k, Fc, &exact, col);
    const unsigned code = perm_dest_code(k, bp);
    if (!PARITY) k3_delta_acc(col, code, s, &dq);
    int dst[4], dcl[4];
    bool mv[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      dst[i] = (int)((code >> (2 * i)) & 3u);
      mv[i] = dst[i] != i;
      dcl[i] = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + dst[i]);  // destination cell of slot i
    }
    const int my_dst = (int)((code >> (2 * s)) & 3u);
    const bool my_mv = my_dst != s;
    const int my_idx = my_idx0;
    __syncwarp();
    if (!WIDE) {
      if (s < nch) {
#pragma unroll
        for (int i = 0; i < 4; i++)
          if (mv[i]) st4(feat + (unsigned)dcl[i] * (unsigned)S + 4 * s, Fc[i]);
      }
    } else {
      // chunk columns: every read of a column precedes its writes
      for (int r = 0; r < (nch + 3) >> 2; r++) {
        const int c = 4 * r + s;
        float4 f[4];
#pragma unroll
        for (int i = 0; i < 4; i++) f[i] = (mv[i] && c < nch) ? ld4v(feat + (long long)rowj[i] * S + 4 * c) : f4zero();
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; i++)
          if (mv[i] && c < nch) st4(feat + (long long)pick4(rowj, dst[i]) * S + 4 * c, f[i]);
        __syncwarp();
      }
    }
    const int dcell = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + my_dst);
    move_index(idx, my_mv, cell, dcell, my_idx, lazy);
    if (stage)
      stage_move(my_mv, dcell, wlist, &wcnt, mo);
    else
      nmv += my_mv;
  }
  if (stage) flush_moves(mo, s_list, wcnt, ps.wcnt, &ps.base);
  k3_cta_epilogue<!PARITY>(mo, nmv, dq);
  const int ex = __reduce_add_sync(PLAS_FULL_MASK, exact);
  if (lane == 0 && ex) atomicAdd(counters + 1, ex);
  gtrace_mark(ctrl, 1);
}

// Gather-regime pass kernel for rows of <= 16 floats, software-pipelined: the
// rows (and element indices) of a team's next group are loaded into registers
// before the current group is decided, so every warp keeps one group's
// gathers in flight while it computes (the plain form waited for them with
// all its warps in the same phase: long-scoreboard stalls dominated).  The
// early loads touch other groups' cells only (a pass's groups are disjoint,
// plas.py:118-121), so they never race with this group's moves.  Same
// decisions and table layout as pass_kernel.
#ifndef K3P_MINB
#define K3P_MINB 2
#endif
template <bool PARITY>
__global__ void __launch_bounds__(256, K3P_MINB) pass_kernel_pipe(float* __restrict__ feat, int* __restrict__ idx,
                                                                  const float* __restrict__ target, int D, int S,
                                                                  const Ctrl* __restrict__ ctrl,
                                                                  const int* __restrict__ sel, long long sel_stride,
                                                                  MoveOut mo, int* __restrict__ counters) {
  __shared__ PassShared ps;
  __shared__ int s_list[8 * WARP_LIST];
  if (ctrl->level_done) return;  // an unrolled pass slot after the level ended
  gtrace_mark(ctrl, 0);
  load_pass_shared(ps, ctrl);
  const int* selp = PARITY ? sel : sel + (long long)(ctrl->pass & 1) * 9 * sel_stride;
  if (!PARITY && blockIdx.x == 0 && threadIdx.x == 0) {
    const_cast<Ctrl*>(ctrl)->gen_pass = ctrl->pass + 1;
    const_cast<Ctrl*>(ctrl)->gen_level = ctrl->level;
  }
  int* wlist = s_list + (threadIdx.x >> 5) * WARP_LIST;
  int wcnt = 0;
  const int side = ctrl->side;
  const int beta = ctrl->beta;
  const bool lazy = ctrl->lazy_idx != 0;
  const int fy = ctrl->first_y, fx = ctrl->first_x;
  const int nby = ctrl->nby, nbx = ctrl->nbx;
  const unsigned cap = (unsigned)ctrl->cap;
  const unsigned g_lo = (unsigned)ctrl->g_lo, total = (unsigned)ctrl->g_hi;  // this rank's groups
  const unsigned cap_m = ctrl->cap_m, nbx_m = ctrl->nbx_m;
  const int cap_l = ctrl->cap_l, nbx_l = ctrl->nbx_l;
  const int nch = S >> 2;
  const int lane = threadIdx.x & 31, s = lane & 3, gl = threadIdx.x >> 2;
  const bool cvalid = s < nch;
  int exact = 0;
  const bool stage = PARITY || ctrl->world > 1;  // moved-cell list (see pass_kernel)
  int nmv = 0;
  __int128 dq = 0;
  // Group g's slot count, block origin and this lane's table entry.  The
  // entry load is issued two groups ahead (pre), so its L2 latency is not
  // exposed between the geometry and the row gathers that depend on it.
  struct Pre {
    int k, base;
    unsigned e;
#ifdef PLAS_DEBUG_BOUNDS
    int hh, ww;
#endif
  };
  auto group_pre = [&](unsigned g) {
    Pre o;
    o.k = 0;
    o.base = 0;
    o.e = 0u;
    if (g < total) {
      const unsigned b = fastdiv(g, cap_m, cap_l);
      const unsigned q = g - b * cap;
      const unsigned by = fastdiv(b, nbx_m, nbx_l);
      const unsigned bx = b - by * (unsigned)nbx;
      const int ty = by == 0 ? 0 : (by == (unsigned)nby - 1 ? 2 : 1);
      const int tx = bx == 0 ? 0 : (bx == (unsigned)nbx - 1 ? 2 : 1);
      const int hh = ps.seg[ty], ww = ps.seg[3 + tx];
      const int rem = hh * ww - 4 * (int)q;
      if (rem >= 2) {  // a single leftover cell never moves
        o.k = rem >= 4 ? 4 : rem;
        const int y0 = by == 0 ? 0 : fy + ((int)by - 1) * beta;
        const int x0 = bx == 0 ? 0 : fx + ((int)bx - 1) * beta;
        o.base = y0 * side + x0;
        if (s < o.k) o.e = group_entry(selp, sel_stride, ty * 3 + tx, q, s);
#ifdef PLAS_DEBUG_BOUNDS
        o.hh = hh;
        o.ww = ww;
#endif
      }
    }
    return o;
  };
  // (slot count, this lane's cell); cell 0 for absent slots
  auto group_cell = [&](const Pre& o, int* k) {
    *k = o.k;
    int cell = s < o.k ? o.base + entry_cell_off(o.e, side) : 0;
#ifdef PLAS_DEBUG_BOUNDS
    if (s < o.k && ((int)(o.e >> 16) >= o.hh || (int)(o.e & 0xffffu) >= o.ww || cell < 0 || cell >= side * side)) {
      printf("K3pipe bad entry: lvl %d pass %d s %d e %08x hh %d ww %d cell %d\n", ctrl->level, ctrl->pass, s, o.e,
             o.hh, o.ww, cell);
      cell = o.base;
    }
#endif
    return cell;
  };
  const unsigned stride = gridDim.x * 64u;
  unsigned g = g_lo + blockIdx.x * 64u + gl;
  int k;
  int cell = group_cell(group_pre(g), &k);
  Pre pre = group_pre(g + stride);  // the next group's entry, in flight
  int rowj[4], rowt[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    rowj[j] = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + j);
    rowt[j] = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + (j ^ s));
  }
  float4 Fc[4], Tc[4];
  load_chunks<true>(feat, target, rowj, rowt, S, s, cvalid, Fc, Tc);
  int my_idx = (!lazy && s < k) ? idx[cell] : 0;
  for (unsigned base = g_lo + blockIdx.x * 64u; base < total; base += stride) {
    // ---- the next group's gathers go out first
    g += stride;
    int nk;
    const int ncell = group_cell(pre, &nk);
    int nrowj[4], nrowt[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      nrowj[j] = __shfl_sync(PLAS_FULL_MASK, ncell, (lane & ~3) + j);
      nrowt[j] = __shfl_sync(PLAS_FULL_MASK, ncell, (lane & ~3) + (j ^ s));
    }
    float4 nFc[4], nTc[4];
    load_chunks<true>(feat, target, nrowj, nrowt, S, s, cvalid, nFc, nTc);
    pre = group_pre(g + stride);  // the entry of the group after next
    const int nidx = (!lazy && s < nk) ? idx[ncell] : 0;
    // ---- decide and apply the current group
    unsigned long long acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) acc[i][j] = 0ull;
    accum_chunks(acc, Fc, Tc);
    float col[4];
    const int bp = decide_from_acc<false>(acc, feat, target, rowj, D, S, k, &exact, col);
    const unsigned code = perm_dest_code(k, bp);
    if (!PARITY) k3_delta_acc(col, code, s, &dq);
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int dst = (int)((code >> (2 * i)) & 3u);
      const int dcl = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + dst);  // destination cell of slot i
      if (dst != i && cvalid) st4(feat + (unsigned)dcl * (unsigned)S + 4 * s, Fc[i]);
    }
    const int my_dst = (int)((code >> (2 * s)) & 3u);
    const bool my_mv = my_dst != s;
    const int dcell = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + my_dst);
    move_index(idx, my_mv, cell, dcell, my_idx, lazy);
    if (stage)
      stage_move(my_mv, dcell, wlist, &wcnt, mo);
    else
      nmv += my_mv;
    // ---- rotate
    k = nk;
    cell = ncell;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      rowj[j] = nrowj[j];
      Fc[j] = nFc[j];
      Tc[j] = nTc[j];
    }
    my_idx = nidx;
  }
  if (stage) flush_moves(mo, s_list, wcnt, ps.wcnt, &ps.base);
  k3_cta_epilogue<!PARITY>(mo, nmv, dq);
  const int ex = __reduce_add_sync(PLAS_FULL_MASK, exact);
  if (lane == 0 && ex) atomicAdd(counters + 1, ex);
  gtrace_mark(ctrl, 1);
}

// Tile-regime pass kernel (small blocks).  A CTA walks blocks b = blockIdx.x,
// +gridDim.x, ... through a TILE_NST-stage shared-memory ring.  A dedicated
// producer warp (warp 8) streams each block's feature and target rows in with
// bulk copies (cp.async.bulk, one per block row and array, counted on the
// stage's "full" mbarrier) as soon as the eight consumer warps have released
// the stage on its "empty" mbarrier; the consumers decide the block's groups
// from shared memory.  Staging costs a few producer instructions per block
// row, no CTA-wide barrier per block, and every block row is contiguous in HBM
// (ww * S floats), so the copies stream.  Element indices are read per group
// from global memory (only moved cells write them back).  Only moved rows are
// written back, from registers (rows <= 16 floats) or the staged copy, so
// in-place swaps need no ordering.  Same decisions as pass_kernel.
// Measured at C2 (beta = 16 passes): 42.6 us with warp 0's lanes issuing the
// copies between their own decisions, 39.6 us with the producer warp; three
// or four stages (fewer CTAs per SM) 48 / 73 us.
constexpr int TILE_THREADS = 256;                    // consumer threads (8 warps)
constexpr int TILE_CTA_THREADS = TILE_THREADS + 32;  // + the producer warp
constexpr int TILE_WARP_LIST = 128;  // moved-cell staging per warp in the tile kernel
#ifndef TILE_NST
#define TILE_NST 2
#endif
#ifndef TILE_MINB
#define TILE_MINB (TILE_NST == 2 ? 3 : 2)
#endif

// bytes of one pipeline stage for blocks of up to bmax x bmax cells (F rows, T rows)
__host__ __device__ __forceinline__ long long tile_stage_bytes(int bmax, int S) {
  const long long m = (long long)bmax * bmax;
  return (2 * m * S * 4 + 127) / 128 * 128;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

struct TileGeom {
  int y0, x0, hh, ww, cls;
};

__device__ __forceinline__ TileGeom tile_geom(int b, int nbx, unsigned nbx_m, int nbx_l, int nby, int fy, int fx,
                                              int beta, const int* seg) {
  TileGeom g;
  const int by = (int)fastdiv((unsigned)b, nbx_m, nbx_l), bx = b - by * nbx;
  const int ty = by == 0 ? 0 : (by == nby - 1 ? 2 : 1);
  const int tx = bx == 0 ? 0 : (bx == nbx - 1 ? 2 : 1);
  g.hh = seg[ty];
  g.ww = seg[3 + tx];
  g.y0 = by == 0 ? 0 : fy + (by - 1) * beta;
  g.x0 = bx == 0 ? 0 : fx + (bx - 1) * beta;
  g.cls = ty * 3 + tx;
  return g;
}

template <bool WIDE, bool PARITY>
__global__ void __launch_bounds__(TILE_CTA_THREADS, WIDE ? 2 : TILE_MINB) tile_pass_kernel(
    float* __restrict__ feat, int* __restrict__ idx, const float* __restrict__ target, int D, int S,
    const Ctrl* __restrict__ ctrl, const int* __restrict__ sel, long long sel_stride, MoveOut mo,
    int* __restrict__ counters) {
  extern __shared__ __align__(128) float4 smem4[];
  __shared__ PassShared ps;
  __shared__ int s_list[9 * TILE_WARP_LIST];  // small lists: 3 CTAs per SM fit in shared memory
  __shared__ unsigned long long s_full[TILE_NST], s_empty[TILE_NST];
  if (ctrl->level_done) return;  // an unrolled pass slot after the level ended
  gtrace_mark(ctrl, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < TILE_NST; i++) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], TILE_THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  load_pass_shared(ps, ctrl);  // (its __syncthreads also publishes the barriers)
  // DEVICE: the grouping tables of this pass's parity (gen_class_tables)
  const int* selp = PARITY ? sel : sel + (long long)(ctrl->pass & 1) * 9 * sel_stride;
  if (!PARITY && blockIdx.x == 0 && threadIdx.x == 0) {
    const_cast<Ctrl*>(ctrl)->gen_pass = ctrl->pass + 1;
    const_cast<Ctrl*>(ctrl)->gen_level = ctrl->level;
  }
  int* wlist = s_list + (threadIdx.x >> 5) * TILE_WARP_LIST;
  int wcnt = 0;
  const int side = ctrl->side;
  const int beta = ctrl->beta;
  const bool lazy = ctrl->lazy_idx != 0;
  const int fy = ctrl->first_y, fx = ctrl->first_x;
  const int nby = ctrl->nby, nbx = ctrl->nbx;
  const unsigned nbx_m = ctrl->nbx_m;
  const int nbx_l = ctrl->nbx_l;
  const int b_lo = ctrl->b_lo, nblocks = ctrl->b_hi;  // this rank's blocks
  const int nch = S >> 2;
  const int mmax = beta * beta;
  const int stage_floats = (int)(tile_stage_bytes(beta, S) / 4);
  float* stage_base = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31, s = lane & 3, gl = threadIdx.x >> 2;
  const int first = b_lo + blockIdx.x;
  const int G = gridDim.x;

  int exact = 0;
  const bool stage = PARITY || ctrl->world > 1;  // moved-cell list (see pass_kernel)
  int nmv = 0;
  __int128 dq = 0;
  if (threadIdx.x >= TILE_THREADS) {
    // ---- producer warp: block it of this CTA into stage it % TILE_NST once
    // the consumers released that stage's previous block (bulk copies are
    // uniform-datapath instructions, so one lane issues them all)
    if (lane == 0) {
      for (int it = 0; first + it * G < nblocks; it++) {
        const int b = first + it * G;
        const int st = it % TILE_NST;
        if (it >= TILE_NST) mbar_wait(&s_empty[st], (unsigned)((it / TILE_NST - 1) & 1));
        const TileGeom g = tile_geom(b, nbx, nbx_m, nbx_l, nby, fy, fx, beta, ps.seg);
        const unsigned rowb = (unsigned)(g.ww * S * 4);
        mbar_expect_tx(&s_full[st], 2u * rowb * (unsigned)g.hh);
        float* sF = stage_base + st * stage_floats;
        float* sT = sF + mmax * S;
        unsigned go = ((unsigned)g.y0 * (unsigned)side + (unsigned)g.x0) * (unsigned)S;
        const unsigned gstep = (unsigned)side * (unsigned)S, sstep = (unsigned)(g.ww * S);
        unsigned so = 0u;
        for (int r = 0; r < g.hh; r++, go += gstep, so += sstep) {
          bulk_g2s(sF + so, feat + go, rowb, &s_full[st]);
          bulk_g2s(sT + so, target + go, rowb, &s_full[st]);
        }
      }
    }
  } else
  for (int it = 0; first + it * G < nblocks; it++) {
    const int b = first + it * G;
    const int st = it % TILE_NST;
    mbar_wait(&s_full[st], (unsigned)((it / TILE_NST) & 1));  // block b's rows have landed
    const TileGeom g = tile_geom(b, nbx, nbx_m, nbx_l, nby, fy, fx, beta, ps.seg);
    const float* sF = stage_base + st * stage_floats;
    const float* sT = sF + mmax * S;
    const int m = g.hh * g.ww;
    const int ngroups = (m + 3) >> 2;
    const int origin = g.y0 * side + g.x0;
    // slot count and table entry of group q (the entry of the next group is
    // loaded one iteration ahead)
    auto group_at = [&](int q, int* k, unsigned* e) {
      *k = 0;
      *e = 0u;
      if (q < ngroups) {
        const int rem = m - 4 * q;
        if (rem >= 2) *k = rem >= 4 ? 4 : rem;
        if (s < *k) *e = group_entry(selp, sel_stride, g.cls, (unsigned)q, s);
      }
    };
    int knext;
    unsigned enext;
    group_at(gl, &knext, &enext);
    for (int q0 = 0; q0 < ngroups; q0 += TILE_THREADS / 4) {
      const int k = knext;
      const unsigned e = enext;
      group_at(q0 + TILE_THREADS / 4 + gl, &knext, &enext);
#ifdef PLAS_DEBUG_BOUNDS
      unsigned e_ = e;
      if (s < k && ((int)(e >> 16) >= g.hh || (int)(e & 0xffffu) >= g.ww)) {
        printf("K3tile bad entry: lvl %d pass %d cls %d q %d s %d e %08x hh %d ww %d\n", ctrl->level, ctrl->pass,
               g.cls, q0 + gl, s, e, g.hh, g.ww);
        e_ = 0u;
      }
      const int mycell = origin + entry_cell_off(e_, side);
#else
      const int mycell = origin + entry_cell_off(e, side);
#endif
      const int my_idx = (!lazy && s < k) ? __ldg(idx + mycell) : 0;  // consumed after the decision
      const int myrow = entry_row(PLAS_DBG_E(e), g.ww);
      int rowj[4], rowt[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        rowj[j] = __shfl_sync(PLAS_FULL_MASK, myrow, (lane & ~3) + j);
        rowt[j] = __shfl_sync(PLAS_FULL_MASK, myrow, (lane & ~3) + (j ^ s));
      }
      float4 Fc[4];
      float col[4];
      const int bp = decide4<WIDE, false>(sF, sT, rowj, rowt, D, S, k, Fc, &exact, col);
      const unsigned code = perm_dest_code(k, bp);
      if (!PARITY) k3_delta_acc(col, code, s, &dq);
      int dst[4];
      bool mv[4];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        dst[i] = (int)((code >> (2 * i)) & 3u);
        mv[i] = dst[i] != i;
      }
      int dcl[4];
#pragma unroll
      for (int i = 0; i < 4; i++) dcl[i] = __shfl_sync(PLAS_FULL_MASK, mycell, (lane & ~3) + dst[i]);
      if (!WIDE) {
        if (s < nch) {
#pragma unroll
          for (int i = 0; i < 4; i++)
            if (mv[i]) st4(feat + (unsigned)dcl[i] * (unsigned)S + 4 * s, Fc[i]);
        }
      } else {
        for (int c = s; c < nch; c += 4) {
#pragma unroll
          for (int i = 0; i < 4; i++)
            if (mv[i]) st4(feat + (unsigned)dcl[i] * (unsigned)S + 4 * c, ld4v(sF + (unsigned)rowj[i] * (unsigned)S + 4 * c));
        }
      }
      const int my_dst = (int)((code >> (2 * s)) & 3u);
      const bool my_mv = my_dst != s;
      const int dcell = __shfl_sync(PLAS_FULL_MASK, mycell, (lane & ~3) + my_dst);
      move_index(idx, my_mv, mycell, dcell, my_idx, lazy);
      if (stage)
        stage_move<TILE_WARP_LIST>(my_mv, dcell, wlist, &wcnt, mo);
      else
        nmv += my_mv;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[st]);  // this warp is done with stage st
  }
  if (stage) flush_moves<TILE_WARP_LIST>(mo, s_list, wcnt, ps.wcnt, &ps.base);
  k3_cta_epilogue<!PARITY>(mo, nmv, dq);
  const int ex = __reduce_add_sync(PLAS_FULL_MASK, exact);
  if (lane == 0 && ex) atomicAdd(counters + 1, ex);
  gtrace_mark(ctrl, 1);
}

// Parity mode: per class (ty, tx) the stable filter master_perm[master_perm < m]
// (plas.py:209), stored as pack_local entries.  One CTA per class; master perm
// of beta^2 entries.
__global__ void __launch_bounds__(1024) class_select_kernel(const int* __restrict__ mp,
                                                             const Ctrl* __restrict__ ctrl,
                                                             int* __restrict__ sel,
                                                             long long sel_stride) {
  __shared__ int counts[1024];
  const int cls = blockIdx.x;
  const int ty = cls / 3, tx = cls % 3;
  const int beta = ctrl->beta;
  const int nby = ctrl->nby, nbx = ctrl->nbx;
  // class exists?  type 0 = first segment, 2 = last (needs >= 2 segments), 1 = interior (>= 3)
  auto exists = [](int t, int n) { return t == 0 || (t == 2 && n >= 2) || (t == 1 && n >= 3); };
  if (!exists(ty, nby) || !exists(tx, nbx)) return;
  const unsigned ww = (unsigned)ctrl->seg_w[tx];
  const long long m = (long long)ctrl->seg_h[ty] * ww;
  const long long n = (long long)beta * beta;
  const long long per = (n + blockDim.x - 1) / blockDim.x;
  const long long s0 = threadIdx.x * per, s1 = min(n, s0 + per);
  int cnt = 0;
  for (long long i = s0; i < s1; i++) cnt += mp[i] < m;
  counts[threadIdx.x] = cnt;
  __syncthreads();
  // inclusive scan (Hillis-Steele on 1024 entries)
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
    if (v < m) out[pos++] = pack_local((unsigned)v, ww);
  }
}

// ABI kernel for _assign_groups on an explicit (G, k) group list (plas.py:113-156).
template <bool WIDE>
__global__ void __launch_bounds__(256) groups_kernel(float* __restrict__ feat,
                                                     long long* __restrict__ idx,
                                                     const float* __restrict__ target, int D, int S,
                                                     const long long* __restrict__ groups,
                                                     long long G, int kk) {
  const int lane = threadIdx.x & 31, s = lane & 3;
  const int nch = S >> 2;
  int exact = 0;
  const long long wstride = ((long long)gridDim.x * blockDim.x) >> 2;  // groups per grid iteration
  for (long long base = ((long long)blockIdx.x * blockDim.x) >> 2; base < G; base += wstride) {
    const long long g = base + (threadIdx.x >> 2);
    const int k = g < G ? kk : 0;
    const int cell = s < k ? (int)groups[g * kk + s] : 0;
    int rowj[4], rowt[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      rowj[j] = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + j);
      rowt[j] = __shfl_sync(PLAS_FULL_MASK, cell, (lane & ~3) + (j ^ s));
    }
    float4 Fc[4];
    float col[4];
    const int bp = decide4<WIDE, true>(feat, target, rowj, rowt, D, S, k, Fc, &exact, col);
    int dst[4];
    bool mv[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      dst[i] = i < k ? perm_dest(k, bp, i) : i;
      mv[i] = bp != 0 && i < k && dst[i] != i;
    }
    const bool my_mv = pick4(mv, s);
    const long long my_idx = my_mv ? idx[cell] : 0;
    __syncwarp();
    for (int r = 0; r < (nch + 3) >> 2; r++) {
      const int c = 4 * r + s;
      float4 f[4];
#pragma unroll
      for (int i = 0; i < 4; i++) f[i] = (mv[i] && c < nch) ? ld4v(feat + (long long)rowj[i] * S + 4 * c) : f4zero();
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; i++)
        if (mv[i] && c < nch) st4(feat + (long long)pick4(rowj, dst[i]) * S + 4 * c, f[i]);
      __syncwarp();
    }
    if (my_mv) idx[pick4(rowj, pick4(dst, s))] = my_idx;
  }
}

// ABI kernel for _assign_groups with a float64 target (plas.py:129-137 as
// numba compiles it when `target` is float64: feat[pi, d] - target[pj, d] is
// an fp64 difference of the widened fp32 feature, squared and summed in fp64;
// the cost is stored to the float32 cost matrix).  One thread per group (an
// API path, not the sort's hot loop); same first-strict-minimum rule.
__global__ void __launch_bounds__(256) groups_f64t_kernel(float* __restrict__ feat, long long* __restrict__ idx,
                                                          const double* __restrict__ target, int D, int S,
                                                          const long long* __restrict__ groups, long long G,
                                                          int kk) {
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < G;
       g += (long long)gridDim.x * blockDim.x) {
    long long cell[4] = {0, 0, 0, 0};
    for (int i = 0; i < kk; i++) cell[i] = groups[g * kk + i];
    float cost[4][4];
    for (int i = 0; i < kk; i++)
      for (int j = 0; j < kk; j++) {
        double acc = 0.0;
        for (int d = 0; d < D; d++) {
          const double df = __dsub_rn((double)feat[cell[i] * S + d], target[cell[j] * S + d]);
          acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
        cost[i][j] = __double2float_rn(__dsqrt_rn(acc));
      }
    int nperm = kk == 4 ? 24 : (kk == 3 ? 6 : 2);
    int best = 0;
    double best_cost = __longlong_as_double(0x7ff0000000000000ll);
    for (int p = 0; p < nperm; p++) {
      double c = 0.0;
      for (int i = 0; i < kk; i++) c = __dadd_rn(c, (double)cost[i][perm_dest(kk, p, i)]);
      if (c < best_cost) {
        best_cost = c;
        best = p;
      }
    }
    if (best == 0) continue;
    float held[4][64];  // rows of up to 64 channels on this path (checked by the ABI)
    long long hidx[4];
    for (int i = 0; i < kk; i++) {
      for (int d = 0; d < D; d++) held[i][d] = feat[cell[i] * S + d];
      hidx[i] = idx[cell[i]];
    }
    for (int i = 0; i < kk; i++) {
      const long long dst = cell[perm_dest(kk, best, i)];
      for (int d = 0; d < D; d++) feat[dst * S + d] = held[i][d];
      idx[dst] = hidx[i];
    }
  }
}

}  // namespace plas
