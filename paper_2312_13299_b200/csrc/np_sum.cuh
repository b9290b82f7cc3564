// NumPy-order grid_distance (plas.py:71-84) for PARITY mode and the API.
//
// The reference computes np.sqrt((diff ** 2).sum(axis=1)).mean() in float64.
// NumPy reduces a contiguous run of m values with pairwise_sum (numpy
// umath loops_utils): m < 8 -> a plain loop from 0.0; m <= 128 -> eight
// running sums r[j] += a[i + j] over the multiples of 8, combined as
// ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), then the tail added in
// order; m > 128 -> split at m2 = m / 2 rounded down to a multiple of 8 and the
// two halves added.  The row sums over D and the mean over n cells follow that
// tree (mean = sum / n), so with every product and add rounded explicitly
// (no FMA contraction) the result equals the reference's bit for bit
// (pinned in tests against numpy itself).
//
// On the GPU: one thread per cell forms sqrt(row sum) (np_cell_*_kernel); one
// thread per leaf of the n-cell tree (8 <= size <= 128) sums its run
// (np_leaf_kernel); one CTA adds the internal nodes level by level, deepest
// first (np_tree_kernel).  The tree depends on n only and is built on the host.
#pragma once
#include <vector>

#include "common.cuh"

namespace plas {

// pairwise_sum of m values v(0..m-1), NumPy's order.  `V` yields value k.
template <typename V>
__device__ __forceinline__ double np_pairwise_small(const V& v, int m) {
  if (m < 8) {
    double res = 0.0;
    for (int i = 0; i < m; i++) res = __dadd_rn(res, v(i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = v(j);
  int i = 8;
  for (; i < m - (m % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], v(i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < m; i++) res = __dadd_rn(res, v(i));
  return res;
}
template <typename V>
__device__ double np_pairwise(const V& v, int off, int m) {
  if (m <= 128) {
    auto w = [&](int k) { return v(off + k); };
    return np_pairwise_small(w, m);
  }
  int m2 = m / 2;
  m2 -= m2 % 8;
  return __dadd_rn(np_pairwise(v, off, m2), np_pairwise(v, off + m2, m - m2));
}

// sqrt(sum_d (f64(F_d) - f64(T_d))^2) per cell of the sort's fp32 rows (stride S)
__global__ void __launch_bounds__(256) np_cell_sort_kernel(const float* __restrict__ feat,
                                                           const float* __restrict__ target, long long n, int D,
                                                           int S, double* __restrict__ out) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const float* f = feat + c * S;
    const float* t = target + c * S;
    auto sq = [&](int d) {
      const double df = __dsub_rn((double)__ldg(f + d), (double)__ldg(t + d));
      return __dmul_rn(df, df);
    };
    out[c] = __dsqrt_rn(np_pairwise(sq, 0, D));
  }
}

// the same for the API's fp64 (n, D) arrays, optional per-channel weights
// (diff * weights, plas.py:81-83)
__global__ void __launch_bounds__(256) np_cell_f64_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                          const double* __restrict__ wts, long long n, int D,
                                                          double* __restrict__ out) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const double* x = a + c * D;
    const double* y = b + c * D;
    auto sq = [&](int d) {
      double df = __dsub_rn(__ldg(x + d), __ldg(y + d));
      if (wts) df = __dmul_rn(df, __ldg(wts + d));
      return __dmul_rn(df, df);
    };
    out[c] = __dsqrt_rn(np_pairwise(sq, 0, D));
  }
}

// Host: the n-cell pairwise tree.  Leaves (start, size) in order; internal
// node k (index nleaves + k) adds its children; `order` lists the internal
// nodes by height (deepest first), `hoff` the height boundaries.
struct NpTree {
  std::vector<long long> leaf_start;
  std::vector<int> leaf_len;
  std::vector<int> left, right;  // per internal node
  std::vector<int> order, hoff;
  int root = 0;
  long long n = 0;
};
inline int np_tree_build(NpTree* t, long long off, long long m) {
  if (m <= 128) {
    t->leaf_start.push_back(off);
    t->leaf_len.push_back((int)m);
    return -(int)t->leaf_start.size();  // leaf k -> -(k + 1)
  }
  long long m2 = m / 2;
  m2 -= m2 % 8;
  const int l = np_tree_build(t, off, m2);
  const int r = np_tree_build(t, off + m2, m - m2);
  t->left.push_back(l);
  t->right.push_back(r);
  return (int)t->left.size() - 1;  // internal k -> k
}
inline void np_tree_make(NpTree* t, long long n) {
  t->leaf_start.clear();
  t->leaf_len.clear();
  t->left.clear();
  t->right.clear();
  t->order.clear();
  t->hoff.clear();
  t->n = n;
  const int root = np_tree_build(t, 0, n);
  const int L = (int)t->leaf_start.size(), I = (int)t->left.size();
  auto idx = [&](int v) { return v < 0 ? (-v - 1) : L + v; };  // node index in the value array
  for (int k = 0; k < I; k++) {
    t->left[k] = idx(t->left[k]);
    t->right[k] = idx(t->right[k]);
  }
  t->root = idx(root);
  // heights (children precede parents in construction order), then the
  // internal nodes bucketed by height (counting sort)
  std::vector<int> h(L + I, 0);
  int hmax = 0;
  for (int k = 0; k < I; k++) {
    h[L + k] = 1 + std::max(h[t->left[k]], h[t->right[k]]);
    hmax = std::max(hmax, h[L + k]);
  }
  t->hoff.assign(hmax + 1, 0);
  for (int k = 0; k < I; k++) t->hoff[h[L + k]]++;  // hoff[lev] counts height lev (1..hmax)
  int acc = 0;
  for (int lev = 1; lev <= hmax; lev++) {
    const int c = t->hoff[lev];
    t->hoff[lev - 1] = acc;
    acc += c;
  }
  t->hoff[hmax] = acc;
  t->order.assign(I, 0);
  std::vector<int> pos(t->hoff.begin(), t->hoff.end());
  for (int k = 0; k < I; k++) t->order[pos[h[L + k] - 1]++] = k;
}

// leaf sums: vals[k] = pairwise sum of v[leaf_start[k] .. + leaf_len[k])
__global__ void __launch_bounds__(256) np_leaf_kernel(const double* __restrict__ v,
                                                      const long long* __restrict__ leaf_start,
                                                      const int* __restrict__ leaf_len, int nleaves,
                                                      double* __restrict__ vals) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nleaves; k += gridDim.x * blockDim.x) {
    const double* p = v + leaf_start[k];
    auto val = [&](int i) { return __ldg(p + i); };
    vals[k] = np_pairwise_small(val, leaf_len[k]);
  }
}

// one CTA: internal nodes height by height; out[0] = total, out[1] = total / n
__global__ void __launch_bounds__(1024) np_tree_kernel(double* __restrict__ vals, const int* __restrict__ left,
                                                       const int* __restrict__ right, const int* __restrict__ order,
                                                       const int* __restrict__ hoff, int nheights, int nleaves,
                                                       int root, long long n, double* __restrict__ out) {
  for (int lev = 0; lev < nheights; lev++) {
    for (int e = hoff[lev] + threadIdx.x; e < hoff[lev + 1]; e += blockDim.x) {
      const int k = order[e];
      vals[nleaves + k] = __dadd_rn(vals[left[k]], vals[right[k]]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tot = vals[root];
    out[0] = tot;
    out[1] = __ddiv_rn(tot, (double)n);
  }
}

// vad (metrics.py:25-40) in NumPy's order: diffs = concatenate(|diff(g, axis=0)|
// in C order of (H-1, W, C), |diff(g, axis=1)| in C order of (H, W-1, C));
// var = pairwise((d - mean)^2) / M with mean = pairwise(d) / M (numpy _var:
// sum, true_divide, subtract, multiply, sum, true_divide).  Element e of the
// pooled array is formed on the fly from the fp32 grid (row stride S).
template <typename T = float>
struct VadElems {
  const T* g;
  unsigned H, W, C, S;
  unsigned long long m0;  // (H - 1) W C axis-0 differences first
  __device__ __forceinline__ double operator()(unsigned long long e) const {
    unsigned long long y, x, c;
    const T* a;
    const T* b;
    if (e < m0) {
      const unsigned long long wc = (unsigned long long)W * C;
      y = e / wc;
      const unsigned long long r = e - y * wc;
      x = r / C;
      c = r - x * C;
      a = g + ((y + 1) * W + x) * S + c;
      b = g + (y * W + x) * S + c;
    } else {
      e -= m0;
      const unsigned long long wc = (unsigned long long)(W - 1) * C;
      y = e / wc;
      const unsigned long long r = e - y * wc;
      x = r / C;
      c = r - x * C;
      a = g + (y * W + x + 1) * S + c;
      b = g + (y * W + x) * S + c;
    }
    return fabs(__dsub_rn((double)__ldg(a), (double)__ldg(b)));
  }
};
// leaf sums of the pooled differences (PASS 0) or of their squared deviations
// from mean[1] (PASS 1)
template <int PASS, typename T = float>
__global__ void __launch_bounds__(256) np_leaf_vad_kernel(VadElems<T> el, const double* __restrict__ mean,
                                                          const long long* __restrict__ leaf_start,
                                                          const int* __restrict__ leaf_len, int nleaves,
                                                          double* __restrict__ vals) {
  const double mu = PASS ? mean[1] : 0.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nleaves; k += gridDim.x * blockDim.x) {
    const unsigned long long e0 = (unsigned long long)leaf_start[k];
    auto val = [&](int i) {
      const double d = el(e0 + (unsigned long long)i);
      if (PASS == 0) return d;
      const double x = __dsub_rn(d, mu);
      return __dmul_rn(x, x);
    };
    vals[k] = np_pairwise_small(val, leaf_len[k]);
  }
}

}  // namespace plas
