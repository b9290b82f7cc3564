// caller-side feature preparation on the GPU, so that
// bundle.compress (bundle.py:134-160) stays device-resident up to quantization.
//
//   prune_to_grid        (splats.py:139-152): keep the `keep` Gaussians of
//                         highest opacity logit; ties broken by index as in a
//                         stable ascending argsort; survivors in index order.
//   normalize_for_sorting (splats.py:184-216): activated attribute channels ->
//                         ((v - lo) / span) * w, constant channels -> 0.
//   values[perm], cloud.select(index) (bundle.py:160, splats.py:95-104): row gather.
//
// Prune = radix select + stable compaction, all on the device (no host sync):
//   key(x) = order-preserving u64 of the fp64 logit (-0 folded onto +0, as
//            NumPy's comparison treats them equal; NaN/Inf are rejected by the
//            SplatCloud validation, splats.py:58-60);
//   the element of ascending rank r = n - keep in the stable order (key, index)
//   is found digit by digit (8 passes of an 8-bit histogram over the keys that
//   match the prefix found so far); that leaves T = its key and d = its rank
//   among the keys equal to T;
//   survivor <=> key > T, or key == T and (its rank among equal keys, in index
//   order) >= d.  Block counts of "key > T" and "key == T" are scanned once
//   (fixed order, one CTA), then every block writes its survivors in index
//   order at gt_before + max(0, eq_before - d) + its local prefix.
#pragma once
#include "common.cuh"

namespace plas {

__device__ __forceinline__ unsigned long long order_key(double x) {
  if (x == 0.0) x = 0.0;  // -0 == +0 (NumPy sorts them as equal)
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct SelectState {
  unsigned long long prefix, mask;  // digits fixed so far
  long long rank;                   // rank still to find inside the current bucket
  long long pad;
};

constexpr int SEL_THREADS = 256;
constexpr int PREP_CHUNK = 4096;  // elements per compaction block

__global__ void __launch_bounds__(SEL_THREADS) select_init_kernel(SelectState* s, long long rank,
                                                                  unsigned* hist) {
  if (threadIdx.x == 0) {
    s->prefix = 0ull;
    s->mask = 0ull;
    s->rank = rank;
  }
  hist[threadIdx.x] = 0u;
}

// histogram of digit `shift` over the keys matching the current prefix
__global__ void __launch_bounds__(SEL_THREADS) select_hist_kernel(const double* __restrict__ x, long long n,
                                                                  const SelectState* __restrict__ s, int shift,
                                                                  unsigned* __restrict__ hist) {
  __shared__ unsigned h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  const unsigned long long prefix = s->prefix, mask = s->mask;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = order_key(x[i]);
    if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// the bucket holding the remaining rank; fixes one more digit, clears the histogram
__global__ void __launch_bounds__(SEL_THREADS) select_pick_kernel(SelectState* s, int shift,
                                                                  unsigned* hist) {
  __shared__ unsigned h[256];
  h[threadIdx.x] = hist[threadIdx.x];
  __syncthreads();
  hist[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    long long r = s->rank, below = 0;
    int b = 0;
    for (; b < 255; b++) {
      if (below + (long long)h[b] > r) break;
      below += h[b];
    }
    s->prefix |= (unsigned long long)b << shift;
    s->mask |= 0xffull << shift;
    s->rank = r - below;
  }
}

// per block of PREP_CHUNK elements: count of keys > T and == T
__global__ void __launch_bounds__(SEL_THREADS) prune_count_kernel(const double* __restrict__ x, long long n,
                                                                  const SelectState* __restrict__ s,
                                                                  int2* __restrict__ counts) {
  __shared__ int cg[SEL_THREADS / 32], ce[SEL_THREADS / 32];
  const unsigned long long T = s->prefix;
  const long long b0 = (long long)blockIdx.x * PREP_CHUNK;
  int gt = 0, eq = 0;
  for (int t = threadIdx.x; t < PREP_CHUNK; t += SEL_THREADS) {
    const long long i = b0 + t;
    if (i < n) {
      const unsigned long long k = order_key(x[i]);
      gt += k > T;
      eq += k == T;
    }
  }
  gt = __reduce_add_sync(PLAS_FULL_MASK, gt);
  eq = __reduce_add_sync(PLAS_FULL_MASK, eq);
  if ((threadIdx.x & 31) == 0) {
    cg[threadIdx.x >> 5] = gt;
    ce[threadIdx.x >> 5] = eq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, e = 0;
    for (int w = 0; w < SEL_THREADS / 32; w++) {
      a += cg[w];
      e += ce[w];
    }
    counts[blockIdx.x] = make_int2(a, e);
  }
}

// exclusive scan of the block counts (one CTA, fixed order)
__global__ void __launch_bounds__(1024) prune_scan_kernel(int2* __restrict__ counts, int nblocks) {
  __shared__ long long carry_g, carry_e;
  __shared__ int wg[32], we[32];
  if (threadIdx.x == 0) carry_g = carry_e = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < nblocks; base += 1024) {
    const int i = base + threadIdx.x;
    const int2 c = i < nblocks ? counts[i] : make_int2(0, 0);
    int g = c.x, e = c.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int tg = __shfl_up_sync(PLAS_FULL_MASK, g, o), te = __shfl_up_sync(PLAS_FULL_MASK, e, o);
      if (lane >= o) {
        g += tg;
        e += te;
      }
    }
    if (lane == 31) {
      wg[wid] = g;
      we[wid] = e;
    }
    __syncthreads();
    if (wid == 0) {
      int sg = wg[lane], se = we[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tg = __shfl_up_sync(PLAS_FULL_MASK, sg, o), te = __shfl_up_sync(PLAS_FULL_MASK, se, o);
        if (lane >= o) {
          sg += tg;
          se += te;
        }
      }
      wg[lane] = sg;
      we[lane] = se;
    }
    __syncthreads();
    const long long pg = carry_g + (wid ? wg[wid - 1] : 0) + g - c.x;  // exclusive
    const long long pe = carry_e + (wid ? we[wid - 1] : 0) + e - c.y;
    if (i < nblocks) counts[i] = make_int2((int)pg, (int)pe);
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_g += wg[31];
      carry_e += we[31];
    }
    __syncthreads();
  }
}

// survivors in index order
__global__ void __launch_bounds__(SEL_THREADS) prune_write_kernel(const double* __restrict__ x, long long n,
                                                                  const SelectState* __restrict__ s,
                                                                  const int2* __restrict__ before,
                                                                  long long* __restrict__ out) {
  __shared__ int wsum_e[SEL_THREADS / 32], wsum_k[SEL_THREADS / 32];
  __shared__ long long run_e, run_k;
  const unsigned long long T = s->prefix;
  const long long d = s->rank;
  const long long b0 = (long long)blockIdx.x * PREP_CHUNK;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    run_e = before[blockIdx.x].y;  // keys == T before this block (index order)
    const long long kept_eq = run_e - d > 0 ? run_e - d : 0;
    run_k = (long long)before[blockIdx.x].x + kept_eq;  // survivors before this block
  }
  __syncthreads();
  for (int t0 = 0; t0 < PREP_CHUNK; t0 += SEL_THREADS) {
    const long long i = b0 + t0 + threadIdx.x;
    unsigned long long k = 0;
    if (i < n) k = order_key(x[i]);
    const bool eq = i < n && k == T, gt = i < n && k > T;
    // rank of this element among the equal keys (index order)
    const unsigned be = __ballot_sync(PLAS_FULL_MASK, eq);
    if (lane == 0) wsum_e[wid] = __popc(be);
    __syncthreads();
    long long eb = run_e;
    for (int w = 0; w < wid; w++) eb += wsum_e[w];
    const long long eqrank = eb + __popc(be & ((1u << lane) - 1u));
    const bool keep = gt || (eq && eqrank >= d);
    const unsigned bk = __ballot_sync(PLAS_FULL_MASK, keep);
    if (lane == 0) wsum_k[wid] = __popc(bk);
    __syncthreads();
    long long kb = run_k;
    for (int w = 0; w < wid; w++) kb += wsum_k[w];
    if (keep) out[kb + __popc(bk & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int se = 0, sk = 0;
      for (int w = 0; w < SEL_THREADS / 32; w++) {
        se += wsum_e[w];
        sk += wsum_k[w];
      }
      run_e += se;
      run_k += sk;
    }
    __syncthreads();
  }
}

// ---- normalize_for_sorting
struct PrepAttr {
  const double* v;
  long long stride;  // elements between rows
  int channels;
  int act;           // 0 identity, 1 sigmoid, 2 exp (splats.py:86-93)
  double weight;
  int col;           // first output column (weight > 0), -1 if dropped
  int ch0;           // first channel in the min/max arrays
};
constexpr int PREP_MAX_ATTRS = 8;
constexpr int PREP_MAX_CH = 64;
struct PrepAttrs {
  PrepAttr a[PREP_MAX_ATTRS];
  int count;
  int total_ch;
};

__device__ __forceinline__ double activate(double x, int act) {
  if (act == 1) return 1.0 / (1.0 + exp(-x));
  if (act == 2) return exp(x);
  return x;
}

// per-CTA per-channel min / max of the activated values.  For an attribute of
// C channels a CTA works as blockDim / C row lanes of C channel threads, so
// consecutive threads read consecutive values of a row and every thread keeps
// one channel's (min, max) in two registers; the row lanes of a channel are
// combined in shared memory (min / max are exact, so the order is immaterial).
__global__ void __launch_bounds__(256) prep_minmax_kernel(PrepAttrs at, long long n, double2* __restrict__ part) {
  __shared__ double2 red[256];
  for (int ai = 0; ai < at.count; ai++) {
    const PrepAttr A = at.a[ai];
    if (A.channels == 0) continue;
    const int C = A.channels;
    const int lanes = (int)blockDim.x / C;  // row lanes per CTA
    const int rl = (int)threadIdx.x / C, c = (int)threadIdx.x - rl * C;
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    if (rl < lanes) {
      const long long step = (long long)gridDim.x * lanes;
      long long i = (long long)blockIdx.x * lanes + rl;
      for (; i + 3 * step < n; i += 4 * step) {  // four independent loads in flight
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = __ldg(A.v + (i + u * step) * A.stride + c);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const double a = activate(v[u], A.act);
          lo = fmin(lo, a);
          hi = fmax(hi, a);
        }
      }
      for (; i < n; i += step) {
        const double a = activate(__ldg(A.v + i * A.stride + c), A.act);
        lo = fmin(lo, a);
        hi = fmax(hi, a);
      }
    }
    red[threadIdx.x] = make_double2(lo, hi);
    __syncthreads();
    if ((int)threadIdx.x < C) {
      double2 r = red[threadIdx.x];
      for (int t = (int)threadIdx.x + C; t < lanes * C; t += C) {
        r.x = fmin(r.x, red[t].x);
        r.y = fmax(r.y, red[t].y);
      }
      part[(long long)blockIdx.x * at.total_ch + A.ch0 + threadIdx.x] = r;
    }
    __syncthreads();
  }
}

// one warp per channel over the CTA partials
__global__ void prep_minmax_final_kernel(const double2* __restrict__ part, int nparts, int total_ch,
                                         double* __restrict__ mins, double* __restrict__ maxs) {
  const int lane = threadIdx.x & 31;
  for (int ch = threadIdx.x >> 5; ch < total_ch; ch += blockDim.x >> 5) {
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    for (int p = lane; p < nparts; p += 32) {
      const double2 v = part[(long long)p * total_ch + ch];
      lo = fmin(lo, v.x);
      hi = fmax(hi, v.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(PLAS_FULL_MASK, lo, o));
      hi = fmax(hi, __shfl_xor_sync(PLAS_FULL_MASK, hi, o));
    }
    if (lane == 0) {
      mins[ch] = lo;
      maxs[ch] = hi;
    }
  }
}

// features[:, col + c] = ((v - lo) / span) * w, span = hi - lo if hi > lo else 1; constant -> 0
__global__ void __launch_bounds__(256) prep_write_kernel(PrepAttrs at, long long n, int fcols,
                                                         const double* __restrict__ mins,
                                                         const double* __restrict__ maxs,
                                                         double* __restrict__ feat) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int ai = 0; ai < at.count; ai++) {
      const PrepAttr A = at.a[ai];
      if (A.col < 0) continue;
      for (int c = 0; c < A.channels; c++) {
        const double lo = mins[A.ch0 + c], hi = maxs[A.ch0 + c];
        double r = 0.0;
        if (hi > lo) r = ((activate(A.v[i * A.stride + c], A.act) - lo) / (hi - lo)) * A.weight;
        feat[i * fcols + A.col + c] = r;
      }
    }
  }
}

// dst[i] = src[index[i]] for rows of row_bytes bytes (16-byte vectors when aligned);
// 32-bit multiply-shift division of the flat vector index (count * row_vecs < 2^32)
template <typename V>
__global__ void __launch_bounds__(256) gather_rows_kernel(const V* __restrict__ src, unsigned row_vecs,
                                                          unsigned rv_m, int rv_l, const long long* __restrict__ index,
                                                          unsigned total, V* __restrict__ dst) {
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned r = fastdiv(t, rv_m, rv_l), c = t - r * row_vecs;
    dst[t] = __ldg(src + index[r] * (long long)row_vecs + c);
  }
}

// ---- correctly rounded ln(1 + x) for the position contraction
// CUDA's log1p is within 1 ulp; the reference's (NumPy -> libm) is correctly
// rounded for ~99.9 % of arguments (52 of 50,000 random ones were not,
// against 60-digit decimal logarithms) -- the two differed in the last bit
// for 7.3 % of values, which moved the manifest's data-driven ranges by an
// ulp in about a third of random attribute sets.  log1p_cr rounds the true
// value instead: from y = log1p(x) it moves to the neighbour whose rounding
// interval holds ln(1 + x), deciding L > m (m an interval end) by comparing
// 1 + x (exact as a double-double) with exp(m) in double-double:
// exp(m) = (Taylor_9(r / 2^10))^(2^10) 2^k, r = m - k ln2, relative error
// below 2^-98; a comparison inside that error keeps y.
struct DDv {
  double hi, lo;
};
__device__ __forceinline__ DDv ddv_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return DDv{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ DDv ddv_norm(double a, double b) {  // |a| >= |b|
  const double s = a + b;
  return DDv{s, b - (s - a)};
}
__device__ __forceinline__ DDv ddv_add(DDv a, DDv b) {
  DDv s = ddv_two_sum(a.hi, b.hi);
  return ddv_norm(s.hi, s.lo + (a.lo + b.lo));
}
__device__ __forceinline__ DDv ddv_mul(DDv a, DDv b) {
  const double p = a.hi * b.hi;
  const double e = fma(a.hi, b.hi, -p) + (a.hi * b.lo + a.lo * b.hi);
  return ddv_norm(p, e);
}
__device__ DDv ddv_exp(DDv m) {
  const DDv LN2{0.6931471805599453, 2.3190468138462996e-17};
  const double k = rint(m.hi / LN2.hi);
  const DDv kl = ddv_mul(LN2, DDv{k, 0.0});
  DDv r = ddv_add(m, DDv{-kl.hi, -kl.lo});
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  // 1/j!, j = 9 .. 2, as double-doubles; Horner from the top
  const double ch[8] = {2.7557319223985893e-06, 2.48015873015873e-05, 0.0001984126984126984,
                        0.001388888888888889, 0.008333333333333333, 0.041666666666666664,
                        0.16666666666666666, 0.5};
  const double cl[8] = {-1.858393274046472e-22, 2.1511947866775882e-23, 1.7209558293420705e-22,
                        -5.300543954373577e-20, 1.1564823173178714e-19, 2.3129646346357427e-18,
                        9.25185853854297e-18, 0.0};
  DDv p{ch[0], cl[0]};
#pragma unroll
  for (int j = 1; j < 8; j++) p = ddv_add(ddv_mul(p, r), DDv{ch[j], cl[j]});
  p = ddv_add(ddv_mul(p, r), DDv{1.0, 0.0});  // 1 + r/1!
  p = ddv_add(ddv_mul(p, r), DDv{1.0, 0.0});  // (exp(r) = 1 + r (1 + r (1/2 + ...)))
  for (int j = 0; j < 10; j++) p = ddv_mul(p, p);
  return DDv{ldexp(p.hi, (int)k), ldexp(p.lo, (int)k)};
}
// sign of (a - b) for double-doubles, 0 when within rel * |b| (undecided)
__device__ __forceinline__ int ddv_cmp(DDv a, DDv b, double rel) {
  const double d = (a.hi - b.hi) + (a.lo - b.lo);
  if (fabs(d) <= rel * fabs(b.hi)) return 0;
  return d > 0.0 ? 1 : -1;
}
__device__ double log1p_cr(double x) {
  const double y = log1p(x);
  if (!(x > 1e-20) || !(y < 700.0)) return y;  // tiny: ln(1 + x) rounds to x; huge / inf / nan: as is
  const DDv A = ddv_two_sum(1.0, x);           // 1 + x exactly
  const double up = nextafter(y, 1e300), dn = nextafter(y, 0.0);
  const double rel = 0x1p-97;
  if (ddv_cmp(A, ddv_exp(DDv{y, (up - y) * 0.5}), rel) > 0) return up;  // ln(1 + x) above the upper midpoint
  if (ddv_cmp(A, ddv_exp(DDv{y, (dn - y) * 0.5}), rel) < 0) return dn;  // below the lower one
  return y;
}

// ---- quantization (quantization.py:8-51, bundle.py:102-115, 158-188)
// contract(x) = sign(x) ln(1 + |x|) (quantization.py:8-11), ln correctly rounded
__device__ __forceinline__ double contract_value(double x) {
  const double s = x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0);  // np.sign: +0 for either zero
  return s * log1p_cr(fabs(x));
}

// per-CTA per-channel min / max of the (optionally contracted) values
__global__ void __launch_bounds__(256) quant_minmax_kernel(const double* __restrict__ v, long long n, int C,
                                                           long long stride, int contract,
                                                           double2* __restrict__ part) {
  __shared__ double2 red[256];
  const int lanes = (int)blockDim.x / C;
  const int rl = (int)threadIdx.x / C, c = (int)threadIdx.x - rl * C;
  double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
  if (rl < lanes) {
    for (long long i = (long long)blockIdx.x * lanes + rl; i < n; i += (long long)gridDim.x * lanes) {
      double x = __ldg(v + i * stride + c);
      if (contract) x = contract_value(x);
      lo = fmin(lo, x);
      hi = fmax(hi, x);
    }
  }
  red[threadIdx.x] = make_double2(lo, hi);
  __syncthreads();
  if ((int)threadIdx.x < C) {
    double2 r = red[threadIdx.x];
    for (int t = (int)threadIdx.x + C; t < lanes * C; t += C) {
      r.x = fmin(r.x, red[t].x);
      r.y = fmax(r.y, red[t].y);
    }
    part[(long long)blockIdx.x * C + threadIdx.x] = r;
  }
}

// data-driven range (bundle.py:106-109): lo = min, hi = max if max > min else min + 1
__global__ void quant_range_kernel(const double2* __restrict__ part, int nparts, int C, double* __restrict__ lo_out,
                                   double* __restrict__ hi_out) {
  const int lane = threadIdx.x & 31;
  for (int c = threadIdx.x >> 5; c < C; c += blockDim.x >> 5) {
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    for (int p = lane; p < nparts; p += 32) {
      lo = fmin(lo, part[(long long)p * C + c].x);
      hi = fmax(hi, part[(long long)p * C + c].y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(PLAS_FULL_MASK, lo, o));
      hi = fmax(hi, __shfl_xor_sync(PLAS_FULL_MASK, hi, o));
    }
    if (lane == 0) {
      lo_out[c] = lo;
      hi_out[c] = hi > lo ? hi : lo + 1.0;
    }
  }
}

__global__ void quant_fill_kernel(double* __restrict__ lo_out, double* __restrict__ hi_out, int C, double lo,
                                  double hi) {
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    lo_out[c] = lo;
    hi_out[c] = hi;
  }
}

// index = floor(((clip(v, lo, hi) - lo) / (hi - lo)) (levels - 1) + 0.5) (quantization.py:28-41),
// written as the encoded image's pixel: image c / per_image, pixel i, sample c % per_image
template <typename P>
__global__ void __launch_bounds__(256) quant_pack_kernel(const double* __restrict__ v, long long n, int C,
                                                         long long stride, int contract,
                                                         const double* __restrict__ lo_in,
                                                         const double* __restrict__ hi_in, int levels,
                                                         int per_image, P* __restrict__ out) {
  const long long total = n * C;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / C;
    const int c = (int)(e - i * C);
    double x = v[i * stride + c];
    if (contract) x = contract_value(x);
    const double lo = lo_in[c], hi = hi_in[c];
    x = fmin(fmax(x, lo), hi);  // np.clip
    const double unit = (x - lo) / (hi - lo);
    const double q = floor(unit * (double)(levels - 1) + 0.5);
    const int img = c / per_image, w = c - img * per_image;
    out[((long long)img * n + i) * per_image + w] = (P)(long long)q;
  }
}

}  // namespace plas
