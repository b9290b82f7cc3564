// K1 large-radius tier: the separable-blur axis passes of the sort computed by
// FFT convolution in fp64, certified against the reference's SciPy fold and
// completed by the exact fallback kernel (blur_fast.cuh) -- same outputs, bit
// for bit, as blur_pad_kernel.
//
// Why: the direct fold costs ~4h fp64 operations per output and axis, so the
// top levels of the schedule (h up to side/2 - 1) are fp64-issue-bound.  A
// zero-padded length-L FFT (L = 2^k >= n + h) costs O(log L) per output
// independent of h.
//
// Arithmetic.  Two real lines a, b (channels c, c+1 of one column / row) form
// one complex line z = a + i b, zero-padded to L.  The Gaussian kernel k is
// symmetric, so its DFT K is real and
//     conv(a) + i conv(b) = IFFT(FFT(z) . K),
// with IFFT(v) = conj(FFT(conj(v))) / L.  FFTs are radix-8/4/2 Stockham
// passes through shared memory (autosort, natural order in and out), twiddles
// from a host-built table of correctly rounded e^{-2 pi i t / L}.
//
// Certification.  Higham (Accuracy and Stability of Numerical Algorithms,
// Thm 24.2): the computed radix-2 FFT satisfies ||y^ - y||_2 <= c ||y||_2,
// c = log2(L) eta / (1 - log2(L) eta), eta = mu + gamma_4 (sqrt2 + mu), mu the
// twiddle error.  Propagating through the pointwise product (|K| <= sum w = 1,
// K itself computed with compensated sums, error eK) and the inverse gives
//     ||z^ - z||_2 <= (c (1 + e2) + e2) ||z_in||_2,
//     e2 = (c + u (1 + c)) (1 + eK) + eK,
// evaluated on the host with a safety factor of 2 (fft_error_constant).  With
// B = that bound + the SciPy fold's own bound (2h+4) 2^-53 2M (blur_fast.cuh),
// an output whose fp32(z^ - B) == fp32(z^ + B) equals the reference's fp32
// value; every other output goes to the fallback list and is recomputed with
// the exact fold.  ||z_in||_2 and M = max|x| are measured per line pair.
#pragma once
#include "blur_fast.cuh"

namespace plas {

struct FftPlan {
  int log2L;
  int L;
  const double2* tw;   // [L] e^{-2 pi i t / L}
  double* spec;        // [L] real spectrum K of the current level (fft_spectrum_kernel)
  double cbound;       // relative FFT convolution error constant (x ||z_in||_2)
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
  return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // a * (-i)

// Global loads the compiler may not hoist above the pass's barrier (an __ldg
// of the twiddle table would be hoisted across every pass and spill).
__device__ __forceinline__ double2 ld_ordered(const double2* p) {
  double2 v;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_ordered(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int R>
__device__ __forceinline__ void dft_small(double2 (&v)[R]) {
  if (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if (R == 4) {
    const double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const double2 t2 = cadd(v[1], v[3]), t3 = mul_mi(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else if (R == 8) {
    // even / odd radix-4 halves, combined with W8^k = e^{-2 pi i k / 8}
    const double s = 0.70710678118654752440;
    double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    {
      const double2 t0 = cadd(e[0], e[2]), t1 = csub(e[0], e[2]);
      const double2 t2 = cadd(e[1], e[3]), t3 = mul_mi(csub(e[1], e[3]));
      e[0] = cadd(t0, t2);
      e[2] = csub(t0, t2);
      e[1] = cadd(t1, t3);
      e[3] = csub(t1, t3);
    }
    {
      const double2 t0 = cadd(o[0], o[2]), t1 = csub(o[0], o[2]);
      const double2 t2 = cadd(o[1], o[3]), t3 = mul_mi(csub(o[1], o[3]));
      o[0] = cadd(t0, t2);
      o[2] = csub(t0, t2);
      o[1] = cadd(t1, t3);
      o[3] = csub(t1, t3);
    }
    const double2 w1 = make_double2(s * (o[1].x + o[1].y), s * (o[1].y - o[1].x));    // (1 - i)/sqrt2
    const double2 w2 = mul_mi(o[2]);                                                   // -i
    const double2 w3 = make_double2(s * (o[3].y - o[3].x), -s * (o[3].x + o[3].y));   // (-1 - i)/sqrt2
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], w1);
    v[5] = csub(e[1], w1);
    v[2] = cadd(e[2], w2);
    v[6] = csub(e[2], w2);
    v[3] = cadd(e[3], w3);
    v[7] = csub(e[3], w3);
  }
}

// One Stockham pass of radix R over L points in shared memory (in place: every
// thread reads its butterflies' inputs, the CTA syncs, then writes).  Ns = size
// of the sub-transforms already done.  LAST: multiply the output by the real
// spectrum and conjugate it (the pointwise step of the convolution).
template <int L> __host__ __device__ constexpr int fft_threads_for() { return L / 8 < 32 ? 32 : (L / 8 > 512 ? 512 : L / 8); }

// resident CTAs per SM the register budget must allow (~85 registers at 256 threads)
template <int L> __host__ __device__ constexpr int fft_min_blocks() { return fft_threads_for<L>() >= 512 ? 1 : 768 / fft_threads_for<L>(); }

template <int LOG2L, int R, int LOG2NS, bool LAST>
__device__ __forceinline__ void stockham_pass(double2* buf, const double2* tw, const double* spec) {
  constexpr int L = 1 << LOG2L;
  constexpr int Ns = 1 << LOG2NS;
  constexpr int T = fft_threads_for<L>();
  constexpr int nb = L / R;
  constexpr int NB = (nb + T - 1) / T;  // butterflies per thread
  double2 v[NB][R];
  int jj[NB];
  // thread index re-read per pass: otherwise the compiler hoists every pass's
  // (thread-only) address arithmetic to the kernel entry and spills it
  unsigned tid;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
#pragma unroll
  for (int t = 0; t < NB; t++) {
    const int j = (int)tid + t * T;
    jj[t] = j;
    if (j < nb) {
#pragma unroll
      for (int r = 0; r < R; r++) v[t][r] = buf[j + r * nb];
      if (Ns > 1) {
        const int k = j & (Ns - 1);
        constexpr int step = L / (Ns * R);  // twiddle W_{Ns R}^{r k} = tw[r k step]
#pragma unroll
        for (int r = 1; r < R; r++) v[t][r] = cmul(v[t][r], ld_ordered(tw + ((r * k * step) & (L - 1))));
      }
      dft_small<R>(v[t]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < NB; t++) {
    const int j = jj[t];
    if (j < nb) {
      const int k = j & (Ns - 1);
      const int d = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; r++) {
        double2 o = v[t][r];
        if (LAST) {
          const double s = ld_ordered(spec + d + r * Ns);
          o = make_double2(o.x * s, -(o.y * s));
        }
        buf[d + r * Ns] = o;
      }
    }
  }
  __syncthreads();
}

// Forward FFT of buf (natural order in and out); LAST_SPEC applies the
// spectrum + conjugation in the final pass.
// radix-8 passes first (sub-transform size 8^i), then one radix-4 / radix-2
// pass for the remaining bits; every pass is a compile-time instance.
template <int LOG2L, bool LAST_SPEC, int PASS>
__device__ __forceinline__ void fft_passes(double2* buf, const FftPlan& p) {
  constexpr int NR8 = LOG2L / 3, REM = LOG2L % 3;
  if constexpr (PASS < NR8) {
    constexpr bool last = REM == 0 && PASS == NR8 - 1;
    stockham_pass<LOG2L, 8, 3 * PASS, last && LAST_SPEC>(buf, p.tw, p.spec);
    fft_passes<LOG2L, LAST_SPEC, PASS + 1>(buf, p);
  } else if constexpr (REM == 2) {
    stockham_pass<LOG2L, 4, 3 * NR8, LAST_SPEC>(buf, p.tw, p.spec);
  } else if constexpr (REM == 1) {
    stockham_pass<LOG2L, 2, 3 * NR8, LAST_SPEC>(buf, p.tw, p.spec);
  }
}

template <int LOG2L, bool LAST_SPEC>
__device__ __forceinline__ void fft_forward(double2* buf, const FftPlan& p) {
  fft_passes<LOG2L, LAST_SPEC, 0>(buf, p);
}

// The convolution's two FFTs.
template <int LOG2L>
__device__ __forceinline__ void fft_convolve(double2* buf, const double2* tw, double* spec) {
  const FftPlan p{LOG2L, 1 << LOG2L, tw, spec, 0.0};
  fft_forward<LOG2L, true>(buf, p);
  fft_forward<LOG2L, false>(buf, p);
}

__device__ __forceinline__ double block_max_sum(double* red, double v, double m, double* out_max) {
  // returns the CTA sum of v and writes the CTA max of m (all threads)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(PLAS_FULL_MASK, v, o);
    m = fmax(m, __shfl_xor_sync(PLAS_FULL_MASK, m, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) {
    red[2 * wid] = v;
    red[2 * wid + 1] = m;
  }
  __syncthreads();
  double s = 0.0, mx = 0.0;
  for (int i = 0; i < nw; i++) {
    s += red[2 * i];
    mx = fmax(mx, red[2 * i + 1]);
  }
  __syncthreads();
  *out_max = mx;
  return s;
}

// One axis pass of the level blur by FFT.  AXIS 0: lines = columns (x, c) of
// feat (row stride W*S), output to the tmp interior (row stride (W+2P)*S).
// AXIS 1: lines = rows (y, c) of tmp, output to target / den32 (EPI 1).
// One CTA of fft_threads_for<L>() threads per line pair (no persistent loop:
// across a loop the compiler hoists every pass's thread-only address
// arithmetic out of it and spills).  The CTA also settles its own uncertain
// outputs with the exact SciPy fold from a shared-memory copy of the two input
// lines (FB_LOCAL of them; any excess goes to the global fallback list).
constexpr int FB_LOCAL = 512;

template <int AXIS, int EPI, int LOG2L>
__global__ void __launch_bounds__(fft_threads_for<(1 << LOG2L)>(), fft_min_blocks<(1 << LOG2L)>())
    blur_fft_kernel(const float* __restrict__ in, float* __restrict__ out, PadGeom pg, BlurLevelRef lvl,
                    FftPlan plan, const float* __restrict__ den32, int* __restrict__ fb, int fb_cap,
                    int* __restrict__ fb_other) {
  constexpr int L = 1 << LOG2L;
  extern __shared__ double2 fbuf[];         // [L] complex line pair
  float* raw = reinterpret_cast<float*>(fbuf + L);  // [2][n] input lines; callers guarantee n <= L/2
  __shared__ double red[64];
  __shared__ int flist[FB_LOCAL];
  __shared__ int nflag;
  if (blockIdx.x == 0 && threadIdx.x == 0 && fb_other) fb_other[0] = 0;
  if (threadIdx.x == 0) nflag = 0;
  const int H = pg.H, W = pg.W, C = pg.C, S = pg.S;
  const int n = AXIS == 0 ? H : W;
  const long long WS = (long long)W * S;
  const long long WSP = (long long)(W + 2 * pg.pad) * S;
  const long long in_stride = AXIS == 0 ? WS : (long long)S;
  const int cpairs = (C + 1) >> 1;
  const long long p = blockIdx.x;
  const long long line = p / cpairs;
  const int c = (int)(p - line * cpairs) * 2;
  const bool has_b = c + 1 < C;
  const long long in_base = AXIS == 0 ? line * S + c : line * WSP + c;
  // ---- load the pair (zero-padded), ||z||_2^2 and max |x|
  double ss = 0.0, mx = 0.0;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    double2 z = make_double2(0.0, 0.0);
    if (i < n) {
      const float* src = in + in_base + (long long)i * in_stride;
      const float a = __ldg(src);
      const float b = has_b ? __ldg(src + 1) : 0.f;
      raw[i] = a;
      raw[n + i] = b;
      z = make_double2((double)a, (double)b);
      ss = fma(z.x, z.x, fma(z.y, z.y, ss));
      mx = fmax(mx, fmax(fabs(z.x), fabs(z.y)));
    }
    fbuf[i] = z;
  }
  double M;
  const double norm2 = block_max_sum(red, ss, mx, &M);  // includes the barrier before the FFT
  // ---- forward FFT, pointwise spectrum + conj, forward FFT again
  fft_convolve<LOG2L>(fbuf, plan.tw, plan.spec);
  // ---- outputs: conv(a) = re / L, conv(b) = -im / L
  int h;
  const double* w;
  lvl.get(&h, &w);
  const long long out_stride = AXIS == 0 ? WSP : (long long)S;
  const long long out_base = AXIS == 0 ? line * S + c : line * WS + c;
  const double invL = 1.0 / (double)L;
  const double fold_scale = (2.0 * h + 4.0) * 2.0 * 1.1102230246251565e-16;
  const double B = (plan.cbound * sqrt(norm2) + fold_scale * M) * 1.0001;
  // warp-uniform trip count (the list append below is warp-collective)
  for (int i0 = 0; i0 < n; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool in_range = i < n;
    const double2 z = fbuf[in_range ? i : 0];
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const bool valid = in_range && (q == 0 || has_b);
      const double acc = q == 0 ? z.x * invL : -(z.y * invL);
      const float lo = __double2float_rn(__dsub_rn(acc, B));
      const float hi = __double2float_rn(__dadd_rn(acc, B));
      const bool unsure = valid && lo != hi;
      if (valid && !unsure) {
        float r = __double2float_rn(acc);
        if (EPI == 1) r = __fdiv_rn(r, den32[(AXIS == 0 ? (long long)i * W + line : line * W + i)]);
        out[out_base + q + (long long)i * out_stride] = r;
      }
      // local list (warp-aggregated), overflow to the global list
      const unsigned bal = __ballot_sync(PLAS_FULL_MASK, unsure);
      if (bal) {
        const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&nflag, __popc(bal));
        base = __shfl_sync(PLAS_FULL_MASK, base, leader);
        if (unsure) {
          const int slot = base + __popc(bal & ((1u << lane) - 1u));
          if (slot < FB_LOCAL) {
            flist[slot] = (q << 30) | i;
          } else {
            const long long o = out_base + q + (long long)i * out_stride;
            const int e = (int)(AXIS == 0 ? (long long)i * WS + line * S + c + q : o);
            const int g = atomicAdd(fb, 1);
            if (g < fb_cap) fb[FB_HEADER + g] = e;
          }
        }
      }
    }
  }
  __syncthreads();
  // ---- exact SciPy fold for this CTA's uncertain outputs (blur.cuh contract)
  const int nf = min(nflag, FB_LOCAL);
  for (int t = threadIdx.x; t < nf; t += blockDim.x) {
    const int e = flist[t];
    const int q = e >> 30, i = e & 0x3fffffff;
    const float* x = raw + q * n;
    double acc = __dmul_rn((double)x[i], __ldg(w));
    for (int j = h; j >= 1; j--) {
      const double a = i - j >= 0 ? (double)x[i - j] : 0.0;
      const double b = i + j < n ? (double)x[i + j] : 0.0;
      acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(a, b), __ldg(w + j)));
    }
    float r = __double2float_rn(acc);
    if (EPI == 1) r = __fdiv_rn(r, den32[(AXIS == 0 ? (long long)i * W + line : line * W + i)]);
    out[out_base + q + (long long)i * out_stride] = r;
  }
}

// Real spectrum of the current level's symmetric kernel on L points:
// K[m] = w0 + 2 sum_{j=1..h} w_j cos(2 pi j m / L), cosines from the twiddle
// table (exact index reduction), compensated (TwoProduct + TwoSum) so the
// error stays ~3 ulp regardless of h.
__global__ void fft_spectrum_kernel(BlurLevelRef lvl, FftPlan plan) {
  int h;
  const double* w;
  lvl.get(&h, &w);
  const int L = plan.L;
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < L; m += gridDim.x * blockDim.x) {
    double s = __ldg(w), comp = 0.0;
    for (int j = 1; j <= h; j++) {
      const double cj = __ldg(&plan.tw[(long long)j * m & (L - 1)].x);
      const double wj2 = 2.0 * __ldg(w + j);
      const double p = wj2 * cj;
      const double pe = fma(wj2, cj, -p);  // exact product error
      const double t = s + p;
      const double bp = t - s;
      const double te = (s - (t - bp)) + (p - bp);  // TwoSum error
      s = t;
      comp += te + pe;
    }
    plan.spec[m] = s + comp;
  }
}

}  // namespace plas
