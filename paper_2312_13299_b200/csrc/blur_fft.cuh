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
  int log2L;          // length code lc (fft_len)
  int L;
  const double2* tw;   // [L] e^{-2 pi i t / L}, then the per-pass tables (fft_pass_twiddle_offset)
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
  if (R == 5) {
    // W5^k = e^{-2 pi i k / 5}: y_k = x0 + sum_{m=1..4} W5^{k m} x_m, paired as
    // (x1 + x4, x1 - x4), (x2 + x3, x2 - x3)
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;  // cos 2pi/5, cos 4pi/5
    const double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;   // sin 2pi/5, sin 4pi/5
    const double2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
    const double2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
    const double2 x0 = v[0];
    const double2 r1 = make_double2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
    const double2 r2 = make_double2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
    // -i (s1 b1 + s2 b2) and -i (s2 b1 - s1 b2)
    const double2 i1 = mul_mi(make_double2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y));
    const double2 i2 = mul_mi(make_double2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y));
    v[0] = cadd(x0, cadd(a1, a2));
    v[1] = cadd(r1, i1);
    v[4] = csub(r1, i1);
    v[2] = cadd(r2, i2);
    v[3] = csub(r2, i2);
  } else if (R == 3) {
    // W3 = e^{-2 pi i / 3} = -1/2 - i sqrt3/2
    const double s3 = 0.86602540378443864676;
    const double2 t = cadd(v[1], v[2]);
    const double2 d = mul_mi(csub(v[1], v[2]));  // -i (x1 - x2)
    const double2 m = make_double2(v[0].x - 0.5 * t.x, v[0].y - 0.5 * t.y);
    const double2 sd = make_double2(s3 * d.x, s3 * d.y);
    v[0] = cadd(v[0], t);
    v[1] = cadd(m, sd);
    v[2] = csub(m, sd);
  } else if (R == 2) {
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

// Composite radices R = R1 R2 (R1 odd or 4, R2 a power of two) in registers,
// Cooley-Tukey: DFT_R1 over n1 for each n2 (inputs x[R2 n1 + n2]), internal
// twiddles W_R^(n2 k1), DFT_R2 over n2 for each k1, output X[k1 + R1 k2].  The
// internal twiddles are correctly rounded constants (exact for multiples of a
// quarter turn).  Error accounting (fft_error_constant): the odd DFT with the
// pass's outer twiddle is charged as for a separate odd pass, and each
// internal twiddle rides on the first radix-2 stage of the power-of-two DFT
// after it, so a composite pass costs exactly the radix-2 stages of its factors.
template <int R>
__device__ __forceinline__ double2 fft_wconst(int m) {  // W_R^m = e^{-2 pi i m / R}, R = 16, 20 or 24
  constexpr double c16[5] = {1.0, 0.9238795325112867, 0.7071067811865476, 0.3826834323650898, 0.0};
  constexpr double c24[7] = {1.0, 0.9659258262890683, 0.8660254037844386, 0.7071067811865476, 0.5,
                             0.25881904510252074, 0.0};
  constexpr double c20[6] = {1.0, 0.9510565162951535, 0.8090169943749475, 0.5877852522924731, 0.30901699437494745,
                             0.0};
  constexpr int Q = R / 4;  // cos over the first quarter turn in Q steps
  const double* cq = Q == 4 ? c16 : (Q == 6 ? c24 : c20);
  m %= R;
  const int quad = m / Q, r = m - quad * Q;
  const double2 b = make_double2(cq[r], -cq[Q - r]);  // (cos, -sin) of 2 pi r / R
  // e^{-i (quad pi/2 + t)} = (-i)^quad e^{-i t}
  return quad == 0 ? b : (quad == 1 ? make_double2(b.y, -b.x) : (quad == 2 ? make_double2(-b.x, -b.y)
                                                                           : make_double2(-b.y, b.x)));
}
template <int R1, int R2>
__device__ __forceinline__ void dft_comp(double2 (&v)[R1 * R2]);
template <int R>
__device__ __forceinline__ void dft_any(double2 (&v)[R]) {
  if constexpr (R == 2 || R == 3 || R == 4 || R == 5 || R == 8) {
    dft_small<R>(v);
  } else if constexpr (R == 6 || R == 12 || R == 24) {
    dft_comp<3, R / 3>(v);
  } else {
    static_assert(R == 10 || R == 20 || R == 40, "unsupported radix");
    dft_comp<5, R / 5>(v);
  }
}
template <int R1, int R2>
__device__ __forceinline__ void dft_comp(double2 (&v)[R1 * R2]) {
  constexpr int R = R1 * R2;
  constexpr int RT = (R == 10 || R == 20) ? 20 : 24;  // constant tables: 6, 12 | 24 and 10 | 20
  constexpr int SC = RT / R;
#pragma unroll
  for (int n2 = 0; n2 < R2; n2++) {
    double2 t[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; n1++) t[n1] = v[R2 * n1 + n2];
    dft_any<R1>(t);
#pragma unroll
    for (int k1 = 0; k1 < R1; k1++) {
      const int m = (n2 * k1) % R;
      if (m != 0) {
        if ((4 * m) % R == 0) {  // a quarter turn: exact
          const int quad = 4 * m / R;
          const double2 b = t[k1];
          t[k1] = quad == 1 ? make_double2(b.y, -b.x) : (quad == 2 ? make_double2(-b.x, -b.y) : make_double2(-b.y, b.x));
        } else {
          t[k1] = cmul(t[k1], fft_wconst<RT>(m * SC));
        }
      }
      v[R2 * k1 + n2] = t[k1];
    }
  }
  double2 o[R];
#pragma unroll
  for (int k1 = 0; k1 < R1; k1++) {
    double2 t[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; n2++) t[n2] = v[R2 * k1 + n2];
    dft_any<R2>(t);
#pragma unroll
    for (int k2 = 0; k2 < R2; k2++) o[k1 + R1 * k2] = t[k2];
  }
#pragma unroll
  for (int k = 0; k < R; k++) v[k] = o[k];
}

// threads per CTA for L > 4096; 0 = L / 8 (640 at 5120, 768 at 6144: one
// radix-8 butterfly per thread and pass, so no pass runs a second partial
// round while most warps wait at its barrier; 96 / 80 registers, no spills).
// Measured at C4: FFT blur 1127 -> 1038 ms per sort vs 512 threads.
#ifndef FFT_LONG_T
#define FFT_LONG_T 0
#endif
#ifndef FFT_LONG_MINB
#define FFT_LONG_MINB 1
#endif
__host__ __device__ constexpr int fft_threads_len(int L) {
  return L > 4096 ? (FFT_LONG_T > 0 ? FFT_LONG_T : L / 8) : (L / 8 < 32 ? 32 : (L / 8 > 512 ? 512 : L / 8));
}
template <int L> __host__ __device__ constexpr int fft_threads_for() { return fft_threads_len(L); }
// resident CTAs per SM the register budget must allow (~85 registers at 256 threads)
// 4 CTAs per SM at 256 threads (64 registers): the passes are latency-bound, so
// occupancy beats the second buffer (measured: C2 144.5 -> 138.5 ms)
#ifndef FFT_MINB
#define FFT_MINB 4
#endif
#ifndef FFT_MINB_3072
#define FFT_MINB_3072 3
#endif
// (L > 4096: one CTA per SM; two with 64 registers spill 150-200 bytes and
// C4 went from 2.61 to 2.75 s.  L = 3072: three CTAs at 56 registers beat two
// at 72 -- C3 1.692 -> 1.672 s; four CTAs at 2560 and 3072 (48 / 40
// registers, 160-280 bytes of spills): C3 1.80 s vs 1.65 s.)
#ifndef FFT_MINB_2560
#define FFT_MINB_2560 3
#endif
template <int L> __host__ __device__ constexpr int fft_min_blocks() {
  return L > 4096 ? FFT_LONG_MINB
                  : (L == 3072 ? FFT_MINB_3072
                               : (L == 2560 ? FFT_MINB_2560 : (FFT_MINB * 256) / fft_threads_for<L>()));
}

// With FFT_MERGE_ODD, the power-of-two remainder (2 or 4) and an odd factor 3
// or 5 share one composite pass (6, 10, 12 or 20) instead of two passes:
// 3072 = 8 8 8 6, 5120 = 8 8 8 10, 6144 = 8 8 8 12 (one barrier pair and
// shared-memory round trip fewer per FFT).
#ifndef FFT_MERGE_ODD
#define FFT_MERGE_ODD 1
#endif
// FFT length code lc = p2 + 32 m: L = M 2^p2 with M = 1, 3, 5, 9 for m = 0..3
// (the odd factors cut the padded length: at side 1024 a level with h <= 128
// uses 1152, h <= 256 1280, h <= 511 1536, instead of 2048).  Pass schedule:
// radix-8 passes over the power-of-two part, one radix-4 or radix-2 pass for
// its remaining bits, then the odd part: one radix-3 (M = 3), one radix-5
// (M = 5) or two radix-3 passes (M = 9).  Pass p has sub-transform size Ns =
// product of the earlier radices.
__host__ __device__ constexpr int fft_mult(int lc) { return (lc >> 5) == 0 ? 1 : ((lc >> 5) == 1 ? 3 : ((lc >> 5) == 2 ? 5 : 9)); }
__host__ __device__ constexpr int fft_p2(int lc) { return lc & 31; }
__host__ __device__ constexpr int fft_len(int lc) { return fft_mult(lc) << fft_p2(lc); }
__host__ __device__ constexpr int fft_np2(int lc) { return fft_p2(lc) / 3 + (fft_p2(lc) % 3 ? 1 : 0); }
__host__ __device__ constexpr int fft_nodd(int lc) { return fft_mult(lc) == 1 ? 0 : (fft_mult(lc) == 9 ? 2 : 1); }
__host__ __device__ constexpr bool fft_merged(int lc) {
  return FFT_MERGE_ODD && fft_p2(lc) % 3 != 0 && (fft_mult(lc) == 3 || fft_mult(lc) == 5);
}
__host__ __device__ constexpr int fft_npasses(int lc) { return fft_np2(lc) + fft_nodd(lc) - (fft_merged(lc) ? 1 : 0); }
__host__ __device__ constexpr int fft_radix(int lc, int p) {
  return fft_merged(lc) && p == fft_p2(lc) / 3
             ? (1 << (fft_p2(lc) % 3)) * fft_mult(lc)
             : (p < fft_np2(lc) ? (p < fft_p2(lc) / 3 ? 8 : (fft_p2(lc) % 3 == 2 ? 4 : 2)) : (fft_mult(lc) == 5 ? 5 : 3));
}
__host__ __device__ constexpr int fft_ns(int lc, int p) {
  int ns = 1;
  for (int q = 0; q < p; q++) ns *= fft_radix(lc, q);
  return ns;
}
// lines of up to fft_out_max(lc) samples fit (n + h <= L checked by the caller):
// L / 2 for powers of two, else the largest power of two below L; the two raw
// input lines need 2 fft_out_max floats of shared memory
__host__ __device__ constexpr int fft_out_max(int lc) {
  return fft_mult(lc) == 1 ? fft_len(lc) / 2 : (fft_mult(lc) == 3 ? 2 : (fft_mult(lc) == 5 ? 4 : 8)) << fft_p2(lc);
}
__host__ __device__ constexpr int fft_raw_floats(int lc) { return 2 * fft_out_max(lc); }
// radix-2-stage equivalents charged to the error bound for the odd passes
__host__ __device__ constexpr int fft_odd_stages(int lc) { return fft_mult(lc) == 1 ? 0 : (fft_mult(lc) == 3 ? 2 : (fft_mult(lc) == 5 ? 3 : 4)); }

// Per-pass twiddle tables follow the L-entry table: pass p (sub-size Ns, radix R)
// holds W_{Ns R}^{r k} at [L + off_p + r Ns + k], k < Ns, r < R, so the lanes
// of a warp (consecutive k) read consecutive entries.
__host__ __device__ constexpr int fft_pass_twiddle_offset(int lc, int p) {
  int off = 0;
  for (int q = 0; q < p; q++) off += fft_radix(lc, q) * fft_ns(lc, q);
  return off;
}
__host__ __device__ constexpr int fft_twiddle_len(int lc) {
  return fft_len(lc) + fft_pass_twiddle_offset(lc, fft_npasses(lc));
}

// Shared-memory layout: one padding slot per 8 complex values, so the radix-8
// scatter of the first pass (stride 8 x 16 B between lanes) is conflict-free.
__host__ __device__ constexpr int fft_pad(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int fft_buf_len(int L) { return L + L / 8; }

// Every pass runs in place in one padded buffer (all threads read their
// butterflies' inputs, the CTA syncs, then all write): half the shared memory
// of ping-pong buffers, so 4 CTAs fit per SM at L = 2048 (and L = 8192 fits).
template <int LOG2L> __host__ __device__ constexpr bool fft_inplace() { return true; }

// Stockham pass p of radix R: butterfly j reads v[r] = src[j + r L/R], applies
// twiddles W_{Ns R}^{r k} (k = j mod Ns), runs the radix-R DFT and writes to
// dst[(j - k) R + k + r Ns] (natural order after the last pass).
template <int LOG2L, int P>
struct FftPass {
  static constexpr int L = fft_len(LOG2L);
  static constexpr int R = fft_radix(LOG2L, P);
  static constexpr int Ns = fft_ns(LOG2L, P);
  static constexpr int T = fft_threads_for<L>();
  static constexpr int NB = (L / R + T - 1) / T;  // butterflies per thread

  __device__ __forceinline__ static void twiddle(double2 (&v)[R], const double2 (&wv)[R]) {
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; r++) v[r] = cmul(v[r], wv[r]);
    }
  }
  __device__ __forceinline__ static int jmod(int j) { return (Ns & (Ns - 1)) == 0 ? (j & (Ns - 1)) : (j % Ns); }
  __device__ __forceinline__ static int dest(int j, int r) {
    const int k = jmod(j);
    return (j - k) * R + k + r * Ns;
  }
  // this thread's twiddles of the pass, loaded BEFORE the barrier that precedes
  // the pass (their latency overlaps the barrier wait instead of the pass)
  struct Tw {
    double2 w[NB][R];
  };
  __device__ __forceinline__ static void load_tw(Tw& t, const double2* tw) {
    if (Ns > 1) {
      unsigned tid;
      asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
#pragma unroll
      for (int b = 0; b < NB; b++) {
        const int j = (int)tid + b * T;
        if (j < L / R) {
          const double2* pt = tw + L + fft_pass_twiddle_offset(LOG2L, P) + jmod(j);
#pragma unroll
          for (int r = 1; r < R; r++) t.w[b][r] = ld_ordered(pt + r * Ns);  // not movable across barriers
        }
      }
    }
  }
  // in place with preloaded twiddles: every thread reads, the CTA syncs, every thread writes
  template <bool SPEC>
  __device__ __forceinline__ static void run_tw(double2* buf, const Tw& twv, const double* spec) {
    unsigned tid;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
    double2 v[NB][R];
#pragma unroll
    for (int t = 0; t < NB; t++) {
      const int j = (int)tid + t * T;
      if (j < L / R) {
#pragma unroll
        for (int r = 0; r < R; r++) v[t][r] = buf[fft_pad(j + r * (L / R))];
        twiddle(v[t], twv.w[t]);
        dft_any<R>(v[t]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NB; t++) {
      const int j = (int)tid + t * T;
      if (j < L / R) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int d = dest(j, r);
          double2 o = v[t][r];
          if (SPEC) {
            const double sp = ld_ordered(spec + d);
            o = make_double2(o.x * sp, -(o.y * sp));
          }
          buf[fft_pad(d)] = o;
        }
      }
    }
  }
};

// Passes P .. LAST-1 in place with twiddle prefetch: pass p + 1's twiddles are
// loaded after pass p's writes and before the barrier between them; after the
// last pass the twiddles of pass LAST (if it exists) go to `next`.
template <int LOG2L, int P, int LAST>
struct FftChainTw {
  template <bool SPEC_LAST, typename NextTw>
  __device__ __forceinline__ static void run(double2* buf, const double2* tw, const double* spec,
                                             const typename FftPass<LOG2L, P>::Tw& cur, NextTw& next) {
    FftPass<LOG2L, P>::template run_tw<SPEC_LAST && P == fft_npasses(LOG2L) - 1>(buf, cur, spec);
    if constexpr (P + 1 < LAST) {
      typename FftPass<LOG2L, P + 1>::Tw nt;
      FftPass<LOG2L, P + 1>::load_tw(nt, tw);
      __syncthreads();
      FftChainTw<LOG2L, P + 1, LAST>::template run<SPEC_LAST>(buf, tw, spec, nt, next);
    } else {
      if constexpr (LAST < fft_npasses(LOG2L)) FftPass<LOG2L, LAST>::load_tw(next, tw);
      __syncthreads();
    }
  }
};
struct NoTw {};

__device__ __forceinline__ double warp_max_sum(double v, double m, double* out_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(PLAS_FULL_MASK, v, o);
    m = fmax(m, __shfl_xor_sync(PLAS_FULL_MASK, m, o));
  }
  *out_max = m;
  return v;
}

// One axis pass of the level blur by FFT.  AXIS 0: lines = columns (x, c) of
// feat (row stride W*S), output to the tmp interior (row stride (W+2P)*S).
// AXIS 1: lines = rows (y, c) of tmp, output to target / den32 (EPI 1).
// One CTA of fft_threads_for<L>() threads per line pair (no persistent loop:
// across a loop the compiler hoists every pass's thread-only address
// arithmetic out of it and spills).  Dataflow: the first pass of the forward
// FFT reads the line pair straight from global memory (indices >= n are the
// zero padding); passes run in place in one padded shared buffer (two
// barriers each); the last pass of the second FFT keeps its outputs in
// registers and certifies / stores them.  The CTA also settles its own
// uncertain outputs with the exact SciPy fold from a shared-memory copy of
// the two input lines (FB_LOCAL of them; any excess goes to the global list).
// Callers guarantee n + h <= L and n <= fft_out_max(lc).
// In-CTA list capacity: 512 entries for L <= 4096 (several CTAs per SM), 4096
// for the long lengths (one CTA per SM, shared memory to spare; the first
// levels of an unsorted grid have hundreds of uncertain outputs per line pair).
#ifndef FFT_FB_LOCAL
#define FFT_FB_LOCAL 512
#endif
#ifndef FFT_FB_LOCAL_LONG
#define FFT_FB_LOCAL_LONG 4096
#endif
template <int L> __host__ __device__ constexpr int fft_fb_local() { return L > 4096 ? FFT_FB_LOCAL_LONG : FFT_FB_LOCAL; }

// A line pair's uncertain outputs: one warp per output runs the certified
// parallel fold (fold_cert.cuh) on the shared copy of its input line; the rare
// output it cannot settle takes the sequential SciPy fold on lane 0.  Not
// inlined: the FFT passes keep their register allocation (inlined, the fold's
// double-double state pushed the 1536 / 2560 / 3072 kernels into spills).
#ifndef FFT_WARP_FOLD_HMIN
#define FFT_WARP_FOLD_HMIN 0
#endif
struct SmemLine {
  const float* x;
  int n;
  __device__ __forceinline__ float operator()(int k) const { return (k >= 0 && k < n) ? x[k] : 0.f; }
};
template <int AXIS, int EPI>
__device__ __noinline__ void fft_cta_folds(const float* raw, int n, const int* flist, int nf, int h,
                                           const double* w, const float* __restrict__ den32, float* out,
                                           long long out_base, long long out_stride, long long line, int W, int nwarps,
                                           int* fb) {
  // cost model (cycles, measured shape): the sequential chain is ~10 per tap
  // on every thread at once; the warp fold ~40 per 32 taps + ~300 fixed, one
  // output per warp at a time.  Many uncertain outputs and short kernels favour
  // the threads (C3's 2560 / 3072 lines), few outputs and long kernels the
  // warps (C4's 5120 / 6144 lines).
  const long long seq_cost = (long long)((nf + nwarps * 32 - 1) / (nwarps * 32)) * h * 10;
  const long long warp_cost = (long long)((nf + nwarps - 1) / nwarps) * (((h + 31) >> 5) * 40 + 300);
  if (h < FFT_WARP_FOLD_HMIN || seq_cost <= warp_cost) {
    // one thread per output runs the sequential fold
    for (int t = threadIdx.x; t < nf; t += nwarps * 32) {
      const int e = flist[t];
      const int q = e >> 30, i = e & 0x3fffffff;
      float res = fold_sequential(SmemLine{raw + q * n, n}, i, h, w);
      if (EPI == 1) res = __fdiv_rn(res, den32[(AXIS == 0 ? (long long)i * W + line : line * W + i)]);
      out[out_base + q + (long long)i * out_stride] = res;
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  for (int t = threadIdx.x >> 5; t < nf; t += nwarps) {
    const int e = flist[t];
    const int q = e >> 30, i = e & 0x3fffffff;
    const SmemLine X{raw + q * n, n};
    float res;
    const bool ok = fold_certified_warp(X, i, h, w, &res);
    if (lane == 0) {
      if (!ok) res = fold_sequential(X, i, h, w);
#ifdef PLAS_FB_STATS
      if (!ok) atomicAdd(fb + 3, 1);  // diagnostics: sequential folds (header slot 3)
#endif
      if (EPI == 1) res = __fdiv_rn(res, den32[(AXIS == 0 ? (long long)i * W + line : line * W + i)]);
      out[out_base + q + (long long)i * out_stride] = res;
    }
  }
}

template <int AXIS, int EPI, int LOG2L>
__global__ void __launch_bounds__(fft_threads_for<fft_len(LOG2L)>(), fft_min_blocks<fft_len(LOG2L)>())
    blur_fft_kernel(const float* __restrict__ in, float* __restrict__ out, PadGeom pg, BlurLevelRef lvl,
                    FftPlan plan, const float* __restrict__ den32, int* __restrict__ fb, int fb_cap,
                    int* __restrict__ fb_other) {
  constexpr int L = fft_len(LOG2L);
  constexpr int T = fft_threads_for<L>();
  constexpr int NP = fft_npasses(LOG2L);
  extern __shared__ double2 fbuf[];
  double2* bufA = fbuf;
  double2* bufB = fft_inplace<LOG2L>() ? fbuf : fbuf + fft_buf_len(L);
  float* raw = reinterpret_cast<float*>(fbuf + (fft_inplace<LOG2L>() ? 1 : 2) * fft_buf_len(L));  // [2][n] lines
  __shared__ double red[64];
  constexpr int FB_LOCAL = fft_fb_local<L>();
  __shared__ int flist[FB_LOCAL > 0 ? FB_LOCAL : 1];
  __shared__ int nflag;
  if (blockIdx.x == 0 && threadIdx.x == 0 && fb_other) fb_other[0] = 0;
  if (threadIdx.x == 0) nflag = 0;
  const int tid = threadIdx.x;
  const int H = pg.H, W = pg.W, C = pg.C, S = pg.S;
  const int n = AXIS == 0 ? H : W;
  const long long WS = (long long)W * S;
  const long long WSP = (long long)(W + 2 * pg.pad) * S;
  const int cpairs = (C + 1) >> 1;
  // lines: columns [c0, c1) (axis 0) or rows [r0, r1) (axis 1), grid = lines x channel pairs
  const long long lline = blockIdx.x / cpairs;
  const long long line = lline + (AXIS == 0 ? pg.c0 : pg.r0);
  const int c = (int)(blockIdx.x - lline * cpairs) * 2;
  const bool has_b = c + 1 < C;
  // ---- forward FFT pass 0 straight from global memory (+ raw copy, ||z||^2, max|x|)
  {
    using P0 = FftPass<LOG2L, 0>;
    const long long in_stride = AXIS == 0 ? WS : (long long)S;
    const float* src = in + (AXIS == 0 ? line * S + c : line * WSP + c);
    double ss = 0.0, mx = 0.0;
#pragma unroll
    for (int t = 0; t < P0::NB; t++) {
      const int j = tid + t * T;
      if (j < L / P0::R) {
        double2 v[P0::R];
#pragma unroll
        for (int r = 0; r < P0::R; r++) {
          const int i = j + r * (L / P0::R);
          v[r] = make_double2(0.0, 0.0);
          if (i < n) {
            float a, b;
            if (has_b) {  // channels c, c+1 are adjacent (c even, rows 16-byte aligned)
              const float2 ab = __ldg(reinterpret_cast<const float2*>(src + (long long)i * in_stride));
              a = ab.x;
              b = ab.y;
            } else {
              a = __ldg(src + (long long)i * in_stride);
              b = 0.f;
            }
            raw[i] = a;
            raw[n + i] = b;
            v[r] = make_double2((double)a, (double)b);
            ss = fma(v[r].x, v[r].x, fma(v[r].y, v[r].y, ss));
            mx = fmax(mx, fmax(fabs(v[r].x), fabs(v[r].y)));
          }
        }
        dft_any<P0::R>(v);
#pragma unroll
        for (int r = 0; r < P0::R; r++) bufA[fft_pad(P0::dest(j, r))] = v[r];
      }
    }
    double m;
    ss = warp_max_sum(ss, mx, &m);
    if ((tid & 31) == 0) {
      red[2 * (tid >> 5)] = ss;
      red[2 * (tid >> 5) + 1] = m;
    }
  }
  typename FftPass<LOG2L, 1>::Tw tw1;
  FftPass<LOG2L, 1>::load_tw(tw1, plan.tw);
  __syncthreads();
  // ---- rest of the forward FFT (spectrum x conj in its last pass), then the
  //      second FFT up to its last pass
  static_assert(fft_inplace<LOG2L>(), "twiddle prefetch assumes the in-place passes");
  (void)bufB;
  typename FftPass<LOG2L, NP - 1>::Tw twl;  // the last pass's twiddles, prefetched by the chain
  {
    typename FftPass<LOG2L, 0>::Tw tw0;  // pass 0 has no twiddles (Ns = 1)
    FftChainTw<LOG2L, 1, NP>::template run<true>(bufA, plan.tw, plan.spec, tw1, tw0);
    FftChainTw<LOG2L, 0, NP - 1>::template run<false>(bufA, plan.tw, plan.spec, tw0, twl);
  }
  const double2* last_src = bufA;
  // ---- bound B for this pair
  int h;
  const double* w;
  lvl.get(&h, &w);
  double norm2 = 0.0, M = 0.0;
  for (int i = 0; i < T / 32; i++) {
    norm2 += red[2 * i];
    M = fmax(M, red[2 * i + 1]);
  }
  const double fold_scale = (2.0 * h + 4.0) * 2.0 * 1.1102230246251565e-16;
  const double B = (plan.cbound * sqrt(norm2) + fold_scale * M) * 1.0001;
  const double invL = 1.0 / (double)L;
  const long long out_stride = AXIS == 0 ? WSP : (long long)S;
  const long long out_base = AXIS == 0 ? line * S + c : line * WS + c;
  // ---- last pass of the second FFT: outputs j + r Ns stay in registers
  {
    using PL = FftPass<LOG2L, NP - 1>;
#pragma unroll
    for (int t = 0; t < PL::NB; t++) {
      const int j = tid + t * T;
      const bool jv = j < L / PL::R;
      double2 v[PL::R];
      const double2(&wv)[PL::R] = twl.w[t];
#pragma unroll
      for (int r = 0; r < PL::R; r++) v[r] = jv ? last_src[fft_pad(j + r * (L / PL::R))] : make_double2(0.0, 0.0);
      PL::twiddle(v, wv);
      dft_any<PL::R>(v);
#pragma unroll
      for (int r = 0; r < PL::R; r++) {
        const int i = PL::dest(j, r);
        if (PL::Ns * r >= fft_out_max(LOG2L)) continue;  // dest(j, r) = j + r Ns >= n: zero padding, unused
        const bool in_range = jv && i < n;
        const float dn = (EPI == 1 && in_range) ? den32[(AXIS == 0 ? (long long)i * W + line : line * W + i)] : 1.f;
        float res[2];
        bool sure[2];
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const double acc = q == 0 ? v[r].x * invL : -(v[r].y * invL);
          sure[q] = __double2float_rn(__dsub_rn(acc, B)) == __double2float_rn(__dadd_rn(acc, B));
          res[q] = __double2float_rn(acc);
          if (EPI == 1) res[q] = __fdiv_rn(res[q], dn);
        }
        float* dsto = out + out_base + (long long)i * out_stride;
        if (in_range) {
          if (has_b && sure[0] && sure[1]) {
            *reinterpret_cast<float2*>(dsto) = make_float2(res[0], res[1]);
          } else {
            if (sure[0]) dsto[0] = res[0];
            if (has_b && sure[1]) dsto[1] = res[1];
          }
        }
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const bool valid = in_range && (q == 0 || has_b);
          const bool unsure = valid && !sure[q];
          // local list (warp-aggregated; trip counts are warp-uniform), overflow to the global list
          const unsigned bal = __ballot_sync(PLAS_FULL_MASK, unsure);
          if (bal) {
            const int lane = tid & 31, leader = __ffs(bal) - 1;
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
    }
  }
  __syncthreads();
  // ---- this CTA's uncertain outputs: one warp per output runs the certified
  // parallel fold (fold_cert.cuh) on the shared copy of its input line; the
  // rare output it cannot settle takes the sequential SciPy fold on lane 0
#ifdef FFT_DEBUG_NO_FOLD
  const int nf = 0;  // diagnostics only (timing without the exact folds): outputs are wrong
#else
  const int nf = min(nflag, FB_LOCAL);
#endif
#ifdef PLAS_FB_STATS
  if (tid == 0 && nf) atomicAdd(fb + 2, nf);  // diagnostics: in-CTA folds (header slot 2)
#endif
  if (nf) fft_cta_folds<AXIS, EPI>(raw, n, flist, nf, h, w, den32, out, out_base, out_stride, line, W, T / 32, fb);
}

// shared memory of blur_fft_kernel for an L-point FFT
inline size_t fft_smem_bytes(int lc) {
  const size_t nbuf = 1;  // fft_inplace
  return sizeof(double2) * nbuf * (size_t)fft_buf_len(fft_len(lc)) + sizeof(float) * (size_t)fft_raw_floats(lc);
}

// Real spectrum of the current level's symmetric kernel on L points:
// K[m] = w0 + 2 sum_{j=1..h} w_j cos(2 pi j m / L), cosines from the twiddle
// table (exact index reduction), compensated (TwoProduct + TwoSum) so the
// error stays ~3 ulp regardless of h.
__device__ __forceinline__ double fft_spectrum_value(int m, int h, const double* __restrict__ w, const FftPlan& plan) {
  const int L = plan.L;
  double s = __ldg(w), comp = 0.0;
  int jm = 0;  // j m mod L
  for (int j = 1; j <= h; j++) {
    jm += m;
    if (jm >= L) jm -= L;
    const double cj = __ldg(&plan.tw[jm].x);
    const double wj2 = 2.0 * __ldg(w + j);
    const double p = wj2 * cj;
    const double pe = fma(wj2, cj, -p);  // exact product error
    const double t = s + p;
    const double bp = t - s;
    const double te = (s - (t - bp)) + (p - bp);  // TwoSum error
    s = t;
    comp += te + pe;
  }
  return s + comp;
}

__global__ void fft_spectrum_kernel(BlurLevelRef lvl, FftPlan plan) {
  int h;
  const double* w;
  lvl.get(&h, &w);
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < plan.L; m += gridDim.x * blockDim.x)
    plan.spec[m] = fft_spectrum_value(m, h, w, plan);
}

}  // namespace plas
