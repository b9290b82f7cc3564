// plas_b200.cu -- C ABI + sort driver of the B200-native PLAS hot path.
//
// Reference call stack: sort_grid_report -> _sort
// (plas.py:226-286) -> per level blur_target + grid_distance, per pass
// rng draws + _reassign_pass -> _assign_groups + grid_distance.
//
// PARITY mode replays that loop from the host with NumPy-exact draws (one
// stream sync per pass to read the device-side convergence flag, with the
// next pass's draws generated while the GPU works).
// DEVICE mode builds the whole sort as ONE CUDA graph: an outer WHILE
// conditional node over levels and an inner WHILE node over passes whose
// condition is set on the device by the controller kernel (K4), so the host
// launches once and syncs once.
#include <cuda_runtime.h>
#include <math.h>
#include <cmath>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/plas_b200.h"
#include "assign.cuh"
#include "prep.cuh"
#include "blur.cuh"
#include "blur_fast.cuh"
#include "blur_fft.cuh"
#include "common.cuh"
#include "control.cuh"
#include "host_rng.h"
#include "np_sum.cuh"
#include "smooth.cuh"

using namespace plas;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return fail(PLAS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));      \
  } while (0)

#define CKL()                                                                               \
  do {                                                                                      \
    cudaError_t _e = cudaGetLastError();                                                    \
    if (_e != cudaSuccess)                                                                  \
      return fail(PLAS_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e) + " @" + \
                                     std::to_string(__LINE__));                             \
  } while (0)

constexpr int MAX_PARTS = 4096;

int num_sms() {
  static std::atomic<int> sms{0};  // lazily initialised caches: atomics, written with the same value by any thread
  if (!sms) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms = v > 0 ? v : 148;
  }
  return sms;
}

int grid_for(long long work, int threads, int per_sm) {
  long long g = (work + threads - 1) / threads;
  long long cap = (long long)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g > MAX_PARTS) g = MAX_PARTS;
  if (g < 1) g = 1;
  return (int)g;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// bump allocator over a caller-provided workspace
struct Carver {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = align_up(off);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += sizeof(T) * count;
    return p;
  }
};

// Dynamic shared-memory limits are per-kernel process state: concurrent calls
// from several host threads may need different amounts for one kernel, so the
// limit only ever grows (a lower request never shrinks it under another
// thread's pending launch).
std::mutex g_smem_mu;
std::vector<std::pair<const void*, int>> g_smem_limits;
cudaError_t raise_smem_limit(const void* fn, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_smem_mu);
  for (auto& e : g_smem_limits)
    if (e.first == fn) {
      if (e.second >= (int)bytes) return cudaSuccess;
      const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (r == cudaSuccess) e.second = (int)bytes;
      return r;
    }
  const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (r == cudaSuccess) g_smem_limits.push_back({fn, (int)bytes});
  return r;
}

int row_stride(int dim) { return (dim + 3) / 4 * 4; }

// ---------------------------------------------------------------- schedule
struct Schedule {
  std::vector<double> radii, weights;
  std::vector<int> betas, hs;
  std::vector<long long> woff;
};

double default_initial_radius(int side) { return std::max(side / 2.0 - 1.0, 2.0); }

void build_schedule(const plas_sort_args* a, int side, Schedule* s) {
  s->radii.clear();
  if (a->radii) {
    s->radii.assign(a->radii, a->radii + a->num_levels);
  } else {
    double r = std::isnan(a->initial_radius) ? default_initial_radius(side) : a->initial_radius;
    while (r >= 1.0) {  // plas.py:251, 274 (repeated multiplication)
      s->radii.push_back(r);
      r *= a->radius_decay;
    }
  }
  const int L = (int)s->radii.size();
  s->betas.resize(L);
  s->hs.resize(L);
  s->woff.resize(L);
  s->weights.clear();
  for (int l = 0; l < L; l++) {
    const double r = s->radii[l];
    int beta = std::max(a->min_block_size, (int)r + 1);  // plas.py:60-61
    s->betas[l] = std::min(beta, side);
    s->hs[l] = (int)ceil(r);
    if (a->weights) {
      s->woff[l] = a->weight_offsets[l];
    } else {
      // scipy _gaussian_kernel1d(sigma=r/2, 0, h): exp(-0.5/sigma^2 x^2) / sum
      const int h = s->hs[l];
      const double sigma = r / 2.0, sigma2 = sigma * sigma;
      std::vector<double> phi(2 * h + 1);
      double sum = 0.0;
      for (int x = -h; x <= h; x++) phi[x + h] = exp(-0.5 / sigma2 * (double)(x * x));
      for (double v : phi) sum += v;
      s->woff[l] = (long long)s->weights.size();
      for (int j = 0; j <= h; j++) s->weights.push_back(phi[h + j] / sum);
    }
  }
  if (a->weights) {
    long long wl = 0;
    for (int l = 0; l < L; l++) wl = std::max(wl, (long long)(s->woff[l] + s->hs[l] + 1));
    s->weights.assign(a->weights, a->weights + wl);
  }
}

// ---------------------------------------------------------------- workspace
struct SortWs {
  Ctrl* ctrl;
  float *feat, *target, *tmp, *den32;  // feat / tmp point at the interior of zero-padded buffers
  float *feat_alloc, *tmp_alloc;
  size_t feat_alloc_floats, tmp_alloc_floats;
  int* fb0;  // blur fallback lists (axis 0 / axis 1)
  int* fb1;
  int fb_cap;
  int pad;
  double* dcache;  // per-cell fp64 distance to the target (level start + pass updates)
  int* idx;
  double* rowweight;
  double* partials;
  int* flags;  // [0] nonfinite, [1] moved
  double* scalars;  // [0] vad mean, [1] vad0, [2] vad1
  double* radii;
  int *betas, *hs;
  long long* woff;
  double* weights;
  long long* level_counts;
  double* trace;
  int4* pdraw;  // DEVICE: per-pass draws of the current level
  int* prec;    // DEVICE: per-pass grouping records (class shapes + Feistel keys)
  int* mp;   // parity: master permutation (beta0^2)
  int* sel;  // parity: 9 class selections
  long long sel_stride;
  int* list;      // moved-cell list of the current pass
  double* spart;  // statistic-kernel partials
  float* orig32;      // sharding: f32 features in element order
  float *xsend, *xrecv;  // sharding: FFT-tier axis-0 band exchange (all-to-all) buffers
  double* lvl_part;      // sharding: level-start partials, XPART doubles per rank (all-gathered in place)
  int* bands;            // sharding: per level [lo[world], hi[world], cs[world + 1]] for the pack kernels
  // PARITY on one GPU: NumPy-order grid_distance (np_sum.cuh)
  double* np_v;          // per-cell sqrt(row sum) [n]
  double* np_vals;       // tree node values [leaves + internal]
  long long* np_lstart;  // leaf starts
  int *np_llen, *np_left, *np_right, *np_order, *np_hoff;
  double* np_out;        // (sum, sum / n)
  // PARITY: NumPy-order vad over M = 2 side (side - 1) D pooled differences
  size_t vad_cap;        // tree leaves the arrays hold
  double* vad_vals;
  long long* vad_lstart;
  int *vad_llen, *vad_left, *vad_right, *vad_order, *vad_hoff;
  double* vad_out;       // (sum, mean, sum of squares, var)
  // FFT tier: up to FFT_PLANS lengths (the shortest that fits each level's h)
  int fft_count;                   // number of lengths
  int fft_codes[4];                // length codes, increasing length
  double2* fft_tws[4];             // twiddles of each length
  double* fft_spec;                // spectrum of the current level (longest length)
  FftPlan* fft_plans;              // device copies of the plans (level_prep_kernel)
  int* lvl_mode;                   // per level: plan index, FFT_PLANS = tile tier, FFT_PLANS + 1 = direct
  int fft_L;                       // longest length (0: no FFT tier)
};

// ---------------------------------------------------------------- direct fold, compile-time h
// Direct-tier levels with h <= PAD_SMALL_HMAX run blur_pad_kernel<AXIS, EPI, h>
// (static tap loop); larger h the runtime-h kernel.  PLAS_PAD_SMALL=0 turns
// the specialisations off (A/B).
constexpr int PAD_SMALL_HMAX = 16;
using PadFn = void (*)(const float*, float*, PadGeom, BlurLevelRef, const float*, int*, int, int*);
template <int H>
PadFn pad_small_fn(int axis) {
  return axis == 0 ? (PadFn)blur_pad_kernel<0, 0, H> : (PadFn)blur_pad_kernel<1, 1, H>;
}
int pad_small_enabled() {
  static std::atomic<int> v{-1};
  if (v < 0) v = getenv("PLAS_PAD_SMALL") ? (atoi(getenv("PLAS_PAD_SMALL")) != 0) : 1;
  return v;
}
PadFn pad_fn(int axis, int h) {
  if (pad_small_enabled()) switch (h) {
      case 1: return pad_small_fn<1>(axis);
      case 2: return pad_small_fn<2>(axis);
      case 3: return pad_small_fn<3>(axis);
      case 4: return pad_small_fn<4>(axis);
      case 5: return pad_small_fn<5>(axis);
      case 6: return pad_small_fn<6>(axis);
      case 7: return pad_small_fn<7>(axis);
      case 8: return pad_small_fn<8>(axis);
      case 9: return pad_small_fn<9>(axis);
      case 10: return pad_small_fn<10>(axis);
      case 11: return pad_small_fn<11>(axis);
      case 12: return pad_small_fn<12>(axis);
      case 13: return pad_small_fn<13>(axis);
      case 14: return pad_small_fn<14>(axis);
      case 15: return pad_small_fn<15>(axis);
      case 16: return pad_small_fn<16>(axis);
    }
  return axis == 0 ? (PadFn)blur_pad_kernel<0, 0> : (PadFn)blur_pad_kernel<1, 1>;
}

// ---------------------------------------------------------------- FFT blur tier
constexpr int FFT_PLANS = 4;  // 32 <= L <= 8192 (16 L bytes of shared memory per CTA)

template <int AXIS, int EPI>
void* fft_kernel_ptr(int lc) {
  switch (lc) {
    case 5: return (void*)blur_fft_kernel<AXIS, EPI, 5>;
    case 6: return (void*)blur_fft_kernel<AXIS, EPI, 6>;
    case 7: return (void*)blur_fft_kernel<AXIS, EPI, 7>;
    case 8: return (void*)blur_fft_kernel<AXIS, EPI, 8>;
    case 9: return (void*)blur_fft_kernel<AXIS, EPI, 9>;
    case 10: return (void*)blur_fft_kernel<AXIS, EPI, 10>;
    case 11: return (void*)blur_fft_kernel<AXIS, EPI, 11>;
    case 12: return (void*)blur_fft_kernel<AXIS, EPI, 12>;
    case 13: return (void*)blur_fft_kernel<AXIS, EPI, 13>;
    case 32 + 9: return (void*)blur_fft_kernel<AXIS, EPI, 32 + 9>;    // 1536
    case 32 + 10: return (void*)blur_fft_kernel<AXIS, EPI, 32 + 10>;  // 3072
    case 32 + 11: return (void*)blur_fft_kernel<AXIS, EPI, 32 + 11>;  // 6144
    case 64 + 9: return (void*)blur_fft_kernel<AXIS, EPI, 64 + 9>;    // 2560
    case 64 + 10: return (void*)blur_fft_kernel<AXIS, EPI, 64 + 10>;  // 5120
  }
  return nullptr;
}

int fft_threads(int L) { return fft_threads_len(L); }

// FFT length for lines of n samples and half-widths up to hmax: the shortest
// instantiated L (2^k, 5 <= k <= 13; 3 * 2^k, 9 <= k <= 11; 5 * 2^k, 9 <= k
// <= 10) with n + hmax <= L and n <= fft_out_max; returns the length code, -1
// if none.  PLAS_FFT3 = bit mask of the odd factors allowed (1: 3, 2: 5; 0
// keeps to powers of two).  Measured: 2560 beats 3072 at C3
// (1.895 vs 2.033 s), 1280 loses to 1536 at C2 (114.9 vs 114.3 ms), so 5 * 2^8
// is not offered; the 9 * 2^k lengths (radix-3 twice) lost at every config.
int fft_choose_code(long long n, long long hmax) {
  static std::atomic<int> odd_mask{-1};
  if (odd_mask < 0) {
    const char* e = getenv("PLAS_FFT3");
    odd_mask = e ? (atoi(e) & 3) : 3;
  }
  static const int codes[] = {5, 6, 7, 8, 9, 10, 11, 12, 13,           // 2^k
                              32 + 9, 32 + 10, 32 + 11,               // 3 2^k
                              64 + 9, 64 + 10};                       // 5 2^k
  int best = -1;
  for (int lc : codes) {
    if (lc >= 32 && !(odd_mask >> (lc / 32 - 1) & 1)) continue;
    if (n + hmax <= fft_len(lc) && n <= fft_out_max(lc) && (best < 0 || fft_len(lc) < fft_len(best))) best = lc;
  }
  return best;
}
// the sort's FFT length code: covers the top level's half-width ceil(side / 2 - 1)
int fft_alloc_code(int side) {
  const long long h0 = (long long)ceil(std::max(side / 2.0 - 1.0, 2.0));
  return fft_choose_code(side, h0);
}
int fft_min_h(int L, int S);
// the lengths a sort at this side can use: the shortest fitting length of every
// half-width from the crossover up to the top level's (sorted by length)
void fft_plan_codes(int side, int S, int* count, int* codes) {
  *count = 0;
  const int top = fft_alloc_code(side);
  if (top < 0) return;
  const long long h0 = (long long)ceil(std::max(side / 2.0 - 1.0, 2.0));
  const int hmin = std::max(fft_min_h(fft_len(top), S), 1);
  for (long long h = hmin; h <= h0; h++) {
    const int lc = fft_choose_code(side, h);
    if (lc < 0) continue;
    bool seen = false;
    for (int i = 0; i < *count; i++) seen |= codes[i] == lc;
    if (!seen && *count < 4) codes[(*count)++] = lc;
  }
  std::sort(codes, codes + *count, [](int a, int b) { return fft_len(a) < fft_len(b); });
}

// smallest half-width that takes the FFT tier for length L (0 = never);
// PLAS_FFT_MIN_H overrides.  Measured crossovers: 48 at C2 (L = 1536: 114.7 vs
// 115.5 ms at 64), 64 at C4 (L = 6144: 2.625 vs 2.641 s at 48).
int fft_min_h(int L, int S) {
  static std::atomic<int> v{-2};
  if (v == -2) {
    const char* e = getenv("PLAS_FFT_MIN_H");
    v = e ? std::max(atoi(e), 0) : -1;
  }
  if (v >= 0) return v;
  if (S > 16) return 40;  // C3 (59 channels): 1.661 s at 40 vs 1.672 s at 64
  return L <= 2048 ? 48 : 64;
}

// largest half-width of the one-kernel tile blur (0 = off); PLAS_TILE_BLUR_HMAX
// overrides.  Measured: 4 is best at C2 (the tile kernel is latency-bound
// above); for rows wider than 16 floats the direct fold wins at every h (C3:
// 1.69 s without the tile tier, 1.75 s with h <= 2, 1.80 s with h <= 4 -- the
// tile kernel reads each row once per channel pair, ~10x its algorithmic bytes)
int tile_blur_hmax(int S) {
  static std::atomic<int> v{-2};
  if (v == -2) {
    const char* e = getenv("PLAS_TILE_BLUR_HMAX");
    v = e ? std::min(std::max(atoi(e), 0), TB_HMAX) : -1;
  }
  if (v >= 0) return v;
  // round 2: the direct fold with compile-time half-widths (converged warps)
  // beats the one-kernel tile tier at every h <= 4 (C2: hmax 4 -> 104.6 ms,
  // 2 -> 104.3, 0 -> 104.05; the tier stays available: PLAS_TILE_BLUR_HMAX,
  // plas_blur_target_tiers tier 2)
  (void)S;
  return 0;
}

// relative error constant of the FFT convolution (blur_fft.cuh), x2 safety
// Higham Thm 24.2 per radix-2 stage (eta); the radix-3 stage (two adds per
// output, a product with the rounded sqrt3 / 2, |A| = sqrt3) is charged 2 eta
double fft_error_constant(int lc) {
  const double u = ldexp(1.0, -53);
  const double mu = 2.0 * u, g4 = 4.0 * u / (1.0 - 4.0 * u);
  const double eta = mu + g4 * (sqrt(2.0) + mu);
  const double ke = (double)(fft_p2(lc) + fft_odd_stages(lc)) * eta;
  const double c = ke / (1.0 - ke);
  const double eK = 4.0 * u;
  const double e2 = (c + u * (1.0 + c)) * (1.0 + eK) + eK;
  return 2.0 * (c * (1.0 + e2) + e2);
}

// e^{-2 pi i t / L} for t < L (correctly rounded from long double), then the
// per-pass tables W_{Ns R}^{r k} = e^{-2 pi i r k step / L} (blur_fft.cuh)
void fft_twiddles(int lc, std::vector<double2>* tw) {
  const int L = fft_len(lc);
  tw->resize(fft_twiddle_len(lc));
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int t = 0; t < L; t++) {
    const long double a = -2.0L * pi * (long double)t / (long double)L;
    (*tw)[t] = make_double2((double)cosl(a), (double)sinl(a));
  }
  for (int p = 0; p < fft_npasses(lc); p++) {
    const int R = fft_radix(lc, p), Ns = fft_ns(lc, p), step = L / (Ns * R);
    for (int r = 0; r < R; r++)
      for (int k = 0; k < Ns; k++)
        (*tw)[L + fft_pass_twiddle_offset(lc, p) + r * Ns + k] = (*tw)[((long long)r * k * step) % L];
  }
}

// zero halo of the padded blur buffers: the largest half-width plus one chunk
int blur_pad(int side) { return (int)ceil(std::max(side / 2.0 - 1.0, 2.0)) + std::max(BLUR_R, BPAD_R) + 1; }

size_t carve_sort(char* base, long long n, int dim, int L, long long wlen, long long tcap,
                  int rng_mode, int side, long long list_cap, SortWs* w, int world = 1) {
  Carver c{base};
  const int S = row_stride(dim);
  const int P = blur_pad(side);
  w->pad = P;
  w->ctrl = c.take<Ctrl>(1);
  w->feat_alloc_floats = (size_t)(side + 2 * P) * side * S;
  w->feat_alloc = c.take<float>(w->feat_alloc_floats);
  w->feat = w->feat_alloc ? w->feat_alloc + (size_t)P * side * S : nullptr;
  w->target = c.take<float>((size_t)n * S);
  w->tmp_alloc_floats = (size_t)side * (side + 2 * P) * S;
  w->tmp_alloc = c.take<float>(w->tmp_alloc_floats);
  w->tmp = w->tmp_alloc ? w->tmp_alloc + (size_t)P * S : nullptr;
  w->fb_cap = (int)std::min<long long>(n * S / 8 + 1024, 1LL << 26);
  w->fb0 = c.take<int>((size_t)FB_HEADER + w->fb_cap);
  w->fb1 = c.take<int>((size_t)FB_HEADER + w->fb_cap);
  w->den32 = c.take<float>((size_t)n);
  w->dcache = c.take<double>((size_t)n);
  w->idx = c.take<int>((size_t)n);
  w->rowweight = c.take<double>((size_t)side);
  w->partials = c.take<double>(MAX_PARTS);
  w->flags = c.take<int>(8);
  w->scalars = c.take<double>(8);
  w->radii = c.take<double>(std::max(L, 1));
  w->betas = c.take<int>(std::max(L, 1));
  w->hs = c.take<int>(std::max(L, 1));
  w->woff = c.take<long long>(std::max(L, 1));
  w->weights = c.take<double>(std::max(wlen, 1LL));
  w->level_counts = c.take<long long>(std::max(L, 1));
  w->trace = c.take<double>(std::max(tcap, 1LL));
  long long b0 = side;  // beta0 <= side
  // per-class grouping tables: PARITY (class_select_kernel) and DEVICE (gen_class_tables)
  w->sel_stride = (b0 * b0 + 3) / 4 * 4;  // every class row 16-byte aligned
  w->mp = c.take<int>(rng_mode == PLAS_RNG_PARITY ? (size_t)(b0 * b0) : 1);
  // two buffers in DEVICE mode (pass parity: pass p reads one while building p + 1's)
  w->sel = c.take<int>((size_t)((rng_mode == PLAS_RNG_PARITY ? 9 : 18) * w->sel_stride));
  w->pdraw = c.take<int4>(rng_mode == PLAS_RNG_PARITY ? 1 : (size_t)PDRAW_MAX);
  w->prec = c.take<int>(rng_mode == PLAS_RNG_PARITY ? 1 : (size_t)PDRAW_MAX * PREC_INTS);
  w->list = c.take<int>((size_t)std::max(list_cap, 1LL));
  w->spart = c.take<double>(MAX_PARTS + 2);  // [MAX_PARTS, +2): the pass statistic's 128-bit accumulator
  w->orig32 = world > 1 ? c.take<float>((size_t)n * S) : nullptr;
  // banded FFT levels: a rank sends its columns of every rank's band (<= 2 side
  // rows in total: bands are side / world + beta <= 2 side / world rows) and
  // receives its band of every column
  const size_t xfl = world > 1 ? (size_t)n * S * 2 / world + (size_t)side * S : 1;
  w->xsend = c.take<float>(xfl);
  w->xrecv = c.take<float>(xfl);
  w->lvl_part = c.take<double>((size_t)XPART * std::max(world, 1));
  w->bands = c.take<int>((size_t)3 * std::max(world, 1) + 1);
  // NumPy tree: leaves hold 8..128 cells (more than n / 128 + 2 of them), as
  // many internal nodes, heights <= 64
  const bool npx = rng_mode == PLAS_RNG_PARITY && world <= 1;
  const size_t nleaf = npx ? (size_t)(n / 64 + 4) : 1;
  w->np_v = c.take<double>(npx ? (size_t)n : 1);
  w->np_vals = c.take<double>(2 * nleaf);
  w->np_lstart = c.take<long long>(nleaf);
  w->np_llen = c.take<int>(nleaf);
  w->np_left = c.take<int>(nleaf);
  w->np_right = c.take<int>(nleaf);
  w->np_order = c.take<int>(nleaf);
  w->np_hoff = c.take<int>(72);
  w->np_out = c.take<double>(2);
  const long long mv = 2LL * side * (side - 1) * dim;
  w->vad_cap = rng_mode == PLAS_RNG_PARITY ? (size_t)(mv / 64 + 4) : 1;
  w->vad_vals = c.take<double>(2 * w->vad_cap);
  w->vad_lstart = c.take<long long>(w->vad_cap);
  w->vad_llen = c.take<int>(w->vad_cap);
  w->vad_left = c.take<int>(w->vad_cap);
  w->vad_right = c.take<int>(w->vad_cap);
  w->vad_order = c.take<int>(w->vad_cap);
  w->vad_hoff = c.take<int>(72);
  w->vad_out = c.take<double>(4);
  fft_plan_codes(side, row_stride(dim), &w->fft_count, w->fft_codes);
  w->fft_L = w->fft_count ? fft_len(w->fft_codes[w->fft_count - 1]) : 0;
  for (int i = 0; i < 4; i++)
    w->fft_tws[i] = i < w->fft_count ? c.take<double2>((size_t)fft_twiddle_len(w->fft_codes[i])) : nullptr;
  w->fft_spec = c.take<double>((size_t)std::max(w->fft_L, 1));
  w->fft_plans = c.take<FftPlan>(4);
  w->lvl_mode = c.take<int>((size_t)std::max(L, 1));
  return align_up(c.off);
}

// ---------------------------------------------------------------- level set-up (graph mode)
// The data-independent set-up of a level in one kernel (one graph node instead
// of four): block ranges [0, nd) build the level's pass draw records
// (pass_draw_item), [nd, nd + nr) the row weights A(y) (border_row_value),
// [nd + nr, nd + nr + ns) the real FFT spectrum if the level uses the FFT
// tier; block 0 thread 0 does level_begin_kernel's bookkeeping.  Every block
// reads only what is stable across the level boundary (Ctrl.level, side, the
// keys, the schedule), so no block waits for another.
__global__ void level_prep_kernel(Ctrl* c, Sched s, unsigned long long blur_switch, unsigned long long tile_cond,
                                  int4* __restrict__ pdraw, int* __restrict__ prec, double* __restrict__ rowweight,
                                  BlurLevelRef lvl, const int* __restrict__ lvl_mode,
                                  const FftPlan* __restrict__ plans, int nplans, int nd, int nr) {
  const int level = c->level, side = c->side;
  const int mode = lvl_mode[level];
  const int beta = s.betas[level];
  int h;
  const double* w;
  lvl.get(&h, &w);
  const int b = blockIdx.x;
  if (b < nd) {
    for (int t = b * blockDim.x + threadIdx.x; t < PDRAW_MAX * 16; t += nd * blockDim.x)
      pass_draw_item(c, level, beta, side, t, pdraw, prec);
    if (b == 0 && threadIdx.x == 0) {
      c->pdraw = pdraw;
      c->prec = prec;
      c->pdraw_level = level;
      // level_begin_kernel
      c->beta = beta;
      c->h = h;
      c->lv_cap = (beta * beta + 3) / 4;
      make_fastdiv((unsigned)c->lv_cap, &c->lv_cap_m, &c->lv_cap_l);
      c->lv_seg_base = num_segments(beta, beta, side);
      make_fastdiv((unsigned)c->lv_seg_base, &c->lv_seg_m[0], &c->lv_seg_l[0]);
      make_fastdiv((unsigned)(c->lv_seg_base + 1), &c->lv_seg_m[1], &c->lv_seg_l[1]);
      set_cond(blur_switch, (unsigned)mode);
      set_cond(tile_cond, use_tile(beta, c->S) ? 1u : 0u);
      c->pass = 0;
      c->strikes = 0;
      c->level_done = 0;
    }
  } else if (b < nd + nr) {
    for (int y = (b - nd) * blockDim.x + threadIdx.x; y < side; y += nr * blockDim.x)
      rowweight[y] = border_row_value(y, side, h, w);
  } else if (mode < nplans) {
    const FftPlan plan = plans[mode];
    const int ns = gridDim.x - nd - nr;
    for (int m = (b - nd - nr) * blockDim.x + threadIdx.x; m < plan.L; m += ns * blockDim.x)
      plan.spec[m] = fft_spectrum_value(m, h, w, plan);
  }
}

// ---------------------------------------------------------------- graph helpers
template <typename... KArgs, typename... Args>
cudaError_t add_kernel(cudaGraphNode_t* out, cudaGraph_t g, const cudaGraphNode_t* deps, int ndeps,
                       void (*kern)(KArgs...), dim3 grid, dim3 block, Args&&... args) {
  std::tuple<typename std::decay<KArgs>::type...> vals(std::forward<Args>(args)...);
  void* ptrs[sizeof...(KArgs) > 0 ? sizeof...(KArgs) : 1];
  std::apply([&](auto&... v) {
    int i = 0;
    ((ptrs[i++] = (void*)&v), ...);
  }, vals);
  cudaKernelNodeParams p{};
  p.func = (void*)kern;
  p.gridDim = grid;
  p.blockDim = block;
  p.sharedMemBytes = 0;
  p.kernelParams = ptrs;
  p.extra = nullptr;
  return cudaGraphAddKernelNode(out, g, deps, ndeps, &p);
}

cudaError_t add_while(cudaGraphNode_t* out, cudaGraph_t g, const cudaGraphNode_t* deps, int ndeps,
                      cudaGraphConditionalHandle h, cudaGraph_t* body) {
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaError_t e = cudaGraphAddNode(out, g, deps, ndeps, &p);
  if (e == cudaSuccess) *body = p.conditional.phGraph_out[0];
  return e;
}

// kernel configuration shared by both modes
struct Launch {
  int S, D, side;
  long long n;
  int blur_grid, fb_grid, den_grid, rows_grid, dist_grid, pass_grid, tile_grid, vad_grid;
  dim3 tb_grid;
  PadGeom pg;
  BlurLevelRef lvl;
  Sched sched;
};

// PLAS_K3_PLAIN=1 selects the unpipelined gather kernel for rows <= 16 floats (A/B)
bool k3_plain() {
  static std::atomic<int> v{-1};
  if (v < 0) v = getenv("PLAS_K3_PLAIN") && atoi(getenv("PLAS_K3_PLAIN")) ? 1 : 0;
  return v == 1;
}
template <bool PARITY>
void* pass_kernel_ptr(int S) {
  if (S <= 16) return k3_plain() ? (void*)pass_kernel<false, PARITY> : (void*)pass_kernel_pipe<PARITY>;
  return (void*)pass_kernel<true, PARITY>;
}

int pass_grid_size(int S) {
  static std::atomic<int> cached[3];
  int which = S <= 16 ? 0 : 1;
  if (!cached[which]) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)pass_kernel_ptr<false>(S), 256, 0);
    if (occ <= 0) occ = 1;
    cached[which] = std::min(num_sms() * occ, MAX_PARTS);
  }
  return cached[which];
}

// Instantiated sort graphs by workspace layout (a few entries; the oldest is
// destroyed when a new shape arrives).
struct GraphKey {
  const void* ws;
  size_t ws_bytes;
  long long n;
  int D, L;
  long long wlen, tcap;
  int mode, device;
  bool operator==(const GraphKey& o) const {
    return ws == o.ws && ws_bytes == o.ws_bytes && n == o.n && D == o.D && L == o.L && wlen == o.wlen &&
           tcap == o.tcap && mode == o.mode && device == o.device;
  }
};
// An entry is shared by its users: eviction only drops the cache's reference,
// and the exec is destroyed when the last sort that fetched it returns (never
// while another thread is launching it).
struct GraphExecHolder {
  cudaGraphExec_t ge = nullptr;
  ~GraphExecHolder() {
    if (ge) cudaGraphExecDestroy(ge);
  }
};
using GraphExecRef = std::shared_ptr<GraphExecHolder>;
std::mutex g_graph_mu;
std::vector<std::pair<GraphKey, GraphExecRef>> g_graphs;
int cudaGetDevice_or(int dflt) {
  int d = dflt;
  return cudaGetDevice(&d) == cudaSuccess ? d : dflt;
}
GraphExecRef graph_cache_get(const GraphKey& k) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (auto& e : g_graphs)
    if (e.first == k) return e.second;
  return nullptr;
}
void graph_cache_put(const GraphKey& k, const GraphExecRef& ge) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  if (g_graphs.size() >= 4) g_graphs.erase(g_graphs.begin());
  g_graphs.push_back({k, ge});
}

// passes per iteration of the graph's pass loop (PLAS_PASS_UNROLL; round 1: 1 -> 122.1, 2 -> 120.2, 3 -> 119.6,
// 4 -> 120.0 ms at C2; round 2 with the lighter statistics node: 3 -> 105.2, 5 -> 104.8, 6 -> 104.6, 8 -> 104.9 ms,
// C3 / C4 unchanged)
int pass_unroll() {
  static std::atomic<int> v{0};
  if (!v) {
    const char* e = getenv("PLAS_PASS_UNROLL");
    v = e ? std::max(1, std::min(8, atoi(e))) : 6;
  }
  return v;
}

// K3 launch configuration (gather regime)
struct PassCfg {
  void* fn;
  int grid, block;
  unsigned smem;
};
template <bool PARITY>
PassCfg pass_cfg(int S) {
  return {pass_kernel_ptr<PARITY>(S), pass_grid_size(S), 256, 0u};
}

template <bool PARITY>
void* tile_kernel_ptr(int S) {
  if (S <= 16) return (void*)tile_pass_kernel<false, PARITY>;
  return (void*)tile_pass_kernel<true, PARITY>;
}

// largest tile block side for row stride S and its two-stage shared memory
int tile_beta_max(int S) {
  int b = 1;
  while (use_tile(b + 1, S)) b++;
  return b;
}
size_t tile_smem_bytes(int S) { return (size_t)(TILE_NST * tile_stage_bytes(tile_beta_max(S), S)); }

int tile_grid_size(int S) {
  static std::atomic<int> cached[65];
  const int key = S <= 64 ? S : 64;
  // the attribute is per kernel, so set it for this S on every sort
  const size_t smem = tile_smem_bytes(S);
  raise_smem_limit((const void*)tile_kernel_ptr<false>(S), smem);
  raise_smem_limit((const void*)tile_kernel_ptr<true>(S), smem);
  if (!cached[key]) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tile_kernel_ptr<false>(S), TILE_CTA_THREADS, smem);
    if (occ <= 0) occ = 1;
    cached[key] = std::min(num_sms() * occ, MAX_PARTS);
  }
  return cached[key];
}

// Capacity of the moved-cell list: every cell changes element at most once per pass.
long long list_capacity(long long n) { return n; }

int stats_grid_size() {
  static std::atomic<int> g{0};
  if (!g) {
    const char* e = getenv("PLAS_STATS_CTAS_PER_SM");
    // measured (C2 / C3 / C4): 1 -> 116.1 ms; 2 -> 115.1 ms / 1.655 s / 2.608 s;
    // 4 -> 115.8 ms / 1.661 s / 2.612 s; 8 -> 120.3 ms (fewer tickets and
    // table workers shorten the kernel's tail)
    const int per = e ? std::max(1, atoi(e)) : 2;
    g = std::min(num_sms() * per, MAX_PARTS);
  }
  return g;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int plas_abi_version(void) { return PLAS_ABI_VERSION; }
size_t plas_sizeof_sort_args(void) { return sizeof(plas_sort_args); }
size_t plas_sizeof_sort_result(void) { return sizeof(plas_sort_result); }

const char* plas_last_error(void) { return g_last_error.c_str(); }

int plas_num_levels(int64_t n, double radius_decay, double initial_radius) {
  int side = (int)llround(sqrt((double)n));
  if (side < 2 || !(radius_decay > 0.0 && radius_decay < 1.0)) return 0;
  double r = std::isnan(initial_radius) ? default_initial_radius(side) : initial_radius;
  int L = 0;
  while (r >= 1.0) {
    L++;
    r *= radius_decay;
  }
  return L;
}

size_t plas_sort_workspace_bytes(int64_t n, int dim, int num_levels, int64_t weights_len,
                                 int64_t trace_capacity, int rng_mode) {
  SortWs w;
  const int side = (int)llround(sqrt((double)n));
  const long long lc = list_capacity(n);
  return carve_sort(nullptr, n, dim, num_levels, weights_len, trace_capacity, rng_mode, side, lc, &w);
}

size_t plas_sort_workspace_bytes_sharded(int64_t n, int dim, int num_levels, int64_t weights_len,
                                         int64_t trace_capacity, int rng_mode, int world) {
  SortWs w;
  const int side = (int)llround(sqrt((double)n));
  const long long lc = list_capacity(n);
  return carve_sort(nullptr, n, dim, num_levels, weights_len, trace_capacity, rng_mode, side, lc, &w,
                    std::max(world, 1));
}

void plas_seed_key(uint64_t seed, uint64_t key[2]) { host::seed_key(seed, key); }

int plas_host_permutation(uint64_t seed, int64_t n, int64_t* out) {
  if (n < 0 || !out) return fail(PLAS_ERR_INVALID, "bad permutation args");
  host::NumpyPhilox r;
  r.seed(seed);
  r.permutation(n, out);
  return PLAS_OK;
}

int plas_sort(const plas_sort_args* a, plas_sort_result* res, void* wsp, size_t ws_bytes) {
  const auto ht0 = std::chrono::steady_clock::now();
  auto hms = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ht0).count(); };
  const bool htrace = getenv("PLAS_HOST_TRACE") && atoi(getenv("PLAS_HOST_TRACE"));
  if (!a || !res || !a->features || !res->perm) return fail(PLAS_ERR_INVALID, "null argument");
  const long long n = a->n;
  const int D = a->dim;
  const int side = (int)llround(sqrt((double)n));
  if (D < 1 || side < 2 || (long long)side * side != n || n >= (1LL << 31))
    return fail(PLAS_ERR_INVALID, "features must be (side^2, D) with side >= 2, D >= 1");
  if ((unsigned long long)n * (unsigned long long)row_stride(D) >= (1ULL << 32))
    return fail(PLAS_ERR_INVALID, "n * padded row width must be < 2^32 (32-bit row offsets in the pass kernels)");
  if (!(a->improvement_threshold > 0.0) || a->min_block_size < 2)
    return fail(PLAS_ERR_INVALID, "bad SortConfig");
  if (a->features_dtype != PLAS_F32 && a->features_dtype != PLAS_F64)
    return fail(PLAS_ERR_INVALID, "features dtype must be f32 or f64");
  const int mode = a->rng_mode;
  if (mode != PLAS_RNG_PARITY && mode != PLAS_RNG_DEVICE) return fail(PLAS_ERR_INVALID, "rng_mode");
  cudaStream_t st = (cudaStream_t)a->stream;

  Schedule sch;
  build_schedule(a, side, &sch);
  const int L = (int)sch.radii.size();
  const long long tcap = std::max<long long>(a->trace_capacity, 1);
  SortWs w;
  const int S = row_stride(D);
  const long long lcap = list_capacity(n);
  const int world = std::max(a->world, 1);
  if (world > 1 && (a->rank < 0 || a->rank >= world || !a->exchange || !a->xchg_send || !a->xchg_recv ||
                    !a->xchg_part || !a->xchg_part_all))
    return fail(PLAS_ERR_INVALID, "sharded sort needs rank < world, an exchange callback and its buffers");
  size_t need = carve_sort(nullptr, n, D, L, (long long)sch.weights.size(), tcap, mode, side, lcap, &w, world);
  if (!wsp || ws_bytes < need)
    return fail(PLAS_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  carve_sort((char*)wsp, n, D, L, (long long)sch.weights.size(), tcap, mode, side, lcap, &w, world);

  // ---- upload schedule + controller
  if (L > 0) {
    CK(cudaMemcpyAsync(w.radii, sch.radii.data(), sizeof(double) * L, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.betas, sch.betas.data(), sizeof(int) * L, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.hs, sch.hs.data(), sizeof(int) * L, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.woff, sch.woff.data(), sizeof(long long) * L, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.weights, sch.weights.data(), sizeof(double) * sch.weights.size(),
                       cudaMemcpyHostToDevice, st));
  }
  Ctrl hc;
  memset(&hc, 0, sizeof(hc));
  hc.num_levels = L;
  hc.side = side;
  hc.S = row_stride(D);
  hc.trace_cap = tcap;
  hc.rng_mode = mode;
  hc.threshold = a->improvement_threshold;
  hc.min_block = a->min_block_size;
  uint64_t key[2];
  host::seed_key(a->seed, key);
  hc.key0 = key[0];
  hc.key1 = key[1];
  // PLAS_GTRACE=1: per-pass globaltimer marks of K3 and the statistics (diagnostics)
  unsigned long long* gtr = nullptr;
  if (getenv("PLAS_GTRACE") && atoi(getenv("PLAS_GTRACE"))) {
    if (cudaMalloc(&gtr, sizeof(unsigned long long) * 6 * (size_t)(tcap + 8)) == cudaSuccess) {
      cudaMemsetAsync(gtr, 0, sizeof(unsigned long long) * 6 * (size_t)(tcap + 8), st);
      hc.gtrace = gtr;
    } else {
      gtr = nullptr;
      cudaGetLastError();
    }
  }
  hc.fft_min_h = fft_min_h(w.fft_L, S);
  hc.fft_L = w.fft_L;
  hc.tile_blur_hmax = tile_blur_hmax(S);
  hc.rank = world > 1 ? a->rank : 0;
  hc.world = world;
  hc.banded = 0;  // whole grid (set per level by set_level_shard_kernel when world > 1)
  // lazy element-index reads in the pass kernels once the index array outgrows
  // what stays in L2 across a pass (PLAS_LAZY_IDX=0/1 overrides)
  hc.lazy_idx = getenv("PLAS_LAZY_IDX") ? (atoi(getenv("PLAS_LAZY_IDX")) != 0) : (n * 4 > (32LL << 20) ? 1 : 0);
  // PARITY on one GPU: strike decisions on the reference's own (NumPy-order)
  // grid_distance, so the trace and every pass count are bit-identical
  // (PLAS_NP_STATS=0: the fixed-point running sum instead, as the sharded path uses)
  hc.exact_stats = (mode == PLAS_RNG_PARITY && world == 1 &&
                    !(getenv("PLAS_NP_STATS") && atoi(getenv("PLAS_NP_STATS")) == 0)) ? 1 : 0;
  hc.own_lo = hc.band_lo = 0;
  hc.own_hi = hc.band_hi = side;
  hc.pdraw = nullptr;
  hc.prec = nullptr;
  hc.pdraw_level = -1;
  CK(cudaMemcpyAsync(w.ctrl, &hc, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
  NpTree npt;
  if (hc.exact_stats) {  // the n-cell pairwise tree of NumPy's mean (depends on n only)
    np_tree_make(&npt, n);
    const size_t nl = npt.leaf_start.size(), ni = npt.left.size();
    if ((long long)nl > n / 64 + 4 || npt.hoff.size() > 72) return fail(PLAS_ERR_INVALID, "numpy tree sizing");
    CK(cudaMemcpyAsync(w.np_lstart, npt.leaf_start.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.np_llen, npt.leaf_len.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, st));
    if (ni) {
      CK(cudaMemcpyAsync(w.np_left, npt.left.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(w.np_right, npt.right.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(w.np_order, npt.order.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(w.np_hoff, npt.hoff.data(), sizeof(int) * npt.hoff.size(), cudaMemcpyHostToDevice, st));
  }
  // NumPy's grid_distance of the current grid vs target into np_out
  auto np_distance = [&]() {
    np_cell_sort_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(w.feat, w.target, n, D, S, w.np_v);
    const int nl = (int)npt.leaf_start.size();
    np_leaf_kernel<<<std::max(1, (nl + 255) / 256), 256, 0, st>>>(w.np_v, w.np_lstart, w.np_llen, nl, w.np_vals);
    np_tree_kernel<<<1, 1024, 0, st>>>(w.np_vals, w.np_left, w.np_right, w.np_order, w.np_hoff,
                                       (int)npt.hoff.size() - 1, nl, npt.root, n, w.np_out);
  };
  CK(cudaMemsetAsync(w.flags, 0, sizeof(int) * 8, st));
  CK(cudaMemsetAsync(w.spart + MAX_PARTS, 0, 2 * sizeof(double), st));  // pass statistic's 128-bit accumulator
  // zero halos of the padded blur buffers, pad channels, fallback counters
  CK(cudaMemsetAsync(w.feat_alloc, 0, sizeof(float) * w.feat_alloc_floats, st));
  CK(cudaMemsetAsync(w.tmp_alloc, 0, sizeof(float) * w.tmp_alloc_floats, st));
  CK(cudaMemsetAsync(w.target, 0, sizeof(float) * n * S, st));
  CK(cudaMemsetAsync(w.fb0, 0, sizeof(int) * FB_HEADER, st));
  CK(cudaMemsetAsync(w.fb1, 0, sizeof(int) * FB_HEADER, st));
  std::vector<std::vector<double2>> htw(w.fft_count);
  for (int i = 0; i < w.fft_count; i++) {
    fft_twiddles(w.fft_codes[i], &htw[i]);
    CK(cudaMemcpyAsync(w.fft_tws[i], htw[i].data(), sizeof(double2) * htw[i].size(), cudaMemcpyHostToDevice, st));
  }

  // ---- initial permutation (plas.py:241)
  host::NumpyPhilox rng;
  rng.seed(a->seed);
  std::vector<int> hperm;
  if (mode == PLAS_RNG_PARITY) {
    hperm.resize(n);
    rng.permutation(n, hperm.data());  // also advances the stream like draw #1
  }
  if (a->initial_perm) {
    perm_i64_to_i32_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>((const long long*)a->initial_perm,
                                                                 w.idx, n);
    CKL();
  } else if (mode == PLAS_RNG_PARITY) {
    CK(cudaMemcpyAsync(w.idx, hperm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  } else {
    init_perm_device_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(w.idx, n, key[0], key[1]);
    CKL();
  }

  cudaEvent_t ev0, ev1;
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  CK(cudaEventRecord(ev0, st));
  if (htrace) fprintf(stderr, "host: ev0 at %.3f ms\n", hms());
  const int gi = grid_for(n * S, 256, 8);
  if (a->features_dtype == PLAS_F32)
    gather_init_kernel<float><<<gi, 256, 0, st>>>((const float*)a->features, w.idx, w.feat, n, D, S,
                                                  w.flags);
  else
    gather_init_kernel<double><<<gi, 256, 0, st>>>((const double*)a->features, w.idx, w.feat, n, D,
                                                   S, w.flags);
  CKL();
  if (world > 1) {
    if (a->features_dtype == PLAS_F32)
      orig32_kernel<float><<<gi, 256, 0, st>>>((const float*)a->features, w.orig32, n, D, S);
    else
      orig32_kernel<double><<<gi, 256, 0, st>>>((const double*)a->features, w.orig32, n, D, S);
    CKL();
  }
  int hflags = 0;
  CK(cudaMemcpyAsync(&hflags, w.flags, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hflags) {
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return fail(PLAS_ERR_NONFINITE, "features must be finite");
  }

  // ---- launch configuration
  Launch lc;
  lc.S = S;
  lc.D = D;
  lc.side = side;
  lc.n = n;
  lc.blur_grid = grid_for((long long)side * S * ((side + BPAD_R - 1) / BPAD_R), 256, 8);
  lc.den_grid = std::min(side, num_sms() * 8);  // border_weight32_kernel: rows per CTA
  lc.fb_grid = num_sms() * 2;
  lc.pg = make_pad_geom(side, side, D, S, w.pad);
  lc.rows_grid = grid_for(side, 128, 1);
  lc.dist_grid = grid_for(n, RED_THREADS, 4);
  lc.vad_grid = grid_for(n * D, RED_THREADS, 4);
  lc.pass_grid = pass_grid_size(S);
  lc.tile_grid = tile_grid_size(S);
  lc.lvl = BlurLevelRef{w.ctrl, w.hs, w.weights, w.woff, 0, nullptr};
  // FFT plans (one per length) and the per-level blur mode: plan index for
  // the FFT tier, FFT_PLANS for the tile tier, FFT_PLANS + 1 for the direct fold
  const int NPL = w.fft_count;
  FftPlan fplans[4];
  void* fft0s[4] = {nullptr, nullptr, nullptr, nullptr};
  void* fft1s[4] = {nullptr, nullptr, nullptr, nullptr};
  int fft_nthreads[4] = {32, 32, 32, 32};
  size_t fft_smems[4] = {0, 0, 0, 0};
  for (int i = 0; i < NPL; i++) {
    const int lcode = w.fft_codes[i];
    fplans[i] = FftPlan{lcode, fft_len(lcode), w.fft_tws[i], w.fft_spec, fft_error_constant(lcode)};
    fft0s[i] = fft_kernel_ptr<0, 0>(lcode);
    fft1s[i] = fft_kernel_ptr<1, 1>(lcode);
    fft_nthreads[i] = fft_threads(fft_len(lcode));
    fft_smems[i] = fft_smem_bytes(lcode);
    CK(raise_smem_limit((const void*)fft0s[i], fft_smems[i]));
    CK(raise_smem_limit((const void*)fft1s[i], fft_smems[i]));
  }
  const int fft_grid = side * ((D + 1) / 2);  // one CTA per line pair
  std::vector<int> hmode(std::max(L, 1));
  // the zero-padded buffers are read at +-h around every output (direct tier,
  // fallback folds): h <= pad - BPAD_R, the reference rule's top half-width
  // plus one; larger start radii are refused (plas.py SortPlan does the same)
  const int hpad = w.pad - std::max(BLUR_R, BPAD_R);
  for (int lv = 0; lv < L; lv++) {
    const int h = sch.hs[lv];
    int m = level_uses_tile_blur(h, side, hc.fft_min_h, hc.fft_L, hc.tile_blur_hmax) ? NPL : NPL + 1;
    if (m == NPL + 1 && h <= PAD_SMALL_HMAX && pad_small_enabled()) m = NPL + 1 + h;  // direct, compile-time h
    if (NPL && level_uses_fft(h, side, hc.fft_min_h, hc.fft_L)) {
      const int lcode = fft_choose_code(side, h);
      int f = -1;
      for (int i = NPL - 1; i >= 0; i--)
        if (w.fft_codes[i] == lcode) f = i;
      // otherwise the longest planned length, if it holds the line and h
      // without wrapping (n + h <= L), else the padded direct tier
      if (f < 0 && side + (long long)h <= fft_len(w.fft_codes[NPL - 1]) && side <= fft_out_max(w.fft_codes[NPL - 1]))
        f = NPL - 1;
      if (f >= 0) m = f;
    }
    if (h > hpad) {  // (the FFT tier's overflow list is folded from the padded buffers too)
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
      return fail(PLAS_ERR_INVALID, "start radius too large for this grid (ceil(r) must be <= ceil(side/2 - 1) + 1)");
    }
    hmode[lv] = m;
  }
  CK(cudaMemcpyAsync(w.lvl_mode, hmode.data(), sizeof(int) * L, cudaMemcpyHostToDevice, st));
  if (NPL) CK(cudaMemcpyAsync(w.fft_plans, fplans, sizeof(FftPlan) * NPL, cudaMemcpyHostToDevice, st));
  lc.tb_grid = dim3((side + TB_T - 1) / TB_T, (side + TB_T - 1) / TB_T);
  if (hc.tile_blur_hmax > 0)
    CK(raise_smem_limit((const void*)blur_tile_kernel, tile_blur_smem_bytes(hc.tile_blur_hmax)));
  lc.sched = Sched{w.radii, w.betas, w.hs, w.level_counts, w.trace};

  // PARITY: the reference's vad float (NumPy order over the pooled
  // differences, np_sum.cuh); the tree over M = 2 side (side - 1) D values is
  // built once per size
  NpTree vtree;
  const bool np_vad = mode == PLAS_RNG_PARITY && !getenv("PLAS_NP_VAD_OFF");
  if (np_vad) {
    np_tree_make(&vtree, 2LL * side * (side - 1) * D);
    const size_t nl = vtree.leaf_start.size(), ni = vtree.left.size();
    if (nl > w.vad_cap || vtree.hoff.size() > 72) return fail(PLAS_ERR_INVALID, "vad tree sizing");
    CK(cudaMemcpyAsync(w.vad_lstart, vtree.leaf_start.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.vad_llen, vtree.leaf_len.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, st));
    if (ni) {
      CK(cudaMemcpyAsync(w.vad_left, vtree.left.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(w.vad_right, vtree.right.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(w.vad_order, vtree.order.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(w.vad_hoff, vtree.hoff.data(), sizeof(int) * vtree.hoff.size(), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // the host tree vectors live on this frame only
  }
  auto vad_launch = [&](double* out) -> int {
    if (np_vad) {
      const VadElems<float> el{w.feat, (unsigned)side, (unsigned)side, (unsigned)D, (unsigned)S,
                        (unsigned long long)(side - 1) * side * D};
      const int nl = (int)vtree.leaf_start.size(), lg = std::max(1, (nl + 255) / 256);
      const long long M = 2LL * side * (side - 1) * D;
      np_leaf_vad_kernel<0><<<lg, 256, 0, st>>>(el, nullptr, w.vad_lstart, w.vad_llen, nl, w.vad_vals);
      np_tree_kernel<<<1, 1024, 0, st>>>(w.vad_vals, w.vad_left, w.vad_right, w.vad_order, w.vad_hoff,
                                         (int)vtree.hoff.size() - 1, nl, vtree.root, M, w.vad_out);
      np_leaf_vad_kernel<1><<<lg, 256, 0, st>>>(el, w.vad_out, w.vad_lstart, w.vad_llen, nl, w.vad_vals);
      np_tree_kernel<<<1, 1024, 0, st>>>(w.vad_vals, w.vad_left, w.vad_right, w.vad_order, w.vad_hoff,
                                         (int)vtree.hoff.size() - 1, nl, vtree.root, M, w.vad_out + 2);
      CK(cudaMemcpyAsync(out, w.vad_out + 3, sizeof(double), cudaMemcpyDeviceToDevice, st));
      CKL();
      return 0;
    }
    vad_kernel<float><<<lc.vad_grid, RED_THREADS, 0, st>>>(w.feat, side, side, D, S, nullptr, w.partials);
    mean_finalize_kernel<<<1, RED_THREADS, 0, st>>>(w.partials, lc.vad_grid,
                                                    2.0 * side * (side - 1) * (double)D, w.scalars);
    vad_kernel<float><<<lc.vad_grid, RED_THREADS, 0, st>>>(w.feat, side, side, D, S, w.scalars, w.partials);
    mean_finalize_kernel<<<1, RED_THREADS, 0, st>>>(w.partials, lc.vad_grid,
                                                    2.0 * side * (side - 1) * (double)D, out);
    CKL();
    return 0;
  };
  if (int e = vad_launch(w.scalars + 1)) return e;

  const int sgrid = stats_grid_size();
  int* counters = w.flags + 2;  // [0] moved cells, [1] exact decisions, [2] moved-list length
  MoveOut ml{w.list, counters + 2, reinterpret_cast<unsigned long long*>(w.spart + MAX_PARTS)};
  int* done = w.flags + 6;      // last-CTA ticket of the statistic kernels
  if (htrace) fprintf(stderr, "host: graph/loop start at %.3f ms\n", hms());
  long long banded_levels = 0;
  if (mode == PLAS_RNG_DEVICE && !a->profile && world == 1) {
    // ------------------------------------------------------------ graph
    // outer WHILE (levels): level_begin, border weight, blur axis 0, blur axis 1,
    //   level statistics, inner WHILE (passes): IF(tile){tile}ELSE{gather},
    //   pass statistics (+controller); level_end.
    // the graph is a function of the workspace layout (every node argument is
    // a workspace pointer or a shape constant), so an instantiated graph is
    // reused by later sorts of the same shape on the same workspace
    const GraphKey gkey{wsp, ws_bytes, n, D, L, (long long)sch.weights.size(), tcap, mode, cudaGetDevice_or(-1)};
    GraphExecRef ger = graph_cache_get(gkey);
    if (!ger) {
    cudaGraphExec_t ge = nullptr;
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle outer_h, tile_h;
    CK(cudaGraphConditionalHandleCreate(&outer_h, g, L > 0 ? 1 : 0, cudaGraphCondAssignDefault));
    cudaGraphNode_t outer_node;
    cudaGraph_t obody;
    CK(add_while(&outer_node, g, nullptr, 0, outer_h, &obody));
    CK(cudaGraphConditionalHandleCreate(&tile_h, obody, 0, 0));
    cudaGraphConditionalHandle blur_h;
    CK(cudaGraphConditionalHandleCreate(&blur_h, obody, 0, 0));
    cudaGraphNode_t nd[8];
    // level set-up in one node: level_begin + pass draw records + row weights
    // (+ FFT spectrum); the sort's grid is square, so the column weights B(x)
    // are the row weights A(x): one fold serves both axes of the certified
    // product (border_weight32)
    {
      const int ndraw = PDRAW_MAX * 16 / 256, nrow = std::max(1, (side + 255) / 256);
      const int nspec = w.fft_L ? std::max(1, w.fft_L / 256) : 0;
      CK(add_kernel(&nd[1], obody, nullptr, 0, level_prep_kernel, dim3(ndraw + nrow + nspec), dim3(256), w.ctrl,
                    lc.sched, (unsigned long long)blur_h, (unsigned long long)tile_h, w.pdraw, w.prec, w.rowweight,
                    lc.lvl, (const int*)w.lvl_mode, (const FftPlan*)w.fft_plans, NPL, ndraw, nrow));
    }
    // the certified border weight (den32) is needed by the blur's axis-1 pass
    // only: each blur body runs it beside the axis-0 pass (a node of its own
    // body, joined before axis 1), off the level's critical path
    auto add_border = [&](cudaGraphNode_t* bw, cudaGraph_t body) {
      return add_kernel(bw, body, nullptr, 0, border_weight32_kernel, dim3(lc.den_grid), dim3(256),
                        (const double*)w.rowweight, (const double*)w.rowweight, w.den32, side, side, lc.lvl);
    };
    nd[2] = nd[1];
    // SWITCH (blur mode of the level) { FFT at length 0 | ... | FFT at length
    // NPL - 1 | one tile kernel | direct fold + fallbacks }
    cudaGraphNode_t blur_if;
    cudaGraph_t bbody[FFT_PLANS + 2 + PAD_SMALL_HMAX];
    {
      cudaGraphNodeParams p{};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = blur_h;
      p.conditional.type = cudaGraphCondTypeSwitch;
      p.conditional.size = NPL + 2 + PAD_SMALL_HMAX;
      CK(cudaGraphAddNode(&blur_if, obody, &nd[2], 1, &p));
      for (int i = 0; i < NPL + 2 + PAD_SMALL_HMAX; i++) bbody[i] = p.conditional.phGraph_out[i];
    }
    for (int i = 0; i < NPL; i++) {
      cudaGraphNode_t fn[5];
      const float* in0 = w.feat;
      float* out0 = w.tmp;
      const float* dnull = nullptr;
      int* fb0 = w.fb0;
      int* fb1 = w.fb1;
      int cap = w.fb_cap;
      PadGeom pg = lc.pg;
      BlurLevelRef lv = lc.lvl;
      FftPlan pl = fplans[i];
      void* a0[] = {&in0, &out0, &pg, &lv, &pl, &dnull, &fb0, &cap, &fb1};
      cudaKernelNodeParams kp{};
      kp.func = fft0s[i];
      kp.gridDim = dim3(fft_grid);
      kp.blockDim = dim3(fft_nthreads[i]);
      kp.sharedMemBytes = (unsigned)fft_smems[i];
      kp.kernelParams = a0;
      CK(cudaGraphAddKernelNode(&fn[1], bbody[i], nullptr, 0, &kp));
      CK(add_kernel(&fn[2], bbody[i], &fn[1], 1, blur_pad_fallback_kernel<0, 0>, dim3(lc.fb_grid), dim3(256),
                    (const float*)w.feat, w.tmp, lc.pg, lc.lvl, (const float*)nullptr, w.fb0, w.fb_cap));
      const float* in1 = w.tmp;
      float* out1 = w.target;
      const float* den = w.den32;
      void* a1[] = {&in1, &out1, &pg, &lv, &pl, &den, &fb1, &cap, &fb0};
      kp.func = fft1s[i];
      kp.kernelParams = a1;
      CK(add_border(&fn[0], bbody[i]));
      {
        cudaGraphNode_t deps[2] = {fn[2], fn[0]};
        CK(cudaGraphAddKernelNode(&fn[3], bbody[i], deps, 2, &kp));
      }
      CK(add_kernel(&fn[4], bbody[i], &fn[3], 1, blur_pad_fallback_kernel<1, 1>, dim3(lc.fb_grid), dim3(256),
                    (const float*)w.tmp, w.target, lc.pg, lc.lvl, (const float*)w.den32, w.fb1, w.fb_cap));
    }
    {
      const float* fin = w.feat;
      float* tout = w.target;
      PadGeom pg = lc.pg;
      BlurLevelRef lv = lc.lvl;
      const float* den = w.den32;
      void* ta[] = {&fin, &tout, &pg, &lv, &den};
      cudaKernelNodeParams kp{};
      kp.func = (void*)blur_tile_kernel;
      kp.gridDim = lc.tb_grid;
      kp.blockDim = dim3(TB_THREADS);
      kp.sharedMemBytes = (unsigned)tile_blur_smem_bytes(std::max(hc.tile_blur_hmax, 1));
      kp.kernelParams = ta;
      cudaGraphNode_t tn, bw;
      CK(add_border(&bw, bbody[NPL]));
      CK(cudaGraphAddKernelNode(&tn, bbody[NPL], &bw, 1, &kp));
    }
    // direct fold: the runtime-h kernels (case NPL + 1) and the compile-time-h
    // kernels of h = 1 .. PAD_SMALL_HMAX (case NPL + 1 + h)
    for (int hb = 0; hb <= PAD_SMALL_HMAX; hb++) {
      cudaGraph_t db = bbody[NPL + 1 + hb];
      cudaGraphNode_t bn[4];
      const PadFn p0 = hb ? pad_fn(0, hb) : (PadFn)blur_pad_kernel<0, 0>;
      const PadFn p1 = hb ? pad_fn(1, hb) : (PadFn)blur_pad_kernel<1, 1>;
      CK(add_kernel(&bn[0], db, nullptr, 0, p0, dim3(lc.blur_grid), dim3(256),
                    (const float*)w.feat, w.tmp, lc.pg, lc.lvl, (const float*)nullptr, w.fb0, w.fb_cap, w.fb1));
      CK(add_kernel(&bn[1], db, &bn[0], 1, blur_pad_fallback_kernel<0, 0>, dim3(lc.fb_grid), dim3(256),
                    (const float*)w.feat, w.tmp, lc.pg, lc.lvl, (const float*)nullptr, w.fb0, w.fb_cap));
      cudaGraphNode_t bw;
      CK(add_border(&bw, db));
      const cudaGraphNode_t d2[2] = {bn[1], bw};
      CK(add_kernel(&bn[2], db, d2, 2, p1, dim3(lc.blur_grid), dim3(256),
                    (const float*)w.tmp, w.target, lc.pg, lc.lvl, (const float*)w.den32, w.fb1, w.fb_cap, w.fb0));
      CK(add_kernel(&bn[3], db, &bn[2], 1, blur_pad_fallback_kernel<1, 1>, dim3(lc.fb_grid), dim3(256),
                    (const float*)w.tmp, w.target, lc.pg, lc.lvl, (const float*)w.den32, w.fb1, w.fb_cap));
    }
    nd[4] = blur_if;
    // IF (tile regime this level) { level statistics, WHILE { tile K3, pass
    // statistics } } ELSE { the same with the gather K3 }: the regime is fixed
    // per level (beta), so the pass loop carries no conditional of its own
    cudaGraphNode_t reg_if;
    cudaGraph_t rbody[2];
    {
      cudaGraphNodeParams p{};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = tile_h;
      p.conditional.type = cudaGraphCondTypeIf;
      p.conditional.size = 2;
      CK(cudaGraphAddNode(&reg_if, obody, &nd[4], 1, &p));
      rbody[0] = p.conditional.phGraph_out[0];  // tile_h != 0: tile regime
      rbody[1] = p.conditional.phGraph_out[1];
    }
    for (int rg = 0; rg < 2; rg++) {
      cudaGraph_t rb = rbody[rg];
      cudaGraphConditionalHandle loop_h;
      CK(cudaGraphConditionalHandleCreate(&loop_h, rb, 0, 0));
      cudaGraphNode_t ls, wl, kn, sn;
      CK(add_kernel(&ls, rb, nullptr, 0, level_stats_kernel, dim3(lc.dist_grid), dim3(RED_THREADS),
                    w.ctrl, lc.sched, (const float*)w.feat, (const float*)w.target, w.dcache, n, D, S,
                    w.spart + MAX_PARTS, done, (unsigned long long)loop_h, (unsigned long long)outer_h, w.sel,
                    w.sel_stride, (double*)nullptr));
      cudaGraph_t lb;
      CK(add_while(&wl, rb, &ls, 1, loop_h, &lb));
      float* feat = w.feat;
      int* idx = w.idx;
      const float* target = w.target;
      const Ctrl* ctrl = w.ctrl;
      const int* sel = w.sel;  // DEVICE-mode tables (gen_class_tables)
      long long sstride = w.sel_stride;
      int Dv = D, Sv = S;
      void* args[] = {&feat, &idx, &target, &Dv, &Sv, &ctrl, &sel, &sstride, &ml, &counters};
      cudaKernelNodeParams kp{};
      if (rg == 0) {
        kp.func = tile_kernel_ptr<false>(S);
        kp.gridDim = dim3(lc.tile_grid);
        kp.blockDim = dim3(TILE_CTA_THREADS);
        kp.sharedMemBytes = (unsigned)tile_smem_bytes(S);
      } else {
        const PassCfg pc = pass_cfg<false>(S);
        kp.func = pc.fn;
        kp.gridDim = dim3(pc.grid);
        kp.blockDim = dim3(pc.block);
        kp.sharedMemBytes = pc.smem;
      }
      kp.kernelParams = args;
      // the loop body holds `unroll` passes; a pass slot after the level ended
      // returns at once (both kernels test Ctrl.level_done), so one loop
      // iteration's overhead is shared by `unroll` passes
      cudaGraphNode_t prev = nullptr;
      for (int u = 0; u < pass_unroll(); u++) {
        CK(cudaGraphAddKernelNode(&kn, lb, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
        CK(add_kernel(&sn, lb, &kn, 1, S > 16 ? pass_stats_kernel<true> : pass_stats_kernel<false>, dim3(sgrid), dim3(RED_THREADS), w.ctrl, lc.sched,
                      (const float*)w.feat, (const float*)w.target, w.dcache, D, S, (const int*)w.list,
                      counters, w.spart + MAX_PARTS, done, n, (unsigned long long)loop_h, (unsigned long long)outer_h,
                      (double*)nullptr, w.sel, w.sel_stride));  // + next pass's tables (+ level end)
        prev = sn;
      }
    }
    if (htrace) fprintf(stderr, "host: graph built at %.3f ms\n", hms());
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    ger = std::make_shared<GraphExecHolder>();
    ger->ge = ge;
    graph_cache_put(gkey, ger);
    if (htrace) fprintf(stderr, "host: instantiated at %.3f ms\n", hms());
    }
    CK(cudaGraphLaunch(ger->ge, st));
    if (htrace) fprintf(stderr, "host: launched at %.3f ms\n", hms());
    CK(cudaStreamSynchronize(st));
  } else {
    // ------------------------------------------------------------ host-stepped loop
    // PARITY (host draws) or DEVICE with profiling (device draws, events per launch)
    const bool parity = mode == PLAS_RNG_PARITY;
    plas_sort_profile* prof = (plas_sort_profile*)a->profile;
    std::vector<cudaEvent_t> evs;
    struct Pending { int kind; int e0; };
    std::vector<Pending> pend;
    auto timed = [&](int kind, auto&& launch) {
      if (!prof) {
        launch();
        return;
      }
      while (evs.size() < (size_t)(2 * pend.size() + 2)) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        evs.push_back(e);
      }
      int e0 = (int)(2 * pend.size());
      cudaEventRecord(evs[e0], st);
      launch();
      cudaEventRecord(evs[e0 + 1], st);
      pend.push_back({kind, e0});
    };
    // PLAS_LEVEL_TRACE=1 (with a profile): one stderr line per level, diagnostics only
    const bool level_trace = prof && getenv("PLAS_LEVEL_TRACE") && atoi(getenv("PLAS_LEVEL_TRACE"));
    double lvl_ms[7] = {0, 0, 0, 0, 0, 0, 0};
    int fbstat[6] = {0, 0, 0, 0, 0, 0};
    int lvl_n[7] = {0, 0, 0, 0, 0, 0, 0};
    auto flush_profile = [&]() {
      if (!prof) return;
      for (auto& pe : pend) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, evs[pe.e0], evs[pe.e0 + 1]);
        lvl_ms[pe.kind] += ms;
        lvl_n[pe.kind] += 1;
        double* slot = &prof->ms_pass + 2 * pe.kind;  // {ms, n} pairs in declaration order
        slot[0] += ms;
        reinterpret_cast<int64_t*>(slot)[1] += 1;
      }
      pend.clear();
    };
    enum { K_PASS = 0, K_BLUR0, K_BLUR1, K_BORDER, K_DIST, K_CTRL, K_SELECT };
    int* pinned = nullptr;
    const long long b0sq = parity ? (long long)side * side : 0;
    CK(cudaMallocHost(&pinned, sizeof(int) * (2 * b0sq + 4)));
    int* hflag = pinned + 2 * b0sq;
    auto cleanup = [&]() {
      cudaFreeHost(pinned);
      for (auto e : evs) cudaEventDestroy(e);
    };
    int pp = 0;
    const PassCfg kpc = parity ? pass_cfg<true>(S) : pass_cfg<false>(S);
    banded_levels = 0;
    void* tfn = parity ? tile_kernel_ptr<true>(S) : tile_kernel_ptr<false>(S);
    for (int lv = 0; lv < L; lv++) {
      const int beta = sch.betas[lv];
      const long long bsq = (long long)beta * beta;
      timed(K_CTRL, [&] {
        level_begin_kernel<<<1, 32, 0, st>>>(w.ctrl, lc.sched, 0ull, 0ull, 0ull);
        if (!parity) pass_draws_kernel<<<PDRAW_MAX * 16 / 256, 256, 0, st>>>(w.ctrl, w.pdraw, w.prec);
      });
      const int mode = hmode[lv];
      const bool use_fft = mode < NPL;
      // ---- sharding of this level (world > 1).  Banded
      // (beta * world <= side): rank r owns rows [Y_r, Y_r+1), Y_r = side r /
      // world, takes the pass's block rows starting there and needs the target
      // on [Y_r, Y_r+1 + beta); otherwise (top levels) every rank holds the
      // whole target and the groups are split evenly.
      PadGeom pgl = lc.pg;  // this rank's output rows [r0, r1) / FFT columns [c0, c1)
      bool fft_split = false;
      std::vector<int> blo(world), bhi(world), bcs(world + 1);
      if (world > 1) {
        const bool banded = (long long)beta * world <= side;
        banded_levels += banded ? 1 : 0;
        for (int q = 0; q <= world; q++) bcs[q] = (int)((long long)side * q / world);
        for (int q = 0; q < world; q++) {
          blo[q] = banded ? bcs[q] : 0;
          bhi[q] = banded ? std::min(side, bcs[q + 1] + beta) : side;
        }
        const int r = a->rank;
        set_level_shard_kernel<<<1, 32, 0, st>>>(w.ctrl, banded ? 1 : 0, bcs[r], bcs[r + 1], blo[r], bhi[r]);
        pgl.r0 = blo[r];
        pgl.r1 = bhi[r];
        fft_split = banded && use_fft;
        if (fft_split) {
          std::vector<int> hb(3 * world + 1);
          for (int q = 0; q < world; q++) hb[q] = blo[q], hb[world + q] = bhi[q];
          for (int q = 0; q <= world; q++) hb[2 * world + q] = bcs[q];
          CK(cudaMemcpyAsync(w.bands, hb.data(), sizeof(int) * hb.size(), cudaMemcpyHostToDevice, st));
          CK(cudaStreamSynchronize(st));  // hb is pageable and local
        }
      }
      timed(K_BORDER, [&] {
        border_rows_kernel<<<lc.rows_grid, 128, 0, st>>>(w.rowweight, side, lc.lvl);
        border_weight32_kernel<<<lc.den_grid, 256, 0, st>>>(w.rowweight, w.rowweight, w.den32, side, side, lc.lvl);
      });
      const int cpairs = (D + 1) / 2;
      if (use_fft) {
        timed(K_BLUR0, [&] {
          fft_spectrum_kernel<<<std::max(1, fplans[mode].L / 128), 128, 0, st>>>(lc.lvl, fplans[mode]);
          // axis 0: every column (one GPU, replicated levels) or this rank's
          // columns [c0, c1) on every row (banded levels, exchanged below)
          PadGeom pg0 = lc.pg;
          if (fft_split) {
            pg0.c0 = bcs[a->rank];
            pg0.c1 = bcs[a->rank + 1];
          }
          {
            const float* in0 = w.feat;
            float* out0 = w.tmp;
            const float* dnull = nullptr;
            BlurLevelRef lv = lc.lvl;
            FftPlan pl = fplans[mode];
            int cap = w.fb_cap;
            void* a0[] = {&in0, &out0, &pg0, &lv, &pl, &dnull, &w.fb0, &cap, &w.fb1};
            cudaLaunchKernel(fft0s[mode], dim3((pg0.c1 - pg0.c0) * cpairs), dim3(fft_nthreads[mode]), a0,
                             fft_smems[mode], st);
          }
          blur_pad_fallback_kernel<0, 0><<<lc.fb_grid, 256, 0, st>>>(w.feat, w.tmp, pg0, lc.lvl, nullptr, w.fb0,
                                                                     w.fb_cap);
        });
        if (fft_split) {
          // every rank's band rows of this rank's columns out, this rank's band
          // of every other rank's columns in (one all-to-all)
          const int r = a->rank;
          const long long WSP = (long long)(side + 2 * w.pad) * S;
          const int* dlo = w.bands;
          const int* dhi = w.bands + world;
          const int* dcs = w.bands + 2 * world;
          band_pack_kernel<<<num_sms() * 4, 256, 0, st>>>(w.tmp, w.xsend, dlo, dhi, world, bcs[r], bcs[r + 1], WSP,
                                                           S);
          CKL();
          std::vector<int64_t> sizes(2 * world);
          for (int q = 0; q < world; q++) {
            sizes[q] = (int64_t)(bhi[q] - blo[q]) * (bcs[r + 1] - bcs[r]) * S * 4;
            sizes[world + q] = (int64_t)(bhi[r] - blo[r]) * (bcs[q + 1] - bcs[q]) * S * 4;
          }
          const int xr = a->exchange(a->exchange_ctx, PLAS_XCHG_ALLTOALL, (int64_t)((char*)w.xsend - (char*)wsp),
                                     (int64_t)((char*)w.xrecv - (char*)wsp), sizes.data());
          if (xr < 0) {
            cleanup();
            return fail(PLAS_ERR_CUDA, "exchange callback failed (band all-to-all)");
          }
          band_unpack_kernel<<<num_sms() * 4, 256, 0, st>>>(w.tmp, w.xrecv, blo[r], bhi[r], dcs, world, r, WSP, S);
          CKL();
        }
        if (level_trace) {
          int h2[4];
          cudaMemcpyAsync(h2, w.fb0, sizeof(int) * 4, cudaMemcpyDeviceToHost, st);
          cudaStreamSynchronize(st);
          fbstat[0] = h2[0];
          fbstat[1] = h2[2];
          fbstat[4] = h2[3];
          cudaMemsetAsync(w.fb0 + 2, 0, sizeof(int) * 2, st);
        }
        timed(K_BLUR1, [&] {
          {
            const float* in1 = w.tmp;
            float* out1 = w.target;
            const float* den = w.den32;
            PadGeom pg = pgl;
            BlurLevelRef lv = lc.lvl;
            FftPlan pl = fplans[mode];
            int cap = w.fb_cap;
            void* a1[] = {&in1, &out1, &pg, &lv, &pl, &den, &w.fb1, &cap, &w.fb0};
            cudaLaunchKernel(fft1s[mode], dim3((pgl.r1 - pgl.r0) * cpairs), dim3(fft_nthreads[mode]), a1,
                             fft_smems[mode], st);
          }
          blur_pad_fallback_kernel<1, 1><<<lc.fb_grid, 256, 0, st>>>(w.tmp, w.target, pgl, lc.lvl, w.den32, w.fb1,
                                                                     w.fb_cap);
        });
        if (level_trace) {
          int h2[4];
          cudaMemcpyAsync(h2, w.fb1, sizeof(int) * 4, cudaMemcpyDeviceToHost, st);
          cudaStreamSynchronize(st);
          fbstat[2] = h2[0];
          fbstat[3] = h2[2];
          fbstat[5] = h2[3];
          cudaMemsetAsync(w.fb1 + 2, 0, sizeof(int) * 2, st);
        }
      } else if (mode == NPL) {
        timed(K_BLUR0, [&] {
          const dim3 tg(lc.tb_grid.x, (pgl.r1 + TB_T - 1) / TB_T - pgl.r0 / TB_T);
          blur_tile_kernel<<<tg, TB_THREADS, tile_blur_smem_bytes(hc.tile_blur_hmax), st>>>(
              w.feat, w.target, pgl, lc.lvl, w.den32);
        });
      } else {
        const int hl = sch.hs[lv];
        const PadFn p0 = pad_fn(0, hl), p1 = pad_fn(1, hl);
        timed(K_BLUR0, [&] {
          p0<<<lc.blur_grid, 256, 0, st>>>(w.feat, w.tmp, pgl, lc.lvl, nullptr, w.fb0, w.fb_cap, w.fb1);
          blur_pad_fallback_kernel<0, 0><<<lc.fb_grid, 256, 0, st>>>(w.feat, w.tmp, pgl, lc.lvl, nullptr, w.fb0,
                                                                     w.fb_cap);
        });
        timed(K_BLUR1, [&] {
          p1<<<lc.blur_grid, 256, 0, st>>>(w.tmp, w.target, pgl, lc.lvl, w.den32, w.fb1, w.fb_cap, w.fb0);
          blur_pad_fallback_kernel<1, 1><<<lc.fb_grid, 256, 0, st>>>(w.tmp, w.target, pgl, lc.lvl, w.den32, w.fb1,
                                                                     w.fb_cap);
        });
      }
      timed(K_DIST, [&] {
        level_stats_kernel<<<lc.dist_grid, RED_THREADS, 0, st>>>(
            w.ctrl, lc.sched, w.feat, w.target, w.dcache, n, D, S, w.spart + MAX_PARTS, done, 0, 0,
            parity ? nullptr : w.sel, w.sel_stride, world > 1 ? w.lvl_part + XPART * a->rank : nullptr);
      });
      if (hc.exact_stats) {
        timed(K_DIST, [&] {
          np_distance();
          np_level_start_kernel<<<1, 32, 0, st>>>(w.ctrl, lc.sched, w.np_out, n);
        });
      }
      CKL();
      if (world > 1) {
        // the ranks' exact 128-bit partials, all-gathered in place, then the
        // identical level-start controller on every rank
        const int xr = a->exchange(a->exchange_ctx, PLAS_XCHG_ALLGATHER, (int64_t)(XPART * sizeof(double)),
                                   (int64_t)((char*)w.lvl_part - (char*)wsp), nullptr);
        if (xr < 0) {
          cleanup();
          return fail(PLAS_ERR_CUDA, "exchange callback failed (level partials)");
        }
        level_start_shard_kernel<<<1, RED_THREADS, 0, st>>>(w.ctrl, lc.sched, w.lvl_part, world, n);
      }
      CKL();
      int dy = 0, dx = 0;
      if (parity) {  // draws for the first pass of the level
        dy = (int)rng.integers(beta);
        dx = (int)rng.integers(beta);
        rng.permutation(bsq, pinned + pp * b0sq);
      }
      for (;;) {
        if (parity) {
          CK(cudaMemcpyAsync(w.mp, pinned + pp * b0sq, sizeof(int) * bsq, cudaMemcpyHostToDevice, st));
          timed(K_SELECT, [&] {
            set_pass_kernel<<<1, 32, 0, st>>>(w.ctrl, dy, dx);
            class_select_kernel<<<9, 1024, 0, st>>>(w.mp, w.ctrl, w.sel, w.sel_stride);
          });
        }
        {
          float* feat = w.feat;
          int* idx = w.idx;
          const float* target = w.target;
          const Ctrl* ctrl = w.ctrl;
          const int* sel = w.sel;  // PARITY: class_select_kernel; DEVICE: gen_class_tables
          long long sstride = w.sel_stride;
          int Dv = D, Sv = S;
          void* args[] = {&feat, &idx, &target, &Dv, &Sv, &ctrl, &sel, &sstride, &ml, &counters};
          cudaError_t le = cudaSuccess;
          if (use_tile(beta, S))
            timed(K_PASS, [&] {
              le = cudaLaunchKernel(tfn, dim3(lc.tile_grid), dim3(TILE_CTA_THREADS), args,
                                    (size_t)(TILE_NST * tile_stage_bytes(beta, S)), st);
            });
          else
            timed(K_PASS, [&] { le = cudaLaunchKernel(kpc.fn, dim3(kpc.grid), dim3(kpc.block), args, kpc.smem, st); });
          if (le != cudaSuccess) {
            cleanup();
            return fail(PLAS_ERR_CUDA, std::string("pass launch: ") + cudaGetErrorString(le));
          }
        }
        timed(K_CTRL, [&] {
          (S > 16 ? pass_stats_kernel<true> : pass_stats_kernel<false>)<<<sgrid, RED_THREADS, 0, st>>>(w.ctrl, lc.sched, w.feat, w.target, w.dcache, D, S,
                                                           w.list, counters, w.spart + MAX_PARTS, done, n, 0, 0, a->xchg_part,
                                                           parity || world > 1 ? nullptr : w.sel, w.sel_stride);
          if (!parity && world > 1) gen_tables_kernel<<<num_sms(), 256, 0, st>>>(w.ctrl, w.sel, w.sel_stride);
          if (hc.exact_stats) {
            np_distance();
            np_pass_control_kernel<<<1, 32, 0, st>>>(w.ctrl, lc.sched, w.np_out);
          }
        });
        CKL();
        if (world > 1) {
          // exchange this rank's updates + partial, apply the others', run the controller
          shard_pack_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(w.list, counters, w.idx, (int2*)a->xchg_send);
          CKL();
          const int m = a->exchange(a->exchange_ctx, PLAS_XCHG_PASS, 0, 0, nullptr);
          if (m < 0) {
            cleanup();
            return fail(PLAS_ERR_CUDA, "exchange callback failed");
          }
          shard_apply_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>((const int2*)a->xchg_recv, m, a->xchg_part_all,
                                                                  world, a->rank, w.orig32, w.feat, w.idx, w.target,
                                                                  w.dcache, D, S, w.ctrl);
          shard_control_kernel<<<1, RED_THREADS, 0, st>>>(w.ctrl, lc.sched, a->xchg_part_all, world, counters, n);
          CKL();
        }
        CK(cudaMemcpyAsync(hflag, &w.ctrl->level_done, sizeof(int), cudaMemcpyDeviceToHost, st));
        // speculative draws for the next pass while the GPU runs this one
        host::NumpyPhilox saved = rng;
        int ndy = 0, ndx = 0;
        if (parity) {
          ndy = (int)rng.integers(beta);
          ndx = (int)rng.integers(beta);
          rng.permutation(bsq, pinned + (1 - pp) * b0sq);
        }
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
          cleanup();
          return fail(PLAS_ERR_CUDA, std::string("pass: ") + cudaGetErrorString(e));
        }
        flush_profile();
        if (*hflag) {
          rng = saved;  // the level ended: these draws belong to the next level's stream
          break;
        }
        dy = ndy;
        dx = ndx;
        pp = 1 - pp;
      }
      timed(K_CTRL, [&] { level_end_kernel<<<1, 32, 0, st>>>(w.ctrl, lc.sched, 0); });
      CKL();
      if (level_trace) {
        CK(cudaStreamSynchronize(st));
        flush_profile();
        char lab[16];
        if (use_fft)
          snprintf(lab, sizeof(lab), "f%d", fplans[mode].L);
        else
          snprintf(lab, sizeof(lab), "%s", mode == NPL ? "tile" : (mode == NPL + 1 ? "dir" : "dirH"));
        if (getenv("PLAS_FB_TRACE")) {  // uncertain blur outputs of the level (FFT: needs -DPLAS_FB_STATS)
          fprintf(stderr, "  fallbacks: axis0 list %d local %d (sequential %d)   axis1 list %d local %d (sequential %d)\n",
                  fbstat[0], fbstat[1], fbstat[4], fbstat[2], fbstat[3], fbstat[5]);
        }
        fprintf(stderr, "level %3d h %4d beta %4d %-5s passes %3d pass %7.1f us blur0 %7.1f blur1 %7.1f border %6.1f "
                "dist %6.1f ctrl %7.1f us (%d)\n", lv, sch.hs[lv], beta,
                lab,
                lvl_n[K_PASS], 1e3 * lvl_ms[K_PASS] / (lvl_n[K_PASS] ? lvl_n[K_PASS] : 1), 1e3 * lvl_ms[K_BLUR0],
                1e3 * lvl_ms[K_BLUR1], 1e3 * lvl_ms[K_BORDER], 1e3 * lvl_ms[K_DIST], 1e3 * lvl_ms[K_CTRL],
                lvl_n[K_CTRL]);
        for (int k = 0; k < 7; k++) lvl_ms[k] = 0, lvl_n[k] = 0;
      }
    }
    CK(cudaStreamSynchronize(st));
    flush_profile();
    cleanup();
  }

  // ---- final VAD, perm, report
  if (int e = vad_launch(w.scalars + 2)) return e;
  perm_i32_to_i64_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(w.idx, (long long*)res->perm, n);
  CKL();
  CK(cudaEventRecord(ev1, st));
  Ctrl out;
  double sc[3];
  int fl[8];
  CK(cudaMemcpyAsync(&out, w.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(fl, w.flags, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(sc, w.scalars, sizeof(double) * 3, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  res->gpu_ms = ms;
  res->initial_vad = sc[1];
  res->final_vad = sc[2];
  res->reorders = out.reorders;
  res->levels_done = out.levels_done;
  res->trace_len = out.trace_pos;
  res->cells_moved = fl[2];
  res->exact_warps = fl[3];
  res->banded_levels = banded_levels;
  if (gtr) {
    std::vector<unsigned long long> g(6 * (size_t)out.reorders);
    cudaMemcpy(g.data(), gtr, sizeof(unsigned long long) * g.size(), cudaMemcpyDeviceToHost);
    cudaFree(gtr);
    double k3 = 0, st_ = 0, gap1 = 0, gap2 = 0, dist = 0, tail = 0, tabs = 0;
    long long n1 = 0, n2 = 0;
    for (long long p = 0; p < out.reorders; p++) {
      const unsigned long long* e = &g[6 * p];
      if (!e[0] || !e[1] || !e[2] || !e[3] || !e[4]) continue;
      const double a0 = (double)~e[0], a1 = (double)e[1], b0 = (double)~e[2], b1 = (double)e[3];
      const double tk = (double)e[4], tb = e[5] ? (double)e[5] : tk;
      k3 += a1 - a0;
      st_ += std::max(b1, tb) - b0;
      gap1 += b0 - a1;
      dist += tk - b0;
      tail += b1 - tk;
      tabs += tb - tk;
      n1++;
      if (p + 1 < out.reorders && g[6 * (p + 1)]) {
        const double c0 = (double)~g[6 * (p + 1)];
        const double end = std::max(b1, tb);
        if (c0 > end && c0 - end < 2e4) {  // within a level (a level boundary carries a blur)
          gap2 += c0 - end;
          n2++;
        }
      }
    }
    if (n1)
      fprintf(stderr, "gtrace: %lld passes  K3 %.2f us  stats %.2f us (to last ticket %.2f, controller tail %.2f, "
              "tables after ticket %.2f)  gap K3->stats %.2f us  gap stats->K3 %.2f us (%lld)\n",
              n1, k3 / n1 / 1e3, st_ / n1 / 1e3, dist / n1 / 1e3, tail / n1 / 1e3, tabs / n1 / 1e3,
              gap1 / n1 / 1e3, n2 ? gap2 / n2 / 1e3 : 0.0, n2);
  }
  if (out.status) return fail(PLAS_ERR_CAPACITY, "trace capacity exceeded");
  if (res->level_counts && L > 0)
    CK(cudaMemcpy(res->level_counts, w.level_counts, sizeof(long long) * L, cudaMemcpyDeviceToHost));
  if (res->trace && out.trace_pos > 0)
    CK(cudaMemcpy(res->trace, w.trace, sizeof(double) * out.trace_pos, cudaMemcpyDeviceToHost));
  return PLAS_OK;
}

int plas_assign_groups(float* feat, int64_t* point_idx, const float* target, int dim, int stride,
                       const int64_t* groups, int64_t num_groups, int group_size, void* stream) {
  if (dim < 1 || stride < dim || stride % 4 || group_size < 2 || group_size > 4)
    return fail(PLAS_ERR_INVALID, "bad assign_groups arguments");
  if (num_groups <= 0) return PLAS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int grid = grid_for(num_groups * 4, 256, 4);
  if (stride <= 16)
    groups_kernel<false><<<grid, 256, 0, st>>>(feat, (long long*)point_idx, target, dim, stride,
                                               (const long long*)groups, num_groups, group_size);
  else
    groups_kernel<true><<<grid, 256, 0, st>>>(feat, (long long*)point_idx, target, dim, stride,
                                              (const long long*)groups, num_groups, group_size);
  CKL();
  return PLAS_OK;
}

int plas_assign_groups_f64t(float* feat, int64_t* point_idx, const double* target, int dim, int stride,
                            const int64_t* groups, int64_t num_groups, int group_size, void* stream) {
  if (dim < 1 || dim > 64 || stride < dim || group_size < 2 || group_size > 4)
    return fail(PLAS_ERR_INVALID, "bad assign_groups_f64t arguments");
  if (num_groups <= 0) return PLAS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  groups_f64t_kernel<<<grid_for(num_groups, 256, 4), 256, 0, st>>>(
      feat, (long long*)point_idx, target, dim, stride, (const long long*)groups, num_groups, group_size);
  CKL();
  return PLAS_OK;
}

static size_t carve_np(char* base, long long n, double** v, double** vals, long long** lstart, int** llen,
                       int** left, int** right, int** order, int** hoff, double** out, bool with_v = true) {
  Carver c{base};
  const size_t nleaf = (size_t)(n / 64 + 4);
  *v = c.take<double>(with_v ? (size_t)n : 1);
  *vals = c.take<double>(2 * nleaf);
  *lstart = c.take<long long>(nleaf);
  *llen = c.take<int>(nleaf);
  *left = c.take<int>(nleaf);
  *right = c.take<int>(nleaf);
  *order = c.take<int>(nleaf);
  *hoff = c.take<int>(72);
  *out = c.take<double>(2);
  return align_up(c.off);
}

// NumPy-order sum of v[0..n) (np_sum.cuh): out2[0] = sum, out2[1] = sum / n.
// The tree tables go up from pageable host memory; cudaMemcpyAsync has staged
// such a copy by the time it returns, so the host vectors may die here.
static int np_sum_device(const double* v, long long n, char* npws, double* out2, cudaStream_t st) {
  double *vv, *vals, *out;
  long long* ls;
  int *ll, *l, *r, *o, *h;
  carve_np(npws, n, &vv, &vals, &ls, &ll, &l, &r, &o, &h, &out, false);
  NpTree t;
  np_tree_make(&t, n);
  const size_t nl = t.leaf_start.size(), ni = t.left.size();
  CK(cudaMemcpyAsync(ls, t.leaf_start.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ll, t.leaf_len.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, st));
  if (ni) {
    CK(cudaMemcpyAsync(l, t.left.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(r, t.right.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(o, t.order.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(h, t.hoff.data(), sizeof(int) * t.hoff.size(), cudaMemcpyHostToDevice, st));
  np_leaf_kernel<<<std::max<int>(1, (int)((nl + 255) / 256)), 256, 0, st>>>(v, ls, ll, (int)nl, vals);
  np_tree_kernel<<<1, 1024, 0, st>>>(vals, l, r, o, h, (int)t.hoff.size() - 1, (int)nl, t.root, n, out2);
  return PLAS_OK;
}

struct AuxWs {
  double *t0, *t1, *t2, *t3, *den64, *rows, *w, *partials, *scalars;
  float* den32;
  char* np;  // NumPy-order sum tables over H W C values (smoothness mean)
};

static size_t carve_aux(char* base, int H, int W, int C, AuxWs* a) {
  Carver c{base};
  size_t cells = (size_t)H * W, tot = cells * C;
  a->t0 = c.take<double>(tot);
  a->t1 = c.take<double>(tot);
  a->t2 = c.take<double>(tot);
  a->t3 = c.take<double>(tot);
  a->den64 = c.take<double>(cells);
  a->den32 = c.take<float>(cells);
  a->rows = c.take<double>(H);
  a->w = c.take<double>((H > W ? H : W) + 4096);
  a->partials = c.take<double>(MAX_PARTS);
  a->scalars = c.take<double>(8);
  double *v, *vals, *out;
  long long* ls;
  int *ll, *l, *r, *o, *h;
  a->np = c.take<char>(carve_np(nullptr, std::max<size_t>(tot, 1), &v, &vals, &ls, &ll, &l, &r, &o, &h, &out, false));
  return align_up(c.off);
}

size_t plas_aux_workspace_bytes(int H, int W, int C) {
  AuxWs a;
  return carve_aux(nullptr, H, W, C, &a);
}

static int launch_blur(const void* in, void* out, int dtype, int H, int W, int C, int S, int h,
                       const AuxWs& a, bool renorm, cudaStream_t st) {
  BlurLevelRef lv{nullptr, nullptr, nullptr, nullptr, h, a.w};
  int grid0 = grid_for((long long)W * S * ((H + BLUR_R - 1) / BLUR_R), 256, 8);
  int grid1 = grid_for((long long)H * S * ((W + BLUR_R - 1) / BLUR_R), 256, 8);
  if (renorm) {
    border_rows_kernel<<<grid_for(H, 128, 1), 128, 0, st>>>(a.rows, H, lv);
    border_weight_kernel<<<grid_for((long long)H * ((W + 1) / 2), 256, 8), 256, 0, st>>>(
        a.rows, a.den32, a.den64, H, W, lv);
  }
  if (dtype == PLAS_F32) {
    float* tmp = (float*)a.t0;
    blur_axis_kernel<float, float, 0, 0><<<grid0, 256, 0, st>>>((const float*)in, tmp, H, W, C, S, lv, nullptr);
    if (renorm)
      blur_axis_kernel<float, float, 1, 1><<<grid1, 256, 0, st>>>(tmp, (float*)out, H, W, C, S, lv, a.den32);
    else
      blur_axis_kernel<float, float, 0, 1><<<grid1, 256, 0, st>>>(tmp, (float*)out, H, W, C, S, lv, nullptr);
  } else {
    double* tmp = a.t0;
    blur_axis_kernel<double, double, 0, 0><<<grid0, 256, 0, st>>>((const double*)in, tmp, H, W, C, S, lv, nullptr);
    if (renorm)
      blur_axis_kernel<double, double, 2, 1><<<grid1, 256, 0, st>>>(tmp, (double*)out, H, W, C, S, lv, a.den64);
    else
      blur_axis_kernel<double, double, 0, 1><<<grid1, 256, 0, st>>>(tmp, (double*)out, H, W, C, S, lv, nullptr);
  }
  CKL();
  return PLAS_OK;
}

// ---- the sort's level blur (fast tiers + exact fallback) on an arbitrary grid
struct TierWs {
  float *feat_alloc, *feat, *tmp_alloc, *tmp, *target, *den32;
  double *rows, *w, *spec;
  double2* tw;
  int *fb0, *fb1;
  int pad, fb_cap, L, lc;
  size_t feat_floats, tmp_floats;
};

static size_t carve_tiers(char* base, int H, int W, int C, int h, TierWs* t) {
  Carver c{base};
  const int S = row_stride(C);
  t->pad = h + std::max(BLUR_R, BPAD_R) + 1;
  t->feat_floats = (size_t)(H + 2 * t->pad) * W * S;
  t->feat_alloc = c.take<float>(t->feat_floats);
  t->feat = t->feat_alloc ? t->feat_alloc + (size_t)t->pad * W * S : nullptr;
  t->tmp_floats = (size_t)H * (W + 2 * t->pad) * S;
  t->tmp_alloc = c.take<float>(t->tmp_floats);
  t->tmp = t->tmp_alloc ? t->tmp_alloc + (size_t)t->pad * S : nullptr;
  t->target = c.take<float>((size_t)H * W * S);
  t->den32 = c.take<float>((size_t)H * W);
  t->rows = c.take<double>((size_t)H);
  t->w = c.take<double>((size_t)h + 1);
  // FFT length: L >= n + h (linear convolution) and n <= fft_out_max (the raw-line buffer)
  t->lc = fft_choose_code(std::max(H, W), h);
  t->L = t->lc >= 0 ? fft_len(t->lc) : 0;
  t->tw = c.take<double2>(t->L ? (size_t)fft_twiddle_len(t->lc) : 1);
  t->spec = c.take<double>((size_t)std::max(t->L, 1));
  t->fb_cap = (int)std::min<long long>((long long)H * W * S / 8 + 1024, 1LL << 26);
  t->fb0 = c.take<int>((size_t)FB_HEADER + t->fb_cap);
  t->fb1 = c.take<int>((size_t)FB_HEADER + t->fb_cap);
  return align_up(c.off);
}

__global__ void pad_rows_kernel(const float* __restrict__ in, float* __restrict__ out, long long cells, int C, int S) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cells * S;
       t += (long long)gridDim.x * blockDim.x) {
    const long long cell = t / S;
    const int c = (int)(t - cell * S);
    out[t] = c < C ? in[cell * C + c] : 0.f;
  }
}

__global__ void unpad_rows_kernel(const float* __restrict__ in, float* __restrict__ out, long long cells, int C, int S) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cells * C;
       t += (long long)gridDim.x * blockDim.x) {
    const long long cell = t / C;
    const int c = (int)(t - cell * C);
    out[t] = in[cell * S + c];
  }
}

size_t plas_blur_tiers_workspace_bytes(int H, int W, int C, int half_width) {
  TierWs t;
  return carve_tiers(nullptr, H, W, C, half_width, &t);
}

int plas_blur_target_tiers(const float* in, float* out, int H, int W, int C, const double* weights, int half_width,
                           int tier, int64_t* fallbacks, void* ws, size_t ws_bytes, void* stream) {
  if (H < 1 || W < 1 || C < 1 || half_width < 1 || !weights || tier < 0 || tier > 2)
    return fail(PLAS_ERR_INVALID, "bad blur tier arguments");
  if (tier == 2 && half_width > TB_HMAX) return fail(PLAS_ERR_INVALID, "tile tier needs half_width <= 16");
  TierWs t;
  if (!ws || ws_bytes < carve_tiers(nullptr, H, W, C, half_width, &t))
    return fail(PLAS_ERR_WORKSPACE, "tier workspace");
  carve_tiers((char*)ws, H, W, C, half_width, &t);
  if (tier == 1 && !t.L) return fail(PLAS_ERR_INVALID, "grid too long for the FFT tier");
  cudaStream_t st = (cudaStream_t)stream;
  const int S = row_stride(C);
  const long long cells = (long long)H * W;
  CK(cudaMemsetAsync(t.feat_alloc, 0, sizeof(float) * t.feat_floats, st));
  CK(cudaMemsetAsync(t.tmp_alloc, 0, sizeof(float) * t.tmp_floats, st));
  CK(cudaMemsetAsync(t.fb0, 0, sizeof(int) * FB_HEADER, st));
  CK(cudaMemsetAsync(t.fb1, 0, sizeof(int) * FB_HEADER, st));
  CK(cudaMemcpyAsync(t.w, weights, sizeof(double) * (half_width + 1), cudaMemcpyHostToDevice, st));
  pad_rows_kernel<<<grid_for(cells * S, 256, 8), 256, 0, st>>>(in, t.feat, cells, C, S);
  BlurLevelRef lv{nullptr, nullptr, nullptr, nullptr, half_width, t.w};
  PadGeom pg = make_pad_geom(H, W, C, S, t.pad);
  border_rows_kernel<<<grid_for(H, 128, 1), 128, 0, st>>>(t.rows, H, lv);
  border_weight_kernel<<<grid_for((long long)H * ((W + 1) / 2), 256, 8), 256, 0, st>>>(t.rows, t.den32, nullptr, H,
                                                                                        W, lv);
  const int fbg = num_sms() * 2;
  int64_t counts[2] = {0, 0};
  int hc[2];
  if (tier == 2) {
    const size_t smem = tile_blur_smem_bytes(half_width);
    CK(raise_smem_limit((const void*)blur_tile_kernel, smem));
    hc[0] = hc[1] = 0;
    blur_tile_kernel<<<dim3((W + TB_T - 1) / TB_T, (H + TB_T - 1) / TB_T), TB_THREADS, smem, st>>>(t.feat, t.target, pg,
                                                                                                  lv, t.den32);
  } else if (tier == 0) {
    const int g0 = grid_for((long long)W * S * ((H + BPAD_R - 1) / BPAD_R), 256, 8);
    pad_fn(0, half_width)<<<g0, 256, 0, st>>>(t.feat, t.tmp, pg, lv, nullptr, t.fb0, t.fb_cap, t.fb1);
    CK(cudaMemcpyAsync(&hc[0], t.fb0, sizeof(int), cudaMemcpyDeviceToHost, st));
    blur_pad_fallback_kernel<0, 0><<<fbg, 256, 0, st>>>(t.feat, t.tmp, pg, lv, nullptr, t.fb0, t.fb_cap);
    pad_fn(1, half_width)<<<g0, 256, 0, st>>>(t.tmp, t.target, pg, lv, t.den32, t.fb1, t.fb_cap, t.fb0);
    CK(cudaMemcpyAsync(&hc[1], t.fb1, sizeof(int), cudaMemcpyDeviceToHost, st));
    blur_pad_fallback_kernel<1, 1><<<fbg, 256, 0, st>>>(t.tmp, t.target, pg, lv, t.den32, t.fb1, t.fb_cap);
  } else {
    std::vector<double2> htw;
    fft_twiddles(t.lc, &htw);
    CK(cudaMemcpyAsync(t.tw, htw.data(), sizeof(double2) * htw.size(), cudaMemcpyHostToDevice, st));
    const int lg = t.lc;
    const FftPlan plan{lg, t.L, t.tw, t.spec, fft_error_constant(lg)};
    void* f0 = fft_kernel_ptr<0, 0>(lg);
    void* f1 = fft_kernel_ptr<1, 1>(lg);
    const size_t smem = fft_smem_bytes(t.lc);
    CK(raise_smem_limit((const void*)f0, smem));
    CK(raise_smem_limit((const void*)f1, smem));
    const int nt = fft_threads(t.L);
    fft_spectrum_kernel<<<std::max(1, t.L / 128), 128, 0, st>>>(lv, plan);
    const float *i0 = t.feat, *i1 = t.tmp, *dn = nullptr, *den = t.den32;
    float *o0 = t.tmp, *o1 = t.target;
    int cap = t.fb_cap;
    void* a0[] = {&i0, &o0, &pg, &lv, (void*)&plan, &dn, &t.fb0, &cap, &t.fb1};
    void* a1[] = {&i1, &o1, &pg, &lv, (void*)&plan, &den, &t.fb1, &cap, &t.fb0};
    const int g0 = W * ((C + 1) / 2);  // one CTA per line pair
    const int g1 = H * ((C + 1) / 2);
    CK(cudaLaunchKernel(f0, dim3(g0), dim3(nt), a0, smem, st));
    CK(cudaMemcpyAsync(&hc[0], t.fb0, sizeof(int), cudaMemcpyDeviceToHost, st));
    blur_pad_fallback_kernel<0, 0><<<fbg, 256, 0, st>>>(t.feat, t.tmp, pg, lv, nullptr, t.fb0, t.fb_cap);
    CK(cudaLaunchKernel(f1, dim3(g1), dim3(nt), a1, smem, st));
    CK(cudaMemcpyAsync(&hc[1], t.fb1, sizeof(int), cudaMemcpyDeviceToHost, st));
    blur_pad_fallback_kernel<1, 1><<<fbg, 256, 0, st>>>(t.tmp, t.target, pg, lv, t.den32, t.fb1, t.fb_cap);
  }
  unpad_rows_kernel<<<grid_for(cells * C, 256, 8), 256, 0, st>>>(t.target, out, cells, C, S);
  CKL();
  CK(cudaStreamSynchronize(st));
  counts[0] = hc[0];
  counts[1] = hc[1];
  if (fallbacks) {
    fallbacks[0] = counts[0];
    fallbacks[1] = counts[1];
  }
  return PLAS_OK;
}

int plas_blur(const void* in, void* out, int dtype, int H, int W, int C, const double* weights,
              int half_width, int op, void* ws, size_t ws_bytes, void* stream) {
  if (H < 1 || W < 1 || C < 1 || half_width < 0 || !weights || (dtype != PLAS_F32 && dtype != PLAS_F64))
    return fail(PLAS_ERR_INVALID, "bad blur arguments");
  AuxWs a;
  if (!ws || ws_bytes < carve_aux(nullptr, H, W, C, &a)) return fail(PLAS_ERR_WORKSPACE, "aux workspace");
  carve_aux((char*)ws, H, W, C, &a);
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(a.w, weights, sizeof(double) * (half_width + 1), cudaMemcpyHostToDevice, st));
  if (op == PLAS_BLUR_BORDER_WEIGHT) {
    BlurLevelRef lv{nullptr, nullptr, nullptr, nullptr, half_width, a.w};
    border_rows_kernel<<<grid_for(H, 128, 1), 128, 0, st>>>(a.rows, H, lv);
    border_weight_kernel<<<grid_for((long long)H * ((W + 1) / 2), 256, 8), 256, 0, st>>>(
        a.rows, nullptr, (double*)out, H, W, lv);
    CKL();
    return PLAS_OK;
  }
  return launch_blur(in, out, dtype, H, W, C, C, half_width, a, op == PLAS_BLUR_RENORMALIZED, st);
}

// workspace of plas_grid_distance: per-cell values + the NumPy tree
size_t plas_grid_distance_workspace_bytes(int64_t n) {
  double *v, *vals, *out;
  long long* ls;
  int *ll, *l, *r, *o, *h;
  return carve_np(nullptr, std::max<int64_t>(n, 1), &v, &vals, &ls, &ll, &l, &r, &o, &h, &out);
}

// grid_distance (plas.py:71-84) in NumPy's summation order (np_sum.cuh):
// bit-identical to the reference's float
int plas_grid_distance(const double* a, const double* b, const double* weights, int64_t n, int dim,
                       double* out_dev, void* ws, size_t ws_bytes, void* stream) {
  if (n < 1 || dim < 1) return fail(PLAS_ERR_INVALID, "bad grid_distance arguments");
  if (!ws || ws_bytes < plas_grid_distance_workspace_bytes(n)) return fail(PLAS_ERR_WORKSPACE, "grid_distance workspace");
  cudaStream_t st = (cudaStream_t)stream;
  double *v, *vals, *out;
  long long* ls;
  int *ll, *l, *r, *o, *h;
  carve_np((char*)ws, n, &v, &vals, &ls, &ll, &l, &r, &o, &h, &out);
  np_cell_f64_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(a, b, weights, n, dim, v);
  if (int e = np_sum_device(v, n, (char*)vals, out, st)) return e;
  CK(cudaMemcpyAsync(out_dev, out + 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
  CKL();
  return PLAS_OK;
}

size_t plas_vad_workspace_bytes(int H, int W, int C) {
  const long long m = std::max<long long>(1, (long long)(H - 1) * W * C + (long long)H * (W - 1) * C);
  double *v, *vals, *out;
  long long* ls;
  int *ll, *l, *r, *o, *h;
  return carve_np(nullptr, m, &v, &vals, &ls, &ll, &l, &r, &o, &h, &out, false) + sizeof(double) * 8;
}

// vad (metrics.py:25-40) in NumPy's order (np_sum.cuh VadElems): the
// reference's float for fp32 and fp64 grids
int plas_vad(const void* grid, int dtype, int H, int W, int C, double* out_dev, void* ws,
             size_t ws_bytes, void* stream) {
  if (H < 2 || W < 2 || C < 1) return fail(PLAS_ERR_INVALID, "vad needs H, W >= 2");
  if (!ws || ws_bytes < plas_vad_workspace_bytes(H, W, C)) return fail(PLAS_ERR_WORKSPACE, "vad workspace");
  cudaStream_t st = (cudaStream_t)stream;
  const long long M = (long long)(H - 1) * W * C + (long long)H * (W - 1) * C;
  double *v, *vals, *out;
  long long* ls;
  int *ll, *l, *r, *o, *h;
  carve_np((char*)ws, M, &v, &vals, &ls, &ll, &l, &r, &o, &h, &out, false);  // values formed on the fly
  double* out4 = (double*)((char*)ws + plas_vad_workspace_bytes(H, W, C) - sizeof(double) * 8);
  NpTree t;
  np_tree_make(&t, M);
  const size_t nl = t.leaf_start.size(), ni = t.left.size();
  CK(cudaMemcpyAsync(ls, t.leaf_start.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ll, t.leaf_len.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, st));
  if (ni) {
    CK(cudaMemcpyAsync(l, t.left.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(r, t.right.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(o, t.order.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(h, t.hoff.data(), sizeof(int) * t.hoff.size(), cudaMemcpyHostToDevice, st));
  const int lg = std::max(1, (int)((nl + 255) / 256)), nh = (int)t.hoff.size() - 1;
  const unsigned long long m0 = (unsigned long long)(H - 1) * W * C;
  if (dtype == PLAS_F32) {
    const VadElems<float> el{(const float*)grid, (unsigned)H, (unsigned)W, (unsigned)C, (unsigned)C, m0};
    np_leaf_vad_kernel<0, float><<<lg, 256, 0, st>>>(el, nullptr, ls, ll, (int)nl, vals);
    np_tree_kernel<<<1, 1024, 0, st>>>(vals, l, r, o, h, nh, (int)nl, t.root, M, out4);
    np_leaf_vad_kernel<1, float><<<lg, 256, 0, st>>>(el, out4, ls, ll, (int)nl, vals);
  } else {
    const VadElems<double> el{(const double*)grid, (unsigned)H, (unsigned)W, (unsigned)C, (unsigned)C, m0};
    np_leaf_vad_kernel<0, double><<<lg, 256, 0, st>>>(el, nullptr, ls, ll, (int)nl, vals);
    np_tree_kernel<<<1, 1024, 0, st>>>(vals, l, r, o, h, nh, (int)nl, t.root, M, out4);
    np_leaf_vad_kernel<1, double><<<lg, 256, 0, st>>>(el, out4, ls, ll, (int)nl, vals);
  }
  np_tree_kernel<<<1, 1024, 0, st>>>(vals, l, r, o, h, nh, (int)nl, t.root, M, out4 + 2);
  CK(cudaMemcpyAsync(out_dev, out4 + 3, sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));  // the host tree vectors live on this frame only
  CKL();
  return PLAS_OK;
}

int plas_smoothness_plane(const double* plane, double* grad, int H, int W, int C, double coeff,
                          double huber_delta, int detach_target, const double* weights,
                          int half_width, double* loss_dev, void* ws, size_t ws_bytes,
                          void* stream) {
  if (H < 1 || W < 1 || C < 1 || !(huber_delta > 0) || half_width < 0)
    return fail(PLAS_ERR_INVALID, "bad smoothness arguments");
  AuxWs a;
  if (!ws || ws_bytes < carve_aux(nullptr, H, W, C, &a)) return fail(PLAS_ERR_WORKSPACE, "aux workspace");
  carve_aux((char*)ws, H, W, C, &a);
  cudaStream_t st = (cudaStream_t)stream;
  const long long cells = (long long)H * W, tot = cells * C;
  const int eg = grid_for(tot, 256, 8);
  const double scale = coeff / (double)tot;
  if (half_width <= 4) {  // fused single-kernel path (kernel_size <= 9)
    if (half_width > 0 && !weights) return fail(PLAS_ERR_INVALID, "weights required");
    const double one = 1.0;
    CK(cudaMemcpyAsync(a.w, half_width > 0 ? weights : &one, sizeof(double) * (half_width + 1),
                       cudaMemcpyHostToDevice, st));
    const dim3 grid((W + SM_TS - 1) / SM_TS, (H + SM_TS - 1) / SM_TS);
    void* fn = nullptr;
    size_t smem = 0;
    switch (half_width) {
      case 0: fn = (void*)smooth_fused_kernel<0>; smem = SmoothTile<0>::smem_doubles * 8; break;
      case 1: fn = (void*)smooth_fused_kernel<1>; smem = SmoothTile<1>::smem_doubles * 8; break;
      case 2: fn = (void*)smooth_fused_kernel<2>; smem = SmoothTile<2>::smem_doubles * 8; break;
      case 3: fn = (void*)smooth_fused_kernel<3>; smem = SmoothTile<3>::smem_doubles * 8; break;
      default: fn = (void*)smooth_fused_kernel<4>; smem = SmoothTile<4>::smem_doubles * 8; break;
    }
    CK(raise_smem_limit((const void*)fn, smem));
    const double* pl = plane;
    double* gr = grad;
    const double* wd = a.w;
    int Hh = H, Ww = W, Cc = C, det = detach_target;
    double dl = huber_delta, sc = scale;
    double* hv = a.t0;
    void* args[] = {&pl, &gr, &Hh, &Ww, &Cc, &wd, &dl, &sc, &det, &hv};
    CK(cudaLaunchKernel(fn, grid, dim3(256), args, smem, st));
    if (int e = np_sum_device(a.t0, tot, a.np, a.scalars, st)) return e;
    CK(cudaMemcpyAsync(loss_dev, a.scalars + 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
    CKL();
    return PLAS_OK;
  }
  if (half_width > 0) {
    if (!weights) return fail(PLAS_ERR_INVALID, "weights required");
    CK(cudaMemcpyAsync(a.w, weights, sizeof(double) * (half_width + 1), cudaMemcpyHostToDevice, st));
    anchor_center_kernel<<<eg, 256, 0, st>>>(plane, a.t1, cells, C);
    if (int e = launch_blur(a.t1, a.t2, PLAS_F64, H, W, C, C, half_width, a, true, st)) return e;
  }
  huber_kernel<<<eg, 256, 0, st>>>(a.t1, a.t2, a.t3, tot, huber_delta, scale, half_width == 0, a.t0);
  if (int e = np_sum_device(a.t0, tot, a.np, a.scalars, st)) return e;
  CK(cudaMemcpyAsync(loss_dev, a.scalars + 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (detach_target || half_width == 0) {
    CK(cudaMemcpyAsync(grad, a.t3, sizeof(double) * tot, cudaMemcpyDeviceToDevice, st));
  } else {
    div_den_kernel<<<eg, 256, 0, st>>>(a.t3, a.den64, a.t1, cells, C);
    if (int e = launch_blur(a.t1, a.t2, PLAS_F64, H, W, C, C, half_width, a, false, st)) return e;
    sub_kernel<<<eg, 256, 0, st>>>(a.t3, a.t2, grad, tot);
  }
  CKL();
  return PLAS_OK;
}

// ---------------------------------------------------------------- feature prep
size_t plas_prune_workspace_bytes(int64_t n) {
  const long long nb = (n + PREP_CHUNK - 1) / PREP_CHUNK;
  return 256 + 256 * sizeof(unsigned) + (size_t)std::max(nb, 1LL) * sizeof(int2) + 256;
}

int plas_prune_to_grid(const double* logit, int64_t n, int64_t keep, int64_t* survivors, void* ws,
                       size_t ws_bytes, void* stream) {
  if (!logit || !survivors || n < 1 || keep < 1 || keep > n || n >= (1LL << 31))
    return fail(PLAS_ERR_INVALID, "prune_to_grid: need 1 <= keep <= n < 2^31");
  if (!ws || ws_bytes < plas_prune_workspace_bytes(n)) return fail(PLAS_ERR_WORKSPACE, "prune workspace");
  cudaStream_t st = (cudaStream_t)stream;
  Carver c{(char*)ws};
  SelectState* s = c.take<SelectState>(1);
  unsigned* hist = c.take<unsigned>(256);
  const long long nb = (n + PREP_CHUNK - 1) / PREP_CHUNK;
  int2* counts = c.take<int2>((size_t)nb);
  const int grid = grid_for(n, SEL_THREADS, 4);
  select_init_kernel<<<1, SEL_THREADS, 0, st>>>(s, n - keep, hist);
  for (int shift = 56; shift >= 0; shift -= 8) {
    select_hist_kernel<<<grid, SEL_THREADS, 0, st>>>(logit, n, s, shift, hist);
    select_pick_kernel<<<1, SEL_THREADS, 0, st>>>(s, shift, hist);
  }
  prune_count_kernel<<<(unsigned)nb, SEL_THREADS, 0, st>>>(logit, n, s, counts);
  prune_scan_kernel<<<1, 1024, 0, st>>>(counts, (int)nb);
  prune_write_kernel<<<(unsigned)nb, SEL_THREADS, 0, st>>>(logit, n, s, counts, (long long*)survivors);
  CKL();
  return PLAS_OK;
}

size_t plas_normalize_workspace_bytes(int64_t n, int total_channels) {
  const int parts = std::min(grid_for(n, 256, 4), 1024);
  return (size_t)parts * std::max(total_channels, 1) * sizeof(double2) + 256;
}

int plas_normalize_for_sorting(const plas_attr* attrs, int num_attrs, int64_t n, double* features,
                               int feat_cols, double* mins, double* maxs, void* ws, size_t ws_bytes,
                               void* stream) {
  if (!attrs || num_attrs < 1 || num_attrs > PREP_MAX_ATTRS || n < 1 || !mins || !maxs)
    return fail(PLAS_ERR_INVALID, "normalize_for_sorting: bad arguments");
  PrepAttrs at{};
  int ch = 0, col = 0;
  for (int i = 0; i < num_attrs; i++) {
    const plas_attr& a = attrs[i];
    if (a.channels < 0 || a.activation < 0 || a.activation > 2 || !(a.weight >= 0.0) ||
        (a.channels > 0 && (!a.values || a.row_stride < a.channels)))
      return fail(PLAS_ERR_INVALID, "normalize_for_sorting: bad attribute");
    PrepAttr& p = at.a[i];
    p.v = a.values;
    p.stride = a.row_stride;
    p.channels = a.channels;
    p.act = a.activation;
    p.weight = a.weight;
    p.ch0 = ch;
    p.col = (a.weight != 0.0 && a.channels > 0) ? col : -1;
    if (p.col >= 0) col += a.channels;
    ch += a.channels;
  }
  at.count = num_attrs;
  at.total_ch = ch;
  if (ch > PREP_MAX_CH) return fail(PLAS_ERR_INVALID, "normalize_for_sorting: too many channels");
  if (col != feat_cols || (col > 0 && !features))
    return fail(PLAS_ERR_INVALID, "normalize_for_sorting: feat_cols != channels of the weighted attributes");
  if (!ws || ws_bytes < plas_normalize_workspace_bytes(n, ch)) return fail(PLAS_ERR_WORKSPACE, "normalize workspace");
  cudaStream_t st = (cudaStream_t)stream;
  if (ch == 0) return PLAS_OK;
  const int parts = std::min(grid_for(n, 256, 4), 1024);
  double2* part = reinterpret_cast<double2*>(ws);
  prep_minmax_kernel<<<parts, 256, 0, st>>>(at, n, part);
  prep_minmax_final_kernel<<<1, 1024, 0, st>>>(part, parts, ch, mins, maxs);
  if (col > 0) prep_write_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(at, n, feat_cols, mins, maxs, features);
  CKL();
  return PLAS_OK;
}

int plas_gather_rows(const void* src, int64_t row_bytes, const int64_t* index, int64_t count, void* dst,
                     void* stream) {
  if (count < 0 || row_bytes < 0 || (count > 0 && (!src || !dst || !index)))
    return fail(PLAS_ERR_INVALID, "gather_rows: bad arguments");
  if (count == 0 || row_bytes == 0) return PLAS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const uintptr_t al = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)row_bytes;
  const int vb = al % 16 == 0 ? 16 : (al % 8 == 0 ? 8 : (al % 4 == 0 ? 4 : 1));
  const long long rv = row_bytes / vb, total = count * rv;
  if (total >= (1LL << 32) - 1) return fail(PLAS_ERR_INVALID, "gather_rows: more than 2^32 vectors");
  unsigned m;
  int l;
  make_fastdiv((unsigned)rv, &m, &l);
  const int grid = grid_for(total, 256, 8);
  const long long* ix = (const long long*)index;
  if (vb == 16)
    gather_rows_kernel<uint4><<<grid, 256, 0, st>>>((const uint4*)src, (unsigned)rv, m, l, ix, (unsigned)total,
                                                    (uint4*)dst);
  else if (vb == 8)
    gather_rows_kernel<unsigned long long><<<grid, 256, 0, st>>>((const unsigned long long*)src, (unsigned)rv, m, l,
                                                                  ix, (unsigned)total, (unsigned long long*)dst);
  else if (vb == 4)
    gather_rows_kernel<unsigned><<<grid, 256, 0, st>>>((const unsigned*)src, (unsigned)rv, m, l, ix, (unsigned)total,
                                                       (unsigned*)dst);
  else
    gather_rows_kernel<unsigned char><<<grid, 256, 0, st>>>((const unsigned char*)src, (unsigned)rv, m, l, ix,
                                                             (unsigned)total, (unsigned char*)dst);
  CKL();
  return PLAS_OK;
}

size_t plas_quantize_workspace_bytes(int64_t n, int channels) {
  const int parts = std::min(grid_for(n, 256, 4), 1024);
  return (size_t)parts * std::max(channels, 1) * sizeof(double2) + 256;
}

int plas_quantize_planes(const double* values, int64_t n, int channels, int64_t row_stride, int contract,
                         int data_driven, double clip_min, double clip_max, int levels, int bit_depth,
                         int per_image, void* planes, double* lo_out, double* hi_out, void* ws, size_t ws_bytes,
                         void* stream) {
  if (n < 1 || channels < 1 || channels > 256 || row_stride < channels || !values || !planes || !lo_out ||
      !hi_out || levels < 2 || (bit_depth != 8 && bit_depth != 16) || per_image < 1 || channels % per_image)
    return fail(PLAS_ERR_INVALID, "quantize_planes: bad arguments");
  if (levels > (1 << bit_depth)) return fail(PLAS_ERR_INVALID, "quantize_planes: levels do not fit bit_depth");
  if (!data_driven && !(clip_min < clip_max)) return fail(PLAS_ERR_INVALID, "clip_min must be below clip_max");
  if (!ws || ws_bytes < plas_quantize_workspace_bytes(n, channels)) return fail(PLAS_ERR_WORKSPACE, "quantize workspace");
  cudaStream_t st = (cudaStream_t)stream;
  if (data_driven) {
    const int parts = std::min(grid_for(n, 256, 4), 1024);
    double2* part = reinterpret_cast<double2*>(ws);
    quant_minmax_kernel<<<parts, 256, 0, st>>>(values, n, channels, row_stride, contract, part);
    quant_range_kernel<<<1, 1024, 0, st>>>(part, parts, channels, lo_out, hi_out);
  } else {
    quant_fill_kernel<<<1, 256, 0, st>>>(lo_out, hi_out, channels, clip_min, clip_max);
  }
  const int grid = grid_for(n * channels, 256, 8);
  if (bit_depth == 8)
    quant_pack_kernel<unsigned char><<<grid, 256, 0, st>>>(values, n, channels, row_stride, contract, lo_out, hi_out,
                                                           levels, per_image, (unsigned char*)planes);
  else
    quant_pack_kernel<unsigned short><<<grid, 256, 0, st>>>(values, n, channels, row_stride, contract, lo_out,
                                                            hi_out, levels, per_image, (unsigned short*)planes);
  CKL();
  return PLAS_OK;
}

}  // extern "C"
