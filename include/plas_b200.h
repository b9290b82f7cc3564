/*
 * plas_b200.h -- C ABI of the B200-native PLAS sort hot path.
 *
 * Drop-in boundary for the reference's sort path (/root/reference/pkg/src/sogs).
 * The reference is pure Python and has no C ABI; each entry point below
 * replaces one reference function (file:line cited) and is what a binding
 * (ctypes / cffi / pybind) of that Python API calls.  Plain pointers and
 * sizes only: device pointers are CUDA device addresses, `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Nothing throws across the
 * ABI; every call returns a plas_status (0 = ok, < 0 = error) and
 * plas_last_error() describes the last failure of the calling thread.
 *
 * All work runs on the current CUDA device; there is no CPU fallback.
 */
#ifndef PLAS_B200_H
#define PLAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLAS_ABI_VERSION 5

enum plas_status {
  PLAS_OK = 0,
  PLAS_ERR_INVALID = -1,   /* bad argument (the Python layer raises ValueError first) */
  PLAS_ERR_CUDA = -2,      /* CUDA runtime error */
  PLAS_ERR_NONFINITE = -3, /* features contain NaN/Inf (plas.py:236-237) */
  PLAS_ERR_CAPACITY = -4,  /* trace buffer too small: retry with a larger capacity */
  PLAS_ERR_WORKSPACE = -5  /* workspace smaller than plas_*_workspace_bytes() */
};

enum plas_dtype { PLAS_F32 = 0, PLAS_F64 = 1 };

/* PARITY: NumPy-exact Generator(Philox(seed)) draws generated on the host,
 *         bit-identical to the reference (plas.py:240-262).
 * DEVICE: counter-based Philox4x64-10 draws on the device keyed like NumPy's
 *         (SeedSequence state); grouping by a keyed bijection per block class;
 *         the whole sort runs as one CUDA graph with no host round trip. */
enum plas_rng_mode { PLAS_RNG_PARITY = 0, PLAS_RNG_DEVICE = 1 };

/* exchange callback operations of a sharded sort (plas_sort_args.exchange) */
enum plas_xchg_op { PLAS_XCHG_PASS = 0, PLAS_XCHG_ALLGATHER = 1, PLAS_XCHG_ALLTOALL = 2 };

enum plas_blur_op {
  PLAS_BLUR_SEPARABLE = 0,     /* blur.py:7-10   separable_blur            */
  PLAS_BLUR_RENORMALIZED = 1,  /* blur.py:18-30  renormalized_blur (= blur_target, plas.py:64-68) */
  PLAS_BLUR_BORDER_WEIGHT = 2  /* blur.py:13-15  border_weight (out is (H, W) f64) */
};

typedef struct plas_sort_args {
  const void* features;          /* device, (n, dim) row-major, PLAS_F32 or PLAS_F64 */
  int features_dtype;
  int dim;                       /* D >= 1 */
  int64_t n;                     /* side * side, side >= 2 */
  /* SortConfig (plas.py:37-51) */
  double improvement_threshold;  /* > 0 */
  double radius_decay;           /* (0, 1); used only when radii == NULL */
  double initial_radius;         /* NaN = reference rule max(side/2-1, 2) (plas.py:54-57) */
  int min_block_size;            /* >= 2 */
  uint64_t seed;                 /* SortConfig.rng_seed */
  int rng_mode;                  /* plas_rng_mode */
  /* schedule (host arrays).  radii[l] by repeated fp64 multiplication
   * (plas.py:246, 274); weights = concatenated Gaussian kernels w[0..h_l]
   * (centre first) as scipy.ndimage._gaussian_kernel1d(r/2, 0, ceil(r))
   * computes them.  NULL -> built by the library (libm exp; may differ from
   * NumPy's exp in the last ulp, so parity callers pass NumPy weights). */
  int num_levels;
  const double* radii;
  const double* weights;
  const int64_t* weight_offsets;
  const int64_t* initial_perm;   /* device [n] int64 or NULL (paired-protocol hook) */
  int64_t trace_capacity;        /* entries of the distance trace buffer */
  void* stream;
  /* optional host plas_sort_profile*: when set, the sort is driven from the
   * host one kernel at a time with CUDA events around every launch (same
   * kernels, same work; DEVICE mode then syncs once per pass instead of
   * running as one graph).  Used by bench.py for per-kernel roofline data. */
  void* profile;
  /* Multi-GPU sharding (world > 1; 0 or 1 = single GPU).  Every rank runs
   * plas_sort on its own device with identical arguments and keeps a full
   * replica of the grid (features and element indices).  Per level: when
   * beta * world <= side (banded levels) rank r owns rows [Y_r, Y_r+1),
   * Y_r = side * r / world, processes the pass's block rows that start there
   * (row bands aligned to the pass's block tiling) and computes the target
   * only on [Y_r, Y_r+1 + beta); on the FFT blur tier the axis-0 transforms
   * are split by columns and exchanged by one all-to-all.  Other levels split
   * each pass's groups evenly and blur the whole grid.  The level-start
   * distance sum and every pass's distance change are exchanged as exact
   * 128-bit fixed-point partials, so the result is bit-identical to one GPU.
   * The library calls exchange(exchange_ctx, op, a, b, sizes):
   *   PLAS_XCHG_PASS: after each pass the library wrote this rank's
   *     (int128 distance change as two 64-bit words, moved-cell count, 0) to
   *     xchg_part[0..3] and its (cell, element) int32 pairs to xchg_send; the
   *     callback all-gathers xchg_part into xchg_part_all[4 * world] (rank
   *     order) and the first m pairs of every rank's xchg_send into
   *     xchg_recv (rank r's pairs at r * m), m >= the largest moved-cell count
   *     (xchg_part_all[4 r + 2]), and returns m.
   *   PLAS_XCHG_ALLGATHER: in-place all-gather of a bytes per rank inside the
   *     workspace: rank r's piece is at ws + b + r * a; returns 0.
   *   PLAS_XCHG_ALLTOALL: workspace byte offsets a (send) and b (recv); host
   *     sizes[q] = bytes sent to rank q (send segments in rank order),
   *     sizes[world + q] = bytes received from rank q (recv segments in rank
   *     order); returns 0.
   * Negative returns abort the sort.  Collectives must be ordered after the
   * work already enqueued on `stream` and before work enqueued after the call
   * returns (torch.distributed over NCCL on the current stream does this). */
  int rank;
  int world;
  int (*exchange)(void* exchange_ctx, int op, int64_t a, int64_t b, const int64_t* sizes);
  void* exchange_ctx;
  void* xchg_send;        /* device int32 [2 * n] */
  void* xchg_recv;        /* device int32 [2 * n * world] */
  double* xchg_part;      /* device [4] */
  double* xchg_part_all;  /* device [4 * world] */
} plas_sort_args;

/* Per-kernel device time (CUDA events, ms) summed over all launches. */
typedef struct plas_sort_profile {
  double ms_pass;      int64_t n_pass;      /* K3 fused assign + distance   */
  double ms_blur0;     int64_t n_blur0;     /* K1 axis-0 blur               */
  double ms_blur1;     int64_t n_blur1;     /* K1 axis-1 blur + renormalize */
  double ms_border;    int64_t n_border;    /* K1b border weight            */
  double ms_distance;  int64_t n_distance;  /* level-start distance         */
  double ms_control;   int64_t n_control;   /* K4 controller kernels        */
  double ms_select;    int64_t n_select;    /* parity class filter          */
} plas_sort_profile;

typedef struct plas_sort_result {
  int64_t* perm;                 /* device [n] out: features[perm] is the sorted grid */
  double initial_vad;            /* metrics.py:25-40 on the fp32 working copy */
  double final_vad;
  int64_t reorders;              /* total passes (plas.py:265) */
  int levels_done;
  int64_t* level_counts;         /* host [num_levels] out: trace entries per level */
  double* trace;                 /* host [trace_capacity] out: radius_trace distances */
  int64_t trace_len;
  double gpu_ms;                 /* device time from init gather to perm ready */
  int64_t cells_moved;           /* elements that changed cell, summed over passes */
  int64_t exact_warps;           /* warps whose decision needed the exact fp64 tier */
  int64_t banded_levels;         /* sharded sorts: levels run in row bands (the rest replicated) */
} plas_sort_result;

int plas_abi_version(void);
/* sizeof the two structs, so bindings can verify their layout */
size_t plas_sizeof_sort_args(void);
size_t plas_sizeof_sort_result(void);
const char* plas_last_error(void);

/* Number of levels the schedule has (0 if side < 2). */
int plas_num_levels(int64_t n, double radius_decay, double initial_radius);

/* Workspace for plas_sort; ws must be 256-byte aligned device memory. */
size_t plas_sort_workspace_bytes(int64_t n, int dim, int num_levels, int64_t weights_len,
                                 int64_t trace_capacity, int rng_mode);
/* Same for a sharded sort on `world` ranks (adds the element-order f32 copy). */
size_t plas_sort_workspace_bytes_sharded(int64_t n, int dim, int num_levels, int64_t weights_len,
                                         int64_t trace_capacity, int rng_mode, int world);

/* sort_grid / sort_grid_report (plas.py:226-301). */
int plas_sort(const plas_sort_args* args, plas_sort_result* result, void* ws, size_t ws_bytes);

/* _assign_groups (plas.py:113-156) on device arrays, in place: feat (rows of
 * `stride` >= dim floats, stride % 4 == 0, 16-byte aligned), point_idx int64,
 * groups (num_groups, group_size) int64 cell indices, group_size in {2,3,4},
 * lexicographic arrangement table PERMUTATIONS[group_size] (plas.py:31-34). */
int plas_assign_groups(float* feat, int64_t* point_idx, const float* target, int dim, int stride,
                       const int64_t* groups, int64_t num_groups, int group_size, void* stream);

/* Same with a float64 target (rows of `stride` doubles, dim <= 64): the
 * reference's numba kernel then differences in fp64 (plas.py:134-136 with a
 * float64 `target`), which this entry reproduces. */
int plas_assign_groups_f64t(float* feat, int64_t* point_idx, const double* target, int dim, int stride,
                            const int64_t* groups, int64_t num_groups, int group_size, void* stream);

/* Workspace for the auxiliary entry points below on an (H, W, C) grid. */
size_t plas_aux_workspace_bytes(int H, int W, int C);

/* blur.py ops on an (H, W, C) grid (device in/out, dtype preserved; f32
 * RENORMALIZED uses the reference's fp32-rounded parity arithmetic).
 * weights: host [half_width + 1], centre first. */
int plas_blur(const void* in, void* out, int dtype, int H, int W, int C, const double* weights,
              int half_width, int op, void* ws, size_t ws_bytes, void* stream);

/* blur_target (plas.py:64-68) of an (H, W, C) f32 grid through the SORT's
 * level-blur tiers: tier 0 = direct fast fold, tier 1 = FFT convolution,
 * tier 2 = one-kernel tile blur (half_width <= 16); all
 * certify every output against the SciPy fold and recompute the uncertain
 * ones exactly, so the result is bit-identical to the reference.  weights:
 * host [half_width + 1], centre first.  fallbacks: optional host [2] out, the
 * outputs recomputed by the exact fold per axis.  Synchronises the stream. */
size_t plas_blur_tiers_workspace_bytes(int H, int W, int C, int half_width);
int plas_blur_target_tiers(const float* in, float* out, int H, int W, int C, const double* weights,
                           int half_width, int tier, int64_t* fallbacks, void* ws, size_t ws_bytes,
                           void* stream);

/* grid_distance (plas.py:71-84): fp64 (n, dim) inputs, optional device
 * weights [dim]; result written to *out_dev (device double).  Summed in
 * NumPy's pairwise order, so the value equals the reference's bit for bit;
 * ws of plas_grid_distance_workspace_bytes(n) bytes. */
size_t plas_grid_distance_workspace_bytes(int64_t n);
int plas_grid_distance(const double* a, const double* b, const double* weights, int64_t n, int dim,
                       double* out_dev, void* ws, size_t ws_bytes, void* stream);

/* vad (metrics.py:25-40) of an (H, W, C) grid (PLAS_F32 or PLAS_F64) in
 * NumPy's summation order: the reference's float; result to *out_dev; ws of
 * plas_vad_workspace_bytes(H, W, C) bytes. */
size_t plas_vad_workspace_bytes(int H, int W, int C);
int plas_vad(const void* grid, int dtype, int H, int W, int C, double* out_dev, void* ws,
             size_t ws_bytes, void* stream);

/* One plane of smoothness_loss (smoothness.py:57-97): fp64 plane (H, W, C),
 * coeff = overall_multiplier * weight, weights/half_width of
 * gaussian(params.sigma, kernel_size // 2) (half_width 0 -> zero residual).
 * *loss_dev = mean(huber(residual)) (the caller scales by coeff exactly as
 * smoothness.py:88 does); grad (H, W, C) f64 is the full gradient. */
int plas_smoothness_plane(const double* plane, double* grad, int H, int W, int C, double coeff,
                          double huber_delta, int detach_target, const double* weights,
                          int half_width, double* loss_dev, void* ws, size_t ws_bytes,
                          void* stream);

/* ---- caller-side feature preparation ---------------------- */

/* prune_to_grid (splats.py:139-152): indices of the `keep` Gaussians that a
 * stable ascending argsort of opacity_logit puts last, in increasing index
 * order, written to survivors (device int64 [keep]).  opacity_logit: device
 * fp64 [n], finite (SplatCloud validation, splats.py:58-60). */
size_t plas_prune_workspace_bytes(int64_t n);
int plas_prune_to_grid(const double* opacity_logit, int64_t n, int64_t keep, int64_t* survivors, void* ws,
                       size_t ws_bytes, void* stream);

/* One attribute of normalize_for_sorting (splats.py:184-216): device fp64
 * rows of `channels` values, `row_stride` values apart; activation 0 = none,
 * 1 = sigmoid, 2 = exp (SplatCloud.activated, splats.py:86-93); weight >= 0
 * (0: min/max only, no output columns). */
typedef struct plas_attr {
  const double* values;
  int64_t row_stride;
  int32_t channels;
  int32_t activation;
  double weight;
} plas_attr;
#define PLAS_MAX_ATTRS 8
#define PLAS_MAX_ATTR_CHANNELS 64

/* normalize_for_sorting: features (device fp64 [n, feat_cols], feat_cols =
 * total channels of the weight > 0 attributes, in attribute order) and the
 * per-channel mins / maxs of every attribute's activated values (device fp64
 * [total channels], attribute order). */
size_t plas_normalize_workspace_bytes(int64_t n, int total_channels);
int plas_normalize_for_sorting(const plas_attr* attrs, int num_attrs, int64_t n, double* features,
                               int feat_cols, double* mins, double* maxs, void* ws, size_t ws_bytes,
                               void* stream);

/* Row gather dst[i] = src[index[i]], i < count, rows of row_bytes bytes
 * (values[perm], bundle.py:160; SplatCloud.select, splats.py:95-104). */
int plas_gather_rows(const void* src, int64_t row_bytes, const int64_t* index, int64_t count, void* dst,
                     void* stream);

/* Quantize one attribute into its encoded image planes:
 * _quantize_attribute (bundle.py:102-115) with contract (quantization.py:8-11)
 * when `contract`, quantize (quantization.py:28-41) per channel, and the
 * plane slicing of compress (bundle.py:170-176): channel c goes to image
 * c / per_image, sample c % per_image; planes = device uint8 (bit_depth 8) or
 * uint16 (16) [channels / per_image][n][per_image].  data_driven: per-channel
 * lo = min, hi = max (min + 1 if constant) of the (contracted) values, else
 * clip_min / clip_max.  lo_out / hi_out: device fp64 [channels] (manifest). */
size_t plas_quantize_workspace_bytes(int64_t n, int channels);
int plas_quantize_planes(const double* values, int64_t n, int channels, int64_t row_stride, int contract,
                         int data_driven, double clip_min, double clip_max, int levels, int bit_depth,
                         int per_image, void* planes, double* lo_out, double* hi_out, void* ws, size_t ws_bytes,
                         void* stream);

/* NumPy SeedSequence(seed).generate_state(2, uint64) -> key (Philox4x64 key). */
void plas_seed_key(uint64_t seed, uint64_t key[2]);

/* Generator(Philox(seed)).permutation(n), NumPy-exact, on the host. */
int plas_host_permutation(uint64_t seed, int64_t n, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* PLAS_B200_H */
