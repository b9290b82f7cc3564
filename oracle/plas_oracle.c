/*
 * plas_oracle.c -- CPU restatement of the reference's PLAS sort hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2312_13299_b200/ links, loads
 * or calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may use it, and only as the checker or
 * the CPU timing arm.  It is pinned against fixtures produced by the real
 * reference (tests/golden/make_golden.py) in tests/test_oracle_golden.py.
 *
 * Restates, from /root/reference/pkg/src/sogs:
 *   plas.py:226-286  _sort (driver, strikes, decay)         -> oracle_sort
 *   plas.py:196-223  _reassign_pass (classes, <m filter)     -> reassign_pass
 *   plas.py:173-193  reassign_block                          -> oracle_reassign_block
 *   plas.py:113-156  _assign_groups (numba arithmetic)       -> oracle_assign_groups
 *   plas.py:64-68 + blur.py:7-30  blur_target / renormalized_blur (SciPy correlate1d order)
 *   plas.py:71-84    grid_distance (NumPy pairwise order)    -> oracle_grid_distance_f32
 *   metrics.py:25-40 vad                                     -> oracle_vad
 *   smoothness.py:57-97 smoothness_loss (one plane)          -> oracle_smoothness_plane
 * and the third-party arithmetic the path delegates to:
 *   NumPy 2.3.5 SeedSequence + Philox4x64-10 + Generator.integers (32-bit Lemire)
 *   + Generator.permutation (Fisher-Yates, masked rejection)  (plas.py:240-262)
 *   SciPy 1.18.1 ndimage.correlate1d symmetric-kernel loop (fp64, zero padding):
 *       out = in[0]*w0; for j = h..1: out += (in[-j] + in[j]) * w_j
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off (no FMA: the reference's
 * numba/SciPy code has none).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------ */
/* NumPy SeedSequence (numpy/random/bit_generator.pyx)                 */
/* ------------------------------------------------------------------ */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t value, uint32_t *hc) {
    value ^= *hc;
    *hc *= SS_MULT_A;
    value *= *hc;
    value ^= value >> 16;
    return value;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

/* key = SeedSequence(seed).generate_state(2, uint64) for a non-negative int seed < 2**64 */
void oracle_seed_key(uint64_t seed, uint64_t key[2]) {
    uint32_t ent[2];
    int nent = 0;
    if (seed == 0) {
        ent[nent++] = 0;
    } else {
        while (seed) {
            ent[nent++] = (uint32_t)(seed & 0xffffffffu);
            seed >>= 32;
        }
    }
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < nent ? ent[i] : 0u, &hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    for (int s = 4; s < nent; s++)
        for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
    uint32_t st[4];
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < 4; i++) {
        uint32_t v = pool[i % 4];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    key[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
    key[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}

/* ------------------------------------------------------------------ */
/* Philox4x64-10 with NumPy's buffering (numpy/random/src/philox)      */
/* ------------------------------------------------------------------ */
typedef struct {
    uint64_t ctr[4];
    uint64_t key[2];
    uint64_t buf[4];
    int pos;      /* next unread word of buf; 4 = empty */
    int has32;    /* buffered upper half available */
    uint32_t u32;
} oracle_rng;

static inline uint64_t mulhi64(uint64_t a, uint64_t b) {
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

static void philox4x64_10(const uint64_t in[4], const uint64_t k_in[2], uint64_t out[4]) {
    uint64_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    uint64_t k0 = k_in[0], k1 = k_in[1];
    for (int r = 0; r < 10; r++) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = mulhi64(0xD2E7470EE14C6C93ull, c0);
        uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = mulhi64(0xCA5A826395121157ull, c2);
        uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

int oracle_rng_size(void) { return (int)sizeof(oracle_rng); }

void oracle_rng_init(oracle_rng *r, uint64_t seed) {
    memset(r, 0, sizeof(*r));
    oracle_seed_key(seed, r->key);
    r->pos = 4;
}

static uint64_t rng_next64(oracle_rng *r) {
    if (r->pos < 4) return r->buf[r->pos++];
    /* counter pre-increment: the first block uses ctr = (1, 0, 0, 0) */
    for (int i = 0; i < 4; i++)
        if (++r->ctr[i]) break;
    philox4x64_10(r->ctr, r->key, r->buf);
    r->pos = 1;
    return r->buf[0];
}

static uint32_t rng_next32(oracle_rng *r) {
    if (r->has32) {
        r->has32 = 0;
        return r->u32;
    }
    uint64_t v = rng_next64(r);
    r->has32 = 1;
    r->u32 = (uint32_t)(v >> 32);
    return (uint32_t)(v & 0xffffffffu);
}

/* Generator.integers(0, high) for 1 <= high <= 2**32 (int64 dtype, Lemire) */
int64_t oracle_rng_integers(oracle_rng *r, int64_t high) {
    uint64_t rng = (uint64_t)(high - 1);
    if (rng == 0) return 0;
    if (rng == 0xffffffffull) return (int64_t)rng_next32(r);
    uint32_t rng_excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)rng_next32(r) * rng_excl;
    uint32_t left = (uint32_t)m;
    if (left < rng_excl) {
        uint32_t thresh = (uint32_t)(0xffffffffu - (uint32_t)rng) % rng_excl;
        while (left < thresh) {
            m = (uint64_t)rng_next32(r) * rng_excl;
            left = (uint32_t)m;
        }
    }
    return (int64_t)(m >> 32);
}

/* Generator.permutation(n): arange then Fisher-Yates i = n-1..1 with masked rejection */
void oracle_rng_permutation(oracle_rng *r, int64_t n, int64_t *out) {
    for (int64_t i = 0; i < n; i++) out[i] = i;
    for (int64_t i = n - 1; i >= 1; i--) {
        uint64_t mask = (uint64_t)i;
        mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
        mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
        uint64_t v;
        if ((uint64_t)i <= 0xffffffffull) {
            while ((v = (rng_next32(r) & mask)) > (uint64_t)i) {}
        } else {
            while ((v = (rng_next64(r) & mask)) > (uint64_t)i) {}
        }
        int64_t t = out[i];
        out[i] = out[v];
        out[v] = t;
    }
}

/* ------------------------------------------------------------------ */
/* Blur (SciPy correlate1d, symmetric kernel, mode constant 0)         */
/* ------------------------------------------------------------------ */
/*
 * One axis of the blur, restated as "for each output line position, for each
 * tap j = h..1 (outermost first), for every element of the slab": the
 * per-element operation sequence is exactly SciPy's
 *     acc = in[i] * w0;  for j = h..1: acc += (in[i-j] + in[i+j]) * w_j
 * while the innermost loop runs over contiguous memory.
 * A slab is `len` contiguous doubles; line positions are `n` slabs apart by
 * `stride` elements; `get` converts the input element to double.
 */
#define AXIS_PASS(TIN, TOUT, in, out, n, nslab, slab_stride, stride, len, w, h)            \
    do {                                                                                 \
        double *acc = (double *)malloc(sizeof(double) * (size_t)(len));                   \
        for (int64_t sl = 0; sl < (nslab); sl++) {                                        \
            const TIN *ib = (in) + sl * (slab_stride);                                    \
            TOUT *ob = (out) + sl * (slab_stride);                                        \
            for (int64_t i = 0; i < (n); i++) {                                           \
                const TIN *ci = ib + i * (stride);                                        \
                for (int64_t e = 0; e < (len); e++) acc[e] = (double)ci[e] * (w)[0];      \
                for (int j = (h); j >= 1; j--) {                                           \
                    const TIN *lo = (i - j >= 0) ? ib + (i - j) * (stride) : NULL;         \
                    const TIN *hi = (i + j < (n)) ? ib + (i + j) * (stride) : NULL;        \
                    double wj = (w)[j];                                                   \
                    for (int64_t e = 0; e < (len); e++) {                                 \
                        double p = (lo ? (double)lo[e] : 0.0) + (hi ? (double)hi[e] : 0.0);\
                        acc[e] = acc[e] + p * wj;                                         \
                    }                                                                     \
                }                                                                         \
                TOUT *co = ob + i * (stride);                                             \
                for (int64_t e = 0; e < (len); e++) co[e] = (TOUT)acc[e];                 \
            }                                                                             \
        }                                                                                 \
        free(acc);                                                                        \
    } while (0)

/* axis-0 pass (along y) then axis-1 pass (along x) over an (H, W, C) grid.
 * f32: f32 in, f32 out after each axis (gaussian_filter1d on float32 arrays).
 * f64: f64 everywhere.
 * w: h+1 weights (w[0] centre), computed by NumPy exactly as scipy's _gaussian_kernel1d. */
void oracle_separable_blur_f32(const float *in, int H, int W, int C, const double *w, int h,
                               float *out) {
    float *tmp = (float *)malloc(sizeof(float) * (size_t)H * W * C);
    const int64_t row = (int64_t)W * C;
    /* axis 0: one slab = a whole row (W*C), positions y */
    AXIS_PASS(float, float, in, tmp, H, 1, 0, row, row, w, h);
    /* axis 1: per row y, positions x, slab = the C channels of a cell */
    for (int y = 0; y < H; y++) {
        const float *ir = tmp + (int64_t)y * row;
        float *orow = out + (int64_t)y * row;
        AXIS_PASS(float, float, ir, orow, W, 1, 0, C, C, w, h);
    }
    free(tmp);
}

void oracle_separable_blur_f64(const double *in, int H, int W, int C, const double *w, int h,
                               double *out) {
    double *tmp = (double *)malloc(sizeof(double) * (size_t)H * W * C);
    const int64_t row = (int64_t)W * C;
    AXIS_PASS(double, double, in, tmp, H, 1, 0, row, row, w, h);
    for (int y = 0; y < H; y++) {
        const double *ir = tmp + (int64_t)y * row;
        double *orow = out + (int64_t)y * row;
        AXIS_PASS(double, double, ir, orow, W, 1, 0, C, C, w, h);
    }
    free(tmp);
}

/* border_weight (blur.py:13-15): separable blur of a ones plane, fp64 throughout */
void oracle_border_weight(int H, int W, const double *w, int h, double *den) {
    double *ones = (double *)malloc(sizeof(double) * (size_t)H * W);
    for (size_t i = 0; i < (size_t)H * W; i++) ones[i] = 1.0;
    oracle_separable_blur_f64(ones, H, W, 1, w, h, den);
    free(ones);
}

/* blur_target (plas.py:64-68) on an f32 grid: f32 out, divided in f32 by f32(den) */
void oracle_blur_target_f32(const float *in, int H, int W, int C, const double *w, int h,
                            float *out) {
    double *den = (double *)malloc(sizeof(double) * (size_t)H * W);
    oracle_border_weight(H, W, w, h, den);
    oracle_separable_blur_f32(in, H, W, C, w, h, out);
    for (size_t i = 0; i < (size_t)H * W; i++) {
        float d = (float)den[i];
        for (int c = 0; c < C; c++) out[i * C + c] = out[i * C + c] / d;
    }
    free(den);
}

/* renormalized_blur (blur.py:18-30) on an f64 grid */
void oracle_blur_target_f64(const double *in, int H, int W, int C, const double *w, int h,
                            double *out) {
    double *den = (double *)malloc(sizeof(double) * (size_t)H * W);
    oracle_border_weight(H, W, w, h, den);
    oracle_separable_blur_f64(in, H, W, C, w, h, out);
    for (size_t i = 0; i < (size_t)H * W; i++)
        for (int c = 0; c < C; c++) out[i * C + c] = out[i * C + c] / den[i];
    free(den);
}

/* ------------------------------------------------------------------ */
/* _assign_groups (plas.py:113-156)                                    */
/* ------------------------------------------------------------------ */
static int PERM_TABLE[5][24][4];
static int PERM_COUNT[5];
static int perm_ready = 0;

static void build_perms(void) {
    if (perm_ready) return;
    for (int k = 1; k <= 4; k++) {
        /* lexicographic order == itertools.permutations(range(k)) */
        int cnt = 0;
        int a[4];
        for (int i = 0; i < k; i++) a[i] = i;
        for (;;) {
            for (int i = 0; i < k; i++) PERM_TABLE[k][cnt][i] = a[i];
            cnt++;
            int i = k - 2;
            while (i >= 0 && a[i] > a[i + 1]) i--;
            if (i < 0) break;
            int j = k - 1;
            while (a[j] < a[i]) j--;
            int t = a[i]; a[i] = a[j]; a[j] = t;
            for (int l = i + 1, r = k - 1; l < r; l++, r--) {
                t = a[l]; a[l] = a[r]; a[r] = t;
            }
        }
        PERM_COUNT[k] = cnt;
    }
    perm_ready = 1;
}

/* groups: (G, k) flat cell indices; feat/target rows have stride S >= D (only D used) */
void oracle_assign_groups(float *feat, int64_t *idx, const float *target, int D, int S,
                          const int64_t *groups, int64_t G, int k) {
    build_perms();
    float cost[4][4];
    float *held = (float *)malloc(sizeof(float) * 4 * (size_t)S);
    int64_t held_idx[4];
    for (int64_t g = 0; g < G; g++) {
        const int64_t *cells = groups + g * k;
        for (int i = 0; i < k; i++)
            for (int j = 0; j < k; j++) {
                double s = 0.0;
                const float *f = feat + cells[i] * S;
                const float *t = target + cells[j] * S;
                for (int d = 0; d < D; d++) {
                    float delta = f[d] - t[d];
                    float sq = delta * delta;
                    s += (double)sq;
                }
                cost[i][j] = (float)sqrt(s);
            }
        int best = 0;
        double best_cost = INFINITY;
        for (int p = 0; p < PERM_COUNT[k]; p++) {
            double c = 0.0;
            for (int i = 0; i < k; i++) c += (double)cost[i][PERM_TABLE[k][p][i]];
            if (c < best_cost) {
                best_cost = c;
                best = p;
            }
        }
        if (best == 0) continue;
        for (int i = 0; i < k; i++) {
            for (int d = 0; d < S; d++) held[i * S + d] = feat[cells[i] * S + d];
            held_idx[i] = idx[cells[i]];
        }
        for (int i = 0; i < k; i++) {
            int64_t dst = cells[PERM_TABLE[k][best][i]];
            for (int d = 0; d < S; d++) feat[dst * S + d] = held[i * S + d];
            idx[dst] = held_idx[i];
        }
    }
    free(held);
}

/* reassign_block (plas.py:173-193) */
void oracle_reassign_block(float *feat, int64_t *idx, const float *target, int D, int S,
                           const int64_t *positions, int64_t m, const int64_t *grouping,
                           int64_t ng) {
    int64_t *ordered = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    int64_t cnt = 0;
    for (int64_t i = 0; i < ng; i++)
        if (grouping[i] < m) ordered[cnt++] = positions[grouping[i]];
    int64_t g4 = (m / 4) * 4;
    if (g4) oracle_assign_groups(feat, idx, target, D, S, ordered, g4 / 4, 4);
    int64_t rest = m - g4;
    if (rest >= 2) oracle_assign_groups(feat, idx, target, D, S, ordered + g4, 1, (int)rest);
    free(ordered);
}

/* ------------------------------------------------------------------ */
/* grid_distance (plas.py:71-84) and vad (metrics.py:25-40)            */
/* ------------------------------------------------------------------ */
/* NumPy's pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), which
 * np.sum / np.mean use on contiguous float64 runs: m < 8 -> plain loop from
 * 0.0; m <= 128 -> eight running sums over the multiples of 8, combined
 * ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), then the tail in order;
 * m > 128 -> split at m2 = m / 2 rounded down to a multiple of 8.  grid_distance
 * (plas.py:83) is np.sqrt((diff ** 2).sum(axis=1)).mean(): row sums over D,
 * then the mean over n in this order.  Compile without FMA contraction
 * (-ffp-contract=off). */
static double np_pairwise(const double *a, int64_t m) {
    if (m < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < m; i++) res += a[i];
        return res;
    }
    if (m <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i = 8;
        for (; i < m - (m % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < m; i++) res += a[i];
        return res;
    }
    int64_t m2 = m / 2;
    m2 -= m2 % 8;
    return np_pairwise(a, m2) + np_pairwise(a + m2, m - m2);
}

double oracle_grid_distance_f32(const float *a, const float *b, int64_t n, int D, int S) {
    double *cell = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *sq = (double *)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
    for (int64_t i = 0; i < n; i++) {
        for (int d = 0; d < D; d++) {
            double df = (double)a[i * S + d] - (double)b[i * S + d];
            sq[d] = df * df;
        }
        cell[i] = sqrt(np_pairwise(sq, D));
    }
    double mean = np_pairwise(cell, n) / (double)n;
    free(cell);
    free(sq);
    return mean;
}

double oracle_vad_f32(const float *g, int H, int W, int C, int S) {
    double n = 0.0, sum = 0.0;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++)
            for (int c = 0; c < C; c++) {
                double v = g[((size_t)y * W + x) * S + c];
                if (y + 1 < H) { sum += fabs((double)g[((size_t)(y + 1) * W + x) * S + c] - v); n += 1; }
                if (x + 1 < W) { sum += fabs((double)g[((size_t)y * W + x + 1) * S + c] - v); n += 1; }
            }
    double mean = sum / n, acc = 0.0;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++)
            for (int c = 0; c < C; c++) {
                double v = g[((size_t)y * W + x) * S + c];
                if (y + 1 < H) { double e = fabs((double)g[((size_t)(y + 1) * W + x) * S + c] - v) - mean; acc += e * e; }
                if (x + 1 < W) { double e = fabs((double)g[((size_t)y * W + x + 1) * S + c] - v) - mean; acc += e * e; }
            }
    return acc / n;
}

/* ------------------------------------------------------------------ */
/* _reassign_pass (plas.py:196-223) and _sort (plas.py:226-286)        */
/* ------------------------------------------------------------------ */
static int segments(int side, int beta, int delta, int *b0, int *b1) {
    int n = 0, prev = 0;
    int x = delta > 0 ? delta : beta;
    while (x < side) {
        b0[n] = prev; b1[n] = x; n++;
        prev = x;
        x += beta;
    }
    b0[n] = prev; b1[n] = side; n++;
    return n;
}

/* filtered master permutation per distinct block size m (memoised per pass) */
typedef struct { int64_t m; int64_t *sel; } sel_entry;

static void reassign_pass(float *feat, int64_t *idx, const float *target, int side, int D, int S,
                          int beta, int dy, int dx, const int64_t *mp, int64_t nmp) {
    int *ry0 = (int *)malloc(sizeof(int) * (side + 2) * 4);
    int *ry1 = ry0 + (side + 2), *rx0 = ry1 + (side + 2), *rx1 = rx0 + (side + 2);
    int ny = segments(side, beta, dy, ry0, ry1);
    int nx = segments(side, beta, dx, rx0, rx1);
    sel_entry cache[9];
    int ncache = 0;
    int64_t groups[4];
    for (int by = 0; by < ny; by++)
        for (int bx = 0; bx < nx; bx++) {
            int hh = ry1[by] - ry0[by], ww = rx1[bx] - rx0[bx];
            int64_t m = (int64_t)hh * ww;
            int64_t *sel = NULL;
            for (int c = 0; c < ncache; c++)
                if (cache[c].m == m) sel = cache[c].sel;
            if (!sel) {
                sel = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
                int64_t cnt = 0;
                for (int64_t i = 0; i < nmp; i++)
                    if (mp[i] < m) sel[cnt++] = mp[i];
                cache[ncache].m = m;
                cache[ncache].sel = sel;
                ncache++;
            }
            int64_t g4 = (m / 4) * 4;
            for (int64_t q = 0; q < g4; q += 4) {
                for (int s = 0; s < 4; s++) {
                    int64_t l = sel[q + s];
                    groups[s] = (int64_t)(ry0[by] + l / ww) * side + rx0[bx] + l % ww;
                }
                oracle_assign_groups(feat, idx, target, D, S, groups, 1, 4);
            }
            int rest = (int)(m - g4);
            if (rest >= 2) {
                for (int s = 0; s < rest; s++) {
                    int64_t l = sel[g4 + s];
                    groups[s] = (int64_t)(ry0[by] + l / ww) * side + rx0[bx] + l % ww;
                }
                oracle_assign_groups(feat, idx, target, D, S, groups, 1, rest);
            }
        }
    for (int c = 0; c < ncache; c++) free(cache[c].sel);
    free(ry0);
}

/*
 * Full sort (plas.py:226-286).  The schedule (radii by repeated fp64
 * multiplication, plas.py:246/274) and the per-level Gaussian weights (NumPy
 * exp, scipy _gaussian_kernel1d) are built by the caller: L levels, level l has
 * half-width hs[l] and weights w + woff[l] (hs[l]+1 values).
 * max_passes / max_seconds bound the run (0 = unbounded) so a bounded CPU
 * sample can be timed (checked before each pass); trace_cap bounds the trace.
 * Returns the number of passes executed, or -1 on trace overflow.
 */
int64_t oracle_sort(const double *features, int64_t n, int D, int64_t seed, double thr,
                    int min_block, int L, const double *radii, const int *hs,
                    const double *w, const int64_t *woff, const int64_t *init_perm,
                    int64_t max_passes, double max_seconds, int64_t *perm_out, int64_t *level_counts,
                    double *trace, int64_t trace_cap, double *vads, int64_t *levels_done) {
    int side = (int)llround(sqrt((double)n));
    int S = D;
    double t_start = now_s();
    oracle_rng rng;
    oracle_rng_init(&rng, (uint64_t)seed);
    int64_t *idx = perm_out;
    if (init_perm) {
        /* paired-protocol hook: the caller supplies draw #1 (plas.py:241) and the
           RNG state is advanced exactly as permutation(n) would have advanced it */
        int64_t *scratch = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
        oracle_rng_permutation(&rng, n, scratch);
        free(scratch);
        memcpy(idx, init_perm, sizeof(int64_t) * (size_t)n);
    } else {
        oracle_rng_permutation(&rng, n, idx);
    }
    float *feat = (float *)malloc(sizeof(float) * (size_t)n * S);
    float *target = (float *)malloc(sizeof(float) * (size_t)n * S);
    for (int64_t i = 0; i < n; i++)
        for (int d = 0; d < D; d++) feat[i * S + d] = (float)features[idx[i] * D + d];
    vads[0] = oracle_vad_f32(feat, side, side, D, S);
    int64_t passes = 0, tpos = 0;
    int64_t *mp = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int lv;
    int stopped = 0;
    for (lv = 0; lv < L && !stopped; lv++) {
        if (max_seconds > 0 && now_s() - t_start >= max_seconds) break;
        double radius = radii[lv];
        const double *wl = w + woff[lv];
        int h = hs[lv];
        oracle_blur_target_f32(feat, side, side, S, wl, h, target);
        int beta = (int)radius + 1;
        if (beta < min_block) beta = min_block;
        if (beta > side) beta = side;
        double previous = oracle_grid_distance_f32(feat, target, n, D, S);
        if (tpos >= trace_cap) return -1;
        trace[tpos++] = previous;
        int64_t count = 1;
        int strikes = 0;
        while (strikes < 2) {
            if ((max_passes > 0 && passes >= max_passes) ||
                (max_seconds > 0 && now_s() - t_start >= max_seconds)) { stopped = 1; break; }
            int dy = (int)oracle_rng_integers(&rng, beta);
            int dx = (int)oracle_rng_integers(&rng, beta);
            oracle_rng_permutation(&rng, (int64_t)beta * beta, mp);
            reassign_pass(feat, idx, target, side, D, S, beta, dy, dx, mp, (int64_t)beta * beta);
            passes++;
            double current = oracle_grid_distance_f32(feat, target, n, D, S);
            if (tpos >= trace_cap) return -1;
            trace[tpos++] = current;
            count++;
            if (previous <= 0.0 || (previous - current) / previous < thr) strikes++;
            else strikes = 0;
            previous = current;
        }
        level_counts[lv] = count;
    }
    *levels_done = lv;
    vads[1] = oracle_vad_f32(feat, side, side, D, S);
    free(mp);
    free(feat);
    free(target);
    return passes;
}

/* ------------------------------------------------------------------ */
/* smoothness_loss for one plane (smoothness.py:57-97)                 */
/* ------------------------------------------------------------------ */
/* plane (H, W, C) f64; coeff = overall_multiplier * weight; w/h as above with
 * sigma = params.sigma and h = kernel_size // 2 (h == 0 -> zero residual).
 * Returns the plane's loss contribution; writes grad (H, W, C). */
double oracle_smoothness_plane(const double *plane, int H, int W, int C, double coeff,
                               double delta, int detach, const double *w, int h, double *grad) {
    size_t n = (size_t)H * W * C;
    if (coeff == 0.0 || n == 0) {
        memset(grad, 0, sizeof(double) * n);
        return 0.0;
    }
    double *res = (double *)malloc(sizeof(double) * n);
    double *den = (double *)malloc(sizeof(double) * (size_t)H * W);
    if (h == 0) {
        for (size_t i = 0; i < n; i++) res[i] = 0.0;
    } else {
        oracle_border_weight(H, W, w, h, den);
        double *cen = (double *)malloc(sizeof(double) * n);
        double *bl = (double *)malloc(sizeof(double) * n);
        for (size_t i = 0; i < (size_t)H * W; i++)
            for (int c = 0; c < C; c++) cen[i * C + c] = plane[i * C + c] - plane[c];
        oracle_separable_blur_f64(cen, H, W, C, w, h, bl);
        for (size_t i = 0; i < (size_t)H * W; i++)
            for (int c = 0; c < C; c++) res[i * C + c] = cen[i * C + c] - bl[i * C + c] / den[i];
        free(cen);
        free(bl);
    }
    /* huber(residual).mean() (smoothness.py:88): elementwise values, then
     * NumPy's pairwise sum over the contiguous array and one division */
    double *hub = (double *)malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; i++) {
        double a = fabs(res[i]);
        hub[i] = a <= delta ? 0.5 * res[i] * res[i] : delta * (a - 0.5 * delta);
    }
    double loss = coeff * (np_pairwise(hub, (int64_t)n) / (double)n);
    free(hub);
    double scale = coeff / (double)n;
    for (size_t i = 0; i < n; i++) {
        double r = res[i];
        double cl = r < -delta ? -delta : (r > delta ? delta : r);
        grad[i] = scale * cl;
    }
    if (!(detach || h == 0)) {
        double *u = (double *)malloc(sizeof(double) * n);
        double *back = (double *)malloc(sizeof(double) * n);
        for (size_t i = 0; i < (size_t)H * W; i++)
            for (int c = 0; c < C; c++) u[i * C + c] = grad[i * C + c] / den[i];
        oracle_separable_blur_f64(u, H, W, C, w, h, back);
        for (size_t i = 0; i < n; i++) grad[i] = grad[i] - back[i];
        free(u);
        free(back);
    }
    free(res);
    free(den);
    return loss;
}
