/*
 * nfft_oracle.c -- CPU restatement of the reference NFFT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * library in paper_1810_09891_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product path never links or calls it.
 *
 * It restates, function by function, the algorithm of the reference package
 * `nfftk` (/root/reference/pkg/src/nfftk, pure Python + numba), citing the
 * file:line each routine follows.  The restatement is pinned against golden
 * vectors produced by the live reference (tests/golden/make_golden.py) in
 * tests/test_oracle_golden.py.
 *
 * Layout conventions (reference-defined):
 *   - spectral vectors f_hat: row-major over I_N, last dim fastest,
 *     k_i in [-N_i/2, N_i/2)                      (indexing.py:32-41)
 *   - oversampled grid: row-major over n, frequency k stored at slot k mod n,
 *     spatial cell l stored at slot l mod n        (transform.py:39-41,
 *                                                   kernels.py:47)
 *   - complex data: C99 double complex == interleaved (re, im) doubles.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define KAISER_BESSEL 0
#define GAUSSIAN 1
#define MODE_DIRECT 0
#define MODE_LUT 2
#define LUT_SIZE (1 << 14) /* plan.py:74 */

static int64_t floor_mod(int64_t a, int64_t n) {
    /* numba/Python `%` (kernels.py:47): result has the sign of n */
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

/* ---------------------------------------------------------------- window */

/* window.py:38-53 -- I0 power series, term-ratio cutoff 1e-16 */
double oracle_bessel_i0(double x) {
    double s = 1.0, t = 1.0, q = 0.25 * x * x;
    long j = 0;
    for (;;) {
        j += 1;
        t *= q / (double)(j * j);
        s += t;
        if (t < 1e-16 * s) return s;
    }
}

/* window.py:56-72 -- scalar window value at offset t */
double oracle_window_factor(int code, double t, double n_i, double m, double b_i) {
    if (code == KAISER_BESSEL) {
        double u = m * m - (n_i * t) * (n_i * t);
        if (u > 0.0) {
            double z = sqrt(u);
            return sinh(b_i * z) / (M_PI * z);
        }
        if (u < 0.0) {
            double z = sqrt(-u);
            return sin(b_i * z) / (M_PI * z);
        }
        return b_i / M_PI;
    }
    return exp(-(n_i * t) * (n_i * t) / b_i) / sqrt(M_PI * b_i);
}

/* window.py:101-111 -- shape parameter b_i from sigma_i = n_i / N_i */
double oracle_window_b(int code, int N_i, int n_i, int m) {
    double sigma = (double)n_i / (double)N_i;
    if (code == KAISER_BESSEL) return M_PI * (2.0 - 1.0 / sigma);
    return 2.0 * sigma * m / ((2.0 * sigma - 1.0) * M_PI);
}

/* window.py:142-164 -- phi_hat(k); returns <= 0 on degenerate input */
double oracle_phi_hat(int code, int k, int n_i, int m, double b_i) {
    if (code == KAISER_BESSEL) {
        double c = 2.0 * M_PI * k / n_i;
        double arg = b_i * b_i - c * c;
        if (arg < 0.0) return -1.0;
        return oracle_bessel_i0(m * sqrt(arg)) / n_i;
    }
    double c = M_PI * k / n_i;
    return exp(-b_i * c * c) / n_i;
}

/* kernels.py:75-82 -- equispaced window samples on [0, m/n_i] */
void oracle_build_lut(int code, double n_i, int m, double b_i, int size, double *out) {
    double h = (m / n_i) / size;
    for (int t = 0; t <= size; ++t) out[t] = oracle_window_factor(code, t * h, n_i, (double)m, b_i);
}

/* kernels.py:30-39 -- linear interpolation of |t| */
static double lut_factor(const double *row, int last, double step, double t) {
    double u = fabs(t) * step;
    int64_t idx = (int64_t)u;
    if (idx >= last) return row[last];
    double frac = u - (double)idx;
    return row[idx] + frac * (row[idx + 1] - row[idx]);
}

/* --------------------------------------------------------------- indexing */

/* indexing.py:114-124 -- lo = ceil(n x - m), width = floor(n x + m) - lo + 1 */
void oracle_node_ranges(int d, const int *n, int m, int64_t M, const double *x,
                        int64_t *lo, int64_t *width) {
    for (int64_t j = 0; j < M; ++j)
        for (int i = 0; i < d; ++i) {
            double y = x[j * d + i] * (double)n[i];
            int64_t l = (int64_t)ceil(y - m);
            lo[j * d + i] = l;
            width[j * d + i] = (int64_t)floor(y + m) - l + 1;
        }
}

/* ------------------------------------------------------------------- FFT */

/* fft.py:33-77 -- iterative radix-2 with bit reversal, unnormalised */
static void fft_pow2(cplx *a, int64_t n, int sign, const cplx *tw) {
    /* tw: concatenated stage twiddles exp(sign 2 pi i k / (2 half)), k < half */
    int bits = 0;
    while (((int64_t)1 << bits) < n) ++bits;
    for (int64_t i = 0; i < n; ++i) {
        int64_t r = 0, v = i;
        for (int b = 0; b < bits; ++b) { r = (r << 1) | (v & 1); v >>= 1; }
        if (r > i) { cplx t = a[i]; a[i] = a[r]; a[r] = t; }
    }
    const cplx *w = tw;
    for (int64_t half = 1; half < n; half *= 2) {
        for (int64_t blk = 0; blk < n; blk += 2 * half)
            for (int64_t k = 0; k < half; ++k) {
                cplx t = a[blk + half + k] * w[k];
                cplx hi = a[blk + k] - t;
                a[blk + k] += t;
                a[blk + half + k] = hi;
            }
        w += half;
    }
    (void)sign;
}

static cplx *pow2_twiddles(int64_t n, int sign) {
    cplx *tw = (cplx *)malloc(sizeof(cplx) * (size_t)(n > 1 ? n : 1));
    int64_t off = 0;
    for (int64_t half = 1; half < n; half *= 2) {
        for (int64_t k = 0; k < half; ++k) {
            double ang = sign * 2.0 * M_PI * (double)k / (double)(2 * half);
            tw[off + k] = cos(ang) + I * sin(ang);
        }
        off += half;
    }
    return tw;
}

typedef struct {
    int64_t n, L;
    int sign;
    int pow2;
    cplx *tw;      /* twiddles for length n (pow2) or L (Bluestein, sign -1) */
    cplx *tw_pos;  /* Bluestein: twiddles for L, sign +1 */
    cplx *chirp;   /* fft.py:80-102 */
    cplx *bhat;
} fft_plan1d;

static fft_plan1d make_plan1d(int64_t n, int sign) {
    fft_plan1d p;
    memset(&p, 0, sizeof(p));
    p.n = n;
    p.sign = sign;
    p.pow2 = (n & (n - 1)) == 0;
    if (p.pow2) {
        p.tw = pow2_twiddles(n, sign);
        return p;
    }
    /* fft.py:80-102 -- Bluestein tables */
    int64_t L = 1;
    while (L < 2 * n - 1) L *= 2;
    p.L = L;
    p.tw = pow2_twiddles(L, -1);
    p.tw_pos = pow2_twiddles(L, +1);
    p.chirp = (cplx *)malloc(sizeof(cplx) * n);
    p.bhat = (cplx *)calloc((size_t)L, sizeof(cplx));
    for (int64_t k = 0; k < n; ++k) {
        int64_t q = (k * k) % (2 * n);
        double ang = sign * M_PI * (double)q / (double)n;
        p.chirp[k] = cos(ang) + I * sin(ang);
    }
    for (int64_t k = 0; k < n; ++k) p.bhat[k] = conj(p.chirp[k]);
    for (int64_t k = 1; k < n; ++k) p.bhat[L - k] = conj(p.chirp[k]);
    fft_pow2(p.bhat, L, -1, p.tw);
    return p;
}

static void free_plan1d(fft_plan1d *p) {
    free(p->tw); free(p->tw_pos); free(p->chirp); free(p->bhat);
}

/* fft.py:105-124 -- one line, in place; scratch >= L entries for Bluestein */
static void fft_line(const fft_plan1d *p, cplx *v, cplx *scratch) {
    if (p->n == 1) return;
    if (p->pow2) { fft_pow2(v, p->n, p->sign, p->tw); return; }
    int64_t n = p->n, L = p->L;
    memset(scratch, 0, sizeof(cplx) * (size_t)L);
    for (int64_t k = 0; k < n; ++k) scratch[k] = v[k] * p->chirp[k];
    fft_pow2(scratch, L, -1, p->tw);
    for (int64_t k = 0; k < L; ++k) scratch[k] *= p->bhat[k];
    fft_pow2(scratch, L, +1, p->tw_pos);
    for (int64_t k = 0; k < n; ++k) v[k] = (scratch[k] / (double)L) * p->chirp[k];
}

/* fft.py:127-139 -- separable nd transform, axes 0..d-1, in place */
void oracle_fft_nd(int d, const int *n, cplx *data, int sign) {
    int64_t total = 1;
    for (int i = 0; i < d; ++i) total *= n[i];
    for (int axis = 0; axis < d; ++axis) {
        int64_t len = n[axis], inner = 1;
        for (int i = axis + 1; i < d; ++i) inner *= n[i];
        int64_t outer = total / (len * inner);
        fft_plan1d p = make_plan1d(len, sign);
        int64_t lines = outer * inner;
        /* lines along a strided axis are moved in blocks of LB neighbours
         * (LB contiguous elements per step instead of one): the same 1-D
         * transforms, cache-friendly gathers */
        int64_t LB = 16;
        while (inner % LB) LB /= 2;
        const int64_t blocks = outer * (inner / LB);
        (void)lines;
#pragma omp parallel
        {
            int64_t sl = p.pow2 ? len : p.L;
            cplx *buf = (cplx *)malloc(sizeof(cplx) * (size_t)(len * LB));
            cplx *scr = (cplx *)malloc(sizeof(cplx) * (size_t)sl);
#pragma omp for schedule(static)
            for (int64_t bi = 0; bi < blocks; ++bi) {
                int64_t o = bi / (inner / LB), in0 = (bi % (inner / LB)) * LB;
                cplx *base = data + o * len * inner + in0;
                for (int64_t k = 0; k < len; ++k)
                    for (int64_t u = 0; u < LB; ++u) buf[u * len + k] = base[k * inner + u];
                for (int64_t u = 0; u < LB; ++u) fft_line(&p, buf + u * len, scr);
                for (int64_t k = 0; k < len; ++k)
                    for (int64_t u = 0; u < LB; ++u) base[k * inner + u] = buf[u * len + k];
            }
            free(buf);
            free(scr);
        }
        free_plan1d(&p);
    }
}

/* ------------------------------------------------------------ transforms */

typedef struct {
    int d;
    int N[3], n[3];
    int m, code, mode;
    double b[3];
    double *lut;      /* d * (LUT_SIZE+1) when mode == MODE_LUT */
    double lut_step[3];
} oplan;

static int setup(oplan *p, int d, const int *N, const int *n, int m, int code, int mode) {
    if (d < 1 || d > 3) return -1;
    p->d = d; p->m = m; p->code = code; p->mode = mode; p->lut = NULL;
    for (int i = 0; i < d; ++i) {
        p->N[i] = N[i]; p->n[i] = n[i];
        p->b[i] = oracle_window_b(code, N[i], n[i], m);
    }
    if (mode == MODE_LUT) {
        /* plan.py:285-295 */
        p->lut = (double *)malloc(sizeof(double) * d * (LUT_SIZE + 1));
        for (int i = 0; i < d; ++i) {
            oracle_build_lut(code, (double)n[i], m, p->b[i], LUT_SIZE, p->lut + i * (LUT_SIZE + 1));
            p->lut_step[i] = LUT_SIZE / ((double)m / n[i]);
        }
    }
    return 0;
}

/* kernels.py:42-53 -- the factors of node j, dim i at cells lo .. lo+w-1 */
static int dim_factors(const oplan *p, const double *x, int64_t j, int i, int64_t *lo_out, double *fac) {
    double n_i = (double)p->n[i];
    double y = x[j * p->d + i] * n_i;
    int64_t lo = (int64_t)ceil(y - p->m);
    int w = (int)((int64_t)floor(y + p->m) - lo + 1);
    for (int t = 0; t < w; ++t) {
        int64_t cell = lo + t;
        double off = x[j * p->d + i] - (double)cell / n_i;
        if (p->mode == MODE_LUT)
            fac[t] = lut_factor(p->lut + i * (LUT_SIZE + 1), LUT_SIZE, p->lut_step[i], off);
        else
            fac[t] = oracle_window_factor(p->code, off, n_i, (double)p->m, p->b[i]);
    }
    *lo_out = lo;
    return w;
}

/* transform.py:44-54 -- per-dim factors over k = -N/2..N/2-1 */
static double **deconv_cols(const oplan *p) {
    double **cols = (double **)malloc(sizeof(double *) * p->d);
    for (int i = 0; i < p->d; ++i) {
        cols[i] = (double *)malloc(sizeof(double) * p->N[i]);
        for (int k = -p->N[i] / 2; k < p->N[i] / 2; ++k)
            cols[i][k + p->N[i] / 2] = oracle_phi_hat(p->code, k, p->n[i], p->m, p->b[i]);
    }
    return cols;
}

static void free_cols(const oplan *p, double **cols) {
    for (int i = 0; i < p->d; ++i) free(cols[i]);
    free(cols);
}

/* transform.py:57-63 division order: /|I_n| first, then each dim's column */
static inline cplx deconv_value(const oplan *p, double **cols, cplx v, const int *kk, double grid_size) {
    cplx out = v / grid_size;
    for (int i = 0; i < p->d; ++i) out = out / cols[i][kk[i]];
    return out;
}

static int64_t grid_total(const oplan *p) {
    int64_t t = 1;
    for (int i = 0; i < p->d; ++i) t *= p->n[i];
    return t;
}

static int64_t freq_total(const oplan *p) {
    int64_t t = 1;
    for (int i = 0; i < p->d; ++i) t *= p->N[i];
    return t;
}

/* linear f_hat index -> grid slot (transform.py:39-41) */
static int64_t freq_slot(const oplan *p, int64_t lin, int *kk) {
    int64_t slot = 0, stride = 1, rem = lin;
    int64_t slots[3];
    for (int i = p->d - 1; i >= 0; --i) {
        int64_t ki = rem % p->N[i];
        rem /= p->N[i];
        kk[i] = (int)ki;
        slots[i] = floor_mod(ki - p->N[i] / 2, p->n[i]);
    }
    for (int i = p->d - 1; i >= 0; --i) { slot += slots[i] * stride; stride *= p->n[i]; }
    return slot;
}

/* ------------------------------------------------------ lexicographic order */

/* Stable LSD radix sort of (key, idx) pairs, 8-bit digits, OpenMP histograms.
 * Ties keep index order, so sorting (key, 0..M-1) reproduces np.lexsort. */
static void sort_pairs(uint64_t *key, int64_t *idx, int64_t M, int bits) {
    uint64_t *k2 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(M > 0 ? M : 1));
    int64_t *i2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M > 0 ? M : 1));
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * 256 * (size_t)nt);
    for (int shift = 0; shift < bits; shift += 8) {
        memset(hist, 0, sizeof(int64_t) * 256 * (size_t)nt);
#pragma omp parallel num_threads(nt)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            int64_t lo = M * t / nt, hi = M * (t + 1) / nt;
            int64_t *h = hist + 256 * t;
            for (int64_t q = lo; q < hi; ++q) h[(key[q] >> shift) & 255]++;
#pragma omp barrier
#pragma omp single
            {
                int64_t run = 0;
                for (int digit = 0; digit < 256; ++digit)
                    for (int u = 0; u < nt; ++u) {
                        int64_t c = hist[256 * u + digit];
                        hist[256 * u + digit] = run;
                        run += c;
                    }
            }
            for (int64_t q = lo; q < hi; ++q) {
                int64_t pos = h[(key[q] >> shift) & 255]++;
                k2[pos] = key[q];
                i2[pos] = idx[q];
            }
        }
        memcpy(key, k2, sizeof(uint64_t) * (size_t)M);
        memcpy(idx, i2, sizeof(int64_t) * (size_t)M);
    }
    free(hist);
    free(k2);
    free(i2);
}

/* plan.py:228-231 -- lexsort of floor(n x), dim 0 primary, stable */
void oracle_node_order(int d, const int *n, int64_t M, const double *x, int64_t *order) {
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(M > 0 ? M : 1));
    uint64_t space = 1;
    for (int i = 0; i < d; ++i) space *= (uint64_t)(n[i] + 1);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < M; ++j) {
        uint64_t k = 0;
        for (int i = 0; i < d; ++i)
            k = k * (uint64_t)(n[i] + 1) + (uint64_t)((int64_t)floor(x[j * d + i] * (double)n[i]) + n[i] / 2);
        key[j] = k;
        order[j] = j;
    }
    int bits = 1;
    while (bits < 64 && ((uint64_t)1 << bits) < space) ++bits;
    sort_pairs(key, order, M, bits);
    free(key);
}

/* ------------------------------------------------------------------ plan */

/* The reference plan's node state and tables (plan.py:202-299): stencil
 * starts and widths (node_ranges, indexing.py:114-124), the lexicographic
 * node order (NFFT_SORT_NODES), and the factor table psi (M, d, 2m+1) --
 * PRE_PSI, kernels.py:56-72; in LUT mode the table holds the interpolated
 * factors, the values kernels.py:30-39 forms per use.  Building them is the
 * reference's set_nodes + precompute; trafo / adjoint then only read them, as
 * the reference's transforms do under its default flags. */
typedef struct {
    oplan p;
    int64_t M;
    int K;
    double *x;        /* (M, d) */
    int64_t *lo;      /* (M, d) */
    int *width;       /* (M, d) */
    double *psi;      /* (M, d, K) */
    int64_t *order;   /* lexicographic order */
    char *wraps;      /* per sorted position: dim-0 rows wrap (transform.py:144-158) */
} oracle_plan;

void oracle_plan_destroy(void *h) {
    oracle_plan *q = (oracle_plan *)h;
    if (!q) return;
    free(q->x); free(q->lo); free(q->width); free(q->psi); free(q->order); free(q->wraps);
    free(q->p.lut);
    free(q);
}

void *oracle_plan_create(int d, const int *N, const int *n, int m, int code, int mode, int64_t M,
                         const double *x) {
    oracle_plan *q = (oracle_plan *)calloc(1, sizeof(oracle_plan));
    if (!q || setup(&q->p, d, N, n, m, code, mode)) { free(q); return NULL; }
    q->M = M;
    q->K = 2 * m + 1;
    size_t nd = (size_t)(M > 0 ? M : 1) * d;
    q->x = (double *)malloc(sizeof(double) * nd);
    q->lo = (int64_t *)malloc(sizeof(int64_t) * nd);
    q->width = (int *)malloc(sizeof(int) * nd);
    q->psi = (double *)malloc(sizeof(double) * nd * q->K);
    q->order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(M > 0 ? M : 1));
    q->wraps = (char *)malloc((size_t)(M > 0 ? M : 1));
    if (!q->x || !q->lo || !q->width || !q->psi || !q->order || !q->wraps) {
        oracle_plan_destroy(q);
        return NULL;
    }
    memcpy(q->x, x, sizeof(double) * (size_t)M * d);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < M; ++j)
        for (int i = 0; i < d; ++i) {
            double *row = q->psi + ((size_t)j * d + i) * q->K;
            int64_t lo;
            int w = dim_factors(&q->p, q->x, j, i, &lo, row);
            for (int t = w; t < q->K; ++t) row[t] = 0.0;
            q->lo[(size_t)j * d + i] = lo;
            q->width[(size_t)j * d + i] = w;
        }
    oracle_node_order(d, n, M, q->x, q->order);
    for (int64_t oi = 0; oi < M; ++oi) {
        size_t j = (size_t)q->order[oi] * d;
        q->wraps[oi] = floor_mod(q->lo[j], n[0]) + q->width[j] > n[0];
    }
    return q;
}

/* Software prefetch of the grid rows node j's stencil reads (d >= 2): the
 * natural-order gather of the reference touches a fresh, random part of the
 * grid per node, so the port issues the next nodes' row loads ahead (the
 * arithmetic and its order are unchanged). */
#define GATHER_AHEAD 4
static inline void prefetch_rows(const oracle_plan *q, const cplx *g, int64_t j) {
    if (j >= q->M) return;
    const int d = q->p.d;
    const int64_t n0 = q->p.n[0], n1 = q->p.n[1], n2 = q->p.n[2];
    const int64_t *lo = q->lo + (size_t)j * d;
    const int *W = q->width + (size_t)j * d;
    if (d == 2) {
        int64_t c1 = floor_mod(lo[1], n1);
        for (int t0 = 0; t0 < W[0]; ++t0) {
            const cplx *r = g + floor_mod(lo[0] + t0, n0) * n1 + c1;
            __builtin_prefetch(r);
            __builtin_prefetch(r + W[1] - 1);
        }
    } else if (d == 3) {
        int64_t c2 = floor_mod(lo[2], n2);
        for (int t0 = 0; t0 < W[0]; ++t0) {
            int64_t b0 = floor_mod(lo[0] + t0, n0) * n1;
            for (int t1 = 0; t1 < W[1]; ++t1) {
                const cplx *r = g + (b0 + floor_mod(lo[1] + t1, n1)) * n2 + c2;
                __builtin_prefetch(r);
                __builtin_prefetch(r + W[2] - 1);
            }
        }
    }
}

/* kernels.py:122-197 -- B: prange over nodes in natural order, lexicographic
 * accumulation ((p0 * f1) * f2) * g */
int oracle_plan_gather_grid(void *h, const cplx *g, cplx *f) {
    const oracle_plan *q = (const oracle_plan *)h;
    const int d = q->p.d, K = q->K;
    const int64_t n0 = q->p.n[0], n1 = q->p.n[1], n2 = q->p.n[2];
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < q->M; ++j) {
        prefetch_rows(q, g, j + GATHER_AHEAD);
        const double *f0 = q->psi + (size_t)j * d * K;
        const int64_t *lo = q->lo + (size_t)j * d;
        const int *W = q->width + (size_t)j * d;
        cplx acc = 0.0;
        if (d == 1) {
            for (int t0 = 0; t0 < W[0]; ++t0) acc += f0[t0] * g[floor_mod(lo[0] + t0, n0)];
        } else if (d == 2) {
            const double *f1 = f0 + K;
            int64_t w1[64];
            for (int t1 = 0; t1 < W[1]; ++t1) w1[t1] = floor_mod(lo[1] + t1, n1);
            for (int t0 = 0; t0 < W[0]; ++t0) {
                int64_t base = floor_mod(lo[0] + t0, n0) * n1;
                double p0 = f0[t0];
                for (int t1 = 0; t1 < W[1]; ++t1) acc += (p0 * f1[t1]) * g[base + w1[t1]];
            }
        } else {
            const double *f1 = f0 + K, *f2 = f0 + 2 * K;
            int64_t w1[64], w2[64];
            for (int t1 = 0; t1 < W[1]; ++t1) w1[t1] = floor_mod(lo[1] + t1, n1);
            for (int t2 = 0; t2 < W[2]; ++t2) w2[t2] = floor_mod(lo[2] + t2, n2);
            for (int t0 = 0; t0 < W[0]; ++t0) {
                int64_t base0 = floor_mod(lo[0] + t0, n0) * n1;
                double p0 = f0[t0];
                for (int t1 = 0; t1 < W[1]; ++t1) {
                    int64_t base1 = (base0 + w1[t1]) * n2;
                    double p01 = p0 * f1[t1];
                    for (int t2 = 0; t2 < W[2]; ++t2) acc += (p01 * f2[t2]) * g[base1 + w2[t2]];
                }
            }
        }
        f[j] = acc;
    }
    return 0;
}

/* transform.py:92-118 -- f = B F D f_hat */
int oracle_plan_trafo(void *h, const cplx *fhat, cplx *f) {
    const oracle_plan *q = (const oracle_plan *)h;
    const oplan *p = &q->p;
    int64_t G = grid_total(p), K = freq_total(p);
    cplx *g = (cplx *)calloc((size_t)G, sizeof(cplx));
    if (!g) return -2;
    double **cols = deconv_cols(p);
    double gs = (double)G;
#pragma omp parallel for schedule(static)
    for (int64_t lin = 0; lin < K; ++lin) {
        int kk[3];
        int64_t slot = freq_slot(p, lin, kk);
        g[slot] = deconv_value(p, cols, fhat[lin], kk, gs);
    }
    free_cols(p, cols);
    oracle_fft_nd(p->d, p->n, g, -1);
    oracle_plan_gather_grid(h, g, f);
    free(g);
    return 0;
}

/* kernels.py:209-281 -- spread one node (all rows, or rows [s_lo, s_hi) of dim 0) */
static void spread_node(const oracle_plan *q, int64_t j, cplx fj, cplx *g,
                        int restrict_rows, int64_t s_lo, int64_t s_hi) {
    const int d = q->p.d, K = q->K;
    const int64_t n0 = q->p.n[0], n1 = q->p.n[1], n2 = q->p.n[2];
    const double *f0 = q->psi + (size_t)j * d * K;
    const int64_t *lo = q->lo + (size_t)j * d;
    const int *W = q->width + (size_t)j * d;
    int t_begin = 0, t_end = W[0];
    if (restrict_rows) {
        /* kernels.py:304-312 -- slab-owned rows of a non-wrapping node */
        int64_t a0 = floor_mod(lo[0], n0);
        t_begin = s_lo > a0 ? (int)(s_lo - a0) : 0;
        int64_t row_end = a0 + W[0] < s_hi ? a0 + W[0] : s_hi;
        t_end = (int)(row_end - a0);
        if (t_begin >= t_end) return;
    }
    if (d == 1) {
        for (int t0 = t_begin; t0 < t_end; ++t0) g[floor_mod(lo[0] + t0, n0)] += fj * f0[t0];
        return;
    }
    const double *f1 = f0 + K;
    int64_t w1[64];
    for (int t1 = 0; t1 < W[1]; ++t1) w1[t1] = floor_mod(lo[1] + t1, n1);
    if (d == 2) {
        for (int t0 = t_begin; t0 < t_end; ++t0) {
            int64_t base = floor_mod(lo[0] + t0, n0) * n1;
            double p0 = f0[t0];
            for (int t1 = 0; t1 < W[1]; ++t1) g[base + w1[t1]] += fj * (p0 * f1[t1]);
        }
        return;
    }
    const double *f2 = f0 + 2 * K;
    int64_t w2[64];
    for (int t2 = 0; t2 < W[2]; ++t2) w2[t2] = floor_mod(lo[2] + t2, n2);
    for (int t0 = t_begin; t0 < t_end; ++t0) {
        int64_t base0 = floor_mod(lo[0] + t0, n0) * n1;
        double p0 = f0[t0];
        for (int t1 = 0; t1 < W[1]; ++t1) {
            int64_t base1 = (base0 + w1[t1]) * n2;
            double p01 = p0 * f1[t1];
            for (int t2 = 0; t2 < W[2]; ++t2) g[base1 + w2[t2]] += fj * (p01 * f2[t2]);
        }
    }
}

/* transform.py:121-171 -- B^H only: the oversampled grid after spreading
 * (before the FFT).  blockwise != 0 restates the slab-owned parallel adjoint
 * (kernels.py:293-401, transform.py:144-158): slab s owns dim-0 rows
 * [n0 s/P, n0 (s+1)/P), every slab walks all sorted nodes, nodes whose rows
 * wrap go to a sequential epilogue; otherwise the sequential natural-order
 * spread (transform.py:159-171).  nthreads <= 0 uses the OpenMP default. */
int oracle_plan_spread_grid(void *h, const cplx *f, cplx *g, int blockwise, int nthreads) {
    const oracle_plan *q = (const oracle_plan *)h;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    int64_t G = grid_total(&q->p);
    memset(g, 0, sizeof(cplx) * (size_t)G);
    const int64_t M = q->M;
    if (blockwise && nthreads > 1) {
        int64_t n0 = q->p.n[0];
#pragma omp parallel for num_threads(nthreads) schedule(static, 1)
        for (int s = 0; s < nthreads; ++s) {
            int64_t s_lo = (n0 * s) / nthreads, s_hi = (n0 * (s + 1)) / nthreads;
            for (int64_t oi = 0; oi < M; ++oi) {
                if (q->wraps[oi]) continue;
                spread_node(q, q->order[oi], f[q->order[oi]], g, 1, s_lo, s_hi);
            }
        }
        for (int64_t oi = 0; oi < M; ++oi)
            if (q->wraps[oi]) spread_node(q, q->order[oi], f[q->order[oi]], g, 0, 0, 0);
    } else {
        for (int64_t j = 0; j < M; ++j) spread_node(q, j, f[j], g, 0, 0, 0);
    }
    return 0;
}

/* transform.py:174-176 -- F^H (sign +1) and D^H of a spread grid (in place) */
static int adjoint_finish_p(const oplan *p, cplx *g, cplx *fhat) {
    int64_t G = grid_total(p), K = freq_total(p);
    oracle_fft_nd(p->d, p->n, g, +1);
    double **cols = deconv_cols(p);
    double gs = (double)G;
#pragma omp parallel for schedule(static)
    for (int64_t lin = 0; lin < K; ++lin) {
        int kk[3];
        int64_t slot = freq_slot(p, lin, kk);
        fhat[lin] = deconv_value(p, cols, g[slot], kk, gs);
    }
    free_cols(p, cols);
    return 0;
}

int oracle_adjoint_finish(int d, const int *N, const int *n, int m, int code, cplx *g, cplx *fhat) {
    oplan p;
    if (setup(&p, d, N, n, m, code, MODE_DIRECT)) return -1;
    return adjoint_finish_p(&p, g, fhat);
}

/* transform.py:121-176 -- f_hat = D^H F^H B^H f */
int oracle_plan_adjoint(void *h, const cplx *f, cplx *fhat, int blockwise, int nthreads) {
    const oracle_plan *q = (const oracle_plan *)h;
    cplx *g = (cplx *)malloc(sizeof(cplx) * (size_t)grid_total(&q->p));
    if (!g) return -2;
    oracle_plan_spread_grid(h, f, g, blockwise, nthreads);
    int rc = adjoint_finish_p(&q->p, g, fhat);
    free(g);
    return rc;
}

/* one-shot forms: plan, transform, release */
int oracle_trafo(int d, const int *N, const int *n, int m, int code, int mode, int64_t M,
                 const double *x, const cplx *fhat, cplx *f) {
    void *h = oracle_plan_create(d, N, n, m, code, mode, M, x);
    if (!h) return -1;
    int rc = oracle_plan_trafo(h, fhat, f);
    oracle_plan_destroy(h);
    return rc;
}

int oracle_gather_grid(int d, const int *N, const int *n, int m, int code, int mode, int64_t M,
                       const double *x, const cplx *g, cplx *f) {
    void *h = oracle_plan_create(d, N, n, m, code, mode, M, x);
    if (!h) return -1;
    int rc = oracle_plan_gather_grid(h, g, f);
    oracle_plan_destroy(h);
    return rc;
}

int oracle_spread_grid(int d, const int *N, const int *n, int m, int code, int mode, int64_t M,
                       const double *x, const cplx *f, cplx *g, int blockwise, int nthreads) {
    void *h = oracle_plan_create(d, N, n, m, code, mode, M, x);
    if (!h) return -1;
    int rc = oracle_plan_spread_grid(h, f, g, blockwise, nthreads);
    oracle_plan_destroy(h);
    return rc;
}

int oracle_adjoint(int d, const int *N, const int *n, int m, int code, int mode, int64_t M,
                   const double *x, const cplx *f, cplx *fhat, int blockwise, int nthreads) {
    void *h = oracle_plan_create(d, N, n, m, code, mode, M, x);
    if (!h) return -1;
    int rc = oracle_plan_adjoint(h, f, fhat, blockwise, nthreads);
    oracle_plan_destroy(h);
    return rc;
}

/* transform.py:188-203 -- exact forward sums sum_k f_hat_k e^{-2 pi i k.x_j} */
int oracle_ndft(int d, const int *N, int64_t M, const double *x, const cplx *fhat, cplx *f) {
    if (d < 1 || d > 3) return -1;
    int64_t K = 1;
    for (int i = 0; i < d; ++i) K *= N[i];
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t j = 0; j < M; ++j) {
        cplx *ph[3];
        for (int i = 0; i < d; ++i) {
            ph[i] = (cplx *)malloc(sizeof(cplx) * N[i]);
            for (int k = 0; k < N[i]; ++k) {
                double ang = -2.0 * M_PI * (double)(k - N[i] / 2) * x[j * d + i];
                ph[i][k] = cos(ang) + I * sin(ang);
            }
        }
        cplx acc = 0.0;
        for (int64_t lin = 0; lin < K; ++lin) {
            int64_t rem = lin;
            cplx e = 1.0;
            for (int i = d - 1; i >= 0; --i) { e *= ph[i][rem % N[i]]; rem /= N[i]; }
            acc += fhat[lin] * e;
        }
        f[j] = acc;
        for (int i = 0; i < d; ++i) free(ph[i]);
    }
    return 0;
}

/* transform.py:206-234 -- exact adjoint sums sum_j f_j e^{+2 pi i k.x_j} */
int oracle_ndft_adjoint(int d, const int *N, int64_t M, const double *x, const cplx *f, cplx *fhat) {
    if (d < 1 || d > 3) return -1;
    int64_t K = 1;
    for (int i = 0; i < d; ++i) K *= N[i];
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t lin = 0; lin < K; ++lin) {
        int kk[3];
        int64_t rem = lin;
        for (int i = d - 1; i >= 0; --i) { kk[i] = (int)(rem % N[i]) - N[i] / 2; rem /= N[i]; }
        cplx acc = 0.0;
        for (int64_t j = 0; j < M; ++j) {
            double ang = 0.0;
            for (int i = 0; i < d; ++i) ang += 2.0 * M_PI * (double)kk[i] * x[j * d + i];
            acc += f[j] * (cos(ang) + I * sin(ang));
        }
        fhat[lin] = acc;
    }
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count for the following parallel regions (torchrun exports
 * OMP_NUM_THREADS=1 to every rank; the CPU baseline wants the host's cores). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
