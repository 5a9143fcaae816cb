/*
 * oracle/stap_oracle.c -- fp64 CPU oracle for the STAP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link,
 * load or execute this file: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg use it.  It shares no code,
 * header, table or constant with paper_2203_06233_b200/ (the CUDA path).
 *
 * What it computes (algorithm c.1; the paper never states the STAP
 * mathematics, so every convention below is a DESIGN.md "reading"):
 *   - the datacube: pulses x channels x samples per pulse
 *     (sec. 5.3 "Multi-node Results (STAP)"), taken after the
 *     per-row Doppler FFT (Table 2 "fft_2D,axis=1"; PAPER.md:420-430
 *     Fig. 7 text) as X[D][C][R] complex (readings c-1, c-14);
 *   - independent outer units fused into one parallel loop (PAPER.md:420-430,
 *     408-418): here, one unit = (Doppler bin d, training block b);
 *   - the three stages named by BASELINE.json north_star: covariance with
 *     diagonal loading, batched Hermitian Cholesky + forward/back solves giving
 *     MVDR weights with the normalising inner products, and application of
 *     the weights to every range cell.
 *
 * Every sum is a sequential fp64 sum in ascending index order.  Complex values
 * are explicit (re, im) pairs of doubles (no C99 complex: no __muldc3 NaN
 * handling, no reordering).  Compiled -O2 -ffp-contract=off, no fast-math.
 *
 * Readings used (ids as in DESIGN.md / SURVEY.md c.3):
 *   c-2 window start d-h, h = floor((T-1)/2);  c-3 circular wrap mod D;
 *   c-4 snapshot element i = t*C + c;          c-5 Rhat = (1/K) sum z z^H;
 *   c-6 delta = lambda * tr(Rhat) / N;          c-7 non-overlapping blocks of K;
 *   c-9 MVDR w = R^-1 s / (s^H R^-1 s);         c-10 gamma = ||L^-1 s||^2;
 *   c-11 LAPACK-potrf-style info, zeroed outputs; c-12 Y = w^H z;
 *   c-13 one steering set [S][N] used as given.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_pins.py
 * (closed forms E1/E2/E3, Sherman-Morrison, invariances, explicit-inverse and
 * exact-rational special cases).  Nothing here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t n_chan;          /* C */
    int32_t tdof;            /* T */
    int32_t n_dop;           /* D (global) */
    int32_t n_range;         /* R */
    int32_t training_block;  /* K */
    int32_t n_steering;      /* S */
    double  diag_load;       /* lambda */
    int32_t dop_begin;       /* first owned bin */
    int32_t dop_count;       /* owned bins */
    int32_t cube_bin0;       /* global bin held in row 0 of the cube buffer */
    int32_t cube_bins;       /* bins held by the cube buffer */
} stap_oracle_params;

enum { OR_OK = 0, OR_BAD = 2, OR_NOMEM = 8 };

static int64_t mod_nonneg(int64_t a, int64_t m) {
    int64_t r = a % m;
    return r < 0 ? r + m : r;
}

static int check_params(const stap_oracle_params* p) {
    if (!p) return OR_BAD;
    if (p->n_chan <= 0 || p->tdof <= 0 || p->n_dop <= 0 || p->n_range <= 0 ||
        p->training_block <= 0 || p->n_steering <= 0) return OR_BAD;
    if (p->n_range % p->training_block) return OR_BAD;
    if (p->tdof > p->n_dop) return OR_BAD;
    if (!(p->diag_load >= 0.0) || !isfinite(p->diag_load)) return OR_BAD;
    if (p->dop_begin < 0 || p->dop_count < 0 || p->dop_begin + p->dop_count > p->n_dop) return OR_BAD;
    if (p->cube_bins <= 0 || p->cube_bins > p->n_dop) return OR_BAD;
    if (p->cube_bin0 < 0 || p->cube_bin0 >= p->n_dop) return OR_BAD;
    return OR_OK;
}

/* Cube row of global bin a (the cube buffer holds bins cube_bin0 .. +cube_bins, wrapping mod D). */
static int64_t cube_row(const stap_oracle_params* p, int64_t a) {
    int64_t loc = mod_nonneg(a - p->cube_bin0, p->n_dop);
    return loc < p->cube_bins ? loc : -1;
}

/* Step 1 (c.1): snapshots Z[i][j] = X[(d-h+t) mod D][c][b*K+j], i = t*C + c.
 * Z is N*K complex, row-major [i][j], (re, im) interleaved. Returns -1 if the
 * cube buffer does not hold a needed bin. */
static int snapshots(const stap_oracle_params* p, const float* cube, int d, int b, double* Z) {
    const int C = p->n_chan, T = p->tdof, K = p->training_block, R = p->n_range;
    const int h = (T - 1) / 2;
    for (int t = 0; t < T; ++t) {
        int64_t a = mod_nonneg((int64_t)d - h + t, p->n_dop);
        int64_t row = cube_row(p, a);
        if (row < 0) return -1;
        for (int c = 0; c < C; ++c) {
            const float* src = cube + 2 * (((row * C) + c) * (int64_t)R + (int64_t)b * K);
            double* dst = Z + 2 * ((int64_t)(t * C + c) * K);
            for (int j = 0; j < K; ++j) {
                dst[2 * j]     = (double)src[2 * j];
                dst[2 * j + 1] = (double)src[2 * j + 1];
            }
        }
    }
    return 0;
}

/* Steps 2-3 (c.1): Rhat[i][l] = (1/K) sum_j Z[i][j] conj(Z[l][j]) for i <= l, mirrored;
 * Im Rhat[i][i] = 0; delta = lambda * tr(Rhat) / N; Rm = Rhat + delta I.
 * Rm is N*N complex row-major. Returns delta. */
static double covariance_loaded(int N, int K, double lambda, const double* Z, double* Rm) {
    for (int i = 0; i < N; ++i) {
        for (int l = i; l < N; ++l) {
            double ar = 0.0, ai = 0.0;
            const double* zi = Z + 2 * (int64_t)i * K;
            const double* zl = Z + 2 * (int64_t)l * K;
            for (int j = 0; j < K; ++j) {
                /* z_i * conj(z_l) */
                ar += zi[2 * j] * zl[2 * j] + zi[2 * j + 1] * zl[2 * j + 1];
                ai += zi[2 * j + 1] * zl[2 * j] - zi[2 * j] * zl[2 * j + 1];
            }
            ar /= (double)K;
            ai /= (double)K;
            Rm[2 * (i * N + l)] = ar;
            Rm[2 * (i * N + l) + 1] = ai;
            Rm[2 * (l * N + i)] = ar;
            Rm[2 * (l * N + i) + 1] = -ai;
        }
        Rm[2 * (i * N + i) + 1] = 0.0;
    }
    double tr = 0.0;
    for (int i = 0; i < N; ++i) tr += Rm[2 * (i * N + i)];
    double delta = lambda * tr / (double)N;
    for (int i = 0; i < N; ++i) Rm[2 * (i * N + i)] += delta;
    return delta;
}

/* Step 4 (c.1): Cholesky-Banachiewicz, row by row: L lower, real positive diagonal.
 * Returns 0, or j+1 for the first failing pivot j. L is N*N complex (upper part zero). */
static int cholesky(int N, const double* Rm, double* L) {
    memset(L, 0, sizeof(double) * 2 * (size_t)N * N);
    for (int i = 0; i < N; ++i) {
        for (int l = 0; l <= i; ++l) {
            double xr = Rm[2 * (i * N + l)], xi = Rm[2 * (i * N + l) + 1];
            for (int m = 0; m < l; ++m) {
                /* x -= L[i][m] * conj(L[l][m]) */
                double ar = L[2 * (i * N + m)], ai = L[2 * (i * N + m) + 1];
                double br = L[2 * (l * N + m)], bi = L[2 * (l * N + m) + 1];
                xr -= ar * br + ai * bi;
                xi -= ai * br - ar * bi;
            }
            if (i == l) {
                if (!(xr > 0.0) || !isfinite(xr)) return i + 1;
                L[2 * (i * N + i)] = sqrt(xr);
                L[2 * (i * N + i) + 1] = 0.0;
            } else {
                double dll = L[2 * (l * N + l)];
                L[2 * (i * N + l)] = xr / dll;
                L[2 * (i * N + l) + 1] = xi / dll;
            }
        }
    }
    return 0;
}

/* Step 5 (c.1), one steering vector: y = L^-1 s (forward), gamma = sum |y_i|^2,
 * v = L^-H y (backward) = Rm^-1 s, w = v / gamma.  Returns 0 or -1 if gamma is
 * not > 0 and finite (then w = 0). */
static int weights_one(int N, const double* L, const double* s, double* y, double* w, double* gamma_out) {
    for (int i = 0; i < N; ++i) {
        double xr = s[2 * i], xi = s[2 * i + 1];
        for (int m = 0; m < i; ++m) {
            double ar = L[2 * (i * N + m)], ai = L[2 * (i * N + m) + 1];
            double br = y[2 * m], bi = y[2 * m + 1];
            xr -= ar * br - ai * bi;
            xi -= ar * bi + ai * br;
        }
        double dii = L[2 * (i * N + i)];
        y[2 * i] = xr / dii;
        y[2 * i + 1] = xi / dii;
    }
    double g = 0.0;
    for (int i = 0; i < N; ++i) g += y[2 * i] * y[2 * i] + y[2 * i + 1] * y[2 * i + 1];
    *gamma_out = g;
    if (!(g > 0.0) || !isfinite(g)) {
        for (int i = 0; i < 2 * N; ++i) w[i] = 0.0;
        return -1;
    }
    /* backward: v_i = (y_i - sum_{m>i} conj(L[m][i]) v_m) / L[i][i]; v stored in w */
    for (int i = N - 1; i >= 0; --i) {
        double xr = y[2 * i], xi = y[2 * i + 1];
        for (int m = i + 1; m < N; ++m) {
            double ar = L[2 * (m * N + i)], ai = -L[2 * (m * N + i) + 1];
            double br = w[2 * m], bi = w[2 * m + 1];
            xr -= ar * br - ai * bi;
            xi -= ar * bi + ai * br;
        }
        double dii = L[2 * (i * N + i)];
        w[2 * i] = xr / dii;
        w[2 * i + 1] = xi / dii;
    }
    for (int i = 0; i < 2 * N; ++i) w[i] /= g;
    return 0;
}

/* Steps 4-5 for one unit: W [S][N], gamma [S]; returns info (c-11). */
static int solve_unit(int N, int S, const double* Rm, const double* steer, double* L, double* y,
                      double* W, double* G) {
    int info = cholesky(N, Rm, L);
    if (info) {
        memset(W, 0, sizeof(double) * 2 * (size_t)S * N);
        if (G) for (int k = 0; k < S; ++k) G[k] = 0.0;
        return info;
    }
    for (int k = 0; k < S; ++k) {
        double g = 0.0;
        int bad = weights_one(N, L, steer + 2 * (int64_t)k * N, y, W + 2 * (int64_t)k * N, &g);
        if (G) G[k] = bad ? 0.0 : g;
        if (bad && info == 0) info = -(k + 1);
    }
    return info;
}

/* Step 6 (c.1): Y[k][j] = sum_i conj(W[k][i]) Z[i][j] for one unit; Yblk is [S][K]. */
static void apply_unit(int N, int K, int S, const double* W, const double* Z, double* Yk, int64_t ystride) {
    for (int k = 0; k < S; ++k) {
        const double* w = W + 2 * (int64_t)k * N;
        double* yrow = Yk + 2 * (int64_t)k * ystride;
        for (int j = 0; j < K; ++j) {
            double ar = 0.0, ai = 0.0;
            for (int i = 0; i < N; ++i) {
                double wr = w[2 * i], wi = -w[2 * i + 1];
                double zr = Z[2 * ((int64_t)i * K + j)], zi = Z[2 * ((int64_t)i * K + j) + 1];
                ar += wr * zr - wi * zi;
                ai += wr * zi + wi * zr;
            }
            yrow[2 * j] = ar;
            yrow[2 * j + 1] = ai;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Exported entry points (ctypes).  All outputs are fp64 complex, interleaved. */

/* Covariance with loading for every owned unit: Rout [Dloc][B][N][N]; delta_out [Dloc][B] (nullable). */
int stap_oracle_covariance(const stap_oracle_params* p, const float* cube, double* Rout, double* delta_out) {
    if (check_params(p) || !cube || !Rout) return OR_BAD;
    const int N = p->n_chan * p->tdof, K = p->training_block, B = p->n_range / K;
    double* Z = (double*)malloc(sizeof(double) * 2 * (size_t)N * K);
    if (!Z) return OR_NOMEM;
    int rc = OR_OK;
    for (int dl = 0; dl < p->dop_count && rc == OR_OK; ++dl) {
        for (int b = 0; b < B; ++b) {
            if (snapshots(p, cube, p->dop_begin + dl, b, Z)) { rc = OR_BAD; break; }
            double* Rm = Rout + 2 * ((int64_t)dl * B + b) * N * N;
            double delta = covariance_loaded(N, K, p->diag_load, Z, Rm);
            if (delta_out) delta_out[(int64_t)dl * B + b] = delta;
        }
    }
    free(Z);
    return rc;
}

/* Solve for `count` independent matrices given as complex64 (promoted exactly to fp64):
 * R [count][N][N], steering [S][N] complex64 -> W [count][S][N], gamma [count][S], info [count]. */
int stap_oracle_solve(int32_t N, int32_t S, int64_t count, const float* R32, const float* steer32,
                      double* W, double* gamma, int32_t* info) {
    if (N <= 0 || S <= 0 || count < 0 || !R32 || !steer32 || !W || !info) return OR_BAD;
    double* Rm = (double*)malloc(sizeof(double) * 2 * (size_t)N * N);
    double* L = (double*)malloc(sizeof(double) * 2 * (size_t)N * N);
    double* y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
    double* s = (double*)malloc(sizeof(double) * 2 * (size_t)S * N);
    if (!Rm || !L || !y || !s) { free(Rm); free(L); free(y); free(s); return OR_NOMEM; }
    for (int64_t q = 0; q < 2 * (int64_t)S * N; ++q) s[q] = (double)steer32[q];
    for (int64_t u = 0; u < count; ++u) {
        for (int64_t q = 0; q < 2 * (int64_t)N * N; ++q) Rm[q] = (double)R32[u * 2 * N * N + q];
        info[u] = solve_unit(N, S, Rm, s, L, y, W + u * 2 * (int64_t)S * N, gamma ? gamma + u * S : NULL);
    }
    free(Rm); free(L); free(y); free(s);
    return OR_OK;
}

/* Same, fp64 inputs (used by the pins on hand-built matrices). */
int stap_oracle_solve_f64(int32_t N, int32_t S, int64_t count, const double* R, const double* steer,
                          double* W, double* gamma, int32_t* info) {
    if (N <= 0 || S <= 0 || count < 0 || !R || !steer || !W || !info) return OR_BAD;
    double* L = (double*)malloc(sizeof(double) * 2 * (size_t)N * N);
    double* y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
    if (!L || !y) { free(L); free(y); return OR_NOMEM; }
    for (int64_t u = 0; u < count; ++u)
        info[u] = solve_unit(N, S, R + u * 2 * (int64_t)N * N, steer, L, y, W + u * 2 * (int64_t)S * N,
                             gamma ? gamma + u * S : NULL);
    free(L); free(y);
    return OR_OK;
}

/* Cholesky factor only (pins): L [N][N]; returns info. */
int stap_oracle_cholesky_f64(int32_t N, const double* R, double* L) {
    if (N <= 0 || !R || !L) return OR_BAD;
    return cholesky(N, R, L);
}

/* Apply given weights (complex64, [Dloc][B][S][N]) to the cube: Y [Dloc][S][R]. */
int stap_oracle_apply(const stap_oracle_params* p, const float* cube, const float* W32, double* Y) {
    if (check_params(p) || !cube || !W32 || !Y) return OR_BAD;
    const int N = p->n_chan * p->tdof, K = p->training_block, B = p->n_range / K, S = p->n_steering;
    const int64_t R = p->n_range;
    double* Z = (double*)malloc(sizeof(double) * 2 * (size_t)N * K);
    double* W = (double*)malloc(sizeof(double) * 2 * (size_t)S * N);
    if (!Z || !W) { free(Z); free(W); return OR_NOMEM; }
    int rc = OR_OK;
    for (int dl = 0; dl < p->dop_count && rc == OR_OK; ++dl) {
        for (int b = 0; b < B; ++b) {
            if (snapshots(p, cube, p->dop_begin + dl, b, Z)) { rc = OR_BAD; break; }
            const float* w32 = W32 + 2 * (((int64_t)dl * B + b) * S * N);
            for (int64_t q = 0; q < 2 * (int64_t)S * N; ++q) W[q] = (double)w32[q];
            apply_unit(N, K, S, W, Z, Y + 2 * ((int64_t)dl * S * R + (int64_t)b * K), R);
        }
    }
    free(Z); free(W);
    return rc;
}

/* The whole path (c.1 steps 1-6) for every owned unit.
 * Outputs: Y [Dloc][S][R] (required), info [Dloc][B] (required),
 *          Rout [Dloc][B][N][N], Wout [Dloc][B][S][N], Gout [Dloc][B][S] (nullable).
 * nthreads > 1 parallelises over Doppler bins (OpenMP); units are independent and
 * every per-unit sum keeps its order, so the result is bitwise independent of nthreads. */
int stap_oracle_run(const stap_oracle_params* p, const float* cube, const float* steer32,
                    double* Y, int32_t* info, double* Rout, double* Wout, double* Gout, int32_t nthreads) {
    if (check_params(p) || !cube || !steer32 || !Y || !info) return OR_BAD;
    const int N = p->n_chan * p->tdof, K = p->training_block, B = p->n_range / K, S = p->n_steering;
    const int64_t R = p->n_range;
    double* s = (double*)malloc(sizeof(double) * 2 * (size_t)S * N);
    if (!s) return OR_NOMEM;
    for (int64_t q = 0; q < 2 * (int64_t)S * N; ++q) s[q] = (double)steer32[q];
    int rc = OR_OK;
    if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
#endif
    {
        double* Z = (double*)malloc(sizeof(double) * 2 * (size_t)N * K);
        double* Rm = (double*)malloc(sizeof(double) * 2 * (size_t)N * N);
        double* L = (double*)malloc(sizeof(double) * 2 * (size_t)N * N);
        double* y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
        double* W = (double*)malloc(sizeof(double) * 2 * (size_t)S * N);
        double* G = (double*)malloc(sizeof(double) * (size_t)S);
        int local_rc = (Z && Rm && L && y && W && G) ? OR_OK : OR_NOMEM;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int dl = 0; dl < p->dop_count; ++dl) {
            if (local_rc != OR_OK) continue;
            const int d = p->dop_begin + dl;
            for (int b = 0; b < B; ++b) {
                const int64_t u = (int64_t)dl * B + b;
                if (snapshots(p, cube, d, b, Z)) { local_rc = OR_BAD; break; }
                covariance_loaded(N, K, p->diag_load, Z, Rm);
                if (Rout) memcpy(Rout + 2 * u * N * N, Rm, sizeof(double) * 2 * (size_t)N * N);
                int inf = solve_unit(N, S, Rm, s, L, y, W, G);
                info[u] = inf;
                if (Wout) memcpy(Wout + 2 * u * S * N, W, sizeof(double) * 2 * (size_t)S * N);
                if (Gout) memcpy(Gout + u * S, G, sizeof(double) * (size_t)S);
                /* failed k (or all k on a Cholesky failure) have W = 0, hence Y = 0 */
                apply_unit(N, K, S, W, Z, Y + 2 * ((int64_t)dl * S * R + (int64_t)b * K), R);
            }
        }
        free(Z); free(Rm); free(L); free(y); free(W); free(G);
        if (local_rc != OR_OK) {
#ifdef _OPENMP
#pragma omp critical
#endif
            rc = local_rc;
        }
    }
    free(s);
    return rc;
}

/* Gauss-Jordan inverse with partial pivoting (complex fp64), an independent
 * path used only by pin P9.  A and Ainv are n*n complex; returns 0 or 1 if singular. */
int stap_oracle_gj_inverse(int32_t n, const double* A, double* Ainv) {
    if (n <= 0 || !A || !Ainv) return OR_BAD;
    const int w = 2 * n;
    double* M = (double*)malloc(sizeof(double) * 2 * (size_t)n * w);
    if (!M) return OR_NOMEM;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < w; ++j) {
            double re = 0.0, im = 0.0;
            if (j < n) { re = A[2 * (i * n + j)]; im = A[2 * (i * n + j) + 1]; }
            else if (j - n == i) re = 1.0;
            M[2 * (i * w + j)] = re;
            M[2 * (i * w + j) + 1] = im;
        }
    for (int col = 0; col < n; ++col) {
        int piv = col;
        double best = -1.0;
        for (int i = col; i < n; ++i) {
            double a = hypot(M[2 * (i * w + col)], M[2 * (i * w + col) + 1]);
            if (a > best) { best = a; piv = i; }
        }
        if (!(best > 0.0)) { free(M); return 1; }
        if (piv != col)
            for (int j = 0; j < w; ++j) {
                double tr = M[2 * (col * w + j)], ti = M[2 * (col * w + j) + 1];
                M[2 * (col * w + j)] = M[2 * (piv * w + j)];
                M[2 * (col * w + j) + 1] = M[2 * (piv * w + j) + 1];
                M[2 * (piv * w + j)] = tr;
                M[2 * (piv * w + j) + 1] = ti;
            }
        /* scale pivot row by 1/pivot */
        double pr = M[2 * (col * w + col)], pi = M[2 * (col * w + col) + 1];
        double den = pr * pr + pi * pi;
        double ir = pr / den, ii = -pi / den;
        for (int j = 0; j < w; ++j) {
            double xr = M[2 * (col * w + j)], xi = M[2 * (col * w + j) + 1];
            M[2 * (col * w + j)] = xr * ir - xi * ii;
            M[2 * (col * w + j) + 1] = xr * ii + xi * ir;
        }
        for (int i = 0; i < n; ++i) {
            if (i == col) continue;
            double fr = M[2 * (i * w + col)], fi = M[2 * (i * w + col) + 1];
            if (fr == 0.0 && fi == 0.0) continue;
            for (int j = 0; j < w; ++j) {
                double xr = M[2 * (col * w + j)], xi = M[2 * (col * w + j) + 1];
                M[2 * (i * w + j)] -= fr * xr - fi * xi;
                M[2 * (i * w + j) + 1] -= fr * xi + fi * xr;
            }
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            Ainv[2 * (i * n + j)] = M[2 * (i * w + n + j)];
            Ainv[2 * (i * n + j) + 1] = M[2 * (i * w + n + j) + 1];
        }
    free(M);
    return 0;
}

/*
 * Doppler front end (reading c-19 in DESIGN.md): the per-row
 * taper and FFT along the pulse axis that turn raw pulses into the datacube
 * (Table 2 "fft_2D,axis=1"; Fig. 7 text):
 *   X[d][c][r] = sum_{p < D} w[p] x[p][c][r] exp(-2 pi i p d / D)
 * written out as the DFT definition: a sequential fp64 sum in ascending p, the phase
 * taken from (p*d mod D) exactly.  raw [batch][D][C][R] complex64 (interleaved
 * floats), window [D] float, out [batch][D][C][R] complex128 (interleaved doubles).
 * The paper's following 2-D x 2-D multiply (its "U") is ambiguous and not modelled.
 */
int stap_oracle_doppler(int32_t D, int32_t C, int32_t R, int32_t batch, const float* window, const float* raw,
                        double* out, int32_t nthreads) {
    if (D <= 0 || C <= 0 || R <= 0 || batch <= 0 || !window || !raw || !out) return OR_BAD;
    double* ct = (double*)malloc(sizeof(double) * (size_t)D);
    double* st = (double*)malloc(sizeof(double) * (size_t)D);
    if (!ct || !st) {
        free(ct);
        free(st);
        return OR_NOMEM;
    }
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t k = 0; k < D; ++k) {  /* exp(-2 pi i k / D) = cos - i sin */
        ct[k] = cos(two_pi * (double)k / (double)D);
        st[k] = -sin(two_pi * (double)k / (double)D);
    }
    const int64_t plane = (int64_t)C * R;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) collapse(2)
#endif
    for (int64_t n = 0; n < batch; ++n) {
        for (int64_t col = 0; col < plane; ++col) {
            const float* xr = raw + 2 * (n * D * plane + col);
            double* xo = out + 2 * (n * D * plane + col);
            for (int64_t d = 0; d < D; ++d) {
                double re = 0.0, im = 0.0;
                for (int64_t q = 0; q < D; ++q) {
                    const double a = (double)window[q] * (double)xr[2 * q * plane];
                    const double bim = (double)window[q] * (double)xr[2 * q * plane + 1];
                    const int64_t k = (q * d) % D;
                    re += a * ct[k] - bim * st[k];
                    im += a * st[k] + bim * ct[k];
                }
                xo[2 * d * plane] = re;
                xo[2 * d * plane + 1] = im;
            }
        }
    }
    free(ct);
    free(st);
    return OR_OK;
}

int stap_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
