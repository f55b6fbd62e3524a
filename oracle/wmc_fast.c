/*
 * oracle/wmc_fast.c -- vectorised CPU restatement of the oracle's per-pixel
 * sequences, fast enough to check the FULL BASELINE configurations (cfg4 is
 * 5.4e10 pixel-updates).  TEST INFRASTRUCTURE ONLY (see wmc_oracle.c header):
 * used by tests/ as the checker and by bench.py's CPU legs, never shipped.
 *
 * Every function here evaluates exactly the expressions of oracle/wmc_px.h
 * (the scalar restatement of SPEC.md:171-179 / :256-272, PAPER.md Eqs.
 * 26-28), in the same operand order, with the same roundings:
 *   - fp32 canonical:  wmc_px_f32_full() + the flow step
 *     fmaf(fl(dt*fl(1/12)), D_m, u) of or_flow_f32, or the map's near-tie rule
 *     (map_best_f32 / wmc_map_px_f32);
 *   - fp64 SPEC-faithful: wmc_px_f64() (row-major taps, s = s + w*x, weights
 *     n/12 rounded once, strict-< first-minimum) + u + dt*H (or_flow_f64).
 * Only the loop structure differs: a row's interior columns run as one loop
 * over x that gcc vectorises (AVX2 + FMA, compiled with -O3 -mavx2 -mfma
 * -ffp-contract=off: vector FMAs only where the source says fmaf/fma, every
 * other + and * rounds once, IEEE compares/blends), the two edge columns go
 * through the scalar wmc_px.h functions.  tests/test_oracle_fast.py checks
 * the result is bit-identical to the scalar oracle on random and edge-case
 * images (odd widths, 1..3 columns, NaN/Inf, huge values, many thread counts).
 *
 * Rows are split like curveflow::parallel::for_rows (parallel.hpp:26-47):
 * contiguous ceil-div blocks, one per worker; results do not depend on it.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_EXPORT __attribute__((visibility("default")))

#include "wmc_px.h"

/* ---- for_rows (parallel.hpp:26-47), one block of rows per worker ------- */
typedef void (*rows_fn)(void* ctx, int y0, int y1);
typedef struct {
    rows_fn fn;
    void* ctx;
    int y0, y1;
} blk_t;
static void* blk_run(void* a) {
    blk_t* b = (blk_t*)a;
    b->fn(b->ctx, b->y0, b->y1);
    return NULL;
}
static void for_row_blocks(int h, int threads, rows_fn fn, void* ctx) {
    int workers = threads < 1 ? 1 : threads;
    if (workers > h) workers = h;
    if (workers <= 1 || h < 16) {
        fn(ctx, 0, h);
        return;
    }
    const int chunk = (h + workers - 1) / workers;
    pthread_t tid[256];
    blk_t blk[256];
    if (workers > 256) workers = 256;
    int started = 0;
    for (int w = 1; w < workers; ++w) {
        const int y0 = w * chunk, y1 = y0 + chunk < h ? y0 + chunk : h;
        if (y0 >= y1) break;
        blk[w] = (blk_t){fn, ctx, y0, y1};
        pthread_create(&tid[w], NULL, blk_run, &blk[w]);
        started = w;
    }
    fn(ctx, 0, chunk < h ? chunk : h);
    for (int w = 1; w <= started; ++w) pthread_join(tid[w], NULL);
}

/* ---- fp32 canonical: one row of H^w (wmc_px_f32_full, inlined) -------- */
static inline float pk32(float l, float r) { return fabsf(r) < fabsf(l) ? r : l; }

/* The canonical D_m of one pixel (same expressions as wmc_px_f32_full). */
#define CANON_BEST(a, b, c, l, u, r, e, f, g, best, n12u_out)                            \
    do {                                                                                 \
        const float n12_ = (u) * -12.0f;                                                 \
        const float Vl = (a) + (e), Vc = (b) + (f), Vr = (c) + (g);                      \
        const float Wm = Vl + Vc, W0 = Vc + Vr;                                          \
        const float Ht = (a) + (c), Hc = (l) + (r), Hb = (e) + (g);                      \
        const float Tm = Ht + Hc, T0 = Hc + Hb;                                          \
        const float D0 = fmaf(2.0f, fmaf(2.0f, (l), Wm), n12_);                          \
        const float D1 = fmaf(2.0f, fmaf(2.0f, (b), Tm), n12_);                          \
        const float D2 = fmaf(2.0f, fmaf(2.0f, (r), W0), n12_);                          \
        const float D3 = fmaf(2.0f, fmaf(2.0f, (f), T0), n12_);                          \
        const float K5 = ((c) + (e)) + n12_, K6 = ((a) + (g)) + n12_;                    \
        const float D4 = fmaf(4.0f, (b) + (l), fmaf(2.0f, (a), K5));                     \
        const float D5 = fmaf(4.0f, (b) + (r), fmaf(2.0f, (c), K6));                     \
        const float D6 = fmaf(4.0f, (r) + (f), fmaf(2.0f, (g), K5));                     \
        const float D7 = fmaf(4.0f, (l) + (f), fmaf(2.0f, (e), K6));                     \
        best = pk32(pk32(pk32(D0, D1), pk32(D2, D3)), pk32(pk32(D4, D5), pk32(D6, D7))); \
        n12u_out = n12_;                                                                 \
        DS[0] = D0; DS[1] = D1; DS[2] = D2; DS[3] = D3;                                  \
        DS[4] = D4; DS[5] = D5; DS[6] = D6; DS[7] = D7;                                  \
    } while (0)

/* mode 0: out = fmaf(fl(dt * fl(1/12)), D_m, u) (flow step);  mode 1: out = H^w with the
 * map's near-tie flag in tie[] (the caller resolves flagged pixels). */
static void row32(const float* R0, const float* R1, const float* R2, float* O, int8_t* tie,
                  int w, int mode, float dt) {
    const float C12 = 1.0f / 12.0f;
    /* edges through the scalar restatement */
    for (int k = 0; k < 2; ++k) {
        const int x = k == 0 ? 0 : w - 1;
        if (k == 1 && w == 1) break;
        const int xm = x > 0 ? x - 1 : 0, xp = x + 1 < w ? x + 1 : w - 1;
        px32 o;
        wmc_px_f32_full(R0[xm], R0[x], R0[xp], R1[xm], R1[x], R1[xp], R2[xm], R2[x], R2[xp], &o);
        if (mode == 0) {
            O[x] = fmaf(dt * C12, o.best, R1[x]);
        } else {
            int t;
            O[x] = map_best_f32(&o, &t) * C12;
            tie[x] = (int8_t)t;
        }
    }
    if (mode == 0) {
        const float dt12 = dt * C12;  /* fl(dt * fl(1/12)) */
        for (int x = 1; x < w - 1; ++x) {
            float DS[8], best, n12u;
            CANON_BEST(R0[x - 1], R0[x], R0[x + 1], R1[x - 1], R1[x], R1[x + 1], R2[x - 1], R2[x],
                       R2[x + 1], best, n12u);
            (void)n12u;
            (void)DS;
            O[x] = fmaf(dt12, best, R1[x]);
        }
    } else {
        for (int x = 1; x < w - 1; ++x) {
            float DS[8], best, n12u;
            CANON_BEST(R0[x - 1], R0[x], R0[x + 1], R1[x - 1], R1[x], R1[x + 1], R2[x - 1], R2[x],
                       R2[x + 1], best, n12u);
            /* map_best_f32 (wmc_px.h), written for the vectoriser */
            uint32_t U, v;
            memcpy(&U, &DS[0], 4);
            int32_t S = (int32_t)U;
            for (int k = 1; k < 8; ++k) {
                memcpy(&v, &DS[k], 4);
                U = v < U ? v : U;
                S = (int32_t)v < S ? (int32_t)v : S;
            }
            float P, N;
            memcpy(&P, &U, 4);
            memcpy(&N, &S, 4);
            const float xs = P + N;
            float b = xs > 0.0f ? N : P;
            const int slow = (U != (uint32_t)S) & !((xs > 0.0f) | (xs < 0.0f));
            b = slow ? best : b;
            const float tau = fmaf(fabsf(n12u), 0x1.8p-19f, fabsf(b) * 0x1.0p-20f);
            const float ax = fabsf(xs);
            tie[x] = (int8_t)((ax <= tau) & (ax < fabsf(b)));
            O[x] = b * C12;
        }
    }
}

typedef struct {
    const float* in;
    float* out;
    int8_t* tie; /* map only: w-wide scratch per row block, or full (planes*h*w) */
    int w, h;
    int64_t pitch;
    int mode;
    float dt;
    int* bad; /* per row (flow) */
} ctx32;

static void rows32(void* vc, int y0, int y1) {
    ctx32* c = (ctx32*)vc;
    int8_t* scratch = NULL;
    if (c->mode == 1 && !c->tie) scratch = (int8_t*)malloc((size_t)c->w);
    for (int y = y0; y < y1; ++y) {
        const int ym = y > 0 ? y - 1 : 0, yp = y + 1 < c->h ? y + 1 : c->h - 1;
        const float* R0 = c->in + (int64_t)ym * c->pitch;
        const float* R1 = c->in + (int64_t)y * c->pitch;
        const float* R2 = c->in + (int64_t)yp * c->pitch;
        float* O = c->out + (int64_t)y * c->pitch;
        if (c->mode == 0) {
            row32(R0, R1, R2, O, NULL, c->w, 0, c->dt);
            int bad = 0;  /* x - x is 0 unless x is NaN or +-Inf */
            for (int x = 0; x < c->w; ++x) bad |= (O[x] - O[x]) != 0.0f;
            c->bad[y] = bad;
        } else {
            int8_t* T = c->tie ? c->tie + (int64_t)y * c->w : scratch;
            row32(R0, R1, R2, O, T, c->w, 1, 0.0f);
            /* flagged pixels: the SPEC-faithful fp64 evaluation (wmc_map_px_f32) */
            for (int x = 0; x < c->w; ++x) {
                if (!T[x]) continue;
                const int xm = x > 0 ? x - 1 : 0, xp = x + 1 < c->w ? x + 1 : c->w - 1;
                int t;
                O[x] = wmc_map_px_f32(R0[xm], R0[x], R0[xp], R1[xm], R1[x], R1[xp], R2[xm],
                                      R2[x], R2[xp], &t);
            }
        }
    }
    free(scratch);
}

/* or_flow_f32 (wmc_oracle.c), vectorised: same arguments, same results. */
OR_EXPORT int or_fast_flow_f32(float* img, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                               int64_t plane_stride, int32_t iters, float dt, int32_t threads,
                               int32_t* bad_iter) {
    if (w <= 0 || h <= 0 || planes <= 0 || iters < 0 || pitch < w) return 1;
    if (!(dt > 0.0f) || dt > 1.0f) return 1;
    if (bad_iter) *bad_iter = 0;
    float* tmp = (float*)malloc(sizeof(float) * (size_t)pitch * (size_t)h);
    int* bad = (int*)calloc((size_t)h, sizeof(int));
    int rc = 0, first = 0;
    for (int p = 0; p < planes && rc == 0; ++p) {
        float* A = img + p * plane_stride;
        float* B = tmp;
        for (int t = 1; t <= iters; ++t) {
            ctx32 c = {A, B, NULL, w, h, pitch, 0, dt, bad};
            for_row_blocks(h, threads, rows32, &c);
            float* s = A; A = B; B = s;
            int any = 0;
            for (int y = 0; y < h; ++y) any |= bad[y];
            if (any) {
                first = t;
                rc = 3;
                break;
            }
        }
        if (A != img + p * plane_stride)
            for (int y = 0; y < h; ++y)
                memcpy(img + p * plane_stride + (int64_t)y * pitch, A + (int64_t)y * pitch,
                       sizeof(float) * (size_t)w);
    }
    if (bad_iter) *bad_iter = first;
    free(tmp);
    free(bad);
    return rc;
}

/* or_wmc_map_f32 (wmc_oracle.c), vectorised: same arguments, same results. */
OR_EXPORT int or_fast_map_f32(const float* in, float* out, int32_t w, int32_t h, int64_t pitch,
                              int32_t planes, int64_t plane_stride, int32_t threads,
                              int8_t* ties) {
    if (w <= 0 || h <= 0 || planes <= 0 || pitch < w) return 1;
    pthread_once(&hw_once, init_hw64);
    for (int p = 0; p < planes; ++p) {
        ctx32 c = {in + p * plane_stride, out + p * plane_stride,
                   ties ? ties + (int64_t)p * w * h : NULL, w, h, pitch, 1, 0.0f, NULL};
        for_row_blocks(h, threads, rows32, &c);
    }
    return 0;
}

/* ---- fp64 SPEC-faithful (wmc_px_f64), one row -------------------------- */
/* Row-major taps t = 0..8 of kernel i, s = s + w*x unfused, zero taps
 * included (0*x is not folded: -fno-fast-math), strict-< first minimum. */
/* h_i weights n/12 (H12 of wmc_px.h), rounded once: the constant n / 12.0
 * folded by the compiler is the IEEE quotient, the value init_hw64 stores. */
static const double W64[8][9] = {
    {2 / 12.0, 2 / 12.0, 0.0, 4 / 12.0, -1.0, 0.0, 2 / 12.0, 2 / 12.0, 0.0},
    {2 / 12.0, 4 / 12.0, 2 / 12.0, 2 / 12.0, -1.0, 2 / 12.0, 0.0, 0.0, 0.0},
    {0.0, 2 / 12.0, 2 / 12.0, 0.0, -1.0, 4 / 12.0, 0.0, 2 / 12.0, 2 / 12.0},
    {0.0, 0.0, 0.0, 2 / 12.0, -1.0, 2 / 12.0, 2 / 12.0, 4 / 12.0, 2 / 12.0},
    {2 / 12.0, 4 / 12.0, 1 / 12.0, 4 / 12.0, -1.0, 0.0, 1 / 12.0, 0.0, 0.0},
    {1 / 12.0, 4 / 12.0, 2 / 12.0, 0.0, -1.0, 4 / 12.0, 0.0, 0.0, 1 / 12.0},
    {0.0, 0.0, 1 / 12.0, 0.0, -1.0, 4 / 12.0, 1 / 12.0, 4 / 12.0, 2 / 12.0},
    {1 / 12.0, 0.0, 0.0, 4 / 12.0, -1.0, 0.0, 2 / 12.0, 4 / 12.0, 1 / 12.0}};

/* OR_EXPORT'ed check that W64 equals the oracle's HW64 (tests). */
OR_EXPORT int or_fast_w64_matches(void) {
    pthread_once(&hw_once, init_hw64);
    for (int i = 0; i < 8; ++i)
        for (int t = 0; t < 9; ++t)
            if (memcmp(&W64[i][t], &HW64[i][t / 3][t % 3], sizeof(double))) return 0;
    return 1;
}

static inline double px64(const double nb[9]) {
    double best = 0.0;
#pragma GCC unroll 8
    for (int i = 0; i < 8; ++i) {
        double s = 0.0;
#pragma GCC unroll 9
        for (int t = 0; t < 9; ++t) s = s + W64[i][t] * nb[t];
        best = (i == 0 || fabs(s) < fabs(best)) ? s : best;
    }
    return best;
}

static void row64(const double* R0, const double* R1, const double* R2, double* O, int w,
                  int flow, double dt) {
    for (int k = 0; k < 2; ++k) {
        const int x = k == 0 ? 0 : w - 1;
        if (k == 1 && w == 1) break;
        const int xm = x > 0 ? x - 1 : 0, xp = x + 1 < w ? x + 1 : w - 1;
        const double nb[9] = {R0[xm], R0[x], R0[xp], R1[xm], R1[x], R1[xp], R2[xm], R2[x], R2[xp]};
        const double best = px64(nb);
        O[x] = flow ? R1[x] + dt * best : best;
    }
    if (flow) {
        for (int x = 1; x < w - 1; ++x) {
            const double nb[9] = {R0[x - 1], R0[x], R0[x + 1], R1[x - 1], R1[x],
                                  R1[x + 1], R2[x - 1], R2[x], R2[x + 1]};
            O[x] = R1[x] + dt * px64(nb);
        }
    } else {
        for (int x = 1; x < w - 1; ++x) {
            const double nb[9] = {R0[x - 1], R0[x], R0[x + 1], R1[x - 1], R1[x],
                                  R1[x + 1], R2[x - 1], R2[x], R2[x + 1]};
            O[x] = px64(nb);
        }
    }
}

typedef struct {
    const double* in;
    double* out;
    int w, h, flow;
    double dt;
    int* bad;
} ctx64;

static void rows64(void* vc, int y0, int y1) {
    ctx64* c = (ctx64*)vc;
    for (int y = y0; y < y1; ++y) {
        const int ym = y > 0 ? y - 1 : 0, yp = y + 1 < c->h ? y + 1 : c->h - 1;
        double* O = c->out + (int64_t)y * c->w;
        row64(c->in + (int64_t)ym * c->w, c->in + (int64_t)y * c->w, c->in + (int64_t)yp * c->w,
              O, c->w, c->flow, c->dt);
        if (c->flow) {
            int bad = 0;
            for (int x = 0; x < c->w; ++x) bad |= (O[x] - O[x]) != 0.0;
            c->bad[y] = bad;
        }
    }
}

/* or_flow_f64 (wmc_oracle.c), vectorised: same arguments, same results. */
OR_EXPORT int or_fast_flow_f64(double* img, int32_t w, int32_t h, int32_t iters, double dt,
                               int32_t threads, int32_t* bad_iter) {
    if (w <= 0 || h <= 0 || iters < 0 || !(dt > 0.0) || dt > 1.0) return 1;
    pthread_once(&hw_once, init_hw64);
    if (bad_iter) *bad_iter = 0;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)w * (size_t)h);
    int* bad = (int*)calloc((size_t)h, sizeof(int));
    double *A = img, *B = tmp;
    int rc = 0;
    for (int t = 1; t <= iters; ++t) {
        ctx64 c = {A, B, w, h, 1, dt, bad};
        for_row_blocks(h, threads, rows64, &c);
        double* s = A; A = B; B = s;
        int any = 0;
        for (int y = 0; y < h; ++y) any |= bad[y];
        if (any) {
            if (bad_iter) *bad_iter = t;
            rc = 3;
            break;
        }
    }
    if (A != img) memcpy(img, A, sizeof(double) * (size_t)w * (size_t)h);
    free(tmp);
    free(bad);
    return rc;
}

/* or_wmc_map_f64 (wmc_oracle.c) without the argmin output, vectorised. */
OR_EXPORT int or_fast_map_f64(const double* in, double* out, int32_t w, int32_t h,
                              int32_t threads) {
    if (w <= 0 || h <= 0) return 1;
    pthread_once(&hw_once, init_hw64);
    ctx64 c = {in, out, w, h, 0, 0.0, NULL};
    for_row_blocks(h, threads, rows64, &c);
    return 0;
}
