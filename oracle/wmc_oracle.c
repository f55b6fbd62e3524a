/*
 * oracle/wmc_oracle.c -- CPU restatement of the reference's WMC path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1903_07189_b200/,
 * include/) includes, links or calls this file.  It is used by tests/,
 * __graft_entry__.smoke() and the cpu_baseline / --impl reference legs of
 * bench.py, always as the checker / the timed reference CPU path, never as
 * the thing shipped.
 *
 * The reference (/root/reference) ships no implementation of this path, only
 * a normative spec; every function below cites the SPEC / PAPER lines it
 * restates.  Two instantiations:
 *
 *  1. fp64 "SPEC-faithful" (or_*_f64): per pixel, the eight stencils h1..h8
 *     (exact rationals lowered to double once) are correlated
 *     with the clamp-to-edge image in row-major tap order (SPEC.md:53-57,
 *     :77-78), and the response with the smallest |d_i| is returned, ties to
 *     the smallest index.  This is
 *     the "reference CPU path" that bench.py times.
 *
 *  2. fp32 "canonical" (or_*_f32): the integer-weight form of SURVEY.md
 *     Appendix A with every rounding pinned (which sums are formed, their
 *     operand order, where an FMA is used).  The CUDA kernels evaluate exactly
 *     this sequence, so GPU-vs-oracle parity is bit-exact.  It is itself
 *     checked against (1) within 1e-5 (tests/test_oracle.py).
 *
 * Flow: U^{t+1} = U^t + dt*H^w(U^t),
 * synchronous (Jacobi), non-finite check after every iteration naming the
 * iteration.
 *
 * Row parallelism follows curveflow::parallel::for_rows
 * (proj/include/curveflow/parallel.hpp:26-47): contiguous ceil-div row
 * blocks, one per worker, caller runs block 0, serial if height < 16 or one
 * worker.  Output is bit-identical for any thread count (parallel.hpp:23-25).
 *
 * Also restated: solve_l2_area / solve_l1_area (the fp32
 * sequences of DESIGN.md §3.5), the WMC energy, fidelity sums and histogram
 * in the fixed reduction order of csrc/wmc_reduce.cu, 8-bit widening and
 * save-time quantisation.
 *
 * Pinning (the reference has no tests, fixtures or golden files for this
 * path -- only its spec and proj/include/curveflow/parallel.hpp): the oracle
 * is pinned by the spec's own examples and acceptance criteria
 * (tests/test_oracle.py: kernel exactness, 1000 random 8x8 vs a naive double
 * loop, constant / impulse / ramp / affine known answers, homogeneity and
 * shift, flow identity / max principle / non-finite naming, the l1 algebra
 * KATs and identity, lambda-sweep SSIM ordering), by golden vectors from
 * independent pure-Python / numpy transcriptions (tests/golden/), and by the
 * fp64 restatement run on the reference's own executor (oracle/_ref/,
 * bit-identical).
 *
 * Build: oracle/Makefile, gcc -O2 -ffp-contract=off (no -ffast-math), SSE
 * arithmetic (x86-64 default), so every + and * rounds once to the declared
 * type and fmaf()/fma() are the only fused operations.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_EXPORT __attribute__((visibility("default")))

#include "wmc_px.h"

OR_EXPORT void or_kernel_bank_numerators(int32_t* out72) { kernel_bank_numerators(out72); }

/* 1 when this CPU can run wmc_fast.c (built with -mavx2 -mfma); the Python
 * wrapper falls back to the scalar functions here otherwise. */
OR_EXPORT int or_fast_supported(void) {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
}

/* ------------------------------------------------------------------------ */
/* for_rows restatement (parallel.hpp:26-47)                                 */
/* ------------------------------------------------------------------------ */
typedef void (*row_fn)(void* ctx, int y);

typedef struct {
    row_fn fn;
    void* ctx;
    int y0, y1;
} row_block;

static void* run_block(void* arg) {
    row_block* b = (row_block*)arg;
    for (int y = b->y0; y < b->y1; ++y) b->fn(b->ctx, y);
    return NULL;
}

static void for_rows(int height, int threads, row_fn fn, void* ctx) {
    int workers = threads < 1 ? 1 : threads;          /* parallel.hpp:28 */
    if (workers > height) workers = height;            /* :29 */
    if (workers <= 1 || height < 16) {                 /* :30-33 */
        for (int y = 0; y < height; ++y) fn(ctx, y);
        return;
    }
    int chunk = (height + workers - 1) / workers;      /* :36 */
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
    row_block* blk = (row_block*)malloc(sizeof(row_block) * (size_t)workers);
    int started = 0;
    for (int w = 1; w < workers; ++w) {                /* :37-44 */
        int y0 = w * chunk;
        int y1 = y0 + chunk < height ? y0 + chunk : height;
        if (y0 >= y1) break;
        blk[w].fn = fn; blk[w].ctx = ctx; blk[w].y0 = y0; blk[w].y1 = y1;
        pthread_create(&tid[w], NULL, run_block, &blk[w]);
        started = w;
    }
    blk[0].fn = fn; blk[0].ctx = ctx; blk[0].y0 = 0;   /* :45 caller runs block 0 */
    blk[0].y1 = chunk < height ? chunk : height;
    run_block(&blk[0]);
    for (int w = 1; w <= started; ++w) pthread_join(tid[w], NULL);  /* :46 */
    free(tid);
    free(blk);
}


/* ------------------------------------------------------------------------ */
/* fp64 SPEC-faithful WMC map                                                */
/* ------------------------------------------------------------------------ */
typedef struct {
    const double* in;
    double* out;
    int w, h;
    int64_t pitch;
    int8_t* argmin; /* optional: index 0..7 of the selected kernel */
} map64_ctx;

static void map64_row(void* vctx, int y) {
    map64_ctx* c = (map64_ctx*)vctx;
    for (int x = 0; x < c->w; ++x) {
        int m;
        c->out[(int64_t)y * c->pitch + x] = wmc_px_f64(c->in, c->w, c->h, c->pitch, y, x, &m);
        if (c->argmin) c->argmin[(int64_t)y * c->w + x] = (int8_t)m;
    }
}

/* wmc_half_laplace, fp64.  Dense row-major, pitch = w. */
OR_EXPORT int or_wmc_map_f64(const double* in, double* out, int32_t w, int32_t h,
                             int32_t threads, int8_t* argmin /* nullable, w*h */) {
    if (w <= 0 || h <= 0) return 1;
    pthread_once(&hw_once, init_hw64);
    map64_ctx c = {in, out, w, h, w, argmin};
    for_rows(h, threads, map64_row, &c);
    return 0;
}

static inline float wmc_at_f32(const float* in, int w, int h, int64_t pitch, int y, int x,
                               int map, int* tie) {
    const int ym = y > 0 ? y - 1 : 0, yp = y + 1 < h ? y + 1 : h - 1;
    const int xm = x > 0 ? x - 1 : 0, xp = x + 1 < w ? x + 1 : w - 1;
    const float* R0 = in + (int64_t)ym * pitch;
    const float* R1 = in + (int64_t)y * pitch;
    const float* R2 = in + (int64_t)yp * pitch;
    if (map)
        return wmc_map_px_f32(R0[xm], R0[x], R0[xp], R1[xm], R1[x], R1[xp], R2[xm], R2[x],
                              R2[xp], tie);
    return wmc_px_f32(R0[xm], R0[x], R0[xp], R1[xm], R1[x], R1[xp], R2[xm], R2[x], R2[xp]);
}

/* The selected D_m (= 12 * d_m) of the flow's canonical evaluation. */
static inline float best_at_f32(const float* in, int w, int h, int64_t pitch, int y, int x) {
    const int ym = y > 0 ? y - 1 : 0, yp = y + 1 < h ? y + 1 : h - 1;
    const int xm = x > 0 ? x - 1 : 0, xp = x + 1 < w ? x + 1 : w - 1;
    const float* R0 = in + (int64_t)ym * pitch;
    const float* R1 = in + (int64_t)y * pitch;
    const float* R2 = in + (int64_t)yp * pitch;
    px32 o;
    wmc_px_f32_full(R0[xm], R0[x], R0[xp], R1[xm], R1[x], R1[xp], R2[xm], R2[x], R2[xp], &o);
    return o.best;
}

typedef struct {
    const float* in;
    float* out;
    int w, h;
    int64_t pitch;
    int flow;  /* 0: map (tie rule) ; 1: out = fmaf(fl(dt*fl(1/12)), D_m, u) ; 2: flow H^w */
    float dt;
    volatile int* bad; /* per-row non-finite marker (flow only) */
    int8_t* ties;      /* map only, nullable: 1 where the fp64 tie rule fired */
} map32_ctx;

static void map32_row(void* vctx, int y) {
    map32_ctx* c = (map32_ctx*)vctx;
    const float* in = c->in;
    float* o = c->out + (int64_t)y * c->pitch;
    int bad = 0;
    const float dt12 = c->dt * C12;  /* fl(dt * fl(1/12)) */
    for (int x = 0; x < c->w; ++x) {
        int tie = 0;
        if (c->flow == 1) {
            const float v = fmaf(dt12, best_at_f32(in, c->w, c->h, c->pitch, y, x),
                                 in[(int64_t)y * c->pitch + x]);
            if (!isfinite(v)) bad = 1;
            o[x] = v;
            continue;
        }
        o[x] = wmc_at_f32(in, c->w, c->h, c->pitch, y, x, !c->flow, &tie);
        if (c->ties) c->ties[(int64_t)y * c->w + x] = (int8_t)tie;
    }
    if (c->flow == 1 && bad) c->bad[y] = 1;
}

/* wmc_half_laplace, fp32 canonical + fp64 near-tie rule; planes independent
 * (SPEC.md:62-69).  ties (nullable, planes*h*w) marks pixels resolved in fp64. */
OR_EXPORT int or_wmc_map_f32(const float* in, float* out, int32_t w, int32_t h, int64_t pitch,
                             int32_t planes, int64_t plane_stride, int32_t threads,
                             int8_t* ties) {
    if (w <= 0 || h <= 0 || planes <= 0 || pitch < w) return 1;
    for (int p = 0; p < planes; ++p) {
        map32_ctx c = {in + p * plane_stride, out + p * plane_stride, w, h, pitch, 0, 0.f, NULL,
                       ties ? ties + (int64_t)p * w * h : NULL};
        for_rows(h, threads, map32_row, &c);
    }
    return 0;
}

/* One flow step's H^w field (canonical fp32, no tie rule): the map the flow
 * iterates, exposed so tests can check U^{t+1} == fmaf(dt, H, U^t). */
OR_EXPORT int or_wmc_flowmap_f32(const float* in, float* out, int32_t w, int32_t h,
                                 int32_t threads) {
    if (w <= 0 || h <= 0) return 1;
    map32_ctx c = {in, out, w, h, w, 2, 0.f, NULL, NULL};
    for_rows(h, threads, map32_row, &c);
    return 0;
}

/* mc_flow(scheme=half_laplace), fp32 canonical, Jacobi ping-pong.
 * Returns 0, or 3 with *bad_iter = first iteration (1-based) whose iterate
 * holds a non-finite value.  img is updated in place
 * (it holds U^iters on success).                                            */
OR_EXPORT int or_flow_f32(float* img, int32_t w, int32_t h, int64_t pitch, int32_t planes,
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
            memset(bad, 0, sizeof(int) * (size_t)h);
            map32_ctx c = {A, B, w, h, pitch, 1, dt, bad, NULL};
            for_rows(h, threads, map32_row, &c);
            float* s = A; A = B; B = s;
            int any = 0;
            for (int y = 0; y < h; ++y) any |= bad[y];
            if (any) {
                if (first == 0 || t < first) first = t;
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

/* solve_l2_area with A = I: U^0 = f, then iters Jacobi
 * steps U' = fmaf(dt, fmaf(lambda, H^w(U), fmaf(U, -1, f)), U), H^w the
 * flow's canonical fp32 map.  u receives U^iters; 3 + *bad_iter on a
 * non-finite iterate. */
typedef struct {
    const float* in;
    const float* f;
    float* out;
    int w, h;
    int64_t pitch;
    float dt, lambda;
    volatile int* bad;
} l2_ctx;

static void l2_row(void* vctx, int y) {
    l2_ctx* c = (l2_ctx*)vctx;
    int bad = 0;
    for (int x = 0; x < c->w; ++x) {
        const int64_t i = (int64_t)y * c->pitch + x;
        const float hw = wmc_at_f32(c->in, c->w, c->h, c->pitch, y, x, 0, NULL);
        const float r = fmaf(c->in[i], -1.0f, c->f[i]);
        const float v = fmaf(c->dt, fmaf(c->lambda, hw, r), c->in[i]);
        if (!isfinite(v)) bad = 1;
        c->out[i] = v;
    }
    if (bad) c->bad[y] = 1;
}

OR_EXPORT int or_solve_l2_area_f32(const float* f, float* u, int32_t w, int32_t h, int64_t pitch,
                                   int32_t planes, int64_t plane_stride, int32_t iters, float dt,
                                   float lambda, int32_t init, int32_t threads,
                                   int32_t* bad_iter) {
    if (w <= 0 || h <= 0 || planes <= 0 || iters < 0 || pitch < w) return 1;
    if (bad_iter) *bad_iter = 0;
    float* tmp = (float*)malloc(sizeof(float) * (size_t)pitch * (size_t)h);
    int* bad = (int*)calloc((size_t)h, sizeof(int));
    int rc = 0;
    for (int p = 0; p < planes && rc == 0; ++p) {
        float* U = u + p * plane_stride;
        const float* F = f + p * plane_stride;
        if (init) memcpy(U, F, sizeof(float) * (size_t)pitch * (size_t)h);
        float *A = U, *B = tmp;
        for (int t = 1; t <= iters; ++t) {
            memset(bad, 0, sizeof(int) * (size_t)h);
            l2_ctx c = {A, F, B, w, h, pitch, dt, lambda, bad};
            for_rows(h, threads, l2_row, &c);
            float* s = A; A = B; B = s;
            int any = 0;
            for (int y = 0; y < h; ++y) any |= bad[y];
            if (any) { if (bad_iter) *bad_iter = t; rc = 3; break; }
        }
        if (A != U) memcpy(U, A, sizeof(float) * (size_t)pitch * (size_t)h);
    }
    free(tmp);
    free(bad);
    return rc;
}

/* solve_l1_area with A = I (Eqs. 32-38), one
 * iteration per pixel in fp32 (the kernel's kModeL1):
 *   r  = fl(fl(u - f) + d)                 (fmaf(f, -1, u) then +)
 *   d' = fminf(fmaxf(r, -alpha), alpha)    (Eq. 37; NaN r -> -alpha)
 *   e  = fmaf(d, -1, d' + d')              (2d' - d; d' + d' exact)
 *   s  = fmaf(lambda, H^w(U), e * nia)     (nia = -fl(1/alpha))
 *   U' = fmaf(dt, s, u)
 * The shrinkage b = r - d' (Eq. 36) never enters the update;
 * or_l1_px exposes it for the KATs.  init: U = f, d = 0. */
OR_EXPORT void or_l1_px(float r, float alpha, float* b, float* d_new) {
    /* Eq. 36 branches and Eq. 37's clamp, literally */
    *b = r > alpha ? r - alpha : (r < -alpha ? r + alpha : 0.0f);
    *d_new = fminf(fmaxf(r, -alpha), alpha);
}

typedef struct {
    const float* in;
    const float* f;
    const float* d;
    float* out;
    float* dout;
    int w, h;
    int64_t pitch;
    float dt, lambda, alpha, nia;
    volatile int* bad;
} l1_ctx;

static void l1_row(void* vctx, int y) {
    l1_ctx* c = (l1_ctx*)vctx;
    int bad = 0;
    for (int x = 0; x < c->w; ++x) {
        const int64_t i = (int64_t)y * c->pitch + x;
        const float u = c->in[i], dv = c->d[i];
        const float hw = wmc_at_f32(c->in, c->w, c->h, c->pitch, y, x, 0, NULL);
        const float r = fmaf(c->f[i], -1.0f, u) + dv;
        const float dn = fminf(fmaxf(r, -c->alpha), c->alpha);
        const float e = fmaf(dv, -1.0f, dn + dn);
        const float v = fmaf(c->dt, fmaf(c->lambda, hw, e * c->nia), u);
        if (!isfinite(v)) bad = 1;
        c->out[i] = v;
        c->dout[i] = dn;
    }
    if (bad) c->bad[y] = 1;
}

OR_EXPORT int or_solve_l1_area_f32(const float* f, float* u, float* d, int32_t w, int32_t h,
                                   int64_t pitch, int32_t planes, int64_t plane_stride,
                                   int32_t iters, float dt, float lambda, float alpha,
                                   int32_t init, int32_t threads, int32_t* bad_iter) {
    if (w <= 0 || h <= 0 || planes <= 0 || iters < 0 || pitch < w || !(alpha > 0.0f)) return 1;
    if (bad_iter) *bad_iter = 0;
    const size_t n = (size_t)pitch * (size_t)h;
    float* tmp = (float*)malloc(sizeof(float) * n);
    float* dtmp = (float*)malloc(sizeof(float) * n);
    int* bad = (int*)calloc((size_t)h, sizeof(int));
    const float nia = -(1.0f / alpha);
    int rc = 0;
    for (int p = 0; p < planes && rc == 0; ++p) {
        float* U = u + p * plane_stride;
        float* D = d + p * plane_stride;
        const float* F = f + p * plane_stride;
        if (init) {
            memcpy(U, F, sizeof(float) * n);
            memset(D, 0, sizeof(float) * n);
        }
        float *A = U, *B = tmp, *DA = D, *DB = dtmp;
        for (int t = 1; t <= iters; ++t) {
            memset(bad, 0, sizeof(int) * (size_t)h);
            l1_ctx c = {A, F, DA, B, DB, w, h, pitch, dt, lambda, alpha, nia, bad};
            for_rows(h, threads, l1_row, &c);
            float* s = A; A = B; B = s;
            s = DA; DA = DB; DB = s;
            int any = 0;
            for (int y = 0; y < h; ++y) any |= bad[y];
            if (any) { if (bad_iter) *bad_iter = t; rc = 3; break; }
        }
        if (A != U) memcpy(U, A, sizeof(float) * n);
        if (DA != D) memcpy(D, DA, sizeof(float) * n);
    }
    free(tmp);
    free(dtmp);
    free(bad);
    return rc;
}

/* Energy sum |H|^q over a dense map (planes x h x w) in the fixed order of
 * paper_1903_07189_b200/csrc/wmc_reduce.cu: per row, 32-column blocks
 * reduced by the xor butterfly (offsets 16,8,4,2,1; lane 0's value), blocks
 * summed in x order, rows in y order, planes in order.  qkind: 1 -> |H|,
 * 2 -> H*H, 3 -> sqrt|H|, 0 -> pow(|H|, q). */
OR_EXPORT double or_energy_from_map(const float* map, int32_t w, int32_t h, int32_t planes,
                                    double q, int32_t qkind) {
    /* the energy's fixed order (csrc/wmc_reduce.cu header): 256-column
     * segments; lane l's terms t0..t7 = columns 4l..4l+3, 128+4l..128+4l+3,
     * summed ((t0+t1)+(t2+t3)) + ((t4+t5)+(t6+t7)); lanes combine by the xor
     * butterfly 16, 8, 4, 2, 1; segments add in x order, rows in y order,
     * planes in plane order. */
    double total = 0.0;
    for (int p = 0; p < planes; ++p)
        for (int y = 0; y < h; ++y) {
            const float* r = map + ((int64_t)p * h + y) * w;
            double row = 0.0;
            for (int x0 = 0; x0 < w; x0 += 256) {
                double v[32];
                for (int l = 0; l < 32; ++l) {
                    double t[8];
                    for (int c = 0; c < 2; ++c)
                        for (int j = 0; j < 4; ++j) {
                            const int x = x0 + 4 * l + 128 * c + j;
                            double tv = 0.0;
                            if (x < w) {
                                const double a = fabs((double)r[x]);
                                tv = qkind == 1 ? a : (qkind == 2 ? a * a : (qkind == 3 ? sqrt(a) : pow(a, q)));
                            }
                            t[4 * c + j] = tv;
                        }
                    v[l] = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
                }
                for (int o = 16; o > 0; o >>= 1) {
                    double nv[32];
                    for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ o];
                    memcpy(v, nv, sizeof(v));
                }
                row = row + v[0];
            }
            total = total + row;
        }
    return total;
}

/* Fidelity sum |u - f|^q (f NULL: sum |u|^q) over pitched planes, the
 * difference in fp64, in the energy's fixed order (wmc_reduce.cu). */
OR_EXPORT double or_fidelity(const float* u, const float* f, int32_t w, int32_t h, int64_t pitch,
                             int32_t planes, int64_t plane_stride, double q, int32_t qkind) {
    /* the energy's order (or_energy_from_map) with terms |u - f|^q */
    double total = 0.0;
    for (int p = 0; p < planes; ++p)
        for (int y = 0; y < h; ++y) {
            const int64_t off = (int64_t)p * plane_stride + (int64_t)y * pitch;
            double row = 0.0;
            for (int x0 = 0; x0 < w; x0 += 256) {
                double v[32];
                for (int l = 0; l < 32; ++l) {
                    double t[8];
                    for (int c = 0; c < 2; ++c)
                        for (int j = 0; j < 4; ++j) {
                            const int x = x0 + 4 * l + 128 * c + j;
                            double tv = 0.0;
                            if (x < w) {
                                const double a = fabs(f ? (double)u[off + x] - (double)f[off + x]
                                                        : (double)u[off + x]);
                                tv = qkind == 1 ? a : (qkind == 2 ? a * a : (qkind == 3 ? sqrt(a) : pow(a, q)));
                            }
                            t[4 * c + j] = tv;
                        }
                    v[l] = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
                }
                for (int o = 16; o > 0; o >>= 1) {
                    double nv[32];
                    for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ o];
                    memcpy(v, nv, sizeof(v));
                }
                row = row + v[0];
            }
            total = total + row;
        }
    return total;
}

/* Histogram bins of a map: floor((v*scale - lo)/width) clamped (NaN -> 0). */
OR_EXPORT void or_histogram_from_map(const float* map, int64_t n, float scale, float lo,
                                     float width, int32_t nbins, int64_t* counts) {
    memset(counts, 0, sizeof(int64_t) * (size_t)nbins);
    for (int64_t i = 0; i < n; ++i) {
        const float t = (map[i] * scale - lo) / width;
        int b = (t != t) ? 0 : (int)floorf(fminf(fmaxf(t, -1.0f), (float)nbins));
        b = b < 0 ? 0 : (b > nbins - 1 ? nbins - 1 : b);
        counts[b]++;
    }
}

/* Save-time quantisation: clamp to [0,1] (NaN -> 0), scale by
 * 255 in fp32, round half to even. */
OR_EXPORT void or_quantize_u8(const float* in, uint8_t* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const float c = fminf(fmaxf(in[i], 0.0f), 1.0f);
        out[i] = (uint8_t)rintf(c * 255.0f);
    }
}

/* 8-bit widening on load: q / 255 in IEEE fp32. */
OR_EXPORT void or_u8_to_f32(const uint8_t* in, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)in[i] / 255.0f;
}

/* ------------------------------------------------------------------------ */
/* fp64 flow (the timed "reference CPU path" of mc_flow).                    */
/* ------------------------------------------------------------------------ */
typedef struct {
    const double* in;
    double* out;
    int w, h;
    double dt;
    volatile int* bad;
} flow64_ctx;

static void flow64_row(void* vctx, int y) {
    flow64_ctx* c = (flow64_ctx*)vctx;
    int bad = 0;
    for (int x = 0; x < c->w; ++x) {
        double hw = wmc_px_f64(c->in, c->w, c->h, c->w, y, x, NULL);
        double v = c->in[(int64_t)y * c->w + x] + c->dt * hw;   /* Eq. 26 */
        if (!isfinite(v)) bad = 1;
        c->out[(int64_t)y * c->w + x] = v;
    }
    if (bad) c->bad[y] = 1;
}

OR_EXPORT int or_flow_f64(double* img, int32_t w, int32_t h, int32_t iters, double dt,
                          int32_t threads, int32_t* bad_iter) {
    if (w <= 0 || h <= 0 || iters < 0 || !(dt > 0.0) || dt > 1.0) return 1;
    pthread_once(&hw_once, init_hw64);
    if (bad_iter) *bad_iter = 0;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)w * (size_t)h);
    int* bad = (int*)calloc((size_t)h, sizeof(int));
    double *A = img, *B = tmp;
    int rc = 0;
    for (int t = 1; t <= iters; ++t) {
        memset(bad, 0, sizeof(int) * (size_t)h);
        flow64_ctx c = {A, B, w, h, dt, bad};
        for_rows(h, threads, flow64_row, &c);
        double* s = A; A = B; B = s;
        int any = 0;
        for (int y = 0; y < h; ++y) any |= bad[y];
        if (any) { if (bad_iter) *bad_iter = t; rc = 3; break; }
    }
    if (A != img) memcpy(img, A, sizeof(double) * (size_t)w * (size_t)h);
    free(tmp);
    free(bad);
    return rc;
}

/* Naive per-pixel double loop without any shared helper: a second, direct   */
/* transcription of Eqs. 27-28 used for SPEC acceptance criterion 2          */
/* (SPEC.md:468): or_wmc_map_f64 must match it bit-exactly.                  */
OR_EXPORT void or_wmc_naive_f64(const double* in, double* out, int32_t w, int32_t h) {
    pthread_once(&hw_once, init_hw64);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double best = 0.0;
            for (int i = 0; i < 8; ++i) {
                double s = 0.0;
                for (int dr = -1; dr <= 1; ++dr)
                    for (int dc = -1; dc <= 1; ++dc) {
                        int yy = y + dr < 0 ? 0 : (y + dr >= h ? h - 1 : y + dr);
                        int xx = x + dc < 0 ? 0 : (x + dc >= w ? w - 1 : x + dc);
                        s = s + HW64[i][dr + 1][dc + 1] * in[yy * w + xx];
                    }
                if (i == 0 || fabs(s) < fabs(best)) best = s;
            }
            out[y * w + x] = best;
        }
}
