/*
 * oracle/synth_ref.c -- the seeded synthetic-image generator restated for
 * the CPU side.  TEST INFRASTRUCTURE ONLY (see wmc_oracle.c header).
 *
 * bench.py's reference arm (--impl reference) and the CPU baseline must not
 * load the product library (paper_1903_07189_b200/libcurveflow_b200.so), so
 * they build their inputs with this file instead of cf_synth_f32 / _u8.  It
 * restates csrc/synth.cpp's pinned generator (BASELINE.json's
 * configs describe only counts, sigma and sizes): xoshiro256** seeded by
 * SplitMix64, ramp + rectangles + discs painted in draw order, counter-based
 * Box-Muller noise per pixel index, clamp to [0,1] in double, then fp32
 * rounding or lrint(255 v).  Same libm calls in the same order, so the bytes
 * equal cf_synth_*'s (tests/test_oracle_fast.py compares them).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#define OR_EXPORT __attribute__((visibility("default")))

static uint64_t sm64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

typedef struct {
    uint64_t s[4];
} xo_t;
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static void xo_seed(xo_t* g, uint64_t seed) {
    uint64_t z = seed;
    for (int i = 0; i < 4; ++i) {
        z = sm64(z);
        g->s[i] = z;
    }
}
static uint64_t xo_next(xo_t* g) {
    uint64_t* s = g->s;
    const uint64_t r = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return r;
}
static double xo_u(xo_t* g) { return (double)(xo_next(g) >> 11) * 0x1.0p-53; }
static double xo_ur(xo_t* g, double lo, double hi) { return lo + (hi - lo) * xo_u(g); }

typedef struct {
    double x0, y0, x1, y1, v;
} rect_t;
typedef struct {
    double cx, cy, r, v;
} disc_t;
typedef struct {
    double v0, v1, ct, st, tmin, tinv;
    rect_t* rects;
    disc_t* discs;
    int nr, nd;
    uint64_t key;
    int w, h;
    double sigma;
} scene_t;

static double dmin(double a, double b) { return a < b ? a : b; }
static double dmax(double a, double b) { return a < b ? b : a; }

static void make_scene(scene_t* sc, int w, int h, uint64_t seed, int nr, int nd) {
    xo_t g;
    xo_seed(&g, seed);
    sc->v0 = xo_u(&g);
    sc->v1 = xo_u(&g);
    const double theta = xo_ur(&g, 0.0, 2.0 * M_PI);
    sc->ct = cos(theta);
    sc->st = sin(theta);
    const double cx[4] = {0.0, (double)w, 0.0, (double)w};
    const double cy[4] = {0.0, 0.0, (double)h, (double)h};
    double tmin = 1e300, tmax = -1e300;
    for (int i = 0; i < 4; ++i) {
        const double t = cx[i] * sc->ct + cy[i] * sc->st;
        tmin = dmin(tmin, t);
        tmax = dmax(tmax, t);
    }
    sc->tmin = tmin;
    sc->tinv = tmax > tmin ? 1.0 / (tmax - tmin) : 0.0;
    sc->rects = (rect_t*)malloc(sizeof(rect_t) * (size_t)(nr > 0 ? nr : 1));
    for (int i = 0; i < nr; ++i) {
        const double rw = xo_ur(&g, w / 64.0, w / 8.0);
        const double rh = xo_ur(&g, h / 64.0, h / 8.0);
        const double x0 = xo_ur(&g, 0.0, dmax(0.0, w - rw));
        const double y0 = xo_ur(&g, 0.0, dmax(0.0, h - rh));
        const double v = xo_u(&g);
        sc->rects[i] = (rect_t){x0, y0, x0 + rw, y0 + rh, v};
    }
    const double m = (double)(w < h ? w : h);
    sc->discs = (disc_t*)malloc(sizeof(disc_t) * (size_t)(nd > 0 ? nd : 1));
    for (int i = 0; i < nd; ++i) {
        const double dx = xo_ur(&g, 0.0, (double)w);
        const double dy = xo_ur(&g, 0.0, (double)h);
        const double r = xo_ur(&g, m / 128.0, m / 16.0);
        const double v = xo_u(&g);
        sc->discs[i] = (disc_t){dx, dy, r, v};
    }
    sc->nr = nr;
    sc->nd = nd;
    sc->key = sm64(seed ^ 0x6E6F697365ull);
    sc->w = w;
    sc->h = h;
}

static double gauss(uint64_t key, uint64_t i) {
    const uint64_t a = sm64(key ^ (2 * i));
    const uint64_t b = sm64(key ^ (2 * i + 1));
    const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(b >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

static void render_row(const scene_t* sc, int y, double* row) {
    const int w = sc->w;
    const double yc = y + 0.5;
    for (int x = 0; x < w; ++x) {
        const double t = ((x + 0.5) * sc->ct + yc * sc->st - sc->tmin) * sc->tinv;
        row[x] = sc->v0 + (sc->v1 - sc->v0) * t;
    }
    for (int i = 0; i < sc->nr; ++i) {
        const rect_t* r = &sc->rects[i];
        if (!(r->y0 <= yc && yc < r->y1)) continue;
        int xa = (int)ceil(r->x0 - 0.5), xb = (int)ceil(r->x1 - 0.5);
        if (xa < 0) xa = 0;
        if (xb > w) xb = w;
        for (int x = xa; x < xb; ++x) row[x] = r->v;
    }
    for (int i = 0; i < sc->nd; ++i) {
        const disc_t* d = &sc->discs[i];
        const double dy = yc - d->cy;
        const double rem = d->r * d->r - dy * dy;
        if (rem < 0.0) continue;
        const double hw = sqrt(rem);
        int xa = (int)floor(d->cx - hw - 0.5) - 1, xb = (int)ceil(d->cx + hw - 0.5) + 2;
        if (xa < 0) xa = 0;
        if (xb > w) xb = w;
        for (int x = xa; x < xb; ++x) {
            const double dx = x + 0.5 - d->cx;
            if (dx * dx + dy * dy <= d->r * d->r) row[x] = d->v;
        }
    }
    const uint64_t base = (uint64_t)y * (uint64_t)w;
    for (int x = 0; x < w; ++x) {
        const double v = row[x] + sc->sigma * gauss(sc->key, base + (uint64_t)x);
        row[x] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
}

typedef struct {
    const scene_t* sc;
    void* out;
    int64_t pitch;
    int u8;
    int y0, y1;
} job_t;

static void* job_run(void* a) {
    job_t* j = (job_t*)a;
    double* row = (double*)malloc(sizeof(double) * (size_t)j->sc->w);
    for (int y = j->y0; y < j->y1; ++y) {
        render_row(j->sc, y, row);
        if (j->u8) {
            uint8_t* o = (uint8_t*)j->out + (int64_t)y * j->pitch;
            for (int x = 0; x < j->sc->w; ++x) o[x] = (uint8_t)lrint(255.0 * row[x]);
        } else {
            float* o = (float*)j->out + (int64_t)y * j->pitch;
            for (int x = 0; x < j->sc->w; ++x) o[x] = (float)row[x];
        }
    }
    free(row);
    return NULL;
}

static int synth(void* out, int u8, int32_t w, int32_t h, int64_t pitch, uint64_t seed,
                 int32_t nr, int32_t nd, double sigma, int32_t threads) {
    if (!out || w <= 0 || h <= 0 || pitch < w || nr < 0 || nd < 0 || !(sigma >= 0.0)) return 1;
    scene_t sc;
    make_scene(&sc, w, h, seed, nr, nd);
    sc.sigma = sigma;
    int workers = threads > 0 ? threads : 1;
    if (workers > 256) workers = 256;
    if (workers > h) workers = h;
    if (h < 16) workers = 1;
    const int chunk = (h + workers - 1) / workers;
    pthread_t tid[256];
    job_t jobs[256];
    int started = 0;
    for (int k = 1; k < workers; ++k) {
        const int y0 = k * chunk, y1 = y0 + chunk < h ? y0 + chunk : h;
        if (y0 >= y1) break;
        jobs[k] = (job_t){&sc, out, pitch, u8, y0, y1};
        pthread_create(&tid[k], NULL, job_run, &jobs[k]);
        started = k;
    }
    jobs[0] = (job_t){&sc, out, pitch, u8, 0, chunk < h ? chunk : h};
    job_run(&jobs[0]);
    for (int k = 1; k <= started; ++k) pthread_join(tid[k], NULL);
    free(sc.rects);
    free(sc.discs);
    return 0;
}

OR_EXPORT int or_synth_f32(float* out, int32_t w, int32_t h, int64_t pitch, uint64_t seed,
                           int32_t n_rects, int32_t n_discs, double sigma, int32_t threads) {
    return synth(out, 0, w, h, pitch, seed, n_rects, n_discs, sigma, threads);
}

OR_EXPORT int or_synth_u8(uint8_t* out, int32_t w, int32_t h, int64_t pitch, uint64_t seed,
                          int32_t n_rects, int32_t n_discs, double sigma, int32_t threads) {
    return synth(out, 1, w, h, pitch, seed, n_rects, n_discs, sigma, threads);
}
