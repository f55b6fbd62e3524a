/*
 * oracle/wmc_px.h -- per-pixel restatements shared by the oracle's C
 * (wmc_oracle.c) and C++ (ref_exec.cpp) translation units.
 * TEST INFRASTRUCTURE ONLY (see wmc_oracle.c header).
 */
#ifndef CF_ORACLE_WMC_PX_H
#define CF_ORACLE_WMC_PX_H
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <pthread.h>

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ------------------------------------------------------------------------ */
/* Kernel bank h1..h8.  Stored as exact   */
/* integer numerators over 12, lowered to double once.         */
/* Index [i][row][col], row = dy+1 (top to bottom), col = dx+1 (left to      */
/* right) -- the Stencil3 orientation of SPEC.md:41 / :77.                   */
/* ------------------------------------------------------------------------ */
static const int H12[8][3][3] = {
    /* h1 left half   */ {{2, 2, 0}, {4, -12, 0}, {2, 2, 0}},
    /* h2 top half    */ {{2, 4, 2}, {2, -12, 2}, {0, 0, 0}},
    /* h3 right half  */ {{0, 2, 2}, {0, -12, 4}, {0, 2, 2}},
    /* h4 bottom half */ {{0, 0, 0}, {2, -12, 2}, {2, 4, 2}},
    /* h5 upper-left  */ {{2, 4, 1}, {4, -12, 0}, {1, 0, 0}},
    /* h6 upper-right */ {{1, 4, 2}, {0, -12, 4}, {0, 0, 1}},
    /* h7 lower-right */ {{0, 0, 1}, {0, -12, 4}, {1, 4, 2}},
    /* h8 lower-left  */ {{1, 0, 0}, {4, -12, 0}, {2, 4, 1}},
};

static inline void kernel_bank_numerators(int32_t* out72) {
    for (int i = 0; i < 8; ++i)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) out72[i * 9 + r * 3 + c] = H12[i][r][c];
}

static double HW64[8][3][3];
static pthread_once_t hw_once = PTHREAD_ONCE_INIT;
static void init_hw64(void) {
    for (int i = 0; i < 8; ++i)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                int n = H12[i][r][c];
                /* exact rationals: n/12 reduced -> 1/6, 1/3, 1/12, -1, 0 */
                HW64[i][r][c] = n == 0 ? 0.0 : (n == -12 ? -1.0 : (double)n / 12.0);
            }
}

static inline double wmc_px_f64(const double* in, int w, int h, int64_t pitch, int y, int x,
                                int* m_out) {
    double d[8];
    for (int i = 0; i < 8; ++i) {
        double s = 0.0;
        for (int r = 0; r < 3; ++r) {          /* SPEC.md:56 correlation, row-major taps */
            int yy = clampi(y + r - 1, 0, h - 1);   /* clamp-to-edge */
            const double* row = in + (int64_t)yy * pitch;
            for (int c = 0; c < 3; ++c) {
                int xx = clampi(x + c - 1, 0, w - 1);
                s = s + HW64[i][r][c] * row[xx];
            }
        }
        d[i] = s;
    }
    int m = 0;                                   /* SPEC.md:173, :195 strict <, first min */
    for (int i = 1; i < 8; ++i)
        if (fabs(d[i]) < fabs(d[m])) m = i;
    if (m_out) *m_out = m;
    return d[m];
}

/* ------------------------------------------------------------------------ */
/* fp32 canonical evaluation, every rounding pinned.  */
/*                                                                           */
/*   a b c        12*d1 = 2((a+e)+(b+f)) + 4l - 12u       (h1)               */
/*   l u r        12*d2 = 2((a+c)+(l+r)) + 4b - 12u       (h2)               */
/*   e f g        12*d3 = 2((b+f)+(c+g)) + 4r - 12u       (h3)               */
/*                12*d4 = 2((l+r)+(e+g)) + 4f - 12u       (h4)               */
/*                12*d5 = 4(b+l) + 2a + ((c+e) - 12u)     (h5)               */
/*                12*d6 = 4(b+r) + 2c + ((a+g) - 12u)     (h6)               */
/*                12*d7 = 4(r+f) + 2g + ((c+e) - 12u)     (h7)               */
/*                12*d8 = 4(l+f) + 2e + ((a+g) - 12u)     (h8)               */
/*                                                                           */
/* ×2 and ×4 are exact, so fmaf(2,x,y) is the single rounding of 2x+y.       */
/* n12u = fl(u * -12) is formed once and ADDED; D1..D4 of a constant image   */
/* are exact zeros (fl(2*fl(6u)) == fl(12u)) and D1 wins the selection, so   */
/* the map / flow of a constant is exact.  D_m selected by strict < on |D|   */
/* scanning 1..8; map H^w = fl(D_m * fl(1/12)); flow step                  */
/* fmaf(fl(dt * fl(1/12)), D_m, u) (the 1/12 folded into the step).          */
/* ------------------------------------------------------------------------ */
static const float C12 = 1.0f / 12.0f; /* fl(1/12) = 0x3DAAAAAB */

/* first-minimum of |.| as a tournament, left operand wins ties; for finite
 * inputs identical to the strict-< scan i = 1..8 of SPEC.md:195. */
static inline float pick_f32(float l, float r) { return fabsf(r) < fabsf(l) ? r : l; }

typedef struct {
    float D[8];   /* 12 * d_i */
    float n12u;   /* fl(-12 u) */
    float best;   /* selected D_m */
} px32;

static inline void wmc_px_f32_full(float a, float b, float c, float l, float u, float r, float e,
                                   float f, float g, px32* o) {
    const float n12u = u * -12.0f;
    const float Vl = a + e, Vc = b + f, Vr = c + g;
    const float Wm = Vl + Vc, W0 = Vc + Vr;
    const float Ht = a + c, Hc = l + r, Hb = e + g;
    const float Tm = Ht + Hc, T0 = Hc + Hb;
    o->n12u = n12u;
    o->D[0] = fmaf(2.0f, fmaf(2.0f, l, Wm), n12u);
    o->D[1] = fmaf(2.0f, fmaf(2.0f, b, Tm), n12u);
    o->D[2] = fmaf(2.0f, fmaf(2.0f, r, W0), n12u);
    o->D[3] = fmaf(2.0f, fmaf(2.0f, f, T0), n12u);
    const float K5 = (c + e) + n12u, K6 = (a + g) + n12u;
    const float Pbl = b + l, Pbr = b + r, Prf = r + f, Plf = l + f;
    o->D[4] = fmaf(4.0f, Pbl, fmaf(2.0f, a, K5));
    o->D[5] = fmaf(4.0f, Pbr, fmaf(2.0f, c, K6));
    o->D[6] = fmaf(4.0f, Prf, fmaf(2.0f, g, K5));
    o->D[7] = fmaf(4.0f, Plf, fmaf(2.0f, e, K6));
    const float* D = o->D;
    o->best = pick_f32(pick_f32(pick_f32(D[0], D[1]), pick_f32(D[2], D[3])),
                       pick_f32(pick_f32(D[4], D[5]), pick_f32(D[6], D[7])));
}

/* H^w of the flow: fl(D_m * fl(1/12)). */
static inline float wmc_px_f32(float a, float b, float c, float l, float u, float r, float e,
                               float f, float g) {
    px32 o;
    wmc_px_f32_full(a, b, c, l, u, r, e, f, g, &o);
    return o.best * C12;
}

/* The map's selection and opposite-sign near-tie test.
 * U = min of the eight D_k's bit patterns as unsigned, S = as signed: when
 * both signs occur (U != S), P = U is the smallest-magnitude non-negative
 * D and N = S the smallest-magnitude negative one, so x = fl(P + N) says
 * which is the minimum magnitude (x > 0: N, x < 0: P) and |x| is the
 * distance of the opposite-sign runner-up, i.e. min_k |fl(D_k + D_m)| over
 * the opposite-sign k (same-sign k are >= 2|D_m| and never near a tie).
 * When all D share a sign, U == S is the minimum.  Only an exact
 * opposite-sign tie (or a NaN x) needs the first index: the tournament.
 * For finite, non-overflowing D this is exactly the strict-< first-minimum
 * scan of SPEC.md:195 and the T = min_k |fl(D_k + D_m)| rule of round 1.
 * tau = fmaf(|n12u|, 1.5*2^-19, fl(|D_m| * 2^-20)); tie iff |x| <= tau and
 * |x| < |D_m|. */
static inline float map_best_f32(const px32* o, int* tie) {
    uint32_t U, v;
    int32_t S, sv;
    memcpy(&U, &o->D[0], 4);
    S = (int32_t)U;
    for (int k = 1; k < 8; ++k) {
        memcpy(&v, &o->D[k], 4);
        sv = (int32_t)v;
        U = v < U ? v : U;
        S = sv < S ? sv : S;
    }
    float P, N;
    memcpy(&P, &U, 4);
    memcpy(&N, &S, 4);
    const float x = P + N;
    float b = x > 0.0f ? N : P;
    if (U != (uint32_t)S && !(x > 0.0f || x < 0.0f)) b = o->best; /* exact tie / NaN */
    const float tau = fmaf(fabsf(o->n12u), 0x1.8p-19f, fabsf(b) * 0x1.0p-20f);
    const float ax = fabsf(x);
    *tie = (ax <= tau) && (ax < fabsf(b));
    return b;
}

/* The map: canonical fp32, with opposite-sign near-ties resolved by the
 * SPEC-faithful fp64 evaluation rounded to fp32. */
static inline float wmc_map_px_f32(float a, float b, float c, float l, float u, float r, float e,
                                   float f, float g, int* tie) {
    px32 o;
    wmc_px_f32_full(a, b, c, l, u, r, e, f, g, &o);
    int t;
    const float best = map_best_f32(&o, &t);
    if (t) {
        pthread_once(&hw_once, init_hw64);
        const double nb[9] = {a, b, c, l, u, r, e, f, g};
        double best64 = 0.0;
        for (int i = 0; i < 8; ++i) {
            double s = 0.0;
            for (int k = 0; k < 9; ++k) s = s + HW64[i][k / 3][k % 3] * nb[k];
            if (i == 0 || fabs(s) < fabs(best64)) best64 = s;
        }
        if (tie) *tie = 1;
        return (float)best64;
    }
    if (tie) *tie = 0;
    return best * C12;
}
#endif
