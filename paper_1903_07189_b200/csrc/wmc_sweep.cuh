// paper_1903_07189_b200/csrc/wmc_sweep.cuh -- the sm_100a WMC stencil and
// temporally blocked WMC-flow kernel.
//
// What it computes (reference: SPEC.md:171-179 wmc_half_laplace, :256-272
// mc_flow scheme=half_laplace; Eqs. 26-28): K synchronous (Jacobi)
// sweeps U <- U + dt * d_m(U) per launch, or (MAP) one evaluation of d_m.
// Arithmetic is the canonical fp32 sequence of DESIGN.md §3 (the same
// sequence oracle/wmc_oracle.c restates), written with explicit _rn
// intrinsics so nvcc can neither contract nor reassociate it.
//
// How: warp-streaming register blocking with packed fp32.
//  * A warp owns column windows of 32*C columns (C adjacent columns per
//    lane) and streams DOWN a strip of rows.  Each window overlaps its
//    neighbours by A >= K columns per side so the K levels of the trapezoid
//    never need another warp's data; horizontal neighbours come from warp
//    shuffles of each produced row.
//  * Packed fp32 across TWO column chunks: a warp owns chunk pair (2c, 2c+1);
//    lane position j (columns xf-1 .. xf+C of each chunk) is ONE 64-bit
//    register pair {chunk 2c value, chunk 2c+1 value}.  Every neighbour of a
//    pixel pair is then an aligned pair, so all canonical arithmetic runs as
//    sm_100 FFMA2/FADD2/FMUL2 (one instruction for two pixels) with no
//    register re-layout; loads/stores are per-column 4-byte accesses that
//    land directly in pair halves (the C accesses of a warp cover whole
//    128-byte lines).
//  * Level l (1..K) keeps a 3-row window of level l-1 in registers; row y of
//    level l lives in slot y mod 3, and the step loop is unrolled by 3 so
//    every slot index is a compile-time constant (no register moves).
//  * Row-shared pair sums (H = l+r, T = (a+c)+(l+r)) are carried down.
//  * Clamp-to-edge is re-applied to the CURRENT iterate at every
//    level: rows via slot copies at rows 0 / h, columns via selects after the
//    halo shuffle.  Only the (at most two) border warps of a row band and the
//    prologue/epilogue steps take this checked path; interior warps run a
//    branch-free steady state.  Level-0 rows are prefetched 3 rows ahead.
//  * Non-finite check: one FFMA2 per pixel pair per level into
//    a per-level accumulator; the first level whose accumulator is NaN is
//    atomically min-ed into a device flag.  A non-finite pixel stays
//    non-finite at every later iteration, so per-level checks
//    of each warp's own columns name the first bad iteration exactly.
//  * MAP mode resolves opposite-sign near-ties of the selection in fp64
//     so the map matches the fp64 SPEC evaluation to 1e-5.
//
// No shared memory, no block barriers: HBM traffic is one 4-byte read and one
// 4-byte write per pixel per launch (the overlap columns hit L2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cfk {

constexpr int kWarpsPerBlock = 4;
constexpr int kThreads = 32 * kWarpsPerBlock;
constexpr unsigned kFull = 0xffffffffu;
constexpr float kC12 = 1.0f / 12.0f;  // fl(1/12)
constexpr int C = 2;                  // columns per lane per chunk
#ifndef CF_MINB_K2
#define CF_MINB_K2 3
#endif
#ifndef CF_PD
#define CF_PD 3
#endif
#ifndef CF_CARRY
#define CF_CARRY 0
#endif

struct SweepParams {
    const void* src;          // global row src_row0 of plane 0 (float or uint8)
    float* dst;               // global row dst_row0 of plane 0
    int64_t src_pitch;        // elements of the source type
    int64_t dst_pitch;        // elements
    int64_t src_plane;        // plane stride, source elements
    int64_t dst_plane;        // plane stride, elements
    int32_t src_row0, dst_row0;
    int32_t w, h;             // global image size (clamp borders)
    int32_t y0, y1;           // output rows
    int32_t strip_rows, n_strips, n_chunks, planes;
    float dt;
    int32_t iter_base;
    int32_t* flag;            // nullable
};

// Column geometry for K levels.
template <int K>
struct Geo {
    static constexpr int A = ((K + C - 1) / C) * C;      // overlap per side, multiple of C
    static constexpr int S = 32 * C - 2 * A;             // output columns per warp
    static constexpr int LANE_LO = A / C;                // first output lane
    static constexpr int LANE_HI = LANE_LO + S / C;      // one past last output lane
    static_assert(A >= K && S > 0 && S % C == 0, "bad geometry");
};

// A packed pair of fp32 values held in ONE 64-bit register pair (PTX .b64),
// operated on with sm_100 add/mul/fma.rn.f32x2 (SASS FADD2/FMUL2/FFMA2).
// Keeping pairs as .b64 end to end avoids the per-use mov.b64 repacking that
// float2 + __fadd2_rn produce.
using f2 = unsigned long long;
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2 pk(float lo, float hi) {
    f2 d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
    return d;
}
__device__ __forceinline__ float lo(f2 v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return a;
}
__device__ __forceinline__ float hi(f2 v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return b;
}
__device__ __forceinline__ constexpr f2 splat_bits(uint32_t b) { return ((f2)b << 32) | b; }
__device__ __forceinline__ f2 splat(float v) { return pk(v, v); }
constexpr f2 kTwo2 = 0x4000000040000000ull;    // {2, 2}
constexpr f2 kFour2 = 0x4080000040800000ull;   // {4, 4}
constexpr f2 kM12x2 = 0xC1400000C1400000ull;   // {-12, -12}
constexpr f2 kC12x2 = 0x3DAAAAAB3DAAAAABull;   // {fl(1/12), fl(1/12)}
constexpr f2 kZero2 = 0ull;

// Level-0 prefetch ring (f32 inputs): each lane cp.async-copies its 2*C
// input values of row t+RD into shared memory, interleaved as
// {chunk0 col j, chunk1 col j} so that one 16-byte LDS returns the pairs
// ready for FFMA2.  No registers are held for in-flight rows.
constexpr int kRingRows = 8;
constexpr int kRingBytesPerWarp = kRingRows * 32 * 16;

__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One window row: positions p0..p5 (columns xf-1 .. xf+4), each a pair
// {chunk 2c, chunk 2c+1}.
struct Row {
    f2 q[C + 2];
};

// A prefetched level-0 row, kept as 32-bit scalars (chunk 0 in a, chunk 1
// in b) so the loads land in their own registers; they are packed into
// pairs only when consumed PD steps later.
struct Staged {
    float a[C], b[C];
};

struct Carry {
    f2 hc[C], tm[C];  // H(y) = l+r and T(y-1) = (a+c)+(l+r) of pixels p1..pC
};

// first-minimum of |.|: a tournament with the left operand
// winning ties; for finite inputs identical to the strict-< scan 1..8.
__device__ __forceinline__ float pick(float l, float r) { return fabsf(r) < fabsf(l) ? r : l; }
__device__ __forceinline__ float select8(float d1, float d2, float d3, float d4, float d5,
                                         float d6, float d7, float d8) {
    return pick(pick(pick(d1, d2), pick(d3, d4)), pick(pick(d5, d6), pick(d7, d8)));
}

// Canonical D_1..D_8 (= 12 * d_i) of a pixel pair.
struct PairD {
    f2 d[8];
    f2 n12u;
};

__device__ __forceinline__ void pair_d(f2 a, f2 b, f2 c, f2 l, f2 u, f2 r, f2 e, f2 f, f2 g,
                                       f2 Wm, f2 W0, f2 Hc, f2 Tm, f2& Hb_out, f2& T0_out,
                                       PairD& P) {
    const f2 two = kTwo2, four = kFour2;
    P.n12u = mul2(u, kM12x2);
    const f2 Hb = add2(e, g);
    const f2 T0 = add2(Hc, Hb);
    P.d[0] = fma2(two, fma2(two, l, Wm), P.n12u);
    P.d[1] = fma2(two, fma2(two, b, Tm), P.n12u);
    P.d[2] = fma2(two, fma2(two, r, W0), P.n12u);
    P.d[3] = fma2(two, fma2(two, f, T0), P.n12u);
    const f2 K5 = add2(c, e), K6 = add2(a, g);
    P.d[4] = add2(fma2(four, add2(b, l), fma2(two, a, K5)), P.n12u);
    P.d[5] = add2(fma2(four, add2(b, r), fma2(two, c, K6)), P.n12u);
    P.d[6] = add2(fma2(four, add2(r, f), fma2(two, g, K5)), P.n12u);
    P.d[7] = add2(fma2(four, add2(l, f), fma2(two, e, K6)), P.n12u);
    Hb_out = Hb;
    T0_out = T0;
}

__device__ __forceinline__ f2 select_pair(const PairD& P) {
    return pk(select8(lo(P.d[0]), lo(P.d[1]), lo(P.d[2]), lo(P.d[3]), lo(P.d[4]), lo(P.d[5]),
                      lo(P.d[6]), lo(P.d[7])),
              select8(hi(P.d[0]), hi(P.d[1]), hi(P.d[2]), hi(P.d[3]), hi(P.d[4]), hi(P.d[5]),
                      hi(P.d[6]), hi(P.d[7])));
}

// ---- fp64 near-tie resolution (MAP only) -------------------
// Opposite-sign near tie: some D_j with D_j + D_m ~ 0 while |D_m| is not ~0.
__device__ __forceinline__ bool near_tie(const PairD& P, int half, float best) {
    float T = 3.0e38f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float dk = half ? hi(P.d[k]) : lo(P.d[k]);
        T = fminf(T, fabsf(__fadd_rn(dk, best)));
    }
    const float n12u = half ? hi(P.n12u) : lo(P.n12u);
    const float tau = __fmaf_rn(fabsf(n12u), 0x1.8p-19f, __fmul_rn(fabsf(best), 0x1.0p-20f));
    return T <= tau && T < fabsf(best);
}

// SPEC-faithful fp64 evaluation of one pixel (oracle/wmc_px.h wmc_px_f64):
// weights n/12 as double, taps in row-major order, s = s + w*x unfused,
// strict-< first-minimum scan.
__device__ __noinline__ float wmc_px_f64(float a, float b, float c, float l, float u, float r,
                                          float e, float f, float g) {
    constexpr signed char H12[8][9] = {
        {2, 2, 0, 4, -12, 0, 2, 2, 0}, {2, 4, 2, 2, -12, 2, 0, 0, 0},
        {0, 2, 2, 0, -12, 4, 0, 2, 2}, {0, 0, 0, 2, -12, 2, 2, 4, 2},
        {2, 4, 1, 4, -12, 0, 1, 0, 0}, {1, 4, 2, 0, -12, 4, 0, 0, 1},
        {0, 0, 1, 0, -12, 4, 1, 4, 2}, {1, 0, 0, 4, -12, 0, 2, 4, 1}};
    const double x[9] = {a, b, c, l, u, r, e, f, g};
    double best = 0.0;
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int n = H12[i][t];
            const double wgt = n == 0 ? 0.0 : (n == -12 ? -1.0 : __ddiv_rn((double)n, 12.0));
            s = __dadd_rn(s, __dmul_rn(wgt, x[t]));
        }
        if (i == 0 || fabs(s) < fabs(best)) best = s;
    }
    return __double2float_rn(best);
}

template <int K, bool MAP, bool VEC, bool U8>
struct SweepWarp {
    using G = Geo<K>;
    static constexpr int NL = K;  // windows for levels 0..K-1
    static constexpr int PD = CF_PD;  // level-0 prefetch distance (rows): 1 or 3

    const SweepParams& P;
    int lane;
    int xf[2];                    // first column of this lane in each chunk
    bool out_lane;                // lane holds output columns
    bool out_h[2];                // chunk h exists (second chunk may be past w)
    bool border;                  // some window touches column 0 or w-1 (uniform)
    bool clampL[2];               // this lane holds column 0 (per chunk)
    int clampR[2];                // position (1..4) holding column w-1, else 0
    int ys, ye;                   // output strip rows
    int rlo[K + 1], rhi[K + 1];   // rows computed per level
    const unsigned char* srcp;    // plane base (bytes)
    float* dstp;                  // plane base

    Row win[NL][3];
    Carry cr[K + 1];
    Staged stage[U8 ? PD : 1];     // u8 inputs: register prefetch
    uint32_t ring;                 // f32 inputs: shared address of this lane's ring row 0
    int rslot;                     // ring slot of the row consumed at the current step
    f2 acc[K + 1];

    __device__ __forceinline__ SweepWarp(const SweepParams& p) : P(p) {}

    static __device__ __forceinline__ constexpr int md3(int r) { return ((r % 3) + 3) % 3; }

    // ---- level-0 loads (raw; widening handled at consume time) ----------
    __device__ __forceinline__ const unsigned char* src_row(int y) const {
        return srcp + (int64_t)(y - P.src_row0) * P.src_pitch * (U8 ? 1 : 4);
    }
    __device__ __forceinline__ float* dst_row(int y) const {
        return dstp + (int64_t)(y - P.dst_row0) * P.dst_pitch;
    }

    // CHECKED: rowp is the row start, columns clamped to [0, w).
    // fast:    rowp already points at column xf[0]; chunk 1 is G::S columns on.
    template <bool CHECKED>
    __device__ __forceinline__ Staged load_row(const unsigned char* rowp) const {
        Staged st;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            int x0 = j, x1 = G::S + j;  // fast: rowp points at column xf[0]
            if (CHECKED) {
                x0 = min(max(xf[0] + j, 0), P.w - 1);
                x1 = min(max(xf[1] + j, 0), P.w - 1);
            }
            if constexpr (U8) {
                st.a[j] = __uint_as_float((uint32_t)__ldg(rowp + x0));
                st.b[j] = __uint_as_float((uint32_t)__ldg(rowp + x1));
            } else {
                const float* row = reinterpret_cast<const float*>(rowp);
                st.a[j] = __ldg(row + x0);
                st.b[j] = __ldg(row + x1);
            }
        }
        return st;
    }

    // f32 prefetch: copy this lane's values of one row into ring slot `slot`.
    template <bool CHECKED>
    __device__ __forceinline__ void ring_issue(const unsigned char* rowp, int slot) const {
        const float* row = reinterpret_cast<const float*>(rowp);
        const uint32_t sa = ring + (uint32_t)slot * (32 * 16);
#pragma unroll
        for (int j = 0; j < C; ++j) {
            int x0 = j, x1 = G::S + j;  // fast: rowp points at column xf[0]
            if (CHECKED) {
                x0 = min(max(xf[0] + j, 0), P.w - 1);
                x1 = min(max(xf[1] + j, 0), P.w - 1);
            }
            cp_async4(sa + 8 * j, row + x0);
            cp_async4(sa + 8 * j + 4, row + x1);
        }
        cp_async_commit();
    }
    __device__ __forceinline__ void ring_consume(int slot, f2 (&v)[C]) const {
        static_assert(C == 2, "ring rows hold 2 pairs per lane");
        const uint32_t sa = ring + (uint32_t)slot * (32 * 16);
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "r"(sa));
    }

    __device__ __forceinline__ f2 widen(float a, float b) const {
        if constexpr (U8) {  // (float)q / 255 in IEEE fp32
            return pk(__fdiv_rn((float)__float_as_uint(a), 255.0f),
                      __fdiv_rn((float)__float_as_uint(b), 255.0f));
        } else {
            return pk(a, b);
        }
    }

    // Build a window row from the lane's positions p1..p4: halo shuffles,
    // then (CLAMP) clamp-to-edge at the image's first/last column.
    template <bool CLAMP>
    __device__ __forceinline__ void make_row(Row& R, const f2 (&v)[C]) const {
#pragma unroll
        for (int j = 0; j < C; ++j) R.q[j + 1] = v[j];
        const float l0 = __shfl_up_sync(kFull, lo(v[C - 1]), 1);  // left lane's pC
        const float l1 = __shfl_up_sync(kFull, hi(v[C - 1]), 1);
        const float r0 = __shfl_down_sync(kFull, lo(v[0]), 1);  // right lane's p1
        const float r1 = __shfl_down_sync(kFull, hi(v[0]), 1);
        R.q[0] = pk(l0, l1);
        R.q[C + 1] = pk(r0, r1);
        if constexpr (CLAMP) {
            float a[C + 2], b[C + 2];
#pragma unroll
            for (int i = 0; i < C + 2; ++i) { a[i] = lo(R.q[i]); b[i] = hi(R.q[i]); }
            if (clampL[0]) a[0] = a[1];
            if (clampL[1]) b[0] = b[1];
#pragma unroll
            for (int i = 1; i <= C; ++i) {
                if (clampR[0] == i) a[i + 1] = a[i];
                if (clampR[1] == i) b[i + 1] = b[i];
            }
            // columns >= w hold pitch padding or clamped loads: keep finite
#pragma unroll
            for (int i = 1; i <= C; ++i) {
                if (xf[0] + i - 1 > P.w) a[i] = 0.0f;
                if (xf[1] + i - 1 > P.w) b[i] = 0.0f;
            }
#pragma unroll
            for (int i = 0; i < C + 2; ++i) R.q[i] = pk(a[i], b[i]);
        }
    }

    // ---- level 0 of one step: consume the prefetched row, prefetch ahead --
    template <int PH, bool CHECKED>
    __device__ __forceinline__ void level0(int t, const unsigned char*& lptr) {
        constexpr int s_y = md3(PH), s_ym = md3(PH - 1);
        f2 v[C];
        if constexpr (!U8) {
            cp_async_wait<kRingRows - 1>();        // row t has landed
            ring_consume(rslot, v);
        }
        if (!CHECKED || (t >= rlo[0] && t < rhi[0])) {
            if constexpr (U8) {
#pragma unroll
                for (int j = 0; j < C; ++j)
                    v[j] = widen(stage[PH % PD].a[j], stage[PH % PD].b[j]);
            }
            make_row<CHECKED>(win[0][s_y], v);
            if (CHECKED && t == 0) win[0][s_ym] = win[0][s_y];  // row -1 := row 0
        } else if (CHECKED && t == P.h && rhi[0] == P.h) {
            win[0][s_y] = win[0][s_ym];                          // row h := row h-1
        }
        constexpr int AHEAD = U8 ? PD : kRingRows;
        if constexpr (U8) {
            if (CHECKED) {
                stage[PH % PD] = load_row<true>(src_row(min(max(t + PD, rlo[0]), rhi[0] - 1)));
            } else {
                stage[PH % PD] = load_row<false>(lptr);  // row t + PD
                lptr += P.src_pitch;
            }
        } else {
            if (CHECKED) {
                ring_issue<true>(src_row(min(max(t + AHEAD, rlo[0]), rhi[0] - 1)), rslot);
            } else {
                ring_issue<false>(lptr, rslot);          // row t + kRingRows
                lptr += P.src_pitch * 4;
            }
            rslot = rslot + 1 == kRingRows ? 0 : rslot + 1;
        }
    }

    // ---- level L >= 1 of one step ---------------------------------------
    template <int PH, int L, bool CHECKED>
    __device__ __forceinline__ void level(int t, float*& sptr) {
        const int y = t - L;
        constexpr int s_y = md3(PH - L);        // slot of row y
        constexpr int s_ym = md3(PH - L - 1);   // slot of row y-1
        constexpr int s_yp = md3(PH - L + 1);   // slot of row y+1
        if (!CHECKED || (y >= rlo[L] && y < rhi[L])) {
            const f2 (&m)[C + 2] = win[L - 1][s_ym].q;
            const f2 (&o)[C + 2] = win[L - 1][s_y].q;
            const f2 (&p)[C + 2] = win[L - 1][s_yp].q;
            Carry& cc = cr[L];
            if ((CHECKED && y == rlo[L]) || !CF_CARRY) {
#pragma unroll
                for (int j = 1; j <= C; ++j) {
                    cc.hc[j - 1] = add2(o[j - 1], o[j + 1]);                       // l + r
                    cc.tm[j - 1] = add2(add2(m[j - 1], m[j + 1]), cc.hc[j - 1]);  // (a+c)+(l+r)
                }
            }
            f2 V[C + 2];
#pragma unroll
            for (int i = 0; i < C + 2; ++i) V[i] = add2(m[i], p[i]);              // a+e / b+f / c+g
            f2 W[C + 1];
#pragma unroll
            for (int i = 0; i < C + 1; ++i) W[i] = add2(V[i], V[i + 1]);          // (a+e)+(b+f)
            f2 nv[C];
#pragma unroll
            for (int j = 1; j <= C; ++j) {
                PairD D;
                f2 hb, t0;
                pair_d(m[j - 1], m[j], m[j + 1], o[j - 1], o[j], o[j + 1], p[j - 1], p[j],
                       p[j + 1], W[j - 1], W[j], cc.hc[j - 1], cc.tm[j - 1], hb, t0, D);
                cc.hc[j - 1] = hb;
                cc.tm[j - 1] = t0;
                const f2 b = select_pair(D);
                f2 hw = mul2(b, kC12x2);
                if constexpr (MAP) {
                    const bool t0_ = near_tie(D, 0, lo(b)), t1_ = near_tie(D, 1, hi(b));
                    if (__any_sync(kFull, t0_ | t1_)) {
                        float h0 = lo(hw), h1 = hi(hw);
                        if (t0_) h0 = wmc_px_f64(lo(m[j - 1]), lo(m[j]), lo(m[j + 1]),
                                                 lo(o[j - 1]), lo(o[j]), lo(o[j + 1]),
                                                 lo(p[j - 1]), lo(p[j]), lo(p[j + 1]));
                        if (t1_) h1 = wmc_px_f64(hi(m[j - 1]), hi(m[j]), hi(m[j + 1]),
                                                 hi(o[j - 1]), hi(o[j]), hi(o[j + 1]),
                                                 hi(p[j - 1]), hi(p[j]), hi(p[j + 1]));
                        hw = pk(h0, h1);
                    }
                    nv[j - 1] = hw;
                } else {
                    nv[j - 1] = fma2(splat(P.dt), hw, o[j]);   // u + dt * H^w
                    acc[L] = fma2(nv[j - 1], kZero2, acc[L]);
                }
            }
            if constexpr (L == K) {
                if (CHECKED) {
                    store_row<true>(dst_row(y), nv);
                } else {
                    store_row<false>(sptr, nv);  // row t - K
                    sptr += P.dst_pitch;
                }
            } else {
                make_row<CHECKED>(win[L][s_y], nv);
                if (CHECKED && y == 0) win[L][s_ym] = win[L][s_y];
            }
        } else if constexpr (L < K) {
            if (y == P.h && rhi[L] == P.h) win[L][s_y] = win[L][s_ym];
        }
    }

    // CHECKED: row is the row start; fast: row points at column xf[0].
    template <bool CHECKED>
    __device__ __forceinline__ void store_row(float* row, const f2 (&nv)[C]) const {
        if (!out_lane) return;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            if (CHECKED) {
                if (out_h[0] && xf[0] + j < P.w) row[xf[0] + j] = lo(nv[j]);
                if (out_h[1] && xf[1] + j < P.w) row[xf[1] + j] = hi(nv[j]);
            } else {
                row[j] = lo(nv[j]);
                row[G::S + j] = hi(nv[j]);
            }
        }
    }

    template <int PH, int L, bool CHECKED>
    __device__ __forceinline__ void levels(int t, float*& sptr) {
        level<PH, L, CHECKED>(t, sptr);
        if constexpr (L < K) levels<PH, L + 1, CHECKED>(t, sptr);
    }

    template <int PH, bool CHECKED>
    __device__ __forceinline__ void step(int t, int t_begin, int t_end,
                                         const unsigned char*& lptr, float*& sptr) {
        level0<PH, CHECKED>(t, lptr);  // prefetch keeps running even for skipped steps
        if (CHECKED && (t < t_begin || t > t_end)) return;
        levels<PH, 1, CHECKED>(t, sptr);
    }

    __device__ __forceinline__ void run() {
        const int t_begin = rlo[0];
        const int t_end = ye - 1 + K;
        // steady steps: every level past its first row, no clamp copies,
        // prefetch in range, no clamp columns
        const int t_s = border ? 0x7fffffff : ys + K + 1;
        constexpr int AHEAD = U8 ? PD : kRingRows;
        const int t_e = min(ye + K, P.h) - 1 - AHEAD;
#pragma unroll
        for (int L = 0; L <= K; ++L) acc[L] = kZero2;
        const int tb0 = t_begin - t_begin % 3;
#pragma unroll
        for (int i = 0; i < AHEAD; ++i) {
            const unsigned char* rp = src_row(min(max(tb0 + i, rlo[0]), rhi[0] - 1));
            if constexpr (U8) stage[i] = load_row<true>(rp);
            else              ring_issue<true>(rp, i);
        }
        rslot = 0;
        const unsigned char* lptr = nullptr;
        float* sptr = nullptr;
        bool fast_prev = false;
        for (int tb = tb0; tb <= t_end; tb += 3) {
            if (tb >= t_s && tb + 2 <= t_e) {
                if (!fast_prev) {  // (re)seed the running row pointers (at column xf[0])
                    lptr = src_row(tb + AHEAD) + (int64_t)xf[0] * (U8 ? 1 : 4);
                    sptr = dst_row(tb - K) + xf[0];
                    fast_prev = true;
                }
                step<0, false>(tb, t_begin, t_end, lptr, sptr);
                step<1, false>(tb + 1, t_begin, t_end, lptr, sptr);
                step<2, false>(tb + 2, t_begin, t_end, lptr, sptr);
            } else {
                fast_prev = false;
                step<0, true>(tb, t_begin, t_end, lptr, sptr);
                step<1, true>(tb + 1, t_begin, t_end, lptr, sptr);
                step<2, true>(tb + 2, t_begin, t_end, lptr, sptr);
            }
        }
    }
};

// Resident blocks per SM the register allocation is held to (occupancy vs
// spills; measured): 16 warps/SM for K <= 2, 12 for K = 3.
template <int K>
struct MinBlocks {
    static constexpr int value = K <= 2 ? CF_MINB_K2 : (K == 3 ? 3 : 2);
};

template <int K, bool MAP, bool VEC, bool U8>
__global__ void __launch_bounds__(kThreads, MinBlocks<K>::value)
    wmc_sweeps_kernel(const SweepParams p) {
    using G = Geo<K>;
    const int warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int n_pairs = (p.n_chunks + 1) / 2;
    const int total = n_pairs * p.n_strips * p.planes;
    if (warp >= total) return;  // warp-uniform
    const int cpair = warp % n_pairs;
    const int rest = warp / n_pairs;
    const int strip = rest % p.n_strips;
    const int plane = rest / p.n_strips;

    SweepWarp<K, MAP, VEC, U8> sw(p);
    sw.lane = threadIdx.x & 31;
    sw.out_lane = sw.lane >= G::LANE_LO && sw.lane < G::LANE_HI;
    sw.border = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int chunk = 2 * cpair + h;
        const int xs = chunk * G::S - G::A;
        sw.out_h[h] = chunk < p.n_chunks;
        // a missing second chunk mirrors the first (finite data, never stored)
        sw.xf[h] = (sw.out_h[h] ? xs : xs - G::S) + sw.lane * C;
        sw.border |= xs < 0 || xs + 32 * C > p.w || !sw.out_h[h];
        sw.clampL[h] = sw.xf[h] == 0;
        sw.clampR[h] = (p.w - 1 >= sw.xf[h] && p.w - 1 < sw.xf[h] + C) ? p.w - sw.xf[h] : 0;
    }
    sw.ys = p.y0 + strip * p.strip_rows;
    sw.ye = min(sw.ys + p.strip_rows, p.y1);
    if (sw.ys >= sw.ye) return;
#pragma unroll
    for (int L = 0; L <= K; ++L) {
        sw.rlo[L] = max(sw.ys - (K - L), 0);
        sw.rhi[L] = min(sw.ye + (K - L), p.h);
    }
    const int esz = U8 ? 1 : 4;
    sw.srcp = reinterpret_cast<const unsigned char*>(p.src) + (int64_t)plane * p.src_plane * esz;
    if constexpr (!U8) {
        extern __shared__ __align__(16) unsigned char smem_ring[];
        sw.ring = (uint32_t)__cvta_generic_to_shared(smem_ring) +
                  (uint32_t)(threadIdx.x >> 5) * kRingBytesPerWarp + (uint32_t)sw.lane * 16;
    }
    sw.dstp = p.dst + (int64_t)plane * p.dst_plane;

    sw.run();

    if constexpr (!MAP) {
        if (p.flag) {
            int bad = 0x7fffffff;
#pragma unroll
            for (int L = K; L >= 1; --L) {
                const float ax = cfk::lo(sw.acc[L]), ay = cfk::hi(sw.acc[L]);
                if (sw.out_lane && (ax != ax || (sw.out_h[1] && ay != ay))) bad = p.iter_base + L;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(kFull, bad, o));
            if (sw.lane == 0 && bad != 0x7fffffff) atomicMin(p.flag, bad);
        }
    }
}

}  // namespace cfk
