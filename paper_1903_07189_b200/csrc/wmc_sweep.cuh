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
// How: warp-streaming register blocking.
//  * A warp owns a column window of 32*C columns (C adjacent columns per lane,
//    loaded with one 16-byte LDG per row) and streams DOWN a strip of rows.
//    The window overlaps its neighbours by A >= K columns per side so the K
//    levels of the trapezoid never need data from another warp; horizontal
//    neighbours come from two warp shuffles per produced row.
//  * Level l (1..K) keeps a 3-row window of level l-1 in registers; row y of
//    level l lives in slot y mod 3, and the step loop is unrolled by 3 so
//    every slot index is a compile-time constant (no register moves).
//  * Pair sums shared between neighbouring pixels (V/W across columns, H/T
//    and the L-shaped pairs across rows) are carried in registers.
//  * Clamp-to-edge is re-applied to the CURRENT iterate at every
//    level: rows via slot copies at rows 0 / h, columns via selects in the
//    two border warps of each row (uniform branch; interior warps pay none).
//  * Non-finite check: one FFMA per output pixel per level
//    into a per-level accumulator; the first level whose accumulator is NaN
//    is atomically min-ed into a device flag.  A non-finite pixel stays
//    non-finite at every later iteration, so per-level checks
//    of each warp's own columns name the first bad iteration exactly.
//
// No shared memory, no block barriers: HBM traffic is one 4-byte read and one
// 4-byte write per pixel per launch (plus the A/32C overlap, served by L2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cfk {

constexpr int kWarpsPerBlock = 4;
constexpr int kThreads = 32 * kWarpsPerBlock;
constexpr unsigned kFull = 0xffffffffu;
constexpr float kC12 = 1.0f / 12.0f;  // fl(1/12)

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

// Column geometry for C columns per lane, K levels.
template <int C, int K>
struct Geo {
    static constexpr int A = ((K + C - 1) / C) * C;      // overlap per side, multiple of C
    static constexpr int S = 32 * C - 2 * A;             // output columns per warp
    static constexpr int LANE_LO = A / C;                // first output lane
    static constexpr int LANE_HI = LANE_LO + S / C;      // one past last output lane
    static_assert(A >= K && S > 0 && S % C == 0, "bad geometry");
};

template <int C>
struct Carry {
    float hb[C], t0[C], q1[C], q2[C];
};

__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float fsel_min_abs(float best, float d) {
    return fabsf(d) < fabsf(best) ? d : best;
}

// Carries for the first row a level produces in a strip: the row-shared pair
// sums of row y computed directly from rows y-1 (m) and y (o), with the same
// operands in the same order as wmc_row forms them for row y+1.
template <int C>
__device__ __forceinline__ void init_carry(const float (&m)[C + 2], const float (&o)[C + 2],
                                           Carry<C>& cr) {
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const float a = m[j], b = m[j + 1], c = m[j + 2];
        const float l = o[j], r = o[j + 2];
        cr.hb[j] = fadd(l, r);                 // H(y)   = l + r
        cr.t0[j] = fadd(fadd(a, c), cr.hb[j]); // T(y-1) = (a + c) + (l + r)
        cr.q1[j] = fadd(b, l);                 // b + l
        cr.q2[j] = fadd(b, r);                 // b + r
    }
}

// One produced row of C pixels from the 3-row window (m, o, p) of the
// previous level (each C+2 wide: position 0 = left halo, C+1 = right halo),
// using the carries of the row above; updates the carries for the row below.
// Writes the selected D_m (= 12 * d_m) of each pixel.
template <int C>
__device__ __forceinline__ void wmc_row(const float (&m)[C + 2], const float (&o)[C + 2],
                                        const float (&p)[C + 2], Carry<C>& cr,
                                        float (&best)[C]) {
    float V[C + 2];
#pragma unroll
    for (int i = 0; i < C + 2; ++i) V[i] = fadd(m[i], p[i]);           // a+e / b+f / c+g
    float W[C + 1];
#pragma unroll
    for (int i = 0; i < C + 1; ++i) W[i] = fadd(V[i], V[i + 1]);       // (a+e)+(b+f)
    float q1n[C], q2n[C];
    q1n[0] = fadd(o[1], p[0]);                                           // next-row b+l at col 0
    q2n[C - 1] = fadd(o[C], p[C + 1]);                                   // next-row b+r at col C-1
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const float a = m[j], b = m[j + 1], c = m[j + 2];
        const float l = o[j], u = o[j + 1], r = o[j + 2];
        const float e = p[j], f = p[j + 1], g = p[j + 2];
        const float n12u = fmul(u, -12.0f);
        const float Hc = cr.hb[j];                       // l + r   (carried)
        const float Hb = fadd(e, g);
        const float Tm = cr.t0[j];                       // (a+c)+(l+r) (carried)
        const float T0 = fadd(Hc, Hb);
        const float D1 = ffma(2.0f, ffma(2.0f, l, W[j]), n12u);
        const float D2 = ffma(2.0f, ffma(2.0f, b, Tm), n12u);
        const float D3 = ffma(2.0f, ffma(2.0f, r, W[j + 1]), n12u);
        const float D4 = ffma(2.0f, ffma(2.0f, f, T0), n12u);
        const float K5 = fadd(c, e), K6 = fadd(a, g);
        const float Pbl = cr.q1[j];                      // b + l   (carried)
        const float Pbr = cr.q2[j];                      // b + r   (carried)
        const float Prf = fadd(r, f);
        const float Plf = fadd(l, f);
        const float D5 = fadd(ffma(4.0f, Pbl, ffma(2.0f, a, K5)), n12u);
        const float D6 = fadd(ffma(4.0f, Pbr, ffma(2.0f, c, K6)), n12u);
        const float D7 = fadd(ffma(4.0f, Prf, ffma(2.0f, g, K5)), n12u);
        const float D8 = fadd(ffma(4.0f, Plf, ffma(2.0f, e, K6)), n12u);
        float bst = D1;                       // strict <, first minimum
        bst = fsel_min_abs(bst, D2);
        bst = fsel_min_abs(bst, D3);
        bst = fsel_min_abs(bst, D4);
        bst = fsel_min_abs(bst, D5);
        bst = fsel_min_abs(bst, D6);
        bst = fsel_min_abs(bst, D7);
        bst = fsel_min_abs(bst, D8);
        best[j] = bst;
        cr.hb[j] = Hb;
        cr.t0[j] = T0;
        if (j + 1 < C) q1n[j + 1] = Prf;
        if (j >= 1) q2n[j - 1] = Plf;
    }
#pragma unroll
    for (int j = 0; j < C; ++j) { cr.q1[j] = q1n[j]; cr.q2[j] = q2n[j]; }
}

template <int C, int K, bool MAP, bool VEC, bool U8>
struct SweepWarp {
    using G = Geo<C, K>;
    static constexpr int NL = K;  // windows for levels 0..K-1

    const SweepParams& P;
    int lane, xf;                 // first column of this lane
    bool out_lane;                // lane holds output columns
    int ys, ye;                   // output strip rows
    int lo[K + 1], hi[K + 1];     // rows computed per level
    const unsigned char* srcp;    // plane base (bytes)
    float* dstp;                  // plane base
    int xload;                    // clamped first column for vector loads

    float win[NL][3][C + 2];
    Carry<C> cr[K + 1];
    float stage[C];
    float acc[K + 1];

    __device__ __forceinline__ SweepWarp(const SweepParams& p) : P(p) {}

    // ---- level-0 loads ---------------------------------------------------
    __device__ __forceinline__ void load_row(int y, float (&v)[C]) const {
        const int64_t r = (int64_t)(y - P.src_row0) * P.src_pitch;
        if constexpr (U8) {
            const unsigned char* row = srcp + r;
            if constexpr (VEC) {
                const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(row + xload));
#pragma unroll
                for (int j = 0; j < C; ++j)
                    v[j] = __fdiv_rn((float)((q >> (8 * j)) & 0xffu), 255.0f);
            } else {
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    int x = min(max(xf + j, 0), P.w - 1);
                    v[j] = __fdiv_rn((float)__ldg(row + x), 255.0f);
                }
            }
        } else {
            const float* row = reinterpret_cast<const float*>(srcp) + r;
            if constexpr (VEC) {
                static_assert(C == 4, "vector path is 16 bytes per lane");
                const float4 q = __ldg(reinterpret_cast<const float4*>(row + xload));
                v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
            } else {
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    int x = min(max(xf + j, 0), P.w - 1);
                    v[j] = __ldg(row + x);
                }
            }
        }
    }

    // Shuffle the halos of a freshly produced row and re-apply clamp-to-edge.
    template <bool BORDER>
    __device__ __forceinline__ void finish_row(float (&v)[C + 2]) const {
        v[0] = __shfl_up_sync(kFull, v[C], 1);
        v[C + 1] = __shfl_down_sync(kFull, v[1], 1);
        if constexpr (BORDER) {
            if (xf == 0) v[0] = v[1];
#pragma unroll
            for (int i = 1; i <= C; ++i)
                if (xf + i - 1 == P.w - 1) v[i + 1] = v[i];
        }
    }

    static __device__ __forceinline__ constexpr int md3(int r) { return ((r % 3) + 3) % 3; }

    template <int L>
    __device__ __forceinline__ void copy_slot(int from, int to) {
        // from/to are compile-time after inlining
#pragma unroll
        for (int i = 0; i < C + 2; ++i) win[L][to][i] = win[L][from][i];
    }

    // ---- one level of one step -----------------------------------------
    template <int PH, int L, bool BORDER>
    __device__ __forceinline__ void level_step(int t) {
        const int y = t - L;
        constexpr int s_y = md3(PH - L);        // slot of row y at level L
        constexpr int s_ym = md3(PH - L - 1);   // slot of row y-1
        constexpr int s_yp = md3(PH - L + 1);   // slot of row y+1
        if constexpr (L == 0) {
            if (y >= lo[0] && y < hi[0]) {
                float v[C];
#pragma unroll
                for (int j = 0; j < C; ++j) v[j] = stage[j];
                if (y + 1 < hi[0]) load_row(y + 1, stage);   // prefetch next row
#pragma unroll
                for (int j = 0; j < C; ++j) win[0][s_y][j + 1] = v[j];
                finish_row<BORDER>(win[0][s_y]);
                if (y == 0) copy_slot<0>(s_y, s_ym);          // row -1 := row 0
            } else if (y == P.h && hi[0] == P.h) {
                copy_slot<0>(s_ym, s_y);                      // row h := row h-1
            }
        } else {
            if (y >= lo[L] && y < hi[L]) {
                const float (&m)[C + 2] = win[L - 1][s_ym];
                const float (&o)[C + 2] = win[L - 1][s_y];
                const float (&pp)[C + 2] = win[L - 1][s_yp];
                float bst[C];
                if (y == lo[L]) init_carry<C>(m, o, cr[L]);
                wmc_row<C>(m, o, pp, cr[L], bst);
                float nv[C];
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    const float hw = fmul(bst[j], kC12);
                    nv[j] = MAP ? hw : ffma(P.dt, hw, o[j + 1]);
                }
                if constexpr (!MAP) {
#pragma unroll
                    for (int j = 0; j < C; ++j) {
                        if (BORDER) {
                            const int x = xf + j;
                            if (x < P.w) acc[L] = ffma(nv[j], 0.0f, acc[L]);
                        } else {
                            acc[L] = ffma(nv[j], 0.0f, acc[L]);
                        }
                    }
                }
                if constexpr (L == K) {
                    store_row<BORDER>(y, nv);
                } else {
#pragma unroll
                    for (int j = 0; j < C; ++j) win[L][s_y][j + 1] = nv[j];
                    finish_row<BORDER>(win[L][s_y]);
                    if (y == 0) copy_slot<L>(s_y, s_ym);
                }
            } else if constexpr (L < K) {
                if (y == P.h && hi[L] == P.h) copy_slot<L>(s_ym, s_y);
            }
        }
    }

    template <bool BORDER>
    __device__ __forceinline__ void store_row(int y, const float (&nv)[C]) const {
        if (!out_lane) return;
        float* row = dstp + (int64_t)(y - P.dst_row0) * P.dst_pitch;
        if constexpr (VEC && !BORDER) {
            *reinterpret_cast<float4*>(row + xf) = make_float4(nv[0], nv[1], nv[2], nv[3]);
        } else {
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const int x = xf + j;
                if (!BORDER || (x >= 0 && x < P.w)) row[x] = nv[j];
            }
        }
    }

    template <int PH, int L, bool BORDER>
    __device__ __forceinline__ void levels(int t) {
        level_step<PH, L, BORDER>(t);
        if constexpr (L < K) levels<PH, L + 1, BORDER>(t);
    }

    template <int PH, bool BORDER>
    __device__ __forceinline__ void step(int t, int t_begin, int t_end) {
        if (t < t_begin || t > t_end) return;
        levels<PH, 0, BORDER>(t);
    }

    template <bool BORDER>
    __device__ __forceinline__ void run() {
        const int t_begin = lo[0];
        const int t_end = ye - 1 + K;
#pragma unroll
        for (int L = 0; L <= K; ++L) acc[L] = 0.0f;
        if (t_begin < hi[0]) load_row(t_begin, stage);
        for (int tb = t_begin - t_begin % 3; tb <= t_end; tb += 3) {
            step<0, BORDER>(tb, t_begin, t_end);
            step<1, BORDER>(tb + 1, t_begin, t_end);
            step<2, BORDER>(tb + 2, t_begin, t_end);
        }
    }
};

template <int C, int K, bool MAP, bool VEC, bool U8>
__global__ void __launch_bounds__(kThreads) wmc_sweeps_kernel(const SweepParams p) {
    using G = Geo<C, K>;
    const int warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int total = p.n_chunks * p.n_strips * p.planes;
    if (warp >= total) return;  // warp-uniform
    const int chunk = warp % p.n_chunks;
    const int rest = warp / p.n_chunks;
    const int strip = rest % p.n_strips;
    const int plane = rest / p.n_strips;

    SweepWarp<C, K, MAP, VEC, U8> sw(p);
    sw.lane = threadIdx.x & 31;
    const int xs = chunk * G::S - G::A;
    sw.xf = xs + sw.lane * C;
    sw.out_lane = sw.lane >= G::LANE_LO && sw.lane < G::LANE_HI;
    sw.ys = p.y0 + strip * p.strip_rows;
    sw.ye = min(sw.ys + p.strip_rows, p.y1);
    if (sw.ys >= sw.ye) return;
#pragma unroll
    for (int L = 0; L <= K; ++L) {
        sw.lo[L] = max(sw.ys - (K - L), 0);
        sw.hi[L] = min(sw.ye + (K - L), p.h);
    }
    const int esz = U8 ? 1 : 4;
    sw.srcp = reinterpret_cast<const unsigned char*>(p.src) + (int64_t)plane * p.src_plane * esz;
    sw.dstp = p.dst + (int64_t)plane * p.dst_plane;
    sw.xload = min(max(sw.xf, 0), (int)(p.src_pitch < 0x7fffffff ? p.src_pitch : 0x7fffffff) - C);

    const bool border = xs < 0 || xs + 32 * C > p.w;
    if (border) sw.template run<true>();
    else        sw.template run<false>();

    if constexpr (!MAP) {
        if (p.flag) {
            int bad = 0x7fffffff;
#pragma unroll
            for (int L = K; L >= 1; --L)
                if (sw.out_lane && sw.acc[L] != sw.acc[L]) bad = p.iter_base + L;
            // warp-reduce then one atomic per warp that saw something
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(kFull, bad, o));
            if (sw.lane == 0 && bad != 0x7fffffff) atomicMin(p.flag, bad);
        }
    }
}

}  // namespace cfk
