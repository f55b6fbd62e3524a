// paper_1903_07189_b200/csrc/wmc_sweep.cuh -- the sm_100a WMC stencil and
// temporally blocked WMC-flow kernel.
//
// What it computes (reference: SPEC.md:171-179 wmc_half_laplace, :256-272
// mc_flow scheme=half_laplace; Eqs. 26-28): K synchronous (Jacobi)
// sweeps U <- U + dt * d_m(U) per launch (the single map evaluation has its
// own kernel, csrc/wmc_map.cuh).
// Arithmetic is the canonical fp32 sequence of DESIGN.md §3 (the same
// sequence oracle/wmc_oracle.c restates), written with explicit _rn
// intrinsics / packed f32x2 PTX so nothing is contracted or reassociated.
//
// How:
//  * Warp streaming.  A warp owns TWO 64-column chunks (2 adjacent columns
//    per lane in each) and streams down a strip of rows.  Each chunk window
//    overlaps its neighbours by A >= K columns per side, so the K levels of
//    the trapezoid never need another warp's data.
//  * Packed fp32 across the two chunks: column c of the warp window is ONE
//    8-byte pair {chunk0[c], chunk1[c]}; every neighbour of a pixel pair is
//    an aligned pair, so the whole canonical sequence runs as sm_100
//    FFMA2/FADD2/FMUL2 (one instruction for two pixels); only the 8-way
//    selection (FSETP+FSEL) is scalar.
//  * Rows live in warp-private SHARED MEMORY, not registers: level 0 in a
//    ring filled RD rows ahead by cp.async (4-byte copies land interleaved
//    as pairs), levels 1..K-1 in 4-row rings written by the producing level.
//    A lane reads its 4-column neighbourhood of a row with two 16-byte LDS
//    (halo columns come from the neighbour lanes' slots -- no shuffles), so
//    registers hold only the pixels in flight and the levels' row sums.
//  * Skewed level pipeline: level L at step t computes row t - (2L - 1), so
//    the K level computations of a step are independent; ring stores are
//    deferred to the end of the step.  Three step loops (checked prologue,
//    fast steady state, checked epilogue); at K <= 2 the steady loop is
//    unrolled over the ring period so every ring address is an immediate.
//  * Clamp-to-edge is applied to the CURRENT iterate at every
//    level: rows by clamping the row index of the slot read (checked steps),
//    columns by an operand fix right after the row loads (edge_fix), so
//    border warps run the fast steady loop too.  Border warps take the
//    lowest warp indices (they start first and share blocks).
//  * Non-finite check: one FFMA2 per pixel pair per level into
//    a per-level accumulator (x*0 + acc is NaN iff x is not finite); the
//    first level whose accumulator is NaN is atomically min-ed into a device
//    flag.  A non-finite pixel stays non-finite at every later iteration
//    (DESIGN.md §3.4), so per-level checks of each warp's own columns name
//    the first bad iteration exactly.
//
// HBM traffic: one 4-byte read and one 4-byte write per pixel per launch
// (overlap columns hit L2); every other access is shared memory.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cfk {

#ifndef CF_RING_UNROLL
#define CF_RING_UNROLL 1  // steady loop unrolled over the ring period (K <= 2)
#endif
#ifndef CF_FAST_UNROLL
#define CF_FAST_UNROLL 2  // steady-state loop unroll (register renaming of the carries)
#endif
constexpr int kFastUnroll = CF_FAST_UNROLL;
// Resident 128-thread blocks per SM the register budget targets (measured on
// B200, 16384^2): K = 1, 3 and the map run best at 4 blocks
// registers); K = 2 at 3 blocks (147 registers with its row-sum carries; 4
// blocks lose 16-20 % even without spills).
#ifndef CF_MINB
#define CF_MINB 4
#endif
#ifndef CF_MINB_EVEN
#define CF_MINB_EVEN 3  // K = 2
#endif
#ifndef CF_WPB
#define CF_WPB 4
#endif
constexpr int kWarpsPerBlock = CF_WPB;
constexpr int kThreads = 32 * kWarpsPerBlock;
constexpr unsigned kFull = 0xffffffffu;
#ifndef CF_COLS
#define CF_COLS 2
#endif
constexpr int C = CF_COLS;            // columns per lane per chunk (2 or 4)
static_assert(C == 2 || C == 4, "2 or 4 columns per lane");
constexpr int kChunk = 32 * C;        // columns per chunk window
constexpr int kRowBytes = 8 * (kChunk + 2);   // pairs for columns -1 .. kChunk
#ifndef CF_RD
#define CF_RD 5
#endif
constexpr int kRD = CF_RD;            // level-0 prefetch distance (rows); kRD + 3 a power of 2
constexpr int kRS = kRD + 3;          // level-0 ring slots (rows t-2 .. t+RD)
static_assert((kRS & (kRS - 1)) == 0, "ring slots must be a power of two");

struct SweepParams {
    const float* src;         // global row src_row0 of plane 0
    float* dst;               // global row dst_row0 of plane 0
    int64_t src_pitch;        // elements
    int64_t dst_pitch;        // elements
    int64_t src_plane;        // plane stride, elements
    int64_t dst_plane;        // plane stride, elements
    int32_t src_row0, dst_row0;
    int32_t w, h;             // global image size (clamp borders)
    int32_t y0, y1;           // output rows
    int32_t strip_rows, n_strips, n_chunks, planes;
    int32_t n_bhi;            // trailing border chunk pairs (host, launch_k)
    int32_t strip_rows_b, n_strips_b;  // border pairs' (shorter) strips
    float dt;
    int32_t iter_base;
    int32_t* flag;            // nullable
    // Fused halo stores (row-band sharding): level-K rows
    // y < peer_up_end are also written into peer_up -- the upper neighbour's
    // destination buffer, whose row 0 is global row peer_up_row0 -- and rows
    // y >= peer_dn_begin into peer_dn.  Both null: no peer stores.  Peer rows
    // are always produced by checked steps, so the fast loop is unchanged.
    float* peer_up;
    float* peer_dn;
    int32_t peer_up_row0, peer_up_end, peer_dn_row0, peer_dn_begin;
    // Fused save-time quantisation (kModeFlowU8, the u8 -> u8 path's last
    // launch): level-K rows go to dst8 as rint(clamp(v,0,1)*255) bytes
    // instead of fp32 to dst.
    uint8_t* dst8;
    int64_t dst8_pitch, dst8_plane;
    int32_t dst8_px;          // bytes between a row's pixels (1 planar; channels interleaved)
    // Fused load-time widening (kModeFlowU8In / kModeFlowU8InOut, the u8
    // paths' first launch): level-0 rows come from u8 bytes at src8 (global
    // row src_row0 of plane 0) instead of src, pixel x of plane p at byte
    // p * src8_plane + x * src8_px of its row.  Host contract (u8_fusable):
    // src8 and the pitch multiples of 4 bytes, w a multiple of 4, and either
    // planar (px 1, plane stride a multiple of 4) or interleaved (plane
    // stride 1, px = channels <= 3, C = 2).
    const uint8_t* src8;
    int64_t src8_pitch, src8_plane;
    int32_t src8_px;
    // MODE == kModeL2 (solve_l2_area): data term f and lambda
    const float* fdata;       // global row 0 of plane 0 (same column geometry as src)
    int64_t f_pitch, f_plane; // elements
    float lambda;
    // MODE == kModeL1 (solve_l1_area): dual planes d (geometry of f)
    const float* dsrc;        // d^t, global row 0 of plane 0
    float* ddst;              // d^{t+K} (output columns/rows only)
    float alpha;              // dual clamp
    float neg_inv_alpha;      // -fl(1/alpha)
};

// Save-time quantisation of the fused u8 stores; wmc_io.cu's
// quantize() is the same clamp-then-round (fminf/fmaxf form, equal bytes).
__device__ __forceinline__ uint32_t quantize_u8(float v) {
    // clamp(v, 0, 1) as one saturating op: NaN -> +0 (the clamp's fmaxf also
    // gives 0; +-0 both quantise to byte 0), then rint(c * 255)
    return (uint32_t)__float2int_rn(__fmul_rn(__saturatef(v), 255.0f));
}

// Load-time widening: fl(q / 255) for a byte q, without the
// division.  r0 = fl(q * fl(1/255)) is off by one ulp for 126 of the 256
// bytes; one residual step r = fma(fma(-r0, 255, q), fl(1/255), r0) equals
// the IEEE quotient for all 256 (checked exhaustively with exact rationals,
// and bit-compared against __fdiv_rn in tests/test_gpu_parity.py).
__device__ __forceinline__ float widen_u8(uint32_t q) {
    const float qf = __uint2float_rn(q);
    const float inv = 0x1.010102p-8f;  // fl(1/255)
    const float r0 = __fmul_rn(qf, inv);
    return __fmaf_rn(__fmaf_rn(-r0, 255.0f, qf), inv, r0);
}

constexpr int kModeFlow = 0;  // U' = U + dt * H^w(U)                      (mc_flow)
// (mode 1, the map, moved to its own kernel: csrc/wmc_map.cuh)
constexpr int kModeL2 = 2;    // U' = U + dt * ((f - U) + lambda * H^w(U))  (solve_l2_area)
constexpr int kModeL1 = 3;    // primal-dual step of solve_l1_area
constexpr int kModeFlowU8 = 4;  // kModeFlow whose level-K rows are stored as u8 bytes
#ifndef CF_U8_EARLY
// 1: widen row t+1 at the end of step t, off the wait -> __syncwarp path
// (measured on cfg5: 0.2 % slower than widening row t in place at step t)
#define CF_U8_EARLY 0
#endif
constexpr int kModeFlowU8In = 5;     // kModeFlow whose level-0 rows are read as u8 bytes
constexpr int kModeFlowU8InOut = 6;  // both (a u8 -> u8 filter done in one launch)
__host__ __device__ constexpr bool mode_u8_in(int m) { return m == kModeFlowU8In || m == kModeFlowU8InOut; }
__host__ __device__ constexpr bool mode_u8_out(int m) { return m == kModeFlowU8 || m == kModeFlowU8InOut; }
__host__ __device__ constexpr bool mode_flow(int m) { return m == kModeFlow || mode_u8_in(m) || mode_u8_out(m); }

// Column geometry for K levels: each chunk window overlaps its neighbours by
// A = K columns per side (the trapezoid shrinks one column per level).
template <int K>
struct Geo {
    static constexpr int A = K;                          // overlap per side
    static constexpr int S = kChunk - 2 * A;             // output columns per chunk
    static_assert(S > 0, "bad geometry");
};

// Rings: level 0 has kRS slots (rows t-2 .. t+RD); levels 1..K-1 have 4
// slots each (skewed pipeline).
constexpr int kLvlSlots = 4;
// Solver modes stage the data term f in a third ring (kFSlots rows, each lane's
// own C column pairs only, 16-byte aligned): rows t-(2K-1) .. t+RD are live.
constexpr int kFSlots = 16;
constexpr int kFRowBytes = 8 * 32 * CF_COLS;
// kModeL1 also stages the incoming dual d (read by level 1 only: rows
// t-1 .. t+RD live).
constexpr int kDSlots = 8;
template <int K>
__host__ __device__ constexpr int ring_bytes_per_warp() {
    return (kRS + kLvlSlots * (K - 1)) * kRowBytes;
}
template <int K, int MODE>
__host__ __device__ constexpr int smem_bytes_per_warp() {
    static_assert(2 * K + CF_RD <= kFSlots && CF_RD + 2 <= kDSlots, "data-term rings too small");
    return ring_bytes_per_warp<K>() + ((MODE == 2 || MODE == 3) ? kFSlots * kFRowBytes : 0) +
           (MODE == 3 ? kDSlots * kFRowBytes : 0);  // f ring: kModeL2/L1; d ring: kModeL1
}

// ---------------------------------------------------------------------------
#ifndef CF_SCALAR
// Packed fp32 pairs in one 64-bit register pair (PTX .b64) and sm_100
// add/mul/fma.rn.f32x2 (SASS FADD2/FMUL2/FFMA2).
// CAUTION (measured, ptxas 12.9): a mul.rn.f32x2 whose only use is an
// add.rn.f32x2 IS contracted into FFMA2 despite .rn and --fmad=false, which
// changes the rounding.  Every packed product here is either multi-use
// (n12u) or a multiplicand of an explicit fma (H^w); keep it that way.
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
#define CF_PAIR_CONST(lo32) (((unsigned long long)(lo32) << 32) | (unsigned long long)(lo32))
#else
// Scalar build of the same sequence (two independent fp32 lanes).
struct f2 {
    float x, y;
};
__device__ __forceinline__ f2 add2(f2 a, f2 b) { return {__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y)}; }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { return {__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)}; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    return {__fmaf_rn(a.x, b.x, c.x), __fmaf_rn(a.y, b.y, c.y)};
}
__device__ __forceinline__ f2 pk(float lo, float hi) { return {lo, hi}; }
__device__ __forceinline__ float lo(f2 v) { return v.x; }
__device__ __forceinline__ float hi(f2 v) { return v.y; }
#endif
__device__ __forceinline__ f2 splat(float v) { return pk(v, v); }
#ifndef CF_SCALAR
constexpr f2 kTwo2 = 0x4000000040000000ull;    // {2, 2}
constexpr f2 kFour2 = 0x4080000040800000ull;   // {4, 4}
constexpr f2 kM12x2 = 0xC1400000C1400000ull;   // {-12, -12}
constexpr f2 kC12x2 = 0x3DAAAAAB3DAAAAABull;   // {fl(1/12), fl(1/12)}
constexpr f2 kZero2 = 0ull;
#else
constexpr f2 kTwo2 = {2.0f, 2.0f};
constexpr f2 kFour2 = {4.0f, 4.0f};
constexpr f2 kM12x2 = {-12.0f, -12.0f};
constexpr f2 kC12x2 = {1.0f / 12.0f, 1.0f / 12.0f};
constexpr f2 kZero2 = {0.0f, 0.0f};
#endif

// ---- shared memory / async copy helpers ----------------------------------
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_rd() {
    asm volatile("cp.async.wait_group %0;" ::"n"(kRD - 1) : "memory");
}
__device__ __forceinline__ void cp_async_wait_rd1() {  // one row further: t + 1
    asm volatile("cp.async.wait_group %0;" ::"n"(kRD - 2) : "memory");
}
// The C+2 pairs (columns C*i-1 .. C*i+C) a lane needs from one row, read
// with 16-byte LDS from byte a = row + 8*C*i (16-aligned).
__device__ __forceinline__ void lds_nb(uint32_t a, f2 (&q)[C + 2]) {
#ifdef CF_EXP_NO_LDS  // diagnostic only (wrong results): cost of the ring loads
#pragma unroll
    for (int k = 0; k < C + 2; ++k)
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(q[k]) : "r"(a + k), "r"(a ^ k));
    return;
#endif
#pragma unroll
    for (int k = 0; k < (C + 2) / 2; ++k) {
#ifndef CF_SCALAR
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                     : "=l"(q[2 * k]), "=l"(q[2 * k + 1]) : "r"(a + 16 * k));
#else
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(q[2 * k].x), "=f"(q[2 * k].y), "=f"(q[2 * k + 1].x),
                       "=f"(q[2 * k + 1].y) : "r"(a + 16 * k));
#endif
    }
}
// Store one pair at byte a (8-aligned).
__device__ __forceinline__ void sts_pair(uint32_t a, f2 v) {
#ifndef CF_SCALAR
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
#else
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
#endif
}
__device__ __forceinline__ void sts1(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

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

// Row-shared sums are carried down a level: Hc = l+r and Tm = (a+c)+(l+r) of
// this row come from the row above (Hb, T0 there); Hb, T0 are returned.
__device__ __forceinline__ void pair_d(f2 a, f2 b, f2 c, f2 l, f2 u, f2 r, f2 e, f2 f, f2 g,
                                       f2 Wm, f2 W0, f2 Hc, f2 Tm, f2& Hb, f2& T0, PairD& P) {
    const f2 two = kTwo2, four = kFour2;
    P.n12u = mul2(u, kM12x2);
    Hb = add2(e, g);                          // e+g
    T0 = add2(Hc, Hb);                        // (l+r)+(e+g)
    P.d[0] = fma2(two, fma2(two, l, Wm), P.n12u);
    P.d[1] = fma2(two, fma2(two, b, Tm), P.n12u);
    P.d[2] = fma2(two, fma2(two, r, W0), P.n12u);
    P.d[3] = fma2(two, fma2(two, f, T0), P.n12u);
    const f2 K5 = add2(add2(c, e), P.n12u), K6 = add2(add2(a, g), P.n12u);
    P.d[4] = fma2(four, add2(b, l), fma2(two, a, K5));
    P.d[5] = fma2(four, add2(b, r), fma2(two, c, K6));
    P.d[6] = fma2(four, add2(r, f), fma2(two, g, K5));
    P.d[7] = fma2(four, add2(l, f), fma2(two, e, K6));
}

__device__ __forceinline__ f2 select_pair(const PairD& P) {
#ifdef CF_EXP_NOSELECT  // diagnostic builds only (wrong results): cost of the selection
    return P.d[0];
#endif
#ifdef CF_EXP_USSELECT  // diagnostic (wrong at exact +-ties / NaN): the map's U/S minimum
    {
        uint32_t U[2], Sx[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            uint32_t v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(hh ? hi(P.d[i]) : lo(P.d[i]));
            const uint32_t a = min(min(v[0], v[1]), v[2]), b = min(min(v[3], v[4]), v[5]);
            U[hh] = min(min(a, b), min(v[6], v[7]));
            const int32_t sa = min(min((int32_t)v[0], (int32_t)v[1]), (int32_t)v[2]);
            const int32_t sb = min(min((int32_t)v[3], (int32_t)v[4]), (int32_t)v[5]);
            Sx[hh] = (uint32_t)min(min(sa, sb), min((int32_t)v[6], (int32_t)v[7]));
        }
        const f2 x = add2(pk(__uint_as_float(U[0]), __uint_as_float(U[1])),
                          pk(__uint_as_float(Sx[0]), __uint_as_float(Sx[1])));
        return pk(lo(x) > 0.0f ? __uint_as_float(Sx[0]) : __uint_as_float(U[0]),
                  hi(x) > 0.0f ? __uint_as_float(Sx[1]) : __uint_as_float(U[1]));
    }
#endif
    return pk(select8(lo(P.d[0]), lo(P.d[1]), lo(P.d[2]), lo(P.d[3]), lo(P.d[4]), lo(P.d[5]),
                      lo(P.d[6]), lo(P.d[7])),
              select8(hi(P.d[0]), hi(P.d[1]), hi(P.d[2]), hi(P.d[3]), hi(P.d[4]), hi(P.d[5]),
                      hi(P.d[6]), hi(P.d[7])));
}

// ---- fp64 evaluation for the map's near ties (csrc/wmc_map.cuh; §3.3) -----
// SPEC-faithful fp64 evaluation of one pixel (oracle/wmc_px.h wmc_px_f64):
// weights n/12 as double, taps in row-major order, s = s + w*x unfused,
// strict-< first-minimum scan.
// fp64 weights n/12 of h1..h8 (row-major taps), rounded once: the constant
// n / 12.0 folded by the compiler is the IEEE quotient __ddiv_rn(n, 12.0).
__device__ __constant__ double kH64[8][9] = {
    {2 / 12.0, 2 / 12.0, 0.0, 4 / 12.0, -1.0, 0.0, 2 / 12.0, 2 / 12.0, 0.0},
    {2 / 12.0, 4 / 12.0, 2 / 12.0, 2 / 12.0, -1.0, 2 / 12.0, 0.0, 0.0, 0.0},
    {0.0, 2 / 12.0, 2 / 12.0, 0.0, -1.0, 4 / 12.0, 0.0, 2 / 12.0, 2 / 12.0},
    {0.0, 0.0, 0.0, 2 / 12.0, -1.0, 2 / 12.0, 2 / 12.0, 4 / 12.0, 2 / 12.0},
    {2 / 12.0, 4 / 12.0, 1 / 12.0, 4 / 12.0, -1.0, 0.0, 1 / 12.0, 0.0, 0.0},
    {1 / 12.0, 4 / 12.0, 2 / 12.0, 0.0, -1.0, 4 / 12.0, 0.0, 0.0, 1 / 12.0},
    {0.0, 0.0, 1 / 12.0, 0.0, -1.0, 4 / 12.0, 1 / 12.0, 4 / 12.0, 2 / 12.0},
    {1 / 12.0, 0.0, 0.0, 4 / 12.0, -1.0, 0.0, 2 / 12.0, 4 / 12.0, 1 / 12.0}};

__device__ __noinline__ float wmc_px_f64(float a, float b, float c, float l, float u, float r,
                                          float e, float f, float g) {
    const double x[9] = {a, b, c, l, u, r, e, f, g};
    double best = 0.0;
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < 9; ++t) s = __dadd_rn(s, __dmul_rn(kH64[i][t], x[t]));
        if (i == 0 || fabs(s) < fabs(best)) best = s;
    }
    return __double2float_rn(best);
}

// ---------------------------------------------------------------------------
template <int K, int MODE>
struct SweepWarp {
    using G = Geo<K>;

    const SweepParams& P;
    int lane;
    int xf[2];                    // first column of this lane in each chunk
    bool outc[C];                 // column j of this lane is an output column
    bool out_h[2];                // chunk h exists (a missing chunk is never stored)
    bool border;                  // some window touches column 0 or w-1 (uniform)
    bool st16;                    // kModeFlowU8: even output rows (16-bit byte-pair stores)
    uint32_t emask;               // image-edge columns of this lane (edge_fix)
    int ys, ye;                   // output strip rows
    // rows computed per level L: [rlo(L), rhi(L)) (recomputed, not stored)
    __device__ __forceinline__ int rlo(int L) const { return max(ys - (K - L), 0); }
    __device__ __forceinline__ int rhi(int L) const { return min(ye + (K - L), P.h); }
    const float* srcp;            // plane base
    float* dstp;                  // plane base
    const float* fp;              // plane base of f (kModeL2, kModeL1)
    const float* dsp;             // plane base of d^t (kModeL1)
    float* ddp;                   // plane base of d^{t+K} (kModeL1)
    uint8_t* d8p;                 // plane base of the u8 output (fused quantisation)
    const uint8_t* s8p;           // u8 input: 4-byte aligned base of this plane's rows
    uint32_t sel8[2];             // byte_perm selectors: chunk h's C input bytes from its words
    int o8[2][2];                 // byte offsets in a u8 row of chunk h's staged words
    int nw8;                      // staged words per chunk (1 or 2)
    uint32_t pend8[4];            // staged words of row t + 1, widened at the end of step t
    uint32_t sbase;               // this warp's shared memory (ring 0, then rings 1..K-1)
    uint32_t lbase;               // sbase + this lane's neighbourhood offset (8*C*lane)
    uint32_t fbase;               // this lane's slice of the data-term ring (solver modes)
    f2 acc[K + 1][C];             // non-finite accumulators per level and column
    // Row sums l+r and (a+c)+(l+r) carried down a level from the row above
    // (K <= 2), or recomputed (K >= 3: the 16 registers buy occupancy there;
    // measured).  Bit-identical either way.
    static constexpr bool kCarry = K <= 2;
    // Ring-period unroll of the steady loop: +2-3 % at K <= 2; at K = 3 the
    // longer live ranges grow the 128-register spill and it loses 3 %.
    static constexpr bool kRingUnroll = CF_RING_UNROLL && K <= 2;
    f2 hc[K + 1][C], tm[K + 1][C];
    f2 onv[K + 1][C];               // results of the current step, per level
    // kModeL1: the dual d_L(y) a level produces is consumed pointwise by
    // level L+1 two steps later (same lane, same columns): a 2-deep register
    // FIFO per level (odv -> dmid -> dold), shifted once per step.
    f2 odv[K + 1][C], dmid[K + 1][C], dold[K + 1][C];

    __device__ __forceinline__ SweepWarp(const SweepParams& p) : P(p) {}

    // Skewed pipeline: level L at step t computes row t - (2L - 1), reading
    // only rows its predecessor produced at earlier steps, so the K level
    // computations of one step are independent (K-way ILP, one __syncwarp
    // per step).
    static __device__ __forceinline__ constexpr int lag(int L) { return 2 * L - 1; }

    // shared address of row y of level L (row index clamped to [0, h):
    // clamp-to-edge on the current iterate).
    template <int L>
    __device__ __forceinline__ uint32_t row_addr(int y) const {
        y = min(max(y, 0), P.h - 1);
        if constexpr (L == 0) {
            return sbase + (uint32_t)(y & (kRS - 1)) * kRowBytes;
        } else {
            return sbase + (uint32_t)(kRS + kLvlSlots * (L - 1) + (y & (kLvlSlots - 1))) *
                               kRowBytes;
        }
    }

    // cp.async this lane's 4 input values of row y into ring slot y % kRS:
    // column c of chunk h lands at byte 8*(c+1) + 4*h of the row.
    __device__ __forceinline__ void prefetch(int y) const {
        if constexpr (kU8In) {
            // u8 input: the 2 aligned words holding chunk h's C bytes,
            // clamped to the row, land in this lane's region at k8Stage;
            // widen8() turns them into the fp32 pairs at step y.
            const uint8_t* row8 = s8p + (int64_t)(y - P.src_row0) * P.src8_pitch;
            const uint32_t s = sbase + (uint32_t)(y & (kRS - 1)) * kRowBytes + 8 * C * lane + k8Stage;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (k < nw8) cp_async4(s + 4 * nw8 * h + 4 * k, row8 + o8[h][k]);
            return;
        }
        const float* row = srcp + (int64_t)(y - P.src_row0) * P.src_pitch;
        const uint32_t s = sbase + (uint32_t)(y & (kRS - 1)) * kRowBytes + 8 * C * lane + 8;
        const float* frow = nullptr;
        if constexpr (kFRing) frow = fp + (int64_t)y * P.f_pitch;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            int x0 = xf[0] + j, x1 = xf[1] + j;
            if (border) {
                x0 = min(max(x0, 0), P.w - 1);
                x1 = min(max(x1, 0), P.w - 1);
            }
            cp_async4(s + 8 * j, row + x0);
            cp_async4(s + 8 * j + 4, row + x1);
            if constexpr (kFRing) {
                const uint32_t fs = fslot(y) + 8 * j;
                cp_async4(fs, frow + x0);
                cp_async4(fs + 4, frow + x1);
            }
            if constexpr (MODE == kModeL1) {
                const float* drow = dsp + (int64_t)y * P.f_pitch;
                const uint32_t ds = dslot(y) + 8 * j;
                cp_async4(ds, drow + x0);
                cp_async4(ds + 4, drow + x1);
            }
        }
    }

    static constexpr bool kU8In = mode_u8_in(MODE);
    // Staged words per chunk and lane (nw8): a lane's C columns start at
    // xf = chunk * S - K + C * lane, so planar rows at C = 2 and even K put
    // them in one aligned word; otherwise they span two.  The 2 * nw8 words
    // sit inside the lane's 8*C-byte region at +8, aligned to their total
    // size (C = 4: at +16).
    static constexpr int k8Stage = C == 4 ? 16 : 8;

    // kU8In: this lane's staged words of row y (landed: after the wait)
    __device__ __forceinline__ void load8(int y, uint32_t (&wd)[4]) const {
        const uint32_t a = sbase + (uint32_t)(y & (kRS - 1)) * kRowBytes + 8 * C * lane + k8Stage;
        if (C == 2 && nw8 == 1) {
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(wd[0]), "=r"(wd[2]) : "r"(a));
            wd[1] = wd[0]; wd[3] = wd[2];
        } else if constexpr (C == 4) {
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(wd[0]), "=r"(wd[1]), "=r"(wd[2]), "=r"(wd[3]) : "r"(a));
        } else {
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(wd[0]), "=r"(wd[1]) : "r"(a));
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(wd[2]), "=r"(wd[3]) : "r"(a + 8));
        }
    }
    __device__ __forceinline__ void widen8(int y) const {
        uint32_t wd[4];
        load8(y, wd);
        cvt8(y, wd);
    }
    // ... widened in place into its C fp32 column pairs, fl(q / 255)
    // exactly as widen_u8 (before the __syncwarp that publishes row y)
    __device__ __forceinline__ void cvt8(int y, const uint32_t (&wd)[4]) const {
        const uint32_t a = sbase + (uint32_t)(y & (kRS - 1)) * kRowBytes + 8 * C * lane;
        const uint32_t q0 = __byte_perm(wd[0], wd[1], sel8[0]);
        const uint32_t q1 = __byte_perm(wd[2], wd[3], sel8[1]);
        const f2 two23 = pk(-8388608.0f, -8388608.0f);  // -2^23
        const f2 inv = pk(0x1.010102p-8f, 0x1.010102p-8f);  // fl(1/255)
        const f2 m255 = pk(-255.0f, -255.0f);
#pragma unroll
        for (int j = 0; j < C; ++j) {
            // 0x4B0000qq = 2^23 + q exactly
            const float lo = __uint_as_float(__byte_perm(q0, 0x4b000000u, 0x7440u | j));
            const float hi = __uint_as_float(__byte_perm(q1, 0x4b000000u, 0x7440u | j));
            const f2 qf = add2(pk(lo, hi), two23);
            const f2 r0 = mul2(qf, inv);   // multi-use: never contracted
            sts_pair(a + 8 + 8 * j, fma2(fma2(r0, m255, qf), inv, r0));
        }
    }

    // Data-term ring (solver modes): this lane's slot of row y, and the pair
    // {f[y][xf[0]+jj], f[y][xf[1]+jj]} from it.
    static constexpr bool kFRing = MODE == kModeL2 || MODE == kModeL1;
    __device__ __forceinline__ uint32_t fslot(int y) const {
        return fbase + (uint32_t)(y & (kFSlots - 1)) * kFRowBytes;
    }
    __device__ __forceinline__ uint32_t dslot(int y) const {
        return fbase + (uint32_t)(kFSlots + (y & (kDSlots - 1))) * kFRowBytes;
    }
    static __device__ __forceinline__ f2 lds_pair(uint32_t a) {
        f2 v;
#ifndef CF_SCALAR
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
#else
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
#endif
        return v;
    }
    __device__ __forceinline__ f2 ld_f(int y, int jj) const { return lds_pair(fslot(y) + 8 * jj); }
    __device__ __forceinline__ f2 ld_d(int y, int jj) const { return lds_pair(dslot(y) + 8 * jj); }

    // Clamp-to-edge at the image's left / right column (border warps): the
    // pixel at x = 0 takes its own column as its x-1 neighbours (a <- b,
    // l <- u, e <- f) and the pixel at x = w-1 as its x+1 neighbours, in each
    // of the three rows right after they are loaded -- exactly the operands
    // of the clamped stencil, so no ring row is ever patched.  Columns
    // outside the image compute finite throw-away values (their level-0 data
    // is the clamped prefetch) and are never stored or read by image pixels.
    // emask bit 2*(2j+h) (+1): column j of chunk half h is x = 0 (x = w-1).
    __device__ __forceinline__ void edge_fix(f2 (&q)[C + 2]) const {
        f2 c[C];
#pragma unroll
        for (int j = 0; j < C; ++j) c[j] = q[j + 1];
#pragma unroll
        for (int j = 0; j < C; ++j) {
            if (emask & (1u << (4 * j + 0))) q[j] = pk(lo(c[j]), hi(q[j]));
            if (emask & (1u << (4 * j + 2))) q[j] = pk(lo(q[j]), hi(c[j]));
            if (emask & (1u << (4 * j + 1))) q[j + 2] = pk(lo(c[j]), hi(q[j + 2]));
            if (emask & (1u << (4 * j + 3))) q[j + 2] = pk(lo(q[j + 2]), hi(c[j]));
        }
    }


    // Compute level L's row for step t.  CHECKED: range check, clamped row
    // indices, predicated stores.  Fast: steady state, rows via R4[] (slot
    // offsets of rows t+c, c = 0..3, in the 4-slot rings) and r0[] (level-0
    // ring rows t-2, t-1, t).  Results are stored (STS / STG) but not yet
    // visible to other lanes: the caller syncs once per step.
    template <int L, bool CHECKED, bool EDGE = false>
    __device__ __forceinline__ void level(int t, const uint32_t (&R4)[4], const uint32_t (&r0)[3],
                                          float* sptr) {
        const int y = t - lag(L);
        if (CHECKED && (y < rlo(L) || y >= rhi(L))) return;  // warp-uniform
        uint32_t am, ao, ap;
        if constexpr (CHECKED) {
            am = row_addr<L - 1>(y - 1);
            ao = row_addr<L - 1>(y);
            ap = row_addr<L - 1>(y + 1);
        } else if constexpr (L == 1) {
            am = r0[0]; ao = r0[1]; ap = r0[2];
        } else {
            // level L-1 row r in slot r & 3; rows y-1, y, y+1 = t - 2L + k
            const uint32_t rb = sbase + (uint32_t)(kRS + kLvlSlots * (L - 2)) * kRowBytes;
            am = rb + R4[(-2 * L + 0 + 64) & 3];
            ao = rb + R4[(-2 * L + 1 + 64) & 3];
            ap = rb + R4[(-2 * L + 2 + 64) & 3];
        }
        f2 m[C + 2], o[C + 2], p[C + 2];
        lds_nb(am + (lbase - sbase), m);
        lds_nb(ao + (lbase - sbase), o);
        lds_nb(ap + (lbase - sbase), p);
        if (CHECKED ? border : EDGE) {
            edge_fix(m);
            edge_fix(o);
            edge_fix(p);
        }
        if (kCarry && CHECKED && y == rlo(L)) {  // first row of this level: no carries yet
#pragma unroll
            for (int j = 1; j <= C; ++j) {
                hc[L][j - 1] = add2(o[j - 1], o[j + 1]);                        // l+r
                tm[L][j - 1] = add2(add2(m[j - 1], m[j + 1]), hc[L][j - 1]);   // (a+c)+(l+r)
            }
        }
        f2 V[C + 2], W[C + 1];
#pragma unroll
        for (int i = 0; i < C + 2; ++i) V[i] = add2(m[i], p[i]);  // a+e / b+f / c+g
#pragma unroll
        for (int i = 0; i < C + 1; ++i) W[i] = add2(V[i], V[i + 1]);  // (a+e)+(b+f)
        f2 nv[C];
#pragma unroll
        for (int j = 1; j <= C; ++j) {
            PairD D;
            f2 hb, t0;
            if constexpr (kCarry) {
                pair_d(m[j - 1], m[j], m[j + 1], o[j - 1], o[j], o[j + 1], p[j - 1], p[j],
                       p[j + 1], W[j - 1], W[j], hc[L][j - 1], tm[L][j - 1], hb, t0, D);
                hc[L][j - 1] = hb;
                tm[L][j - 1] = t0;
            } else {  // recompute the row sums (bit-identical to the carried ones)
                const f2 hcr = add2(o[j - 1], o[j + 1]);
                const f2 tmr = add2(add2(m[j - 1], m[j + 1]), hcr);
                pair_d(m[j - 1], m[j], m[j + 1], o[j - 1], o[j], o[j + 1], p[j - 1], p[j],
                       p[j + 1], W[j - 1], W[j], hcr, tmr, hb, t0, D);
            }
            const f2 b = select_pair(D);
            f2 hw = mul2(b, kC12x2);
            if constexpr (MODE == kModeL2) {
                // SPEC.md:298 with A = I: U' = U + dt*((f - U) + lambda*H^w(U))
                const f2 fv = ld_f(y, j - 1);
                const f2 r = fma2(o[j], splat(-1.0f), fv);         // f - u
                const f2 sdir = fma2(splat(P.lambda), hw, r);      // (f-u) + lambda*H
                nv[j - 1] = fma2(splat(P.dt), sdir, o[j]);
                acc[L][j - 1] = fma2(nv[j - 1], kZero2, acc[L][j - 1]);
            } else if constexpr (MODE == kModeL1) {
                // SPEC.md:306 with A = I:
                //   r = (u - f) + d;  d' = clamp(r, -alpha, alpha)
                //   U' = u + dt*(lambda*H^w - (2d' - d)/alpha)
                const f2 fv = ld_f(y, j - 1);
                f2 dv;
                if constexpr (L == 1) dv = ld_d(y, j - 1);
                else dv = dold[L - 1][j - 1];
                const f2 r = add2(fma2(fv, splat(-1.0f), o[j]), dv);
                const f2 dn = pk(fminf(fmaxf(lo(r), -P.alpha), P.alpha),
                                 fminf(fmaxf(hi(r), -P.alpha), P.alpha));
                const f2 e = fma2(dv, splat(-1.0f), add2(dn, dn));  // 2d' - d
                const f2 sdir = fma2(splat(P.lambda), hw, mul2(e, splat(P.neg_inv_alpha)));
                nv[j - 1] = fma2(splat(P.dt), sdir, o[j]);
                odv[L][j - 1] = dn;
                acc[L][j - 1] = fma2(nv[j - 1], kZero2, acc[L][j - 1]);
            } else {
                // U' = fma(c, D_m, u), c = fl(dt * fl(1/12)): the 1/12 folded
                // into the step (one rounding)
                nv[j - 1] = fma2(splat(__fmul_rn(P.dt, 0x1.555556p-4f)), b, o[j]);
                acc[L][j - 1] = fma2(nv[j - 1], kZero2, acc[L][j - 1]);
            }
        }
#pragma unroll
        for (int j = 0; j < C; ++j) onv[L][j] = nv[j];
    }

    // Store phase of a step (after every level computed, so no shared-memory
    // store precedes a later level's loads: the compiler is free to overlap
    // the K independent level computations).
    template <int L, bool CHECKED, bool EDGE = false>
    __device__ __forceinline__ void store(int t, const uint32_t (&R4)[4], float* sptr) {
        store_one<L, CHECKED, EDGE>(t, R4, sptr);
        if constexpr (L < K) store<L + 1, CHECKED, EDGE>(t, R4, sptr);
    }

    // This lane's output columns of a level-K row as quantised bytes.  FAST
    // (interior warp, unchecked step) with K even: a lane's C = 2 columns
    // start at an even column (chunk origin chunk*S - K) and are both output
    // or both halo, so each chunk's pair is one aligned 16-bit store.
    template <bool FAST>
    __device__ __forceinline__ void store_row8(uint8_t* row, const f2 (&nv)[C]) const {
        if constexpr (FAST && C == 2 && (G::A & 1) == 0) {
            if (!outc[0]) return;
            if (st16) {  // planar, even row addresses (base and pitch)
                const uint32_t b0 = quantize_u8(lo(nv[0])) | (quantize_u8(lo(nv[1])) << 8);
                const uint32_t b1 = quantize_u8(hi(nv[0])) | (quantize_u8(hi(nv[1])) << 8);
                *reinterpret_cast<uint16_t*>(row + xf[0]) = (uint16_t)b0;
                *reinterpret_cast<uint16_t*>(row + xf[1]) = (uint16_t)b1;
                return;
            }
        }
        const int px = P.dst8_px;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            if (!outc[j]) continue;
            if (out_h[0] && xf[0] + j < P.w) row[px * (xf[0] + j)] = (uint8_t)quantize_u8(lo(nv[j]));
            if (out_h[1] && xf[1] + j < P.w) row[px * (xf[1] + j)] = (uint8_t)quantize_u8(hi(nv[j]));
        }
    }

    // This lane's output columns of a level-K row (bounds-checked).
    __device__ __forceinline__ void store_row(float* row, const f2 (&nv)[C]) const {
#pragma unroll
        for (int j = 0; j < C; ++j) {
            if (!outc[j]) continue;
            if (out_h[0] && xf[0] + j < P.w) row[xf[0] + j] = lo(nv[j]);
            if (out_h[1] && xf[1] + j < P.w) row[xf[1] + j] = hi(nv[j]);
        }
    }

    template <int L, bool CHECKED, bool EDGE = false>
    __device__ __forceinline__ void store_one(int t, const uint32_t (&R4)[4], float* sptr) {
        const int y = t - lag(L);
        if (CHECKED && (y < rlo(L) || y >= rhi(L))) return;  // warp-uniform
        const f2 (&nv)[C] = onv[L];
        if constexpr (L == K && MODE == kModeL1) {
            float* drow = ddp + (int64_t)y * P.f_pitch;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                if (!outc[j]) continue;
                if (out_h[0] && (!(CHECKED || EDGE) || xf[0] + j < P.w))
                    drow[xf[0] + j] = lo(odv[K][j]);
                if (out_h[1] && (!(CHECKED || EDGE) || xf[1] + j < P.w))
                    drow[xf[1] + j] = hi(odv[K][j]);
            }
        }
        if constexpr (L == K && mode_u8_out(MODE)) {  // quantise in the store
            store_row8<!(CHECKED || EDGE)>(d8p + (int64_t)(y - P.dst_row0) * P.dst8_pitch, nv);
            return;
        }
        if constexpr (L == K) {
            if (CHECKED || EDGE) {
                float* row = dstp + (int64_t)(y - P.dst_row0) * P.dst_pitch;
                store_row(row, nv);
                if (CHECKED && P.peer_up && y < P.peer_up_end)  // into the neighbour's halo
                    store_row(P.peer_up + (int64_t)(y - P.peer_up_row0) * P.dst_pitch, nv);
                if (CHECKED && P.peer_dn && y >= P.peer_dn_begin)
                    store_row(P.peer_dn + (int64_t)(y - P.peer_dn_row0) * P.dst_pitch, nv);
            } else {  // sptr: row y at column xf[0]; chunk 1 is G::S columns on
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    if (!outc[j]) continue;
                    sptr[j] = lo(nv[j]);
                    sptr[G::S + j] = hi(nv[j]);
                }
            }
        } else {
            uint32_t rb;
            if constexpr (CHECKED) {
                rb = row_addr<L>(y);
            } else {  // row y = t - 2L + 1 in slot y & 3
                rb = sbase + (uint32_t)(kRS + kLvlSlots * (L - 1)) * kRowBytes +
                     R4[(-2 * L + 1 + 64) & 3];
            }
#pragma unroll
            for (int j = 0; j < C; ++j) sts_pair(rb + 8 * C * lane + 8 + 8 * j, nv[j]);
        }
    }

    template <int L, bool CHECKED, bool EDGE = false>
    __device__ __forceinline__ void levels(int t, const uint32_t (&R4)[4],
                                           const uint32_t (&r0)[3], float* sptr) {
        level<L, CHECKED, EDGE>(t, R4, r0, sptr);
        if constexpr (L < K) levels<L + 1, CHECKED, EDGE>(t, R4, r0, sptr);
    }

    // kModeL1: end of step -- level L's dual of row t-lag(L) becomes level
    // L+1's input at step t+2 (rows outside a level's range are never read).
    __device__ __forceinline__ void shift_duals() {
        if constexpr (MODE == kModeL1) {
#pragma unroll
            for (int L = 1; L < K; ++L)
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    dold[L][j] = dmid[L][j];
                    dmid[L][j] = odv[L][j];
                }
        }
    }

    __device__ __forceinline__ void run() {
        const int t_begin = rlo(0);
        const int t_end = ye - 1 + lag(K);
        // steady steps: every level in range with unclamped neighbour rows,
        // interior warp
        int t_s = 0, t_e = rhi(0) - 1;
#pragma unroll
        for (int L = 1; L <= K; ++L) {
            t_s = max(t_s, max(rlo(L) + 1, 1) + lag(L));    // y-1 >= 0, y > rlo (carries)
            t_e = min(t_e, min(rhi(L) - 1, P.h - 2) + lag(L));  // y+1 <= h-1, y < rhi
        }
        if (P.peer_up) t_s = max(t_s, P.peer_up_end + lag(K));       // peer rows: checked
        if (P.peer_dn) t_e = min(t_e, P.peer_dn_begin - 1 + lag(K));
#pragma unroll
        for (int L = 0; L <= K; ++L)
#pragma unroll
            for (int j = 0; j < C; ++j) acc[L][j] = kZero2;
        // prologue: rows t_begin .. t_begin+RD-1 (one commit group per row)
#pragma unroll
        for (int i = 0; i < kRD; ++i) {
            const int y = t_begin + i;
            if (y < rhi(0)) prefetch(y);
            cp_async_commit();
        }
        // running pointers: prefetch source (row t+RD, column xf[0]) and the
        // level-K store row (t - lag(K), column xf[0])
        const float* lptr = srcp + (int64_t)(t_begin + kRD - P.src_row0) * P.src_pitch + xf[0];
        float* sptr = dstp + (int64_t)(t_begin - lag(K) - P.dst_row0) * P.dst_pitch + xf[0];
        // Three loops -- checked prologue, fast steady state, checked
        // epilogue -- so the steady-state loop's carried registers never
        // join the checked path's (a per-step if/else costs ~5 register
        // moves per pixel-update at the join).
        const int f0 = min(t_s, t_end + 1), f1 = min(t_e, t_end);
        int t = t_begin;
        for (; t < f0; ++t) step<false>(t, lptr, sptr);
        if (border) {  // image-edge columns: fast steps with the edge fix
            for (; t <= f1; ++t) step<true, -1, true>(t, lptr, sptr);
        } else if constexpr (kRingUnroll) {
            // Steady state unrolled over the ring period (4 steps from t = 0
            // mod 4): every ring row address is a compile-time offset from
            // sbase or from the group's two level-0 half-ring bases -- no
            // per-step slot arithmetic (IMAD work on the saturated FMA pipe).
            for (; t <= f1 && (t & 3); ++t) step<true>(t, lptr, sptr);
            for (; t + 3 <= f1; t += 4) {
                const uint32_t g0 = sbase + (uint32_t)(t & 4) * kRowBytes;
                const uint32_t g1 = sbase + (uint32_t)((t & 4) ^ 4) * kRowBytes;
                step<true, 0>(t, lptr, sptr, g0, g1);
                step<true, 1>(t + 1, lptr, sptr, g0, g1);
                step<true, 2>(t + 2, lptr, sptr, g0, g1);
                step<true, 3>(t + 3, lptr, sptr, g0, g1);
            }
            for (; t <= f1; ++t) step<true>(t, lptr, sptr);
        } else {
#pragma unroll kFastUnroll
            for (; t <= f1; ++t) step<true>(t, lptr, sptr);
        }
        for (; t <= t_end; ++t) step<false>(t, lptr, sptr);
    }

    // Level-0 ring row t0 + D (t0 = 0 mod 4 the group start, -2 <= D <= 8)
    // in the 8-slot ring: slot ((t0 & 4) + D) & 7, i.e. the group's own half
    // ring (g0) when bit 2 of D is clear (D = 0..3, 8) and the other half
    // (g1) when it is set (D = -2, -1, 4..7), at offset D & 3.
    template <int D>
    static __device__ __forceinline__ uint32_t ring0(uint32_t g0, uint32_t g1) {
        static_assert(kRS == 8, "phase addressing assumes an 8-slot level-0 ring");
        static_assert(D >= -4 && D < 12, "row outside the ring's reach");
        if constexpr ((((D + 8) >> 2) & 1) == 0) return g0 + (uint32_t)((D + 8) & 3) * kRowBytes;
        else return g1 + (uint32_t)((D + 8) & 3) * kRowBytes;
    }

    // PH >= 0: steady step at phase PH of a 4-step group (t = t0 + PH).
    template <bool FAST, int PH = -1, bool EDGE = false>
    __device__ __forceinline__ void step(int t, const float*& lptr, float*& sptr,
                                         uint32_t g0 = 0, uint32_t g1 = 0) {
        if constexpr (kU8In && CF_U8_EARLY) {
            // row t was widened at the end of step t-1 (the first row here);
            // row t+1's words are read now, widened after this step's levels
            cp_async_wait_rd1();
            if (t == rlo(0)) widen8(t);
            if (t + 1 < rhi(0)) load8(t + 1, pend8);
        } else {
            cp_async_wait_rd();       // this lane's copies of row t landed
            if constexpr (kU8In) {
                if (t < rhi(0)) widen8(t);
            }
        }
        __syncwarp();             // rows of step t-1 and row t visible to all lanes
        if (t + kRD < rhi(0)) {
            if constexpr (kU8In) {
                prefetch(t + kRD);   // first launch only: the generic form is enough
            } else if ((FAST && !EDGE) || !border) {
                // (a coalesced copy mapping -- lane L filling ring word 2 +
                // 32k + L -- was measured here too: +8 registers, no gain at
                // K = 2, where the sweeps, not the copies, bound the kernel;
                // the single-sweep map uses it, csrc/wmc_map.cuh)
                uint32_t sa;
                if constexpr (PH >= 0) sa = ring0<PH + kRD>(g0, g1) + 8 * C * lane + 8;
                else sa = sbase + (uint32_t)((t + kRD) & (kRS - 1)) * kRowBytes + 8 * C * lane + 8;
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    cp_async4(sa + 8 * j, lptr + j);
                    cp_async4(sa + 8 * j + 4, lptr + G::S + j);
                }
                if constexpr (kFRing) {  // interior warp: both chunks present
                    const float* frow = fp + (int64_t)(t + kRD) * P.f_pitch + xf[0];
                    const uint32_t fs = fslot(t + kRD);
#pragma unroll
                    for (int j = 0; j < C; ++j) {
                        cp_async4(fs + 8 * j, frow + j);
                        cp_async4(fs + 8 * j + 4, frow + G::S + j);
                    }
                }
                if constexpr (MODE == kModeL1) {
                    const float* drow = dsp + (int64_t)(t + kRD) * P.f_pitch + xf[0];
                    const uint32_t ds = dslot(t + kRD);
#pragma unroll
                    for (int j = 0; j < C; ++j) {
                        cp_async4(ds + 8 * j, drow + j);
                        cp_async4(ds + 8 * j + 4, drow + G::S + j);
                    }
                }
            } else {
                prefetch(t + kRD);
            }
        }
        lptr += P.src_pitch;
        cp_async_commit();
        const int ph = PH >= 0 ? PH : t;
        const uint32_t R4[4] = {(uint32_t)(ph & 3) * kRowBytes,
                                (uint32_t)((ph + 1) & 3) * kRowBytes,
                                (uint32_t)((ph + 2) & 3) * kRowBytes,
                                (uint32_t)((ph + 3) & 3) * kRowBytes};
        if constexpr (FAST) {
            uint32_t r0[3];
            if constexpr (PH >= 0) {
                r0[0] = ring0<PH - 2>(g0, g1);
                r0[1] = ring0<PH - 1>(g0, g1);
                r0[2] = ring0<PH>(g0, g1);
            } else {
                r0[0] = sbase + (uint32_t)((t - 2) & (kRS - 1)) * kRowBytes;
                r0[1] = sbase + (uint32_t)((t - 1) & (kRS - 1)) * kRowBytes;
                r0[2] = sbase + (uint32_t)(t & (kRS - 1)) * kRowBytes;
            }
            levels<1, false, EDGE>(t, R4, r0, sptr);
            store<1, false, EDGE>(t, R4, sptr);
            shift_duals();
        } else {
            const uint32_t r0[3] = {0, 0, 0};
            levels<1, true>(t, R4, r0, sptr);
            store<1, true>(t, R4, sptr);
            shift_duals();
        }
        if constexpr (kU8In && CF_U8_EARLY) {
            if (t + 1 < rhi(0)) cvt8(t + 1, pend8);
        }
        sptr += P.dst_pitch;
    }
};

template <int K, int MODE>
// The solver modes carry f (and the dual FIFO): 3 blocks/SM = 168 registers,
// no spills at the filter's K = 2.
__global__ void __launch_bounds__(kThreads,
                                  (MODE == kModeL2 || MODE == kModeL1)                    ? 3
                                  : (mode_flow(MODE) && K == 2)                           ? CF_MINB_EVEN
                                                                                           : CF_MINB)
    wmc_sweeps_kernel(const SweepParams p) {
    using G = Geo<K>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int n_pairs = (p.n_chunks + 1) / 2;
    const int nb = min(n_pairs, 1 + p.n_bhi), ni = n_pairs - nb;
    const int btasks = nb * p.n_strips_b * p.planes;
    const int total = btasks + ni * p.n_strips * p.planes;
    if (warp >= total) return;  // warp-uniform
    // Border chunk pairs (pair 0 and the last n_bhi) do extra per-step work
    // (edge fix, clamped prefetch): their tasks take the lowest warp indices,
    // so they start first and share blocks with each other rather than
    // stretching the residency of otherwise-fast blocks (a block frees its
    // slot only when its slowest warp ends).
    // Border pairs also get shorter strips (strip_rows_b): their steps cost
    // more, and with equal strips they were the tail of every launch.
    int cpair, strip, plane, srows;
    if (warp < btasks) {
        const int k = warp % nb, rest = warp / nb;
        cpair = k == 0 ? 0 : n_pairs - nb + k;
        strip = rest % p.n_strips_b;
        plane = rest / p.n_strips_b;
        srows = p.strip_rows_b;
    } else {
        const int i = warp - btasks, rest = i / ni;
        cpair = 1 + i % ni;
        strip = rest % p.n_strips;
        plane = rest / p.n_strips;
        srows = p.strip_rows;
    }

    SweepWarp<K, MODE> sw(p);
    sw.lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const int c = sw.lane * C + j;  // window column
        sw.outc[j] = c >= G::A && c < G::A + G::S;
    }
    sw.border = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int chunk = 2 * cpair + h;
        const int xs = chunk * G::S - G::A;
        sw.out_h[h] = chunk < p.n_chunks;
        // a missing second chunk mirrors the first (finite data, never stored)
        sw.xf[h] = (sw.out_h[h] ? xs : xs - G::S) + sw.lane * C;
        sw.border |= xs < 0 || xs + kChunk > p.w || !sw.out_h[h];
    }
    sw.emask = 0;
#pragma unroll
    for (int j = 0; j < C; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int x = sw.xf[h] + j;
            if (x == 0) sw.emask |= 1u << (4 * j + 2 * h);
            if (x == p.w - 1) sw.emask |= 1u << (4 * j + 2 * h + 1);
        }
    sw.ys = p.y0 + strip * srows;
    sw.ye = min(sw.ys + srows, p.y1);
    if (sw.ys >= sw.ye) return;
#ifdef CF_EXP_SKIP_BORDER  // diagnostic only (wrong results): cost of the border tasks
    if (sw.border) return;
#endif
    sw.srcp = p.src + (int64_t)plane * p.src_plane;
    sw.dstp = p.dst + (int64_t)plane * p.dst_plane;
    sw.fp = (MODE == kModeL2 || MODE == kModeL1) ? p.fdata + (int64_t)plane * p.f_plane : nullptr;
    sw.dsp = MODE == kModeL1 ? p.dsrc + (int64_t)plane * p.f_plane : nullptr;
    sw.ddp = MODE == kModeL1 ? p.ddst + (int64_t)plane * p.f_plane : nullptr;
    sw.d8p = mode_u8_out(MODE) ? p.dst8 + (int64_t)plane * p.dst8_plane : nullptr;
    sw.s8p = nullptr;
    if constexpr (mode_u8_in(MODE)) {
        // Pixel x of this plane is byte c8 + px * x of the aligned row base
        // (c8: the plane offset's low two bits -- an interleaved channel).
        // Column x of chunk h comes from byte b & 3 of staged word 0 or 1,
        // b = c8 + px * xc, xc = x clamped to the row: the words of a lane's
        // clamped columns are always the two clamped words prefetch() stages
        // (w = 0 mod 4; px <= 3 at C = 2).
        const uintptr_t a8 = reinterpret_cast<uintptr_t>(p.src8 + (int64_t)plane * p.src8_plane);
        const int c8 = (int)(a8 & 3u), px = p.src8_px;
        sw.s8p = reinterpret_cast<const uint8_t*>(a8 - (uintptr_t)c8);
        const int nw = ((c8 + px * (p.w - 1)) >> 2) + 1;  // words holding the row's pixels
        sw.nw8 = (C == 2 && K % 2 == 0 && px == 1 && c8 == 0) ? 1 : 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int w0 = (c8 + px * sw.xf[h]) >> 2;  // floor (xf may be negative)
            const int wa = min(max(w0, 0), nw - 1);
            sw.o8[h][0] = 4 * wa;
            sw.o8[h][1] = 4 * min(max(w0 + 1, 0), nw - 1);
            uint32_t sel = 0;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const int b = c8 + px * min(max(sw.xf[h] + j, 0), p.w - 1);
                sel |= (uint32_t)(((b >> 2) == wa ? 0 : 4) + (b & 3)) << (4 * j);
            }
            sw.sel8[h] = sel;
        }
    }
    sw.st16 = p.dst8_px == 1 &&
              ((reinterpret_cast<uintptr_t>(sw.d8p) | (uintptr_t)p.dst8_pitch) & 1) == 0;
    sw.sbase = (uint32_t)__cvta_generic_to_shared(smem) +
               (uint32_t)(threadIdx.x >> 5) * smem_bytes_per_warp<K, MODE>();
    sw.lbase = sw.sbase + 8 * C * sw.lane;
    sw.fbase = sw.sbase + ring_bytes_per_warp<K>() + 8 * C * sw.lane;

    sw.run();

    {
        if (p.flag) {
            int bad = 0x7fffffff;
#pragma unroll
            for (int L = K; L >= 1; --L) {
#pragma unroll
                for (int j = 0; j < C; ++j) {  // only this warp's output columns count
                    const float ax = cfk::lo(sw.acc[L][j]), ay = cfk::hi(sw.acc[L][j]);
                    if (sw.outc[j] && (ax != ax || (sw.out_h[1] && ay != ay)))
                        bad = p.iter_base + L;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(kFull, bad, o));
            if (sw.lane == 0 && bad != 0x7fffffff) atomicMin(p.flag, bad);
        }
    }
}

}  // namespace cfk
