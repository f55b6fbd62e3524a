// paper_1903_07189_b200/csrc/wmc_map.cuh -- the WMC map (wmc_half_laplace,
// SPEC.md:171-179) as a dedicated streaming kernel, and the map's selection
// rule shared with the small-image flat kernel.  DESIGN.md §3.3, §4.
//
// One evaluation per pixel: nothing to block temporally, so the kernel is
// built for memory-pipeline and issue efficiency (map).
//  * A warp owns 256 contiguous columns -- two 128-column chunks packed as
//    pairs {chunk 0 col c, chunk 1 col c}, so the canonical sequence runs as
//    FFMA2 / FADD2 as in the flow kernel -- and streams a strip of rows; lane
//    i computes columns 4i .. 4i+3 of each chunk (4 pixel pairs a row).
//  * Rows are staged in a warp-private shared-memory ring by cp.async with
//    CLAMPED source coordinates (window columns -1 / 128 and the rows above /
//    below the image hold the edge pixels), so the clamp-to-edge stencil
//     needs no checked path: border warps run the same loop.
//  * The copies use their own lane mapping (lane L fills ring word 32k + L):
//    each copy instruction reads two 64-byte runs and writes 128 contiguous
//    bytes of shared memory.  The lane-per-column mapping of the flow kernel
//    read 4 lines and hit one bank 8 times per instruction; with it, data
//    movement alone ran at 0.54 of the HBM roofline, with this one at 0.77.
//  * 16-byte output stores where the rows are 16-byte aligned.
//  * Selection by the U/S rule (map_fast below): two 8-way integer minimum
//    trees (3-input VIMNMX3) over the D_k bit patterns and one packed add
//    give the first-index minimum AND the opposite-sign runner-up distance
//    the near-tie test needs -- instead of the 7-pick FSETP/FSEL tournament
//    plus a separate 8-sum near-tie scan.  A two-predicate superset test
//    flags the pixels that may need more; one warp vote per row sends them
//    to map_pair_fix (out of line), which applies the exact rule: fp64 for
//    near ties, the first-index tournament for exact +-0 / NaN ties.
#pragma once
#include "wmc_sweep.cuh"

namespace cfk {

// min over 8 as 3-input trees (ptxas: VIMNMX3 / VIMNMX, 4 ops each)
__device__ __forceinline__ uint32_t umin8(const uint32_t (&v)[8]) {
    const uint32_t a = min(min(v[0], v[1]), v[2]);
    const uint32_t b = min(min(v[3], v[4]), v[5]);
    const uint32_t c = min(v[6], v[7]);
    return min(min(a, b), c);
}
__device__ __forceinline__ int32_t smin8(const uint32_t (&v)[8]) {
    const int32_t a = min(min((int32_t)v[0], (int32_t)v[1]), (int32_t)v[2]);
    const int32_t b = min(min((int32_t)v[3], (int32_t)v[4]), (int32_t)v[5]);
    const int32_t c = min((int32_t)v[6], (int32_t)v[7]);
    return min(min(a, b), c);
}

// The map's selection and near-tie test (oracle/wmc_px.h
// map_best_f32 is the same rule), per pixel:
//   U = min_k bits(D_k) unsigned, S = min_k bits(D_k) signed;
//   x = fl(float(U) + float(S));  b = x > 0 ? float(S) : float(U);
//   U != S and x neither > 0 nor < 0 (exact opposite-sign tie, or NaN):
//     b = the first-index tournament;
//   tie iff |x| <= tau && |x| < |b|, tau = fmaf(|n12u|, 1.5*2^-19, fl(|b|*2^-20)).
// The tie test is evaluated with the fast b: where the tournament is needed
// x is 0 (|b| is the tied magnitude either way) or NaN (no tie either way).
// The fast path returns b and a "rare" flag per pixel (tie, or tournament
// needed); map_pair_fix redoes flagged pixels.
__device__ __forceinline__ void map_fast_s(const PairD& D, float& b0, float& b1, bool& rare) {
    uint32_t dl[8], dh[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        dl[k] = __float_as_uint(lo(D.d[k]));
        dh[k] = __float_as_uint(hi(D.d[k]));
    }
    const uint32_t U0 = umin8(dl), U1 = umin8(dh);
    const int32_t S0 = smin8(dl), S1 = smin8(dh);
    const f2 x = add2(pk(__uint_as_float(U0), __uint_as_float(U1)),
                      pk(__int_as_float(S0), __int_as_float(S1)));
    const float x0 = lo(x), x1 = hi(x);
    b0 = x0 > 0.0f ? __int_as_float(S0) : __uint_as_float(U0);
    b1 = x1 > 0.0f ? __int_as_float(S1) : __uint_as_float(U1);
    const float tau0 = __fmaf_rn(fabsf(lo(D.n12u)), 0x1.8p-19f, __fmul_rn(fabsf(b0), 0x1.0p-20f));
    const float tau1 = __fmaf_rn(fabsf(hi(D.n12u)), 0x1.8p-19f, __fmul_rn(fabsf(b1), 0x1.0p-20f));
    // A superset of {near tie} u {tournament needed}, two predicates a pixel:
    // both need mixed signs (U != S; with one sign |x| = 2|b| >= |b|), and
    // |x| <= tau (a near tie needs it; x == 0 satisfies it) or x NaN -- the
    // unordered compare.  map_pair_fix applies the exact rule.
    rare = ((U0 != (uint32_t)S0) & !(fabsf(x0) > tau0)) |
           ((U1 != (uint32_t)S1) & !(fabsf(x1) > tau1));
}
__device__ __forceinline__ f2 map_fast(const PairD& D, bool& rare) {
    float b0, b1;
    map_fast_s(D, b0, b1, rare);
    return pk(b0, b1);
}

// The complete rule for one pixel of a flagged pair: tie -> the SPEC-faithful
// fp64 evaluation, else the first-index tournament.  Recomputes D from the
// neighbourhood with the same operands in the same order (V = a+e | b+f |
// c+g, W = V + V', H = l+r, T = (a+c)+(l+r) -- bit-identical to the
// streamed / carried sums).  Out of line: rare, and kept out of the loop's
// instruction-cache footprint.
__device__ __forceinline__ f2 map_pair_fix_inl(f2 a, f2 b, f2 c, f2 l, f2 u, f2 r, f2 e, f2 f,
                                               f2 g, f2 hw) {
    const f2 Vl = add2(a, e), Vc = add2(b, f), Vr = add2(c, g);
    const f2 Wm = add2(Vl, Vc), W0 = add2(Vc, Vr);
    const f2 Hc = add2(l, r);
    const f2 Tm = add2(add2(a, c), Hc);
    PairD D;
    f2 hb, t0;
    pair_d(a, b, c, l, u, r, e, f, g, Wm, W0, Hc, Tm, hb, t0, D);
    float h[2] = {lo(hw), hi(hw)};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        float d[8];
        uint32_t bits[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            d[i] = k ? hi(D.d[i]) : lo(D.d[i]);
            bits[i] = __float_as_uint(d[i]);
        }
        const uint32_t U = umin8(bits);
        const int32_t S = smin8(bits);
        const float x = __fadd_rn(__uint_as_float(U), __int_as_float(S));
        const float bf = x > 0.0f ? __int_as_float(S) : __uint_as_float(U);
        const float n12 = k ? hi(D.n12u) : lo(D.n12u);
        const float tau = __fmaf_rn(fabsf(n12), 0x1.8p-19f, __fmul_rn(fabsf(bf), 0x1.0p-20f));
        if (fabsf(x) <= tau && fabsf(x) < fabsf(bf))  // near tie: SPEC-faithful fp64
            h[k] = k ? wmc_px_f64(hi(a), hi(b), hi(c), hi(l), hi(u), hi(r), hi(e), hi(f), hi(g))
                     : wmc_px_f64(lo(a), lo(b), lo(c), lo(l), lo(u), lo(r), lo(e), lo(f), lo(g));
        else if (U != (uint32_t)S && !(x > 0.0f || x < 0.0f))  // exact tie: first index
            h[k] = __fmul_rn(select8(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7]),
                             0x1.555556p-4f);  // fl(1/12)
    }
    return pk(h[0], h[1]);
}

__device__ __noinline__ f2 map_pair_fix(f2 a, f2 b, f2 c, f2 l, f2 u, f2 r, f2 e, f2 f, f2 g,
                                        f2 hw) {
    return map_pair_fix_inl(a, b, c, l, u, r, e, f, g, hw);
}

// H^w of the map for a pixel pair (fast path), `rare` if either pixel may
// need map_pair_fix; the row sums carried in Hc / Tm.
__device__ __forceinline__ f2 map_pair(f2 a, f2 b, f2 c, f2 l, f2 u, f2 r, f2 e, f2 f, f2 g,
                                       f2 Wm, f2 W0, f2& Hc, f2& Tm, bool& rare) {
    PairD D;
    f2 hb, t0;
    pair_d(a, b, c, l, u, r, e, f, g, Wm, W0, Hc, Tm, hb, t0, D);
    Hc = hb;
    Tm = t0;
    const f2 best = map_fast(D, rare);
    return mul2(best, kC12x2);
}
// The same with the pair's two results as scalars (h0: chunk 0, h1: chunk
// 1): the streaming kernel's 16-byte stores take four chunk-0 values in
// consecutive registers, which a packed pair would have to be unpacked into.
__device__ __forceinline__ void map_pair_s(f2 a, f2 b, f2 c, f2 l, f2 u, f2 r, f2 e, f2 f, f2 g,
                                           f2 Wm, f2 W0, f2& Hc, f2& Tm, float& h0, float& h1,
                                           bool& rare) {
    PairD D;
    f2 hb, t0;
    pair_d(a, b, c, l, u, r, e, f, g, Wm, W0, Hc, Tm, hb, t0, D);
    Hc = hb;
    Tm = t0;
    float b0, b1;
    map_fast_s(D, b0, b1, rare);
    h0 = __fmul_rn(b0, 0x1.555556p-4f);  // fl(1/12): the lanes of mul2(best, kC12x2)
    h1 = __fmul_rn(b1, 0x1.555556p-4f);
}

// ---- the streaming map kernel ---------------------------------------------
// Lane i owns columns 4i .. 4i+3 of each of the warp's two 128-column chunks
// (4 pixel pairs per row: 4 independent chains for the scheduler, and the
// per-row costs -- ring wait, copies, loads, vote -- spread over 8 pixels).
#ifndef CF_MAP_COLS
#define CF_MAP_COLS 4
#endif
constexpr int kMapCols = CF_MAP_COLS;         // columns per lane per chunk (2 or 4)
static_assert(kMapCols == 2 || kMapCols == 4, "2 or 4 columns per lane");
constexpr int kMapChunk = 32 * kMapCols;      // 128
constexpr int kMapNb = kMapCols + 2;          // pairs of a lane's neighbourhood row
constexpr int kMapCopies = 2 * kMapCols;      // full 32-word copies per ring row (+ a 4-word tail)
#ifndef CF_MAP_PD
#define CF_MAP_PD 6
#endif
constexpr int kMapPD = CF_MAP_PD;             // prefetch distance (rows)
#ifndef CF_MAP_RING
#define CF_MAP_RING 8
#endif
constexpr int kMapRing = CF_MAP_RING;         // ring rows (>= kMapPD + 2, power of 2)
constexpr int kMapRowBytes = 8 * (kMapChunk + 2);  // pairs for window columns -1 .. 128
#ifndef CF_MAP_WARPS
#define CF_MAP_WARPS 4
#endif
constexpr int kMapWarps = CF_MAP_WARPS;       // warps per block
static_assert(kMapRing >= kMapPD + 2, "ring too small for the prefetch distance");
#ifndef CF_MAP_ROLL
#define CF_MAP_ROLL 0   // 1: rows rolled through registers, loop unrolled x3 (experiment)
#endif

struct MapParams {
    const float* src;
    float* dst;            // nullable with seg_sums set: the energy alone, no map stored
    // Fused WMC energy (csrc/wmc_reduce.cu's fixed order):
    // per row and 256-column segment, the sum of |H|^q -- lane i's columns
    // 4i..4i+3 then 128+4i..128+4i+3 sequentially, then the xor butterfly --
    // into seg_sums[segment * planes * h + plane * h + y].
    double* seg_sums;      // nullable
    double q;
    int32_t qkind;         // 1: |H|, 2: H*H, 3: sqrt|H|, 0: pow(|H|, q)
    int64_t src_pitch, src_plane, dst_pitch, dst_plane;
    int32_t w, h, planes;
    int32_t n_pairs;       // 256-column chunk pairs per row
    int32_t strip_rows, n_strips;
    int32_t st128;         // every output row 16-byte aligned
};

// Ring rows are stored with their 16-byte chunks swizzled (4 columns a
// lane): chunk q lives at q ^ ((q >> 3) & 1).  A lane's neighbourhood is
// chunks 2i .. 2i+2 (lane stride 32 bytes), which unswizzled hit each bank
// group twice per LDS.128 (8 shared-memory wavefronts instead of 4); the
// swizzle spreads every 8 consecutive lanes over all 8 groups.  The copies
// write whole 128-byte groups of 8 chunks, so they stay conflict-free.
#ifndef CF_MAP_SWZ
#define CF_MAP_SWZ 1
#endif
constexpr bool kMapSwz = CF_MAP_SWZ && kMapCols == 4;
__host__ __device__ constexpr uint32_t map_swz_chunk(uint32_t q) {
    return kMapSwz ? (q ^ ((q >> 3) & 1u)) : q;
}

// the kMapNb pairs (window columns C*i-1 .. C*i+C) of one ring row: one
// LDS.128 per 16-byte chunk, at the lane's (swizzled) chunk offsets
__device__ __forceinline__ void lds_row6(uint32_t row, const uint32_t (&co)[kMapNb / 2],
                                         f2 (&q)[kMapNb]) {
#pragma unroll
    for (int k = 0; k < kMapNb / 2; ++k)
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                     : "=l"(q[2 * k]), "=l"(q[2 * k + 1]) : "r"(row + co[k]));
}

// |H|^q in fp64 (csrc/wmc_reduce.cu term(): the same expressions); the
// general power out of line (eight inlined pow() copies per row flooded the
// instruction cache)
__device__ __noinline__ double energy_pow(double a, double q) { return pow(a, q); }
template <int QK>  // 1: |H|, 2: H*H, 3: sqrt|H|, 4: pow(|H|, q)
__device__ __forceinline__ double energy_term(float hv, double q) {
    const double a = fabs((double)hv);
    if constexpr (QK == 1) return a;
    else if constexpr (QK == 2) return __dmul_rn(a, a);
    else if constexpr (QK == 3) return __dsqrt_rn(a);
    else return energy_pow(a, q);
}

// The energy order's in-lane sum of the 8 terms (csrc/wmc_reduce.cu): a
// pairwise tree, ((t0+t1)+(t2+t3)) + ((t4+t5)+(t6+t7)) -- depth 3.
__device__ __forceinline__ double lane_tree8(const double (&t)[8]) {
    return __dadd_rn(__dadd_rn(__dadd_rn(t[0], t[1]), __dadd_rn(t[2], t[3])),
                     __dadd_rn(__dadd_rn(t[4], t[5]), __dadd_rn(t[6], t[7])));
}
// (CF_MAP_COLS=2 experiment builds only: not the energy's pinned order)
__device__ __forceinline__ double lane_tree8(const double (&t)[4]) {
    return __dadd_rn(__dadd_rn(t[0], t[1]), __dadd_rn(t[2], t[3]));
}

// One warp's strip.  Ring slot of row r: (r - (ys - 1)) & 7.
// INTERIOR: every column x0-1 .. x0+256 inside the image (no clamping);
// ST128: INTERIOR with 16-byte aligned output rows (vector stores).
template <bool INTERIOR, int QK, bool ST128 = false>  // QK > 0: the fused energy epilogue
struct MapWarp {
    static constexpr bool ENERGY = QK > 0;
    const MapParams& p;
    int lane, ys, ye, x0;
    const float* src;      // plane base
    int64_t pf_step;       // src row pitch in bytes
    bool tail4;            // lanes 0-3 also copy the row's last 4 words
    const char* pf;        // column x0 of the next row to prefetch (row clamp(yp))
    int yp;
    uint32_t sbase;
    int64_t plane_row0;        // plane * h (the energy's row index base)
    uint32_t co[kMapNb / 2];   // this lane's neighbourhood chunks (byte offsets in a ring row)
    uint32_t cpe, cpo;         // this lane's copy word offset for even / odd copies
    f2 hc[kMapCols], tm[kMapCols];

    __device__ __forceinline__ MapWarp(const MapParams& p_) : p(p_) {}

    __device__ __forceinline__ uint32_t slot(int k) const {
        return sbase + (uint32_t)(k & (kMapRing - 1)) * kMapRowBytes;
    }
    // cp.async row yp (clamped) into ring slot k, then step to the next row.
    // The copy's lane mapping is NOT the compute mapping: copy k (0..8) of
    // lane L fills ring word 32k + L, i.e. pair (32k + L)/2 - 1 of chunk L&1
    // (window columns -1 .. 128 of both chunks, interleaved as pairs), so
    // every copy instruction reads two 64-byte runs of the row and writes 128
    // contiguous bytes of shared memory (no bank conflicts); a lane-per-
    // column mapping read 4 lines and hit one bank 8 times per instruction.
    __device__ __forceinline__ void prefetch_next(int k) {
        const uint32_t s = slot(k);
        const int c0 = lane / 2 - 1 + kMapChunk * (lane & 1);  // window column (chunk offset) of copy 0
        if (INTERIOR) {
            const char* g = pf + 4 * c0;
#pragma unroll
            for (int kk = 0; kk < kMapCopies; ++kk)
                cp_async4(s + 128 * kk + ((kk & 1) ? cpo : cpe), g + 64 * kk);
            if (tail4) cp_async4(s + 128 * kMapCopies + cpe, g + 64 * kMapCopies);
        } else {  // image-edge warp: clamped columns
            const float* row = reinterpret_cast<const float*>(pf);
#pragma unroll
            for (int kk = 0; kk < kMapCopies; ++kk)
                cp_async4(s + 128 * kk + ((kk & 1) ? cpo : cpe),
                          row + min(max(x0 + c0 + 16 * kk, 0), p.w - 1));
            if (tail4)
                cp_async4(s + 128 * kMapCopies + cpe,
                          row + min(max(x0 + c0 + 16 * kMapCopies, 0), p.w - 1));
        }
        // clamp-to-edge rows: rows < 0 read row 0, rows >= h read row h-1
        if ((unsigned)yp < (unsigned)(p.h - 1)) pf += pf_step;
        ++yp;
    }

    // 16-byte stores (chunk 0 = lo halves at x0 + 4i .., chunk 1 = hi halves
    // at x0 + 128 + 4i ..) where the rows are 16-byte aligned
    __device__ __forceinline__ void store(float* row, const float (&ol)[kMapCols],
                                          const float (&oh)[kMapCols]) const {
        if (ST128) {
            if constexpr (kMapCols == 4) {
                asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row), "f"(ol[0]),
                             "f"(ol[1]), "f"(ol[2]), "f"(ol[3]) : "memory");
                asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + kMapChunk),
                             "f"(oh[0]), "f"(oh[1]), "f"(oh[2]), "f"(oh[3]) : "memory");
            } else {
                asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(row), "f"(ol[0]), "f"(ol[1])
                             : "memory");
                asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(row + kMapChunk), "f"(oh[0]),
                             "f"(oh[1]) : "memory");
            }
            return;
        }
#pragma unroll
        for (int j = 0; j < kMapCols; ++j) {
            const int xa = x0 + kMapCols * lane + j;
            if (INTERIOR || xa < p.w) row[j] = ol[j];
            if (INTERIOR || xa + kMapChunk < p.w) row[kMapChunk + j] = oh[j];
        }
    }

    // One output row y: rows y-1, y in m, o (ROLL) or loaded here, y+1 into q.
    template <bool ROLL>
    __device__ __forceinline__ void row_step(int y, f2 (&m)[kMapNb], f2 (&o)[kMapNb],
                                             f2 (&q)[kMapNb], float*& sp, int64_t dpitch) {
        const int k = y - ys;  // slot of row y-1
        // rows y-1 .. y+1 landed: of the PD + k groups issued (rows up to
        // y+PD-2), at most PD-3 may still be pending
        asm volatile("cp.async.wait_group %0;" ::"n"(kMapPD - 3) : "memory");
        __syncwarp();
        if (yp <= ye) prefetch_next(k + kMapPD);  // row y+PD-1 (the strip needs rows <= ye)
        cp_async_commit();
        if (!ROLL) {  // rows y-1 and y too (rolled: already in registers)
            lds_row6(slot(k), co, m);
            lds_row6(slot(k + 1), co, o);
        }
        lds_row6(slot(k + 2), co, q);
        f2 V[kMapNb], W[kMapNb - 1];
        float ol[kMapCols], oh[kMapCols];  // chunk 0 / chunk 1 results
#pragma unroll
        for (int i = 0; i < kMapNb; ++i) V[i] = add2(m[i], q[i]);
#pragma unroll
        for (int i = 0; i < kMapNb - 1; ++i) W[i] = add2(V[i], V[i + 1]);
        bool rare = false;
#pragma unroll
        for (int j = 0; j < kMapCols; ++j) {
            bool r;
#if defined(CF_MAP_EXP) && CF_MAP_EXP == 1  // diagnostic (wrong results): data movement only
            {
                const f2 v = add2(add2(m[j + 1], q[j + 1]), W[j]);
                ol[j] = lo(v);
                oh[j] = hi(v);
            }
            r = false;
#elif defined(CF_MAP_EXP) && CF_MAP_EXP == 2  // diagnostic (wrong results): no selection
            {
                PairD D;
                f2 hb, t0;
                pair_d(m[j], m[j + 1], m[j + 2], o[j], o[j + 1], o[j + 2], q[j], q[j + 1],
                       q[j + 2], W[j], W[j + 1], hc[j], tm[j], hb, t0, D);
                hc[j] = hb;
                tm[j] = t0;
                const f2 v = add2(add2(add2(D.d[0], D.d[1]), add2(D.d[2], D.d[3])),
                                  add2(add2(D.d[4], D.d[5]), add2(D.d[6], D.d[7])));
                ol[j] = lo(v);
                oh[j] = hi(v);
                r = false;
            }
#else
            map_pair_s(m[j], m[j + 1], m[j + 2], o[j], o[j + 1], o[j + 2], q[j], q[j + 1],
                       q[j + 2], W[j], W[j + 1], hc[j], tm[j], ol[j], oh[j], r);
#endif
            rare |= r;
        }
        if (__any_sync(kFull, rare)) {  // rare: near ties / exact opposite-sign ties
            if (rare) {
#pragma unroll
                for (int j = 0; j < kMapCols; ++j) {
                    const f2 hw = map_pair_fix(m[j], m[j + 1], m[j + 2], o[j], o[j + 1],
                                               o[j + 2], q[j], q[j + 1], q[j + 2],
                                               pk(ol[j], oh[j]));
                    ol[j] = lo(hw);
                    oh[j] = hi(hw);
                }
            }
        }
        if constexpr (ENERGY) {  // the energy's segment sum of this row
            double t[2 * kMapCols];
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int j = 0; j < kMapCols; ++j) {
                    const int xa = x0 + kMapCols * lane + kMapChunk * c + j;
                    const float hv = c ? oh[j] : ol[j];
                    t[kMapCols * c + j] =
                        (INTERIOR || xa < p.w) ? energy_term<QK>(hv, p.q) : 0.0;
                }
            double acc = lane_tree8(t);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, o));
            if (lane == 0)
                p.seg_sums[(int64_t)(x0 / (2 * kMapChunk)) * p.planes * p.h + plane_row0 + y] =
                    acc;
        }
        if (!ENERGY || p.dst) {
            store(sp, ol, oh);
            sp += dpitch;
        }
    }

    __device__ __forceinline__ void run(float* dst) {
        // prologue: rows ys-1 .. ys-1+PD-1 -> slots 0 .. PD-1, a group each
#pragma unroll
        for (int k = 0; k < kMapPD; ++k) {
            prefetch_next(k);
            cp_async_commit();
        }
        // the first row's row sums (what it would have carried): rows ys-1, ys
        asm volatile("cp.async.wait_group %0;" ::"n"(kMapPD - 2) : "memory");
        __syncwarp();
        {
            f2 m[kMapNb], o[kMapNb];
            lds_row6(slot(0), co, m);
            lds_row6(slot(1), co, o);
#pragma unroll
            for (int j = 0; j < kMapCols; ++j) {
                hc[j] = add2(o[j], o[j + 2]);
                tm[j] = add2(add2(m[j], m[j + 2]), hc[j]);
            }
        }
        float* sp = dst ? dst + (int64_t)ys * p.dst_pitch + x0 + kMapCols * lane : nullptr;
        const int64_t dpitch = p.dst_pitch;
#if CF_MAP_ROLL
        // rows rolled through three register sets: one LDS row per step
        {
            f2 ra[kMapNb], rb[kMapNb], rc[kMapNb];
            lds_row6(slot(0), co, ra);
            lds_row6(slot(1), co, rb);
            int y = ys;
            for (; y + 3 <= ye; y += 3) {
                row_step<true>(y, ra, rb, rc, sp, dpitch);
                row_step<true>(y + 1, rb, rc, ra, sp, dpitch);
                row_step<true>(y + 2, rc, ra, rb, sp, dpitch);
            }
            for (; y < ye; ++y) {
                f2 m[kMapNb], o[kMapNb], q[kMapNb];
                row_step<false>(y, m, o, q, sp, dpitch);
            }
        }
#else
        for (int y = ys; y < ye; ++y) {
            f2 m[kMapNb], o[kMapNb], q[kMapNb];
            row_step<false>(y, m, o, q, sp, dpitch);
        }
#endif
        asm volatile("cp.async.wait_group 0;" ::: "memory");  // no copy outlives the warp
    }
};

#ifndef CF_MAP_MINB
#define CF_MAP_MINB 3  // resident blocks per SM the register budget targets
#endif
#ifndef CF_MAP_MINB_ENERGY
#define CF_MAP_MINB_ENERGY CF_MAP_MINB
#endif
// QK > 0: the fused energy epilogue (p.seg_sums; 1: |H|, 2: H*H, 3: sqrt,
// 4: pow), the map store then optional (p.dst nullable)
template <int QK>
__global__ void __launch_bounds__(32 * kMapWarps, QK ? CF_MAP_MINB_ENERGY : CF_MAP_MINB)
    wmc_map_kernel(const MapParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t task = (int64_t)blockIdx.x * kMapWarps + (threadIdx.x >> 5);
    const int64_t per_plane = (int64_t)p.n_pairs * p.n_strips;
    if (task >= per_plane * p.planes) return;  // warp-uniform
    const int plane = (int)(task / per_plane);
    const int64_t rest = task - (int64_t)plane * per_plane;
    const int strip = (int)(rest / p.n_pairs);
    const int cpair = (int)(rest - (int64_t)strip * p.n_pairs);
    const int lane = threadIdx.x & 31;
    const int x0 = cpair * 2 * kMapChunk;
    const float* src = p.src + (int64_t)plane * p.src_plane;
    float* dst = p.dst ? p.dst + (int64_t)plane * p.dst_plane : nullptr;
    const int ys = strip * p.strip_rows;
    const float* row0 = src + (int64_t)max(ys - 1, 0) * p.src_pitch;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem) +
                           (uint32_t)(threadIdx.x >> 5) * (kMapRing * kMapRowBytes);
    auto init = [&](auto& mw) {
        mw.lane = lane;
        mw.plane_row0 = (int64_t)plane * p.h;
        mw.ys = ys;
        mw.ye = min(ys + p.strip_rows, p.h);
        mw.x0 = x0;
        mw.src = src;
        mw.pf_step = p.src_pitch * 4;
        mw.tail4 = lane < 4;
        mw.yp = ys - 1;
        mw.sbase = sbase;
        // window columns C*i-1 .. C*i+C: 16-byte chunks C*i/2 + k (swizzled)
#pragma unroll
        for (int k = 0; k < kMapNb / 2; ++k)
            mw.co[k] = 16u * map_swz_chunk((uint32_t)(kMapCols * lane / 2 + k));
        // copy kk writes word 32kk + lane, i.e. chunk 8kk + lane/4: for odd kk
        // the swizzle flips bit 0 of the chunk (kk even: no change)
        mw.cpe = 16u * map_swz_chunk((uint32_t)(lane >> 2)) + 4u * (lane & 3);
        mw.cpo = 16u * (map_swz_chunk((uint32_t)(8 + (lane >> 2))) - 8u) + 4u * (lane & 3);
    };
    if (x0 > 0 && x0 + 2 * kMapChunk < p.w && p.st128) {
        MapWarp<true, QK, true> mw(p);
        init(mw);
        mw.pf = reinterpret_cast<const char*>(row0 + x0);
        mw.run(dst);
    } else if (x0 > 0 && x0 + 2 * kMapChunk < p.w) {
        MapWarp<true, QK> mw(p);
        init(mw);
        mw.pf = reinterpret_cast<const char*>(row0 + x0);
        mw.run(dst);
    } else {
        MapWarp<false, QK> mw(p);
        init(mw);
        mw.pf = reinterpret_cast<const char*>(row0);
        mw.run(dst);
    }
}

// ---------------------------------------------------------------------------
// Flat map kernel for small images: one thread per horizontal
// pixel pair loads its clamped 3x4 neighbourhood from global memory (L1/L2
// served) and runs map_pair with the same operands in the same order
// (V = a+e | b+f | c+g, W = V+V', H = l+r, T = (a+c)+(l+r)), so it is
// bit-identical to the streaming kernel.  A single small map is latency
// bound: every pixel pair in flight at once beats warps streaming strips.
__global__ void __launch_bounds__(256) wmc_map_flat_kernel(const float* __restrict__ src,
                                                          float* __restrict__ dst, int32_t w,
                                                          int32_t h, int64_t src_pitch,
                                                          int64_t src_plane, int64_t dst_pitch,
                                                          int64_t dst_plane, int32_t planes) {
    const int32_t pw = (w + 1) / 2;  // pixel pairs per row
    const int64_t n = (int64_t)pw * h * planes;
    // grid-stride with a warp-uniform trip count (map_pair votes)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t base = blockIdx.x * (int64_t)blockDim.x;
    for (int64_t i0 = base; i0 < n; i0 += stride) {
        const int64_t i = min(i0 + threadIdx.x, n - 1);  // tail lanes redo the last pair
        const bool live = i0 + threadIdx.x < n;
        const int32_t px = (int32_t)(i % pw);
        const int64_t r = i / pw;
        const int32_t y = (int32_t)(r % h);
        const int32_t pl = (int32_t)(r / h);
        const float* plane = src + pl * src_plane;
        const int x0 = 2 * px;
        int cxs[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) cxs[k] = min(max(x0 - 1 + k, 0), w - 1);
        const float* rows[3] = {plane + (int64_t)max(y - 1, 0) * src_pitch,
                                plane + (int64_t)y * src_pitch,
                                plane + (int64_t)min(y + 1, h - 1) * src_pitch};
        float v[3][4];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
            for (int k = 0; k < 4; ++k) v[rr][k] = __ldg(rows[rr] + cxs[k]);
        // pair k = {column x0-1+k, column x0+k}: the neighbourhood of the pixel pair
        f2 m[3], o[3], q[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            m[k] = pk(v[0][k], v[0][k + 1]);
            o[k] = pk(v[1][k], v[1][k + 1]);
            q[k] = pk(v[2][k], v[2][k + 1]);
        }
        const f2 V0 = add2(m[0], q[0]), V1 = add2(m[1], q[1]), V2 = add2(m[2], q[2]);
        const f2 Wm = add2(V0, V1), W0 = add2(V1, V2);
        f2 Hc = add2(o[0], o[2]);
        f2 Tm = add2(add2(m[0], m[2]), Hc);
        bool rare;
        f2 hw = map_pair(m[0], m[1], m[2], o[0], o[1], o[2], q[0], q[1], q[2], Wm, W0, Hc, Tm, rare);
        if (rare) hw = map_pair_fix(m[0], m[1], m[2], o[0], o[1], o[2], q[0], q[1], q[2], hw);
        if (live) {
            float* out = dst + pl * dst_plane + (int64_t)y * dst_pitch;
            out[x0] = lo(hw);
            if (x0 + 1 < w) out[x0 + 1] = hi(hw);
        }
    }
}

}  // namespace cfk
