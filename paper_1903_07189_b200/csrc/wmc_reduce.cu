// paper_1903_07189_b200/csrc/wmc_reduce.cu -- reductions over the WMC map
// (SURVEY.md §8f rank 2): the WMC regularisation energy and the WMC value
// histogram; plus the solvers' data-fidelity sums (SolveReport series).
//
// Reference semantics:
//  * energy(img, kind = WMC, q) = sum over pixels of |H^w|^q with H^w from
//    wmc_half_laplace, q > 0 (default 1); "parallel
//    reduction allowed with fixed summation order per row then ordered row
//    combine (deterministic)".
//  * corpus_stats histograms wmc_half_laplace values with bins of width 1
//    over [-256, 256]; counts are integers.
//
// Fixed order of the ENERGY (round 2; restated by the oracle, bit-exact) --
// the map kernel's own layout (csrc/wmc_map.cuh), so the reduction can run
// as the map's epilogue:
//  per plane, per row y: the row is cut into 256-column segments; lane i of
//  a segment owns columns 4i .. 4i+3 and 128+4i .. 128+4i+3, terms t0..t7 in
//  that order (|H|^q in fp64; columns past w give 0), summed as the tree
//  ((t0+t1)+(t2+t3)) + ((t4+t5)+(t6+t7)); the 32 lane sums combine by the
//  butterfly tree of a warp xor-shuffle reduction (offsets 16, 8, 4, 2, 1);
//  a row sum is the sequential sum of its segment sums in x order (from 0);
//  the plane's energy is the sequential sum of its row sums in y order, and
//  planes add in plane order.
// The FIDELITY sums (SolveReport series) use the same order with terms
// |u - f|^q, the difference taken in fp64.
//  q = 1 -> |H|, q = 2 -> H*H, q = 0.5 -> sqrt(|H|) (correctly rounded, so
//  bit-exact); any other q uses pow() (documented 1e-12 relative tolerance).
// The map itself is cf_wmc_map_f32 (fp32, fp64 near-tie rule).
#include <algorithm>
#include <climits>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/curveflow/capi.h"

extern "C" void cf_internal_set_cuda_error(int e);  // wmc_capi.cu (not exported)
extern "C" int cf_internal_map_energy_segs(const float* in, int32_t w, int32_t h, int64_t pitch,
                                           int32_t planes, int64_t plane_stride, double q,
                                           int32_t qkind, double* seg_sums, void* stream);

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double term_abs(double a, double q, int qkind) {
    switch (qkind) {
        case 1: return a;
        case 2: return __dmul_rn(a, a);
        case 3: return __dsqrt_rn(a);
        default: return pow(a, q);
    }
}

__device__ __forceinline__ double term(float hw, double q, int qkind) {
    return term_abs(fabs((double)hw), q, qkind);
}

// One warp per (row, 256-column segment): the reduction order's segment sum
// (lane terms as a pairwise tree, then the xor butterfly), written by lane 0
// into seg_sums[segment][row].  Terms: |map|^q, or (fidelity, f2 set or not)
// |u - f|^q with the difference in fp64.
__global__ void seg_sum_kernel(const float* __restrict__ map, const float* __restrict__ f2,
                               bool fid, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                               int64_t plane_stride, double q, int qkind, int32_t nseg,
                               double* __restrict__ seg_sums) {
    const int lane = threadIdx.x & 31;
    const int64_t task = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (task >= (int64_t)h * planes * nseg) return;
    const int64_t row = task / nseg;
    const int s = (int)(task - row * nseg);
    const int64_t p = row / h, y = row % h;
    const int64_t off = p * plane_stride + y * pitch;
    const float* r = map + off;
    const int x0 = 256 * s + 4 * lane;
    double t[8];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = x0 + 128 * c + j;
            double v = 0.0;
            if (x < w) {
                if (fid) {
                    const double a = f2 ? __dsub_rn((double)r[x], (double)f2[off + x]) : (double)r[x];
                    v = term_abs(fabs(a), q, qkind);
                } else {
                    v = term(r[x], q, qkind);
                }
            }
            t[4 * c + j] = v;
        }
    double acc = __dadd_rn(__dadd_rn(__dadd_rn(t[0], t[1]), __dadd_rn(t[2], t[3])),
                           __dadd_rn(__dadd_rn(t[4], t[5]), __dadd_rn(t[6], t[7])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(kFull, acc, o));
    if (lane == 0) seg_sums[(int64_t)s * h * planes + row] = acc;  // [segment][row]
}

// Row sums: the segment sums of each row added in x order (one thread a
// row; segment sums stored [segment][row], so every step reads coalesced).
__global__ void row_from_segs_kernel(const double* __restrict__ seg_sums, int32_t nseg,
                                     int64_t nrows, double* __restrict__ row_sums) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= nrows) return;
    double acc = 0.0;
    for (int i = 0; i < nseg; ++i) acc = __dadd_rn(acc, seg_sums[(int64_t)i * nrows + row]);
    row_sums[row] = acc;
}

// Ordered combine of the row sums: h*planes sequential adds by one thread,
// the operands staged through shared memory by the whole block (the adds are
// a dependent chain; the loads are not, so they must not sit in it).
__global__ void __launch_bounds__(1024) ordered_sum_kernel(const double* __restrict__ row_sums,
                                                           int64_t n, double* __restrict__ out) {
    __shared__ double buf[4096];
    double s = 0.0;
    for (int64_t base = 0; base < n; base += 4096) {
        const int m = n - base < 4096 ? (int)(n - base) : 4096;
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) buf[i] = row_sums[base + i];
        __syncthreads();
        if (threadIdx.x == 0)
            for (int i = 0; i < m; ++i) s = __dadd_rn(s, buf[i]);
    }
    if (threadIdx.x == 0) *out = s;
}

// bin = floor((v*scale - lo) / width), out-of-range -> clamped ends, NaN -> 0
__device__ __forceinline__ int hist_bin(float v, float scale, float lo, float width, int nbins) {
    const float d = __fsub_rn(__fmul_rn(v, scale), lo);
    const float t = width == 1.0f ? d : __fdiv_rn(d, width);  // x / 1 == x exactly
    int b = (t != t) ? 0 : (int)floorf(fminf(fmaxf(t, -1.0f), (float)nbins));
    return min(max(b, 0), nbins - 1);
}

// Warp-private histograms in shared memory (32-bit counts, one per warp when
// they fit, else one per block); the block's counts then go to the global
// 64-bit counts.  Rows are walked whole
// (coalesced loads, no per-element division).  WMC values pile into a few
// bins, so global atomics per element serialised on them: 52 ms for 16384^2.
__global__ void histogram_smem_kernel(const float* __restrict__ map, int32_t w, int32_t h,
                                      int64_t pitch, int32_t planes, int64_t plane_stride,
                                      float scale, float lo, float width, int32_t nbins,
                                      unsigned long long* __restrict__ counts) {
    extern __shared__ unsigned int shm[];
    // one sub-histogram per warp when they fit (no contention between the
    // warps on the hot bins), else one per block
    const int nsub = (int)(blockDim.x >> 5) * nbins <= 12288 ? (int)(blockDim.x >> 5) : 1;
    for (int i = threadIdx.x; i < nsub * nbins; i += blockDim.x) shm[i] = 0u;
    __syncthreads();
    unsigned int* sh = shm + (nsub > 1 ? (threadIdx.x >> 5) * nbins : 0);
    const int64_t rows = (int64_t)h * planes;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int64_t p = r / h, y = r - p * h;
        const float* row = map + p * plane_stride + y * pitch;
        for (int x0 = 0; x0 < w; x0 += blockDim.x) {  // warp-uniform trip count
            const int x = x0 + (int)threadIdx.x;
            const bool live = x < w;
            // (merging same-bin lanes with __match_any_sync first cost more than
            // the shared atomics it saves: 1.90 vs 1.08 ms for 16384^2)
            if (live) atomicAdd(&sh[hist_bin(row[x], scale, lo, width, nbins)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) {
        unsigned long long c = 0;
        for (int k = 0; k < nsub; ++k) c += shm[k * nbins + i];
        if (c) atomicAdd(counts + i, c);
    }
}

__global__ void histogram_kernel(const float* __restrict__ map, int32_t w, int32_t h,
                                 int64_t pitch, int32_t planes, int64_t plane_stride, float scale,
                                 float lo, float width, int32_t nbins,
                                 unsigned long long* __restrict__ counts) {
    const int64_t n = (int64_t)w * h * planes;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)w * h), rem = i % ((int64_t)w * h);
        const float v = map[p * plane_stride + (rem / w) * pitch + rem % w];
        atomicAdd(counts + hist_bin(v, scale, lo, width, nbins), 1ull);
    }
}

int fail() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        cf_internal_set_cuda_error((int)e);
        return CF_ECUDA;
    }
    return CF_OK;
}

int qkind_of(double q) { return q == 1.0 ? 1 : (q == 2.0 ? 2 : (q == 0.5 ? 3 : 0)); }

}  // namespace

extern "C" {

CF_API size_t cf_wmc_reduce_workspace_bytes(int32_t w, int32_t h, int32_t planes) {
    if (w <= 0 || h <= 0 || planes <= 0) return 0;
    const size_t map = (((size_t)w * h * planes * sizeof(float)) + 255) & ~(size_t)255;
    const size_t nseg = ((size_t)w + 255) / 256;
    // map | row sums | segment sums
    return map + (((size_t)h * planes * sizeof(double) + 255) & ~(size_t)255) +
           (size_t)h * planes * nseg * sizeof(double) + 256;
}

CF_API int cf_wmc_energy_f64(const float* img, int32_t w, int32_t h, int64_t pitch,
                             int32_t planes, int64_t plane_stride, double q, double* d_out,
                             void* workspace, size_t workspace_bytes, void* stream) {
    if (!img || !d_out || !workspace || w <= 0 || h <= 0 || planes <= 0 || pitch < w)
        return CF_EINVAL;
    if (planes > 1 && plane_stride < pitch * (int64_t)h) return CF_EINVAL;
    if (!(q > 0.0) || !(q < 1e300)) return CF_EINVAL;
    if (workspace_bytes < cf_wmc_reduce_workspace_bytes(w, h, planes)) return CF_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    float* map = reinterpret_cast<float*>(workspace);
    const size_t map_bytes = (((size_t)w * h * planes * sizeof(float)) + 255) & ~(size_t)255;
    double* rows = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + map_bytes);
    const int64_t nrows = (int64_t)h * planes;
    const int32_t nseg = (w + 255) / 256;
    double* segs = reinterpret_cast<double*>(
        reinterpret_cast<char*>(rows) + ((nrows * sizeof(double) + 255) & ~(size_t)255));
    // large images: the segment sums come straight out of the map kernel's
    // epilogue (no map stored or re-read); small ones: map, then reduce it
    const int fused = cf_internal_map_energy_segs(img, w, h, pitch, planes, plane_stride, q,
                                                  qkind_of(q), segs, stream);
    if (fused != CF_OK && fused != CF_EINVAL) return fused;
    if (fused == CF_EINVAL) {
        // dense copy of the map (pitch = w) so the layout is independent of the input's
        for (int p = 0; p < planes; ++p) {
            int rc = cf_wmc_map_f32(img + p * plane_stride, map + (int64_t)p * w * h, w, h, pitch,
                                    1, (int64_t)w * h, stream);
            if (rc) return rc;
        }
        const int64_t tasks = nrows * nseg;
        seg_sum_kernel<<<(unsigned)((tasks + 7) / 8), 256, 0, s>>>(
            map, nullptr, false, w, h, w, planes, (int64_t)w * h, q, qkind_of(q), nseg, segs);
    }
    row_from_segs_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(segs, nseg, nrows, rows);
    ordered_sum_kernel<<<1, 1024, 0, s>>>(rows, nrows, d_out);
    return fail();
}

CF_API int cf_wmc_fidelity_f64(const float* u, const float* f, int32_t w, int32_t h,
                               int64_t pitch, int32_t planes, int64_t plane_stride, double q,
                               double* d_out, void* workspace, size_t workspace_bytes,
                               void* stream) {
    if (!u || !d_out || !workspace || w <= 0 || h <= 0 || planes <= 0 || pitch < w)
        return CF_EINVAL;
    if (planes > 1 && plane_stride < pitch * (int64_t)h) return CF_EINVAL;
    if (!(q > 0.0) || !(q < 1e300)) return CF_EINVAL;
    if (workspace_bytes < cf_wmc_reduce_workspace_bytes(w, h, planes)) return CF_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    double* rows = reinterpret_cast<double*>(workspace);
    const int64_t nrows = (int64_t)h * planes;
    const int32_t nseg = (w + 255) / 256;
    double* segs = reinterpret_cast<double*>(
        reinterpret_cast<char*>(rows) + ((nrows * sizeof(double) + 255) & ~(size_t)255));
    const int64_t tasks = nrows * nseg;
    seg_sum_kernel<<<(unsigned)((tasks + 7) / 8), 256, 0, s>>>(
        u, f, true, w, h, pitch, planes, plane_stride, q, qkind_of(q), nseg, segs);
    row_from_segs_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(segs, nseg, nrows, rows);
    ordered_sum_kernel<<<1, 1024, 0, s>>>(rows, nrows, d_out);
    return fail();
}

CF_API int cf_wmc_histogram(const float* img, int32_t w, int32_t h, int64_t pitch,
                            int32_t planes, int64_t plane_stride, float scale, float lo,
                            float width, int32_t nbins, uint64_t* d_counts, void* workspace,
                            size_t workspace_bytes, void* stream) {
    if (!img || !d_counts || !workspace || w <= 0 || h <= 0 || planes <= 0 || pitch < w)
        return CF_EINVAL;
    if (planes > 1 && plane_stride < pitch * (int64_t)h) return CF_EINVAL;
    if (nbins <= 0 || !(width > 0.0f) || !(scale == scale) || !(lo == lo)) return CF_EINVAL;
    if (workspace_bytes < cf_wmc_reduce_workspace_bytes(w, h, planes)) return CF_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    float* map = reinterpret_cast<float*>(workspace);
    for (int p = 0; p < planes; ++p) {
        int rc = cf_wmc_map_f32(img + p * plane_stride, map + (int64_t)p * w * h, w, h, pitch, 1,
                                (int64_t)w * h, stream);
        if (rc) return rc;
    }
    if (cudaMemsetAsync(d_counts, 0, sizeof(uint64_t) * nbins, s) != cudaSuccess) return fail();
    auto* c64 = reinterpret_cast<unsigned long long*>(d_counts);
    const int64_t rows = (int64_t)h * planes;
    // shared-memory path: up to 12288 bins (48 KB) and fewer than 2^32
    // pixels per block (the 32-bit shared counts cannot overflow)
    const int blocks = (int)std::min<int64_t>(rows, 148 * 8);
    const int64_t per_block = ((rows + blocks - 1) / blocks) * (int64_t)w;
    if (nbins <= 12288 && per_block < (int64_t)UINT32_MAX) {
        const size_t shb = (size_t)(8 * nbins <= 12288 ? 8 : 1) * nbins * sizeof(unsigned);
        histogram_smem_kernel<<<blocks, 256, shb, s>>>(
            map, w, h, w, planes, (int64_t)w * h, scale, lo, width, nbins, c64);
    } else {
        histogram_kernel<<<1184, 256, 0, s>>>(map, w, h, w, planes, (int64_t)w * h, scale, lo,
                                              width, nbins, c64);
    }
    return fail();
}

}  // extern "C"
