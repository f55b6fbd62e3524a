// paper_1903_07189_b200/csrc/wmc_f64.cu -- the SPEC-faithful fp64 path:
// wmc_half_laplace and mc_flow(scheme=half_laplace) on fp64 images with the
// reference CPU path's own arithmetic ("fp64 internally"), so the
// results are BIT-IDENTICAL to the reference CPU implementation
// (oracle/wmc_px.h wmc_px_f64, run on the reference's executor by
// oracle/_ref), not merely within a tolerance.  DESIGN.md §3.6.
//
// The reference evaluation of one pixel (SPEC.md:53-61, :96-111, :171-179,
// :195): for each kernel h_i, s = 0; s = s + w_t * x_t over the 9 taps in
// row-major order (weights n/12 rounded to fp64 once, multiply and add
// rounded separately); m = the first i with the strictly smallest |s_i|.
// Here, exactly the same roundings:
//  * zero-weight taps are skipped: s + (+-0) == s because s is never -0
//    (it starts as 0 + p, and RN sums are -0 only when both operands are),
//    and images are finite (a non-finite iterate aborts the
//    flow in the iteration that produced it, the same one here);
//  * the centre tap's product (-1) * u is the exact negation -u;
//  * each (neighbour, weight) product fl(w * x) is formed once and reused by
//    every kernel that has that tap (16 DMUL per pixel), each kernel's sum
//    keeps its own row-major order (the 0 + p first step kept: it maps a -0
//    product to +0), and h2 / h5 share their identical two-term prefix;
//  * the argmin is the reference's sequential strict-< scan (NaN-faithful).
// The flow step is v = u + dt * d (two roundings), dt == 1 skips the exact
// multiplication.  Jacobi ping-pong through the workspace; non-finite values
// are flagged per iteration (atomicMin of the iteration into the flag), the
// first bad iteration named as SPEC.md:259 asks.
//
// The kernel is FP64-pipe bound (~60 DP ops per pixel-update): one warp
// per 32 columns streams a strip of rows with the 3x3 window in registers
// (clamped loads, L1-served), no shared memory.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>

#include "../../include/curveflow/capi.h"

extern "C" void cf_internal_set_cuda_error(int e);
extern "C" int cf_internal_graph_run(const void* key_bytes, size_t key_len, void* stream,
                                     int (*enqueue)(void* ctx, void* stream), void* ctx);

namespace {

constexpr int kStripRows = 64;   // rows per warp task
constexpr int kWarps = 4;        // warps per block
constexpr size_t kWsHeader = 256;

#define CF64_CUDA(x)                                                  \
    do {                                                              \
        cudaError_t e_ = (x);                                         \
        if (e_ != cudaSuccess) {                                      \
            cf_internal_set_cuda_error((int)e_);                      \
            return CF_ECUDA;                                          \
        }                                                             \
    } while (0)

// fl(n/12) for n = 1, 2, 4 (the compiler's constant folding of n / 12.0 is
// the IEEE quotient, as the oracle's (double)n / 12.0)
constexpr double kW1 = 1.0 / 12.0, kW2 = 2.0 / 12.0, kW4 = 4.0 / 12.0;

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// The SPEC-faithful fp64 d_m of one pixel from its (clamped) neighbourhood.
__device__ __forceinline__ double wmc_px64(double a, double b, double c, double l, double u,
                                          double r, double e, double f, double g) {
    const double a1 = dmul(kW1, a), a2 = dmul(kW2, a);
    const double b2 = dmul(kW2, b), b4 = dmul(kW4, b);
    const double c1 = dmul(kW1, c), c2 = dmul(kW2, c);
    const double l2 = dmul(kW2, l), l4 = dmul(kW4, l);
    const double r2 = dmul(kW2, r), r4 = dmul(kW4, r);
    const double e1 = dmul(kW1, e), e2 = dmul(kW2, e);
    const double f2 = dmul(kW2, f), f4 = dmul(kW4, f);
    const double g1 = dmul(kW1, g), g2 = dmul(kW2, g);
    const double nu = -u;
    // first terms 0 + p (a -0 product becomes +0, as in the reference)
    const double za2 = dadd(0.0, a2), zb2 = dadd(0.0, b2), zl2 = dadd(0.0, l2);
    const double za1 = dadd(0.0, a1), zc1 = dadd(0.0, c1);
    const double pab4 = dadd(za2, b4);  // shared prefix of h2 and h5
    double d[8];
    d[0] = dadd(dadd(dadd(dadd(dadd(za2, b2), l4), nu), e2), f2);      // h1: a b l u e f
    d[1] = dadd(dadd(dadd(dadd(pab4, c2), l2), nu), r2);               // h2: a b c l u r
    d[2] = dadd(dadd(dadd(dadd(dadd(zb2, c2), nu), r4), f2), g2);      // h3: b c u r f g
    d[3] = dadd(dadd(dadd(dadd(dadd(zl2, nu), r2), e2), f4), g2);      // h4: l u r e f g
    d[4] = dadd(dadd(dadd(dadd(pab4, c1), l4), nu), e1);               // h5: a b c l u e
    d[5] = dadd(dadd(dadd(dadd(dadd(za1, b4), c2), nu), r4), g1);      // h6: a b c u r g
    d[6] = dadd(dadd(dadd(dadd(dadd(zc1, nu), r4), e1), f4), g2);      // h7: c u r e f g
    d[7] = dadd(dadd(dadd(dadd(dadd(za1, l4), nu), e2), f4), g1);      // h8: a l u e f g
    double best = d[0];
#pragma unroll
    for (int i = 1; i < 8; ++i)  // strict <, first minimum, sequential scan
        if (fabs(d[i]) < fabs(best)) best = d[i];
    return best;
}

struct Step64 {
    const double* src;
    double* dst;
    int64_t src_pitch, src_plane, dst_pitch, dst_plane;
    int32_t w, h, planes;
    int32_t n_colw;       // warps across a row (ceil(w / 32))
    int32_t n_strips;     // strips down a plane
    double dt;
    int32_t flow;         // 0: map (dst = d_m), 1: flow step (dst = u + dt * d_m)
    int32_t iter;         // 1-based iteration of this step (flow)
    int32_t* flag;        // nullable: atomicMin(flag, iter) on a non-finite output
};

__global__ void __launch_bounds__(32 * kWarps) wmc_f64_kernel(const Step64 p) {
    const int64_t task = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int64_t per_plane = (int64_t)p.n_colw * p.n_strips;
    if (task >= per_plane * p.planes) return;
    const int plane = (int)(task / per_plane);
    const int64_t rest = task - (int64_t)plane * per_plane;
    const int strip = (int)(rest / p.n_colw), cw = (int)(rest - (int64_t)strip * p.n_colw);
    const int lane = threadIdx.x & 31;
    const int x = cw * 32 + lane;
    const bool live = x < p.w;
    const int xc = min(x, p.w - 1);
    const int xl = max(xc - 1, 0), xr = min(xc + 1, p.w - 1);
    const int y0 = strip * kStripRows, y1 = min(y0 + kStripRows, p.h);
    const double* src = p.src + (int64_t)plane * p.src_plane;
    double* dst = p.dst + (int64_t)plane * p.dst_plane;
    auto row = [&](int y) { return src + (int64_t)min(max(y, 0), p.h - 1) * p.src_pitch; };
    const double* rm = row(y0 - 1);
    const double* r0 = row(y0);
    const double* r1 = row(y0 + 1);
    double a = __ldg(rm + xl), b = __ldg(rm + xc), c = __ldg(rm + xr);
    double l = __ldg(r0 + xl), u = __ldg(r0 + xc), r = __ldg(r0 + xr);
    double e = __ldg(r1 + xl), f = __ldg(r1 + xc), g = __ldg(r1 + xr);
    // software pipeline: rows y+2 and y+3 are in flight while row y computes
    // (with one row ahead the DMULs still waited on their loads: ncu
    // long-scoreboard 40 % of stall samples)
    const double* rn = row(y0 + 2);
    double n1e = __ldg(rn + xl), n1f = __ldg(rn + xc), n1g = __ldg(rn + xr);
    if (y0 + 2 < p.h - 1) rn += p.src_pitch;
    double n2e = __ldg(rn + xl), n2f = __ldg(rn + xc), n2g = __ldg(rn + xr);
    if (y0 + 3 < p.h - 1) rn += p.src_pitch;
    bool bad = false;
#pragma unroll 2
    for (int y = y0; y < y1; ++y) {
        const double n3e = __ldg(rn + xl), n3f = __ldg(rn + xc), n3g = __ldg(rn + xr);  // row y+4
        if (y + 4 < p.h - 1) rn += p.src_pitch;  // clamp at the last row
        const double dm = wmc_px64(a, b, c, l, u, r, e, f, g);
        double v;
        if (p.flow) {
            v = dadd(u, p.dt == 1.0 ? dm : dmul(p.dt, dm));  // 1 * d == d exactly
            bad |= !isfinite(v);
        } else {
            v = dm;
        }
        if (live) dst[(int64_t)y * p.dst_pitch + x] = v;
        a = l; b = u; c = r;
        l = e; u = f; r = g;
        e = n1e; f = n1f; g = n1g;
        n1e = n2e; n1f = n2f; n1g = n2g;
        n2e = n3e; n2f = n3f; n2g = n3g;
    }
    if (p.flag && __any_sync(0xffffffffu, bad && live) && lane == 0) atomicMin(p.flag, p.iter);
}

// u8 -> fp64 widening q / 255.0 with IEEE division (the
// reference widens on load in fp64).
__global__ void u8_to_f64_kernel(const uint8_t* in, int64_t in_pitch, int64_t in_plane,
                                 double* out, int64_t pitch, int64_t plane, int32_t w, int32_t h,
                                 int32_t planes) {
    const int64_t n = (int64_t)w * h * planes;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % w, r = i / w, y = r % h, pl = r / h;
        const uint8_t q = in[pl * in_plane + y * in_pitch + x];
        out[pl * plane + y * pitch + x] = __ddiv_rn((double)q, 255.0);
    }
}

struct DevCount {
    int sms = 0;
};

int sm_count(int* out) {
    int dev = 0, sms = 0, maj = 0, min_ = 0;
    CF64_CUDA(cudaGetDevice(&dev));
    CF64_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CF64_CUDA(cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev));
    CF64_CUDA(cudaDeviceGetAttribute(&min_, cudaDevAttrComputeCapabilityMinor, dev));
    if (maj != 10 || min_ != 0) return CF_ENODEV;
    *out = sms;
    return CF_OK;
}

bool shape_ok64(int32_t w, int32_t h, int64_t pitch, int32_t planes, int64_t plane_stride) {
    if (w <= 0 || h <= 0 || planes <= 0 || pitch < w) return false;
    if (planes > 1 && plane_stride < pitch * (int64_t)h) return false;
    if ((int64_t)w > (1 << 30) || (int64_t)h > (1 << 30)) return false;
    return true;
}

int launch_step(const double* src, int64_t src_pitch, int64_t src_plane, double* dst,
                int64_t dst_pitch, int64_t dst_plane, int32_t w, int32_t h, int32_t planes,
                bool flow, double dt, int32_t iter, int32_t* flag, cudaStream_t s) {
    Step64 p{};
    p.src = src; p.dst = dst;
    p.src_pitch = src_pitch; p.src_plane = src_plane;
    p.dst_pitch = dst_pitch; p.dst_plane = dst_plane;
    p.w = w; p.h = h; p.planes = planes;
    p.n_colw = (w + 31) / 32;
    p.n_strips = (h + kStripRows - 1) / kStripRows;
    p.dt = dt; p.flow = flow ? 1 : 0; p.iter = iter; p.flag = flag;
    const int64_t tasks = (int64_t)p.n_colw * p.n_strips * planes;
    const int64_t blocks = (tasks + kWarps - 1) / kWarps;
    if (blocks > INT_MAX) return CF_EINVAL;
    wmc_f64_kernel<<<(unsigned)blocks, 32 * kWarps, 0, s>>>(p);
    CF64_CUDA(cudaGetLastError());
    return CF_OK;
}

struct Flow64 {
    const uint8_t* src8;  // nullable: widen from u8 first
    int64_t src8_pitch, src8_plane;
    double* img;
    int32_t w, h;
    int64_t pitch;
    int32_t planes;
    int64_t plane_stride;
    int32_t iters;
    double dt;
    void* ws;
};

int enqueue_flow64(void* ctx, void* stream) {
    const Flow64& f = *static_cast<const Flow64*>(ctx);
    cudaStream_t s = (cudaStream_t)stream;
    int sms = 0;
    if (int rc = sm_count(&sms)) return rc;
    int32_t* flag = static_cast<int32_t*>(f.ws);
    double* tmp = reinterpret_cast<double*>(static_cast<char*>(f.ws) + kWsHeader);
    CF64_CUDA(cudaMemsetAsync(flag, 0x7f, sizeof(int32_t), s));
    double* cur = f.img;
    double* nxt = tmp;
    if (f.iters % 2 == 1) std::swap(cur, nxt);  // the last step lands in img
    if (f.src8) {
        const int64_t n = (int64_t)f.w * f.h * f.planes;
        const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16);
        u8_to_f64_kernel<<<(unsigned)blocks, 256, 0, s>>>(f.src8, f.src8_pitch, f.src8_plane, cur,
                                                          f.pitch, f.plane_stride, f.w, f.h,
                                                          f.planes);
        CF64_CUDA(cudaGetLastError());
    } else if (cur != f.img) {
        for (int pl = 0; pl < f.planes; ++pl)
            CF64_CUDA(cudaMemcpy2DAsync(cur + pl * f.plane_stride, f.pitch * 8,
                                        f.img + pl * f.plane_stride, f.pitch * 8,
                                        (size_t)f.w * 8, f.h, cudaMemcpyDeviceToDevice, s));
    }
    for (int t = 1; t <= f.iters; ++t) {
        if (int rc = launch_step(cur, f.pitch, f.plane_stride, nxt, f.pitch, f.plane_stride, f.w,
                                 f.h, f.planes, true, f.dt, t, flag, s))
            return rc;
        std::swap(cur, nxt);
    }
    return CF_OK;
}

int query_flag(const void* ws, int32_t* first_bad_iter, cudaStream_t s) {
    int32_t host = 0x7f7f7f7f;
    CF64_CUDA(cudaMemcpyAsync(&host, ws, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CF64_CUDA(cudaStreamSynchronize(s));
    if (host >= 0x7f7f7f7f || host <= 0) {
        *first_bad_iter = 0;
        return CF_OK;
    }
    *first_bad_iter = host;
    return CF_ENONFINITE;
}

int run_flow64(const Flow64& f, int32_t* first_bad_iter, cudaStream_t s) {
    // graph-cache key: every argument (the flow is a chain of `iters` launches)
    struct Key {
        char tag[4];
        const void* src8; int64_t src8_pitch, src8_plane;
        void* img; int32_t w, h; int64_t pitch; int32_t planes; int64_t plane_stride;
        int32_t iters; double dt; void* ws;
    } key;
    std::memset(&key, 0, sizeof(key));
    std::memcpy(key.tag, "f64", 4);
    key.src8 = f.src8; key.src8_pitch = f.src8_pitch; key.src8_plane = f.src8_plane;
    key.img = f.img; key.w = f.w; key.h = f.h; key.pitch = f.pitch; key.planes = f.planes;
    key.plane_stride = f.plane_stride; key.iters = f.iters; key.dt = f.dt; key.ws = f.ws;
    Flow64 copy = f;
    if (int rc = cf_internal_graph_run(&key, sizeof(key), s, enqueue_flow64, &copy)) return rc;
    if (first_bad_iter) return query_flag(f.ws, first_bad_iter, s);
    return CF_OK;
}

}  // namespace

extern "C" {

CF_API int cf_wmc_map_f64(const double* in, double* out, int32_t w, int32_t h, int64_t pitch,
                          int32_t planes, int64_t plane_stride, void* stream) {
    if (!in || !out || in == out || !shape_ok64(w, h, pitch, planes, plane_stride))
        return CF_EINVAL;
    int sms = 0;
    if (int rc = sm_count(&sms)) return rc;
    return launch_step(in, pitch, plane_stride, out, pitch, plane_stride, w, h, planes, false, 0.0,
                       0, nullptr, (cudaStream_t)stream);
}

CF_API size_t cf_wmc_filter_f64_workspace_bytes(int32_t w, int32_t h, int64_t pitch,
                                                int32_t planes, int64_t plane_stride) {
    if (!shape_ok64(w, h, pitch, planes, plane_stride)) return 0;
    const int64_t elems = (planes - 1) * (planes > 1 ? plane_stride : 0) + pitch * (int64_t)h;
    return kWsHeader + (size_t)elems * sizeof(double);
}

CF_API int cf_wmc_filter_f64(double* img, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                             int64_t plane_stride, int32_t iters, double dt, void* workspace,
                             size_t workspace_bytes, int32_t* first_bad_iter, void* stream) {
    if (!img || !shape_ok64(w, h, pitch, planes, plane_stride) || iters < 0) return CF_EINVAL;
    if (!(dt > 0.0) || dt > 1.0) return CF_EINVAL;
    if (first_bad_iter) *first_bad_iter = 0;
    if (iters == 0) return CF_OK;                   // identity
    if (!workspace ||
        workspace_bytes < cf_wmc_filter_f64_workspace_bytes(w, h, pitch, planes, plane_stride))
        return CF_EINVAL;
    Flow64 f{};
    f.img = img; f.w = w; f.h = h; f.pitch = pitch; f.planes = planes;
    f.plane_stride = plane_stride; f.iters = iters; f.dt = dt; f.ws = workspace;
    return run_flow64(f, first_bad_iter, (cudaStream_t)stream);
}

CF_API int cf_wmc_filter_u8_f64(const uint8_t* in, int64_t in_pitch, int64_t in_plane_stride,
                                double* out, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                                int64_t plane_stride, int32_t iters, double dt, void* workspace,
                                size_t workspace_bytes, int32_t* first_bad_iter, void* stream) {
    if (!in || !out || !shape_ok64(w, h, pitch, planes, plane_stride) || iters < 0)
        return CF_EINVAL;
    if (in_pitch < w || (planes > 1 && in_plane_stride < in_pitch * (int64_t)h)) return CF_EINVAL;
    if (!(dt > 0.0) || dt > 1.0) return CF_EINVAL;
    if (first_bad_iter) *first_bad_iter = 0;
    if (!workspace ||
        workspace_bytes < cf_wmc_filter_f64_workspace_bytes(w, h, pitch, planes, plane_stride))
        return CF_EINVAL;
    Flow64 f{};
    f.src8 = in; f.src8_pitch = in_pitch; f.src8_plane = in_plane_stride;
    f.img = out; f.w = w; f.h = h; f.pitch = pitch; f.planes = planes;
    f.plane_stride = plane_stride; f.iters = iters; f.dt = dt; f.ws = workspace;
    return run_flow64(f, first_bad_iter, (cudaStream_t)stream);
}

CF_API int cf_wmc_filter_f64_query_nonfinite(const void* workspace, int32_t* first_bad_iter,
                                             void* stream) {
    if (!workspace || !first_bad_iter) return CF_EINVAL;
    return query_flag(workspace, first_bad_iter, (cudaStream_t)stream);
}

}  // extern "C"
