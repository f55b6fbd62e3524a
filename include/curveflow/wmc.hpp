// include/curveflow/wmc.hpp -- C++ host API of the B200 WMC path.
//
// Mirrors the reference's C++ surface in namespace curveflow (SPEC.md:29-89
// core types, :250-253 FlowConfig, :171 wmc_half_laplace, :256 mc_flow;
// the reference's only shipped header is curveflow/parallel.hpp) on top of
// the C-ABI in capi.h.  Header-only; link libcurveflow_b200.so and cudart.
//
//   curveflow::Image2D img = ...;                         // host, row-major
//   auto hw  = curveflow::cuda::wmc_half_laplace(img);     // H2D, kernel, D2H
//   auto out = curveflow::cuda::mc_flow(img, {1.0, 100});  // throws FlowError
//   curveflow::Image2D64 ref = ...;                       // fp64, the reference's type
//   auto same = curveflow::cuda::exact::mc_flow(ref, {1.0, 100});  // == reference CPU path
//
// Device-pointer overloads (curveflow::cuda::device::...) skip the copies and
// are stream-ordered.  There is no CPU fallback.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "capi.h"

namespace curveflow {

// SPEC.md:34-39.  This build computes in fp32; data.size()
// == width * height, row-major, x = column, y = row.
struct Image2D {
    int width = 0, height = 0;
    std::vector<float> data;
    Image2D() = default;
    Image2D(int w, int h, float v = 0.0f) : width(w), height(h), data((size_t)w * h, v) {}
    float& at(int y, int x) { return data[(size_t)y * width + x]; }
    float at(int y, int x) const { return data[(size_t)y * width + x]; }
};

// SPEC.md:34-39 in the reference's own precision: fp64 images, processed by
// curveflow::cuda::exact:: with the reference CPU path's arithmetic
// -- results bit-identical to the reference's.
struct Image2D64 {
    int width = 0, height = 0;
    std::vector<double> data;
    Image2D64() = default;
    Image2D64(int w, int h, double v = 0.0) : width(w), height(h), data((size_t)w * h, v) {}
    double& at(int y, int x) { return data[(size_t)y * width + x]; }
    double at(int y, int x) const { return data[(size_t)y * width + x]; }
};

// SPEC.md:250-253.  dt default 1.0 for half_laplace; 0 < dt <= 1.
struct FlowConfig {
    double dt = 1.0;
    int iters = 0;
    enum class Scheme { half_laplace, fd } scheme = Scheme::half_laplace;
};

// SPEC.md:286-289 with operator A = identity.
struct SolverConfig {
    double lambda = 0.0;
    double alpha = 1.0;   // l1 dual constant
    double dt = 0.15;
    int iters = 500;
    enum class Model { l2_area, l1_area } model = Model::l2_area;
};

// SPEC.md:290-293 (final state; the per-iteration series are built by the
// Python SolverConfig.report mode).  fidelity: l2 0.5*||U-f||^2, l1 ||U-f||_1.
struct SolveReport {
    Image2D image;
    Image2D dual;         // l1: final d; empty for l2
    int iters = 0;
    double fidelity = 0.0;
};

class Error : public std::runtime_error {
   public:
    Error(int status, const std::string& what)
        : std::runtime_error(what + ": " + cf_status_string(status)), status_(status) {}
    int status() const { return status_; }

   private:
    int status_;
};

// mc_flow aborts naming the iteration that went non-finite.
class FlowError : public Error {
   public:
    explicit FlowError(int iteration)
        : Error(CF_ENONFINITE, "mc_flow: non-finite value at iteration " +
                                   std::to_string(iteration)),
          iteration_(iteration) {}
    int iteration() const { return iteration_; }

   private:
    int iteration_;
};

namespace detail {
inline void check(int st, const char* what) {
    if (st != CF_OK) throw Error(st, what);
}
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, n ? n : 1), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};
}  // namespace detail

namespace cuda {

// Device-pointer entry points (stream-ordered; pointers owned by the caller).
namespace device {
inline void wmc_half_laplace(const float* in, float* out, int w, int h, cudaStream_t s = nullptr) {
    detail::check(cf_wmc_map_f32(in, out, w, h, w, 1, (int64_t)w * h, s), "wmc_half_laplace");
}
inline void mc_flow(float* img, int w, int h, const FlowConfig& cfg, void* workspace,
                    size_t workspace_bytes, cudaStream_t s = nullptr) {
    if (cfg.scheme != FlowConfig::Scheme::half_laplace)
        throw std::invalid_argument("scheme=fd is outside this build (DESIGN.md §9)");
    int32_t bad = 0;
    const int st = cf_wmc_filter_f32(img, w, h, w, 1, (int64_t)w * h, cfg.iters, (float)cfg.dt,
                                     workspace, workspace_bytes, &bad, s);
    if (st == CF_ENONFINITE) throw FlowError(bad);
    detail::check(st, "mc_flow");
}
inline size_t flow_workspace_bytes(int w, int h) {
    return cf_wmc_filter_workspace_bytes(w, h, w, 1, (int64_t)w * h);
}
}  // namespace device

// wmc_half_laplace(img) -> Image2D, host in / host out.
inline Image2D wmc_half_laplace(const Image2D& img, cudaStream_t s = nullptr) {
    Image2D out(img.width, img.height);
    const size_t n = img.data.size() * sizeof(float);
    detail::DevBuf din(n), dout(n);
    detail::cuda_check(cudaMemcpyAsync(din.p, img.data.data(), n, cudaMemcpyHostToDevice, s),
                       "H2D");
    device::wmc_half_laplace((const float*)din.p, (float*)dout.p, img.width, img.height, s);
    detail::cuda_check(cudaMemcpyAsync(out.data.data(), dout.p, n, cudaMemcpyDeviceToHost, s),
                       "D2H");
    detail::cuda_check(cudaStreamSynchronize(s), "sync");
    return out;
}

// mc_flow(img, cfg) -> Image2D (scheme = half_laplace).
inline Image2D mc_flow(const Image2D& img, const FlowConfig& cfg, cudaStream_t s = nullptr) {
    Image2D out = img;
    if (cfg.iters == 0) return out;
    const size_t n = img.data.size() * sizeof(float);
    detail::DevBuf dimg(n), ws(device::flow_workspace_bytes(img.width, img.height));
    detail::cuda_check(cudaMemcpyAsync(dimg.p, img.data.data(), n, cudaMemcpyHostToDevice, s),
                       "H2D");
    device::mc_flow((float*)dimg.p, img.width, img.height, cfg, ws.p,
                    device::flow_workspace_bytes(img.width, img.height), s);
    detail::cuda_check(cudaMemcpyAsync(out.data.data(), dimg.p, n, cudaMemcpyDeviceToHost, s),
                       "D2H");
    detail::cuda_check(cudaStreamSynchronize(s), "sync");
    return out;
}

// solve_l2_area / solve_l1_area, host in / host out;
// throws FlowError on divergence.
inline SolveReport solve(const Image2D& f, const SolverConfig& cfg, cudaStream_t s = nullptr) {
    const int w = f.width, h = f.height;
    const int64_t plane = (int64_t)w * h;
    const size_t n = f.data.size() * sizeof(float);
    const bool l1 = cfg.model == SolverConfig::Model::l1_area;
    const size_t wsb = l1 ? cf_wmc_solve_l1_area_workspace_bytes(w, h, w, 1, plane)
                          : cf_wmc_filter_workspace_bytes(w, h, w, 1, plane);
    detail::DevBuf df(n), du(n), dd(n), ws(wsb), red(cf_wmc_reduce_workspace_bytes(w, h, 1)),
        fid(sizeof(double));
    detail::cuda_check(cudaMemcpyAsync(df.p, f.data.data(), n, cudaMemcpyHostToDevice, s), "H2D");
    int32_t bad = 0;
    const int st =
        l1 ? cf_wmc_solve_l1_area_f32((const float*)df.p, (float*)du.p, (float*)dd.p, w, h, w, 1,
                                      plane, cfg.iters, (float)cfg.dt, (float)cfg.lambda,
                                      (float)cfg.alpha, 1, ws.p, wsb, &bad, s)
           : cf_wmc_solve_l2_area_f32((const float*)df.p, (float*)du.p, w, h, w, 1, plane,
                                      cfg.iters, (float)cfg.dt, (float)cfg.lambda, 1, ws.p, wsb,
                                      &bad, s);
    if (st == CF_ENONFINITE) throw FlowError(bad);
    detail::check(st, l1 ? "solve_l1_area" : "solve_l2_area");
    detail::check(cf_wmc_fidelity_f64((const float*)du.p, (const float*)df.p, w, h, w, 1, plane,
                                      l1 ? 1.0 : 2.0, (double*)fid.p, red.p,
                                      cf_wmc_reduce_workspace_bytes(w, h, 1), s),
                  "fidelity");
    SolveReport rep;
    rep.image = Image2D(w, h);
    rep.iters = cfg.iters;
    detail::cuda_check(cudaMemcpyAsync(rep.image.data.data(), du.p, n, cudaMemcpyDeviceToHost, s),
                       "D2H");
    if (l1) {
        rep.dual = Image2D(w, h);
        detail::cuda_check(
            cudaMemcpyAsync(rep.dual.data.data(), dd.p, n, cudaMemcpyDeviceToHost, s), "D2H");
    }
    double fv = 0.0;
    detail::cuda_check(cudaMemcpyAsync(&fv, fid.p, sizeof(double), cudaMemcpyDeviceToHost, s),
                       "D2H");
    detail::cuda_check(cudaStreamSynchronize(s), "sync");
    rep.fidelity = l1 ? fv : 0.5 * fv;
    return rep;
}
inline SolveReport solve_l2_area(const Image2D& f, SolverConfig cfg, cudaStream_t s = nullptr) {
    cfg.model = SolverConfig::Model::l2_area;
    return solve(f, cfg, s);
}
inline SolveReport solve_l1_area(const Image2D& f, SolverConfig cfg, cudaStream_t s = nullptr) {
    cfg.model = SolverConfig::Model::l1_area;
    return solve(f, cfg, s);
}

// mc_flow of one image split into `parts` row bands over `devices` (the
// reference's for_rows chunking; cf_wmc_filter_sharded_f32): host in / host
// out.  devices.empty(): every part on the current device.
inline Image2D mc_flow_sharded(const Image2D& img, const FlowConfig& cfg, int parts,
                               std::vector<int> devices = {}) {
    if (cfg.iters == 0) return img;
    const int w = img.width, h = img.height;
    int cur = 0;
    detail::cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
    if (devices.empty()) devices.assign(parts, cur);
    if ((int)devices.size() != parts) throw std::invalid_argument("one device per part");
    cf_shard_plan plan;
    detail::check(cf_shard_plan_init(h, w, parts, cf_wmc_filter_sweeps_per_launch(w, h, 1), &plan),
                  "cf_shard_plan_init");
    struct Part {
        int dev;
        void *a = nullptr, *b = nullptr, *flag = nullptr;
    };
    std::vector<Part> ps(parts);
    std::vector<float*> va(parts), vb(parts);
    std::vector<int32_t*> vf(parts);
    auto release = [&]() {
        for (auto& p : ps) {
            cudaSetDevice(p.dev);
            cudaFree(p.a);
            cudaFree(p.b);
            cudaFree(p.flag);
        }
        cudaSetDevice(cur);
    };
    try {
        for (int p = 0; p < parts; ++p) {
            ps[p].dev = devices[p];
            detail::cuda_check(cudaSetDevice(devices[p]), "cudaSetDevice");
            const size_t bytes = (size_t)plan.rows[p] * w * sizeof(float);
            detail::cuda_check(cudaMalloc(&ps[p].a, bytes), "cudaMalloc");
            detail::cuda_check(cudaMalloc(&ps[p].b, bytes), "cudaMalloc");
            detail::cuda_check(cudaMalloc(&ps[p].flag, 256), "cudaMalloc");
            const size_t own = (size_t)(plan.row1[p] - plan.row0[p]) * w;
            detail::cuda_check(
                cudaMemcpy((float*)ps[p].a + (size_t)plan.top[p] * w,
                           img.data.data() + (size_t)plan.row0[p] * w, own * sizeof(float),
                           cudaMemcpyHostToDevice),
                "H2D");
            va[p] = (float*)ps[p].a;
            vb[p] = (float*)ps[p].b;
            vf[p] = (int32_t*)ps[p].flag;
        }
        detail::cuda_check(cudaSetDevice(cur), "cudaSetDevice");
        int32_t bad = 0;
        const int st = cf_wmc_filter_sharded_f32(&plan, va.data(), vb.data(), vf.data(),
                                                 devices.data(), nullptr, cfg.iters,
                                                 (float)cfg.dt, &bad);
        if (st == CF_ENONFINITE) throw FlowError(bad);
        detail::check(st, "mc_flow_sharded");
        Image2D out(w, h);
        for (int p = 0; p < parts; ++p) {
            detail::cuda_check(cudaSetDevice(devices[p]), "cudaSetDevice");
            const size_t own = (size_t)(plan.row1[p] - plan.row0[p]) * w;
            detail::cuda_check(cudaMemcpy(out.data.data() + (size_t)plan.row0[p] * w,
                                          va[p] + (size_t)plan.top[p] * w, own * sizeof(float),
                                          cudaMemcpyDeviceToHost),
                               "D2H");
        }
        release();
        return out;
    } catch (...) {
        release();
        throw;
    }
}

// The reference's own fp64 arithmetic: wmc_half_laplace and
// mc_flow on fp64 images, BIT-identical to the reference CPU implementation.
namespace exact {
namespace device {
inline void wmc_half_laplace(const double* in, double* out, int w, int h,
                             cudaStream_t s = nullptr) {
    detail::check(cf_wmc_map_f64(in, out, w, h, w, 1, (int64_t)w * h, s), "wmc_half_laplace");
}
inline size_t flow_workspace_bytes(int w, int h) {
    return cf_wmc_filter_f64_workspace_bytes(w, h, w, 1, (int64_t)w * h);
}
inline void mc_flow(double* img, int w, int h, const FlowConfig& cfg, void* workspace,
                    size_t workspace_bytes, cudaStream_t s = nullptr) {
    if (cfg.scheme != FlowConfig::Scheme::half_laplace)
        throw std::invalid_argument("scheme=fd is outside this build (DESIGN.md §9)");
    int32_t bad = 0;
    const int st = cf_wmc_filter_f64(img, w, h, w, 1, (int64_t)w * h, cfg.iters, cfg.dt,
                                     workspace, workspace_bytes, &bad, s);
    if (st == CF_ENONFINITE) throw FlowError(bad);
    detail::check(st, "mc_flow");
}
}  // namespace device

inline Image2D64 wmc_half_laplace(const Image2D64& img, cudaStream_t s = nullptr) {
    Image2D64 out(img.width, img.height);
    const size_t n = img.data.size() * sizeof(double);
    detail::DevBuf din(n), dout(n);
    detail::cuda_check(cudaMemcpyAsync(din.p, img.data.data(), n, cudaMemcpyHostToDevice, s),
                       "H2D");
    device::wmc_half_laplace((const double*)din.p, (double*)dout.p, img.width, img.height, s);
    detail::cuda_check(cudaMemcpyAsync(out.data.data(), dout.p, n, cudaMemcpyDeviceToHost, s),
                       "D2H");
    detail::cuda_check(cudaStreamSynchronize(s), "sync");
    return out;
}

inline Image2D64 mc_flow(const Image2D64& img, const FlowConfig& cfg, cudaStream_t s = nullptr) {
    Image2D64 out = img;
    if (cfg.iters == 0) return out;
    const size_t n = img.data.size() * sizeof(double);
    const size_t wsb = device::flow_workspace_bytes(img.width, img.height);
    detail::DevBuf dimg(n), ws(wsb);
    detail::cuda_check(cudaMemcpyAsync(dimg.p, img.data.data(), n, cudaMemcpyHostToDevice, s),
                       "H2D");
    device::mc_flow((double*)dimg.p, img.width, img.height, cfg, ws.p, wsb, s);
    detail::cuda_check(cudaMemcpyAsync(out.data.data(), dimg.p, n, cudaMemcpyDeviceToHost, s),
                       "D2H");
    detail::cuda_check(cudaStreamSynchronize(s), "sync");
    return out;
}
}  // namespace exact

// Per-channel processing: planes are independent.
inline std::vector<Image2D> mc_flow(const std::vector<Image2D>& channels, const FlowConfig& cfg) {
    if (channels.size() != 1 && channels.size() != 3)
        throw std::invalid_argument("unsupported channel count (SPEC.md:65)");
    std::vector<Image2D> out;
    for (const auto& c : channels) out.push_back(mc_flow(c, cfg));
    return out;
}

}  // namespace cuda
}  // namespace curveflow
