// paper_1903_07189_b200/csrc/wmc_shard.cpp -- single-process sharded WMC
// filter over P device buffers (SURVEY.md §8b export 4).
//
// Row bands follow the reference's parallel::for_rows chunking
// (proj/include/curveflow/parallel.hpp:36-44: chunk = ceil(h / P), part p
// owns [p*chunk, min(h, (p+1)*chunk))).  Per launch of kk fused sweeps:
//   1. every part records "iterate ready" on its stream;
//   2. every part waits for its neighbours' "ready" and pulls their kk
//      boundary rows into its own halo (cudaMemcpyPeerAsync: NVLink P2P
//      between GPUs, a device copy when parts share one), then records
//      "copied";
//   3. every part waits for its neighbours' "copied" (they read the buffer
//      this launch overwrites) and runs the row-band kernel
//      (cf_wmc_sweeps_band_f32) from its buffer to the other one.
// Jacobi semantics make the result bit-identical to the single-buffer
// filter for any P.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "../../include/curveflow/capi.h"

extern "C" void cf_internal_set_cuda_error(int e);
extern "C" int cf_internal_schedule(int32_t iters, int32_t levels, int32_t* out, int32_t cap);

namespace {

struct DeviceGuard {  // restores the caller's current device
    int dev = 0;
    bool ok = false;
    DeviceGuard() { ok = cudaGetDevice(&dev) == cudaSuccess; }
    ~DeviceGuard() {
        if (ok) cudaSetDevice(dev);
    }
};

int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return CF_OK;
    cf_internal_set_cuda_error((int)e);
    return CF_ECUDA;
}

#define SH_CUDA(x)                                \
    do {                                          \
        const int rc_ = cuda_status(x);           \
        if (rc_ != CF_OK) return rc_;             \
    } while (0)

// Per part: ready / copied.  Destroyed on scope exit; CUDA releases an event
// whose last record is still pending once the device completes it.
struct Events {
    std::vector<cudaEvent_t> ready, copied;
    std::vector<int> dev;
    ~Events() {
        for (size_t i = 0; i < ready.size(); ++i) {
            cudaSetDevice(dev[i]);
            if (ready[i]) cudaEventDestroy(ready[i]);
            if (copied[i]) cudaEventDestroy(copied[i]);
        }
    }
};

}  // namespace

extern "C" {

CF_API int cf_shard_plan_init(int32_t h, int32_t w, int32_t parts, int32_t k,
                              cf_shard_plan* plan) {
    if (!plan || h <= 0 || w <= 0 || parts < 1 || parts > CF_MAX_PARTS || parts > h) return CF_EINVAL;
    if (k < 1 || k > cf_wmc_max_sweeps_per_launch()) return CF_EINVAL;
    const int32_t chunk = (h + parts - 1) / parts;  // parallel.hpp:36
    if ((int64_t)chunk * (parts - 1) >= h) return CF_EINVAL;  // a part would own no rows
    *plan = cf_shard_plan{};
    plan->h = h;
    plan->w = w;
    plan->parts = parts;
    plan->k = k;
    for (int p = 0; p < parts; ++p) {
        plan->row0[p] = p * chunk;
        plan->row1[p] = std::min(h, (p + 1) * chunk);
        plan->top[p] = p > 0 ? k : 0;
        plan->bot[p] = p < parts - 1 ? k : 0;
        const int own = plan->row1[p] - plan->row0[p];
        if (parts > 1 && own < k) return CF_EINVAL;  // halos come from the adjacent part only
        plan->rows[p] = plan->top[p] + own + plan->bot[p];
    }
    return CF_OK;
}

CF_API int cf_wmc_filter_sharded_f32(const cf_shard_plan* plan, float* const* bufs_a,
                                     float* const* bufs_b, int32_t* const* flags,
                                     const int32_t* devices, void* const* streams, int32_t iters,
                                     float dt, int32_t* first_bad_iter) {
    if (!plan || !bufs_a || !bufs_b || !flags || !devices || iters < 0) return CF_EINVAL;
    const int P = plan->parts;
    if (P < 1 || P > CF_MAX_PARTS || plan->k < 1) return CF_EINVAL;
    if (!(dt > 0.0f) || dt > 1.0f) return CF_EINVAL;
    for (int p = 0; p < P; ++p)
        if (!bufs_a[p] || !bufs_b[p] || !flags[p] || bufs_a[p] == bufs_b[p]) return CF_EINVAL;
    if (first_bad_iter) *first_bad_iter = 0;
    if (iters == 0) return CF_OK;
    std::vector<int32_t> ks(2 * iters + 2);
    const int n = cf_internal_schedule(iters, plan->k, ks.data(), (int32_t)ks.size());
    if (n <= 0) return CF_EINVAL;
    const int64_t w = plan->w;
    auto stream = [&](int p) { return streams ? (cudaStream_t)streams[p] : (cudaStream_t)0; };

    DeviceGuard guard;
    Events ev;
    ev.ready.assign(P, nullptr);
    ev.copied.assign(P, nullptr);
    ev.dev.assign(devices, devices + P);
    for (int p = 0; p < P; ++p) {
        SH_CUDA(cudaSetDevice(devices[p]));
        SH_CUDA(cudaEventCreateWithFlags(&ev.ready[p], cudaEventDisableTiming));
        SH_CUDA(cudaEventCreateWithFlags(&ev.copied[p], cudaEventDisableTiming));
        for (int q : {p - 1, p + 1}) {  // P2P over NVLink where the topology has it
            if (q < 0 || q >= P || devices[q] == devices[p]) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, devices[p], devices[q]) == cudaSuccess && can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else SH_CUDA(e);
            }
        }
        SH_CUDA(cudaMemsetAsync(flags[p], 0x7f, sizeof(int32_t), stream(p)));
        SH_CUDA(cudaEventRecord(ev.copied[p], stream(p)));
    }
    std::vector<float*> cur(bufs_a, bufs_a + P), nxt(bufs_b, bufs_b + P);
    int iter = 0;
    for (int i = 0; i < n; ++i) {
        const int kk = ks[i];
        for (int p = 0; p < P; ++p) {  // 1. this part's iterate is complete
            SH_CUDA(cudaSetDevice(devices[p]));
            SH_CUDA(cudaEventRecord(ev.ready[p], stream(p)));
        }
        for (int p = 0; p < P; ++p) {  // 2. pull the neighbours' boundary rows
            if (P == 1) break;
            SH_CUDA(cudaSetDevice(devices[p]));
            const int own = plan->row1[p] - plan->row0[p];
            if (p > 0) {
                const int q = p - 1, own_q = plan->row1[q] - plan->row0[q];
                SH_CUDA(cudaStreamWaitEvent(stream(p), ev.ready[q], 0));
                SH_CUDA(cudaMemcpyPeerAsync(cur[p] + (plan->top[p] - kk) * w, devices[p],
                                            cur[q] + (plan->top[q] + own_q - kk) * w, devices[q],
                                            sizeof(float) * kk * w, stream(p)));
            }
            if (p < P - 1) {
                const int q = p + 1;
                SH_CUDA(cudaStreamWaitEvent(stream(p), ev.ready[q], 0));
                SH_CUDA(cudaMemcpyPeerAsync(cur[p] + (plan->top[p] + own) * w, devices[p],
                                            cur[q] + plan->top[q] * w, devices[q],
                                            sizeof(float) * kk * w, stream(p)));
            }
            SH_CUDA(cudaEventRecord(ev.copied[p], stream(p)));
        }
        for (int p = 0; p < P; ++p) {  // 3. advance the band (writes nxt[p])
            SH_CUDA(cudaSetDevice(devices[p]));
            for (int q : {p - 1, p + 1})  // neighbours have read what nxt[p] held
                if (q >= 0 && q < P) SH_CUDA(cudaStreamWaitEvent(stream(p), ev.copied[q], 0));
            const int32_t buf_row0 = plan->row0[p] - plan->top[p];
            const int rc = cf_wmc_sweeps_band_f32(cur[p], buf_row0, plan->rows[p], nxt[p], buf_row0,
                                                  plan->w, plan->h, plan->w, plan->row0[p],
                                                  plan->row1[p], kk, dt, iter, flags[p], stream(p));
            if (rc) return rc;
        }
        iter += kk;
        std::swap(cur, nxt);
    }
    if (cur[0] != bufs_a[0]) {  // iters == 1: one launch wrote bufs_b
        for (int p = 0; p < P; ++p) {
            SH_CUDA(cudaSetDevice(devices[p]));
            SH_CUDA(cudaMemcpyAsync(bufs_a[p] + plan->top[p] * w, cur[p] + plan->top[p] * w,
                                    sizeof(float) * (plan->row1[p] - plan->row0[p]) * w,
                                    cudaMemcpyDeviceToDevice, stream(p)));
        }
    }
    if (!first_bad_iter) return CF_OK;
    int32_t bad = 0x7fffffff;
    for (int p = 0; p < P; ++p) {
        SH_CUDA(cudaSetDevice(devices[p]));
        int32_t host = 0x7f7f7f7f;
        SH_CUDA(cudaMemcpyAsync(&host, flags[p], sizeof(int32_t), cudaMemcpyDeviceToHost, stream(p)));
        SH_CUDA(cudaStreamSynchronize(stream(p)));
        if (host > 0 && host < 0x7f7f7f7f) bad = std::min(bad, host);
    }
    if (bad != 0x7fffffff) {
        *first_bad_iter = bad;
        return CF_ENONFINITE;
    }
    return CF_OK;
}

}  // extern "C"
