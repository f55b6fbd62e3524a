// paper_1903_07189_b200/csrc/wmc_capi.cu -- host side of the C-ABI
// (include/curveflow/capi.h): validation, launch planning, ping-pong
// scheduling of the temporally blocked flow, non-finite flag plumbing.
//
// Reference interfaces replaced (the SPEC operations on the path; the
// reference ships no code for them): wmc_half_laplace SPEC.md:171-179,
// mc_flow(scheme=half_laplace) SPEC.md:256-272.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <tuple>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/curveflow/capi.h"
#include "wmc_map.cuh"

namespace {

constexpr int kMaxLevels = 4;            // max sweeps fused per launch (band API)
// Sweeps per launch the filter schedules (measured on B200):
// K = 2 wins or ties K = 3 on every BASELINE config and 9 of 10 probed
// geometries (tools/probe_geometry.py) since border warps take the fast
// path; CF_FLOW_LEVELS overrides it for experiments.
#ifndef CF_FLOW_LEVELS
#define CF_FLOW_LEVELS 2
#endif
constexpr int kFlowLevels = CF_FLOW_LEVELS;
#ifndef CF_FLAT_MAP_PIXELS
#define CF_FLAT_MAP_PIXELS (1 << 19)  // measured crossover: +23 % at 512^2, equal at 1024^2
#endif
constexpr int64_t kFlatMapPixels = CF_FLAT_MAP_PIXELS;  // maps up to this size: flat kernel
#ifndef CF_BORDER_SPLIT
#define CF_BORDER_SPLIT 2
#endif
constexpr int kBorderSplit = CF_BORDER_SPLIT;  // border-pair strips are this much shorter
constexpr int kBorderSplitMinRows = 32;         // ... when interior strips are this long
constexpr size_t kWsHeader = 256;        // workspace: [flag | pad] then image
constexpr int32_t kFlagNone = 0x7f7f7f7f;  // memset(0x7f) pattern

thread_local int g_last_cuda = 0;

int cuda_fail(cudaError_t e) {
    g_last_cuda = (int)e;
    return CF_ECUDA;
}
#define CF_CUDA(x)                                  \
    do {                                            \
        cudaError_t e_ = (x);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_); \
    } while (0)

struct DevInfo {
    int sms = 0;
    int cc_major = 0, cc_minor = 0;
};

std::mutex g_dev_mu;
std::vector<DevInfo> g_dev;

int device_info(DevInfo* out) {
    int dev = 0;
    CF_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
    DevInfo& d = g_dev[dev];
    if (d.sms == 0) {
        CF_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
        CF_CUDA(cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev));
        CF_CUDA(cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
    }
    if (d.cc_major != 10 || d.cc_minor != 0) return CF_ENODEV;
    *out = d;
    return CF_OK;
}

template <int K, int MODE>
constexpr size_t smem_bytes() {
    return (size_t)cfk::kWarpsPerBlock * cfk::smem_bytes_per_warp<K, MODE>();
}

template <int K, int MODE>
int kernel_occupancy_warps() {
    // per instantiation; identical on every B200.  Atomic: first calls may
    // come from several host threads at once (the ABI is re-entrant); they
    // compute the same value.
    static std::atomic<int> cached{-1};
    int v = cached.load(std::memory_order_acquire);
    if (v < 0) {
        if (smem_bytes<K, MODE>() > 48 * 1024)
            cudaFuncSetAttribute(cfk::wmc_sweeps_kernel<K, MODE>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<K, MODE>());
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &blocks, cfk::wmc_sweeps_kernel<K, MODE>, cfk::kThreads, smem_bytes<K, MODE>()) !=
                cudaSuccess ||
            blocks <= 0)
            blocks = 2;
        v = blocks * cfk::kWarpsPerBlock;
        cached.store(v, std::memory_order_release);
    }
    return v;
}

// Strip planner: choose rows per warp-task so that the number of waves times
// the per-task length (rows + temporal warm-up + fixed cost) is minimal.
// Border pairs' strip height: kBorderSplit x shorter for long strips (there
// they were the launch's tail); short strips (latency-bound small images)
// keep the interior height -- extra warps cost more than the tail there.
int border_strip_rows(int sr) {
    return sr >= kBorderSplitMinRows ? (sr + kBorderSplit - 1) / kBorderSplit : sr;
}

void plan_strips(cfk::SweepParams& p, int K, int slots) {
    const int rows = p.y1 - p.y0;
    const int64_t n_pairs = (p.n_chunks + 1) / 2;
    const int64_t nb = std::min<int64_t>(n_pairs, 1 + p.n_bhi), ni = n_pairs - nb;
#ifndef CF_PLAN_OVH
#define CF_PLAN_OVH 3.0  // measured: 1-4 rows +0.6 % on cfg4 over 6, cfg3 unchanged, 1 row -11 % on cfg3
#endif
    const double overhead = (K - 1) + CF_PLAN_OVH;  // warm-up rows + fixed per-task cost (rows)
#ifndef CF_MIN_STRIP
#define CF_MIN_STRIP 8   // output rows per strip at least max(CF_MIN_STRIP, CF_MIN_STRIP_K * K)
#endif
#ifndef CF_MIN_STRIP_K
#define CF_MIN_STRIP_K 4
#endif
    const int max_strips = std::max(1, rows / std::max(CF_MIN_STRIP, CF_MIN_STRIP_K * K));
    double best_cost = 1e300;
    int best = 1;
    for (int ns = 1; ns <= max_strips; ++ns) {
        const int sr = (rows + ns - 1) / ns;
        const int ns_eff = (rows + sr - 1) / sr;
        const int sr_b = border_strip_rows(sr);
        const int ns_b = (rows + sr_b - 1) / sr_b;
        // all tasks, border ones included (kBorderSplit x more, shorter)
        const int64_t tasks = (ni * ns_eff + nb * ns_b) * p.planes;
        const int64_t waves = (tasks + slots - 1) / slots;
        const double cost = (double)waves * (sr + overhead);
        if (cost < best_cost * 0.999) { best_cost = cost; best = ns; }
        if (tasks > (int64_t)slots * 64) break;
    }
#ifdef CF_FORCE_NS  // experiments: a fixed number of strips
    best = CF_FORCE_NS;
#endif
    p.strip_rows = (rows + best - 1) / best;
    p.n_strips = (rows + p.strip_rows - 1) / p.strip_rows;
    p.strip_rows_b = border_strip_rows(p.strip_rows);
    p.n_strips_b = (rows + p.strip_rows_b - 1) / p.strip_rows_b;
}

template <int K, int MODE>
int launch_k(cfk::SweepParams p, const DevInfo& d, cudaStream_t s) {
    using G = cfk::Geo<K>;
    p.n_chunks = (p.w + G::S - 1) / G::S;
    {  // trailing chunk pairs whose window leaves the image (kernel task order)
        const int n_pairs = (p.n_chunks + 1) / 2;
        int nbh = 0;
        for (int pp = n_pairs - 1; pp >= 1; --pp) {
            bool b = false;
            for (int h = 0; h < 2; ++h) {
                const int c = 2 * pp + h;
                if (c >= p.n_chunks || c * G::S - G::A + cfk::kChunk > p.w) b = true;
            }
            if (!b) break;
            ++nbh;
        }
        p.n_bhi = nbh;
    }
    plan_strips(p, K, d.sms * kernel_occupancy_warps<K, MODE>());
    const int64_t n_pairs = (p.n_chunks + 1) / 2;
    const int64_t nb = std::min<int64_t>(n_pairs, 1 + p.n_bhi);
    const int64_t tasks = (nb * p.n_strips_b + (n_pairs - nb) * p.n_strips) * p.planes;
    const int64_t blocks = (tasks + cfk::kWarpsPerBlock - 1) / cfk::kWarpsPerBlock;
    if (blocks > INT_MAX) return CF_EINVAL;
    cfk::wmc_sweeps_kernel<K, MODE><<<(unsigned)blocks, cfk::kThreads, smem_bytes<K, MODE>(), s>>>(p);
    CF_CUDA(cudaGetLastError());
    return CF_OK;
}

template <int MODE>
int launch(const cfk::SweepParams& p, int K, const DevInfo& d, cudaStream_t s) {
    switch (K) {
        case 1: return launch_k<1, MODE>(p, d, s);
        case 2: return launch_k<2, MODE>(p, d, s);
        case 3: return launch_k<3, MODE>(p, d, s);
        case 4: return launch_k<4, MODE>(p, d, s);
        default: return CF_EINVAL;
    }
}


// The streaming map (csrc/wmc_map.cuh): one warp per 256 columns x strip;
// strips sized so waves x (rows + warm-up) is minimal over the resident slots.
int launch_map(const float* in, float* out, int32_t w, int32_t h, int64_t pitch, int32_t planes,
               int64_t plane_stride, const DevInfo& d, cudaStream_t s,
               double* seg_sums = nullptr, double q = 1.0, int qkind = 1) {
    constexpr size_t smem = (size_t)cfk::kMapWarps * cfk::kMapRing * cfk::kMapRowBytes;
    // 0: plain map; 1..4: the fused energy epilogue for q = 1, 2, 0.5, other
    const int qk = seg_sums == nullptr ? 0 : (qkind >= 1 && qkind <= 3 ? qkind : 4);
    void (*const kerns[5])(cfk::MapParams) = {cfk::wmc_map_kernel<0>, cfk::wmc_map_kernel<1>,
                                              cfk::wmc_map_kernel<2>, cfk::wmc_map_kernel<3>,
                                              cfk::wmc_map_kernel<4>};
    auto kern = kerns[qk];
    static std::atomic<int> occ_cache[5] = {-1, -1, -1, -1, -1};  // warps per SM (every B200)
    std::atomic<int>& occ = occ_cache[qk];
    int warps = occ.load(std::memory_order_acquire);
    if (warps < 0) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern,
                                                          32 * cfk::kMapWarps, smem) != cudaSuccess ||
            blocks <= 0)
            blocks = 2;
        warps = blocks * cfk::kMapWarps;
        occ.store(warps, std::memory_order_release);
    }
    cfk::MapParams p{};
    p.src = in; p.dst = out;
    p.src_pitch = p.dst_pitch = pitch;
    p.src_plane = p.dst_plane = plane_stride;
    p.w = w; p.h = h; p.planes = planes;
    p.seg_sums = seg_sums; p.q = q; p.qkind = qkind;
    p.n_pairs = (w + 2 * cfk::kMapChunk - 1) / (2 * cfk::kMapChunk);
    // 16-byte (4 columns a lane) or 8-byte (2) output stores need aligned rows
    constexpr int kAl = cfk::kMapCols;  // elements
    p.st128 = ((reinterpret_cast<uintptr_t>(out) & (4 * kAl - 1)) == 0 && (pitch % kAl) == 0 &&
               (planes == 1 || (plane_stride % kAl) == 0)) ? 1 : 0;
    const int64_t slots = (int64_t)d.sms * warps;
    const int64_t cols = (int64_t)p.n_pairs * planes;
    double best_cost = 1e300;
    int best = 1;
    const int max_strips = std::max(1, h / 8);
    for (int ns = 1; ns <= max_strips; ++ns) {
        const int sr = (h + ns - 1) / ns;
        const int64_t tasks = cols * ((h + sr - 1) / sr);
        const int64_t waves = (tasks + slots - 1) / slots;
        const double cost = (double)waves * (sr + 8.0);  // + warm-up / fixed cost (rows)
        if (cost < best_cost * 0.999) { best_cost = cost; best = ns; }
        if (tasks > slots * 32) break;
    }
#ifndef CF_MAP_TAIL_MODEL
#define CF_MAP_TAIL_MODEL 1
#endif
    // Images that need several waves: the block scheduler balances many
    // short tasks better than a few whole waves of long ones, so cost the
    // work spread over the slots plus one task of tail instead (16384^2:
    // 55 strips of 298 rows in 2 waves -> ~240 of 69 rows, 0.565 -> 0.547
    // ms; one-wave images keep the wave count, where it measured better).
    const int sr_w = (h + best - 1) / best;  // the wave model's choice
    if (CF_MAP_TAIL_MODEL && cols * ((h + sr_w - 1) / sr_w) > slots) {
        best_cost = 1e300;
        for (int ns = 1; ns <= max_strips; ++ns) {
            const int sr = (h + ns - 1) / ns;
            const int64_t tasks = cols * ((h + sr - 1) / sr);
#ifndef CF_MAP_TAIL_OVH
#define CF_MAP_TAIL_OVH 8.0
#endif
            const double cost = ((double)tasks / (double)slots + 1.0) * (sr + CF_MAP_TAIL_OVH);
            if (cost < best_cost * 0.999) { best_cost = cost; best = ns; }
            if (tasks > slots * 32) break;
        }
    }
#ifdef CF_MAP_FORCE_NS  // experiments: a fixed number of strips
    best = std::min(CF_MAP_FORCE_NS, h);
#endif
    p.strip_rows = (h + best - 1) / best;
    p.n_strips = (h + p.strip_rows - 1) / p.strip_rows;
    const int64_t tasks = cols * p.n_strips;
    const int64_t blocks = (tasks + cfk::kMapWarps - 1) / cfk::kMapWarps;
    if (blocks > INT_MAX) return CF_EINVAL;
    kern<<<(unsigned)blocks, 32 * cfk::kMapWarps, smem, s>>>(p);
    CF_CUDA(cudaGetLastError());
    return CF_OK;
}

bool shape_ok(int32_t w, int32_t h, int64_t pitch, int32_t planes, int64_t plane_stride) {
    if (w <= 0 || h <= 0 || planes <= 0 || pitch < w) return false;
    if (planes > 1 && plane_stride < pitch * (int64_t)h) return false;
    if ((int64_t)w > (1 << 30) || (int64_t)h > (1 << 30)) return false;
    return true;
}

int flow_levels(int32_t, int32_t, int32_t) { return kFlowLevels; }

// Launch schedule: sweeps per launch, at most `levels` each, an EVEN number
// of launches when iters >= 2 (unless levels == 1 and iters is odd) so the
// ping-pong ends in the caller's buffer:
// n = the smallest even count >= ceil(iters / levels), sweeps spread evenly
// (200 at 3 levels -> 64 x 3 + 4 x 2: no single-sweep launch, each of which
// would cost a full HBM pass).
std::vector<int> schedule(int iters, int levels) {
    if (iters <= 0) return {};
    if (iters == 1) return {1};
    int n = (iters + levels - 1) / levels;
    n += n & 1;
    n = std::min(n, iters);  // levels == 1, odd iters: odd count, callers copy back
    std::vector<int> ks(n, iters / n);
    for (int i = 0; i < iters % n; ++i) ks[i] += 1;
    return ks;
}

__global__ void u8_to_f32_kernel(const uint8_t* in, int64_t in_pitch, int64_t in_plane, float* out,
                                 int64_t pitch, int64_t plane, int32_t w, int32_t h,
                                 int32_t planes) {
    // one row per block iteration (a single index division per row); rows
    // whose source is 4-byte and destination 16-byte aligned move 4 pixels
    // per thread (one 32-bit load, one 128-bit store), others 1
    const int64_t rows = (int64_t)h * planes;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int64_t p = r / h, y = r - p * h;
        const uint8_t* src = in + p * in_plane + y * in_pitch;
        float* dst = out + p * plane + y * pitch;
        int x0 = 0;
        if ((reinterpret_cast<uintptr_t>(src) & 3) == 0 &&
            (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            const int n4 = w >> 2;
            const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
            float4* d4 = reinterpret_cast<float4*>(dst);
            for (int i = threadIdx.x; i < n4; i += blockDim.x) {
                const uint32_t v = __ldg(s4 + i);
                d4[i] = make_float4(cfk::widen_u8(v & 0xffu), cfk::widen_u8((v >> 8) & 0xffu),
                                    cfk::widen_u8((v >> 16) & 0xffu), cfk::widen_u8(v >> 24));
            }
            x0 = n4 << 2;
        }
        for (int x = x0 + threadIdx.x; x < w; x += blockDim.x) dst[x] = cfk::widen_u8(src[x]);
    }
}

__device__ __forceinline__ float4 widen4(uint32_t v) {
    return make_float4(cfk::widen_u8(v & 0xffu), cfk::widen_u8((v >> 8) & 0xffu),
                       cfk::widen_u8((v >> 16) & 0xffu), cfk::widen_u8(v >> 24));
}

__global__ void u8_to_f32_dense_kernel(const uint32_t* in, float4* out, int64_t n4) {
    // dense planes (pitch w, plane stride h*w): the batch is one flat array
    // of 4-pixel words.  Consecutive threads take consecutive words, so every
    // warp load is 128 contiguous bytes and every float4 store 512; four
    // words per thread (grid-stride apart) are loaded before any is stored.
    const int64_t S = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * S < n4; i += 4 * S) {
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldg(in + i + k * S);
#pragma unroll
        for (int k = 0; k < 4; ++k) out[i + k * S] = widen4(v[k]);
    }
    for (; i < n4; i += S) out[i] = widen4(__ldg(in + i));
}

// u8 -> fp32 widening of a plane batch, flat when dense.
int launch_widen(const uint8_t* in, int64_t in_pitch, int64_t in_plane, float* out, int64_t pitch,
                 int64_t plane, int32_t w, int32_t h, int32_t planes, int sms, cudaStream_t s) {
    const int64_t hw = (int64_t)h * w, n = hw * planes;
    const bool dense = in_pitch == w && pitch == w && (planes == 1 || (in_plane == hw && plane == hw));
    if (dense && (reinterpret_cast<uintptr_t>(in) & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(out) & 15) == 0 && n >= 4) {
        const int64_t n4 = n / 4;
        const int64_t blocks = std::min<int64_t>((n4 + 255) / 256, (int64_t)sms * 8);
        u8_to_f32_dense_kernel<<<(unsigned)blocks, 256, 0, s>>>(
            reinterpret_cast<const uint32_t*>(in), reinterpret_cast<float4*>(out), n4);
        CF_CUDA(cudaGetLastError());
        if (n4 * 4 == n) return CF_OK;
        // tail (< 4 pixels, contiguous: may span rows when w < 4): one
        // "row" of n - done pixels through the row kernel
        const int64_t done = n4 * 4;
        u8_to_f32_kernel<<<1, 256, 0, s>>>(in + done, 0, 0, out + done, 0, 0,
                                           (int32_t)(n - done), 1, 1);
        CF_CUDA(cudaGetLastError());
        return CF_OK;
    }
    u8_to_f32_kernel<<<sms * 16, 256, 0, s>>>(in, in_pitch, in_plane, out, pitch, plane, w, h,
                                           planes);
    CF_CUDA(cudaGetLastError());
    return CF_OK;
}

// ---- launch-graph cache -----------------------------------------------------
// A run is tens to hundreds of dependent launches; on small (L2-resident)
// images each is ~10 us and the stream's launch-to-launch gap costs ~18 %
// (1024^2, 100 iterations).  A call repeated with identical arguments (a
// frame loop over fixed buffers) is captured once into a CUDA graph on an
// internal capture stream and replayed on the caller's stream from then on.
// The graph is built on the SECOND identical call, so one-off calls never pay
// the instantiation.  Callers that are themselves capturing get the plain
// launches (their graph already holds them).  CF_GRAPHS=0 disables the cache.
struct FlowKey {
    int dev;
    const void* src0; bool src_u8; int64_t src_pitch, src_plane;
    float* out; int32_t w, h; int64_t pitch; int32_t planes; int64_t plane_stride;
    int32_t iters; uint32_t dt; void* ws;
    const float* f; uint32_t lambda; float* d; float* d_ws; uint32_t alpha;
    uint8_t* o8; int64_t o8_pitch, o8_plane;
    int32_t src_px, o8_px;
    // field-by-field bytes (no padding): the cache's key
    std::string bytes() const {
        std::string k;
        auto put = [&k](const auto& v) { k.append(reinterpret_cast<const char*>(&v), sizeof(v)); };
        put('F'); put(src0); put(src_u8); put(src_pitch); put(src_plane); put(out); put(w);
        put(h); put(pitch); put(planes); put(plane_stride); put(iters); put(dt); put(ws); put(f);
        put(lambda); put(d); put(d_ws); put(alpha); put(o8); put(o8_pitch); put(o8_plane);
        put(src_px); put(o8_px);
        return k;
    }
};

struct GraphEntry {
    int dev = 0;
    std::string key;                 // argument bytes of the run (per entry point family)
    cudaGraphExec_t exec = nullptr;  // null: seen once, not captured yet
    bool no_graph = false;           // capture failed once: plain launches for this key
    uint64_t last_use = 0;
};

constexpr size_t kGraphCap = 32;
std::mutex g_graph_mu;
std::vector<GraphEntry> g_graphs;
uint64_t g_graph_clock = 0;
std::vector<cudaStream_t> g_capture_streams;  // one per device, created on demand

bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CF_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}

uint32_t f32_bits(float v) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    return b;
}

// Runs `enqueue` directly or through a cached graph.  g_graph_mu covers the
// lookup, the capture (once per key: the capture stream is shared per device)
// and cudaGraphLaunch (an exec must not be evicted mid-launch); a key's
// first, plain run happens outside it.
template <typename Fn>
int run_cached(int dev, const std::string& key, cudaStream_t s, Fn&& enqueue) {
    if (!graphs_enabled()) return enqueue(s);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
        (void)cudaGetLastError();
        return enqueue(s);
    }
    if (cs != cudaStreamCaptureStatusNone) return enqueue(s);
    std::unique_lock<std::mutex> lk(g_graph_mu);
    const uint64_t now = ++g_graph_clock;
    GraphEntry* hit = nullptr;
    for (GraphEntry& e : g_graphs)
        if (e.dev == dev && e.key == key) { hit = &e; break; }
    if (!hit) {  // first sighting: remember the key, launch directly
        if (g_graphs.size() >= kGraphCap) {
            auto lru = std::min_element(g_graphs.begin(), g_graphs.end(),
                                        [](const GraphEntry& a, const GraphEntry& b) {
                                            return a.last_use < b.last_use;
                                        });
            if (lru->exec) cudaGraphExecDestroy(lru->exec);  // freed after in-flight runs
            g_graphs.erase(lru);
        }
        GraphEntry e;
        e.dev = dev;
        e.key = key;
        e.last_use = now;
        g_graphs.push_back(e);
        lk.unlock();  // plain launches need no lock (other threads keep going)
        return enqueue(s);
    }
    hit->last_use = now;
    if (hit->no_graph) {
        lk.unlock();
        return enqueue(s);
    }
    if (!hit->exec) {  // second sighting: capture on the device's capture stream
        if ((int)g_capture_streams.size() <= dev) g_capture_streams.resize(dev + 1, nullptr);
        cudaStream_t& cap = g_capture_streams[dev];
        bool ok = cap || cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess;
        if (ok && cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            const int rc = enqueue(cap);
            cudaGraph_t g = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(cap, &g);
            ok = !rc && ec == cudaSuccess && g &&
                 cudaGraphInstantiate(&hit->exec, g, 0) == cudaSuccess;
            if (g) cudaGraphDestroy(g);
        } else {
            ok = false;
        }
        if (!ok) {  // capture refused or failed: plain launches for this key from now
            hit->exec = nullptr;  // on (a genuine argument error recurs there and is returned)
            hit->no_graph = true;
            (void)cudaGetLastError();
            lk.unlock();
            return enqueue(s);
        }
    }
    if (cudaGraphLaunch(hit->exec, s) != cudaSuccess) {
        // e.g. the exec was invalidated (device reset): drop it, run plain launches
        (void)cudaGetLastError();
        cudaGraphExecDestroy(hit->exec);
        hit->exec = nullptr;
        hit->no_graph = true;
        lk.unlock();
        return enqueue(s);
    }
    return CF_OK;
}

}  // namespace

// The WMC energy's segment sums computed in the streaming map kernel's
// epilogue, without storing the map (wmc_reduce.cu).  CF_EINVAL when the
// image is small enough for the flat map kernel (the caller then reduces a
// stored map).  seg_sums: [ceil(w / 256)][planes * h].
extern "C" int cf_internal_map_energy_segs(const float* in, int32_t w, int32_t h, int64_t pitch,
                                           int32_t planes, int64_t plane_stride, double q,
                                           int32_t qkind, double* seg_sums, void* stream) {
    if (cfk::kMapCols != 4 || (int64_t)w * h * planes <= kFlatMapPixels) return CF_EINVAL;
    DevInfo d;
    if (int rc = device_info(&d)) return rc;
    return launch_map(in, nullptr, w, h, pitch, planes, plane_stride, d, (cudaStream_t)stream,
                      seg_sums, q, qkind);
}

// Shared with wmc_io.cu / wmc_shard.cpp; hidden (not part of the C-ABI).
extern "C" void cf_internal_set_cuda_error(int e) { g_last_cuda = e; }
// The same cache for the other entry-point families (wmc_f64.cu): `key` is
// the caller's argument bytes (padding-free), `enqueue(ctx, stream)` the run.
extern "C" int cf_internal_graph_run(const void* key, size_t key_len, void* stream,
                                     int (*enqueue)(void* ctx, void* stream), void* ctx) {
    int dev = 0;
    CF_CUDA(cudaGetDevice(&dev));
    return run_cached(dev, std::string(static_cast<const char*>(key), key_len),
                      (cudaStream_t)stream,
                      [&](cudaStream_t st) { return enqueue(ctx, (void*)st); });
}
extern "C" int cf_internal_schedule(int32_t iters, int32_t levels, int32_t* out, int32_t cap) {
    const std::vector<int> ks = schedule(iters, levels);
    if ((int32_t)ks.size() > cap) return -1;
    for (size_t i = 0; i < ks.size(); ++i) out[i] = ks[i];
    return (int32_t)ks.size();
}

extern "C" {

CF_API const char* cf_version(void) { return "curveflow-b200 0.1.0 (sm_100a)"; }

CF_API const char* cf_status_string(int status) {
    switch (status) {
        case CF_OK: return "ok";
        case CF_EINVAL: return "invalid argument (shape, pitch, planes, iters, dt or workspace)";
        case CF_ECUDA: return "CUDA runtime error";
        case CF_ENONFINITE: return "non-finite value produced (instability)";
        case CF_ENODEV: return "no sm_100 (B200) device";
        default: return "unknown status";
    }
}

CF_API int cf_last_cuda_error(void) { return g_last_cuda; }

CF_API int32_t cf_wmc_max_sweeps_per_launch(void) { return kMaxLevels; }

CF_API int32_t cf_wmc_filter_sweeps_per_launch(int32_t w, int32_t h, int32_t planes) {
    if (w <= 0 || h <= 0 || planes <= 0) return 0;
    return flow_levels(w, h, planes);
}

CF_API int32_t cf_wmc_filter_launches(int32_t w, int32_t h, int32_t planes, int32_t iters) {
    if (iters <= 0 || w <= 0 || h <= 0 || planes <= 0) return 0;
    return (int32_t)schedule(iters, flow_levels(w, h, planes)).size();
}

static bool u8_fusable(const void* src0, int64_t pitch, int64_t plane, int32_t w, int32_t px,
                       int32_t planes);
CF_API int32_t cf_wmc_filter_u8_fused(const void* in, int64_t in_pitch, int64_t in_plane_stride,
                                      int32_t w, int32_t iters) {
    return iters > 0 && in && w > 0 && u8_fusable(in, in_pitch, in_plane_stride, w, 1, 1) ? 1 : 0;
}

CF_API void cf_kernel_bank_x12(int32_t* out72) {
    // PAPER.md:411-444; SPEC.md:96-111 -- h_i * 12, [i][row][col]
    static const int32_t H12[72] = {
        2, 2, 0, 4, -12, 0, 2, 2, 0,    // h1
        2, 4, 2, 2, -12, 2, 0, 0, 0,    // h2
        0, 2, 2, 0, -12, 4, 0, 2, 2,    // h3
        0, 0, 0, 2, -12, 2, 2, 4, 2,    // h4
        2, 4, 1, 4, -12, 0, 1, 0, 0,    // h5
        1, 4, 2, 0, -12, 4, 0, 0, 1,    // h6
        0, 0, 1, 0, -12, 4, 1, 4, 2,    // h7
        1, 0, 0, 4, -12, 0, 2, 4, 1,    // h8
    };
    std::memcpy(out72, H12, sizeof(H12));
}

CF_API int cf_wmc_map_f32(const float* in, float* out, int32_t w, int32_t h, int64_t pitch,
                          int32_t planes, int64_t plane_stride, void* stream) {
    if (!in || !out || in == out || !shape_ok(w, h, pitch, planes, plane_stride)) return CF_EINVAL;
    DevInfo d;
    if (int rc = device_info(&d)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if ((int64_t)w * h * planes <= kFlatMapPixels) {  // latency-bound size: flat kernel
        const int64_t pairs = (int64_t)((w + 1) / 2) * h * planes;
        const int64_t blocks = std::min<int64_t>((pairs + 255) / 256, (int64_t)d.sms * 16);
        cfk::wmc_map_flat_kernel<<<(unsigned)blocks, 256, 0, s>>>(
            in, out, w, h, pitch, plane_stride, pitch, plane_stride, planes);
        CF_CUDA(cudaGetLastError());
        return CF_OK;
    }
    return launch_map(in, out, w, h, pitch, planes, plane_stride, d, s);
}

CF_API size_t cf_wmc_filter_workspace_bytes(int32_t w, int32_t h, int64_t pitch, int32_t planes,
                                            int64_t plane_stride) {
    if (!shape_ok(w, h, pitch, planes, plane_stride)) return 0;
    const int64_t elems = (planes - 1) * (planes > 1 ? plane_stride : 0) + pitch * (int64_t)h;
    return kWsHeader + (size_t)elems * sizeof(float);
}

struct DataTerm {            // solve_l2_area / solve_l1_area (f != nullptr)
    const float* f = nullptr;
    float lambda = 0.0f;
    // solve_l1_area only (d != nullptr): dual planes, ping-ponged with d_ws
    float* d = nullptr;
    float* d_ws = nullptr;
    float alpha = 1.0f;
};

// The first launch can read u8 rows itself (cfk::kModeFlowU8In) when every
// row starts on a 4-byte boundary and w % 4 == 0, so the words holding a
// row's pixels never reach past its last pixel's word: planar rows (pixel
// stride px = 1, plane stride a multiple of 4) or interleaved channels
// (plane stride 1, px = planes <= 3; two staged words per lane need C = 2).
// CF_U8_FUSE=0 forces the separate widening pass (A/B measurements).
static bool u8_fusable(const void* src0, int64_t pitch, int64_t plane, int32_t w, int32_t px,
                       int32_t planes) {
    static const bool enabled = [] {
        const char* e = std::getenv("CF_U8_FUSE");
        return !(e && e[0] == '0');
    }();
    if (!enabled || w % 4 != 0 || ((reinterpret_cast<uintptr_t>(src0) | (uintptr_t)pitch) & 3))
        return false;
    if (px == 1) return (plane & 3) == 0;
    return cfk::C == 2 && px <= 3 && plane == 1 && planes == px;
}

struct Out8 {               // fused save-time quantisation of the last launch
    uint8_t* p = nullptr;
    int64_t pitch = 0, plane = 0;
    int32_t px = 1;         // bytes between a row's pixels (channels when interleaved)
};

// Enqueue one filter / solver run: the launches of schedule(iters) on `s`.
static int enqueue_flow(const void* src0, bool src_u8, int64_t src_pitch, int64_t src_plane,
                        float* out, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                        int64_t plane_stride, int32_t iters, float dt, void* workspace,
                        cudaStream_t s, const DataTerm& dterm, const Out8& out8,
                        int32_t src_px) {
    DevInfo d;
    if (int rc = device_info(&d)) return rc;
    int32_t* flag = reinterpret_cast<int32_t*>(workspace);
    float* ws = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + kWsHeader);
    CF_CUDA(cudaMemsetAsync(flag, 0x7f, sizeof(int32_t), s));

    const std::vector<int> ks = schedule(iters, flow_levels(w, h, planes));
    // Ping-pong between the caller's buffer and the workspace, arranged so
    // the last launch writes `out` (even launch count; iters == 1 copies).
    float* cur = out;
    float* nxt = ws;
    float* dcur = dterm.d;      // kModeL1: follows the same ping-pong as U
    float* dnxt = dterm.d_ws;
    // u8 input: widened inside the first launch's row loads
    // when the bytes allow 4-byte copies, else by a separate pass
    const bool fuse8 = src_u8 && !ks.empty() &&
                       u8_fusable(src0, src_pitch, src_plane, w, src_px, planes) && !dterm.f;
    if (src_u8 && src_px != 1 && !fuse8) return CF_EINVAL;  // interleaved: fused only
    if (src_u8) {
        // the widened image (or the first launch's output) goes to whichever
        // buffer makes the final launch land in `out`
        if (ks.size() % 2 == 1) std::swap(cur, nxt);
        if (!fuse8)
            if (int rc = launch_widen(static_cast<const uint8_t*>(src0), src_pitch, src_plane, cur,
                                      pitch, plane_stride, w, h, planes, d.sms, s))
                return rc;
    }
    int iter = 0;
    for (size_t i = 0; i < ks.size(); ++i) {
        cfk::SweepParams p{};
        p.src = cur; p.dst = nxt;
        p.src_pitch = p.dst_pitch = pitch;
        p.src_plane = p.dst_plane = plane_stride;
        p.src_row0 = p.dst_row0 = 0;
        p.w = w; p.h = h; p.y0 = 0; p.y1 = h; p.planes = planes;
        p.dt = dt; p.iter_base = iter; p.flag = flag;
        p.fdata = dterm.f; p.f_pitch = pitch; p.f_plane = plane_stride; p.lambda = dterm.lambda;
        p.dsrc = dcur; p.ddst = dnxt;
        p.alpha = dterm.alpha; p.neg_inv_alpha = -(1.0f / dterm.alpha);
        if (out8.p && i + 1 == ks.size()) {  // last launch: u8 bytes instead of fp32
            p.dst8 = out8.p; p.dst8_pitch = out8.pitch; p.dst8_plane = out8.plane;
            p.dst8_px = out8.px;
        }
        const bool in8 = fuse8 && i == 0;    // first launch: u8 rows in
        if (in8) {
            p.src8 = static_cast<const uint8_t*>(src0);
            p.src8_pitch = src_pitch; p.src8_plane = src_plane; p.src8_px = src_px;
        }
        const int rc = dterm.d          ? launch<cfk::kModeL1>(p, ks[i], d, s)
                       : dterm.f        ? launch<cfk::kModeL2>(p, ks[i], d, s)
                       : in8 && p.dst8  ? launch<cfk::kModeFlowU8InOut>(p, ks[i], d, s)
                       : in8            ? launch<cfk::kModeFlowU8In>(p, ks[i], d, s)
                       : p.dst8         ? launch<cfk::kModeFlowU8>(p, ks[i], d, s)
                                        : launch<cfk::kModeFlow>(p, ks[i], d, s);
        if (rc) return rc;
        iter += ks[i];
        std::swap(cur, nxt);
        std::swap(dcur, dnxt);
    }
    if (cur != out && !out8.p) {
        // iters == 1 on an in-place f32 image: the single launch wrote ws
        for (int pl = 0; pl < planes; ++pl)
            CF_CUDA(cudaMemcpy2DAsync(out + pl * plane_stride, pitch * 4, cur + pl * plane_stride,
                                      pitch * 4, (size_t)w * 4, h, cudaMemcpyDeviceToDevice, s));
        if (dterm.d)
            for (int pl = 0; pl < planes; ++pl)
                CF_CUDA(cudaMemcpy2DAsync(dterm.d + pl * plane_stride, pitch * 4,
                                          dcur + pl * plane_stride, pitch * 4, (size_t)w * 4, h,
                                          cudaMemcpyDeviceToDevice, s));
    }
    return CF_OK;
}

static int run_flow(const void* src0, bool src_u8, int64_t src_pitch, int64_t src_plane,
                    float* out, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                    int64_t plane_stride, int32_t iters, float dt, void* workspace,
                    int32_t* first_bad_iter, cudaStream_t s, DataTerm dterm = {},
                    Out8 out8 = {}, int32_t src_px = 1) {
    FlowKey key{};
    CF_CUDA(cudaGetDevice(&key.dev));
    key.src0 = src0; key.src_u8 = src_u8; key.src_pitch = src_pitch; key.src_plane = src_plane;
    key.out = out; key.w = w; key.h = h; key.pitch = pitch; key.planes = planes;
    key.plane_stride = plane_stride; key.iters = iters; key.dt = f32_bits(dt);
    key.ws = workspace; key.f = dterm.f; key.lambda = f32_bits(dterm.lambda);
    key.d = dterm.d; key.d_ws = dterm.d_ws; key.alpha = f32_bits(dterm.alpha);
    key.o8 = out8.p; key.o8_pitch = out8.pitch; key.o8_plane = out8.plane;
    key.src_px = src_px; key.o8_px = out8.px;
    const int rc = run_cached(key.dev, key.bytes(), s, [&](cudaStream_t st) {
        return enqueue_flow(src0, src_u8, src_pitch, src_plane, out, w, h, pitch, planes,
                            plane_stride, iters, dt, workspace, st, dterm, out8, src_px);
    });
    if (rc) return rc;
    if (first_bad_iter) return cf_wmc_filter_query_nonfinite(workspace, first_bad_iter, s);
    return CF_OK;
}

// Interleaved 8-bit image in and out (wmc_io.cu's cf_wmc_filter_image8;
// arguments validated there): channel c is plane c with plane stride 1 and
// pixel stride `channels`, widened in the first launch and quantised in the
// last, when cf_internal_image8_fusable() says the input can be read that way.
extern "C" int cf_internal_image8_fusable(const uint8_t* in, int64_t in_pitch, int32_t w,
                                          int32_t channels, int32_t iters) {
    // gray: one plane (its stride unused); RGB: interleaved, plane stride 1
    return iters > 0 && u8_fusable(in, in_pitch, channels == 1 ? 0 : 1, w, channels, channels) ? 1
                                                                                               : 0;
}
CF_API int32_t cf_wmc_filter_image8_fused(const uint8_t* in, int64_t in_pitch, int32_t w,
                                          int32_t channels, int32_t iters) {
    return in && w > 0 && (channels == 1 || channels == 3)
               ? cf_internal_image8_fusable(in, in_pitch, w, channels, iters)
               : 0;
}
extern "C" int cf_internal_filter_image8(const uint8_t* in, int64_t in_pitch, int32_t channels,
                                         float* fbuf, int32_t w, int32_t h, int32_t iters,
                                         float dt, void* fws, uint8_t* out, int64_t out_pitch,
                                         int32_t* first_bad_iter, void* stream) {
    Out8 o8;
    const int64_t plane = channels == 1 ? 0 : 1;
    o8.p = out; o8.pitch = out_pitch; o8.plane = plane; o8.px = channels;
    return run_flow(in, true, in_pitch, plane, fbuf, w, h, w, channels, (int64_t)w * h, iters, dt,
                    fws, first_bad_iter, (cudaStream_t)stream, DataTerm{}, o8, channels);
}

// u8 frames in, u8 frames out with the quantisation fused into the last
// launch (wmc_io.cu's cf_wmc_filter_u8_u8; arguments validated there).
// fbuf: dense fp32 planes (pitch w), fws: the filter workspace.
extern "C" int cf_internal_filter_u8_u8(const uint8_t* in, int64_t in_pitch, int64_t in_plane,
                                        float* fbuf, int32_t w, int32_t h, int32_t planes,
                                        int32_t iters, float dt, void* fws, uint8_t* out,
                                        int64_t out_pitch, int64_t out_plane,
                                        int32_t* first_bad_iter, void* stream) {
    Out8 o8;
    o8.p = out; o8.pitch = out_pitch; o8.plane = out_plane;
    return run_flow(in, true, in_pitch, in_plane, fbuf, w, h, w, planes, (int64_t)w * h, iters,
                    dt, fws, first_bad_iter, (cudaStream_t)stream, DataTerm{}, o8);
}

CF_API int cf_wmc_filter_f32(float* img, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                             int64_t plane_stride, int32_t iters, float dt, void* workspace,
                             size_t workspace_bytes, int32_t* first_bad_iter, void* stream) {
    if (!img || !shape_ok(w, h, pitch, planes, plane_stride) || iters < 0) return CF_EINVAL;
    if (!(dt > 0.0f) || dt > 1.0f) return CF_EINVAL;
    if (first_bad_iter) *first_bad_iter = 0;
    if (iters == 0) return CF_OK;                     // identity
    if (!workspace ||
        workspace_bytes < cf_wmc_filter_workspace_bytes(w, h, pitch, planes, plane_stride))
        return CF_EINVAL;
    return run_flow(img, false, pitch, plane_stride, img, w, h, pitch, planes, plane_stride,
                    iters, dt, workspace, first_bad_iter, (cudaStream_t)stream);
}

CF_API int cf_wmc_filter_u8_f32(const uint8_t* in, int64_t in_pitch, int64_t in_plane_stride,
                                float* out, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                                int64_t plane_stride, int32_t iters, float dt, void* workspace,
                                size_t workspace_bytes, int32_t* first_bad_iter, void* stream) {
    if (!in || !out || !shape_ok(w, h, pitch, planes, plane_stride) || iters < 0)
        return CF_EINVAL;
    if (in_pitch < w || (planes > 1 && in_plane_stride < in_pitch * (int64_t)h)) return CF_EINVAL;
    if (!(dt > 0.0f) || dt > 1.0f) return CF_EINVAL;
    if (first_bad_iter) *first_bad_iter = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (iters == 0) {
        DevInfo d;
        if (int rc = device_info(&d)) return rc;
        return launch_widen(in, in_pitch, in_plane_stride, out, pitch, plane_stride, w, h, planes,
                            d.sms, s);
    }
    if (!workspace ||
        workspace_bytes < cf_wmc_filter_workspace_bytes(w, h, pitch, planes, plane_stride))
        return CF_EINVAL;
    return run_flow(in, true, in_pitch, in_plane_stride, out, w, h, pitch, planes, plane_stride,
                    iters, dt, workspace, first_bad_iter, s);
}

CF_API int cf_wmc_solve_l2_area_f32(const float* f, float* u, int32_t w, int32_t h,
                                    int64_t pitch, int32_t planes, int64_t plane_stride,
                                    int32_t iters, float dt, float lambda, int32_t init,
                                    void* workspace, size_t workspace_bytes,
                                    int32_t* first_bad_iter, void* stream) {
    if (!f || !u || f == u || !shape_ok(w, h, pitch, planes, plane_stride) || iters < 0)
        return CF_EINVAL;
    if (!(dt > 0.0f) || !(dt < 3.0e38f) || !(lambda >= 0.0f) || !(lambda < 3.0e38f))
        return CF_EINVAL;
    if (first_bad_iter) *first_bad_iter = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (init)
        for (int pl = 0; pl < planes; ++pl)  // U^0 = f
            CF_CUDA(cudaMemcpy2DAsync(u + pl * plane_stride, pitch * 4, f + pl * plane_stride,
                                      pitch * 4, (size_t)w * 4, h, cudaMemcpyDeviceToDevice, s));
    if (iters == 0) return CF_OK;
    if (!workspace ||
        workspace_bytes < cf_wmc_filter_workspace_bytes(w, h, pitch, planes, plane_stride))
        return CF_EINVAL;
    DataTerm dterm;
    dterm.f = f;
    dterm.lambda = lambda;
    return run_flow(u, false, pitch, plane_stride, u, w, h, pitch, planes, plane_stride, iters,
                    dt, workspace, first_bad_iter, s, dterm);
}

CF_API size_t cf_wmc_solve_l1_area_workspace_bytes(int32_t w, int32_t h, int64_t pitch,
                                                   int32_t planes, int64_t plane_stride) {
    if (!shape_ok(w, h, pitch, planes, plane_stride)) return 0;
    const int64_t elems = (planes - 1) * (planes > 1 ? plane_stride : 0) + pitch * (int64_t)h;
    const size_t img = ((size_t)elems * sizeof(float) + 255) & ~(size_t)255;
    return kWsHeader + img + (size_t)elems * sizeof(float);
}

CF_API int cf_wmc_solve_l1_area_f32(const float* f, float* u, float* d, int32_t w, int32_t h,
                                    int64_t pitch, int32_t planes, int64_t plane_stride,
                                    int32_t iters, float dt, float lambda, float alpha,
                                    int32_t init, void* workspace, size_t workspace_bytes,
                                    int32_t* first_bad_iter, void* stream) {
    if (!f || !u || !d || f == u || f == d || u == d ||
        !shape_ok(w, h, pitch, planes, plane_stride) || iters < 0)
        return CF_EINVAL;
    if (!(dt > 0.0f) || !(dt < 3.0e38f) || !(lambda >= 0.0f) || !(lambda < 3.0e38f))
        return CF_EINVAL;
    if (!(alpha > 0.0f) || !(alpha <= 1.0e30f)) return CF_EINVAL;
    if (first_bad_iter) *first_bad_iter = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (init) {
        for (int pl = 0; pl < planes; ++pl) {  // U^0 = f, d^0 = 0
            CF_CUDA(cudaMemcpy2DAsync(u + pl * plane_stride, pitch * 4, f + pl * plane_stride,
                                      pitch * 4, (size_t)w * 4, h, cudaMemcpyDeviceToDevice, s));
            CF_CUDA(cudaMemset2DAsync(d + pl * plane_stride, pitch * 4, 0, (size_t)w * 4, h, s));
        }
    }
    if (iters == 0) return CF_OK;
    if (!workspace ||
        workspace_bytes < cf_wmc_solve_l1_area_workspace_bytes(w, h, pitch, planes, plane_stride))
        return CF_EINVAL;
    const int64_t elems = (planes - 1) * (planes > 1 ? plane_stride : 0) + pitch * (int64_t)h;
    DataTerm dterm;
    dterm.f = f;
    dterm.lambda = lambda;
    dterm.d = d;
    dterm.d_ws = reinterpret_cast<float*>(
        reinterpret_cast<char*>(workspace) + kWsHeader +
        (((size_t)elems * sizeof(float) + 255) & ~(size_t)255));
    dterm.alpha = alpha;
    return run_flow(u, false, pitch, plane_stride, u, w, h, pitch, planes, plane_stride, iters,
                    dt, workspace, first_bad_iter, s, dterm);
}

CF_API int cf_wmc_filter_query_nonfinite(const void* workspace, int32_t* first_bad_iter,
                                         void* stream) {
    if (!workspace || !first_bad_iter) return CF_EINVAL;
    int32_t host = kFlagNone;
    cudaStream_t s = (cudaStream_t)stream;
    CF_CUDA(cudaMemcpyAsync(&host, workspace, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    if (host >= kFlagNone || host <= 0) {
        *first_bad_iter = 0;
        return CF_OK;
    }
    *first_bad_iter = host;
    return CF_ENONFINITE;
}

CF_API int cf_wmc_sweeps_band_peer_f32(const float* src, int32_t src_row0, int32_t src_rows,
                                       float* dst, int32_t dst_row0, int32_t w, int32_t h,
                                       int64_t pitch, int32_t y0, int32_t y1, int32_t sweeps,
                                       float dt, int32_t iter_base, int32_t* d_flag,
                                       float* peer_up, int32_t peer_up_row0, int32_t peer_up_end,
                                       float* peer_dn, int32_t peer_dn_row0,
                                       int32_t peer_dn_begin, void* stream) {
    if (!src || !dst || w <= 0 || h <= 0 || pitch < w) return CF_EINVAL;
    if (sweeps < 1 || sweeps > kMaxLevels || !(dt > 0.0f) || dt > 1.0f) return CF_EINVAL;
    if (y0 < 0 || y1 > h || y0 >= y1) return CF_EINVAL;
    const int need0 = std::max(0, y0 - sweeps), need1 = std::min(h, y1 + sweeps);
    if (src_row0 > need0 || src_row0 + src_rows < need1) return CF_EINVAL;
    if (peer_up && (peer_up_end < y0 || peer_up_end > y1 || peer_up_row0 > y0)) return CF_EINVAL;
    if (peer_dn && (peer_dn_begin < y0 || peer_dn_begin > y1)) return CF_EINVAL;
    DevInfo d;
    if (int rc = device_info(&d)) return rc;
    cfk::SweepParams p{};
    p.src = src; p.dst = dst;
    p.src_pitch = p.dst_pitch = pitch;
    p.src_plane = p.dst_plane = 0;
    p.src_row0 = src_row0; p.dst_row0 = dst_row0;
    p.w = w; p.h = h; p.y0 = y0; p.y1 = y1; p.planes = 1;
    p.dt = dt; p.iter_base = iter_base; p.flag = d_flag;
    p.peer_up = peer_up; p.peer_up_row0 = peer_up_row0; p.peer_up_end = peer_up_end;
    p.peer_dn = peer_dn; p.peer_dn_row0 = peer_dn_row0; p.peer_dn_begin = peer_dn_begin;
    return launch<cfk::kModeFlow>(p, sweeps, d, (cudaStream_t)stream);
}

CF_API int cf_wmc_sweeps_band_f32(const float* src, int32_t src_row0, int32_t src_rows,
                                  float* dst, int32_t dst_row0, int32_t w, int32_t h,
                                  int64_t pitch, int32_t y0, int32_t y1, int32_t sweeps,
                                  float dt, int32_t iter_base, int32_t* d_flag, void* stream) {
    if (!src || !dst || w <= 0 || h <= 0 || pitch < w) return CF_EINVAL;
    if (sweeps < 1 || sweeps > kMaxLevels || !(dt > 0.0f) || dt > 1.0f) return CF_EINVAL;
    if (y0 < 0 || y1 > h || y0 >= y1) return CF_EINVAL;
    const int need0 = std::max(0, y0 - sweeps), need1 = std::min(h, y1 + sweeps);
    if (src_row0 > need0 || src_row0 + src_rows < need1) return CF_EINVAL;
    DevInfo d;
    if (int rc = device_info(&d)) return rc;
    cfk::SweepParams p{};
    p.src = src; p.dst = dst;
    p.src_pitch = p.dst_pitch = pitch;
    p.src_plane = p.dst_plane = 0;
    p.src_row0 = src_row0; p.dst_row0 = dst_row0;
    p.w = w; p.h = h; p.y0 = y0; p.y1 = y1; p.planes = 1;
    p.dt = dt; p.iter_base = iter_base; p.flag = d_flag;
    return launch<cfk::kModeFlow>(p, sweeps, d, (cudaStream_t)stream);
}

}  // extern "C"
