// paper_1903_07189_b200/csrc/cf_cli.cpp -- `curveflow` command-line driver
// in C++ over the C++ API (include/curveflow/wmc.hpp) and the C-ABI.
//
// Mirrors the reference CLI shapes for this path (SPEC.md:201 `op --kind wmc`,
// :274 `flow --scheme half`, :458 `bench`) on seeded synthetic inputs
// (PGM/PNG file I/O is out of scope):
//
//   curveflow_b200 op    --size H W --seed S [--fp64]  -> checksum of the map
//                                                       (--fp64: curveflow::cuda::exact, the
//                                                        reference's own fp64 arithmetic)
//   curveflow_b200 flow  --size H W --iters N --dt D [--parts P]
//                                                       -> checksum of U^N (P row bands:
//                                                          the single-process sharded filter)
//   curveflow_b200 bench --size H W --iters N --reps R -> Gpixel-updates/s
//   curveflow_b200 smooth --model l1|l2 --lambda L --alpha A --iters N --dt D
//                                                       -> checksum of U
//
// Output: one JSON object per invocation on stdout.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/curveflow/wmc.hpp"

namespace {

template <typename T>
uint64_t fnv1a(const std::vector<T>& v) {
    uint64_t h = 1469598103934665603ull;
    const unsigned char* p = reinterpret_cast<const unsigned char*>(v.data());
    for (size_t i = 0; i < v.size() * sizeof(T); ++i) h = (h ^ p[i]) * 1099511628211ull;
    return h;
}

curveflow::Image2D64 widen(const curveflow::Image2D& img) {
    curveflow::Image2D64 out(img.width, img.height);
    for (size_t i = 0; i < img.data.size(); ++i) out.data[i] = img.data[i];
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s op|flow|bench|smooth [--size H W] [--seed S] "
                             "[--iters N] [--dt D] [--reps R] [--model l1|l2] [--lambda L] "
                             "[--alpha A]\n", argv[0]);
        return 2;
    }
    const std::string cmd = argv[1];
    int H = 512, W = 512, iters = 100, reps = 3;
    uint64_t seed = 1;
    double dt = 1.0, lambda = 0.0, alpha = 1.0;
    int parts = 1;
    bool dt_set = false, fp64 = false;
    std::string model = "l2";
    for (int i = 2; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--size") && i + 2 < argc) {
            H = std::atoi(argv[++i]);
            W = std::atoi(argv[++i]);
        } else if (!std::strcmp(argv[i], "--seed") && i + 1 < argc) {
            seed = std::strtoull(argv[++i], nullptr, 10);
        } else if (!std::strcmp(argv[i], "--iters") && i + 1 < argc) {
            iters = std::atoi(argv[++i]);
        } else if (!std::strcmp(argv[i], "--dt") && i + 1 < argc) {
            dt = std::atof(argv[++i]);
            dt_set = true;
        } else if (!std::strcmp(argv[i], "--parts") && i + 1 < argc) {
            parts = std::atoi(argv[++i]);
        } else if (!std::strcmp(argv[i], "--model") && i + 1 < argc) {
            model = argv[++i];
        } else if (!std::strcmp(argv[i], "--lambda") && i + 1 < argc) {
            lambda = std::atof(argv[++i]);
        } else if (!std::strcmp(argv[i], "--alpha") && i + 1 < argc) {
            alpha = std::atof(argv[++i]);
        } else if (!std::strcmp(argv[i], "--fp64")) {
            fp64 = true;
        } else if (!std::strcmp(argv[i], "--reps") && i + 1 < argc) {
            reps = std::atoi(argv[++i]);
        }
    }
    curveflow::Image2D img(W, H);
    if (cf_synth_f32(img.data.data(), W, H, W, seed, 20, 20, 0.1, 0) != CF_OK) return 1;
    try {
        if (cmd == "op" && fp64) {
            auto m = curveflow::cuda::exact::wmc_half_laplace(widen(img));
            std::printf("{\"op\": \"wmc\", \"fp64\": true, \"h\": %d, \"w\": %d, "
                        "\"fnv1a\": \"%016llx\"}\n", H, W, (unsigned long long)fnv1a(m.data));
        } else if (cmd == "flow" && fp64) {
            auto u = curveflow::cuda::exact::mc_flow(widen(img), {dt, iters});
            std::printf("{\"op\": \"flow\", \"fp64\": true, \"h\": %d, \"w\": %d, "
                        "\"iters\": %d, \"fnv1a\": \"%016llx\"}\n", H, W, iters,
                        (unsigned long long)fnv1a(u.data));
        } else if (cmd == "op") {
            auto m = curveflow::cuda::wmc_half_laplace(img);
            std::printf("{\"op\": \"wmc\", \"h\": %d, \"w\": %d, \"fnv1a\": \"%016llx\"}\n", H, W,
                        (unsigned long long)fnv1a(m.data));
        } else if (cmd == "flow") {
            auto u = parts > 1 ? curveflow::cuda::mc_flow_sharded(img, {dt, iters}, parts)
                               : curveflow::cuda::mc_flow(img, {dt, iters});
            std::printf("{\"op\": \"flow\", \"h\": %d, \"w\": %d, \"iters\": %d, \"fnv1a\": "
                        "\"%016llx\"}\n", H, W, iters, (unsigned long long)fnv1a(u.data));
        } else if (cmd == "smooth") {
            curveflow::SolverConfig cfg;
            cfg.lambda = lambda;
            cfg.alpha = alpha;
            cfg.iters = iters;
            if (dt_set) cfg.dt = dt;  // else the SPEC default 0.15
            if (model == "l1") cfg.model = curveflow::SolverConfig::Model::l1_area;
            else if (model != "l2") throw std::invalid_argument("--model must be l1 or l2");
            auto rep = curveflow::cuda::solve(img, cfg);
            std::printf("{\"op\": \"smooth\", \"model\": \"%s\", \"h\": %d, \"w\": %d, "
                        "\"iters\": %d, \"fidelity\": %.17g, \"fnv1a\": \"%016llx\"}\n",
                        model.c_str(), H, W, iters, rep.fidelity,
                        (unsigned long long)fnv1a(rep.image.data));
        } else if (cmd == "bench") {
            // device-resident timing of mc_flow (SPEC.md:437-456 median of reps)
            const size_t n = img.data.size() * sizeof(float);
            curveflow::detail::DevBuf d(n), ws(curveflow::cuda::device::flow_workspace_bytes(W, H));
            std::vector<double> ms;
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int r = 0; r < reps + 1; ++r) {
                cudaMemcpy(d.p, img.data.data(), n, cudaMemcpyHostToDevice);
                cudaEventRecord(a);
                curveflow::cuda::device::mc_flow((float*)d.p, W, H, {dt, iters}, ws.p,
                                                 curveflow::cuda::device::flow_workspace_bytes(W, H));
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float t = 0;
                cudaEventElapsedTime(&t, a, b);
                if (r > 0) ms.push_back(t);  // first run is warm-up
            }
            std::sort(ms.begin(), ms.end());
            const double med = ms[ms.size() / 2];
            std::printf("{\"op\": \"bench\", \"h\": %d, \"w\": %d, \"iters\": %d, \"reps\": %d, "
                        "\"median_ms\": %.4f, \"gpixel_updates_per_s\": %.3f}\n", H, W, iters,
                        reps, med, (double)H * W * iters / (med * 1e-3) / 1e9);
        } else {
            std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
            return 2;
        }
    } catch (const curveflow::FlowError& e) {
        std::printf("{\"error\": \"%s\", \"iteration\": %d}\n", e.what(), e.iteration());
        return 3;
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
