// oracle/ref_exec.cpp -- TEST INFRASTRUCTURE ONLY (see wmc_oracle.c header).
//
// The reference ships exactly one compilable native component on this path:
// its row-parallel executor curveflow::parallel
// (/root/reference/proj/include/curveflow/parallel.hpp:7-49).  This file is
// compiled against that header IN PLACE (oracle/Makefile, -I into
// /root/reference/proj/include; the header is never copied into this repo)
// into oracle/_ref/libcf_ref.so, so the fp64 restatement of wmc_half_laplace
// / mc_flow can be run on the reference's own executor.  tests/ check it is
// bit-identical to the oracle's for_rows restatement for every thread count
// (parallel.hpp:23-25).
#include <curveflow/parallel.hpp>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" {
#include "wmc_px.h"
}

extern "C" __attribute__((visibility("default"))) int ref_wmc_map_f64(const double* in, double* out,
                                                                     int32_t w, int32_t h,
                                                                     int32_t threads) {
    if (w <= 0 || h <= 0) return 1;
    pthread_once(&hw_once, init_hw64);
    curveflow::parallel::set_num_threads(threads);
    curveflow::parallel::for_rows(h, [&](int y) {
        for (int x = 0; x < w; ++x) out[(int64_t)y * w + x] = wmc_px_f64(in, w, h, w, y, x, nullptr);
    });
    return 0;
}

extern "C" __attribute__((visibility("default"))) int ref_flow_f64(double* img, int32_t w, int32_t h,
                                                                  int32_t iters, double dt,
                                                                  int32_t threads, int32_t* bad_iter) {
    if (w <= 0 || h <= 0 || iters < 0 || !(dt > 0.0) || dt > 1.0) return 1;
    pthread_once(&hw_once, init_hw64);
    curveflow::parallel::set_num_threads(threads);
    if (bad_iter) *bad_iter = 0;
    std::vector<double> tmp((size_t)w * h);
    std::vector<int> bad(h);
    double* A = img;
    double* B = tmp.data();
    int rc = 0;
    for (int t = 1; t <= iters; ++t) {
        std::fill(bad.begin(), bad.end(), 0);
        curveflow::parallel::for_rows(h, [&](int y) {
            int b = 0;
            for (int x = 0; x < w; ++x) {
                double v = A[(int64_t)y * w + x] + dt * wmc_px_f64(A, w, h, w, y, x, nullptr);
                if (!std::isfinite(v)) b = 1;
                B[(int64_t)y * w + x] = v;
            }
            bad[y] = b;
        });
        std::swap(A, B);
        int any = 0;
        for (int y = 0; y < h; ++y) any |= bad[y];
        if (any) { if (bad_iter) *bad_iter = t; rc = 3; break; }
    }
    if (A != img) std::memcpy(img, A, sizeof(double) * (size_t)w * h);
    return rc;
}
