// paper_1903_07189_b200/csrc/synth.cpp -- seeded synthetic-image generator.
//
// Stand-in for the inputs BASELINE.json's five configs describe ("seeded
// piecewise-smooth synthetic image: random axis-aligned rectangles and discs
// of uniform-random constant intensity over a linear ramp background, plus
// i.i.d. Gaussian noise, clamped to [0,1]").  The reference names no public
// dataset for this path; the paper's own images are
// not used.  Every free choice is pinned here and in DESIGN.md §6:
//
//  - shape parameters: xoshiro256** seeded by SplitMix64(seed), drawn in the
//    order ramp (v0, v1, theta), then each rectangle (w, h, x, y, value), then
//    each disc (cx, cy, radius, value); doubles are (next >> 11) * 2^-53;
//  - ramp: v0 + (v1 - v0) * t, t = projection of the pixel centre on
//    (cos theta, sin theta), normalised over the image corners to [0, 1];
//  - rectangle: sides U[W/64, W/8] x U[H/64, H/8], corner uniform so it fits;
//    covers pixel (x, y) iff x0 <= x + 0.5 < x0 + w (and likewise in y);
//  - disc: centre U[0,W] x U[0,H], radius U[min(W,H)/128, min(W,H)/16];
//    covers pixel iff |(x+0.5, y+0.5) - c| <= r;
//  - painted rectangles first, then discs, in draw order (later wins);
//  - noise: counter-based, n = sqrt(-2 ln u1) cos(2 pi u2) with u1, u2 from
//    SplitMix64(key ^ (2i)), SplitMix64(key ^ (2i+1)) of the pixel's linear
//    index i = y*W + x, so the image is identical for any thread count;
//  - value = clamp(base + sigma * n, 0, 1) in double, then rounded to fp32
//    (f32) or lrint(255 * value) (u8).
//
// Host code; runs on the CPU cores of the box (rows split like
// curveflow::parallel::for_rows, proj/include/curveflow/parallel.hpp:26-47).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/curveflow/capi.h"

namespace {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct Xoshiro256ss {
    uint64_t s[4];
    explicit Xoshiro256ss(uint64_t seed) {
        uint64_t z = seed;
        for (auto& v : s) { z = splitmix64(z); v = z; }
    }
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t next() {
        const uint64_t r = rotl(s[1] * 5, 7) * 9;
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
        s[2] ^= t; s[3] = rotl(s[3], 45);
        return r;
    }
    double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

struct Rect { double x0, y0, x1, y1, v; };
struct Disc { double cx, cy, r, v; };

struct Scene {
    double v0, v1, ct, st, tmin, tinv;
    std::vector<Rect> rects;
    std::vector<Disc> discs;
    uint64_t noise_key;
};

Scene make_scene(int w, int h, uint64_t seed, int n_rects, int n_discs) {
    Scene sc;
    Xoshiro256ss rng(seed);
    sc.v0 = rng.uniform();
    sc.v1 = rng.uniform();
    const double theta = rng.uniform(0.0, 2.0 * M_PI);
    sc.ct = std::cos(theta);
    sc.st = std::sin(theta);
    const double cx[4] = {0.0, (double)w, 0.0, (double)w};
    const double cy[4] = {0.0, 0.0, (double)h, (double)h};
    double tmin = 1e300, tmax = -1e300;
    for (int i = 0; i < 4; ++i) {
        const double t = cx[i] * sc.ct + cy[i] * sc.st;
        tmin = std::min(tmin, t);
        tmax = std::max(tmax, t);
    }
    sc.tmin = tmin;
    sc.tinv = tmax > tmin ? 1.0 / (tmax - tmin) : 0.0;
    sc.rects.reserve(n_rects);
    for (int i = 0; i < n_rects; ++i) {
        const double rw = rng.uniform(w / 64.0, w / 8.0);
        const double rh = rng.uniform(h / 64.0, h / 8.0);
        const double x0 = rng.uniform(0.0, std::max(0.0, w - rw));
        const double y0 = rng.uniform(0.0, std::max(0.0, h - rh));
        const double v = rng.uniform();
        sc.rects.push_back({x0, y0, x0 + rw, y0 + rh, v});
    }
    const double m = (double)std::min(w, h);
    sc.discs.reserve(n_discs);
    for (int i = 0; i < n_discs; ++i) {
        const double dx = rng.uniform(0.0, (double)w);
        const double dy = rng.uniform(0.0, (double)h);
        const double r = rng.uniform(m / 128.0, m / 16.0);
        const double v = rng.uniform();
        sc.discs.push_back({dx, dy, r, v});
    }
    sc.noise_key = splitmix64(seed ^ 0x6E6F697365ull /* "noise" */);
    return sc;
}

inline double gauss(uint64_t key, uint64_t i) {
    const uint64_t a = splitmix64(key ^ (2 * i));
    const uint64_t b = splitmix64(key ^ (2 * i + 1));
    const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = (double)(b >> 11) * 0x1.0p-53;          // [0, 1)
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// Fill one row of clamped double values.
void render_row(const Scene& sc, int w, int y, double sigma, std::vector<double>& row) {
    const double yc = y + 0.5;
    for (int x = 0; x < w; ++x) {
        const double t = ((x + 0.5) * sc.ct + yc * sc.st - sc.tmin) * sc.tinv;
        row[x] = sc.v0 + (sc.v1 - sc.v0) * t;
    }
    for (const Rect& r : sc.rects) {
        if (!(r.y0 <= yc && yc < r.y1)) continue;
        // x + 0.5 in [x0, x1)  <=>  x in [ceil(x0 - 0.5), ceil(x1 - 0.5))
        const int xa = std::max(0, (int)std::ceil(r.x0 - 0.5));
        const int xb = std::min(w, (int)std::ceil(r.x1 - 0.5));
        for (int x = xa; x < xb; ++x) row[x] = r.v;
    }
    for (const Disc& d : sc.discs) {
        const double dy = yc - d.cy;
        const double rem = d.r * d.r - dy * dy;
        if (rem < 0.0) continue;
        const double hw = std::sqrt(rem);
        const int xa = std::max(0, (int)std::floor(d.cx - hw - 0.5) - 1);
        const int xb = std::min(w, (int)std::ceil(d.cx + hw - 0.5) + 2);
        for (int x = xa; x < xb; ++x) {
            const double dx = x + 0.5 - d.cx;
            if (dx * dx + dy * dy <= d.r * d.r) row[x] = d.v;
        }
    }
    const uint64_t base = (uint64_t)y * (uint64_t)w;
    for (int x = 0; x < w; ++x) {
        double v = row[x] + sigma * gauss(sc.noise_key, base + (uint64_t)x);
        row[x] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
}

template <typename Fn>
void parallel_rows(int h, int threads, Fn&& fn) {
    int workers = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    workers = std::min(workers, h);
    if (workers <= 1 || h < 16) {
        for (int y = 0; y < h; ++y) fn(y);
        return;
    }
    const int chunk = (h + workers - 1) / workers;
    std::vector<std::thread> pool;
    for (int wk = 1; wk < workers; ++wk) {
        const int y0 = wk * chunk, y1 = std::min(h, y0 + chunk);
        if (y0 >= y1) break;
        pool.emplace_back([&fn, y0, y1] { for (int y = y0; y < y1; ++y) fn(y); });
    }
    for (int y = 0; y < std::min(chunk, h); ++y) fn(y);
    for (auto& t : pool) t.join();
}

template <typename T, typename Conv>
int synth(T* out, int32_t w, int32_t h, int64_t pitch, uint64_t seed, int32_t n_rects,
          int32_t n_discs, double sigma, int32_t threads, Conv conv) {
    if (!out || w <= 0 || h <= 0 || pitch < w || n_rects < 0 || n_discs < 0 || !(sigma >= 0.0))
        return CF_EINVAL;
    const Scene sc = make_scene(w, h, seed, n_rects, n_discs);
    parallel_rows(h, threads, [&](int y) {
        thread_local std::vector<double> row;
        row.resize((size_t)w);
        render_row(sc, w, y, sigma, row);
        T* o = out + (int64_t)y * pitch;
        for (int x = 0; x < w; ++x) o[x] = conv(row[x]);
    });
    return CF_OK;
}

}  // namespace

extern "C" CF_API int cf_synth_f32(float* out, int32_t w, int32_t h, int64_t pitch, uint64_t seed,
                                   int32_t n_rects, int32_t n_discs, double sigma,
                                   int32_t threads) {
    return synth(out, w, h, pitch, seed, n_rects, n_discs, sigma, threads,
                 [](double v) { return (float)v; });
}

extern "C" CF_API int cf_synth_u8(uint8_t* out, int32_t w, int32_t h, int64_t pitch, uint64_t seed,
                                  int32_t n_rects, int32_t n_discs, double sigma,
                                  int32_t threads) {
    return synth(out, w, h, pitch, seed, n_rects, n_discs, sigma, threads,
                 [](double v) { return (uint8_t)std::lrint(255.0 * v); });
}
