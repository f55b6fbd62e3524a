/*
 * include/curveflow/capi.h -- C-ABI of the B200-native WMC path
 * (libcurveflow_b200.so, built from paper_1903_07189_b200/csrc/).
 *
 * The reference (arXiv 1903.07189, /root/reference) declares this path only
 * in its spec; its proj/include holds just the CPU executor
 * curveflow::parallel (proj/include/curveflow/parallel.hpp:7-49).  The entry
 * points below are the drop-in for the two SPEC operations on the path:
 *
 *   wmc_half_laplace(img: Image2D) -> Image2D
 *   mc_flow(img: Image2D, cfg: FlowConfig) -> Image2D
 *                                  (cfg.scheme == half_laplace only)
 *
 * and the pieces of the spec they rely on: per-channel planes
 * (SPEC.md:62-69), 8-bit widening on load, non-finite abort
 * naming the iteration, bit-identical output for any
 * parallel decomposition (parallel.hpp:23-25).
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *  - Image pointers passed to cf_wmc_* are DEVICE pointers owned by the
 *    caller, valid until the work enqueued on `stream` (a cudaStream_t passed
 *    as void*, NULL = legacy default stream) completes.  Calls are
 *    stream-ordered and asynchronous unless stated otherwise.
 *  - Images are planar fp32, row-major: element (plane p, row y, col x) is
 *    base[p*plane_stride + y*pitch + x], pitch >= w, all in ELEMENTS.
 *  - Returns CF_OK (0) or a status below; no exceptions cross the ABI.
 *    CF_ECUDA keeps the CUDA error in thread-local state (cf_last_cuda_error).
 *  - Re-entrant: concurrent calls on different streams are safe.
 *  - The filter / solver entry points keep a small LRU of CUDA graphs keyed
 *    on all of their arguments.  From the second identical call on, the
 *    launch chain replays as one graph on `stream`: same results, no
 *    per-launch gaps.  Calls made while `stream` is capturing launch
 *    directly.  Environment CF_GRAPHS=0 disables the cache.
 *  - Results are bit-identical for every launch configuration, temporal
 *    depth and band decomposition, and equal to the canonical fp32
 *    evaluation documented in DESIGN.md §3 (oracle/wmc_oracle.c).
 */
#ifndef CURVEFLOW_CAPI_H
#define CURVEFLOW_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CF_API __attribute__((visibility("default")))
#else
#define CF_API
#endif

enum cf_status {
    CF_OK = 0,
    CF_EINVAL = 1,      /* bad shape / pitch / planes / iters / dt / workspace */
    CF_ECUDA = 2,       /* CUDA runtime error, see cf_last_cuda_error()         */
    CF_ENONFINITE = 3,  /* mc_flow produced a non-finite value    */
    CF_ENODEV = 4       /* no usable sm_100 device                              */
};

/* Library version string, e.g. "curveflow-b200 0.1.0 (sm_100a)". */
CF_API const char* cf_version(void);
/* Human-readable text for a cf_status value. */
CF_API const char* cf_status_string(int status);
/* Last CUDA error code recorded on this thread by a call returning CF_ECUDA. */
CF_API int cf_last_cuda_error(void);

/* ---------------------------------------------------------------------- */
/* wmc_half_laplace (Eqs. 27-28)                  */
/* out[p][y][x] = d_m, m = argmin_i |(h_i * in)(y,x)|, ties -> smallest i,  */
/* clamp-to-edge borders.  out must not alias in.      */
/* ---------------------------------------------------------------------- */
CF_API int cf_wmc_map_f32(const float* in, float* out, int32_t w, int32_t h, int64_t pitch,
                          int32_t planes, int64_t plane_stride, void* stream);

/* ---------------------------------------------------------------------- */
/* mc_flow, scheme = half_laplace (Eq. 26)        */
/* img <- U^iters with U^{t+1} = U^t + dt * wmc_half_laplace(U^t), Jacobi.  */
/* In-place API; ping-pongs through `workspace`                            */
/* (>= cf_wmc_filter_workspace_bytes bytes of device memory).              */
/* dt in (0, 1], iters >= 0 (0 = identity).     */
/* If first_bad_iter != NULL the call synchronises `stream` and returns    */
/* CF_ENONFINITE with *first_bad_iter = the first iteration t (1-based)    */
/* whose iterate holds a NaN/Inf, else sets it to 0.   */
/* If first_bad_iter == NULL the call is fully asynchronous and the check  */
/* result can be read later with cf_wmc_filter_query_nonfinite().          */
/* ---------------------------------------------------------------------- */
CF_API size_t cf_wmc_filter_workspace_bytes(int32_t w, int32_t h, int64_t pitch, int32_t planes,
                                            int64_t plane_stride);
CF_API int cf_wmc_filter_f32(float* img, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                             int64_t plane_stride, int32_t iters, float dt, void* workspace,
                             size_t workspace_bytes, int32_t* first_bad_iter, void* stream);
/* Synchronises `stream`; returns CF_OK / CF_ENONFINITE for the last filter
 * call that used `workspace`, writing the iteration to *first_bad_iter.   */
CF_API int cf_wmc_filter_query_nonfinite(const void* workspace, int32_t* first_bad_iter,
                                         void* stream);

/* 8-bit batch variant (BASELINE cfg 5): in is u8, widened on device to    */
/* the IEEE quotient fl(q / 255) (computed division-free as an */
/* FMA-corrected reciprocal product, bit-identical for all 256 bytes):     */
/* inside the first sweep launch when cf_wmc_filter_u8_fused() says so     */
/* (4-byte aligned rows, w % 4 == 0), else by a widening pass before it;   */
/* out receives U^iters in fp32.  in_pitch / in_plane_stride in BYTES.     */
/* iters == 0 writes the widened image.                                    */
CF_API int cf_wmc_filter_u8_f32(const uint8_t* in, int64_t in_pitch, int64_t in_plane_stride,
                                float* out, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                                int64_t plane_stride, int32_t iters, float dt, void* workspace,
                                size_t workspace_bytes, int32_t* first_bad_iter, void* stream);

/* ---------------------------------------------------------------------- */
/* solve_l2_area, A = identity (Eq. 30 with      */
/* -dR_area/dU ~ H^w): u <- f when init != 0 (else continue from u), then   */
/* iters explicit steps                                                    */
/*   U' = U + dt * ((f - U) + lambda * wmc(U))                             */
/* with wmc the flow's canonical fp32 H^w.  f and u are    */
/* distinct device images of the same geometry; dt > 0, lambda >= 0.        */
/* Workspace / non-finite reporting as cf_wmc_filter_f32.                   */
/* ---------------------------------------------------------------------- */
CF_API int cf_wmc_solve_l2_area_f32(const float* f, float* u, int32_t w, int32_t h,
                                    int64_t pitch, int32_t planes, int64_t plane_stride,
                                    int32_t iters, float dt, float lambda, int32_t init,
                                    void* workspace, size_t workspace_bytes,
                                    int32_t* first_bad_iter, void* stream);

/* ---------------------------------------------------------------------- */
/* solve_l1_area, A = identity (Eqs. 32-38):      */
/* init != 0: u <- f, d <- 0; else continue from (u, d).*/
/* Each of the iters steps, per pixel (fp32):               */
/*   r = (U - f) + d;  d' = clamp(r, -alpha, alpha)                         */
/*   U' = U + dt * (lambda * wmc(U) - (2 d' - d) / alpha)                   */
/* (the shrinkage b = r - d' of Eq. 36 is eliminated).  f, u,  */
/* d: distinct device images of one geometry; dt > 0, lambda >= 0,          */
/* 0 < alpha <= 1e30.  Workspace: cf_wmc_solve_l1_area_workspace_bytes.     */
/* ---------------------------------------------------------------------- */
CF_API size_t cf_wmc_solve_l1_area_workspace_bytes(int32_t w, int32_t h, int64_t pitch,
                                                   int32_t planes, int64_t plane_stride);
CF_API int cf_wmc_solve_l1_area_f32(const float* f, float* u, float* d, int32_t w, int32_t h,
                                    int64_t pitch, int32_t planes, int64_t plane_stride,
                                    int32_t iters, float dt, float lambda, float alpha,
                                    int32_t init, void* workspace, size_t workspace_bytes,
                                    int32_t* first_bad_iter, void* stream);

/* ---------------------------------------------------------------------- */
/* Single-process sharded filter over P device buffers (SURVEY.md §8b      */
/* export 4; BASELINE cfg 4 row bands).  The plan splits the h rows like    */
/* the reference's parallel::for_rows (ceil-div blocks, parallel.hpp:36-44) */
/* and gives each part k halo rows above / below (k = sweeps per launch,   */
/* 1 <= k <= cf_wmc_max_sweeps_per_launch()).  Part p's buffers hold        */
/* rows[p] x w floats (pitch w): global rows [row0-top, row1+bot); the      */
/* caller places the band's owned rows at buffer row top[p] of bufs_a[p].   */
/* Halo rows move between parts with cudaMemcpyPeerAsync (NVLink / NVSwitch */
/* when the parts live on different GPUs), ordered by events, and each part */
/* advances with the row-band kernel on streams[p] of devices[p].  The      */
/* result is in bufs_a (an even number of launches); bit-identical to       */
/* cf_wmc_filter_f32 for any P.  flags[p]: a device int32 on devices[p].    */
/* first_bad_iter (nullable): synchronises all streams, as the filter.      */
/* ---------------------------------------------------------------------- */
#define CF_MAX_PARTS 64
typedef struct {
    int32_t h, w, parts, k;
    int32_t row0[CF_MAX_PARTS], row1[CF_MAX_PARTS]; /* owned rows [row0, row1)   */
    int32_t top[CF_MAX_PARTS], bot[CF_MAX_PARTS];   /* halo rows above / below   */
    int32_t rows[CF_MAX_PARTS];                     /* buffer rows of each part  */
} cf_shard_plan;
CF_API int cf_shard_plan_init(int32_t h, int32_t w, int32_t parts, int32_t k, cf_shard_plan* plan);
CF_API int cf_wmc_filter_sharded_f32(const cf_shard_plan* plan, float* const* bufs_a,
                                     float* const* bufs_b, int32_t* const* flags,
                                     const int32_t* devices, void* const* streams, int32_t iters,
                                     float dt, int32_t* first_bad_iter);

/* ---------------------------------------------------------------------- */
/* Fused-halo row bands across processes.  As              */
/* cf_wmc_sweeps_band_f32, and the launch also stores level-K rows          */
/* y < peer_up_end into peer_up (the upper neighbour's destination buffer,  */
/* whose row 0 is global row peer_up_row0) and rows y >= peer_dn_begin into */
/* peer_dn: the halo exchange is part of the compute kernel's stores (peer  */
/* memory mapped with cf_ipc_open_mem; NVLink between GPUs).  Null peers:   */
/* identical to cf_wmc_sweeps_band_f32.                                     */
/* ---------------------------------------------------------------------- */
CF_API int cf_wmc_sweeps_band_peer_f32(const float* src, int32_t src_row0, int32_t src_rows,
                                       float* dst, int32_t dst_row0, int32_t w, int32_t h,
                                       int64_t pitch, int32_t y0, int32_t y1, int32_t sweeps,
                                       float dt, int32_t iter_base, int32_t* d_flag,
                                       float* peer_up, int32_t peer_up_row0, int32_t peer_up_end,
                                       float* peer_dn, int32_t peer_dn_row0,
                                       int32_t peer_dn_begin, void* stream);
/* CUDA IPC / event plumbing for that protocol (handles are 64 bytes).       */
CF_API int cf_device_alloc(size_t bytes, void** dptr);
CF_API int cf_device_free(void* dptr);
/* cudaMemsetAsync of `bytes` bytes to `value` on `stream` (the band flow's
 * non-finite flag is reset with 0x7f before every run). */
CF_API int cf_device_memset(void* dptr, int value, size_t bytes, void* stream);
CF_API int cf_copy(void* dst, const void* src, size_t bytes, void* stream);
CF_API int cf_ipc_mem_handle(const void* dptr, void* handle_out);
CF_API int cf_ipc_open_mem(const void* handle, void** dptr);
CF_API int cf_ipc_close_mem(void* dptr);
CF_API int cf_ipc_event_create(void** event);
CF_API int cf_ipc_event_handle(void* event, void* handle_out);
CF_API int cf_ipc_open_event(const void* handle, void** event);
CF_API int cf_event_record(void* event, void* stream);
CF_API int cf_stream_wait_event(void* stream, void* event);
CF_API int cf_event_destroy(void* event);
CF_API int cf_stream_synchronize(void* stream);

/* ---------------------------------------------------------------------- */
/* Row-band primitive for sharded filtering (BASELINE cfg 4).               */
/* Runs `sweeps` (1 <= sweeps <= cf_wmc_max_sweeps_per_launch()) Jacobi     */
/* sweeps of the flow in ONE launch, producing global rows [y0, y1) of the  */
/* iterate U^{iter_base+sweeps} into dst, from U^{iter_base} in src.        */
/* src holds global rows [src_row0, src_row0 + src_rows) at                */
/* src + (y - src_row0) * pitch and must cover                             */
/* [max(0, y0 - sweeps), min(h, y1 + sweeps)); dst row y is written at      */
/* dst + (y - dst_row0) * pitch.  h is the GLOBAL height (clamp-to-edge    */
/* applies only at rows 0 and h-1).  d_flag (device int32, nullable) is    */
/* atomically min-ed with the first iteration producing a non-finite value.*/
/* ---------------------------------------------------------------------- */
CF_API int32_t cf_wmc_max_sweeps_per_launch(void);
/* Number of kernel launches cf_wmc_filter_f32 / _u8_f32 (and the solvers) */
/* enqueue for iters on a w x h x planes image, and the sweeps fused per    */
/* launch they schedule (at most; the geometry argument is kept so a       */
/* geometry-dependent schedule needs no ABI change -- currently 2).          */
CF_API int32_t cf_wmc_filter_launches(int32_t w, int32_t h, int32_t planes, int32_t iters);
CF_API int32_t cf_wmc_filter_sweeps_per_launch(int32_t w, int32_t h, int32_t planes);
/* 1 if the u8 entry points (_u8_f32, _u8_u8, _u8_f64 excluded) read these  */
/* u8 rows inside the first sweep launch (4-byte aligned rows, w % 4 == 0,  */
/* iters > 0), 0 if they run a separate widening launch first.             */
CF_API int32_t cf_wmc_filter_u8_fused(const void* in, int64_t in_pitch, int64_t in_plane_stride,
                                      int32_t w, int32_t iters);
CF_API int cf_wmc_sweeps_band_f32(const float* src, int32_t src_row0, int32_t src_rows,
                                  float* dst, int32_t dst_row0, int32_t w, int32_t h,
                                  int64_t pitch, int32_t y0, int32_t y1, int32_t sweeps,
                                  float dt, int32_t iter_base, int32_t* d_flag, void* stream);

/* ---------------------------------------------------------------------- */
/* 8-bit interleaved images (SPEC.md:62-69 per-channel processing, :79     */
/* widen on load / clamp + round at save).  channels = 1 or 3 (else        */
/* CF_EINVAL); in/out are HWC u8 with row pitch in BYTES;      */
/* planes are planar fp32 on [0,1].                                        */
/*   load: v = (float)q / 255.0f;  save: q = rint(fl(clamp(v,0,1) * 255)) */
/* ---------------------------------------------------------------------- */
CF_API int cf_image8_to_planes_f32(const uint8_t* in, int64_t in_pitch, int32_t w, int32_t h,
                                   int32_t channels, float* planes, int64_t pitch,
                                   int64_t plane_stride, void* stream);
CF_API int cf_planes_f32_to_image8(const float* planes, int64_t pitch, int64_t plane_stride,
                                   int32_t w, int32_t h, int32_t channels, uint8_t* out,
                                   int64_t out_pitch, void* stream);
/* mc_flow on a planar batch of 8-bit images (planes independent): widen    */
/* q/255, filter, re-quantise rint(clamp(v,0,1)*255) -- u8 frames in, u8     */
/* frames out.  Workspace: cf_wmc_filter_u8_u8_workspace_bytes.*/
CF_API size_t cf_wmc_filter_u8_u8_workspace_bytes(int32_t w, int32_t h, int32_t planes);
CF_API int cf_wmc_filter_u8_u8(const uint8_t* in, int64_t in_pitch, int64_t in_plane_stride,
                               uint8_t* out, int64_t out_pitch, int64_t out_plane_stride,
                               int32_t w, int32_t h, int32_t planes, int32_t iters, float dt,
                               void* workspace, size_t workspace_bytes, int32_t* first_bad_iter,
                               void* stream);
/* mc_flow on an interleaved 8-bit image, per channel, result re-quantised. */
/* With 4-byte aligned rows and w % 4 == 0 (cf_wmc_filter_image8_fused()   */
/* == 1) the first sweep launch reads the interleaved bytes and the last    */
/* writes them; otherwise separate deinterleave / interleave passes run.   */
CF_API size_t cf_wmc_filter_image8_workspace_bytes(int32_t w, int32_t h, int32_t channels);
CF_API int32_t cf_wmc_filter_image8_fused(const uint8_t* in, int64_t in_pitch, int32_t w,
                                          int32_t channels, int32_t iters);
CF_API int cf_wmc_filter_image8(const uint8_t* in, int64_t in_pitch, uint8_t* out,
                                int64_t out_pitch, int32_t w, int32_t h, int32_t channels,
                                int32_t iters, float dt, void* workspace, size_t workspace_bytes,
                                int32_t* first_bad_iter, void* stream);

/* ---------------------------------------------------------------------- */
/* Reductions over the WMC map.    */
/* energy: *d_out (device double) = sum |H^w|^q, q > 0, in the fixed order */
/*   of csrc/wmc_reduce.cu (32-column butterfly blocks, blocks in x order, */
/*   rows in y order, planes in order) -- deterministic, bit-exact for     */
/*   q in {0.5, 1, 2}.                                                     */
/* histogram: d_counts[nbins] (device u64) of floor((H^w*scale - lo)/width) */
/*   clamped to [0, nbins-1] (NaN -> bin 0); the reference's binning is    */
/*   scale = 255 (0-255 intensities), lo = -256, width = 1, nbins = 512.   */
/* ---------------------------------------------------------------------- */
CF_API size_t cf_wmc_reduce_workspace_bytes(int32_t w, int32_t h, int32_t planes);
CF_API int cf_wmc_energy_f64(const float* img, int32_t w, int32_t h, int64_t pitch,
                             int32_t planes, int64_t plane_stride, double q, double* d_out,
                             void* workspace, size_t workspace_bytes, void* stream);
CF_API int cf_wmc_histogram(const float* img, int32_t w, int32_t h, int64_t pitch,
                            int32_t planes, int64_t plane_stride, float scale, float lo,
                            float width, int32_t nbins, uint64_t* d_counts, void* workspace,
                            size_t workspace_bytes, void* stream);
/* fidelity: *d_out = sum |u - f|^q (f nullable: sum |u|^q), the difference */
/*   taken in fp64, same fixed order and q handling as the energy; the      */
/*   solvers' SolveReport series: l1 fidelity q = 1, l2   */
/*   0.5 * (q = 2), relative update from q = 2 sums.                        */
CF_API int cf_wmc_fidelity_f64(const float* u, const float* f, int32_t w, int32_t h,
                               int64_t pitch, int32_t planes, int64_t plane_stride, double q,
                               double* d_out, void* workspace, size_t workspace_bytes,
                               void* stream);

/* ---------------------------------------------------------------------- */
/* Seeded synthetic image generator (BASELINE.json configs). */
/* HOST memory, deterministic for a given (seed, params) on any thread     */
/* count: linear ramp background, n_rects axis-aligned rectangles then     */
/* n_discs discs of U(0,1) intensity, + N(0, sigma^2) noise, clamp [0,1].  */
/* f32: value rounded to nearest fp32.  u8: lrint(255 * value).            */
/* threads <= 0 -> hardware concurrency.                                   */
/* ---------------------------------------------------------------------- */
CF_API int cf_synth_f32(float* out, int32_t w, int32_t h, int64_t pitch, uint64_t seed,
                        int32_t n_rects, int32_t n_discs, double sigma, int32_t threads);
CF_API int cf_synth_u8(uint8_t* out, int32_t w, int32_t h, int64_t pitch, uint64_t seed,
                       int32_t n_rects, int32_t n_discs, double sigma, int32_t threads);

/* ---------------------------------------------------------------------- */
/* Kernel bank: h_i weights times 12 as exact integers,  */
/* out72[i*9 + r*3 + c], i = 0..7 for h1..h8, r/c = dy+1 / dx+1.          */
/* ---------------------------------------------------------------------- */
CF_API void cf_kernel_bank_x12(int32_t* out72);

/* ---------------------------------------------------------------------- */
/* The SPEC-faithful fp64 path (csrc/wmc_f64.cu)            */
/* fp64 images (the reference computes in fp64) and the */
/* reference CPU path's own arithmetic: per kernel s = s + w*x over the     */
/* row-major taps with w = n/12 rounded to fp64, multiply and add rounded   */
/* separately, strict-< first-minimum scan; */
/* flow step u + dt*d.  Results are BIT-IDENTICAL to the  */
/* reference CPU implementation for finite images (not a tolerance); the    */
/* price is the FP64 pipe (about 60 DP operations per pixel-update).        */
/* Layout and conventions as the fp32 entry points, elements of 8 bytes.    */
/* ---------------------------------------------------------------------- */
/* wmc_half_laplace in fp64 (replaces SPEC.md:171's operation bit-exactly). */
CF_API int cf_wmc_map_f64(const double* in, double* out, int32_t w, int32_t h, int64_t pitch,
                          int32_t planes, int64_t plane_stride, void* stream);
/* Workspace of cf_wmc_filter_f64 / cf_wmc_filter_u8_f64: 256-byte header
 * (non-finite flag) + one fp64 image of the given geometry. */
CF_API size_t cf_wmc_filter_f64_workspace_bytes(int32_t w, int32_t h, int64_t pitch,
                                                int32_t planes, int64_t plane_stride);
/* mc_flow in fp64, in place, Jacobi (replaces SPEC.md:256's operation
 * bit-exactly).  dt in (0, 1], iters >= 0 (0: identity).  first_bad_iter
 * non-null: synchronises `stream`, returns CF_ENONFINITE naming the first
 * iteration that produced a non-finite value. */
CF_API int cf_wmc_filter_f64(double* img, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                             int64_t plane_stride, int32_t iters, double dt, void* workspace,
                             size_t workspace_bytes, int32_t* first_bad_iter, void* stream);
/* u8 planes widened as (double)q / 255.0 (IEEE division), then
 * cf_wmc_filter_f64 into `out` (fp64 planes of the given geometry). */
CF_API int cf_wmc_filter_u8_f64(const uint8_t* in, int64_t in_pitch, int64_t in_plane_stride,
                                double* out, int32_t w, int32_t h, int64_t pitch, int32_t planes,
                                int64_t plane_stride, int32_t iters, double dt, void* workspace,
                                size_t workspace_bytes, int32_t* first_bad_iter, void* stream);
/* Read back the fp64 filter's non-finite flag (synchronises `stream`). */
CF_API int cf_wmc_filter_f64_query_nonfinite(const void* workspace, int32_t* first_bad_iter,
                                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CURVEFLOW_CAPI_H */
