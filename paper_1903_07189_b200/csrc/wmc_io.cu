// paper_1903_07189_b200/csrc/wmc_io.cu -- 8-bit images on either side of the
// WMC filter: interleaved 1/3-channel images and
// planar u8 batches (cfg5 frames in, frames out).
//
// Reference semantics: images are processed per channel (SPEC.md:62-69,
// PAPER.md:674 "performed on each color channel separately"); 8-bit inputs
// are widened on load and outputs are clamped to the 8-bit range and rounded
// only at save time.  This build works on [0,1] floats:
//   load : v = (float)q / 255.0f                         (IEEE division)
//   save : q = rint(fl(clamp(v, 0, 1) * 255.0f))          (round half to even)
// Channels: 1 (gray) or 3 (RGB); anything else is a format error.
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/curveflow/capi.h"

extern "C" void cf_internal_set_cuda_error(int e);  // wmc_capi.cu (not exported)
extern "C" int cf_internal_image8_fusable(const uint8_t* in, int64_t in_pitch, int32_t w,
                                          int32_t channels, int32_t iters);
extern "C" int cf_internal_filter_image8(const uint8_t* in, int64_t in_pitch, int32_t channels,
                                         float* fbuf, int32_t w, int32_t h, int32_t iters,
                                         float dt, void* fws, uint8_t* out, int64_t out_pitch,
                                         int32_t* first_bad_iter, void* stream);
extern "C" int cf_internal_filter_u8_u8(const uint8_t* in, int64_t in_pitch, int64_t in_plane,
                                        float* fbuf, int32_t w, int32_t h, int32_t planes,
                                        int32_t iters, float dt, void* fws, uint8_t* out,
                                        int64_t out_pitch, int64_t out_plane,
                                        int32_t* first_bad_iter, void* stream);

namespace {

constexpr size_t align256(size_t n) { return (n + 255) & ~(size_t)255; }

__global__ void deinterleave_kernel(const uint8_t* __restrict__ in, int64_t in_pitch, int32_t w,
                                    int32_t h, int32_t ch, float* __restrict__ out,
                                    int64_t pitch, int64_t plane_stride) {
    for (int64_t y = blockIdx.x; y < h; y += gridDim.x) {
        const uint8_t* row = in + y * in_pitch;
        for (int x = threadIdx.x; x < w; x += blockDim.x)
            for (int c = 0; c < ch; ++c)
                out[c * plane_stride + y * pitch + x] = __fdiv_rn((float)row[x * ch + c], 255.0f);
    }
}

__device__ __forceinline__ uint8_t quantize(float v) {
    const float c = fminf(fmaxf(v, 0.0f), 1.0f);  // NaN -> 0 (fmaxf returns the number)
    return (uint8_t)__float2int_rn(__fmul_rn(c, 255.0f));
}

__global__ void interleave_kernel(const float* __restrict__ in, int64_t pitch,
                                  int64_t plane_stride, int32_t w, int32_t h, int32_t ch,
                                  uint8_t* __restrict__ out, int64_t out_pitch) {
    for (int64_t y = blockIdx.x; y < h; y += gridDim.x) {
        uint8_t* row = out + y * out_pitch;
        for (int x = threadIdx.x; x < w; x += blockDim.x)
            for (int c = 0; c < ch; ++c) row[x * ch + c] = quantize(in[c * plane_stride + y * pitch + x]);
    }
}

// Planar quantisation of a batch (one byte per pixel per plane).
__global__ void quantize_planes_kernel(const float* __restrict__ in, int64_t pitch,
                                       int64_t plane_stride, int32_t w, int32_t h, int32_t planes,
                                       uint8_t* __restrict__ out, int64_t out_pitch,
                                       int64_t out_plane_stride) {
    // one row per block iteration: a single index division per row
    const int64_t rows = (int64_t)h * planes;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int64_t p = r / h, y = r - p * h;
        const float* src = in + p * plane_stride + y * pitch;
        uint8_t* dst = out + p * out_plane_stride + y * out_pitch;
        for (int x = threadIdx.x; x < w; x += blockDim.x) dst[x] = quantize(src[x]);
    }
}

bool io_shape_ok(int32_t w, int32_t h, int32_t ch, int64_t pitch8, int64_t pitch,
                 int64_t plane_stride) {
    if (w <= 0 || h <= 0 || (ch != 1 && ch != 3)) return false;
    if (pitch8 < (int64_t)w * ch || pitch < w) return false;
    if (ch > 1 && plane_stride < pitch * (int64_t)h) return false;
    return true;
}

int io_launch_check() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        cf_internal_set_cuda_error((int)e);
        return CF_ECUDA;
    }
    return CF_OK;
}

}  // namespace

extern "C" {

CF_API int cf_image8_to_planes_f32(const uint8_t* in, int64_t in_pitch, int32_t w, int32_t h,
                                   int32_t channels, float* planes, int64_t pitch,
                                   int64_t plane_stride, void* stream) {
    if (!in || !planes || !io_shape_ok(w, h, channels, in_pitch, pitch, plane_stride))
        return CF_EINVAL;
    deinterleave_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(in, in_pitch, w, h, channels,
                                                                 planes, pitch, plane_stride);
    return io_launch_check();
}

CF_API int cf_planes_f32_to_image8(const float* planes, int64_t pitch, int64_t plane_stride,
                                   int32_t w, int32_t h, int32_t channels, uint8_t* out,
                                   int64_t out_pitch, void* stream) {
    if (!planes || !out || !io_shape_ok(w, h, channels, out_pitch, pitch, plane_stride))
        return CF_EINVAL;
    interleave_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(planes, pitch, plane_stride, w, h,
                                                               channels, out, out_pitch);
    return io_launch_check();
}

CF_API size_t cf_wmc_filter_image8_workspace_bytes(int32_t w, int32_t h, int32_t channels) {
    if (w <= 0 || h <= 0 || (channels != 1 && channels != 3)) return 0;
    const int64_t plane = (int64_t)w * h;
    // planar fp32 image + the filter's own workspace (header + one image)
    return align256((size_t)(channels * plane) * sizeof(float)) +
           cf_wmc_filter_workspace_bytes(w, h, w, channels, plane);
}

CF_API int cf_wmc_filter_image8(const uint8_t* in, int64_t in_pitch, uint8_t* out,
                                int64_t out_pitch, int32_t w, int32_t h, int32_t channels,
                                int32_t iters, float dt, void* workspace, size_t workspace_bytes,
                                int32_t* first_bad_iter, void* stream) {
    if (!in || !out || !workspace) return CF_EINVAL;
    if (!io_shape_ok(w, h, channels, in_pitch, w, (int64_t)w * h) || out_pitch < (int64_t)w * channels)
        return CF_EINVAL;
    if (workspace_bytes < cf_wmc_filter_image8_workspace_bytes(w, h, channels)) return CF_EINVAL;
    const int64_t plane = (int64_t)w * h;
    float* planes = reinterpret_cast<float*>(workspace);
    // the filter workspace follows the planes, 256-byte aligned
    const size_t off = align256((size_t)(channels * plane) * sizeof(float));
    void* fws = reinterpret_cast<char*>(workspace) + off;
    const size_t fws_bytes = workspace_bytes - off;
    if (cf_internal_image8_fusable(in, in_pitch, w, channels, iters)) {
        // deinterleave + widen inside the first sweep launch, clamp + round +
        // interleave inside the last (4-byte aligned rows, w % 4 == 0)
        if (!(dt > 0.0f) || dt > 1.0f) return CF_EINVAL;
        if (first_bad_iter) *first_bad_iter = 0;
        return cf_internal_filter_image8(in, in_pitch, channels, planes, w, h, iters, dt, fws, out,
                                         out_pitch, first_bad_iter, stream);
    }
    int rc = cf_image8_to_planes_f32(in, in_pitch, w, h, channels, planes, w, plane, stream);
    if (rc) return rc;
    rc = cf_wmc_filter_f32(planes, w, h, w, channels, plane, iters, dt, fws, fws_bytes,
                           first_bad_iter, stream);
    if (rc) return rc;
    return cf_planes_f32_to_image8(planes, w, plane, w, h, channels, out, out_pitch, stream);
}

CF_API size_t cf_wmc_filter_u8_u8_workspace_bytes(int32_t w, int32_t h, int32_t planes) {
    if (w <= 0 || h <= 0 || planes <= 0) return 0;
    const int64_t plane = (int64_t)w * h;
    return align256((size_t)(planes * plane) * sizeof(float)) +
           cf_wmc_filter_workspace_bytes(w, h, w, planes, plane);
}

CF_API int cf_wmc_filter_u8_u8(const uint8_t* in, int64_t in_pitch, int64_t in_plane_stride,
                               uint8_t* out, int64_t out_pitch, int64_t out_plane_stride,
                               int32_t w, int32_t h, int32_t planes, int32_t iters, float dt,
                               void* workspace, size_t workspace_bytes, int32_t* first_bad_iter,
                               void* stream) {
    if (!in || !out || !workspace || w <= 0 || h <= 0 || planes <= 0 || iters < 0)
        return CF_EINVAL;
    if (in_pitch < w || out_pitch < w) return CF_EINVAL;
    if (planes > 1 && (in_plane_stride < in_pitch * (int64_t)h ||
                       out_plane_stride < out_pitch * (int64_t)h))
        return CF_EINVAL;
    if (workspace_bytes < cf_wmc_filter_u8_u8_workspace_bytes(w, h, planes)) return CF_EINVAL;
    const int64_t plane = (int64_t)w * h;
    float* f = reinterpret_cast<float*>(workspace);
    const size_t off = align256((size_t)(planes * plane) * sizeof(float));
    if (!(dt > 0.0f) || dt > 1.0f) return CF_EINVAL;
    if (iters > 0)  // the last sweep launch stores quantised bytes (no fp32 round trip)
        return cf_internal_filter_u8_u8(in, in_pitch, in_plane_stride, f, w, h, planes, iters, dt,
                                        reinterpret_cast<char*>(workspace) + off, out, out_pitch,
                                        out_plane_stride, first_bad_iter, stream);
    int rc = cf_wmc_filter_u8_f32(in, in_pitch, in_plane_stride, f, w, h, w, planes, plane, 0, dt,
                                  reinterpret_cast<char*>(workspace) + off, workspace_bytes - off,
                                  first_bad_iter, stream);
    if (rc) return rc;
    quantize_planes_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(
        f, w, plane, w, h, planes, out, out_pitch, out_plane_stride);
    return io_launch_check();
}

}  // extern "C"
