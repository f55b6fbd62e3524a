// paper_1903_07189_b200/csrc/wmc_ipc.cpp -- the CUDA IPC plumbing of the
// fused-halo row-band flow across processes: device buffers
// whose IPC handles a neighbour process maps (its band kernel then stores
// boundary rows straight into them, over NVLink when the processes own
// different GPUs), and interprocess events ordering the launches.  Thin
// C-ABI wrappers so host code in any language can drive the protocol.
#include <cuda_runtime.h>

#include <cstring>

#include "../../include/curveflow/capi.h"

extern "C" void cf_internal_set_cuda_error(int e);

namespace {
int st(cudaError_t e) {
    if (e == cudaSuccess) return CF_OK;
    cf_internal_set_cuda_error((int)e);
    return CF_ECUDA;
}
}  // namespace

extern "C" {

CF_API int cf_device_alloc(size_t bytes, void** dptr) {
    if (!dptr || bytes == 0) return CF_EINVAL;
    return st(cudaMalloc(dptr, bytes));  // a whole allocation: its IPC handle maps its base
}

CF_API int cf_device_free(void* dptr) { return st(cudaFree(dptr)); }

CF_API int cf_device_memset(void* dptr, int value, size_t bytes, void* stream) {
    if (!dptr) return CF_EINVAL;
    return st(cudaMemsetAsync(dptr, value, bytes, (cudaStream_t)stream));
}

CF_API int cf_copy(void* dst, const void* src, size_t bytes, void* stream) {
    if (!dst || !src) return CF_EINVAL;
    return st(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
}

CF_API int cf_ipc_mem_handle(const void* dptr, void* handle_out) {
    if (!dptr || !handle_out) return CF_EINVAL;
    cudaIpcMemHandle_t h;
    const int rc = st(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
    if (rc == CF_OK) std::memcpy(handle_out, &h, sizeof(h));
    return rc;
}

CF_API int cf_ipc_open_mem(const void* handle, void** dptr) {
    if (!handle || !dptr) return CF_EINVAL;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    return st(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
}

CF_API int cf_ipc_close_mem(void* dptr) { return st(cudaIpcCloseMemHandle(dptr)); }

CF_API int cf_ipc_event_create(void** event) {
    if (!event) return CF_EINVAL;
    cudaEvent_t e;
    const int rc = st(cudaEventCreateWithFlags(&e, cudaEventInterprocess | cudaEventDisableTiming));
    if (rc == CF_OK) *event = e;
    return rc;
}

CF_API int cf_ipc_event_handle(void* event, void* handle_out) {
    if (!event || !handle_out) return CF_EINVAL;
    cudaIpcEventHandle_t h;
    const int rc = st(cudaIpcGetEventHandle(&h, (cudaEvent_t)event));
    if (rc == CF_OK) std::memcpy(handle_out, &h, sizeof(h));
    return rc;
}

CF_API int cf_ipc_open_event(const void* handle, void** event) {
    if (!handle || !event) return CF_EINVAL;
    cudaIpcEventHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    cudaEvent_t e;
    const int rc = st(cudaIpcOpenEventHandle(&e, h));
    if (rc == CF_OK) *event = e;
    return rc;
}

CF_API int cf_event_record(void* event, void* stream) {
    return st(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
}

CF_API int cf_stream_wait_event(void* stream, void* event) {
    return st(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0));
}

CF_API int cf_event_destroy(void* event) { return st(cudaEventDestroy((cudaEvent_t)event)); }

CF_API int cf_stream_synchronize(void* stream) {
    return st(cudaStreamSynchronize((cudaStream_t)stream));
}

}  // extern "C"
