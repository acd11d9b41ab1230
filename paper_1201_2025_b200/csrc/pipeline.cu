// hsad_pipeline_host: reduce_cube + detect on HOST buffers — the composition the
// reference CLI runs (`hsad reduce` then `hsad detect`, proj/tools/hsad_main.cpp:112-198)
// minus file I/O. H2D of the fp32 cube, K1 reduction into a device-resident
// reduced cube, one fused K2-K4 pass for every request, D2H of every map.
// Device buffers are cached per host thread so repeated calls do not re-allocate.
#include <cstdint>
#include <string>

#include "hsad_internal.h"

namespace hsad_b200 {

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int device = -1;
    cudaError_t reserve(size_t n) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (p && bytes >= n && device == dev) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, n ? n : 1);
        if (e == cudaSuccess) {
            bytes = n;
            device = dev;
        }
        return e;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct PipelineCache {
    DevBuf cube, reduced, out[kMaxRequests], counts[kMaxRequests];
};
thread_local PipelineCache g_cache;

}  // namespace
}  // namespace hsad_b200

using namespace hsad_b200;

extern "C" hsad_status hsad_pipeline_host(const float* h_cube, int64_t lines, int64_t samples,
                                          int32_t bands, int32_t order, int32_t target_bands,
                                          const hsad_detect_request* host_requests,
                                          int32_t n_requests, hsad_pixel_error* err,
                                          void* stream) {
    if (!h_cube && lines * samples * bands > 0) return set_error(HSAD_E_INVALID_VALUE, "null cube");
    if (n_requests < 1 || n_requests > kMaxRequests || !host_requests)
        return set_error(HSAD_E_INVALID_VALUE, "between 1 and 4 requests per call");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t npix = lines * samples;
    const int32_t det_bands = order > 0 ? target_bands : bands;
    if (order > 0) {
        hsad_status st = wavelet_plan(bands, order, target_bands, nullptr);
        if (st != HSAD_OK) return st;
    }
    PipelineCache& c = g_cache;
    const size_t cube_bytes = static_cast<size_t>(npix) * bands * sizeof(float);
    HSAD_CUDA_TRY(c.cube.reserve(cube_bytes));
    if (cube_bytes) HSAD_CUDA_TRY(cudaMemcpyAsync(c.cube.p, h_cube, cube_bytes, cudaMemcpyHostToDevice, s));
    const void* d_det = c.cube.p;
    int32_t det_elem = 4;
    FuseSrc fuse{static_cast<const float*>(c.cube.p), bands, order, nullptr};
    if (order > 0) {
        HSAD_CUDA_TRY(c.reduced.reserve(static_cast<size_t>(npix) * target_bands * sizeof(double)));
        if (npix) {
            hsad_status st = device_wavelet_map(bands, order, target_bands, &fuse.wmap);
            if (st != HSAD_OK) return st;
        }
        d_det = c.reduced.p;
        det_elem = 8;
    }
    hsad_detect_request dev_req[kMaxRequests];
    for (int q = 0; q < n_requests; ++q) {
        dev_req[q] = host_requests[q];
        const int sb = host_requests[q].score_bytes;
        HSAD_CUDA_TRY(c.out[q].reserve(static_cast<size_t>(npix) * (sb == 4 ? 4 : 8)));
        dev_req[q].d_scores = c.out[q].p;
        if (host_requests[q].algorithm == HSAD_DWEST && host_requests[q].d_eigcount) {
            HSAD_CUDA_TRY(c.counts[q].reserve(static_cast<size_t>(npix)));
            dev_req[q].d_eigcount = static_cast<int8_t*>(c.counts[q].p);
        } else {
            dev_req[q].d_eigcount = nullptr;
        }
    }
    // order > 0: the DWT runs inside the detector launch (or K1 first, see detect.cu)
    hsad_status st = detect_multi_impl(d_det, det_elem, lines, samples, det_bands, 0, lines, 0,
                                       lines, dev_req, n_requests, nullptr, err, s,
                                       order > 0 ? &fuse : nullptr);
    if (st != HSAD_OK) return st;
    for (int q = 0; q < n_requests; ++q) {
        const int sb = host_requests[q].score_bytes;
        if (npix)
            HSAD_CUDA_TRY(cudaMemcpyAsync(host_requests[q].d_scores, c.out[q].p,
                                          static_cast<size_t>(npix) * sb, cudaMemcpyDeviceToHost, s));
        if (dev_req[q].d_eigcount && npix)
            HSAD_CUDA_TRY(cudaMemcpyAsync(host_requests[q].d_eigcount, c.counts[q].p,
                                          static_cast<size_t>(npix), cudaMemcpyDeviceToHost, s));
    }
    HSAD_CUDA_TRY(cudaStreamSynchronize(s));
    return HSAD_OK;
}
