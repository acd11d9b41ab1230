// hsad_pipeline_sharded: one process drives G GPUs. The image splits
// into row strips aligned to hsad_row_quantum (so every pixel's arithmetic, and map, is
// the one a single-GPU run produces); a host thread per strip selects its device, copies
// the strip's buffer rows (strip + reflected window halo, hsad_strip_rows) from the host
// cube, reduces them, runs the fused detectors on the strip's output rows and copies
// those map rows straight into the caller's host maps. With host outputs no collective
// is needed: each GPU writes its own rows over its own PCIe link (the torch.distributed
// path, sharded.py, is the one that gathers device maps to rank 0 with NCCL).
//
// Strips outnumbering devices run round-robin (strip g on device g % ndev), which is
// also how the strip logic is exercised on a one-GPU machine.
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "hsad_internal.h"

namespace hsad_b200 {
hsad_status detect_multi_impl(const void* d_cube, int32_t elem_bytes, int64_t lines, int64_t samples,
                              int32_t bands, int64_t buf_row0, int64_t buf_rows, int64_t row_begin,
                              int64_t row_end, const hsad_detect_request* requests, int32_t n_requests,
                              uint64_t* d_status, hsad_pixel_error* err, cudaStream_t s);
int64_t row_quantum(int64_t lines, int64_t samples);
}  // namespace hsad_b200

using namespace hsad_b200;

namespace {

struct StripResult {
    hsad_status status = HSAD_OK;
    hsad_pixel_error err{HSAD_OK, -1, -1};
    std::string message;
};

// one strip on the current device: rows [r0, r1) of the maps, buffer rows [b0, b0 + nb)
void run_strip(const float* h_cube, int64_t lines, int64_t samples, int32_t bands, int32_t order,
               int32_t target, int64_t r0, int64_t r1, const hsad_detect_request* host_requests,
               int32_t n, int device, StripResult* out) {
    auto fail = [&](hsad_status st) {
        out->status = st;
        out->message = hsad_last_error_message();
    };
    if (cudaSetDevice(device) != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "cudaSetDevice"));
    int64_t b0 = 0, nb = 0;
    hsad_status st = hsad_strip_rows(lines, r0, r1, host_requests, n, &b0, &nb);
    if (st != HSAD_OK) return fail(st);
    const int32_t det_bands = order > 0 ? target : bands;
    const size_t row_px = static_cast<size_t>(samples);
    cudaStream_t s = nullptr;
    std::vector<void*> bufs;
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess) return nullptr;
        bufs.push_back(p);
        return p;
    };
    auto cleanup = [&]() {
        if (s) cudaStreamSynchronize(s);
        for (void* p : bufs) cudaFree(p);
        if (s) cudaStreamDestroy(s);
    };
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
        s = nullptr;
        return fail(set_error(HSAD_E_CUDA, "stream creation failed"));
    }
    float* d_cube = static_cast<float*>(alloc(static_cast<size_t>(nb) * row_px * bands * sizeof(float)));
    double* d_red = order > 0 ? static_cast<double*>(alloc(static_cast<size_t>(nb) * row_px * target * sizeof(double)))
                              : nullptr;
    uint64_t* d_status = static_cast<uint64_t*>(alloc(sizeof(uint64_t)));
    hsad_detect_request dev_req[kMaxCallRequests];
    bool ok = d_cube && d_status && (order <= 0 || d_red);
    for (int q = 0; q < n && ok; ++q) {
        dev_req[q] = host_requests[q];
        const int sb = host_requests[q].score_bytes == 4 ? 4 : 8;
        dev_req[q].d_scores = alloc(static_cast<size_t>(r1 - r0) * row_px * sb);
        dev_req[q].d_eigcount = (host_requests[q].algorithm == HSAD_DWEST && host_requests[q].d_eigcount)
                                    ? static_cast<int8_t*>(alloc(static_cast<size_t>(r1 - r0) * row_px))
                                    : nullptr;
        ok = dev_req[q].d_scores != nullptr;
    }
    if (!ok) {
        cleanup();
        return fail(set_error(HSAD_E_CUDA, "device allocation failed for strip rows [" + std::to_string(r0) +
                                               ", " + std::to_string(r1) + ")"));
    }
    cudaError_t e = cudaMemcpyAsync(d_cube, h_cube + static_cast<size_t>(b0) * row_px * bands,
                                    static_cast<size_t>(nb) * row_px * bands * sizeof(float),
                                    cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_status, 0xff, sizeof(uint64_t), s);
    if (e != cudaSuccess) {
        cleanup();
        return fail(cuda_fail(e, "strip H2D"));
    }
    if (order > 0) {
        st = hsad_reduce(d_cube, 4, nb, samples, bands, order, target, d_red, 8, s);
        if (st != HSAD_OK) {
            cleanup();
            return fail(st);
        }
    }
    // synchronous detector call: reports the strip's first failing pixel with its message
    st = detect_multi_impl(order > 0 ? static_cast<const void*>(d_red) : d_cube, order > 0 ? 8 : 4, lines,
                           samples, det_bands, b0, nb, r0, r1, dev_req, n, nullptr, &out->err, s);
    if (st != HSAD_OK) {
        cleanup();
        return fail(st);
    }
    for (int q = 0; q < n && e == cudaSuccess; ++q) {
        const int sb = host_requests[q].score_bytes == 4 ? 4 : 8;
        e = cudaMemcpyAsync(static_cast<char*>(host_requests[q].d_scores) + static_cast<size_t>(r0) * row_px * sb,
                            dev_req[q].d_scores, static_cast<size_t>(r1 - r0) * row_px * sb,
                            cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && dev_req[q].d_eigcount)
            e = cudaMemcpyAsync(host_requests[q].d_eigcount + static_cast<size_t>(r0) * row_px,
                                dev_req[q].d_eigcount, static_cast<size_t>(r1 - r0) * row_px,
                                cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cleanup();
    if (e != cudaSuccess) return fail(cuda_fail(e, "strip D2H"));
}

}  // namespace

extern "C" hsad_status hsad_pipeline_sharded(const float* h_cube, int64_t lines, int64_t samples,
                                             int32_t bands, int32_t order, int32_t target_bands,
                                             const hsad_detect_request* host_requests, int32_t n_requests,
                                             int32_t n_strips, hsad_pixel_error* err) {
    if (err) {
        err->code = HSAD_OK;
        err->row = err->col = -1;
    }
    if (lines < 0 || samples < 0) return set_error(HSAD_E_INVALID_VALUE, "negative cube extent");
    if (n_requests < 1 || n_requests > kMaxCallRequests || !host_requests)
        return set_error(HSAD_E_INVALID_VALUE, "between 1 and 16 requests per call");
    if (n_strips < 1) return set_error(HSAD_E_INVALID_VALUE, "n_strips must be >= 1");
    if (!h_cube && lines * samples * bands > 0) return set_error(HSAD_E_INVALID_VALUE, "null cube");
    if (order > 0) {
        hsad_status st = wavelet_plan(bands, order, target_bands, nullptr);
        if (st != HSAD_OK) return st;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
        return set_error(HSAD_E_CUDA, "no CUDA device");
    if (lines == 0 || samples == 0) return HSAD_OK;
    // strips of the row quantum (bit-identical maps at any strip count)
    const int64_t q = row_quantum(lines, samples);
    const int64_t per = (lines + static_cast<int64_t>(n_strips) * q - 1) / (static_cast<int64_t>(n_strips) * q) * q;
    std::vector<StripResult> res(n_strips);
    std::vector<std::thread> threads;
    for (int g = 0; g < n_strips; ++g) {
        const int64_t r0 = g * per < lines ? g * per : lines;
        const int64_t r1 = (g + 1) * per < lines ? (g + 1) * per : lines;
        if (r1 <= r0) continue;
        threads.emplace_back(run_strip, h_cube, lines, samples, bands, order, target_bands, r0, r1,
                             host_requests, n_requests, g % ndev, &res[g]);
    }
    for (auto& t : threads) t.join();
    // report like one sequential call: the first failing pixel in row-major order
    // (strips are in row order), else the first other failure
    for (int g = 0; g < n_strips; ++g)
        if (res[g].status != HSAD_OK) {
            if (err) *err = res[g].err;
            return set_error(res[g].status, res[g].message.substr(res[g].message.find(": ") + 2));
        }
    return HSAD_OK;
}
