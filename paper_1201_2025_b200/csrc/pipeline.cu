// hsad_pipeline_host: reduce_cube + detect on HOST buffers — the composition the
// reference CLI runs (`hsad reduce` then `hsad detect`, proj/tools/hsad_main.cpp:112-198)
// minus file I/O.
//
// The cube is streamed in row strips so that PCIe and the kernels overlap:
//
//   copy stream   : H2D strip i (fp32 rows [r0, r1))            -> event h[i]
//   caller stream : wait h[i]; K1 reduce of rows [r0, r1);
//                   detect the output rows whose windows are now complete
//                   ([d0, d1), multiples of hsad_row_quantum)    -> event d[i]
//   D2H stream    : wait d[i]; D2H of those map rows
//
// Strip boundaries on the row quantum keep every map bit-identical to a single
// whole-image hsad_reduce + hsad_detect_multi (the detector's strip property).
// The step is then bound by the H2D of the fp32 cube (PCIe), with the kernels and
// the map D2H hidden under it except for the last strip. Device buffers, streams
// and events are cached per host thread so repeated calls do not re-allocate.
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "hsad_internal.h"

namespace hsad_b200 {

hsad_status detect_multi_impl(const void* d_cube, int32_t elem_bytes, int64_t lines,
                              int64_t samples, int32_t bands, int64_t buf_row0, int64_t buf_rows,
                              int64_t row_begin, int64_t row_end,
                              const hsad_detect_request* requests, int32_t n_requests,
                              uint64_t* d_status, hsad_pixel_error* err, cudaStream_t s);
int64_t row_quantum(int64_t lines, int64_t samples);

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

constexpr int kMaxStrips = 16;

struct PipelineCache {
    DevBuf cube, reduced, out[kMaxCallRequests], counts[kMaxCallRequests], status;
    int device = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr, comp = nullptr;  // comp: hsad_pipeline_sharded
    cudaEvent_t ev_h[kMaxStrips] = {}, ev_d[kMaxStrips] = {}, ev_start = nullptr;
    cudaError_t init() {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (h2d && device == dev) return cudaSuccess;
        // a device switch leaks the old handles; they belong to the other device
        h2d = d2h = nullptr;
        if ((e = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking)) != cudaSuccess) return e;
        for (int i = 0; i < kMaxStrips; ++i) {
            if ((e = cudaEventCreateWithFlags(&ev_h[i], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&ev_d[i], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        if ((e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming)) != cudaSuccess) return e;
        device = dev;
        return cudaSuccess;
    }
};
thread_local PipelineCache g_cache;

}  // namespace hsad_b200

using namespace hsad_b200;

extern "C" hsad_status hsad_reduce(const void* d_cube, int32_t elem_bytes, int64_t lines,
                                   int64_t samples, int32_t bands, int32_t order,
                                   int32_t target_bands, void* d_out, int32_t out_bytes,
                                   void* stream);

namespace hsad_b200 {

// Output rows [row0, row1) of the maps (row0 a multiple of the row quantum), streamed
// from the HOST cube on the current device with the given cache: the buffer rows the
// windows need ([b0, b0 + nb), hsad_strip_rows) move H2D in sub-strips on the copy
// stream, are reduced on `s`, and every quantum-aligned block of output rows whose
// windows are resident is detected and copied back on the D2H stream into rows
// [row0, row1) of the caller's full-image host maps. *fail receives the call's packed
// failure word (UINT64_MAX: none); err / the thread's message describe it.
hsad_status pipeline_rows(PipelineCache& c, const float* h_cube, int64_t lines, int64_t samples,
                          int32_t bands, int32_t order, int32_t target_bands,
                          const hsad_detect_request* host_requests, int32_t n_requests, int64_t row0,
                          int64_t row1, hsad_pixel_error* err, cudaStream_t s,
                          unsigned long long* fail) {
    if (fail) *fail = ~0ull;
    const int32_t det_bands = order > 0 ? target_bands : bands;
    HSAD_CUDA_TRY(c.init());
    int64_t b0 = 0, nb = 0;
    hsad_status st = hsad_strip_rows(lines, row0, row1, host_requests, n_requests, &b0, &nb);
    if (st != HSAD_OK) return st;
    const size_t row_px = static_cast<size_t>(samples);
    const int64_t nout = row1 - row0;
    HSAD_CUDA_TRY(c.cube.reserve(static_cast<size_t>(nb) * row_px * bands * sizeof(float)));
    const void* d_det = c.cube.p;
    int32_t det_elem = 4;
    if (order > 0) {
        HSAD_CUDA_TRY(c.reduced.reserve(static_cast<size_t>(nb) * row_px * target_bands * sizeof(double)));
        d_det = c.reduced.p;
        det_elem = 8;
    }
    hsad_detect_request dev_req[kMaxCallRequests];
    for (int q = 0; q < n_requests; ++q) {
        dev_req[q] = host_requests[q];
        const int sb = host_requests[q].score_bytes;
        HSAD_CUDA_TRY(c.out[q].reserve(static_cast<size_t>(nout) * row_px * (sb == 4 ? 4 : 8)));
        dev_req[q].d_scores = c.out[q].p;
        if (host_requests[q].algorithm == HSAD_DWEST && host_requests[q].d_eigcount) {
            HSAD_CUDA_TRY(c.counts[q].reserve(static_cast<size_t>(nout) * row_px));
            dev_req[q].d_eigcount = static_cast<int8_t*>(c.counts[q].p);
        } else {
            dev_req[q].d_eigcount = nullptr;
        }
    }
    // request validation before any transfer (an empty range validates only)
    st = detect_multi_impl(d_det, det_elem, lines, samples, det_bands, b0, nb, row0, row0, dev_req,
                           n_requests, nullptr, err, s);
    if (st != HSAD_OK || nout == 0 || samples == 0) return st;
    HSAD_CUDA_TRY(c.status.reserve(sizeof(uint64_t)));
    uint64_t* d_status = static_cast<uint64_t*>(c.status.p);
    HSAD_CUDA_TRY(cudaMemsetAsync(d_status, 0xff, sizeof(uint64_t), s));

    int64_t rmax = 0;  // rows a window reaches beyond its pixel
    for (int q = 0; q < n_requests; ++q) {
        const hsad_window& w = host_requests[q].window;
        const int64_t r = (w.mode == HSAD_WINDOW_SINGLE ? w.single_size : w.outer_size) / 2;
        rmax = r > rmax ? r : rmax;
    }
    const int64_t quantum = row_quantum(lines, samples);
    int64_t strip = (nb + kMaxStrips - 1) / kMaxStrips;
    // a sub-strip moves at least ~8 MB (~150 us of PCIe): smaller ones only add launch and
    // event overhead (a 64 x 64 x 189 cube is one 3 MB strip)
    const int64_t row_bytes = samples * bands * static_cast<int64_t>(sizeof(float));
    const int64_t min_rows = row_bytes > 0 ? ((8 << 20) + row_bytes - 1) / row_bytes : nb;
    if (strip < min_rows) strip = min_rows;
    strip = (strip + quantum - 1) / quantum * quantum;
    if (strip < quantum) strip = quantum;

    // the copy streams start after the caller's earlier work on `stream`
    HSAD_CUDA_TRY(cudaEventRecord(c.ev_start, s));
    HSAD_CUDA_TRY(cudaStreamWaitEvent(c.h2d, c.ev_start, 0));
    HSAD_CUDA_TRY(cudaStreamWaitEvent(c.d2h, c.ev_start, 0));
    int64_t d_done = row0;
    int i = 0;
    for (int64_t r0 = b0; r0 < b0 + nb; r0 += strip, ++i) {
        const int64_t r1 = r0 + strip < b0 + nb ? r0 + strip : b0 + nb;
        const size_t off = static_cast<size_t>(r0 - b0) * row_px * bands;
        HSAD_CUDA_TRY(cudaMemcpyAsync(static_cast<float*>(c.cube.p) + off,
                                      h_cube + static_cast<size_t>(r0) * row_px * bands,
                                      static_cast<size_t>(r1 - r0) * row_px * bands * sizeof(float),
                                      cudaMemcpyHostToDevice, c.h2d));
        HSAD_CUDA_TRY(cudaEventRecord(c.ev_h[i], c.h2d));
        HSAD_CUDA_TRY(cudaStreamWaitEvent(s, c.ev_h[i], 0));
        if (order > 0) {
            st = hsad_reduce(static_cast<const float*>(c.cube.p) + off, 4, r1 - r0, samples, bands,
                             order, target_bands,
                             static_cast<double*>(c.reduced.p) +
                                 static_cast<size_t>(r0 - b0) * row_px * target_bands,
                             8, s);
            if (st != HSAD_OK) break;
        }
        // output rows whose windows lie inside the resident rows [b0, r1)
        int64_t d1 = r1 == b0 + nb ? row1 : (r1 - rmax) / quantum * quantum;
        if (d1 > row1) d1 = row1;
        if (d1 <= d_done) continue;
        hsad_detect_request part[kMaxCallRequests];
        for (int q = 0; q < n_requests; ++q) {
            part[q] = dev_req[q];
            const int sb = dev_req[q].score_bytes;
            part[q].d_scores = static_cast<char*>(dev_req[q].d_scores) + (d_done - row0) * row_px * sb;
            if (part[q].d_eigcount) part[q].d_eigcount += (d_done - row0) * row_px;
        }
        st = detect_multi_impl(d_det, det_elem, lines, samples, det_bands, b0, r1 - b0, d_done, d1, part,
                               n_requests, d_status, err, s);
        if (st != HSAD_OK) break;
        HSAD_CUDA_TRY(cudaEventRecord(c.ev_d[i], s));
        HSAD_CUDA_TRY(cudaStreamWaitEvent(c.d2h, c.ev_d[i], 0));
        const size_t rows_px = static_cast<size_t>(d1 - d_done) * row_px;
        for (int q = 0; q < n_requests; ++q) {
            const int sb = host_requests[q].score_bytes;
            HSAD_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(host_requests[q].d_scores) + d_done * row_px * sb,
                                          part[q].d_scores, rows_px * sb, cudaMemcpyDeviceToHost, c.d2h));
            if (part[q].d_eigcount)
                HSAD_CUDA_TRY(cudaMemcpyAsync(host_requests[q].d_eigcount + d_done * row_px,
                                              part[q].d_eigcount, rows_px, cudaMemcpyDeviceToHost, c.d2h));
        }
        d_done = d1;
    }
    // drain all three streams before returning (or reporting a launch error)
    const cudaError_t e1 = cudaStreamSynchronize(c.h2d);
    const cudaError_t e2 = cudaStreamSynchronize(c.d2h);
    const cudaError_t e3 = cudaStreamSynchronize(s);
    if (st != HSAD_OK) return st;
    HSAD_CUDA_TRY(e1);
    HSAD_CUDA_TRY(e2);
    HSAD_CUDA_TRY(e3);
    unsigned long long packed = 0;
    HSAD_CUDA_TRY(cudaMemcpy(&packed, d_status, sizeof(packed), cudaMemcpyDeviceToHost));
    if (fail) *fail = packed;
    if (packed == ~0ull) return HSAD_OK;
    // a pixel failed: re-run its row chunk synchronously for the reference message
    // (identical arithmetic: same rows resident, chunk-aligned range)
    const int64_t row = failure_pixel(packed) / samples;
    const int64_t a = row / quantum * quantum > row0 ? row / quantum * quantum : row0;
    const int64_t b = a + quantum < row1 ? a + quantum : row1;
    hsad_detect_request part[kMaxCallRequests];
    for (int q = 0; q < n_requests; ++q) {
        part[q] = dev_req[q];
        const int sb = dev_req[q].score_bytes;
        part[q].d_scores = static_cast<char*>(dev_req[q].d_scores) + (a - row0) * row_px * sb;
        if (part[q].d_eigcount) part[q].d_eigcount += (a - row0) * row_px;
    }
    st = detect_multi_impl(d_det, det_elem, lines, samples, det_bands, b0, nb, a, b, part, n_requests,
                           nullptr, err, s);
    return st != HSAD_OK ? st : set_error(HSAD_E_CUDA, "pipeline: failing pixel not reproduced");
}

// hsad_pipeline_sharded's per-device work: rows [row0, row1) on `device` with that
// device's persistent cache (buffers, streams and events live across calls; one host
// thread per device at a time holds its lock).
hsad_status pipeline_rows_device(int device, const float* h_cube, int64_t lines, int64_t samples,
                                 int32_t bands, int32_t order, int32_t target_bands,
                                 const hsad_detect_request* host_requests, int32_t n_requests,
                                 int64_t row0, int64_t row1, hsad_pixel_error* err,
                                 unsigned long long* fail) {
    static std::mutex guard;
    static std::vector<std::unique_ptr<PipelineCache>> caches;
    static std::vector<std::unique_ptr<std::mutex>> locks;
    PipelineCache* c = nullptr;
    std::mutex* mu = nullptr;
    {
        std::lock_guard<std::mutex> lock(guard);
        while (static_cast<int>(caches.size()) <= device) {
            caches.emplace_back(new PipelineCache());
            locks.emplace_back(new std::mutex());
        }
        c = caches[device].get();
        mu = locks[device].get();
    }
    std::lock_guard<std::mutex> lock(*mu);
    HSAD_CUDA_TRY(cudaSetDevice(device));
    HSAD_CUDA_TRY(c->init());
    return pipeline_rows(*c, h_cube, lines, samples, bands, order, target_bands, host_requests,
                         n_requests, row0, row1, err, c->comp, fail);
}

}  // namespace hsad_b200

extern "C" hsad_status hsad_pipeline_host(const float* h_cube, int64_t lines, int64_t samples,
                                          int32_t bands, int32_t order, int32_t target_bands,
                                          const hsad_detect_request* host_requests,
                                          int32_t n_requests, hsad_pixel_error* err,
                                          void* stream) {
    if (err) {
        err->code = HSAD_OK;
        err->row = err->col = -1;
    }
    if (lines < 0 || samples < 0) return set_error(HSAD_E_INVALID_VALUE, "negative cube extent");
    if (!h_cube && lines * samples * bands > 0) return set_error(HSAD_E_INVALID_VALUE, "null cube");
    if (n_requests < 1 || n_requests > kMaxCallRequests || !host_requests)
        return set_error(HSAD_E_INVALID_VALUE, "between 1 and 16 requests per call");
    if (order > 0) {
        hsad_status st = wavelet_plan(bands, order, target_bands, nullptr);
        if (st != HSAD_OK) return st;
    }
    return pipeline_rows(g_cache, h_cube, lines, samples, bands, order, target_bands, host_requests,
                         n_requests, 0, lines, err, static_cast<cudaStream_t>(stream), nullptr);
}

// hsad_pipeline_raw: the same streamed composition starting from the raw bytes of an
// ENVI file (read_cube + reduce_cube + detect, cube.cpp:198-253 -> wavelet.cpp:148-167 ->
// detect.cpp:159-289) for BSQ / BIL cubes of any supported type. Strip i's rows move
// host -> device into their place of a device copy of the raw image (BSQ: one 2D copy
// of `bands` plane segments; BIL: one contiguous block), are decoded and reduced in one
// pass (reduce_raw_rows), and detected / copied back as in hsad_pipeline_host. int16
// files move half the PCIe bytes of the fp32 cube. A non-finite element anywhere is
// reported first (read_cube runs before the detectors in the reference).
extern "C" hsad_status hsad_pipeline_raw(const void* h_raw, int64_t raw_bytes, const hsad_cube_header* header,
                                         int32_t order, int32_t target_bands,
                                         const hsad_detect_request* host_requests, int32_t n_requests,
                                         hsad_pixel_error* err, void* stream) {
    if (err) {
        err->code = HSAD_OK;
        err->row = err->col = -1;
    }
    if (!header) return set_error(HSAD_E_INVALID_VALUE, "null header");
    const hsad_cube_header& h = *header;
    hsad_status st = validate_raw(h, raw_bytes);
    if (st != HSAD_OK) return st;
    if (h.interleave == HSAD_BIP)
        return set_error(HSAD_E_UNSUPPORTED, "BIP input: decode with hsad_read_cube or use hsad_pipeline_host");
    if (order <= 0) return set_error(HSAD_E_UNSUPPORTED, "hsad_pipeline_raw reduces (order >= 1)");
    if (!h_raw) return set_error(HSAD_E_INVALID_VALUE, "null raw buffer");
    if (n_requests < 1 || n_requests > kMaxCallRequests || !host_requests)
        return set_error(HSAD_E_INVALID_VALUE, "between 1 and 16 requests per call");
    st = wavelet_plan(h.bands, order, target_bands, nullptr);
    if (st != HSAD_OK) return st;
    if (target_bands != 1 && target_bands != 2 && target_bands != 4 && target_bands != 8 && target_bands != 16)
        return set_error(HSAD_E_UNSUPPORTED, "raw-cube reduction supports 1..16 target bands");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t lines = h.lines, samples = h.samples;
    const int64_t npix = lines * samples;
    const size_t es = static_cast<size_t>(raw_bytes / (npix * h.bands));
    PipelineCache& c = g_cache;
    HSAD_CUDA_TRY(c.init());
    const size_t row_px = static_cast<size_t>(samples);
    HSAD_CUDA_TRY(c.cube.reserve(static_cast<size_t>(raw_bytes)));
    HSAD_CUDA_TRY(c.reduced.reserve(static_cast<size_t>(npix) * target_bands * sizeof(double)));
    hsad_detect_request dev_req[kMaxCallRequests];
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
    st = detect_multi_impl(c.reduced.p, 8, lines, samples, target_bands, 0, lines, 0, 0, dev_req,
                           n_requests, nullptr, err, s);
    if (st != HSAD_OK) return st;
    // two status words: [0] detector failures, [1] first non-finite raw element
    HSAD_CUDA_TRY(c.status.reserve(2 * sizeof(uint64_t)));
    uint64_t* d_status = static_cast<uint64_t*>(c.status.p);
    unsigned long long* d_nonfinite = reinterpret_cast<unsigned long long*>(d_status + 1);
    HSAD_CUDA_TRY(cudaMemsetAsync(d_status, 0xff, 2 * sizeof(uint64_t), s));

    int64_t rmax = 0;
    for (int q = 0; q < n_requests; ++q) {
        const hsad_window& w = host_requests[q].window;
        const int64_t r = (w.mode == HSAD_WINDOW_SINGLE ? w.single_size : w.outer_size) / 2;
        rmax = r > rmax ? r : rmax;
    }
    const int64_t quantum = row_quantum(lines, samples);
    int64_t strip = (lines + kMaxStrips - 1) / kMaxStrips;
    const int64_t row_bytes = samples * h.bands * static_cast<int64_t>(es);
    const int64_t min_rows = ((8 << 20) + row_bytes - 1) / row_bytes;
    if (strip < min_rows) strip = min_rows;
    strip = (strip + quantum - 1) / quantum * quantum;
    if (strip < quantum) strip = quantum;

    HSAD_CUDA_TRY(cudaEventRecord(c.ev_start, s));
    HSAD_CUDA_TRY(cudaStreamWaitEvent(c.h2d, c.ev_start, 0));
    HSAD_CUDA_TRY(cudaStreamWaitEvent(c.d2h, c.ev_start, 0));
    const size_t plane_bytes = static_cast<size_t>(npix) * es;
    int64_t d_done = 0;
    int i = 0;
    cudaError_t ce = cudaSuccess;
    for (int64_t r0 = 0; r0 < lines && ce == cudaSuccess; r0 += strip, ++i) {
        const int64_t r1 = r0 + strip < lines ? r0 + strip : lines;
        if (h.interleave == HSAD_BSQ) {  // rows [r0, r1) of every band plane
            const size_t off = static_cast<size_t>(r0) * row_px * es;
            ce = cudaMemcpy2DAsync(static_cast<char*>(c.cube.p) + off, plane_bytes,
                                   static_cast<const char*>(h_raw) + off, plane_bytes,
                                   static_cast<size_t>(r1 - r0) * row_px * es, h.bands,
                                   cudaMemcpyHostToDevice, c.h2d);
        } else {  // BIL: lines are contiguous
            const size_t off = static_cast<size_t>(r0) * row_bytes;
            ce = cudaMemcpyAsync(static_cast<char*>(c.cube.p) + off, static_cast<const char*>(h_raw) + off,
                                 static_cast<size_t>(r1 - r0) * row_bytes, cudaMemcpyHostToDevice, c.h2d);
        }
        if (ce != cudaSuccess) break;
        if ((ce = cudaEventRecord(c.ev_h[i], c.h2d)) != cudaSuccess) break;
        if ((ce = cudaStreamWaitEvent(s, c.ev_h[i], 0)) != cudaSuccess) break;
        if ((ce = reduce_raw_rows(h, c.cube.p, order, target_bands, c.reduced.p, 8, d_nonfinite, s, r0, r1)) !=
            cudaSuccess)
            break;
        int64_t d1 = r1 == lines ? lines : (r1 - rmax) / quantum * quantum;
        if (d1 <= d_done) continue;
        hsad_detect_request part[kMaxCallRequests];
        for (int q = 0; q < n_requests; ++q) {
            part[q] = dev_req[q];
            const int sb = dev_req[q].score_bytes;
            part[q].d_scores = static_cast<char*>(dev_req[q].d_scores) + d_done * row_px * sb;
            if (part[q].d_eigcount) part[q].d_eigcount += d_done * row_px;
        }
        st = detect_multi_impl(c.reduced.p, 8, lines, samples, target_bands, 0, r1, d_done, d1, part,
                               n_requests, d_status, err, s);
        if (st != HSAD_OK) break;
        if ((ce = cudaEventRecord(c.ev_d[i], s)) != cudaSuccess) break;
        if ((ce = cudaStreamWaitEvent(c.d2h, c.ev_d[i], 0)) != cudaSuccess) break;
        const size_t rows_px = static_cast<size_t>(d1 - d_done) * row_px;
        for (int q = 0; q < n_requests && ce == cudaSuccess; ++q) {
            const int sb = host_requests[q].score_bytes;
            ce = cudaMemcpyAsync(static_cast<char*>(host_requests[q].d_scores) + d_done * row_px * sb,
                                 part[q].d_scores, rows_px * sb, cudaMemcpyDeviceToHost, c.d2h);
            if (ce == cudaSuccess && part[q].d_eigcount)
                ce = cudaMemcpyAsync(host_requests[q].d_eigcount + d_done * row_px, part[q].d_eigcount,
                                     rows_px, cudaMemcpyDeviceToHost, c.d2h);
        }
        d_done = d1;
    }
    const cudaError_t e1 = cudaStreamSynchronize(c.h2d);
    const cudaError_t e2 = cudaStreamSynchronize(c.d2h);
    const cudaError_t e3 = cudaStreamSynchronize(s);
    if (st != HSAD_OK) return st;
    HSAD_CUDA_TRY(ce);
    HSAD_CUDA_TRY(e1);
    HSAD_CUDA_TRY(e2);
    HSAD_CUDA_TRY(e3);
    unsigned long long words[2] = {~0ull, ~0ull};
    HSAD_CUDA_TRY(cudaMemcpy(words, d_status, sizeof(words), cudaMemcpyDeviceToHost));
    if (words[1] != ~0ull) return nonfinite_error(h, words[1]);  // read_cube fails first
    if (words[0] == ~0ull) return HSAD_OK;
    // a pixel failed: its row chunk again, synchronously, for the reference message
    const int64_t row = failure_pixel(words[0]) / samples;
    const int64_t a = row / quantum * quantum;
    const int64_t b = a + quantum < lines ? a + quantum : lines;
    hsad_detect_request part[kMaxCallRequests];
    for (int q = 0; q < n_requests; ++q) {
        part[q] = dev_req[q];
        const int sb = dev_req[q].score_bytes;
        part[q].d_scores = static_cast<char*>(dev_req[q].d_scores) + a * row_px * sb;
        if (part[q].d_eigcount) part[q].d_eigcount += a * row_px;
    }
    st = detect_multi_impl(c.reduced.p, 8, lines, samples, target_bands, 0, lines, a, b, part, n_requests,
                           nullptr, err, s);
    return st != HSAD_OK ? st : set_error(HSAD_E_CUDA, "pipeline: failing pixel not reproduced");
}
