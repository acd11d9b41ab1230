// hsad_pipeline_sharded: one process drives G GPUs. The image splits
// into row strips aligned to hsad_row_quantum (so every pixel's arithmetic, and map, is
// the one a single-GPU run produces). Strips are dealt to the devices in contiguous
// blocks, so each device owns one row range; a host thread per device runs the same
// streamed pipeline as hsad_pipeline_host on that range (pipeline.cu: H2D of the
// range's buffer rows, strip + reflected window halo, overlapped with the reduction,
// the fused detectors and the D2H of the finished map rows) with the device's
// persistent buffers and streams, writing its rows straight into the caller's host
// maps: with host outputs no collective is needed, each GPU uses its own PCIe link.
// Device-resident maps are gathered to a root rank with hsad_gather_maps (NCCL).
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "hsad_internal.h"

namespace hsad_b200 {
int64_t row_quantum(int64_t lines, int64_t samples);
hsad_status pipeline_rows_device(int device, const float* h_cube, int64_t lines, int64_t samples,
                                 int32_t bands, int32_t order, int32_t target_bands,
                                 const hsad_detect_request* host_requests, int32_t n_requests,
                                 int64_t row0, int64_t row1, hsad_pixel_error* err,
                                 unsigned long long* fail);
}  // namespace hsad_b200

using namespace hsad_b200;

namespace {

struct RangeResult {
    hsad_status status = HSAD_OK;
    hsad_pixel_error err{HSAD_OK, -1, -1};
    unsigned long long fail = ~0ull;
    std::string message;
};

}  // namespace

extern "C" hsad_status hsad_strip_plan(int64_t lines, int64_t samples, int32_t world, int32_t rank,
                                       int64_t* row0, int64_t* row1, int64_t* strip_rows) {
    if (world < 1 || rank < 0 || rank >= world)
        return set_error(HSAD_E_INVALID_VALUE, "rank outside [0, world)");
    if (lines < 0 || samples < 0) return set_error(HSAD_E_INVALID_VALUE, "negative cube extent");
    const int64_t q = row_quantum(lines, samples);
    const int64_t per = (lines + static_cast<int64_t>(world) * q - 1) / (static_cast<int64_t>(world) * q) * q;
    const int64_t a = rank * per < lines ? rank * per : lines;
    const int64_t b = (rank + 1) * per < lines ? (rank + 1) * per : lines;
    if (row0) *row0 = a;
    if (row1) *row1 = b;
    if (strip_rows) *strip_rows = per;
    return HSAD_OK;
}

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
    // strips of the row quantum (bit-identical maps at any strip count), dealt to the
    // devices in contiguous blocks: device d owns strips [d k, (d + 1) k)
    int64_t per = 0;
    hsad_strip_plan(lines, samples, n_strips, 0, nullptr, nullptr, &per);
    const int used = n_strips < ndev ? n_strips : ndev;
    const int64_t k = (n_strips + used - 1) / used;
    std::vector<RangeResult> res(used);
    std::vector<std::thread> threads;
    for (int d = 0; d < used; ++d) {
        const int64_t r0 = d * k * per < lines ? d * k * per : lines;
        const int64_t r1 = (d + 1) * k * per < lines ? (d + 1) * k * per : lines;
        if (r1 <= r0) continue;
        threads.emplace_back([=, &res] {
            RangeResult& out = res[d];
            out.status = pipeline_rows_device(d, h_cube, lines, samples, bands, order, target_bands,
                                              host_requests, n_requests, r0, r1, &out.err, &out.fail);
            if (out.status != HSAD_OK) out.message = hsad_last_error_message();
        });
    }
    for (auto& t : threads) t.join();
    // report like one sequential call: a device failure first (in device order), else the
    // first failing request at its first pixel (the minimum packed failure word)
    int pick = -1;
    for (int d = 0; d < used; ++d)
        if (res[d].status != HSAD_OK && res[d].fail == ~0ull) {
            pick = d;
            break;
        }
    if (pick < 0)
        for (int d = 0; d < used; ++d)
            if (res[d].status != HSAD_OK && (pick < 0 || res[d].fail < res[pick].fail)) pick = d;
    if (pick < 0) return HSAD_OK;
    if (err) *err = res[pick].err;
    const std::string& m = res[pick].message;
    const size_t colon = m.find(": ");
    return set_error(res[pick].status, colon == std::string::npos ? m : m.substr(colon + 2));
}
