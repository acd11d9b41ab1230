// Two small data-parallel pieces of the reference's detector surface that are not
// detectors themselves:
//   * dual_window_samples (detect.cpp:150-157; gather_box / gather_annulus,
//     detect.cpp:83-117): the inner-box and annulus sample sets of one pixel, in the
//     reference's row-major scan order with mirror_index reflection;
//   * the fp32 little-endian payload of save_score_map (detect.cpp:291-318).
#include "hsad_internal.h"

namespace hsad_b200 {
namespace {

// One thread per (outer-window position, band). Position p = (dr, dc) in row-major order
// over the outer box; positions inside the inner box go to the inner set (in the inner
// box's own row-major order), the others to the annulus in scan order, i.e. at p minus the
// number of inner-box positions scanned before p.
template <typename T>
__global__ void window_samples_kernel(const T* __restrict__ cube, int64_t lines, int64_t samples, int bands,
                                      int64_t row, int64_t col, int inner, int outer,
                                      double* __restrict__ d_inner, double* __restrict__ d_outer) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = static_cast<int64_t>(outer) * outer * bands;
    if (e >= total) return;
    const int b = static_cast<int>(e % bands);
    const int p = static_cast<int>(e / bands);
    const int oh = outer / 2, ih = inner / 2;
    const int dr = p / outer - oh, dc = p % outer - oh;
    const int64_t rr = mirror_index(row + dr, lines), cc = mirror_index(col + dc, samples);
    const double v = static_cast<double>(cube[(rr * samples + cc) * bands + b]);
    const bool in_hole = abs(dr) <= ih && abs(dc) <= ih;
    if (in_hole) {
        d_inner[(static_cast<int64_t>(dr + ih) * inner + (dc + ih)) * bands + b] = v;
    } else {
        // inner-box positions before p: whole hole rows above dr, plus this row's hole when
        // the scan has passed it
        int before = min(max(dr + ih, 0), inner) * inner;
        if (abs(dr) <= ih && dc > ih) before += inner;
        d_outer[static_cast<int64_t>(p - before) * bands + b] = v;
    }
}

template <typename T>
__global__ void encode_f32le_kernel(const T* __restrict__ scores, int64_t n, float* __restrict__ out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = static_cast<float>(scores[i]);  // the device is little-endian, like the file
}

}  // namespace
}  // namespace hsad_b200

using namespace hsad_b200;

extern "C" {

hsad_status hsad_dual_window_samples(const void* d_cube, int32_t elem_bytes, int64_t lines, int64_t samples,
                                     int32_t bands, int64_t row, int64_t col, const hsad_window* window,
                                     double* d_inner, double* d_outer, void* stream) {
    if (!window) return set_error(HSAD_E_INVALID_VALUE, "null window");
    if (const hsad_status st = window_validate(*window); st != HSAD_OK) return st;
    if (window->mode != HSAD_WINDOW_DUAL)
        return set_error(HSAD_E_CONFIG_MISMATCH, "dual_window_samples requires a dual window");
    if (elem_bytes != 4 && elem_bytes != 8) return set_error(HSAD_E_INVALID_VALUE, "elem_bytes must be 4 or 8");
    if (lines < 1 || samples < 1 || bands < 1 || !d_cube || !d_inner || !d_outer)
        return set_error(HSAD_E_INVALID_VALUE, "null buffer or empty cube");
    if (row < 0 || row >= lines || col < 0 || col >= samples)
        return set_error(HSAD_E_INVALID_VALUE, "pixel (" + std::to_string(row) + ", " + std::to_string(col) +
                                                   ") is outside the cube");
    if (hsad_device_check() != HSAD_OK) return HSAD_E_CUDA;
    const int64_t total = static_cast<int64_t>(window->outer_size) * window->outer_size * bands;
    const int nt = 256;
    const unsigned grid = static_cast<unsigned>((total + nt - 1) / nt);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (elem_bytes == 8)
        window_samples_kernel<double><<<grid, nt, 0, s>>>(static_cast<const double*>(d_cube), lines, samples, bands,
                                                          row, col, window->inner_size, window->outer_size,
                                                          d_inner, d_outer);
    else
        window_samples_kernel<float><<<grid, nt, 0, s>>>(static_cast<const float*>(d_cube), lines, samples, bands,
                                                         row, col, window->inner_size, window->outer_size,
                                                         d_inner, d_outer);
    HSAD_CUDA_TRY(cudaGetLastError());
    return HSAD_OK;
}

hsad_status hsad_encode_score_map(const void* d_scores, int32_t score_bytes, int64_t n, void* d_raw,
                                  void* stream) {
    if (score_bytes != 4 && score_bytes != 8) return set_error(HSAD_E_INVALID_VALUE, "score_bytes must be 4 or 8");
    if (n < 0 || (n > 0 && (!d_scores || !d_raw))) return set_error(HSAD_E_INVALID_VALUE, "null buffer");
    if (hsad_device_check() != HSAD_OK) return HSAD_E_CUDA;
    if (n == 0) return HSAD_OK;
    const int nt = 256;
    const int64_t want = (n + nt - 1) / nt;
    const unsigned grid = static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (score_bytes == 8)
        encode_f32le_kernel<double><<<grid, nt, 0, s>>>(static_cast<const double*>(d_scores), n,
                                                        static_cast<float*>(d_raw));
    else
        encode_f32le_kernel<float><<<grid, nt, 0, s>>>(static_cast<const float*>(d_scores), n,
                                                       static_cast<float*>(d_raw));
    HSAD_CUDA_TRY(cudaGetLastError());
    return HSAD_OK;
}

}  // extern "C"
