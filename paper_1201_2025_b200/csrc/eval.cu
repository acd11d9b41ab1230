// Evaluation of score maps on the device (proj/core/src/eval.cpp):
//
//   hsad_roc                 roc_curve (eval.cpp:10-57): exact integer AUC, optional points
//   hsad_top_k               the k highest-scoring pixels (the parity gate's top-k sets)
//   hsad_adaptive_threshold  adaptive_threshold (eval.cpp:69-90)
//   hsad_render_pgm          render_pgm's min-max stretch (eval.cpp:92-109)
//
// Scores are mapped to order-preserving 64-bit keys (IEEE bits with the sign
// folded; -0.0 == 0.0 as the reference's == comparison treats them), so every
// comparison is an integer one and the results are exact.
//
// AUC without a full sort: the reference's numerator sum_steps fp_step (2 tp_before
// + tp_step) equals, summed per negative pixel, 2 #{positives scoring higher} +
// #{positives scoring equal}. The positives (0.1-0.2% of a scene) are compacted
// and sorted (bitonic, in HBM), a shared-memory splitter table narrows each
// negative's two binary searches, and the per-negative counts reduce into one
// 64-bit integer. The ROC points need every distinct score in descending order:
// they use a device radix sort of all keys (CUB, the CUDA toolkit's library
// sort) and per-distinct-value counts from the sorted positives.
//
// Top-k: an 8-pass radix select (8-bit digits, shared-memory histograms) finds
// the k-th largest key; a scan-ordered compaction writes the selected indices in
// ascending order, ties at the k-th value going to the lowest indices.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "hsad_internal.h"

namespace hsad_b200 {
namespace {

__device__ __forceinline__ uint64_t okey(double s) {
    if (s == 0.0) s = 0.0;  // -0.0 ties with +0.0
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double score_at(const void* p, int bytes, int64_t i) {
    return bytes == 8 ? __ldg(static_cast<const double*>(p) + i)
                      : static_cast<double>(__ldg(static_cast<const float*>(p) + i));
}

constexpr int kThreads = 256;
unsigned grid_for(int64_t n) {
    const int64_t b = (n + kThreads - 1) / kThreads;
    return static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(b, 1), 148 * 8));
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// positives count
__global__ void count_positive_kernel(const uint8_t* __restrict__ truth, int64_t n,
                                      unsigned long long* out) {
    unsigned long long c = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        c += truth[i] != 0;
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// positive keys -> keys[0..k) (any order), pad [k, kp) with UINT64_MAX
__global__ void compact_positive_kernel(const void* __restrict__ scores, int bytes,
                                        const uint8_t* __restrict__ truth, int64_t n,
                                        uint64_t* keys, unsigned long long* cursor) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (truth[i]) keys[atomicAdd(cursor, 1ull)] = okey(score_at(scores, bytes, i));
}
__global__ void fill_kernel(uint64_t* keys, int64_t from, int64_t to, uint64_t v) {
    for (int64_t i = from + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < to;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        keys[i] = v;
}

// one bitonic compare-exchange step over a power-of-two array (ascending)
__global__ void bitonic_step_kernel(uint64_t* keys, int64_t n, int64_t j, int64_t k) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t l = i ^ j;
        if (l > i) {
            const uint64_t a = keys[i], b = keys[l];
            const bool up = (i & k) == 0;
            if ((a > b) == up) {
                keys[i] = b;
                keys[l] = a;
            }
        }
    }
}

// bitonic steps with stride j < 2 * kThreads, fused through shared memory
__global__ void bitonic_local_kernel(uint64_t* keys, int64_t k, int64_t jmax) {
    __shared__ uint64_t s[2 * kThreads];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * 2 * kThreads;
    s[threadIdx.x] = keys[base + threadIdx.x];
    s[threadIdx.x + kThreads] = keys[base + threadIdx.x + kThreads];
    __syncthreads();
    for (int64_t j = jmax; j > 0; j >>= 1) {
        // thread t handles the pair (i, i ^ j) with i the lower index
        const int t = threadIdx.x;
        const int64_t lo = (t / j) * 2 * j + (t % j);
        const int64_t i = base + lo;
        const uint64_t a = s[lo], b = s[lo + j];
        const bool up = (i & k) == 0;
        if ((a > b) == up) {
            s[lo] = b;
            s[lo + j] = a;
        }
        __syncthreads();
    }
    keys[base + threadIdx.x] = s[threadIdx.x];
    keys[base + threadIdx.x + kThreads] = s[threadIdx.x + kThreads];
}

void bitonic_sort(uint64_t* keys, int64_t n_pow2, cudaStream_t s) {
    const unsigned g = grid_for(n_pow2);
    for (int64_t k = 2; k <= n_pow2; k <<= 1) {
        int64_t j = k >> 1;
        for (; j >= 2 * kThreads; j >>= 1) bitonic_step_kernel<<<g, kThreads, 0, s>>>(keys, n_pow2, j, k);
        if (n_pow2 >= 2 * kThreads) {
            bitonic_local_kernel<<<static_cast<unsigned>(n_pow2 / (2 * kThreads)), kThreads, 0, s>>>(keys, k, j);
        } else {
            for (; j > 0; j >>= 1) bitonic_step_kernel<<<g, kThreads, 0, s>>>(keys, n_pow2, j, k);
        }
    }
}

constexpr int kSplit = 4096;  // splitter table entries in shared memory

// lower_bound / upper_bound of key in sorted[0..k) using splitters spl[i] = sorted[i*step]
__device__ __forceinline__ int64_t bound(const uint64_t* __restrict__ sorted, int64_t k,
                                         const uint64_t* spl, int nspl, int64_t step, uint64_t key,
                                         bool upper) {
    // first splitter index with spl > key (upper) / >= key (lower)
    int lo = 0, hi = nspl;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const bool go_right = upper ? spl[mid] <= key : spl[mid] < key;
        if (go_right) lo = mid + 1;
        else hi = mid;
    }
    // answer lies in ((lo-1)*step, lo*step]
    int64_t a = lo == 0 ? 0 : static_cast<int64_t>(lo - 1) * step + 1;
    int64_t b = lo >= nspl ? k : static_cast<int64_t>(lo) * step;
    if (lo == 0) b = 0;
    while (a < b) {
        const int64_t mid = (a + b) >> 1;
        const uint64_t v = __ldg(sorted + mid);
        const bool go_right = upper ? v <= key : v < key;
        if (go_right) a = mid + 1;
        else b = mid;
    }
    return a;
}

__global__ void __launch_bounds__(kThreads)
    auc_count_kernel(const void* __restrict__ scores, int bytes, const uint8_t* __restrict__ truth,
                     int64_t n, const uint64_t* __restrict__ sorted, int64_t k,
                     unsigned long long* num) {
    __shared__ uint64_t spl[kSplit];
    const int64_t step = (k + kSplit - 1) / kSplit;
    const int nspl = static_cast<int>((k + step - 1) / step);
    for (int i = threadIdx.x; i < nspl; i += blockDim.x) spl[i] = sorted[static_cast<int64_t>(i) * step];
    __syncthreads();
    unsigned long long acc = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (truth[i]) continue;
        const uint64_t key = okey(score_at(scores, bytes, i));
        const int64_t lb = bound(sorted, k, spl, nspl, step, key, false);
        const int64_t ub = bound(sorted, k, spl, nspl, step, key, true);
        acc += 2ull * static_cast<unsigned long long>(k - ub) + static_cast<unsigned long long>(ub - lb);
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(num, acc);
}

__global__ void keys_kernel(const void* __restrict__ scores, int bytes, int64_t n, uint64_t* keys) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        keys[i] = okey(score_at(scores, bytes, i));
}

// sorted descending keys: head flags of distinct runs
__global__ void run_heads_kernel(const uint64_t* __restrict__ desc, int64_t n, uint32_t* head) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        head[i] = (i == 0 || desc[i] != desc[i - 1]) ? 1u : 0u;
}
// per run (segment): total count and positives at that value
__global__ void run_counts_kernel(const uint64_t* __restrict__ desc, int64_t n,
                                  const uint32_t* __restrict__ head, const uint64_t* __restrict__ run_of,
                                  const uint64_t* __restrict__ sorted_pos, int64_t k,
                                  unsigned long long* tp_step, unsigned long long* fp_step) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!head[i]) continue;
        const uint64_t key = desc[i];
        // run end: next head (runs are contiguous); binary search the run length
        int64_t a = i + 1, b = n;
        while (a < b) {
            const int64_t m = (a + b) >> 1;
            if (desc[m] == key) a = m + 1;
            else b = m;
        }
        const int64_t cnt = a - i;
        int64_t lo = 0, hi = k;  // lower bound in ascending sorted positives
        while (lo < hi) {
            const int64_t m = (lo + hi) >> 1;
            if (sorted_pos[m] < key) lo = m + 1;
            else hi = m;
        }
        int64_t up = lo, hi2 = k;
        while (up < hi2) {
            const int64_t m = (up + hi2) >> 1;
            if (sorted_pos[m] <= key) up = m + 1;
            else hi2 = m;
        }
        const int64_t tp = up - lo;
        const uint64_t r = run_of[i];
        tp_step[r] = static_cast<unsigned long long>(tp);
        fp_step[r] = static_cast<unsigned long long>(cnt - tp);
    }
}
// points[j+1] = (fp_cum / negatives, tp_cum / positives), eval.cpp:49-50
__global__ void roc_points_kernel(const unsigned long long* tp_cum, const unsigned long long* fp_cum,
                                  int64_t runs, double pos, double neg, double* far, double* td) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= runs;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i == 0) {
            far[0] = 0.0;
            td[0] = 0.0;
        } else {
            far[i] = static_cast<double>(fp_cum[i - 1]) / neg;
            td[i] = static_cast<double>(tp_cum[i - 1]) / pos;
        }
    }
}

// ---- top-k radix select ----
__global__ void __launch_bounds__(kThreads)
    select_hist_kernel(const void* __restrict__ scores, int bytes, int64_t n, uint64_t prefix,
                       uint64_t prefix_mask, int shift, unsigned long long* hist) {
    __shared__ unsigned int h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t key = okey(score_at(scores, bytes, i));
        if ((key & prefix_mask) == prefix) atomicAdd(&h[(key >> shift) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(h[i]));
}

// per-block counts of (key > kth) and (key == kth) over fixed index ranges
__global__ void __launch_bounds__(kThreads)
    select_count_kernel(const void* __restrict__ scores, int bytes, int64_t n, uint64_t kth,
                        int64_t per_block, unsigned long long* gt, unsigned long long* eq) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * per_block;
    const int64_t b = n < a + per_block ? n : a + per_block;
    unsigned long long g = 0, e = 0;
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
        const uint64_t key = okey(score_at(scores, bytes, i));
        g += key > kth;
        e += key == kth;
    }
    __shared__ unsigned long long sg[kThreads / 32], se[kThreads / 32];
    g = warp_sum(g);
    e = warp_sum(e);
    if ((threadIdx.x & 31) == 0) {
        sg[threadIdx.x >> 5] = g;
        se[threadIdx.x >> 5] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tg = 0, te = 0;
        for (int w = 0; w < kThreads / 32; ++w) {
            tg += sg[w];
            te += se[w];
        }
        gt[blockIdx.x] = tg;
        eq[blockIdx.x] = te;
    }
}

// write the selected indices in ascending order: position = greater_before +
// min(ties_before, ties_needed); block offsets are exclusive scans of the counts
__global__ void __launch_bounds__(kThreads)
    select_write_kernel(const void* __restrict__ scores, int bytes, int64_t n, uint64_t kth,
                        int64_t per_block, const unsigned long long* gt_off,
                        const unsigned long long* eq_off, unsigned long long ties_needed,
                        int64_t* out) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * per_block;
    const int64_t b = n < a + per_block ? n : a + per_block;
    unsigned long long g_run = gt_off[blockIdx.x], e_run = eq_off[blockIdx.x];
    __shared__ unsigned int wg[kThreads / 32], we[kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = a; base < b; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        bool isg = false, ise = false;
        if (i < b) {
            const uint64_t key = okey(score_at(scores, bytes, i));
            isg = key > kth;
            ise = key == kth;
        }
        const unsigned mg = __ballot_sync(0xffffffffu, isg), me = __ballot_sync(0xffffffffu, ise);
        if (lane == 0) {
            wg[warp] = __popc(mg);
            we[warp] = __popc(me);
        }
        __syncthreads();
        unsigned long long gb = g_run, eb = e_run;
        for (int w = 0; w < warp; ++w) {
            gb += wg[w];
            eb += we[w];
        }
        const unsigned lower = (1u << lane) - 1u;
        gb += __popc(mg & lower);
        eb += __popc(me & lower);
        if (isg) out[gb + (eb < ties_needed ? eb : ties_needed)] = i;
        if (ise && eb < ties_needed) out[gb + eb] = i;
        unsigned long long tg = 0, te = 0;
        for (int w = 0; w < kThreads / 32; ++w) {
            tg += wg[w];
            te += we[w];
        }
        g_run += tg;
        e_run += te;
        __syncthreads();
    }
}

// ---- threshold / pgm ----
__device__ __forceinline__ void two_sum(double& s, double& c, double x) {
    const double t = s + x;
    const double bp = t - s;
    c += (s - (t - bp)) + (x - bp);
    s = t;
}
// per-block compensated partial sums of f(s) = s (mode 0) or (s - mean)^2 (mode 1)
__global__ void __launch_bounds__(kThreads)
    moment_kernel(const void* __restrict__ scores, int bytes, int64_t n, double mean, int mode,
                  double* partial_hi, double* partial_lo) {
    double s = 0.0, c = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = score_at(scores, bytes, i);
        two_sum(s, c, mode == 0 ? v : (v - mean) * (v - mean));
    }
    __shared__ double sh[kThreads], sl[kThreads];
    sh[threadIdx.x] = s;
    sl[threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x == 0) {  // fixed-order block combine (deterministic)
        double bs = 0.0, bc = 0.0;
        for (int t = 0; t < kThreads; ++t) {
            two_sum(bs, bc, sh[t]);
            bc += sl[t];
        }
        partial_hi[blockIdx.x] = bs;
        partial_lo[blockIdx.x] = bc;
    }
}
__global__ void mask_kernel(const void* __restrict__ scores, int bytes, int64_t n, double tau,
                            uint8_t* mask) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        mask[i] = score_at(scores, bytes, i) > tau ? 1 : 0;
}
__global__ void __launch_bounds__(kThreads)
    minmax_kernel(const void* __restrict__ scores, int bytes, int64_t n, unsigned long long* kmin,
                  unsigned long long* kmax) {
    uint64_t lo = ~0ull, hi = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t k = okey(score_at(scores, bytes, i));
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(kmin, static_cast<unsigned long long>(lo));
        atomicMax(kmax, static_cast<unsigned long long>(hi));
    }
}
__global__ void pgm_kernel(const void* __restrict__ scores, int bytes, int64_t n, double lo, double scale,
                           int stretch, uint8_t* px) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        px[i] = stretch ? static_cast<uint8_t>(lround((score_at(scores, bytes, i) - lo) * scale)) : 0;
}

// RAII device scratch on a stream
struct Scratch {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    template <typename T>
    T* get(size_t count) {
        void* p = nullptr;
        if (scratch_alloc(&p, std::max<size_t>(count, 1) * sizeof(T), s) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Scratch() {
        for (void* p : ptrs) scratch_free(p, s);
    }
};

hsad_status check_scores(const void* d, int32_t bytes, int64_t n) {
    if (bytes != 8 && bytes != 4) return set_error(HSAD_E_INVALID_VALUE, "score_bytes must be 8 or 4");
    if (n < 0) return set_error(HSAD_E_INVALID_VALUE, "negative length");
    if (n > 0 && !d) return set_error(HSAD_E_INVALID_VALUE, "null score buffer");
    return HSAD_OK;
}

}  // namespace
}  // namespace hsad_b200

using namespace hsad_b200;

#define HSAD_TRY_CUDA_EVAL(expr)                                          \
    do {                                                                  \
        cudaError_t e__ = (expr);                                         \
        if (e__ != cudaSuccess) return cuda_fail(e__, #expr);             \
    } while (0)

extern "C" hsad_status hsad_roc(const void* d_scores, int32_t score_bytes, const uint8_t* d_truth,
                                int64_t n, hsad_roc_summary* out, double* d_far, double* d_td,
                                int64_t points_capacity, void* stream) {
    hsad_status st = check_scores(d_scores, score_bytes, n);
    if (st != HSAD_OK) return st;
    if (!out || (n > 0 && !d_truth)) return set_error(HSAD_E_INVALID_VALUE, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch sc(s);
    unsigned long long* cnt = sc.get<unsigned long long>(2);
    if (!cnt) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    HSAD_TRY_CUDA_EVAL(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s));
    if (n > 0) count_positive_kernel<<<grid_for(n), kThreads, 0, s>>>(d_truth, n, cnt);
    unsigned long long h[2] = {0, 0};
    HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    const uint64_t positives = h[0], negatives = static_cast<uint64_t>(n) - h[0];
    if (positives == 0 || negatives == 0)  // eval.cpp:20-21
        return set_error(HSAD_E_DEGENERATE_TRUTH, "truth mask must contain both classes");
    const int64_t k = static_cast<int64_t>(positives);
    int64_t kp = 1;
    while (kp < k) kp <<= 1;
    if (kp < 2 * kThreads) kp = 2 * kThreads;
    uint64_t* pos = sc.get<uint64_t>(kp);
    if (!pos) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    HSAD_TRY_CUDA_EVAL(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s));
    compact_positive_kernel<<<grid_for(n), kThreads, 0, s>>>(d_scores, score_bytes, d_truth, n, pos, cnt);
    fill_kernel<<<grid_for(kp - k), kThreads, 0, s>>>(pos, k, kp, ~0ull);
    bitonic_sort(pos, kp, s);
    auc_count_kernel<<<grid_for(n), kThreads, 0, s>>>(d_scores, score_bytes, d_truth, n, pos, k, cnt + 1);
    HSAD_TRY_CUDA_EVAL(cudaGetLastError());
    HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    out->positives = positives;
    out->negatives = negatives;
    out->auc_twice_num = h[1];
    out->auc = static_cast<double>(h[1]) /
               (2.0 * static_cast<double>(positives) * static_cast<double>(negatives));
    out->distinct = 0;
    if (!d_far && !d_td) return HSAD_OK;
    if (!d_far || !d_td) return set_error(HSAD_E_INVALID_VALUE, "far and td buffers go together");

    // ROC points: all keys sorted descending (CUB radix sort), distinct runs
    uint64_t* keys = sc.get<uint64_t>(n);
    uint64_t* desc = sc.get<uint64_t>(n);
    uint32_t* head = sc.get<uint32_t>(n);
    uint64_t* run_of = sc.get<uint64_t>(n);
    if (!keys || !desc || !head || !run_of) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    keys_kernel<<<grid_for(n), kThreads, 0, s>>>(d_scores, score_bytes, n, keys);
    size_t tmp_bytes = 0;
    HSAD_TRY_CUDA_EVAL(cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp_bytes, keys, desc,
                                                                static_cast<int64_t>(n), 0, 64, s));
    size_t scan_bytes = 0;
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, head, run_of, n, s));
    void* tmp = sc.get<char>(std::max(tmp_bytes, scan_bytes));
    if (!tmp) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    HSAD_TRY_CUDA_EVAL(cub::DeviceRadixSort::SortKeysDescending(tmp, tmp_bytes, keys, desc,
                                                                static_cast<int64_t>(n), 0, 64, s));
    run_heads_kernel<<<grid_for(n), kThreads, 0, s>>>(desc, n, head);
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, head, run_of, n, s));
    uint64_t last_run = 0;
    uint32_t last_head = 0;
    HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(&last_run, run_of + n - 1, sizeof(last_run), cudaMemcpyDeviceToHost, s));
    HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(&last_head, head + n - 1, sizeof(last_head), cudaMemcpyDeviceToHost, s));
    HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    const int64_t runs = static_cast<int64_t>(last_run + last_head);
    out->distinct = static_cast<uint64_t>(runs);
    if (points_capacity < runs + 1)
        return set_error(HSAD_E_OUT_OF_BOUNDS, "ROC needs " + std::to_string(runs + 1) +
                                                   " points, buffers hold " +
                                                   std::to_string(points_capacity));
    unsigned long long* tp_step = sc.get<unsigned long long>(runs);
    unsigned long long* fp_step = sc.get<unsigned long long>(runs);
    unsigned long long* tp_cum = sc.get<unsigned long long>(runs);
    unsigned long long* fp_cum = sc.get<unsigned long long>(runs);
    if (!tp_step || !fp_step || !tp_cum || !fp_cum) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    run_counts_kernel<<<grid_for(n), kThreads, 0, s>>>(desc, n, head, run_of, pos, k, tp_step, fp_step);
    size_t s2 = 0;
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::InclusiveSum(nullptr, s2, tp_step, tp_cum, runs, s));
    void* tmp2 = sc.get<char>(s2);
    if (!tmp2) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::InclusiveSum(tmp2, s2, tp_step, tp_cum, runs, s));
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::InclusiveSum(tmp2, s2, fp_step, fp_cum, runs, s));
    roc_points_kernel<<<grid_for(runs + 1), kThreads, 0, s>>>(tp_cum, fp_cum, runs,
                                                              static_cast<double>(positives),
                                                              static_cast<double>(negatives), d_far, d_td);
    HSAD_TRY_CUDA_EVAL(cudaGetLastError());
    HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    return HSAD_OK;
}

extern "C" hsad_status hsad_top_k(const void* d_scores, int32_t score_bytes, int64_t n, int64_t k,
                                  int64_t* d_indices, double* kth, void* stream) {
    hsad_status st = check_scores(d_scores, score_bytes, n);
    if (st != HSAD_OK) return st;
    if (k < 1 || k > n)
        return set_error(HSAD_E_INVALID_VALUE, "k must be in [1, " + std::to_string(n) + "], got " +
                                                   std::to_string(k));
    if (!d_indices) return set_error(HSAD_E_INVALID_VALUE, "null index buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch sc(s);
    unsigned long long* hist = sc.get<unsigned long long>(256);
    if (!hist) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    // radix select, most significant digit first: the k-th largest key
    uint64_t prefix = 0, mask = 0;
    unsigned long long need = static_cast<unsigned long long>(k);  // rank within the prefix, from the top
    for (int shift = 56; shift >= 0; shift -= 8) {
        HSAD_TRY_CUDA_EVAL(cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), s));
        select_hist_kernel<<<grid_for(n), kThreads, 0, s>>>(d_scores, score_bytes, n, prefix, mask, shift, hist);
        unsigned long long hh[256];
        HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, s));
        HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
        int d = 255;
        for (; d > 0; --d) {
            if (hh[d] >= need) break;
            need -= hh[d];
        }
        prefix |= static_cast<uint64_t>(d) << shift;
        mask |= 0xffull << shift;
    }
    const uint64_t kth_key = prefix;
    // selected = all keys > kth plus the first `need` keys == kth in index order
    const int64_t per_block = 4096;
    const int64_t blocks = (n + per_block - 1) / per_block;
    unsigned long long* gt = sc.get<unsigned long long>(blocks);
    unsigned long long* eq = sc.get<unsigned long long>(blocks);
    unsigned long long* gt_off = sc.get<unsigned long long>(blocks);
    unsigned long long* eq_off = sc.get<unsigned long long>(blocks);
    if (!gt || !eq || !gt_off || !eq_off) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    select_count_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(d_scores, score_bytes, n, kth_key,
                                                                           per_block, gt, eq);
    size_t tb = 0;
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::ExclusiveSum(nullptr, tb, gt, gt_off, blocks, s));
    void* tmp = sc.get<char>(tb);
    if (!tmp) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::ExclusiveSum(tmp, tb, gt, gt_off, blocks, s));
    HSAD_TRY_CUDA_EVAL(cub::DeviceScan::ExclusiveSum(tmp, tb, eq, eq_off, blocks, s));
    select_write_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(
        d_scores, score_bytes, n, kth_key, per_block, gt_off, eq_off, need, d_indices);
    HSAD_TRY_CUDA_EVAL(cudaGetLastError());
    HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    if (kth) {
        // okey -> double (sign-folded inverse)
        const uint64_t b = (kth_key >> 63) ? (kth_key & 0x7fffffffffffffffull) : ~kth_key;
        double v;
        std::memcpy(&v, &b, sizeof(v));
        *kth = v;
    }
    return HSAD_OK;
}

extern "C" hsad_status hsad_adaptive_threshold(const void* d_scores, int32_t score_bytes, int64_t n,
                                               double z_alpha, double* tau, uint8_t* d_mask,
                                               void* stream) {
    hsad_status st = check_scores(d_scores, score_bytes, n);
    if (st != HSAD_OK) return st;
    if (n == 0) return set_error(HSAD_E_INVALID_VALUE, "cannot threshold an empty score map");
    if (!tau) return set_error(HSAD_E_INVALID_VALUE, "null tau");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch sc(s);
    const unsigned g = grid_for(n);
    double* hi = sc.get<double>(g);
    double* lo = sc.get<double>(g);
    if (!hi || !lo) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    std::vector<double> hh(g), hl(g);
    auto total = [&](int mode, double mean, double& out_sum) -> hsad_status {
        moment_kernel<<<g, kThreads, 0, s>>>(d_scores, score_bytes, n, mean, mode, hi, lo);
        HSAD_TRY_CUDA_EVAL(cudaGetLastError());
        HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(hh.data(), hi, g * sizeof(double), cudaMemcpyDeviceToHost, s));
        HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(hl.data(), lo, g * sizeof(double), cudaMemcpyDeviceToHost, s));
        HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
        double a = 0.0, c = 0.0;
        for (unsigned i = 0; i < g; ++i) {  // compensated, fixed order
            const double t = a + hh[i];
            const double bp = t - a;
            c += (a - (t - bp)) + (hh[i] - bp) + hl[i];
            a = t;
        }
        out_sum = a + c;
        return HSAD_OK;
    };
    const double dn = static_cast<double>(n);
    double sum = 0.0, ssq = 0.0;
    if ((st = total(0, 0.0, sum)) != HSAD_OK) return st;
    const double mean = sum / dn;
    if ((st = total(1, mean, ssq)) != HSAD_OK) return st;
    const double var = ssq / dn;  // population variance, eval.cpp:77-79
    *tau = mean + z_alpha * std::sqrt(var);
    if (d_mask) {
        mask_kernel<<<g, kThreads, 0, s>>>(d_scores, score_bytes, n, *tau, d_mask);
        HSAD_TRY_CUDA_EVAL(cudaGetLastError());
        HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    }
    return HSAD_OK;
}

extern "C" hsad_status hsad_render_pgm(const void* d_scores, int32_t score_bytes, int64_t n,
                                       uint8_t* d_pixels, void* stream) {
    hsad_status st = check_scores(d_scores, score_bytes, n);
    if (st != HSAD_OK) return st;
    if (n == 0) return HSAD_OK;
    if (!d_pixels) return set_error(HSAD_E_INVALID_VALUE, "null pixel buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch sc(s);
    unsigned long long* mm = sc.get<unsigned long long>(2);
    if (!mm) return set_error(HSAD_E_CUDA, "scratch allocation failed");
    const unsigned long long init[2] = {~0ull, 0ull};
    HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
    minmax_kernel<<<grid_for(n), kThreads, 0, s>>>(d_scores, score_bytes, n, mm, mm + 1);
    unsigned long long h[2];
    HSAD_TRY_CUDA_EVAL(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, s));
    HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    auto to_d = [](unsigned long long k) {
        const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        double v;
        std::memcpy(&v, &b, sizeof(v));
        return v;
    };
    const double lo = to_d(h[0]), hi = to_d(h[1]);
    const bool stretch = hi > lo;
    const double scale = stretch ? 255.0 / (hi - lo) : 0.0;  // eval.cpp:101-106
    pgm_kernel<<<grid_for(n), kThreads, 0, s>>>(d_scores, score_bytes, n, lo, scale, stretch ? 1 : 0, d_pixels);
    HSAD_TRY_CUDA_EVAL(cudaGetLastError());
    HSAD_TRY_CUDA_EVAL(cudaStreamSynchronize(s));
    return HSAD_OK;
}
