// Host-side entry points of the C-ABI that do not launch kernels: status names,
// last-error text, limits, window validation, mirror index, Daubechies taps and
// the composed wavelet map used by the reduction kernel.
//
// References: proj/core/src/error.cpp:5-30 (names), proj/core/src/detect.cpp:29-76
// (window validation + mirror), proj/core/src/wavelet.cpp:16-146 (taps, stage,
// padding, cascade and their error contract).
#include <bit>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "hsad_internal.h"

namespace hsad_b200 {

// Library-owned stream-ordered pools, one per device, created on first use.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (static_cast<int>(pools.size()) <= dev) pools.resize(dev + 1, nullptr);
        if (!pools[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&pools[dev], &props);
            if (e != cudaSuccess) return e;
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes > 0 ? bytes : 1, pool, s);
}

void scratch_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

namespace {

thread_local std::string g_last_error;

// Daubechies scaling taps h[n], orders 1..10: the standard published
// minimal-phase constants normalised to sum sqrt(2) (the same constants the
// reference tabulates at proj/core/src/wavelet.cpp:16-49).
const double kTaps1[] = {0.70710678118654752, 0.70710678118654752};
const double kTaps2[] = {0.48296291314453414, 0.83651630373780791, 0.22414386804201338,
                         -0.12940952255126038};
const double kTaps3[] = {0.33267055295008262, 0.80689150931109258, 0.45987750211849157,
                         -0.13501102001025459, -0.085441273882026662, 0.035226291885709537};
const double kTaps4[] = {0.23037781330889650, 0.71484657055291565, 0.63088076792985891,
                         -0.027983769416859854, -0.18703481171909308, 0.030841381835560764,
                         0.032883011666885200, -0.010597401785069032};
const double kTaps5[] = {0.16010239797419291, 0.60382926979718967, 0.72430852843777293,
                         0.13842814590132073, -0.24229488706638203, -0.032244869584638375,
                         0.077571493840045714, -0.0062414902127982743, -0.012580751999081999,
                         0.0033357252854737713};
const double kTaps6[] = {0.11154074335010946, 0.49462389039845309, 0.75113390802109535,
                         0.31525035170919763, -0.22626469396543982, -0.12976686756726194,
                         0.097501605587323049, 0.027522865530305729, -0.031582039317486030,
                         0.00055384220116149614, 0.0047772575109455106, -0.0010773010853084796};
const double kTaps7[] = {0.077852054085009179, 0.39653931948191731, 0.72913209084623512,
                         0.46978228740519312, -0.14390600392856498, -0.22403618499387498,
                         0.071309219266830265, 0.080612609151083072, -0.038029936935014414,
                         -0.016574541630666881, 0.012550998556099841, 0.00042957797292136652,
                         -0.0018016407040474909, 0.00035371379997452025};
const double kTaps8[] = {0.054415842243104010, 0.31287159091429997, 0.67563073629728981,
                         0.58535468365420671, -0.015829105256349306, -0.28401554296154693,
                         0.00047248457391328277, 0.12874742662047846, -0.017369301001807546,
                         -0.044088253930794752, 0.013981027917398282, 0.0087460940474057767,
                         -0.0048703529934515743, -0.00039174037337694705,
                         0.00067544940645056937, -0.00011747678412476953};
const double kTaps9[] = {0.038077947363878347, 0.24383467461259035, 0.60482312369011111,
                         0.65728807805130054, 0.13319738582500758, -0.29327378327917491,
                         -0.096840783222976461, 0.14854074933810638, 0.030725681479333379,
                         -0.067632829061329974, 0.00025094711483145196, 0.022361662123679097,
                         -0.0047232047577513973, -0.0042815036824634298, 0.0018476468830562265,
                         0.00023038576352319597, -0.00025196318894271014,
                         0.000039347320316271599};
const double kTaps10[] = {0.026670057900555554, 0.18817680007769149, 0.52720118893172559,
                          0.68845903945360357, 0.28117234366057746, -0.24984642432731538,
                          -0.19594627437737704, 0.12736934033579326, 0.093057364603572351,
                          -0.071394147166397087, -0.029457536821875813, 0.033212674059341002,
                          0.0036065535669561697, -0.010733175483330575, 0.0013953517470529012,
                          0.0019924052951850561, -0.00068585669495971163,
                          -0.00011646685512928545, 0.000093588670320069591,
                          -0.000013264202894521245};
const double* const kTaps[10] = {kTaps1, kTaps2, kTaps3, kTaps4, kTaps5,
                                 kTaps6, kTaps7, kTaps8, kTaps9, kTaps10};

}  // namespace

const char* status_name(int32_t code) {
    static const char* names[] = {"Ok",
                                  "MissingKey",
                                  "InvalidValue",
                                  "SizeMismatch",
                                  "NonFiniteValue",
                                  "OutOfBounds",
                                  "UnsupportedOrder",
                                  "OddLength",
                                  "TooShort",
                                  "LengthMismatch",
                                  "TargetTooLarge",
                                  "EmptySampleSet",
                                  "TooFewSamples",
                                  "SingularAfterRidge",
                                  "NotSymmetric",
                                  "NoConvergence",
                                  "ConfigMismatch",
                                  "FractionOutOfRange",
                                  "OutOfBoundsImplant",
                                  "DimensionMismatch",
                                  "DegenerateTruth",
                                  "IoFailure"};
    if (code >= 0 && code <= HSAD_E_IO_FAILURE) return names[code];
    if (code == HSAD_E_CUDA) return "CudaError";
    if (code == HSAD_E_UNSUPPORTED) return "Unsupported";
    if (code == HSAD_E_NCCL) return "NcclError";
    return "UnknownError";
}

hsad_status set_error(hsad_status code, const std::string& message) {
    g_last_error = std::string(status_name(code)) + ": " + message;
    return code;
}

hsad_status cuda_fail(cudaError_t e, const char* what) {
    return set_error(HSAD_E_CUDA, std::string(what) + " failed: " + cudaGetErrorString(e));
}

hsad_status window_validate(const hsad_window& w) {
    // proj/core/src/detect.cpp:46-64 (same messages)
    if (w.mode == HSAD_WINDOW_SINGLE) {
        if (w.single_size < 3 || w.single_size % 2 == 0)
            return set_error(HSAD_E_INVALID_VALUE, "single window size must be odd and >= 3, got " +
                                                       std::to_string(w.single_size));
        return HSAD_OK;
    }
    if (w.mode != HSAD_WINDOW_DUAL) return set_error(HSAD_E_INVALID_VALUE, "unknown window mode");
    if (w.inner_size < 1 || w.inner_size % 2 == 0)
        return set_error(HSAD_E_INVALID_VALUE, "inner window size must be odd and >= 1, got " +
                                                   std::to_string(w.inner_size));
    if (w.outer_size <= w.inner_size || w.outer_size % 2 == 0)
        return set_error(HSAD_E_INVALID_VALUE, "outer window size must be odd and > inner, got " +
                                                   std::to_string(w.outer_size));
    if (w.outer_size - w.inner_size < 2)
        return set_error(HSAD_E_INVALID_VALUE, "outer window must exceed inner by at least 2");
    if (w.outer_size * w.outer_size - w.inner_size * w.inner_size < 2)
        return set_error(HSAD_E_INVALID_VALUE, "outer annulus must contain at least 2 pixels");
    return HSAD_OK;
}

// wavelet.cpp:122-146: pad to P = bit_ceil(bands) by appending x[n-1], x[n-2], ...
// then run the low-pass stage (approx[k] = sum_j h[j] x[(2k+j) mod n]) until the
// length equals `target`. The map is linear, so it is composed once here in
// fp64 by pushing the unit vectors e_b through the exact same cascade.
hsad_status wavelet_plan(int32_t bands, int32_t order, int32_t target, std::vector<double>* map) {
    if (order < 1 || order > 10)
        return set_error(HSAD_E_UNSUPPORTED_ORDER,
                         "Daubechies order must be in 1..10, got " + std::to_string(order));
    if (target < 2 || !std::has_single_bit(static_cast<unsigned>(target)))
        return set_error(HSAD_E_INVALID_VALUE,
                         "target bands must be a power of two >= 2, got " + std::to_string(target));
    // the reference's fail-fast probe (wavelet.cpp:153-156) then raises the
    // multilevel_approx contract errors for a `bands`-long spectrum
    if (bands <= 0) return set_error(HSAD_E_TOO_SHORT, "empty signal");
    const std::size_t padded = std::bit_ceil(static_cast<std::size_t>(bands));
    if (static_cast<std::size_t>(target) > padded)
        return set_error(HSAD_E_TARGET_TOO_LARGE, "target length " + std::to_string(target) +
                                                      " exceeds padded length " +
                                                      std::to_string(padded));
    const int taps = 2 * order;
    for (std::size_t n = padded; n > static_cast<std::size_t>(target); n /= 2) {
        if (n % 2 != 0)
            return set_error(HSAD_E_ODD_LENGTH, "signal length " + std::to_string(n) + " is odd");
        if (n < static_cast<std::size_t>(taps))
            return set_error(HSAD_E_TOO_SHORT, "signal length " + std::to_string(n) +
                                                   " shorter than filter length " +
                                                   std::to_string(taps));
    }
    if (!map) return HSAD_OK;
    if (bands > kMaxReduceBands)
        return set_error(HSAD_E_UNSUPPORTED, "hsad_reduce supports at most " +
                                                 std::to_string(kMaxReduceBands) + " bands");
    const double* h = kTaps[order - 1];
    map->assign(static_cast<std::size_t>(target) * bands, 0.0);
    std::vector<double> cur(padded), next;
    for (int b = 0; b < bands; ++b) {
        std::vector<double> x(bands, 0.0);
        x[b] = 1.0;
        cur.assign(x.begin(), x.end());
        for (std::size_t k = 0; cur.size() < padded; ++k) cur.push_back(x[bands - 1 - k]);
        while (cur.size() > static_cast<std::size_t>(target)) {
            const std::size_t n = cur.size();
            next.assign(n / 2, 0.0);
            for (std::size_t k = 0; k < n / 2; ++k) {
                double a = 0.0;
                for (int j = 0; j < taps; ++j) {
                    std::size_t idx = 2 * k + j;
                    if (idx >= n) idx -= n;
                    a += h[j] * cur[idx];
                }
                next[k] = a;
            }
            cur.swap(next);
        }
        for (int k = 0; k < target; ++k) (*map)[static_cast<std::size_t>(k) * bands + b] = cur[k];
    }
    return HSAD_OK;
}

}  // namespace hsad_b200

using namespace hsad_b200;

extern "C" {

int32_t hsad_abi_version(void) { return HSAD_ABI_VERSION; }

const char* hsad_status_name(int32_t status) { return status_name(status); }

const char* hsad_last_error_message(void) { return g_last_error.c_str(); }

void hsad_get_limits(hsad_limits* out) {
    if (!out) return;
    out->max_detect_bands = 224;  // LRX/DWRX full band (fullband.cu); DWEST up to 200 (fullband_dwest.cu)
    out->max_window = 2 * kMaxRadius + 1;
    out->max_reduce_bands = kMaxReduceBands;
}

hsad_status hsad_device_check(void) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    cudaDeviceProp prop{};
    e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10)
        return set_error(HSAD_E_CUDA, "this build targets sm_100a; device is sm_" +
                                          std::to_string(prop.major * 10 + prop.minor));
    return HSAD_OK;
}

int32_t hsad_mirror_index(int32_t i, int32_t n) {
    return static_cast<int32_t>(mirror_index(i, n));
}

hsad_status hsad_window_validate(const hsad_window* window) {
    if (!window) return set_error(HSAD_E_INVALID_VALUE, "null window");
    return window_validate(*window);
}

hsad_status hsad_daubechies_filters(int32_t order, double* low, double* high, int32_t* length) {
    // proj/core/src/wavelet.cpp:60-74: high[n] = (-1)^n low[len-1-n]
    if (order < 1 || order > 10)
        return set_error(HSAD_E_UNSUPPORTED_ORDER,
                         "Daubechies order must be in 1..10, got " + std::to_string(order));
    const int len = 2 * order;
    const double* h = kTaps[order - 1];
    for (int n = 0; n < len; ++n) {
        if (low) low[n] = h[n];
        if (high) high[n] = (n % 2 == 0) ? h[len - 1 - n] : -h[len - 1 - n];
    }
    if (length) *length = len;
    return HSAD_OK;
}

hsad_status hsad_decode_status(uint64_t packed, int64_t samples, hsad_pixel_error* err) {
    if (!err) return HSAD_OK;
    if (packed == ~0ull || samples <= 0) {
        err->code = HSAD_OK;
        err->row = err->col = -1;
        return HSAD_OK;
    }
    const uint64_t lin = static_cast<uint64_t>(failure_pixel(packed));
    err->code = failure_code(packed);
    err->row = static_cast<int64_t>(lin / static_cast<uint64_t>(samples));
    err->col = static_cast<int64_t>(lin % static_cast<uint64_t>(samples));
    return static_cast<hsad_status>(err->code);
}

}  // extern "C"
