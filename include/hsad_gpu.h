/*
 * hsad_gpu.h — C-ABI of the B200-native hsad hot path (sm_100a).
 *
 * The reference ("hsad", arXiv 1201.2025) exposes its hot path only as a C++
 * library API; it has no FFI of its own. These entry points are what a
 * maintainer binds to replace it (see INTEGRATION.md for the C++ shim and the
 * ctypes binding). Each entry point names the reference interface it replaces:
 *
 *   hsad_daubechies_filters  <- hsad::daubechies_filters   proj/core/include/hsad/wavelet.hpp:24
 *                                                           (impl proj/core/src/wavelet.cpp:60-74)
 *   hsad_reduce              <- hsad::reduce_cube           proj/core/include/hsad/wavelet.hpp:55-56
 *                                                           (impl proj/core/src/wavelet.cpp:148-167)
 *   hsad_detect              <- hsad::detect / local_rx / dwrx / dwest
 *                                                           proj/core/include/hsad/detect.hpp:77-92
 *                                                           (impl proj/core/src/detect.cpp:159-289)
 *   hsad_detect_multi        <- several hsad::detect calls on one cube that share
 *                               window statistics (the fused B200 path; same per-detector
 *                               semantics as hsad_detect)
 *   hsad_reduce_detect       <- hsad::reduce_cube followed by hsad_detect_multi on the reduced
 *                               cube (device buffers, one call)
 *   hsad_pipeline_host       <- hsad::reduce_cube + hsad::detect on HOST buffers, i.e. the
 *                               `hsad reduce` + `hsad detect` CLI composition
 *                               (proj/tools/hsad_main.cpp:112-198) without file I/O
 *   hsad_mirror_index        <- hsad::mirror_index          proj/core/include/hsad/detect.hpp:68
 *   hsad_window_validate     <- hsad::WindowConfig::validate proj/core/src/detect.cpp:46-64
 *
 * Conventions
 *  - Cubes are BIP (band fastest), index (row*samples + col)*bands + band, exactly
 *    hsad::HyperCube (proj/core/include/hsad/cube.hpp:53-58). Element type is fp32
 *    (elem_bytes = 4, the on-disk type widened by the reference at load,
 *    cube.cpp:219) or fp64 (elem_bytes = 8, the HyperCube type).
 *  - Score maps are row-major (row*samples + col), like ScoreMap::scores
 *    (detect.hpp:52), stored as fp64 (score_bytes = 8, the "fp64 path") or fp32
 *    (score_bytes = 4, the "fp32 path"; the reference's .raw files are fp32,
 *    detect.cpp:291-318). All arithmetic is fp64 in both cases.
 *  - Pointers named d_* are device pointers on the current CUDA device; work is
 *    enqueued on `stream` (a cudaStream_t, 0 = legacy default stream). Pointers
 *    named h_* are host pointers.
 *  - Every call validates its arguments exactly like the reference and returns
 *    the reference's error category (hsad_status mirrors hsad::errc,
 *    proj/core/include/hsad/error.hpp:10-32, shifted by one so 0 = success).
 *    hsad_last_error_message() returns the reference-formatted message of the
 *    calling thread's last failure: "<Name>: <message>[ at pixel (r, c)]"
 *    (error.hpp:36-45, detect.cpp:127-130).
 *  - Per-pixel failures (singular covariance, ...) are reported for the first
 *    failing pixel in row-major order — the reference's workers=1 semantics
 *    (parallel.hpp:17-40).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns HSAD_E_CUDA.
 */
#ifndef HSAD_GPU_H
#define HSAD_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSAD_ABI_VERSION 1

typedef enum hsad_status {
    HSAD_OK = 0,
    /* hsad::errc + 1 (proj/core/include/hsad/error.hpp:10-32) */
    HSAD_E_MISSING_KEY = 1,
    HSAD_E_INVALID_VALUE = 2,
    HSAD_E_SIZE_MISMATCH = 3,
    HSAD_E_NON_FINITE_VALUE = 4,
    HSAD_E_OUT_OF_BOUNDS = 5,
    HSAD_E_UNSUPPORTED_ORDER = 6,
    HSAD_E_ODD_LENGTH = 7,
    HSAD_E_TOO_SHORT = 8,
    HSAD_E_LENGTH_MISMATCH = 9,
    HSAD_E_TARGET_TOO_LARGE = 10,
    HSAD_E_EMPTY_SAMPLE_SET = 11,
    HSAD_E_TOO_FEW_SAMPLES = 12,
    HSAD_E_SINGULAR_AFTER_RIDGE = 13,
    HSAD_E_NOT_SYMMETRIC = 14,
    HSAD_E_NO_CONVERGENCE = 15,
    HSAD_E_CONFIG_MISMATCH = 16,
    HSAD_E_FRACTION_OUT_OF_RANGE = 17,
    HSAD_E_OUT_OF_BOUNDS_IMPLANT = 18,
    HSAD_E_DIMENSION_MISMATCH = 19,
    HSAD_E_DEGENERATE_TRUTH = 20,
    HSAD_E_IO_FAILURE = 21,
    /* B200 path only */
    HSAD_E_CUDA = 64,        /* no device / launch or runtime failure */
    HSAD_E_UNSUPPORTED = 65, /* outside this build's kernel limits (see hsad_limits) */
    HSAD_E_NCCL = 66         /* NCCL missing or an NCCL call failed (hsad_gather_maps) */
} hsad_status;

typedef enum hsad_algorithm { /* hsad::Algorithm, detect.hpp:13 */
    HSAD_LRX = 0,
    HSAD_DWRX = 1,
    HSAD_DWEST = 2
} hsad_algorithm;

typedef enum hsad_window_mode { HSAD_WINDOW_SINGLE = 0, HSAD_WINDOW_DUAL = 1 } hsad_window_mode;

/* hsad::WindowConfig (detect.hpp:20-33): Single = one odd window (LRX),
 * Dual = inner box + outer annulus (DWRX, DWEST). */
typedef struct hsad_window {
    int32_t mode;
    int32_t single_size;
    int32_t inner_size;
    int32_t outer_size;
} hsad_window;

/* One detector request. Mirrors hsad::detect(cube, algo, window, options)
 * (detect.hpp:91-92) with DetectOptions {ridge, dwest.eigen_fraction}
 * (detect.hpp:35-45) plus two B200-path extensions:
 *   guard      LRX only: background = single_size box minus a guard x guard box
 *              centred on the pixel (1 = the reference: only the centre position
 *              is excluded, detect.cpp:83-99). Extension, unpinned by the reference.
 *   d_eigcount DWEST only, nullable: int8 per pixel = number of eigenvectors the
 *              DWEST loop summed (detect.cpp:258-262). Extension.                */
typedef struct hsad_detect_request {
    int32_t algorithm;       /* hsad_algorithm */
    hsad_window window;
    int32_t guard;           /* LRX guard box (>= 1, odd); ignored otherwise */
    double ridge;            /* LRX / DWRX ridge fraction (default 1e-6) */
    double eigen_fraction;   /* DWEST cutoff fraction in (0, 1] (default 0.1) */
    void* d_scores;          /* output rows x samples, row-major */
    int32_t score_bytes;     /* 8 = fp64, 4 = fp32 */
    int8_t* d_eigcount;      /* DWEST only, nullable */
} hsad_detect_request;

/* First failing pixel, row-major (global image coordinates). */
typedef struct hsad_pixel_error {
    int32_t code;   /* hsad_status, HSAD_OK when no pixel failed */
    int64_t row;
    int64_t col;
} hsad_pixel_error;

/* Kernel limits of this build. */
typedef struct hsad_limits {
    int32_t max_detect_bands;   /* bands accepted by hsad_detect* for LRX/DWRX (DWEST: 200) */
    int32_t max_window;         /* largest single/outer window edge */
    int32_t max_reduce_bands;   /* bands accepted by hsad_reduce */
} hsad_limits;

/* ---- library ---------------------------------------------------------------- */
int32_t hsad_abi_version(void);
const char* hsad_status_name(int32_t status);      /* errc_name, error.cpp:5-30 */
const char* hsad_last_error_message(void);          /* thread-local */
void hsad_get_limits(hsad_limits* out);
/* 0 when an sm_100-class device is usable; HSAD_E_CUDA otherwise. */
hsad_status hsad_device_check(void);

/* ---- geometry (host, no device needed) ------------------------------------- */
int32_t hsad_mirror_index(int32_t i, int32_t n);
hsad_status hsad_window_validate(const hsad_window* window);
/* low/high: >= 2*order doubles; *length = 2*order. */
hsad_status hsad_daubechies_filters(int32_t order, double* low, double* high, int32_t* length);

/* ---- wavelet reduction (reduce_cube) ---------------------------------------- */
/* d_cube: lines*samples*bands BIP (elem_bytes 4|8); d_out: lines*samples*target_bands
 * BIP (out_bytes 8|4). Filter: Daubechies `order` (1..10), target_bands a power of
 * two >= 2 and <= bit_ceil(bands). Errors exactly as wavelet.cpp:122-167. */
hsad_status hsad_reduce(const void* d_cube, int32_t elem_bytes, int64_t lines, int64_t samples,
                        int32_t bands, int32_t order, int32_t target_bands, void* d_out,
                        int32_t out_bytes, void* stream);

/* ---- detectors ---------------------------------------------------------------- */
/* Whole-image single detector: hsad::detect semantics. Synchronous (the stream is
 * synchronised to report per-pixel errors); `err` may be NULL. */
hsad_status hsad_detect(const void* d_cube, int32_t elem_bytes, int64_t lines, int64_t samples,
                        int32_t bands, const hsad_detect_request* request,
                        hsad_pixel_error* err, void* stream);

/* symmetric_eigen + the DWEST selection loop (stats.cpp:64-89, detect.cpp:252-263) on a
 * batch of n 4 x 4 symmetric matrices: d_cdiff n*16 doubles (row-major; the upper triangle
 * is read), d_mdiff n*4. d_scores[i] = |sum over {lambda_j > 0, lambda_j >= f lambda_max} of
 * v_j . m_diff| with the sign rule of stats.cpp:83-85, d_counts[i] (optional) the size of that
 * set, d_route[i] (optional) 0 when the two-pair tridiagonal route settled the matrix and 1
 * when it went through the general Jacobi route. The device code is the fused detectors'. */
hsad_status hsad_dwest_pairs(const double* d_cdiff, const double* d_mdiff, int64_t n,
                             double eigen_fraction, double* d_scores, int8_t* d_counts,
                             int8_t* d_route, void* stream);

/* dual_window_samples (detect.cpp:150-157): the inner-box and annulus sample sets of pixel
 * (row, col) in the reference's scan order (gather_box / gather_annulus, detect.cpp:83-117,
 * mirror_index reflection). d_inner: inner^2 x bands doubles, d_outer: (outer^2 - inner^2) x
 * bands doubles, sample-major (= the column-major `dimension x count` SampleSet::vectors).
 * Errors: the window's validation errors, ConfigMismatch "dual_window_samples requires a
 * dual window". */
hsad_status hsad_dual_window_samples(const void* d_cube, int32_t elem_bytes, int64_t lines,
                                     int64_t samples, int32_t bands, int64_t row, int64_t col,
                                     const hsad_window* window, double* d_inner, double* d_outer,
                                     void* stream);

/* The payload of save_score_map (detect.cpp:291-318): n scores (score_bytes 8|4) -> n
 * little-endian fp32 values, the .raw file of a 1-band ENVI BSQ data type 4 map. */
hsad_status hsad_encode_score_map(const void* d_scores, int32_t score_bytes, int64_t n, void* d_raw,
                                  void* stream);

/* Fused multi-detector over a row strip. The image is `lines` x `samples` x
 * `bands`; the buffer d_cube holds global rows [buf_row0, buf_row0 + buf_rows)
 * (row strip plus mirror halo; hsad_strip_rows() computes the range) and the
 * requests' score buffers receive output rows [row_begin, row_end). Window
 * reflection uses global coordinates, so any row split yields bit-identical maps.
 * Asynchronous: when d_status (device, 1 x uint64) is non-NULL the first failing
 * pixel is recorded there as (row*samples+col) << 8 | code (UINT64_MAX = none)
 * and the call returns without synchronising; decode it with
 * hsad_decode_status(). With d_status NULL the call synchronises and fills err. */
hsad_status hsad_detect_multi(const void* d_cube, int32_t elem_bytes, int64_t lines,
                              int64_t samples, int32_t bands, int64_t buf_row0, int64_t buf_rows,
                              int64_t row_begin, int64_t row_end,
                              const hsad_detect_request* requests, int32_t n_requests,
                              uint64_t* d_status, hsad_pixel_error* err, void* stream);

/* reduce_cube + hsad_detect_multi in one call (the `hsad reduce` + `hsad detect`
 * composition on device buffers). d_cube (fp32 BIP, `bands` bands) and d_reduced
 * (fp64 BIP, target_bands bands) both hold global rows [buf_row0, buf_row0 +
 * buf_rows); on return d_reduced holds reduce_cube of those rows and the requests'
 * maps hold rows [row_begin, row_end), bit-identical to hsad_reduce followed by
 * hsad_detect_multi. Reduction errors (wavelet.cpp:122-167) come first, then the
 * detectors' errors. Asynchrony as hsad_detect_multi (d_status). */
hsad_status hsad_reduce_detect(const float* d_cube, int64_t lines, int64_t samples, int32_t bands,
                               int32_t order, int32_t target_bands, int64_t buf_row0,
                               int64_t buf_rows, int64_t row_begin, int64_t row_end,
                               double* d_reduced, const hsad_detect_request* requests,
                               int32_t n_requests, uint64_t* d_status, hsad_pixel_error* err,
                               void* stream);

/* 1 when the calling thread's last hsad_reduce_detect folded the reduction into its first
 * detector launch (opt-in with HSAD_FUSE=1: the DWT of each row is
 * computed by the CTAs that need it, as that row enters their windows, with hsad_reduce's
 * exact arithmetic; measured slower than the two-step path on B200), 0 when it ran
 * hsad_reduce first. */
int32_t hsad_last_reduce_detect_fused(void);

/* Rows [*buf_row0, *buf_row0 + *buf_rows) that output rows [row_begin, row_end) of a
 * `lines`-row image read for the given requests (window halo + reflection). */
hsad_status hsad_strip_rows(int64_t lines, int64_t row_begin, int64_t row_end,
                            const hsad_detect_request* requests, int32_t n_requests,
                            int64_t* buf_row0, int64_t* buf_rows);
/* Row-chunk height the detector grid is anchored to for this image; strip
 * boundaries that are multiples of it keep per-pixel arithmetic identical. */
int64_t hsad_row_quantum(int64_t lines, int64_t samples);

hsad_status hsad_decode_status(uint64_t packed, int64_t samples, hsad_pixel_error* err);

/* ---- end to end on host buffers ---------------------------------------------- */
/* h_cube (fp32 BIP, host; pinned memory recommended) -> H2D -> reduce (order,
 * target_bands; order 0 = no reduction, detect on the full-band cube) -> all
 * requests (their d_scores must be HOST pointers here, rows x samples) -> D2H.
 * Synchronous. Device buffers are cached per thread between calls. */
hsad_status hsad_pipeline_host(const float* h_cube, int64_t lines, int64_t samples, int32_t bands,
                               int32_t order, int32_t target_bands,
                               const hsad_detect_request* host_requests, int32_t n_requests,
                               hsad_pixel_error* err, void* stream);

/* One process, G GPUs: the image splits into n_strips row strips aligned to
 * hsad_row_quantum (hsad_strip_plan), dealt to the devices in contiguous blocks; a host
 * thread per device streams its row range like hsad_pipeline_host (buffer rows = range +
 * reflected window halo from h_cube, H2D overlapped with reduce, fused detectors and the
 * D2H of finished rows, on the device's persistent buffers and streams) and writes its
 * map rows straight into the HOST maps of host_requests. Maps are bit-identical to a
 * one-strip run. Errors: the first failing request at its first failing pixel, as one
 * sequential call would report it. Synchronous. */
hsad_status hsad_pipeline_sharded(const float* h_cube, int64_t lines, int64_t samples, int32_t bands,
                                  int32_t order, int32_t target_bands,
                                  const hsad_detect_request* host_requests, int32_t n_requests,
                                  int32_t n_strips, hsad_pixel_error* err);

/* ---- multi-GPU row strips and the NCCL score-map gather ----------------- */
/* Rank `rank` of `world` owns output rows [*row0, *row1): strips of *strip_rows rows, a
 * multiple of hsad_row_quantum (so every map is bit-identical to a one-GPU run). The
 * reference's analogue is parallel_rows' row split, proj/core/src/parallel.hpp:17-40. */
hsad_status hsad_strip_plan(int64_t lines, int64_t samples, int32_t world, int32_t rank,
                            int64_t* row0, int64_t* row1, int64_t* strip_rows);

typedef struct hsad_map_desc {
    const void* d_strip;   /* this rank's rows [row0, row1) x samples (device) */
    void* d_full;          /* root only: the lines x samples map (device); may hold d_strip */
    int32_t elem_bytes;    /* 8 fp64 scores, 4 fp32 scores, 1 int8 DWEST eigen-counts */
} hsad_map_desc;

/* Gathers every rank's strip of each map into the root's full maps: one grouped
 * ncclSend per map on the other ranks, ncclRecv straight into place on the root (strips
 * are contiguous row blocks), a device copy for the root's own strip. nccl_comm is the
 * caller's ncclComm_t over `world` ranks (ncclCommInitRank / hsad_nccl_comm_init_*);
 * single-process multi-GPU callers issue one call per device from one host thread per
 * device. Enqueued on `stream`; NCCL is loaded at run time (libnccl.so.2). */
hsad_status hsad_gather_maps(void* nccl_comm, int32_t world, int32_t rank, int32_t root,
                             int64_t lines, int64_t samples, const hsad_map_desc* maps,
                             int32_t n_maps, void* stream);
/* Communicator helpers for callers without their own NCCL setup (thin wrappers of
 * ncclGetUniqueId / ncclCommInitRank / ncclCommInitAll / ncclCommDestroy). */
hsad_status hsad_nccl_available(void);
hsad_status hsad_nccl_unique_id(uint8_t* id128);
hsad_status hsad_nccl_comm_init_rank(void** comm, int32_t world, const uint8_t* id128, int32_t rank);
hsad_status hsad_nccl_comm_init_all(void** comms, int32_t ndev);
hsad_status hsad_nccl_comm_destroy(void* comm);

/* ---- ENVI ingest --------------------------------------------- */
typedef enum hsad_interleave { /* hsad::Interleave, cube.hpp:20 */
    HSAD_BSQ = 0,
    HSAD_BIL = 1,
    HSAD_BIP = 2
} hsad_interleave;

typedef struct hsad_cube_header { /* hsad::CubeHeader, cube.hpp:26-37 */
    int32_t samples, lines, bands;
    int32_t interleave;     /* hsad_interleave */
    int32_t data_type_code; /* 1=u8, 2=i16, 4=f32, 5=f64, 12=u16 */
    int32_t byte_order;     /* 0 little-endian, 1 big-endian */
} hsad_cube_header;

/* Replaces hsad::read_cube (proj/core/src/cube.cpp:198-253): validate the header
 * (cube.cpp:22-45), check raw_bytes == samples*lines*bands*element_size
 * (SizeMismatch), decode every element (byte swap, widen) from the header's
 * interleave into the BIP cube d_out (out_bytes 8 = the reference's fp64
 * HyperCube; 4 = fp32, only for u8/i16/u16/f32 sources, which fp32 holds
 * exactly), and reject non-finite values with NonFiniteValue
 * "at (row=r, col=c, band=b)" for the first one in (row, col, band) order.
 * d_raw, d_out: device pointers. Synchronous (the status is read back). */
hsad_status hsad_read_cube(const void* d_raw, int64_t raw_bytes, const hsad_cube_header* header,
                           void* d_out, int32_t out_bytes, void* stream);

/* read_cube followed by reduce_cube (wavelet.cpp:148-167) without the BIP intermediate:
 * a BSQ / BIL raw cube is decoded and reduced in one pass (composed wavelet map applied
 * per band plane row segment); BIP raw input goes through hsad_read_cube + hsad_reduce.
 * Header / size errors as hsad_read_cube, then the wavelet parameter errors of
 * hsad_reduce, then NonFiniteValue for the first non-finite element. d_out: BIP
 * (lines x samples x target_bands), out_bytes 8 or 4. target_bands 1..16 (powers of 2).
 * Synchronous. */
hsad_status hsad_reduce_raw(const void* d_raw, int64_t raw_bytes, const hsad_cube_header* header,
                            int32_t order, int32_t target_bands, void* d_out, int32_t out_bytes,
                            void* stream);

/* read_cube + reduce_cube + detect on HOST buffers (the CLI's reduce + detect on an ENVI
 * file minus file reading): h_raw holds the raw file bytes of a BSQ or BIL cube; row
 * strips stream to the device (BSQ as 2D copies of the band-plane segments), are decoded
 * and reduced in one pass, detected and copied back as in hsad_pipeline_host. Errors:
 * header / size (read_cube), wavelet parameters, request validation, then NonFiniteValue
 * anywhere in the cube before any detector failure. host_requests' d_scores / d_eigcount
 * are HOST pointers (lines x samples). Synchronous. */
hsad_status hsad_pipeline_raw(const void* h_raw, int64_t raw_bytes, const hsad_cube_header* header,
                              int32_t order, int32_t target_bands,
                              const hsad_detect_request* host_requests, int32_t n_requests,
                              hsad_pixel_error* err, void* stream);

/* ---- evaluation on device ------------------------------------ */
typedef struct hsad_roc_summary {
    uint64_t positives, negatives;
    /* sum over (positive, negative) pairs of 2 [s_pos > s_neg] + [s_pos == s_neg]:
     * the reference's exact integer AUC numerator (eval.cpp:33-46) */
    uint64_t auc_twice_num;
    double auc;         /* auc_twice_num / (2 positives negatives), eval.cpp:54-55 */
    uint64_t distinct;  /* distinct score values = ROC points - 1 */
} hsad_roc_summary;

/* hsad::roc_curve's AUC (proj/core/src/eval.cpp:10-57) for n scores (score_bytes
 * 8 or 4) and a 0/1 truth mask (nonzero = positive, synth.cpp:15-18), all on the
 * device. DegenerateTruth when either class is empty. When d_far / d_td are
 * non-null they receive the ROC points (distinct + 1 each, far/td as in
 * eval.cpp:30-52: (0,0) first, one step per distinct score, descending). The
 * points need a full sort of the scores (a device radix sort); the AUC alone
 * sorts only the positives. Synchronous. */
hsad_status hsad_roc(const void* d_scores, int32_t score_bytes, const uint8_t* d_truth, int64_t n,
                     hsad_roc_summary* out, double* d_far, double* d_td, int64_t points_capacity,
                     void* stream);

/* Indices (ascending) of the k largest scores; ties at the k-th value are broken
 * towards lower indices. *kth = the k-th largest score. Synchronous. */
hsad_status hsad_top_k(const void* d_scores, int32_t score_bytes, int64_t n, int64_t k,
                       int64_t* d_indices, double* kth, void* stream);

/* hsad::adaptive_threshold (eval.cpp:69-90): tau = mean + z_alpha * sqrt(population
 * variance) (two passes, fp64 with compensated per-thread sums), d_mask[i] =
 * scores[i] > tau. InvalidValue on an empty map. Synchronous. */
hsad_status hsad_adaptive_threshold(const void* d_scores, int32_t score_bytes, int64_t n,
                                    double z_alpha, double* tau, uint8_t* d_mask, void* stream);

/* hsad::render_pgm's pixel stretch (eval.cpp:92-109): lo/hi = min/max score,
 * pixel = lround((s - lo) * (255 / (hi - lo))) when hi > lo, else 0. Synchronous. */
hsad_status hsad_render_pgm(const void* d_scores, int32_t score_bytes, int64_t n,
                            uint8_t* d_pixels, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* HSAD_GPU_H */
