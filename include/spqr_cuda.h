/*
 * spqr_cuda.h -- C ABI of the B200-native SpQR decode path.
 *
 * Plain C: pointers, sizes and status codes only (no torch, no C++ types).
 * Every entry point names the reference interface it replaces
 * (/root/reference/proj/include/spqr/<file>:<line>).  The reference is a
 * header-only C++ library with no FFI of its own; these are the functions a
 * binding (ctypes / cgo / JNI) for its decode path binds.
 * shows the bindings.
 *
 * Status codes: 0 = OK; 1 + Errc for the reference's error enum, in the same
 * enumerator order as common.hpp:10-27; SPQR_E_CUDA for CUDA runtime
 * failures; SPQR_E_UNSUPPORTED is never returned for a valid stream -- layers
 * outside the fast-path geometry run the generic CUDA kernels.  There is no
 * CPU fallback for any compute entry point.  spqr_last_error() returns the
 * calling thread's last message ("<ErrcName>: <what>", as spqr::Error::what()).
 *
 * Layout of the stream arguments: a complete .spqr stream (48-byte header,
 * optional permutation, column-block-major group records, CSR outliers) as
 * produced by the reference encode (format.hpp:269-352).
 */
#ifndef SPQR_CUDA_H
#define SPQR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum spqr_status {
    SPQR_OK = 0,
    SPQR_E_MALFORMED_HEADER = 1,
    SPQR_E_SHAPE_MISMATCH = 2,
    SPQR_E_NON_FINITE_VALUE = 3,
    SPQR_E_IO_FAILURE = 4,
    SPQR_E_PARSE_ERROR = 5,
    SPQR_E_MISSING_FILE = 6,
    SPQR_E_EMPTY_INPUT = 7,
    SPQR_E_NOT_POSITIVE_DEFINITE = 8,
    SPQR_E_DIMENSION_MISMATCH = 9,
    SPQR_E_CONFIG_INVALID = 10,
    SPQR_E_COLUMN_INDEX_OVERFLOW = 11,
    SPQR_E_MALFORMED_STREAM = 12,
    SPQR_E_VERSION_UNSUPPORTED = 13,
    SPQR_E_CORRUPT_CSR = 14,
    SPQR_E_ILL_CONDITIONED = 15,
    SPQR_E_OUTLIER_BUDGET_EXCEEDED = 16,
    SPQR_E_CUDA = 100,
    SPQR_E_BUFFER_TOO_SMALL = 101,
    SPQR_E_NCCL = 102
};

enum spqr_dtype { SPQR_F16 = 0, SPQR_F32 = 1 };

/* Header fields of a validated stream (format.hpp:366-398). */
typedef struct spqr_layer_info {
    uint32_t rows, cols;
    int32_t weight_bits, scale_bits, zero_bits;
    uint32_t beta1, beta2;
    uint32_t outlier_count;
    uint32_t flags;             /* stream flag bits (format.hpp:21-27) */
    int32_t has_permutation;    /* SpqrTensor::has_permutation() (non-identity order) */
    float tau, lambda_rel;
    uint64_t payload_bytes;     /* stream_payload_bytes (layout.hpp:47-64): algorithmic bytes */
    uint64_t device_bytes;      /* HBM held by a layer handle (0 from spqr_stream_validate) */
    int32_t fast_path;          /* 1 when the fused tiled kernel serves this layer */
    int32_t device;             /* CUDA ordinal of a layer handle */
} spqr_layer_info;

/* Size model -- LayoutSpec + stream_payload_bytes, layout.hpp:18-64. */
typedef struct spqr_layout_spec {
    uint32_t rows, cols;
    int32_t weight_bits, scale_bits, zero_bits;
    uint32_t beta1, beta2;
    uint32_t outlier_count;
    int32_t has_permutation;
} spqr_layout_spec;

/* Flat view of an in-memory SpqrTensor (format.hpp:32-67).  Arrays are
 * row-major / block-major exactly as the reference's vectors:
 *   codes          rows*cols           CodeMatrix::codes (solve order)
 *   scale_codes    nblocks*rows        BlockStats::scale_codes, block k at k*rows (bits<=8)
 *   zero_codes     nblocks*rows        BlockStats::zero_codes
 *   raw_scales     nblocks*rows        BlockStats::raw_scales (bits==16)
 *   raw_zeros      nblocks*rows        BlockStats::raw_zeros
 *   group_scalars  nblocks*ngroups*4   StatGroupScalars {scale_s,scale_z,zero_s,zero_z}
 *   order          cols or NULL        Permutation::order (NULL = identity)
 *   outlier_*      outlier_count       OutlierSet::items (row, col, value16)
 * For spqr_decode_arrays the caller allocates every array it passes (sizes
 * from spqr_stream_validate); NULL arrays are skipped. */
typedef struct spqr_tensor_arrays {
    uint32_t rows, cols;
    int32_t weight_bits, scale_bits, zero_bits;
    uint32_t beta1, beta2;
    uint32_t flags;  /* act_order / integer_zero / full_range_sign / outliers_enabled bits */
    float tau, lambda_rel;
    uint32_t* order;
    uint8_t* codes;
    uint8_t* scale_codes;
    uint8_t* zero_codes;
    float* raw_scales;
    float* raw_zeros;
    uint16_t* group_scalars;
    uint32_t outlier_count;
    uint32_t* outlier_rows;
    uint32_t* outlier_cols;
    uint16_t* outlier_vals;
} spqr_tensor_arrays;

typedef struct spqr_layer spqr_layer;

typedef struct spqr_layer_opts {
    int32_t device;        /* CUDA ordinal; -1 = current device */
    int32_t force_generic; /* 1: never build the tiled planes (tests / comparison) */
    int32_t keep_stream;   /* 1: keep the raw stream on the device even on the fast path (matvec,
                              dequantize and export read the cells; the stream is for debugging) */
    uint32_t row_begin;    /* row band [row_begin, row_end) of the stream; 0,0 = all rows */
    uint32_t row_end;
    int32_t host_transcode; /* 1: build the HBM layout on the host (comparison); 0: on the GPU */
} spqr_layer_opts;

/* ---------------------------------------------------------------- host -- */
/* Last error message of the calling thread ("" when none). */
const char* spqr_last_error(void);
/* Library / layout version string. */
const char* spqr_version(void);

/* decode()'s validation without materialising codes (format.hpp:354-500).
 * Returns the reference's Errc for every malformed input. */
int spqr_stream_validate(const uint8_t* stream, size_t nbytes, spqr_layer_info* info);

/* decode(std::span<const uint8_t>) -> SpqrTensor, format.hpp:354. */
int spqr_decode_arrays(const uint8_t* stream, size_t nbytes, spqr_tensor_arrays* out);

/* encode(const SpqrTensor&) -> bytes, format.hpp:269.  *len receives the
 * required size; SPQR_E_BUFFER_TOO_SMALL when cap < *len (out may be NULL). */
int spqr_encode_arrays(const spqr_tensor_arrays* t, uint8_t* out, size_t cap, size_t* len);

/* stream_payload_bytes(const LayoutSpec&), layout.hpp:47. */
uint64_t spqr_payload_bytes(const spqr_layout_spec* ls);

/* estimate_avg_bits(...), format.hpp:531.  out5 = {avg, base, first, second, outliers}. */
int spqr_estimate_avg_bits(int b_w, int b_s, int b_z, uint32_t beta1, uint32_t beta2, double r_o,
                           double* out5);

/* measure_actual_bits(const SpqrTensor&), format.hpp:550, from a stream.
 * out3 = {bits_per_param, per_outlier_bits, payload_bytes}. */
int spqr_measure_actual_bits(const uint8_t* stream, size_t nbytes, double* out3);

/* Row band [r0, r1) of a stream as a standalone, valid stream (CSR rebased,
 * same permutation).  The row-sharded multi-GPU wrapper loads these. */
int spqr_stream_slice_rows(const uint8_t* stream, size_t nbytes, uint32_t r0, uint32_t r1,
                           uint8_t* out, size_t cap, size_t* len);

/* Host-only check of the device-layout transcoder: stream -> tiled planes ->
 * stream, no GPU involved.  Returns SPQR_E_CONFIG_INVALID if the layer is
 * outside the fast-path geometry. */
int spqr_transcode_roundtrip_host(const uint8_t* stream, size_t nbytes, uint8_t* out, size_t cap,
                                  size_t* len);

/* Test hook: the tiled HBM image the loader would upload, in host memory.
 * dims4 = {Gn, Pn, cell_bytes, record_bytes}.  Call with NULL buffers to
 * query dims; then cells (record_bytes: cell records = cell + its outlier
 * entries, 16-B padded with 0xffffffff), cell_off (Gn*Pn+1 byte offsets).
 * `entries` is unused (kept for ABI stability). */
int spqr_debug_tiled_host(const uint8_t* stream, size_t nbytes, uint32_t* dims4, uint8_t* cells,
                          uint32_t* cell_off, uint32_t* entries);

/* -------------------------------------------------------------- device -- */
/* decode (format.hpp:354) + build_tile_plan (kernel.hpp:54) + upload:
 * validates exactly like decode, transcodes to the HBM layout, uploads once. */
int spqr_layer_create(const uint8_t* stream, size_t nbytes, const spqr_layer_opts* opts,
                      spqr_layer** out);
/* Extension (no reference counterpart; the reference decodes one tensor at a
 * time): layers sharing their input -- q/k/v, gate/up -- stacked row-wise in
 * one handle, so one launch writes all outputs (layer i's rows follow layer
 * i-1's in y).  Same columns, widths, group sizes and permutation required;
 * rows % 32 == 0 for all but the last.  matvec / matvec_ws / matvec_host only
 * (dequantize and export return SPQR_E_CONFIG_INVALID). */
int spqr_layer_create_stacked(const uint8_t* const* streams, const size_t* sizes, int count,
                              const spqr_layer_opts* opts, spqr_layer** out);
void spqr_layer_destroy(spqr_layer* layer);
int spqr_layer_get_info(const spqr_layer* layer, spqr_layer_info* info);
/* Batched-decode precision mode (default 0: batch >= 5 on gemm_tc, weights
 * rounded to fp16).  exact != 0: every batch on exact-code kernels (fp32
 * rounding only).  Changes the workspace size spqr_workspace_bytes reports.
 * Not for a layer in use on another thread or stream. */
int spqr_layer_set_exact(spqr_layer* layer, int exact);

/* encode() of the device-resident layer (format.hpp:269): reads the HBM
 * layout back and re-encodes it; byte-identical to the input stream. */
int spqr_layer_export_stream(const spqr_layer* layer, uint8_t* out, size_t cap, size_t* len);

/* dequantize_full (kernel.hpp:17-25): W (rows x cols, fp32, row-major,
 * ORIGINAL column order) into caller device memory.  Bit-exact.  Fast-path
 * layers decode their cell records (dequant_cells, one launch); others the
 * raw stream (dequant_raw + outliers_raw). */
int spqr_dequantize(const spqr_layer* layer, float* w_dev, void* cuda_stream);

/* Scratch for spqr_matvec_ws (bytes).  The workspace carries arrival
 * counters between launches: zero-fill it once before its first use
 * (cudaMemsetAsync(ws, 0, bytes)); every launch leaves its counters zero
 * again.  A workspace belongs to ONE layer and one stream at a time (its
 * counter and partial regions sit at layer-specific offsets): zero it again
 * before handing it to another layer.  Size it for the largest batch used. */
uint64_t spqr_workspace_bytes(const spqr_layer* layer, int batch);

/* matvec (kernel.hpp:89-124) on device buffers: y[b] = W * x[b] for b < batch.
 * x: batch x cols (f16 or f32, original column order), y: batch x rows fp32.
 * Asynchronous on cuda_stream; allocates nothing.  spqr_matvec uses the
 * layer's own workspace (one stream at a time); spqr_matvec_ws takes a caller
 * workspace (concurrent streams; size from spqr_workspace_bytes(layer, batch)).
 * Fast-path layers: batch 1-4 run fused gemv_cta launches -- fp16 x two
 * columns per launch (each weight decoded once for both), an odd column and
 * fp32 x one column per launch (exact codes, fp32 accumulation: ~1e-7
 * relative to the reference); batch >= 5 run xprep_tc + gemm_tc per 64
 * columns (weights rounded to fp16, tcgen05 tensor cores: ~1e-4 relative on
 * well-conditioned layers, the north star's bar is 1e-3) -- unless the layer
 * is in exact mode (spqr_layer_set_exact): then batch < 7 runs the
 * gemv_cta launches and batch >= 7 xprep_bm + gemm_bm per 32 fp16 columns (batch in the
 * mma.sync M dimension) or xprep_ex + gemm_ex per 64 columns (fp32 x, wider
 * batches; tcgen05) -- exact codes, per-block fp32 scales: ~1e-6 relative. */
int spqr_matvec(const spqr_layer* layer, const void* x_dev, int x_dtype, float* y_dev, int batch,
                void* cuda_stream);
int spqr_matvec_ws(const spqr_layer* layer, const void* x_dev, int x_dtype, float* y_dev,
                   int batch, void* workspace, uint64_t ws_bytes, void* cuda_stream);

/* Fused all-gather for the row-sharded wrapper ("optional
 * B200-native fusion"; 8f rank 2): instead of spqr_matvec on the band followed
 * by an NCCL all-gather of y, each rank's gemv_cta stores every finished y
 * row straight into every rank's full-y buffer (peer addresses from CUDA IPC:
 * NVLink P2P stores between GPUs); its last CTA bumps this rank's round
 * counter on every rank and waits for all ranks' counters, so the launch
 * completes with y whole (spqr_gather_wait is kept for callers and launches
 * nothing).  Rounds live on the device: the launch replays in a CUDA graph.  Protocol: spqr_gather_create on every rank -> spqr_gather_handle ->
 * exchange the world x SPQR_GATHER_HANDLE_BYTES handles and the bands' first
 * rows (any transport, e.g. torch.distributed) -> spqr_gather_open -> per
 * step spqr_matvec_gather + spqr_gather_wait, then read spqr_gather_y.
 * Batch 1; the layer is this rank's band (rows row_base[rank] ...).
 * Round safety: a rank's band kernel of round R stores into peer j's y only
 * after peer j's band kernel of round R has started (each band kernel posts
 * its round to every rank first), so everything peer j issued on its stream
 * before spqr_matvec_gather of round R -- its readers of round R-1's y -- has
 * completed: consumers of spqr_gather_y must be stream-ordered before the
 * rank's next spqr_matvec_gather (no host barrier is needed between rounds). */
#define SPQR_GATHER_HANDLE_BYTES 64
typedef struct spqr_gather spqr_gather;
int spqr_gather_create(int device, uint32_t rows, int world, int rank, spqr_gather** out);
int spqr_gather_handle(const spqr_gather* g, void* handle_out);
int spqr_gather_open(spqr_gather* g, const void* handles, const uint32_t* row_base);
float* spqr_gather_y(const spqr_gather* g);
int spqr_matvec_gather(const spqr_layer* layer, const void* x_dev, int x_dtype, spqr_gather* g,
                       void* cuda_stream);
int spqr_gather_wait(spqr_gather* g, void* cuda_stream);
void spqr_gather_destroy(spqr_gather* g);

/* Row-sharded decode over NCCL (SURVEY 8b "spqr_sharded_create(..., ncclComm_t)
 * + spqr_sharded_matvec", 8e; BASELINE north_star: row-sharded layers with an
 * NCCL all-gather of y).  One process per GPU.  Rank r holds the contiguous
 * row band edges[r] .. edges[r+1] of the layer -- or of `count` layers stacked
 * row-wise (q/k/v, gate/up: all but the last with rows % 32 == 0), cut in the
 * stacked row order so the gathered y is [layer 0; layer 1; ...] -- with
 * bands of lcm(32, beta2)-row units, sizes differing by at most one unit
 * (sharded.py row_bands computes the same edges).  spqr_sharded_matvec: the
 * band's spqr_matvec, then ncclAllGather of the y bands on cuda_stream; y
 * (batch x rows fp32, on this rank's device) is complete on every rank when
 * the stream reaches that point.  The handle's band layer and gather slots
 * are used one call at a time (calls serialise on the handle); NCCL's rules
 * apply (every rank issues the same sequence of calls).  NCCL is bound at
 * run time (dlopen libnccl.so.2); NCCL failures return SPQR_E_NCCL.
 * Communicator: spqr_nccl_unique_id on one rank, broadcast the
 * SPQR_NCCL_ID_BYTES bytes (any transport), spqr_nccl_comm_init on every
 * rank -- or pass an ncclComm_t the application already has. */
#define SPQR_NCCL_ID_BYTES 128
typedef struct spqr_sharded spqr_sharded;
/* The band edges (world + 1 values) every rank computes for `rows` stacked rows. */
int spqr_row_bands(uint32_t rows, uint32_t beta2, int world, uint32_t* edges);
int spqr_nccl_unique_id(uint8_t* id_out);
int spqr_nccl_comm_init(const uint8_t* id, int world, int rank, int device, void** nccl_comm_out);
int spqr_nccl_comm_destroy(void* nccl_comm);
int spqr_sharded_create(const uint8_t* const* streams, const size_t* sizes, int count, int rank, int world,
                        void* nccl_comm, const spqr_layer_opts* opts, spqr_sharded** out);
int spqr_sharded_band(const spqr_sharded* s, uint32_t* rows, uint32_t* band_begin, uint32_t* band_end,
                      spqr_layer** band_layer);
int spqr_sharded_matvec(spqr_sharded* s, const void* x_dev, int x_dtype, float* y_dev, int batch,
                        void* cuda_stream);
void spqr_sharded_destroy(spqr_sharded* s);

/* The encoder on the GPU (the path's producer): Hessian
 * accumulation H += 2 X X^T (hessian.hpp:59-69, binary64), damped inverse
 * Cholesky (hessian.hpp:103-143), block-GPTQ with the leave-one-out outlier
 * screen and the bilevel statistics fit (spqr_quantize, solver.hpp:417-533),
 * then encode (format.hpp:269-352) -- the reference's arithmetic in binary64
 * with rows in parallel, the trailing updates / products on cuBLAS DGEMM and
 * the factorizations on cuSOLVER (bound at run time).  The stream equals the
 * reference encoder's (tests/test_gpu_encoder.py). */
typedef struct spqr_encoder_cfg {
    int32_t weight_bits, scale_bits, zero_bits;  /* b_w; b_s, b_z (16: raw fp32 statistics) */
    uint32_t beta1, beta2;                       /* beta1 <= 256 */
    int32_t order;                               /* 0 natural, 1 act_order, 2 shuffled (seed) */
    int32_t act_order_key;                       /* 0 Hessian diagonal, 1 inverse diagonal */
    int32_t outliers_enabled, integer_zero, full_range_sign;
    double tau, lambda_rel;
    uint64_t seed;
} spqr_encoder_cfg;
typedef struct spqr_hessian spqr_hessian;
int spqr_hessian_create(uint32_t n, int device, spqr_hessian** out);
/* x: n x samples fp32, row-major, on the Hessian's device. */
int spqr_hessian_accumulate(spqr_hessian* h, const float* x_dev, uint32_t samples, void* cuda_stream);
int spqr_hessian_read(const spqr_hessian* h, double* h_host);  /* n x n binary64 */
void spqr_hessian_destroy(spqr_hessian* h);
/* W: m x n fp32 row-major (original column order) on the device; out: the
 * .spqr stream; report[3] = {relative layer error, outlier rate, bits/param}. */
int spqr_quantize_layer(const spqr_hessian* h, const float* w_dev, uint32_t m, const spqr_encoder_cfg* cfg,
                        uint8_t* out, size_t cap, size_t* len, double* report);
/* tune_tau (solver.hpp:546-640): binary search of the 0.05-step tau grid over
 * [0.1, 1.0] for the smallest tau with outlier rate <= target_rate (cfg.tau is
 * ignored); report[5] = {relative error, outlier rate, bits/param, tau,
 * target reached (1/0)}.  cap must hold the stream (the encoded layer). */
int spqr_quantize_layer_tuned(const spqr_hessian* h, const float* w_dev, uint32_t m, const spqr_encoder_cfg* cfg,
                              double target_rate, uint8_t* out, size_t cap, size_t* len, double* report);

/* Profiling split of spqr_matvec: stage 1 = x preparation only, stage 2 = the
 * product only, 0 = both.  On the fast path x preparation is fused into the
 * product kernel, so stage 1 launches nothing and stage 2 equals stage 0;
 * the generic (raw-stream) path still has two kernels. */
int spqr_matvec_stage(const spqr_layer* layer, const void* x_dev, int x_dtype, float* y_dev, int batch,
                      int stage, void* cuda_stream);

/* matvec(const SpqrTensor&, std::span<const float>) drop-in with HOST buffers
 * (kernel.hpp:126-128): copies x in, computes, copies y out, synchronises. */
int spqr_matvec_host(const spqr_layer* layer, const float* x_host, float* y_host, int batch);

/* Comparator: dense fp16 GEMV y = W16 * x (our own 128-bit-load kernel),
 * W16 rows x cols row-major fp16, x fp16, y fp32. */
int spqr_dense_gemv_f16(const void* w_dev, const void* x_dev, float* y_dev, uint32_t rows,
                        uint32_t cols, void* cuda_stream);

/* Test hook: the device-resident cell records (len bytes) and record offsets
 * (Gn*Pn + 1 entries) of a fast-path layer; cells == NULL queries len. */
int spqr_debug_layer_cells(const spqr_layer* layer, uint8_t* cells, size_t cap, size_t* len, uint32_t* cell_off);

/* Number of kernel launches the last spqr_matvec* on this thread issued. */
int spqr_last_launch_count(void);

/* bench_matvec (kernel.hpp:185-226) timings on the device, CUDA-event timed,
 * median over `repeats`: ns3 = {fused matvec, dequantize_full (the naive
 * path's reconstruction), dense fp16 GEMV of the same shape}. */
int spqr_bench_layer(const spqr_layer* layer, int repeats, double* ns3);

/* Minimal device-memory helpers for C/C++ hosts without a CUDA toolchain. */
int spqr_dev_alloc(void** ptr, size_t bytes);
void spqr_dev_free(void* ptr);
int spqr_dev_copy_to_host(void* dst, const void* src, size_t bytes);
int spqr_dev_copy_to_device(void* dst, const void* src, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* SPQR_CUDA_H */
