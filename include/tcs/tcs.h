/*
 * tcs.h -- C-ABI of the B200-native FlashSparse hot path
 *          (CSR -> ME-BCRS conversion, SpMM, SDDMM; sm_100a).
 *
 * This is the drop-in boundary for the reference's C++ API in
 * /root/reference/proj/include/tcsparse ("ref:" below).  Every entry point is
 * extern "C", takes plain pointers and sizes, throws nothing, and reports
 * errors through tcs_status plus a thread-local message (tcs_last_error).
 * The status codes map one-to-one onto the reference's exception taxonomy
 * (ref: errors.hpp:11-38); include/tcsparse/gpu.hpp rethrows them as those
 * exact types.
 *
 * Device entry points (tcs_mebcrs_encode, tcs_spmm, tcs_sddmm) take DEVICE
 * pointers and are stream-ordered: they enqueue work on `stream` and return.
 * tcs_mebcrs_encode synchronises once (the output sizes are data dependent).
 * The *_host entry points take HOST pointers (pinned for full bandwidth),
 * copy, compute and copy back on `stream`, and synchronise before returning
 * -- the value semantics of the reference API.
 *
 * There is no CPU fallback: without a CUDA device every call returns
 * TCS_ERR_CUDA.
 */
#ifndef TCS_TCS_H_
#define TCS_TCS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tcs_stream_t; /* == cudaStream_t; NULL = legacy default stream */

/* ref: errors.hpp -- FormatError(:24), ShapeError(:30), ArgumentError(:36). */
typedef enum tcs_status {
    TCS_OK = 0,
    TCS_ERR_ARGUMENT = 1, /* ref ArgumentError: bad precision / vector height / null pointer */
    TCS_ERR_SHAPE = 2,    /* ref ShapeError: operand dimensions disagree               */
    TCS_ERR_FORMAT = 3,   /* ref FormatError: ME-BCRS / CSR invariants violated         */
    TCS_ERR_CUDA = 4,     /* CUDA runtime error (no device, launch failure, ...)        */
    TCS_ERR_NCCL = 5,     /* reserved for the multi-GPU layer                           */
    TCS_ERR_OOM = 6,      /* device allocation failed                                   */
    TCS_ERR_PARSE = 7,    /* ref ParseError (errors.hpp:11-22): malformed MatrixMarket;
                             the message carries "line N: " as the reference's          */
    TCS_ERR_IO = 8        /* a container / output file cannot be opened or written      */
} tcs_status;

/* ref: precision.hpp:13 (Precision{fp16=0, tf32=1}). */
typedef enum tcs_precision { TCS_FP16 = 0, TCS_TF32 = 1 } tcs_precision;

/* Element type of a buffer. */
typedef enum tcs_dtype { TCS_DTYPE_F16 = 0, TCS_DTYPE_F32 = 1 } tcs_dtype;

/* ref: access_pattern.hpp:15 (ThreadMapping). No numerical effect
 * (ref tests/acceptance.cpp:103-104): both give bit-identical results.
 * COALESCED (default) runs the memory-efficient mapping; DIRECT runs, for
 * FP16 SpMM, the paper's direct mapping (each lane loads its own fragment
 * elements as 2-byte gathers) as the ablation baseline.  TF32 mappings
 * coincide (ref access_pattern.hpp:110-119). */
typedef enum tcs_mapping { TCS_MAP_DIRECT = 0, TCS_MAP_COALESCED = 1 } tcs_mapping;

/* ref: matrix.hpp:20-49 (CsrMatrix). u32 indices, f32 values; column
 * indices strictly ascending within a row; explicit zeros are entries. */
typedef struct tcs_csr {
    uint64_t rows;
    uint64_t cols;
    uint64_t nnz;
    const uint32_t* row_ptr; /* rows+1 */
    const uint32_t* col_idx; /* nnz    */
    const float* values;     /* nnz    */
} tcs_csr;

/* ref: mebcrs.hpp:23-78 (MeBcrsMatrix).  Windows of 8 rows; vector v of
 * window w (0-based, ascending column) sits in block b = v / k at
 *   values[8 * (row_pointers[w] + b * k) + r * width_b + v % k],
 *   width_b = min(k, nv_w - b * k)                 (ref mebcrs.hpp:46-56).
 * value_dtype F16 stores RNE-rounded binary16 (bit-identical to the
 * reference's round_to_fp16, applied by the reference at MMA time); F32
 * stores the reference's raw binary32 values.  TF32 always uses F32. */
typedef struct tcs_mebcrs {
    uint64_t rows;
    uint64_t cols;
    uint32_t vector_height; /* 8 */
    uint32_t k;             /* storage block width: 8 (FP16), 4 (TF32); ref mma.hpp:23 */
    tcs_precision precision;
    tcs_dtype value_dtype;
    uint64_t num_windows;     /* ceil(rows / 8)                   */
    uint64_t num_vectors;     /* nv = row_pointers[num_windows]   */
    uint32_t* row_pointers;   /* device, num_windows + 1           */
    uint32_t* column_indices; /* device, num_vectors               */
    void* values;             /* device, 8 * num_vectors elements  */
    uint32_t flags;           /* TCS_MEBCRS_OWN_* : which arrays tcs_mebcrs_free releases */
    uint32_t max_window_vectors; /* filled by tcs_mebcrs_prepare      */
    uint64_t num_blocks;         /* sum_w ceil(nv_w / k)              */
    uint64_t num_groups16;       /* sum_w ceil(nv_w / 16)             */
    void* plan;                  /* library-private work list; NULL until prepared */
} tcs_mebcrs;

#define TCS_MEBCRS_OWN_STRUCTURE 0x1u /* row_pointers + column_indices */
#define TCS_MEBCRS_OWN_VALUES 0x2u
#define TCS_MEBCRS_BORROWED_PLAN 0x4u /* work list shared with the handle the structure came from */

/* ref: spmm.hpp:17-21 (KernelConfig). */
typedef struct tcs_kernel_config {
    tcs_precision precision;
    uint32_t vector_height; /* must be 8 (ref spmm.hpp:106) */
    tcs_mapping mapping;
    uint32_t flags; /* TCS_CFG_* */
} tcs_kernel_config;

/* SpMM instruction path.  Default (0 or TCS_CFG_PATH_MMA_SYNC): warp-level
 * mma.sync fed by quarter-warp-coalesced 128-bit gathers -- the faster path
 * on B200 for 8x1 vectors.  TCS_CFG_PATH_TCGEN05 selects
 * tcgen05.mma (TMEM accumulators) fed by TMA gather4 (FP16, binary16
 * values, N <= 256; ARGUMENT error otherwise). */
#define TCS_CFG_PATH_MMA_SYNC 0x1u
#define TCS_CFG_PATH_TCGEN05 0x2u
/* Also fill counters->transactions / transaction_bytes / useful_bytes with
 * the reference's access model (tcs_mebcrs_cost, one extra kernel). */
#define TCS_CFG_COUNT_ACCESS 0x4u
/* SDDMM (and the fused SDDMM -> softmax): the mask's values do not change
 * between calls.  The sampling rule (value != 0) is then read from one
 * liveness byte per stored vector, built from the values on first use and
 * cached in the handle's work list, instead of from the 8 stored values
 * (16 or 32 bytes per vector).  Results are identical; a caller that edits
 * the values in place must call tcs_mebcrs_prepare (fresh work list) before
 * relying on this flag again. */
#define TCS_CFG_STATIC_MASK 0x8u
/* TF32 SpMM, N > 32: gather the f32 dense operand as given instead of its
 * per-call repack into 2.5 bytes per feature (the top 19 bits the TF32 MMA
 * reads).  Same results bit for bit; kept as the ablation. */
#define TCS_CFG_TF32_F32_GATHER 0x10u

/* ref: spmm.hpp:23-28 (KernelCounters).  mma_invocations is reported in the
 * reference's units (storage-k blocks x 16-wide tiles, ref analysis.hpp:34);
 * the transaction fields belong to the reference's analytic cost model:
 * 0 unless cfg->flags has TCS_CFG_COUNT_ACCESS (real coalescing is measured
 * with ncu). */
typedef struct tcs_counters {
    uint64_t mma_invocations;
    uint64_t transactions;
    uint64_t transaction_bytes;
    uint64_t useful_bytes;
} tcs_counters;

/* ------------------------------------------------------------------ misc */
const char* tcs_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* tcs_last_error(void);
/* Number of kernels this library has launched in this process (a monotone
 * counter, used by benchmarks to report gpu_launches). */
uint64_t tcs_launch_count(void);

/* Diagnostics: applies, on the device, exactly the operand rounding the
 * kernels use -- RNE to binary16 (__float2half_rn; ref round_to_fp16,
 * precision.hpp:51-64) or RNE to TF32 (cvt.rn.tf32.f32; ref round_to_tf32,
 * precision.hpp:42-46) -- and widens back to f32.  in/out are device arrays
 * of n floats. */
tcs_status tcs_round_values(tcs_precision precision, const float* in, float* out, uint64_t n, tcs_stream_t stream);

/* ------------------------------------------------------------- conversion */
/* ref: encode_mebcrs(const CsrMatrix&, Precision)  (mebcrs.hpp:80).
 * Device CSR in; ME-BCRS out with library-allocated device arrays (release
 * with tcs_mebcrs_free).  value_dtype: F16 or F32 for TCS_FP16, F32 for
 * TCS_TF32.  row_pointers / column_indices are bit-identical to the
 * reference's; values are bit-identical (F32) or equal to the reference's
 * round_to_fp16 of them (F16).  Also prepares the SpMM/SDDMM work list. */
tcs_status tcs_mebcrs_encode(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype,
                             tcs_mebcrs* out, tcs_stream_t stream);

/* ref: partition_windows(m, vector_height, k) (partition.hpp:40-66) +
 * the ME-BCRS layout of mebcrs.hpp:80-114 at either vector height.
 * vector_height 8 is tcs_mebcrs_encode.  vector_height 16 builds the
 * 16-row-window layout of the reference's 16x1 baseline (spmm.hpp:187-257:
 * windows of 16 rows, blocks 16 x k, value (r, j) of block b of window w at
 * 16 * (row_pointers[w] + b * k) + r * width_b + j); such a handle is accepted
 * only by tcs_spmm_baseline16, download, validate, prepare and free.  Other
 * heights -> ARGUMENT (ref partition.hpp:42-43). */
tcs_status tcs_mebcrs_encode_v(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype,
                               uint32_t vector_height, tcs_mebcrs* out, tcs_stream_t stream);

/* Builds (or rebuilds) the work list and the block/group counts for an
 * ME-BCRS whose arrays were filled by the caller.  Synchronises. */
tcs_status tcs_mebcrs_prepare(tcs_mebcrs* m, tcs_stream_t stream);

/* Host-side structural checks of ref mebcrs.hpp:58-77 on device arrays
 * (copies them back; test/debug use).  Returns TCS_ERR_FORMAT on violation. */
tcs_status tcs_mebcrs_validate(const tcs_mebcrs* m, tcs_stream_t stream);

/* ref: decode_mebcrs(const MeBcrsMatrix&) (mebcrs.hpp:116-138): device
 * ME-BCRS -> device CSR (library-allocated arrays, release with
 * tcs_csr_free).  Every stored value != 0 becomes an entry (+-0.0 fill is
 * dropped), rows sorted by column, f32 values (binary16 storage widened).
 * The arrays are assumed valid (the reference validates first:
 * tcs_mebcrs_validate). */
tcs_status tcs_mebcrs_decode(const tcs_mebcrs* m, tcs_csr* out, tcs_stream_t stream);
/* Copies a device CSR into caller-sized host arrays (rows+1, nnz, nnz); any
 * pointer may be NULL.  Synchronises. */
tcs_status tcs_csr_download(const tcs_csr* m, uint32_t* row_ptr, uint32_t* col_idx, float* values,
                            tcs_stream_t stream);

/* Releases the arrays flagged as owned and the work list; zeroes *m. */
tcs_status tcs_mebcrs_free(tcs_mebcrs* m, tcs_stream_t stream);

/* ------------------------------------------------------------------- SpMM */
/* ref: spmm(const MeBcrsMatrix&, const DenseMatrix&, const KernelConfig&)
 * (spmm.hpp:173).  C[rows x n] (f32, row stride ldc) = A * B, B is
 * [b_rows x n] with row stride ldb in b_dtype.  Errors as the reference:
 * cfg->vector_height != 8 or cfg->precision != a->precision -> ARGUMENT;
 * a->cols != b_rows -> SHAPE.  Empty windows produce zero rows.
 * FP16 needs b_dtype F16 (or F32, converted with RNE into a workspace);
 * TF32 needs F32 (rounded RNE to TF32 in-register). */
tcs_status tcs_spmm(const tcs_mebcrs* a, const void* b, tcs_dtype b_dtype, int64_t ldb, int64_t b_rows,
                    int64_t n, float* c, int64_t ldc, const tcs_kernel_config* cfg,
                    tcs_counters* counters, tcs_stream_t stream);

/* ref: spmm_baseline16(const CsrMatrix&, const DenseMatrix&, const KernelConfig&)
 * (spmm.hpp:187-257) -- the paper's non-swapped 16x1 ablation: sparse
 * 16 x k blocks as the m=16 left MMA operand, k x 8 dense tiles.  `a` is a
 * vector_height-16 handle from tcs_mebcrs_encode_v.  Same numerical
 * contract as tcs_spmm.  Errors: cfg->vector_height != 16 -> ARGUMENT (ref
 * :190); precision mismatch -> ARGUMENT; a->cols != b_rows -> SHAPE.
 * counters->mma_invocations = sum_w ceil(nv_w / k) * ceil(n / 8) (ref
 * analysis.hpp:34-38, Strategy::baseline16). */
tcs_status tcs_spmm_baseline16(const tcs_mebcrs* a, const void* b, tcs_dtype b_dtype, int64_t ldb, int64_t b_rows,
                               int64_t n, float* c, int64_t ldc, const tcs_kernel_config* cfg,
                               tcs_counters* counters, tcs_stream_t stream);

/* -------------------------------------------- SR-BCRS (padded ablation) */
/* ref: srbcrs.hpp:11-38 (SrBcrsMatrix) -- the zero-vector padded baseline
 * format of the paper's footprint ablation: every window is widened to a
 * multiple of k vectors, so every block is a full 8 x k tile; padded
 * vectors carry TCS_SR_PADDING as column index and zero values.  The
 * pointer array holds a (begin, end) pair per window.  Value (r, j) of block
 * b of window w sits at 8 * (row_pointer_pairs[2w] + b * k) + r * k + j. */
#define TCS_SR_PADDING 0xFFFFFFFFu /* ref kPaddingSentinel (srbcrs.hpp:12) */
typedef struct tcs_srbcrs {
    uint64_t rows;
    uint64_t cols;
    uint32_t vector_height; /* 8 */
    uint32_t k;             /* 8 (FP16), 4 (TF32) */
    tcs_precision precision;
    tcs_dtype value_dtype;
    uint64_t num_windows;
    uint64_t num_padded;         /* stored (padded) vectors = column_indices length */
    uint32_t* row_pointer_pairs; /* device, 2 * num_windows */
    uint32_t* column_indices;    /* device, num_padded      */
    void* values;                /* device, 8 * num_padded  */
    void* impl;                  /* library-private gather view + work list */
} tcs_srbcrs;

/* ref: encode_srbcrs(const CsrMatrix&, Precision) (srbcrs.hpp:40-72), on the
 * GPU: CSR -> ME-BCRS -> padded.  All arrays bit-identical to the
 * reference's (values as F32, or their binary16 rounding as F16). */
tcs_status tcs_srbcrs_encode(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype, tcs_srbcrs* out,
                             tcs_stream_t stream);
/* The padding step alone (ref srbcrs.hpp:49-70), from a device ME-BCRS. */
tcs_status tcs_srbcrs_from_mebcrs(const tcs_mebcrs* me, tcs_srbcrs* out, tcs_stream_t stream);
/* Host arrays (2W pairs, padded column indices, 8 * padded f32 values) ->
 * device handle.  Windows must be stored back to back (pairs[2w+1] ==
 * pairs[2w+2], as encode_srbcrs produces them) and each a multiple of k
 * vectors; FORMAT error otherwise. */
tcs_status tcs_srbcrs_upload(uint64_t rows, uint64_t cols, tcs_precision precision,
                             const uint32_t* row_pointer_pairs, const uint32_t* column_indices, const float* values,
                             tcs_srbcrs* out, tcs_stream_t stream);
/* Device handle -> caller-sized host arrays (values widened to f32); any
 * pointer may be NULL.  Synchronises. */
tcs_status tcs_srbcrs_download(const tcs_srbcrs* m, uint32_t* row_pointer_pairs, uint32_t* column_indices,
                               float* values, tcs_stream_t stream);
tcs_status tcs_srbcrs_free(tcs_srbcrs* m, tcs_stream_t stream);
/* ref: decode_srbcrs (srbcrs.hpp:74-90): device CSR (library-allocated,
 * release with tcs_csr_free) of the stored values != 0; padded vectors
 * decode to nothing. */
tcs_status tcs_srbcrs_decode(const tcs_srbcrs* m, tcs_csr* out, tcs_stream_t stream);
/* ref: spmm(const SrBcrsMatrix&, const DenseMatrix&, const KernelConfig&)
 * (spmm.hpp:181-185): the swapped 8x1 kernel over the padded format;
 * padded vectors gather a zero row (the reference's kAbsentRow) and are
 * numerically inert.  The result equals tcs_spmm on the compact format bit
 * for bit wherever the sums are exact (the reference's small-integer
 * inputs); with real values, windows long enough to be split across work
 * items may associate their partial sums differently.  Arguments,
 * errors and counters as tcs_spmm (mma_invocations = sum_w padded_w / k *
 * ceil(n / 16)). */
tcs_status tcs_spmm_srbcrs(const tcs_srbcrs* a, const void* b, tcs_dtype b_dtype, int64_t ldb, int64_t b_rows,
                           int64_t n, float* c, int64_t ldc, const tcs_kernel_config* cfg, tcs_counters* counters,
                           tcs_stream_t stream);
/* tcs_spmm_srbcrs with host operands (the reference's value semantics): A
 * given by host SR-BCRS arrays (f32 values), B host f32 [b_rows x n], C host
 * f32 [rows x n]. */
tcs_status tcs_spmm_srbcrs_host(uint64_t rows, uint64_t cols, tcs_precision precision,
                                const uint32_t* row_pointer_pairs, const uint32_t* column_indices,
                                const float* values, const float* b, int64_t b_rows, int64_t n, float* c,
                                const tcs_kernel_config* cfg, tcs_counters* counters, tcs_stream_t stream);


/* ------------------------------------------------------------ cost model */
/* ref analysis.hpp:34-131 + footprint.hpp:13-25: the structural cost of one
 * SpMM over `m` with n_cols dense columns -- swapped 8x1 strategy for a
 * vector-height-8 handle, the 16x1 baseline for a vector-height-16 one --
 * evaluated on the GPU (the dense-operand gather of the reference's warp
 * model replayed per block and tile, 32-byte segments merged into aligned
 * 64/128-byte transactions).  nnz = the source CSR's entry count. */
typedef struct tcs_cost {
    uint64_t mma_count;              /* ref count_mma                                  */
    uint64_t zero_fill;              /* ref count_zero_fill: vh * nv - nnz             */
    uint64_t access_bytes;           /* ref data_access_cost(...).total()              */
    uint64_t transactions;           /* ref count_spmm_transactions (tiles 0,1 extrapolated) */
    uint64_t exec_transactions;      /* summed over all tiles == the executing kernel's */
    uint64_t exec_transaction_bytes; /*   KernelCounters (ref spmm.hpp:146-151, :236-240) */
    uint64_t exec_useful_bytes;
    uint64_t footprint_me;           /* ref footprint_me_bytes                          */
    uint64_t footprint_sr;           /* ref footprint_sr_bytes                          */
    uint64_t padded_vectors;         /* ref WindowPartition::padded_vectors             */
} tcs_cost;
tcs_status tcs_mebcrs_cost(const tcs_mebcrs* m, uint64_t nnz, int64_t n_cols, tcs_mapping mapping, tcs_cost* out,
                           tcs_stream_t stream);

/* ------------------------------------------------------------------ SDDMM */
/* ref: sddmm(const SddmmOperands&, const KernelConfig&)  (sddmm.hpp:84).
 * out.values[pos] = sum_l A[i][l] * Bt[j][l] at every mask position whose
 * stored value is != 0; every other slot of the output blocks is 0.
 * A is [a_rows x f_a] (row stride lda), Bt = B^T is [bt_rows x f_b]
 * (row stride ldbt).  `out` receives the mask's structure (aliased, not
 * owned) and values of out_dtype; if out->values is NULL they are
 * library-allocated (owned).  Errors: cfg precision != mask precision ->
 * ARGUMENT; a_rows != mask rows, bt_rows != mask cols, f_a != f_b -> SHAPE. */
tcs_status tcs_sddmm(const tcs_mebcrs* mask, const void* a, tcs_dtype a_dtype, int64_t lda, int64_t a_rows,
                     int64_t f_a, const void* bt, tcs_dtype bt_dtype, int64_t ldbt, int64_t bt_rows,
                     int64_t f_b, tcs_mebcrs* out, tcs_dtype out_dtype, const tcs_kernel_config* cfg,
                     tcs_counters* counters, tcs_stream_t stream);

/* ---------------------------------------------------- AGNN row softmax */
/* Row-wise softmax over the ME-BCRS pattern, the middle stage of the AGNN
 * attention layer (SDDMM -> row softmax -> SpMM).  Not a
 * reference operator.  For every row r of every window:
 *   out[pos] = exp(scale*scores[pos] - max_r) / sum_r  at live positions,
 * live = mask value != 0 (the SDDMM sampling rule, ref sddmm.hpp:131); all
 * other slots 0.  scores and mask share one structure (an SDDMM output and
 * its mask).  `out` receives that structure (aliased) and values of
 * out_dtype, library-allocated if out->values is NULL. */
tcs_status tcs_mebcrs_row_softmax(const tcs_mebcrs* scores, const tcs_mebcrs* mask, float scale, tcs_mebcrs* out,
                                  tcs_dtype out_dtype, tcs_stream_t stream);

/* Fused AGNN attention front half (no reference
 * counterpart): out = row_softmax(S, mask, scale) with S = tcs_sddmm(mask,
 * A, Bt) stored as score_dtype -- the result of tcs_sddmm followed by
 * tcs_mebcrs_row_softmax up to the order of the per-row exp sums.  The
 * SDDMM kernel publishes per-row softmax partials, so the scores are
 * normalised in one streaming pass with no mask re-read.  Arguments and
 * errors as tcs_sddmm; score_dtype as its out_dtype.  `out` as in
 * tcs_mebcrs_row_softmax. */
tcs_status tcs_sddmm_row_softmax(const tcs_mebcrs* mask, const void* a, tcs_dtype a_dtype, int64_t lda,
                                 int64_t a_rows, int64_t f_a, const void* bt, tcs_dtype bt_dtype, int64_t ldbt,
                                 int64_t bt_rows, int64_t f_b, float scale, tcs_dtype score_dtype, tcs_mebcrs* out,
                                 tcs_dtype out_dtype, const tcs_kernel_config* cfg, tcs_stream_t stream);

/* AGNN aggregation (no reference counterpart):
 *   C[rows x n] (f32, stride ldc) = row_softmax(scale * S) . Hc,
 *   S[i][j] = Hn[row0 + i] . Hn[j] sampled at the mask's live slots
 *   (tcs_sddmm's rule),
 * bit for bit the result of tcs_sddmm_row_softmax(mask, Hn[row0..], Hn,
 * scale, binary16 scores, binary16 P) followed by tcs_spmm(P, Hc), without
 * writing P: the softmax is applied to each sparse value inside the SpMM.
 * The mask is the adjacency rows [row0, row0 + rows) of a graph with
 * mask->cols nodes (row0 = 0 and rows = cols for the whole graph; a row
 * shard otherwise).  Hn [cols x f] (stride ldhn), Hc [cols x n] (stride
 * ldhc), F16 or F32 (rounded RNE to binary16).  FP16 masks only
 * (ARGUMENT otherwise).  cfg->flags may carry TCS_CFG_STATIC_MASK. */
tcs_status tcs_agnn_aggregate(const tcs_mebcrs* mask, const void* hn, tcs_dtype hn_dtype, int64_t ldhn, int64_t row0,
                              int64_t rows, int64_t f, float scale, const void* hc, tcs_dtype hc_dtype, int64_t ldhc,
                              int64_t n, float* c, int64_t ldc, const tcs_kernel_config* cfg, tcs_stream_t stream);

/* Fused AGNN attention (no reference counterpart):
 *   C[i] (f32, rows x f, stride ldc) = sum_j softmax_j(scale * cos(h[row0 + i], h[j])) h[j]
 * over the mask's live slots (tcs_sddmm's rule: mask value != 0), in ONE
 * pass: every neighbour row is gathered once and feeds both the score MMA
 * and the aggregation MMA (online softmax, flash-attention style).  h
 * [cols x f] f16 (stride ldh, 16-byte aligned rows), f = 32 or 64; the cosine
 * uses 1 / max(||h_j||, eps).  Tolerance-level agreement with
 * tcs_agnn_aggregate (scores are not rounded to binary16 here, P is
 * rounded to binary16 before the aggregation MMA).  Any mask precision
 * (only its pattern and liveness are read); cfg->flags may carry
 * TCS_CFG_STATIC_MASK.  SHAPE for other f, ARGUMENT for misaligned buffers. */
tcs_status tcs_agnn_attend(const tcs_mebcrs* mask, const void* h, tcs_dtype h_dtype, int64_t ldh, int64_t row0,
                           int64_t f, float scale, float eps, float* c, int64_t ldc, const tcs_kernel_config* cfg,
                           tcs_stream_t stream);

/* AGNN input transform (no reference counterpart): hn[i] = h[i] /
 * max(||h[i]||_2, eps) and hc[i] = h[i], rounded to out_dtype (F16/F32),
 * from one read of the f32 rows h [rows][ldh].  hn or hc may be NULL. */
tcs_status tcs_rows_normalize(const float* h, int64_t rows, int64_t f, int64_t ldh, void* hn, void* hc, int64_t ldo,
                              tcs_dtype out_dtype, float eps, tcs_stream_t stream);

/* ------------------------------------------------------ ingest / containers */
/* ref: parse_matrix_market (matrix_market.hpp:28-94) -- coordinate
 * real/integer/pattern, general/symmetric (expanded), pattern -> 1.0,
 * duplicates summed (csr_from_coords, matrix.hpp:96-128).  The text is
 * tokenised by all host cores; the coordinate -> CSR assembly (sort, run
 * sums, row pointers) runs on the GPU.  `out` receives library-allocated
 * HOST arrays (release with tcs_csr_free_host).  Malformed input ->
 * TCS_ERR_PARSE with the reference's message and line number. */
tcs_status tcs_matrix_market_parse(const char* text, uint64_t len, tcs_csr* out, tcs_stream_t stream);
/* As above from a file; an unreadable file -> TCS_ERR_PARSE "cannot open '<path>'"
 * (ref cli.hpp:34-38). */
tcs_status tcs_matrix_market_read(const char* path, tcs_csr* out, tcs_stream_t stream);
/* ref write_matrix_market (matrix_market.hpp:97-104), host CSR. */
tcs_status tcs_matrix_market_write(const char* path, const tcs_csr* host_csr);
tcs_status tcs_csr_free_host(tcs_csr* m);
/* ref csr_from_coords (matrix.hpp:96-128) on the device: n DEVICE
 * coordinates (0-based, in range) -> device CSR with library-allocated
 * arrays (release with tcs_csr_free).  Duplicates are summed in input order. */
tcs_status tcs_coo_to_csr(uint64_t rows, uint64_t cols, uint64_t n, const uint32_t* row, const uint32_t* col,
                          const float* values, tcs_csr* out, tcs_stream_t stream);
tcs_status tcs_csr_free(tcs_csr* m, tcs_stream_t stream);
/* ref write_mebcrs / read_mebcrs (container_io.hpp:56-91): the MEBC v1
 * container ("MEBC", u32 version, u64 rows, u64 cols, u32 vector_height,
 * u32 k, u8 precision, then u32-length-prefixed row_pointers, column_indices
 * and f32 values; little endian).  Write downloads the handle (binary16
 * values are widened, so a file is byte-identical to the reference's only
 * for F32-valued handles or fp16-representable values).  Read validates like
 * the reference (FORMAT errors with its messages) and returns a device handle
 * with F32 values, prepared.  Unopenable files -> TCS_ERR_IO. */
tcs_status tcs_mebcrs_write(const char* path, const tcs_mebcrs* m, tcs_stream_t stream);
tcs_status tcs_mebcrs_read(const char* path, tcs_mebcrs* out, tcs_stream_t stream);

/* ------------------------------------------------- host-buffer entry points */
/* Value semantics of the reference API: host arrays in, host arrays out.  */

/* Host CSR -> device ME-BCRS (then tcs_mebcrs_download for host arrays). */
tcs_status tcs_mebcrs_encode_host(const tcs_csr* host_csr, tcs_precision precision, tcs_dtype value_dtype,
                                  tcs_mebcrs* out, tcs_stream_t stream);
/* Copies a device ME-BCRS into caller-sized host arrays (values widened to
 * f32).  Any pointer may be NULL to skip that array.  Synchronises. */
tcs_status tcs_mebcrs_download(const tcs_mebcrs* m, uint32_t* row_pointers, uint32_t* column_indices,
                               float* values, tcs_stream_t stream);
/* Host arrays -> device ME-BCRS (values uploaded as F32) + prepare. */
tcs_status tcs_mebcrs_upload(uint64_t rows, uint64_t cols, tcs_precision precision,
                             const uint32_t* row_pointers, const uint32_t* column_indices,
                             const float* values, tcs_mebcrs* out, tcs_stream_t stream);

/* ref spmm with host operands: A given by host ME-BCRS arrays (f32 values),
 * B host f32 [b_rows x n], C host f32 [rows x n]. */
tcs_status tcs_spmm_host(uint64_t rows, uint64_t cols, tcs_precision precision, const uint32_t* row_pointers,
                         const uint32_t* column_indices, const float* values, const float* b, int64_t b_rows,
                         int64_t n, float* c, const tcs_kernel_config* cfg, tcs_counters* counters,
                         tcs_stream_t stream);

/* ref sddmm with host operands; out_values has 8 * nv floats. */
tcs_status tcs_sddmm_host(uint64_t rows, uint64_t cols, tcs_precision precision, const uint32_t* row_pointers,
                          const uint32_t* column_indices, const float* mask_values, const float* a,
                          int64_t a_rows, int64_t f_a, const float* bt, int64_t bt_rows, int64_t f_b,
                          float* out_values, const tcs_kernel_config* cfg, tcs_counters* counters,
                          tcs_stream_t stream);

/* The reference CLI's spmm pipeline (ref cli.hpp:162-200: encode_mebcrs
 * then spmm) from host buffers: host CSR + host f32 B -> host f32 C.
 * Pipelined over row-window chunks on side streams forked from and joined
 * back to `stream` (returns when C is in host memory): B uploads first,
 * then each chunk's column indices and values; a chunk is converted (no
 * host round trip) and multiplied as soon as it has landed, and its C rows
 * are copied back while later chunks upload.  row_ptr is validated on the
 * host before any chunk is queued; column indices are validated by the
 * chunk conversions, and a violation is reported (FORMAT, the reference's
 * message) after the pipeline drains -- C is then unspecified. */
tcs_status tcs_spmm_csr_host(const tcs_csr* host_csr, tcs_precision precision, const float* b, int64_t n,
                             float* c, const tcs_kernel_config* cfg, tcs_counters* counters,
                             tcs_stream_t stream);

/* ref spmm_baseline16(const CsrMatrix&, const DenseMatrix&, const
 * KernelConfig&) (spmm.hpp:187-257) with host operands: host CSR + host f32
 * B [b_rows x n] -> host f32 C [rows x n].  The CSR is partitioned into
 * 16-row windows on the GPU (ref partition_windows(sparse, 16, k), :195) and
 * multiplied by tcs_spmm_baseline16.  Errors in the reference's order:
 * cfg->vector_height != 16 -> ARGUMENT (:190), host_csr->cols != b_rows ->
 * SHAPE (:191). */
tcs_status tcs_spmm_baseline16_csr_host(const tcs_csr* host_csr, const float* b, int64_t b_rows, int64_t n,
                                        float* c, const tcs_kernel_config* cfg, tcs_counters* counters,
                                        tcs_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* TCS_TCS_H_ */
