// tcsparse/gpu.hpp -- header-only drop-in adapter: the reference API
// (proj/include/tcsparse) executed by the B200 library through the C-ABI.
//
//   tcsparse::encode_mebcrs(m, p)   ->  tcsparse::gpu::encode_mebcrs(m, p)
//   tcsparse::spmm(a, b, cfg)       ->  tcsparse::gpu::spmm(a, b, cfg)
//   tcsparse::sddmm(ops, cfg)       ->  tcsparse::gpu::sddmm(ops, cfg)
//   tcsparse::spmm_baseline16(m, b, cfg) -> tcsparse::gpu::spmm_baseline16(m, b, cfg)
//   (multi-GPU extension, no reference counterpart)
//                                   tcsparse::gpu::spmm_sharded(m, b, cfg, comm)
//
// Same parameter and return types as the reference (ref mebcrs.hpp:80,
// spmm.hpp:173, sddmm.hpp:84) -- this header includes the reference's own
// type definitions from whichever tcsparse include directory is on the
// include path, so code written against the reference switches by changing
// the namespace qualifier.  Value semantics are kept: host data in, host
// data out; each call uploads, runs the sm_100a kernels on the default
// stream and synchronises before returning.  Status codes are rethrown as
// the reference's exception types (ref errors.hpp).  Link with
// -ltcsparse_b200.
//
// Numerical contract (BASELINE.json north star): encode_mebcrs is
// bit-identical to the reference; spmm / sddmm are bit-identical on the
// reference's small-integer inputs and within rel-L2 1e-2 (FP16) / 1e-3
// (TF32) -- in practice ~1e-7 -- otherwise (the tensor core sums in a
// different order than the reference's sequential binary32 loop).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tcs/tcs.h"
#include "tcs/tcs_dist.h"
#include "tcsparse/mebcrs.hpp"
#include "tcsparse/sddmm.hpp"
#include "tcsparse/spmm.hpp"

namespace tcsparse::gpu {

namespace detail {

inline void check(tcs_status s) {
    if (s == TCS_OK) return;
    const std::string msg = tcs_last_error();
    switch (s) {
        case TCS_ERR_ARGUMENT: throw ArgumentError(msg);
        case TCS_ERR_SHAPE: throw ShapeError(msg);
        case TCS_ERR_FORMAT: throw FormatError(msg);
        case TCS_ERR_NCCL: throw std::runtime_error("tcsparse-b200 (NCCL): " + msg);
        default: throw std::runtime_error("tcsparse-b200: " + msg);
    }
}

// TCS_CFG_COUNT_ACCESS: the transaction counters are filled in the
// reference's units (its warp gather model, ref spmm.hpp:146-151, replayed
// on the GPU by the cost model) so every KernelCounters field matches.
inline tcs_kernel_config config(const KernelConfig& cfg) {
    return tcs_kernel_config{static_cast<tcs_precision>(cfg.precision),
                             static_cast<uint32_t>(cfg.vector_height),
                             static_cast<tcs_mapping>(cfg.mapping), TCS_CFG_COUNT_ACCESS};
}

inline KernelCounters counters(const tcs_counters& c) {
    KernelCounters k;
    k.mma_invocations = c.mma_invocations;
    k.transactions = c.transactions;
    k.transaction_bytes = c.transaction_bytes;
    k.useful_bytes = c.useful_bytes;
    return k;
}

// Array lengths must be consistent before their contents are handed to the
// device (ref mebcrs.hpp:58-66).
inline void require_lengths(const MeBcrsMatrix& m) {
    const std::size_t windows = (m.rows + m.vector_height - 1) / m.vector_height;
    if (m.row_pointers.size() != windows + 1) throw FormatError("row_pointers length must be numWindows+1");
    if (m.row_pointers.back() != m.column_indices.size())
        throw FormatError("row_pointers end must equal stored vector count");
    if (m.values.size() != m.vector_height * m.column_indices.size())
        throw FormatError("values length must be vectorHeight * stored vectors");
}

}  // namespace detail

/// ref mebcrs.hpp:80 -- CSR -> ME-BCRS, converted on the GPU.
inline MeBcrsMatrix encode_mebcrs(const CsrMatrix& m, Precision p) {
    const tcs_csr c{m.rows, m.cols, m.nnz(), m.row_ptr.data(), m.col_idx.data(), m.values.data()};
    tcs_mebcrs d{};
    detail::check(tcs_mebcrs_encode_host(&c, static_cast<tcs_precision>(p), TCS_DTYPE_F32, &d, nullptr));
    MeBcrsMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.vector_height = d.vector_height;
    out.k = d.k;
    out.precision = p;
    out.row_pointers.resize(d.num_windows + 1);
    out.column_indices.resize(d.num_vectors);
    out.values.resize(8 * d.num_vectors);
    const tcs_status s = tcs_mebcrs_download(&d, out.row_pointers.data(), out.column_indices.data(),
                                             out.values.data(), nullptr);
    tcs_mebcrs_free(&d, nullptr);
    detail::check(s);
    return out;
}

/// ref mebcrs.hpp:117 -- ME-BCRS -> CSR on the GPU (stored zeros dropped).
inline CsrMatrix decode_mebcrs(const MeBcrsMatrix& m) {
    m.validate();  // the reference's FormatError checks, in its order
    tcs_mebcrs d{};
    detail::check(tcs_mebcrs_upload(m.rows, m.cols, static_cast<tcs_precision>(m.precision), m.row_pointers.data(),
                                    m.column_indices.data(), m.values.data(), &d, nullptr));
    tcs_csr c{};
    tcs_status s = tcs_mebcrs_decode(&d, &c, nullptr);
    tcs_mebcrs_free(&d, nullptr);
    detail::check(s);
    CsrMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.row_ptr.resize(m.rows + 1);
    out.col_idx.resize(c.nnz);
    out.values.resize(c.nnz);
    s = tcs_csr_download(&c, out.row_ptr.data(), out.col_idx.data(), out.values.data(), nullptr);
    tcs_csr_free(&c, nullptr);
    detail::check(s);
    return out;
}

/// ref spmm.hpp:173 -- C = A * B with the 8x1 swap-and-transpose kernel.
inline SpmmResult spmm(const MeBcrsMatrix& sparse, const DenseMatrix& dense, const KernelConfig& cfg) {
    const tcs_kernel_config kc = detail::config(cfg);
    // the reference's checks, in its order (ref spmm.hpp:106-109)
    if (cfg.vector_height != 8) throw ArgumentError("swap-and-transpose path requires vector height 8");
    if (cfg.precision != sparse.precision) throw ArgumentError("config precision must match the encoded matrix");
    if (sparse.cols != dense.rows) throw ShapeError("sparse cols must equal dense rows");
    detail::require_lengths(sparse);
    SpmmResult res;
    res.output = DenseMatrix(sparse.rows, dense.cols);
    tcs_counters cn{};
    detail::check(tcs_spmm_host(sparse.rows, sparse.cols, static_cast<tcs_precision>(sparse.precision),
                                sparse.row_pointers.data(), sparse.column_indices.data(), sparse.values.data(),
                                dense.data.data(), static_cast<int64_t>(dense.rows),
                                static_cast<int64_t>(dense.cols), res.output.data.data(), &kc, &cn, nullptr));
    res.counters = detail::counters(cn);
    return res;
}

/// Multi-GPU extension of the CLI's encode + spmm pipeline (ref
/// cli.hpp:162-200; the reference itself has no communication layer, its
/// rows are independent per 8-row window): every rank of the
/// NCCL communicator `nccl_comm` (an ncclComm_t) calls this with the same
/// CSR; rank `root`'s dense operand is broadcast (the others' content is
/// ignored, only its shape is checked).  The row windows are cut by nnz,
/// each rank converts and multiplies its own rows, and every rank returns
/// the whole C.  An NCCL error, or no completion within timeout_ms, aborts
/// the communicator and throws std::runtime_error.  counters are this
/// rank's shard's.
inline SpmmResult spmm_sharded(const CsrMatrix& sparse, const DenseMatrix& dense, const KernelConfig& cfg,
                               void* nccl_comm, int root = 0, int64_t timeout_ms = 60000) {
    if (cfg.vector_height != 8) throw ArgumentError("swap-and-transpose path requires vector height 8");
    if (sparse.cols != dense.rows) throw ShapeError("sparse cols must equal dense rows");
    tcs_dist d{};
    detail::check(tcs_dist_init(&d, nccl_comm, timeout_ms));
    const tcs_kernel_config kc = detail::config(cfg);
    const tcs_csr c{sparse.rows, sparse.cols, sparse.nnz(), sparse.row_ptr.data(), sparse.col_idx.data(),
                    sparse.values.data()};
    SpmmResult res;
    res.output = DenseMatrix(sparse.rows, dense.cols);
    tcs_counters cn{};
    detail::check(tcs_spmm_sharded_csr_host(&d, &c, static_cast<tcs_precision>(cfg.precision), dense.data.data(),
                                            static_cast<int64_t>(dense.cols), root, res.output.data.data(), &kc,
                                            &cn, nullptr));
    res.counters = detail::counters(cn);
    return res;
}

/// ref spmm.hpp:187-257 -- the non-swapped 16x1 baseline over 16-row
/// windows of the CSR (the paper's ablation), on the GPU.
inline SpmmResult spmm_baseline16(const CsrMatrix& sparse, const DenseMatrix& dense, const KernelConfig& cfg) {
    // the reference's checks, in its order (ref spmm.hpp:190-191)
    if (cfg.vector_height != 16) throw ArgumentError("baseline path requires vector height 16");
    if (sparse.cols != dense.rows) throw ShapeError("sparse cols must equal dense rows");
    const tcs_kernel_config kc = detail::config(cfg);
    const tcs_csr c{sparse.rows, sparse.cols, sparse.nnz(), sparse.row_ptr.data(), sparse.col_idx.data(),
                    sparse.values.data()};
    SpmmResult res;
    res.output = DenseMatrix(sparse.rows, dense.cols);
    tcs_counters cn{};
    detail::check(tcs_spmm_baseline16_csr_host(&c, dense.data.data(), static_cast<int64_t>(dense.rows),
                                               static_cast<int64_t>(dense.cols), res.output.data.data(), &kc, &cn,
                                               nullptr));
    res.counters = detail::counters(cn);
    return res;
}

/// ref srbcrs.hpp:40 -- CSR -> SR-BCRS (the zero-vector padded baseline
/// format of the footprint ablation), converted on the GPU.
inline SrBcrsMatrix encode_srbcrs(const CsrMatrix& m, Precision p) {
    const tcs_csr c{m.rows, m.cols, m.nnz(), m.row_ptr.data(), m.col_idx.data(), m.values.data()};
    tcs_mebcrs d{};
    detail::check(tcs_mebcrs_encode_host(&c, static_cast<tcs_precision>(p), TCS_DTYPE_F32, &d, nullptr));
    tcs_srbcrs sr{};
    const tcs_status rc = tcs_srbcrs_from_mebcrs(&d, &sr, nullptr);
    tcs_mebcrs_free(&d, nullptr);
    detail::check(rc);
    SrBcrsMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.vector_height = sr.vector_height;
    out.k = sr.k;
    out.precision = p;
    out.row_pointer_pairs.resize(2 * sr.num_windows);
    out.column_indices.resize(sr.num_padded);
    out.values.resize(8 * sr.num_padded);
    const tcs_status s = tcs_srbcrs_download(&sr, out.row_pointer_pairs.data(), out.column_indices.data(),
                                             out.values.data(), nullptr);
    tcs_srbcrs_free(&sr, nullptr);
    detail::check(s);
    return out;
}

/// ref srbcrs.hpp:74 -- SR-BCRS -> CSR on the GPU (padding decodes to nothing).
inline CsrMatrix decode_srbcrs(const SrBcrsMatrix& m) {
    tcs_srbcrs d{};
    detail::check(tcs_srbcrs_upload(m.rows, m.cols, static_cast<tcs_precision>(m.precision),
                                    m.row_pointer_pairs.data(), m.column_indices.data(), m.values.data(), &d,
                                    nullptr));
    tcs_csr c{};
    tcs_status s = tcs_srbcrs_decode(&d, &c, nullptr);
    tcs_srbcrs_free(&d, nullptr);
    detail::check(s);
    CsrMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.row_ptr.resize(m.rows + 1);
    out.col_idx.resize(c.nnz);
    out.values.resize(c.nnz);
    s = tcs_csr_download(&c, out.row_ptr.data(), out.col_idx.data(), out.values.data(), nullptr);
    tcs_csr_free(&c, nullptr);
    detail::check(s);
    return out;
}

/// ref spmm.hpp:181 -- the same swapped kernel over the padded format.
inline SpmmResult spmm(const SrBcrsMatrix& sparse, const DenseMatrix& dense, const KernelConfig& cfg) {
    const tcs_kernel_config kc = detail::config(cfg);
    if (cfg.vector_height != 8) throw ArgumentError("swap-and-transpose path requires vector height 8");
    if (cfg.precision != sparse.precision) throw ArgumentError("config precision must match the encoded matrix");
    if (sparse.cols != dense.rows) throw ShapeError("sparse cols must equal dense rows");
    if (sparse.row_pointer_pairs.size() != 2 * ((sparse.rows + 7) / 8))
        throw FormatError("row_pointer_pairs length must be 2 * numWindows");
    SpmmResult res;
    res.output = DenseMatrix(sparse.rows, dense.cols);
    tcs_counters cn{};
    detail::check(tcs_spmm_srbcrs_host(sparse.rows, sparse.cols, static_cast<tcs_precision>(sparse.precision),
                                       sparse.row_pointer_pairs.data(), sparse.column_indices.data(),
                                       sparse.values.data(), dense.data.data(), static_cast<int64_t>(dense.rows),
                                       static_cast<int64_t>(dense.cols), res.output.data.data(), &kc, &cn, nullptr));
    res.counters = detail::counters(cn);
    return res;
}

/// ref sddmm.hpp:84 -- sampled dense-dense product over the mask pattern.
inline SddmmResult sddmm(const SddmmOperands& ops, const KernelConfig& cfg) {
    const tcs_kernel_config kc = detail::config(cfg);
    // the reference's checks, in its order (ref sddmm.hpp:86-90)
    if (cfg.precision != ops.mask.precision) throw ArgumentError("config precision must match the encoded mask");
    if (ops.a.rows != ops.mask.rows) throw ShapeError("A rows must equal mask rows");
    if (ops.b_t.rows != ops.mask.cols) throw ShapeError("B cols must equal mask cols");
    if (ops.b_t.cols != ops.a.cols) throw ShapeError("inner dimensions of A and B must agree");
    detail::require_lengths(ops.mask);
    SddmmResult res;
    res.output = ops.mask;
    tcs_counters cn{};
    detail::check(tcs_sddmm_host(ops.mask.rows, ops.mask.cols, static_cast<tcs_precision>(ops.mask.precision),
                                 ops.mask.row_pointers.data(), ops.mask.column_indices.data(),
                                 ops.mask.values.data(), ops.a.data.data(), static_cast<int64_t>(ops.a.rows),
                                 static_cast<int64_t>(ops.a.cols), ops.b_t.data.data(),
                                 static_cast<int64_t>(ops.b_t.rows), static_cast<int64_t>(ops.b_t.cols),
                                 res.output.values.data(), &kc, &cn, nullptr));
    res.counters = detail::counters(cn);
    return res;
}

}  // namespace tcsparse::gpu
