// SR-BCRS, the zero-vector padded baseline format of the paper's footprint
// ablation (ref srbcrs.hpp; Table 5), and the swapped SpMM over it
// (ref spmm.hpp:181-185, SrBlockSource :77-93).
//
// Conversion (ref encode_srbcrs, srbcrs.hpp:40-72) runs on the device from
// an ME-BCRS handle: per-window padded counts ceil(nv_w / k) * k, a scan for
// the window starts, then one thread per padded vector writes its column
// index (TCS_SR_PADDING past nv_w) and its 8 values re-laid from the
// compact width_b-wide block to the full k-wide block (zeros past nv_w).
//
// SpMM: with every window a multiple of k vectors, the SR-BCRS value array
// IS an ME-BCRS value array (width_b == k for every block), so the format
// runs through the same kernel.  The handle keeps a gather view: the window
// starts as CSR-style row pointers and a copy of the column indices with the
// padding sentinel mapped to an appended zero row of B -- the reference's
// kAbsentRow gather (spmm.hpp:86) -- so padded vectors are numerically
// inert (0 * 0).  The result equals the compact-format SpMM bit for bit when
// the sums are exact; long windows may be split at other points (the
// work-list segment follows the vector count), so real-valued partial sums
// of split windows can associate differently.
#include <algorithm>
#include <cstring>
#include <vector>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

struct SrImpl {
    tcs_mebcrs view{};  // rows, cols + 1, rp = window starts (W+1), ci = gather indices, values aliased
};

__global__ void sr_padded_counts(const uint32_t* __restrict__ rp, uint64_t W, uint32_t k, uint32_t* __restrict__ cnt) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t nv = rp[w + 1] - rp[w];
        cnt[w] = (nv + k - 1) / k * k;  // ref WindowPartition::padded_vectors / srbcrs.hpp:51
    }
}

__global__ void sr_pairs(const uint32_t* __restrict__ srp, uint64_t W, uint32_t* __restrict__ pairs) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W; w += (uint64_t)gridDim.x * blockDim.x) {
        pairs[2 * w] = srp[w];
        pairs[2 * w + 1] = srp[w + 1];
    }
}

// One thread per padded vector p: window by binary search over the padded
// starts, then column index + the 8 values of slot j (ref srbcrs.hpp:53-69).
template <typename V>
__global__ void sr_fill(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci, const V* __restrict__ vals,
                        const uint32_t* __restrict__ srp, uint64_t W, uint64_t P, uint32_t k, uint32_t gather_sentinel,
                        uint32_t* __restrict__ sci, uint32_t* __restrict__ gci, V* __restrict__ svals) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < P; p += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = W;  // largest w with srp[w] <= p (and srp[w+1] > p)
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (srp[mid] <= p) lo = mid; else hi = mid;
        }
        const uint64_t w = lo;
        const uint32_t j = static_cast<uint32_t>(p - srp[w]);
        const uint32_t base = rp[w], nv = rp[w + 1] - base;
        const uint32_t b = j / k, jj = j % k;
        const uint64_t out = 8ull * (srp[w] + b * k) + jj;
        if (j < nv) {
            const uint32_t c = ci[base + j];
            sci[p] = c;
            gci[p] = c;
            const uint32_t width = min(k, nv - b * k);
            const uint64_t in = 8ull * (base + b * k) + jj;
#pragma unroll
            for (int r = 0; r < 8; ++r) svals[out + r * k] = vals[in + r * width];
        } else {
            sci[p] = TCS_SR_PADDING;
            gci[p] = gather_sentinel;
#pragma unroll
            for (int r = 0; r < 8; ++r) svals[out + r * k] = V(0);
        }
    }
}

__global__ void sr_gather_view(const uint32_t* __restrict__ sci, uint64_t P, uint32_t gather_sentinel,
                               uint32_t* __restrict__ gci) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < P; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = sci[p];
        gci[p] = c == TCS_SR_PADDING ? gather_sentinel : c;
    }
}

int grid_for(uint64_t n) { return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16))); }

void check_sr(const tcs_srbcrs* m) {
    if (!m) fail(TCS_ERR_ARGUMENT, "null SR-BCRS handle");
    if (m->vector_height != 8) fail(TCS_ERR_ARGUMENT, "SR-BCRS vector height must be 8");
    if (m->precision != TCS_FP16 && m->precision != TCS_TF32) fail(TCS_ERR_ARGUMENT, "unknown precision");
    if (m->k != (m->precision == TCS_FP16 ? 8u : 4u)) fail(TCS_ERR_FORMAT, "block width k does not match precision");
    if (!m->impl) fail(TCS_ERR_ARGUMENT, "SR-BCRS handle not prepared");
}

// Allocates the handle's arrays + gather view for `P` padded vectors over
// window starts `srp` (device, W+1, owned by the view from here on).
void sr_alloc(tcs_srbcrs* out, uint64_t rows, uint64_t cols, tcs_precision prec, tcs_dtype vdt, uint64_t W, uint64_t P,
              uint32_t* srp, cudaStream_t s) {
    const size_t esz = vdt == TCS_DTYPE_F16 ? 2 : 4;
    tcs_srbcrs m{};
    m.rows = rows;
    m.cols = cols;
    m.vector_height = 8;
    m.k = prec == TCS_FP16 ? 8 : 4;
    m.precision = prec;
    m.value_dtype = vdt;
    m.num_windows = W;
    m.num_padded = P;
    m.row_pointer_pairs = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, 2 * W) * 4, s));
    m.column_indices = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, P) * 4, s));
    m.values = dalloc(std::max<uint64_t>(1, 8 * P) * esz, s);
    auto* impl = new SrImpl;
    tcs_mebcrs& v = impl->view;
    v.rows = rows;
    v.cols = cols + 1;  // + the zero row padded vectors gather
    v.vector_height = 8;
    v.k = m.k;
    v.precision = prec;
    v.value_dtype = vdt;
    v.num_windows = W;
    v.num_vectors = P;
    v.row_pointers = srp;
    v.column_indices = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, P) * 4, s));
    v.values = m.values;
    v.flags = TCS_MEBCRS_OWN_STRUCTURE;  // srp + gather indices; values belong to the SR handle
    m.impl = impl;
    *out = m;
}

void sr_release(tcs_srbcrs* m, cudaStream_t s) {
    if (!m) return;
    dfree(m->row_pointer_pairs, s);
    dfree(m->column_indices, s);
    dfree(m->values, s);
    if (auto* impl = static_cast<SrImpl*>(m->impl)) {
        tcs_mebcrs_free(&impl->view, reinterpret_cast<tcs_stream_t>(s));
        delete impl;
    }
    std::memset(m, 0, sizeof(*m));
}

void sr_prepare(tcs_srbcrs* m, cudaStream_t s) {
    tcs_status rc = tcs_mebcrs_prepare(&static_cast<SrImpl*>(m->impl)->view, reinterpret_cast<tcs_stream_t>(s));
    if (rc != TCS_OK) fail(rc, tcs_last_error());
}

void from_mebcrs(const tcs_mebcrs* me, tcs_srbcrs* out, cudaStream_t s) {
    check_mebcrs(me);
    if (!out) fail(TCS_ERR_ARGUMENT, "null output handle");
    const uint64_t W = me->num_windows;
    DBuf cnt(std::max<uint64_t>(1, W) * 4, s);
    uint32_t* srp = static_cast<uint32_t*>(dalloc((W + 1) * 4, s));
    if (W) {
        sr_padded_counts<<<grid_for(W), 256, 0, s>>>(me->row_pointers, W, me->k, cnt.as<uint32_t>());
        TCS_LAUNCHED("sr_padded_counts");
    }
    // the padded total must fit the reference's u32 pointers
    const uint64_t bound = me->num_vectors + W * (me->k - 1);
    if (bound >= (1ull << 32)) {
        dfree(srp, s);
        fail(TCS_ERR_FORMAT, "padded vector count exceeds u32 row pointers");
    }
    exclusive_scan_u32(cnt.as<uint32_t>(), srp, W, s);
    uint32_t P32 = 0;
    TCS_CUDA(cudaMemcpyAsync(&P32, srp + W, 4, cudaMemcpyDeviceToHost, s));
    TCS_CUDA(cudaStreamSynchronize(s));
    const uint64_t P = P32;
    tcs_srbcrs m{};
    sr_alloc(&m, me->rows, me->cols, me->precision, me->value_dtype, W, P, srp, s);
    try {
        auto* impl = static_cast<SrImpl*>(m.impl);
        if (W) {
            sr_pairs<<<grid_for(W), 256, 0, s>>>(srp, W, m.row_pointer_pairs);
            TCS_LAUNCHED("sr_pairs");
        }
        if (P) {
            const uint32_t zero_row = static_cast<uint32_t>(me->cols);
            if (me->value_dtype == TCS_DTYPE_F16)
                sr_fill<unsigned short><<<grid_for(P), 256, 0, s>>>(
                    me->row_pointers, me->column_indices, static_cast<const unsigned short*>(me->values), srp, W, P,
                    me->k, zero_row, m.column_indices, impl->view.column_indices, static_cast<unsigned short*>(m.values));
            else
                sr_fill<uint32_t><<<grid_for(P), 256, 0, s>>>(
                    me->row_pointers, me->column_indices, static_cast<const uint32_t*>(me->values), srp, W, P, me->k,
                    zero_row, m.column_indices, impl->view.column_indices, static_cast<uint32_t*>(m.values));
            TCS_LAUNCHED("sr_fill");
        }
        sr_prepare(&m, s);
    } catch (...) {
        sr_release(&m, s);
        throw;
    }
    *out = m;
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_srbcrs_from_mebcrs(const tcs_mebcrs* me, tcs_srbcrs* out, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_srbcrs_from_mebcrs"); from_mebcrs(me, out, st(stream)); });
}

extern "C" tcs_status tcs_srbcrs_encode(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype,
                                        tcs_srbcrs* out, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_srbcrs_encode");
        tcs_mebcrs me{};
        tcs_status rc = tcs_mebcrs_encode(csr, precision, value_dtype, &me, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        struct Free {
            tcs_mebcrs* m;
            tcs_stream_t s;
            ~Free() { tcs_mebcrs_free(m, s); }
        } fr{&me, stream};
        from_mebcrs(&me, out, st(stream));
    });
}

extern "C" tcs_status tcs_srbcrs_upload(uint64_t rows, uint64_t cols, tcs_precision precision,
                                        const uint32_t* row_pointer_pairs, const uint32_t* column_indices,
                                        const float* values, tcs_srbcrs* out, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_srbcrs_upload");
        if (!out || (rows && !row_pointer_pairs)) fail(TCS_ERR_ARGUMENT, "null argument");
        if (precision != TCS_FP16 && precision != TCS_TF32) fail(TCS_ERR_ARGUMENT, "unknown precision");
        cudaStream_t s = st(stream);
        const uint32_t k = precision == TCS_FP16 ? 8 : 4;
        const uint64_t W = (rows + 7) / 8;
        std::vector<uint32_t> srp(W + 1, 0);
        for (uint64_t w = 0; w < W; ++w) {
            const uint32_t b = row_pointer_pairs[2 * w], e = row_pointer_pairs[2 * w + 1];
            if (b != (w ? row_pointer_pairs[2 * w - 1] : 0u))
                fail(TCS_ERR_FORMAT, "SR-BCRS windows must be stored back to back");
            if (e < b || (e - b) % k) fail(TCS_ERR_FORMAT, "SR-BCRS window length must be a multiple of k");
            srp[w] = b;
            srp[w + 1] = e;
        }
        const uint64_t P = srp[W];
        for (uint64_t p = 0; p < P; ++p)
            if (column_indices[p] != TCS_SR_PADDING && column_indices[p] >= cols)
                fail(TCS_ERR_FORMAT, "column index out of range");
        uint32_t* dsrp = static_cast<uint32_t*>(dalloc((W + 1) * 4, s));
        TCS_CUDA(cudaMemcpyAsync(dsrp, srp.data(), (W + 1) * 4, cudaMemcpyHostToDevice, s));
        tcs_srbcrs m{};
        sr_alloc(&m, rows, cols, precision, TCS_DTYPE_F32, W, P, dsrp, s);
        try {
            if (W)
                TCS_CUDA(cudaMemcpyAsync(m.row_pointer_pairs, row_pointer_pairs, 2 * W * 4, cudaMemcpyHostToDevice, s));
            if (P) {
                TCS_CUDA(cudaMemcpyAsync(m.column_indices, column_indices, P * 4, cudaMemcpyHostToDevice, s));
                TCS_CUDA(cudaMemcpyAsync(m.values, values, 8 * P * 4, cudaMemcpyHostToDevice, s));
                sr_gather_view<<<grid_for(P), 256, 0, s>>>(m.column_indices, P, static_cast<uint32_t>(cols),
                                                           static_cast<SrImpl*>(m.impl)->view.column_indices);
                TCS_LAUNCHED("sr_gather_view");
            }
            sr_prepare(&m, s);
        } catch (...) {
            sr_release(&m, s);
            throw;
        }
        *out = m;
    });
}

extern "C" tcs_status tcs_srbcrs_download(const tcs_srbcrs* m, uint32_t* row_pointer_pairs, uint32_t* column_indices,
                                          float* values, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_srbcrs_download");
        check_sr(m);
        cudaStream_t s = st(stream);
        if (row_pointer_pairs && m->num_windows)
            TCS_CUDA(cudaMemcpyAsync(row_pointer_pairs, m->row_pointer_pairs, 2 * m->num_windows * 4,
                                     cudaMemcpyDeviceToHost, s));
        if (column_indices && m->num_padded)
            TCS_CUDA(cudaMemcpyAsync(column_indices, m->column_indices, m->num_padded * 4, cudaMemcpyDeviceToHost, s));
        if (values && m->num_padded) {
            const uint64_t n = 8 * m->num_padded;
            if (m->value_dtype == TCS_DTYPE_F32) {
                TCS_CUDA(cudaMemcpyAsync(values, m->values, n * 4, cudaMemcpyDeviceToHost, s));
            } else {
                DBuf wide(n * 4, s);
                pad_convert(m->values, TCS_DTYPE_F16, (int64_t)n, wide.p, TCS_DTYPE_F32, (int64_t)n, 1, (int64_t)n,
                            (int64_t)n, s);
                TCS_CUDA(cudaMemcpyAsync(values, wide.p, n * 4, cudaMemcpyDeviceToHost, s));
            }
        }
        TCS_CUDA(cudaStreamSynchronize(s));
    });
}

extern "C" tcs_status tcs_srbcrs_free(tcs_srbcrs* m, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_srbcrs_free"); sr_release(m, st(stream)); });
}

extern "C" tcs_status tcs_spmm_srbcrs(const tcs_srbcrs* A, const void* b, tcs_dtype b_dtype, int64_t ldb,
                                      int64_t b_rows, int64_t n, float* c, int64_t ldc, const tcs_kernel_config* cfg,
                                      tcs_counters* counters, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_srbcrs");
        if (!cfg) fail(TCS_ERR_ARGUMENT, "null kernel config");
        // ref spmm.hpp:106-109 (spmm_swapped's checks, shared by both formats)
        if (cfg->vector_height != 8) fail(TCS_ERR_ARGUMENT, "swap-and-transpose path requires vector height 8");
        check_sr(A);
        if (cfg->precision != A->precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded matrix");
        if (static_cast<int64_t>(A->cols) != b_rows) fail(TCS_ERR_SHAPE, "sparse cols must equal dense rows");
        if (n < 0 || b_rows < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        if (n > 0 && b_rows > 0 && (!b || ldb < n)) fail(TCS_ERR_ARGUMENT, "bad dense buffer / ldb");
        if (b_dtype != TCS_DTYPE_F16 && b_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown dtype");
        if (A->precision == TCS_TF32 && b_dtype != TCS_DTYPE_F32)
            fail(TCS_ERR_ARGUMENT, "TF32 SpMM needs an f32 dense operand");
        cudaStream_t s = st(stream);
        // B with the appended zero row (the padded vectors' gather target),
        // feature-padded as the kernel wants it.
        const int64_t npad = n <= 32 ? 32 : n <= 64 ? 64 : (n + 127) / 128 * 128;
        const tcs_dtype need = A->precision == TCS_FP16 ? TCS_DTYPE_F16 : TCS_DTYPE_F32;
        const size_t esz = need == TCS_DTYPE_F16 ? 2 : 4;
        DBuf bext(static_cast<size_t>(b_rows + 1) * npad * esz, s);
        if (n > 0 && b_rows > 0) pad_convert(b, b_dtype, ldb, bext.p, need, npad, b_rows, n, npad, s);
        TCS_CUDA(cudaMemsetAsync(static_cast<char*>(bext.p) + static_cast<size_t>(b_rows) * npad * esz, 0, npad * esz, s));
        const tcs_status rc = tcs_spmm(&static_cast<SrImpl*>(A->impl)->view, bext.p, need, npad, b_rows + 1, n, c, ldc,
                                       cfg, counters, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
    });
}

extern "C" tcs_status tcs_spmm_srbcrs_host(uint64_t rows, uint64_t cols, tcs_precision precision,
                                           const uint32_t* row_pointer_pairs, const uint32_t* column_indices,
                                           const float* values, const float* b, int64_t b_rows, int64_t n, float* c,
                                           const tcs_kernel_config* cfg, tcs_counters* counters,
                                           tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_srbcrs_host");
        if (!cfg) fail(TCS_ERR_ARGUMENT, "null kernel config");
        if (cfg->vector_height != 8) fail(TCS_ERR_ARGUMENT, "swap-and-transpose path requires vector height 8");
        if (cfg->precision != precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded matrix");
        if (static_cast<int64_t>(cols) != b_rows) fail(TCS_ERR_SHAPE, "sparse cols must equal dense rows");
        cudaStream_t s = st(stream);
        tcs_srbcrs m{};
        tcs_status rc = tcs_srbcrs_upload(rows, cols, precision, row_pointer_pairs, column_indices, values, &m, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        struct Free {
            tcs_srbcrs* m;
            tcs_stream_t s;
            ~Free() { tcs_srbcrs_free(m, s); }
        } fr{&m, stream};
        DBuf db(std::max<int64_t>(1, b_rows * n) * 4, s), dc(std::max<uint64_t>(1, rows * n) * 4, s);
        if (b_rows > 0 && n > 0) TCS_CUDA(cudaMemcpyAsync(db.p, b, b_rows * n * 4, cudaMemcpyHostToDevice, s));
        rc = tcs_spmm_srbcrs(&m, db.p, TCS_DTYPE_F32, n, b_rows, n, dc.as<float>(), n, cfg, counters, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        if (rows > 0 && n > 0) TCS_CUDA(cudaMemcpyAsync(c, dc.p, rows * n * 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
    });
}

// ref decode_srbcrs (srbcrs.hpp:74-90): padded vectors hold zero values, so
// decoding the gather view (padding -> the extra zero row `cols`) drops them
// like every other stored zero.
extern "C" tcs_status tcs_srbcrs_decode(const tcs_srbcrs* m, tcs_csr* out, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_srbcrs_decode");
        check_sr(m);
        if (!out) fail(TCS_ERR_ARGUMENT, "null output");
        tcs_status rc = tcs_mebcrs_decode(&static_cast<SrImpl*>(m->impl)->view, out, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        out->cols = m->cols;
    });
}
