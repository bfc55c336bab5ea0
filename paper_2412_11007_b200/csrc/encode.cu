// CSR -> ME-BCRS conversion as a GPU pipeline, bit-exact with the reference
// encoder (ref mebcrs.hpp:80-114, partition.hpp:40-66).
//
//   K0 csr_check     one thread per row: CSR invariants (ref matrix.hpp:31-48)
//                    + longest window (entries) -> picks the merge kernel.
//   K1 window_merge  one CTA per 8-row window: the window's 8 rows are 8
//                    sorted runs of column indices; three rounds of CTA-wide
//                    merge-path merging (keys = col<<32 | entry) give the
//                    window's entries in (column, row) order; a block scan of
//                    "first of its column" flags yields, per entry, the rank
//                    of its column among the window's distinct columns (its
//                    vector slot) and the window's vector count nv_w.
//                    Runs in shared memory (<= 2048 entries, 128 threads;
//                    <= 12288 entries, 512 threads) or, for hub windows,
//                    in a global scratch buffer with the same code.
//   K2 scan          row_pointers = exclusive scan of nv_w (u32, as the ref).
//   K3 window_scatter one CTA per window: writes column_indices and places
//                    every CSR value at 8*(rp[w]+b*k) + r*width_b + j,
//                    width_b = min(k, nv_w - b*k) (ref mebcrs.hpp:46-56), all
//                    other slots 0.  F16 storage rounds with __float2half_rn
//                    (bit-identical to ref round_to_fp16); F32 keeps raw bits.
#include <algorithm>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

constexpr uint32_t kSmallCap = 2048;    // entries per window, 128-thread CTA, 32 KB smem
constexpr uint32_t kSmallThreads = 128;
constexpr uint32_t kBigCap = 12288;     // 512-thread CTA, 192 KB smem
constexpr uint32_t kBigThreads = 512;
constexpr uint64_t kSentinel = ~0ull;

struct CheckOut {
    uint32_t max_window_entries;
    uint32_t bad;  // nonzero = first violated invariant code
};

__global__ void csr_check(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci, uint64_t rows,
                          uint64_t cols, uint64_t nnz, CheckOut* out) {
    uint32_t mx = 0, bad = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = rp[r], e = rp[r + 1];
        if (b > e) { bad = 1; continue; }
        if (e > nnz) { bad = 2; continue; }
        uint32_t prev = 0;
        for (uint32_t p = b; p < e; ++p) {
            const uint32_t c = ci[p];
            if (c >= cols) bad = 3;
            if (p > b && prev >= c) bad = 4;
            prev = c;
        }
        if ((r & 7) == 0) mx = max(mx, rp[min(r + 8, rows)] - b);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        bad = max(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out->max_window_entries, mx);
        if (bad) atomicMax(&out->bad, bad);
    }
}

// Merge adjacent pairs of sorted runs src[bnd[2q] .. bnd[2q+1]) and
// src[bnd[2q+1] .. bnd[2q+2]) into dst (same span).  Every thread produces a
// contiguous slice of the output: a merge-path binary search locates its
// start, then a sequential two-pointer merge.  Keys are unique.
__device__ void merge_pass(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, const uint32_t* bnd,
                           int nruns, uint32_t n) {
    const uint32_t nt = blockDim.x;
    const uint32_t ipt = (n + nt - 1) / nt;
    uint32_t p = min(n, threadIdx.x * ipt);
    const uint32_t pend = min(n, p + ipt);
    while (p < pend) {
        int q = 0;
        while (bnd[min(2 * q + 2, nruns)] <= p) ++q;
        const uint32_t a0 = bnd[2 * q], a1 = bnd[min(2 * q + 1, nruns)], b1 = bnd[min(2 * q + 2, nruns)];
        const int64_t la = a1 - a0, lb = b1 - a1, d = p - a0;
        int64_t lo = d - lb > 0 ? d - lb : 0, hi = d < la ? d : la;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (src[a0 + mid] < src[a1 + d - 1 - mid]) lo = mid + 1;
            else hi = mid;
        }
        int64_t i = lo, j = d - lo;
        const uint32_t end = min(pend, b1);
        uint64_t va = i < la ? src[a0 + i] : kSentinel;
        uint64_t vb = j < lb ? src[a1 + j] : kSentinel;
        for (; p < end; ++p) {
            if (va < vb) {
                dst[p] = va;
                ++i;
                va = i < la ? src[a0 + i] : kSentinel;
            } else {
                dst[p] = vb;
                ++j;
                vb = j < lb ? src[a1 + j] : kSentinel;
            }
        }
    }
}

// One window's merge + unique + rank, executed by the whole CTA.
// bufA/bufB hold >= n keys each (shared or global).
__device__ void window_sort_rank(const uint32_t* __restrict__ csr_rp, const uint32_t* __restrict__ ci,
                                 uint64_t rows, uint64_t w, uint64_t* bufA, uint64_t* bufB,
                                 uint32_t* __restrict__ tmp_cols, uint32_t* __restrict__ rank,
                                 uint32_t* __restrict__ nv_out) {
    __shared__ uint32_t bnd[9];
    __shared__ uint32_t bnd2[5];
    __shared__ uint32_t bnd3[3];
    const uint64_t r0 = 8 * w;
    const uint32_t e0 = csr_rp[r0];
    if (threadIdx.x < 9) bnd[threadIdx.x] = csr_rp[min(r0 + threadIdx.x, rows)] - e0;
    __syncthreads();
    const uint32_t n = bnd[8];
    if (threadIdx.x < 5) bnd2[threadIdx.x] = bnd[2 * threadIdx.x];
    if (threadIdx.x < 3) bnd3[threadIdx.x] = bnd[4 * threadIdx.x];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
        bufA[i] = (static_cast<uint64_t>(ci[e0 + i]) << 32) | i;
    __syncthreads();
    merge_pass(bufA, bufB, bnd, 8, n);
    __syncthreads();
    merge_pass(bufB, bufA, bnd2, 4, n);
    __syncthreads();
    merge_pass(bufA, bufB, bnd3, 2, n);
    __syncthreads();
    // bufB: entries sorted by (column, entry) -- the first entry of each
    // column run is the column's representative (ref partition.hpp:60-62:
    // sort + unique).
    const uint32_t nt = blockDim.x, ipt = (n + nt - 1) / nt;
    const uint32_t p0 = min(n, threadIdx.x * ipt), p1 = min(n, p0 + ipt);
    uint32_t cnt = 0;
    for (uint32_t p = p0; p < p1; ++p)
        cnt += (p == 0 || (bufB[p] >> 32) != (bufB[p - 1] >> 32)) ? 1u : 0u;
    uint32_t total;
    uint32_t run = dev::block_exclusive_scan(cnt, &total);
    for (uint32_t p = p0; p < p1; ++p) {
        const uint64_t key = bufB[p];
        const uint32_t col = static_cast<uint32_t>(key >> 32);
        if (p == 0 || col != static_cast<uint32_t>(bufB[p - 1] >> 32)) {
            tmp_cols[e0 + run] = col;
            ++run;
        }
        rank[e0 + static_cast<uint32_t>(key)] = run - 1;
    }
    if (threadIdx.x == 0) nv_out[w] = total;
    __syncthreads();  // bnd / buffers are reused by the next window
}

__global__ void __launch_bounds__(kSmallThreads) window_merge_small(const uint32_t* __restrict__ csr_rp,
                                                                    const uint32_t* __restrict__ ci, uint64_t rows,
                                                                    uint64_t W, uint32_t* __restrict__ tmp_cols,
                                                                    uint32_t* __restrict__ rank,
                                                                    uint32_t* __restrict__ nv_out) {
    __shared__ uint64_t bufA[kSmallCap];
    __shared__ uint64_t bufB[kSmallCap];
    for (uint64_t w = blockIdx.x; w < W; w += gridDim.x) {
        const uint32_t n = csr_rp[min(8 * w + 8, rows)] - csr_rp[8 * w];
        if (n > kSmallCap) continue;  // block-uniform
        window_sort_rank(csr_rp, ci, rows, w, bufA, bufB, tmp_cols, rank, nv_out);
    }
}

__global__ void __launch_bounds__(kBigThreads) window_merge_big(const uint32_t* __restrict__ csr_rp,
                                                                const uint32_t* __restrict__ ci, uint64_t rows,
                                                                uint64_t W, uint64_t* __restrict__ scratch,
                                                                uint32_t* __restrict__ tmp_cols,
                                                                uint32_t* __restrict__ rank,
                                                                uint32_t* __restrict__ nv_out) {
    extern __shared__ uint64_t smem_keys[];
    for (uint64_t w = blockIdx.x; w < W; w += gridDim.x) {
        const uint32_t e0 = csr_rp[8 * w];
        const uint32_t n = csr_rp[min(8 * w + 8, rows)] - e0;
        if (n <= kSmallCap) continue;
        uint64_t *a, *b;
        if (n <= kBigCap) {
            a = smem_keys;
            b = smem_keys + kBigCap;
        } else {
            a = scratch + 2ull * e0;  // window-private slice of a 2*nnz scratch
            b = a + n;
        }
        window_sort_rank(csr_rp, ci, rows, w, a, b, tmp_cols, rank, nv_out);
    }
}

template <typename V>
__device__ __forceinline__ V store_cvt(float x);
template <>
__device__ __forceinline__ float store_cvt<float>(float x) { return x; }
template <>
__device__ __forceinline__ __half store_cvt<__half>(float x) { return __float2half_rn(x); }

template <typename V>
__global__ void __launch_bounds__(256) window_scatter(const uint32_t* __restrict__ csr_rp,
                                                      const float* __restrict__ csr_vals, uint64_t rows, uint64_t W,
                                                      uint32_t k, const uint32_t* __restrict__ rp,
                                                      const uint32_t* __restrict__ tmp_cols,
                                                      const uint32_t* __restrict__ rank,
                                                      uint32_t* __restrict__ out_ci, V* __restrict__ out_vals) {
    __shared__ uint32_t rb[9];
    for (uint64_t w = blockIdx.x; w < W; w += gridDim.x) {
        const uint64_t r0 = 8 * w;
        if (threadIdx.x < 9) rb[threadIdx.x] = csr_rp[min(r0 + threadIdx.x, rows)];
        const uint32_t base = rp[w], nvw = rp[w + 1] - base;
        __syncthreads();
        const uint32_t e0 = rb[0], e1 = rb[8];
        for (uint32_t i = threadIdx.x; i < nvw; i += blockDim.x) out_ci[base + i] = tmp_cols[e0 + i];
        V* vals = out_vals + 8ull * base;
        for (uint32_t i = threadIdx.x; i < 8 * nvw; i += blockDim.x) vals[i] = store_cvt<V>(0.0f);
        __syncthreads();
        for (uint32_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            uint32_t r = 0;
#pragma unroll
            for (int q = 1; q < 8; ++q) r += (e >= rb[q]) ? 1u : 0u;
            const uint32_t v = rank[e];
            const uint32_t b = v / k, j = v - b * k;
            const uint32_t width = min(k, nvw - b * k);
            vals[static_cast<uint64_t>(b) * k * 8 + r * width + j] = store_cvt<V>(csr_vals[e]);
        }
        __syncthreads();
    }
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_mebcrs_encode(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype,
                                        tcs_mebcrs* out, tcs_stream_t stream) {
    return guard([&] {
        if (!csr || !out) fail(TCS_ERR_ARGUMENT, "null argument");
        if (precision != TCS_FP16 && precision != TCS_TF32) fail(TCS_ERR_ARGUMENT, "unknown precision");
        if (precision == TCS_TF32 && value_dtype != TCS_DTYPE_F32)
            fail(TCS_ERR_ARGUMENT, "TF32 ME-BCRS values must be stored as f32");
        if (value_dtype != TCS_DTYPE_F16 && value_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown dtype");
        if (!csr->row_ptr || (csr->nnz && (!csr->col_idx || !csr->values))) fail(TCS_ERR_ARGUMENT, "null CSR array");
        if (csr->nnz >= (1ull << 32)) fail(TCS_ERR_FORMAT, "nnz exceeds u32 row_ptr");
        cudaStream_t s = st(stream);
        const uint64_t rows = csr->rows, W = (rows + 7) / 8, nnz = csr->nnz;
        const uint32_t k = precision == TCS_FP16 ? 8 : 4;
        const int sms = num_sms();

        tcs_mebcrs m{};
        m.rows = rows;
        m.cols = csr->cols;
        m.vector_height = 8;
        m.k = k;
        m.precision = precision;
        m.value_dtype = value_dtype;
        m.num_windows = W;
        m.flags = TCS_MEBCRS_OWN_STRUCTURE | TCS_MEBCRS_OWN_VALUES;
        m.row_pointers = static_cast<uint32_t*>(dalloc((W + 1) * 4, s));

        uint32_t nv = 0;
        if (W) {
            // K0: validate + longest window
            DBuf chk(sizeof(CheckOut), s);
            TCS_CUDA(cudaMemsetAsync(chk.p, 0, sizeof(CheckOut), s));
            const int g0 = static_cast<int>(std::min<uint64_t>((rows + 255) / 256, uint64_t(sms) * 8));
            csr_check<<<g0, 256, 0, s>>>(csr->row_ptr, csr->col_idx, rows, csr->cols, nnz, chk.as<CheckOut>());
            TCS_LAUNCHED("csr_check");
            CheckOut h{};
            uint32_t last = 0;
            TCS_CUDA(cudaMemcpyAsync(&h, chk.p, sizeof(h), cudaMemcpyDeviceToHost, s));
            TCS_CUDA(cudaMemcpyAsync(&last, csr->row_ptr + rows, 4, cudaMemcpyDeviceToHost, s));
            uint32_t first = 0;
            TCS_CUDA(cudaMemcpyAsync(&first, csr->row_ptr, 4, cudaMemcpyDeviceToHost, s));
            TCS_CUDA(cudaStreamSynchronize(s));
            if (first != 0 || last != nnz) {
                dfree(m.row_pointers, s);
                fail(TCS_ERR_FORMAT, "row_ptr endpoints inconsistent with nnz");
            }
            if (h.bad) {
                dfree(m.row_pointers, s);
                static const char* msg[] = {"", "row_ptr must be nondecreasing", "row_ptr exceeds nnz",
                                            "column index out of range",
                                            "column indices must be strictly ascending within a row"};
                fail(TCS_ERR_FORMAT, msg[h.bad < 5 ? h.bad : 0]);
            }

            DBuf tmp_cols(std::max<uint64_t>(1, nnz) * 4, s), rank(std::max<uint64_t>(1, nnz) * 4, s);
            DBuf nvw(W * 4, s);
            const int g1 = static_cast<int>(std::min<uint64_t>(W, uint64_t(sms) * 16));
            window_merge_small<<<g1, kSmallThreads, 0, s>>>(csr->row_ptr, csr->col_idx, rows, W,
                                                            tmp_cols.as<uint32_t>(), rank.as<uint32_t>(),
                                                            nvw.as<uint32_t>());
            TCS_LAUNCHED("window_merge_small");
            if (h.max_window_entries > kSmallCap) {
                DBuf scratch;
                if (h.max_window_entries > kBigCap) scratch = DBuf(2 * nnz * 8, s);
                const size_t smem = 2 * kBigCap * sizeof(uint64_t);
                TCS_CUDA(cudaFuncSetAttribute(window_merge_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem)));
                const int g2 = static_cast<int>(std::min<uint64_t>(W, uint64_t(sms)));
                window_merge_big<<<g2, kBigThreads, smem, s>>>(csr->row_ptr, csr->col_idx, rows, W,
                                                                scratch.as<uint64_t>(), tmp_cols.as<uint32_t>(),
                                                                rank.as<uint32_t>(), nvw.as<uint32_t>());
                TCS_LAUNCHED("window_merge_big");
            }
            exclusive_scan_u32(nvw.as<uint32_t>(), m.row_pointers, W, s);
            TCS_CUDA(cudaMemcpyAsync(&nv, m.row_pointers + W, 4, cudaMemcpyDeviceToHost, s));
            TCS_CUDA(cudaStreamSynchronize(s));
            m.num_vectors = nv;
            const size_t vw = value_dtype == TCS_DTYPE_F16 ? 2 : 4;
            m.column_indices = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, nv) * 4, s));
            m.values = dalloc(std::max<uint64_t>(1, 8ull * nv) * vw, s);
            const int g3 = static_cast<int>(std::min<uint64_t>(W, uint64_t(sms) * 8));
            if (value_dtype == TCS_DTYPE_F16)
                window_scatter<__half><<<g3, 256, 0, s>>>(csr->row_ptr, csr->values, rows, W, k, m.row_pointers,
                                                          tmp_cols.as<uint32_t>(), rank.as<uint32_t>(),
                                                          m.column_indices, static_cast<__half*>(m.values));
            else
                window_scatter<float><<<g3, 256, 0, s>>>(csr->row_ptr, csr->values, rows, W, k, m.row_pointers,
                                                         tmp_cols.as<uint32_t>(), rank.as<uint32_t>(),
                                                         m.column_indices, static_cast<float*>(m.values));
            TCS_LAUNCHED("window_scatter");
        } else {
            TCS_CUDA(cudaMemsetAsync(m.row_pointers, 0, 4, s));
            m.column_indices = static_cast<uint32_t*>(dalloc(4, s));
            m.values = dalloc(4, s);
        }
        *out = m;
        const tcs_status rc = tcs_mebcrs_prepare(out, stream);
        if (rc != TCS_OK) {
            const std::string msg = tcs_last_error();
            tcs_mebcrs_free(out, stream);
            fail(rc, msg);
        }
    });
}

extern "C" tcs_status tcs_mebcrs_encode_host(const tcs_csr* host_csr, tcs_precision precision,
                                             tcs_dtype value_dtype, tcs_mebcrs* out, tcs_stream_t stream) {
    return guard([&] {
        if (!host_csr || !out || !host_csr->row_ptr) fail(TCS_ERR_ARGUMENT, "null argument");
        cudaStream_t s = st(stream);
        const uint64_t rows = host_csr->rows, nnz = host_csr->nnz;
        DBuf rp((rows + 1) * 4, s), ci(std::max<uint64_t>(1, nnz) * 4, s), v(std::max<uint64_t>(1, nnz) * 4, s);
        TCS_CUDA(cudaMemcpyAsync(rp.p, host_csr->row_ptr, (rows + 1) * 4, cudaMemcpyHostToDevice, s));
        if (nnz) {
            TCS_CUDA(cudaMemcpyAsync(ci.p, host_csr->col_idx, nnz * 4, cudaMemcpyHostToDevice, s));
            TCS_CUDA(cudaMemcpyAsync(v.p, host_csr->values, nnz * 4, cudaMemcpyHostToDevice, s));
        }
        tcs_csr d{rows, host_csr->cols, nnz, rp.as<uint32_t>(), ci.as<uint32_t>(), v.as<float>()};
        const tcs_status rc = tcs_mebcrs_encode(&d, precision, value_dtype, out, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
    });
}
