// ME-BCRS -> CSR on the GPU (ref decode_mebcrs, mebcrs.hpp:116-138): every
// stored value v != 0 (so +-0.0 fill is dropped) becomes the CSR entry
// (8w + r, column_indices[rp[w] + vector]).  Vectors ascend by column inside
// a window, so walking a window's vectors in order yields each row's entries
// already sorted -- the order csr_from_coords produces.
//
// Two warp-per-window passes: per-row counts (8 rows at once, lanes strided
// over the window's vectors), an exclusive scan into row_ptr, then the fill,
// which keeps the order with a per-row ballot over each 32-vector chunk.
#include <algorithm>
#include <cstring>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

// Value of row r at window-relative vector v of a window with nvw vectors
// (block b = v / k of width min(k, nvw - b*k); ref mebcrs.hpp:46-56).
template <typename V>
__device__ __forceinline__ float value_at(const V* vals, uint64_t vbase, uint32_t nvw, uint32_t k, uint32_t v,
                                          uint32_t r) {
    const uint32_t b = v / k, j = v % k, width = min(k, nvw - b * k);
    const V x = vals[vbase + 8ull * b * k + r * width + j];
    if constexpr (sizeof(V) == 2) return __half2float(x);
    else return x;
}

template <typename V>
__global__ void __launch_bounds__(256) decode_count(const uint32_t* __restrict__ rp, uint64_t W, uint64_t rows,
                                                    const V* __restrict__ vals, uint32_t k, uint32_t* __restrict__ cnt) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    for (uint64_t w = w0; w < W; w += nw) {
        const uint32_t base = rp[w], nvw = rp[w + 1] - base;
        uint32_t c[8] = {};
        for (uint32_t v = lane; v < nvw; v += 32)
#pragma unroll
            for (int r = 0; r < 8; ++r) c[r] += value_at(vals, 8ull * base, nvw, k, v, r) != 0.f;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) c[r] += __shfl_xor_sync(0xffffffffu, c[r], o);
            const uint64_t row = 8 * w + r;
            if (lane == 0 && row < rows) cnt[row] = c[r];
        }
    }
}

template <typename V>
__global__ void __launch_bounds__(256) decode_fill(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                                   uint64_t W, uint64_t rows, const V* __restrict__ vals, uint32_t k,
                                                   const uint32_t* __restrict__ row_ptr, uint32_t* __restrict__ col_idx,
                                                   float* __restrict__ out_vals) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    const uint32_t below = (1u << lane) - 1u;
    for (uint64_t w = w0; w < W; w += nw) {
        const uint32_t base = rp[w], nvw = rp[w + 1] - base;
        uint32_t pos[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) pos[r] = 8 * w + r < rows ? row_ptr[8 * w + r] : 0u;
        for (uint32_t v0 = 0; v0 < nvw; v0 += 32) {
            const uint32_t v = v0 + lane;
            const bool in = v < nvw;
            const uint32_t col = in ? ci[base + v] : 0u;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (8 * w + r >= rows) continue;  // warp-uniform
                const float x = in ? value_at(vals, 8ull * base, nvw, k, v, r) : 0.f;
                const bool nz = x != 0.f;
                const uint32_t m = __ballot_sync(0xffffffffu, nz);
                if (nz) {
                    const uint32_t p = pos[r] + __popc(m & below);
                    col_idx[p] = col;
                    out_vals[p] = x;
                }
                pos[r] += __popc(m);
            }
        }
    }
}

template <typename V>
void decode(const tcs_mebcrs* m, tcs_csr* out, cudaStream_t s) {
    const uint64_t W = m->num_windows, rows = m->rows;
    const V* vals = static_cast<const V*>(m->values);
    DBuf cnt(std::max<uint64_t>(1, rows) * 4, s);
    uint32_t* row_ptr = static_cast<uint32_t*>(dalloc((rows + 1) * 4, s));
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((W + 7) / 8, uint64_t(num_sms()) * 16)));
    if (W && m->num_vectors) {
        decode_count<V><<<grid, 256, 0, s>>>(m->row_pointers, W, rows, vals, m->k, cnt.as<uint32_t>());
        TCS_LAUNCHED("decode_count");
    } else if (rows) {
        TCS_CUDA(cudaMemsetAsync(cnt.p, 0, rows * 4, s));
    }
    exclusive_scan_u32(cnt.as<uint32_t>(), row_ptr, rows, s);
    uint32_t nnz = 0;
    TCS_CUDA(cudaMemcpyAsync(&nnz, row_ptr + rows, 4, cudaMemcpyDeviceToHost, s));
    TCS_CUDA(cudaStreamSynchronize(s));
    uint32_t* col_idx = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, nnz) * 4, s));
    float* out_vals = static_cast<float*>(dalloc(std::max<uint64_t>(1, nnz) * 4, s));
    if (nnz) {
        decode_fill<V><<<grid, 256, 0, s>>>(m->row_pointers, m->column_indices, W, rows, vals, m->k, row_ptr, col_idx,
                                            out_vals);
        TCS_LAUNCHED("decode_fill");
    }
    *out = tcs_csr{rows, m->cols, nnz, row_ptr, col_idx, out_vals};
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_mebcrs_decode(const tcs_mebcrs* m, tcs_csr* out, tcs_stream_t stream) {
    return guard([&] {
        check_mebcrs(m);
        if (!out) fail(TCS_ERR_ARGUMENT, "null output");
        if (m->value_dtype == TCS_DTYPE_F16) decode<__half>(m, out, st(stream));
        else decode<float>(m, out, st(stream));
    });
}

extern "C" tcs_status tcs_csr_download(const tcs_csr* m, uint32_t* row_ptr, uint32_t* col_idx, float* values,
                                       tcs_stream_t stream) {
    return guard([&] {
        if (!m) fail(TCS_ERR_ARGUMENT, "null argument");
        cudaStream_t s = st(stream);
        if (row_ptr && m->row_ptr)
            TCS_CUDA(cudaMemcpyAsync(row_ptr, m->row_ptr, (m->rows + 1) * 4, cudaMemcpyDeviceToHost, s));
        if (col_idx && m->nnz) TCS_CUDA(cudaMemcpyAsync(col_idx, m->col_idx, m->nnz * 4, cudaMemcpyDeviceToHost, s));
        if (values && m->nnz) TCS_CUDA(cudaMemcpyAsync(values, m->values, m->nnz * 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
    });
}
