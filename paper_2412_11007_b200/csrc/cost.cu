// Structural cost model of one SpMM (ref analysis.hpp,
// access_pattern.hpp, footprint.hpp) evaluated on the GPU from a device
// ME-BCRS structure -- the reference's analytic counters at any matrix size
// (the reference itself needs the O(rows x cols) dense copy).
//
// For every TC block and output tile the dense-operand gather of the
// reference's warp model is replayed: the lanes' byte accesses of each load
// step (ref map_threads_rows, access_pattern.hpp:72-121, for the swapped 8x1
// path; one step of 16-byte chunks per gathered row for the 16x1 baseline,
// ref spmm.hpp:225-231 / analysis.hpp:112-121) are reduced to their touched
// 32-byte segments, which merge greedily into naturally aligned 64/128-byte
// transactions (ref count_transactions, access_pattern.hpp:135-170).  A warp
// owns a window, its lanes stride over the window's blocks.
//
//   transactions      tiles 0 and 1 extrapolated, as count_spmm_transactions
//                     (analysis.hpp:84-131) -- the `stats` report column
//   exec_*            summed over every tile, as the executing kernels'
//                     KernelCounters (spmm.hpp:146-151, :236-240)
#include <algorithm>
#include <vector>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

struct CostTotals {
    unsigned long long t0, t1;            // transactions of tiles 0 and 1
    unsigned long long exec_tx, exec_bytes, exec_useful;
    unsigned long long nonempty;          // windows with >= 1 vector
};

struct CostArgs {
    const uint32_t* rp;
    const uint32_t* ci;
    uint64_t W;
    uint32_t k;
    uint32_t vw;        // value width (2 FP16, 4 TF32)
    uint32_t tw;        // output tile width: 16 (swap8) / 8 (baseline16)
    uint64_t tiles;
    uint64_t stride;    // padded row stride in bytes = tiles * tw * vw
    int mode;           // 0 swap8 FP16 coalesced, 1 swap8 FP16 direct, 2 swap8 TF32, 3 baseline16
    CostTotals* out;
};

// Segment list of one load step (<= 16 distinct entries in every mode).
struct Segs {
    unsigned long long s[32];
    int n = 0;
    __device__ void add(unsigned long long addr, uint32_t width) {
        const unsigned long long first = addr / 32, last = (addr + width - 1) / 32;
        for (unsigned long long x = first; x <= last && n < 32; ++x)
            if (n == 0 || s[n - 1] != x) s[n++] = x;  // lanes of one row share segments
    }
    // ref count_transactions: sort + unique, then greedy 128/64/32-byte merge.
    __device__ void flush(unsigned long long& tx, unsigned long long& bytes) {
        for (int i = 1; i < n; ++i) {  // insertion sort
            const unsigned long long v = s[i];
            int j = i - 1;
            while (j >= 0 && s[j] > v) s[j + 1] = s[j], --j;
            s[j + 1] = v;
        }
        int m = 0;
        for (int i = 0; i < n; ++i)
            if (m == 0 || s[m - 1] != s[i]) s[m++] = s[i];
        auto touched = [&](unsigned long long v) {
            for (int i = 0; i < m; ++i)
                if (s[i] == v) return true;
            return false;
        };
        for (int i = 0; i < m;) {
            const unsigned long long v = s[i];
            unsigned long long span = 1;
            if (v % 4 == 0 && touched(v + 1) && touched(v + 2) && touched(v + 3)) span = 4;
            else if (v % 2 == 0 && touched(v + 1)) span = 2;
            tx += 1;
            bytes += span * 32;
            while (i < m && s[i] < v + span) ++i;
        }
        n = 0;
    }
};

// One (block, tile): transactions, transaction bytes and useful bytes.
__device__ void block_tile(const CostArgs& a, const uint32_t* cols, uint32_t width, uint64_t t,
                           unsigned long long& tx, unsigned long long& bytes, unsigned long long& useful) {
    Segs sg;
    if (a.mode == 0) {  // FP16 coalesced: lane (g,t') reads row 2t'+dr, cols 2g..2g+1 as 4 bytes
        for (uint32_t dr = 0; dr < 2; ++dr) {
            for (uint32_t tt = 0; tt < 4; ++tt) {
                const uint32_t j = 2 * tt + dr;
                if (j >= width) continue;
                const unsigned long long addr = cols[j] * a.stride + t * a.tw * a.vw;
                for (uint32_t g = 0; g < 8; ++g) sg.add(addr + 4 * g, 4);
                useful += 32;
            }
            sg.flush(tx, bytes);
        }
    } else if (a.mode == 1) {  // FP16 direct: (row 2t'+dr, col g+dc) as 2 bytes
        for (uint32_t dr = 0; dr < 2; ++dr)
            for (uint32_t dc = 0; dc <= 8; dc += 8) {
                for (uint32_t tt = 0; tt < 4; ++tt) {
                    const uint32_t j = 2 * tt + dr;
                    if (j >= width) continue;
                    const unsigned long long addr = cols[j] * a.stride + t * a.tw * a.vw;
                    for (uint32_t g = 0; g < 8; ++g) sg.add(addr + 2 * (g + dc), 2);
                    useful += 16;
                }
                sg.flush(tx, bytes);
            }
    } else if (a.mode == 2) {  // TF32 (both mappings): row t', col g+dc as 4 bytes
        for (uint32_t dc = 0; dc <= 8; dc += 8) {
            for (uint32_t j = 0; j < 4; ++j) {
                if (j >= width) continue;
                const unsigned long long addr = cols[j] * a.stride + t * a.tw * a.vw;
                for (uint32_t g = 0; g < 8; ++g) sg.add(addr + 4 * (g + dc), 4);
                useful += 32;
            }
            sg.flush(tx, bytes);
        }
    } else {  // baseline16: one step, each gathered row as 16-byte chunks
        const uint32_t len = a.tw * a.vw;
        for (uint32_t j = 0; j < width; ++j) {
            const unsigned long long addr = cols[j] * a.stride + t * len;
            for (uint32_t off = 0; off < len; off += 16) sg.add(addr + off, min(16u, len - off));
            useful += len;
        }
        sg.flush(tx, bytes);
    }
}

__global__ void cost_kernel(const CostArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long t0 = 0, t1 = 0, etx = 0, eby = 0, eus = 0, ne = 0;
    for (uint64_t w = warp; w < a.W; w += nwarps) {
        const uint32_t base = a.rp[w], nvw = a.rp[w + 1] - base;
        if (lane == 0 && nvw) ++ne;
        const uint32_t nb = (nvw + a.k - 1) / a.k;
        for (uint32_t b = lane; b < nb; b += 32) {
            uint32_t cols[8];
            const uint32_t width = min(a.k, nvw - b * a.k);
            for (uint32_t j = 0; j < width; ++j) cols[j] = a.ci[base + b * a.k + j];
            for (uint64_t t = 0; t < a.tiles; ++t) {
                unsigned long long tx = 0, by = 0, us = 0;
                block_tile(a, cols, width, t, tx, by, us);
                if (t == 0) t0 += tx;
                if (t == 1) t1 += tx;
                etx += tx;
                eby += by;
                eus += us;
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
        etx += __shfl_xor_sync(0xffffffffu, etx, o);
        eby += __shfl_xor_sync(0xffffffffu, eby, o);
        eus += __shfl_xor_sync(0xffffffffu, eus, o);
        ne += __shfl_xor_sync(0xffffffffu, ne, o);
    }
    if (lane == 0) {
        atomicAdd(&a.out->t0, t0);
        atomicAdd(&a.out->t1, t1);
        atomicAdd(&a.out->exec_tx, etx);
        atomicAdd(&a.out->exec_bytes, eby);
        atomicAdd(&a.out->exec_useful, eus);
        atomicAdd(&a.out->nonempty, ne);
    }
}

}  // namespace

void mebcrs_cost(const tcs_mebcrs* m, uint64_t nnz, int64_t n_cols, tcs_mapping mapping, tcs_cost* out,
                 cudaStream_t s) {
    check_mebcrs(m, true);
    if (!out) fail(TCS_ERR_ARGUMENT, "null argument");
    if (n_cols < 0) fail(TCS_ERR_SHAPE, "negative dimension");
    const bool swap8 = m->vector_height == 8;
    const uint64_t vh = m->vector_height, k = m->k, vw = m->precision == TCS_FP16 ? 2 : 4;
    const uint64_t tw = swap8 ? 16 : 8;
    const uint64_t tiles = (static_cast<uint64_t>(n_cols) + tw - 1) / tw;
    uint64_t blocks = m->num_blocks;
    if (!m->plan) {  // structure filled by the caller and never prepared: count blocks on the host
        std::vector<uint32_t> rp(m->num_windows + 1);
        TCS_CUDA(cudaMemcpyAsync(rp.data(), m->row_pointers, rp.size() * 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
        blocks = 0;
        for (uint64_t w = 0; w < m->num_windows; ++w) blocks += (rp[w + 1] - rp[w] + k - 1) / k;
    }
    CostTotals h{};
    if (m->num_windows) {
        DBuf tot(sizeof(CostTotals), s);
        TCS_CUDA(cudaMemsetAsync(tot.p, 0, sizeof(CostTotals), s));
        CostArgs a{m->row_pointers, m->column_indices, m->num_windows, m->k, static_cast<uint32_t>(vw),
                   static_cast<uint32_t>(tw), tiles, tiles * tw * vw,
                   !swap8 ? 3 : (vw == 4 ? 2 : (mapping == TCS_MAP_DIRECT ? 1 : 0)), tot.as<CostTotals>()};
        const uint64_t warps = std::min<uint64_t>(m->num_windows, uint64_t(num_sms()) * 64);
        cost_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(a);
        TCS_LAUNCHED("cost_kernel");
        TCS_CUDA(cudaMemcpyAsync(&h, tot.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
    }
    tcs_cost c{};
    c.mma_count = blocks * tiles;                                   // ref analysis.hpp:34-38
    c.zero_fill = vh * m->num_vectors - nnz;                        // :41-43
    c.access_bytes = blocks * tiles * (vh * k * vw + k * tw * vw)   // :58-77
                     + h.nonempty * tiles * vh * tw * vw;
    c.transactions = tiles == 0 ? 0 : tiles == 1 ? h.t0 : (tiles + 1) / 2 * h.t0 + tiles / 2 * h.t1;  // :126-130
    c.exec_transactions = h.exec_tx;
    c.exec_transaction_bytes = h.exec_bytes;
    c.exec_useful_bytes = h.exec_useful;
    c.padded_vectors = blocks * k;                                  // partition.hpp:35-36
    c.footprint_me = (m->num_windows + 1) * 4 + m->num_vectors * 4 + m->num_vectors * vh * vw;  // footprint.hpp:13-18
    c.footprint_sr = 2 * m->num_windows * 4 + c.padded_vectors * 4 + c.padded_vectors * vh * vw;  // :20-25
    *out = c;
}

}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_mebcrs_cost(const tcs_mebcrs* m, uint64_t nnz, int64_t n_cols, tcs_mapping mapping,
                                      tcs_cost* out, tcs_stream_t stream) {
    return guard([&] { mebcrs_cost(m, nnz, n_cols, mapping, out, st(stream)); });
}
