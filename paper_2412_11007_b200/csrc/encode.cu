// CSR -> ME-BCRS conversion as a GPU pipeline, bit-exact with the reference
// encoder (ref mebcrs.hpp:80-114, partition.hpp:40-66).
//
// The reference partitions each 8-row window by concatenating its rows'
// column lists, sorting and de-duplicating (ref partition.hpp:55-64); the
// k-th distinct column is vector slot k (ascending).  Here every window is
// one CTA task and the per-entry output is the RANK of its column among the
// window's distinct columns:
//
//   K0 window_stats   thread per window: row_ptr invariants (ref
//                     matrix.hpp:31-48) and the longest window -> kernel pick.
//   K1 window ranks, one of:
//      window_sort    <= 2048 entries (128 thr) / <= 12288 (512 thr, 192 KB smem)
//                     / longer (global scratch): the window's 8 rows are 8
//                     sorted runs; three rounds of CTA-wide merge-path merging
//                     (keys col<<32 | entry) + a block scan of "first of its
//                     column" flags give each entry's rank and nv_w.
//      window_bitmap  long windows when the column space fits shared memory
//                     (<= 819,200 columns): set one bit per column, prefix-
//                     popcount the words -> rank(c) = prefix[c/32] +
//                     popc(word & below(c)).  O(cols/32 + entries) per window.
//                     Both validate the column indices of their window (range,
//                     strictly ascending within a row).
//   K2 scan           row_pointers = exclusive scan of nv_w (u32, as the ref).
//   K3 window_scatter CTA per window: column_indices (each entry stores its
//                     column at slot rank; duplicates store the same value),
//                     and every CSR value to
//                     8*(rp[w]+b*k) + r*width_b + j, width_b = min(k, nv_w-b*k)
//                     (ref mebcrs.hpp:46-56); all other slots 0.  F16 storage
//                     rounds with __float2half_rn (== ref round_to_fp16, checked
//                     exhaustively on device by the tests); F32 keeps raw bits.
#include <algorithm>
#include <cstddef>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

#ifndef TCS_ENC_TINY_CAP
#define TCS_ENC_TINY_CAP 256
#endif
constexpr uint32_t kTinyCap = TCS_ENC_TINY_CAP;  // entries per window, one warp (window_sort_warp)
constexpr int kTinyWarps = 8;           // warps per CTA of window_sort_warp
constexpr uint32_t kSmallCap = 2048;    // entries per window, 128-thread CTA, 32 KB smem
constexpr uint32_t kSmallThreads = 128;
constexpr uint32_t kBigCap = 12288;     // medium / huge class boundary (entries)
// window_sort_big (column spaces too wide for the bitmap): windows of up to
// kSortCap entries merge in shared memory (2 x 8 B per entry), longer ones in
// global scratch
#ifndef TCS_ENC_SORT_CAP
#define TCS_ENC_SORT_CAP 12288
#endif
#ifndef TCS_ENC_SORT_THREADS
#define TCS_ENC_SORT_THREADS 512
#endif
constexpr uint32_t kSortCap = TCS_ENC_SORT_CAP;
#ifndef TCS_ENC_SORT_SPLIT
#define TCS_ENC_SORT_SPLIT 6144
#endif
constexpr uint32_t kSortCapA = TCS_ENC_SORT_SPLIT;  // 0: one launch
// hub windows of wide column spaces ranked with a global-memory bitmap
// (A/B knob; 0 = merged in global scratch)
#ifndef TCS_ENC_HUB_BITMAP
#define TCS_ENC_HUB_BITMAP 1
#endif
constexpr uint32_t kBigThreads = TCS_ENC_SORT_THREADS;
// the global-memory hub bitmap's popcount / prefix passes as coalesced warp
// scans (A/B knob; 0 = thread-contiguous runs, as the shared-memory bitmap)
#ifndef TCS_ENC_GBM_WARPSCAN
#define TCS_ENC_GBM_WARPSCAN 1
#endif
#ifndef TCS_ENC_BITMAP_THREADS
#define TCS_ENC_BITMAP_THREADS 512
#endif
constexpr uint32_t kBitmapThreads = TCS_ENC_BITMAP_THREADS;
constexpr uint32_t kBitmapMaxWords = 25600;
// resident CTAs per SM the register budget is sized for (C3's 233 K-column
// bitmap + prefix take 58 KB of shared memory, so three fit)
#ifndef TCS_ENC_BITMAP_MINB
#define TCS_ENC_BITMAP_MINB 3
#endif
constexpr int kBitmapMinBlocks = TCS_ENC_BITMAP_MINB;
#ifndef TCS_ENC_BITMAP_KEEP
#define TCS_ENC_BITMAP_KEEP 1
#endif
constexpr bool kBitmapKeep = TCS_ENC_BITMAP_KEEP;
// column_indices written by the entries (every entry stores its column at
// slot base + rank; entries sharing a column store the same value) instead of
// a copy of the rank kernels' distinct-column list: the bitmap ranking then
// writes no column list at all, and the CTA scatter has no copy pass
#ifndef TCS_ENC_COLS_FROM_ENTRIES
#define TCS_ENC_COLS_FROM_ENTRIES 1
#endif
constexpr bool kColsFromEntries = TCS_ENC_COLS_FROM_ENTRIES;
#ifndef TCS_ENC_BITMAP_U
#define TCS_ENC_BITMAP_U 4
#endif
constexpr int kBitmapU = TCS_ENC_BITMAP_U;  // entries per thread in flight (window_bitmap)  // 2 x 100 KB of smem -> <= 819,200 columns
constexpr uint64_t kSentinel = ~0ull;

struct CheckOut {
    uint32_t max_window_entries;
    uint32_t bad;  // nonzero = violated invariant code (see kBadMsg)
    // window lists by size class (K0): small (<= kSmallCap entries) in
    // `small`, huge (> kBigCap) from the front and medium from the back of
    // `big` -- so the big-window kernels start the longest windows first and
    // no kernel walks (and skips) the windows of another class
    uint32_t n_small, n_medium, n_huge;
    uint32_t n_tiny;  // tiny (<= kTinyCap entries) from the front of `small`, small from its back
    // dynamic window queues of the big-window kernels (a hub window of 10^5+
    // entries must not delay the windows behind it on a fixed CTA stride)
    uint32_t next_sort_big, next_bitmap, next_scatter_big;
    uint32_t next_sort_big2;  // window_sort_big's second (large-window) launch
    // set by the F16 scatter when a nonzero f32 value rounds to a binary16
    // zero (0 < |v| <= 2^-25): the reference still samples it in SDDMM
    // (ref sddmm.hpp:131 tests the f32 value), so the handle gets exact
    // liveness bytes built from the f32 CSR values
    uint32_t tiny;
    // scatter work units of the huge windows: one per (window, value tile),
    // tile_off = their exclusive prefix over the huge list (huge_tile_prefix)
    uint32_t huge_tiles;
};

// CTA-wide queue claim: thread 0 takes the next index, every thread gets it.
__device__ __forceinline__ uint32_t cta_next(uint32_t* counter) {
    __shared__ uint32_t s_next;
    __syncthreads();  // the previous claim has been read by every thread
    if (threadIdx.x == 0) s_next = atomicAdd(counter, 1u);
    __syncthreads();
    return s_next;
}

// i-th window of the big list: huge ones first (front), then medium (back).
__device__ __forceinline__ uint32_t big_window(const uint32_t* big, uint64_t W, uint32_t n_huge, uint32_t i) {
    return i < n_huge ? big[i] : big[W - 1 - (i - n_huge)];
}

// Appends w to a list with one atomic per warp and class.
__device__ __forceinline__ void list_push(bool mine, uint32_t w, uint32_t* counter, uint32_t* list, bool from_back,
                                          uint64_t W) {
    const uint32_t m = __ballot_sync(0xffffffffu, mine);
    if (!m) return;
    const uint32_t lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (mine) {
        const uint32_t idx = base + __popc(m & ((1u << lane) - 1u));
        list[from_back ? W - 1 - idx : idx] = w;
    }
}

// nvw_zero (pipelined encode): every window's vector count starts at 0, so
// a window that fails validation (in no list) scans as empty.
template <int VH>
__global__ void window_stats(const uint32_t* __restrict__ rp, uint64_t rows, uint64_t W, uint64_t nnz,
                             CheckOut* out, uint32_t* __restrict__ small, uint32_t* __restrict__ big,
                             uint32_t* __restrict__ nvw_zero) {
    uint32_t mx = 0, bad = 0;
    const uint64_t W32 = (W + 31) / 32 * 32;  // whole warps iterate (ballots below)
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W32; w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t n = 0;
        bool ok = false;
        if (nvw_zero && w < W) nvw_zero[w] = 0u;
        if (w < W) {
            const uint64_t r0 = VH * w, r1 = min(r0 + VH, rows);
            uint32_t prev = rp[r0];
            bool wbad = false;
            for (uint64_t r = r0 + 1; r <= r1; ++r) {
                const uint32_t x = rp[r];
                if (x < prev) bad = max(bad, 1u), wbad = true;
                prev = x;
            }
            if (prev > nnz) bad = max(bad, 2u), wbad = true;
            if (!wbad) {
                n = prev - rp[r0];
                mx = max(mx, n);
                ok = true;
            }
        }
        list_push(ok && n <= kTinyCap, static_cast<uint32_t>(w), &out->n_tiny, small, false, W);
        list_push(ok && n > kTinyCap && n <= kSmallCap, static_cast<uint32_t>(w), &out->n_small, small, true, W);
        list_push(ok && n > kBigCap, static_cast<uint32_t>(w), &out->n_huge, big, false, W);
        list_push(ok && n > kSmallCap && n <= kBigCap, static_cast<uint32_t>(w), &out->n_medium, big, true, W);
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

// Column index i (window-local) of the window whose row boundaries are rb[0..VH]:
// in range and strictly greater than its predecessor in the same row.
template <int VH>
__device__ __forceinline__ uint32_t check_col(const uint32_t* __restrict__ ci, uint32_t e0, uint32_t i, uint32_t c,
                                              const uint32_t* rb, uint64_t cols) {
    uint32_t bad = c >= cols ? 3u : 0u;
    bool row_start = false;
#pragma unroll
    for (int r = 0; r < VH; ++r) row_start |= (i == rb[r]);
    if (!row_start && __ldg(ci + e0 + i - 1) >= c) bad = 4u;
    return bad;
}

// Merge adjacent pairs of sorted runs src[bnd[2q] .. bnd[2q+1]) and
// src[bnd[2q+1] .. bnd[2q+2]) into dst (same span).  Every thread produces a
// contiguous slice of the output: a merge-path binary search locates its
// start, then a sequential two-pointer merge.  Keys are unique.
__device__ __forceinline__ void merge_pass(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, const uint32_t* bnd,
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

// One window's merge + unique + rank, executed by the whole CTA: the VH
// rows are VH sorted runs, merged pairwise in log2(VH) passes.
// bufA/bufB hold >= n keys each (shared or global).
template <int VH>
__device__ __forceinline__ void window_sort_rank(const uint32_t* __restrict__ csr_rp, const uint32_t* __restrict__ ci,
                                 uint64_t rows, uint64_t cols, uint64_t w, uint64_t* bufA, uint64_t* bufB,
                                 uint32_t* __restrict__ tmp_cols, uint32_t* __restrict__ rank,
                                 uint32_t* __restrict__ nv_out, CheckOut* chk) {
    __shared__ uint32_t bnd[2 * VH + 8];  // run boundaries of every pass: VH+1, VH/2+1, ..., 2 entries
    const uint64_t r0 = VH * w;
    const uint32_t e0 = csr_rp[r0];
    if (threadIdx.x <= VH) bnd[threadIdx.x] = csr_rp[min(r0 + threadIdx.x, rows)] - e0;
    __syncthreads();
    const uint32_t n = bnd[VH];
    {
        int off = VH + 1;
        for (int runs = VH / 2; runs >= 1; runs /= 2) {  // boundaries of the pass producing `runs` runs
            if (threadIdx.x <= runs) bnd[off + threadIdx.x] = bnd[threadIdx.x * (VH / runs)];
            off += runs + 1;
        }
    }
    uint32_t bad = 0;
    {
        // 4 entries per thread in flight; the row-order predecessor is lane
        // - 1's column (consecutive lanes hold consecutive entries), loaded
        // only by lane 0.  Warp-uniform trip count (the shuffle needs every lane).
        constexpr int U = 4;
        const uint32_t lane = threadIdx.x & 31, nt = blockDim.x;
        for (uint32_t i0 = threadIdx.x; i0 - lane < n; i0 += U * nt) {
            uint32_t c[U], cp0[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * nt;
                c[u] = i < n ? ci[e0 + i] : 0xFFFFFFFFu;
                cp0[u] = lane == 0 && i < n && i > 0 ? ci[e0 + i - 1] : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * nt;
                uint32_t cp = __shfl_up_sync(0xffffffffu, c[u], 1);
                if (lane == 0) cp = cp0[u];
                if (i >= n) continue;
                uint32_t b = c[u] >= cols ? 3u : 0u;
                if (i > 0 && cp >= c[u]) {
                    bool row_start = false;
#pragma unroll
                    for (int r = 1; r < VH; ++r) row_start |= (i == bnd[r]);
                    if (!row_start) b = 4u;
                }
                bad = max(bad, b);
                // an out-of-range column (reported via chk->bad) must not reach the
                // output: the pipelined encode multiplies before the host sees the flag
                bufA[i] = (static_cast<uint64_t>(c[u] < cols ? c[u] : 0u) << 32) | i;
            }
        }
    }
    if (bad) atomicMax(&chk->bad, bad);
    __syncthreads();
    {
        int off = 0;
        for (int runs = VH; runs > 1; runs /= 2) {
            merge_pass(bufA, bufB, bnd + off, runs, n);
            __syncthreads();
            uint64_t* t = bufA;
            bufA = bufB;
            bufB = t;
            off += runs + 1;
        }
    }
    bufB = bufA;  // the merged keys
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
            if (!kColsFromEntries) tmp_cols[e0 + run] = col;  // else the scatter's entries write them
            ++run;
        }
        rank[e0 + static_cast<uint32_t>(key)] = run - 1;
    }
    if (threadIdx.x == 0) nv_out[w] = total;
    __syncthreads();  // bnd / buffers are reused by the next window
}

template <int VH>
__global__ void __launch_bounds__(kSmallThreads) window_sort_small(const uint32_t* __restrict__ csr_rp,
                                                                   const uint32_t* __restrict__ ci, uint64_t rows,
                                                                   uint64_t cols, uint64_t W,
                                                                   uint32_t* __restrict__ tmp_cols,
                                                                   uint32_t* __restrict__ rank,
                                                                   uint32_t* __restrict__ nv_out, CheckOut* chk,
                                                                   const uint32_t* __restrict__ small) {
    __shared__ uint64_t bufA[kSmallCap];
    __shared__ uint64_t bufB[kSmallCap];
    const uint32_t n_small = chk->n_small;  // class counts come from window_stats on the device
    for (uint32_t i = blockIdx.x; i < n_small; i += gridDim.x)  // small windows sit at the back of the list
        window_sort_rank<VH>(csr_rp, ci, rows, cols, small[W - 1 - i], bufA, bufB, tmp_cols, rank, nv_out, chk);
}

// Tiny windows (<= kTinyCap entries, most of an R-MAT graph's 10^6 windows):
// one warp per window, no CTA barriers.  The VH rows are sorted runs staged
// in shared memory; an entry's position in the stable (column, row) merge is
// its offset in its own row plus, per other row, the number of entries with
// a smaller column (a larger-or-equal one for rows above it) -- binary
// searches.  The merged columns then give the first-occurrence flags, whose
// warp prefix is the rank (ref partition.hpp:55-64: sort + unique).
template <int VH>
__global__ void __launch_bounds__(kTinyWarps * 32) window_sort_warp(const uint32_t* __restrict__ csr_rp,
                                                                    const uint32_t* __restrict__ ci, uint64_t rows,
                                                                    uint64_t cols, uint32_t* __restrict__ tmp_cols,
                                                                    uint32_t* __restrict__ rank,
                                                                    uint32_t* __restrict__ nv_out, CheckOut* chk,
                                                                    const uint32_t* __restrict__ tiny) {
    constexpr uint32_t kPer = kTinyCap / 32;  // entries per lane
    const uint32_t n_tiny = chk->n_tiny;
    __shared__ uint32_t s_col[kTinyWarps][kTinyCap];
    __shared__ uint32_t s_mrg[kTinyWarps][kTinyCap];
    __shared__ uint32_t s_rb[kTinyWarps][VH + 1];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* col = s_col[wid];
    uint32_t* mrg = s_mrg[wid];
    uint32_t* rb = s_rb[wid];
    uint32_t bad = 0;
    for (uint32_t i = blockIdx.x * kTinyWarps + wid; i < n_tiny; i += gridDim.x * kTinyWarps) {
        const uint64_t w = tiny[i], r0 = VH * w;
        uint32_t b = 0;
        if (lane <= VH) b = __ldg(csr_rp + min(r0 + lane, rows));
        const uint32_t e0 = __shfl_sync(0xffffffffu, b, 0);
        if (lane <= VH) rb[lane] = b - e0;
        const uint32_t n = __shfl_sync(0xffffffffu, b, VH) - e0;
        for (uint32_t j = lane; j < n; j += 32) col[j] = __ldg(ci + e0 + j);
        __syncwarp();
        uint32_t pos[kPer];
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) {
            const uint32_t j = lane + 32 * k;
            pos[k] = 0;
            if (j >= n) continue;
            const uint32_t c = col[j] < cols ? col[j] : 0u;  // out of range: flagged below, never output
            uint32_t r = 0;  // row of entry j: the last r with rb[r] <= j (empty rows share boundaries)
            bool row_start = false;
#pragma unroll
            for (int q = 0; q < VH; ++q) {
                r = rb[q] <= j ? q : r;
                row_start |= rb[q] == j;
            }
            if (col[j] >= cols) bad = max(bad, 3u);
            if (!row_start && col[j - 1] >= col[j]) bad = max(bad, 4u);
            uint32_t p = j - rb[r];
#pragma unroll
            for (int q = 0; q < VH; ++q) {
                if (q == static_cast<int>(r)) continue;
                // rows above: entries with column <= c precede; rows below: < c
                uint32_t lo = rb[q], hi = rb[q + 1];
                const uint32_t base = lo;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    const uint32_t x = col[mid];
                    if (q < static_cast<int>(r) ? x <= c : x < c) lo = mid + 1;
                    else hi = mid;
                }
                p += lo - base;
            }
            pos[k] = min(p, n - 1);  // invalid input (flagged above) must not write out of range
            mrg[pos[k]] = c;
        }
        __syncwarp();
        // first-occurrence flags of the merged columns -> inclusive prefix U
        // (stored over `col`, no longer needed); U - 1 is the rank
        uint32_t nv = 0;
        for (uint32_t p0 = 0; p0 < n; p0 += 32) {
            const uint32_t p = p0 + lane;
            const bool valid = p < n;
            const uint32_t x = valid ? mrg[p] : 0u;
            const bool first = valid && (p == 0 || mrg[p - 1] != x);
            const uint32_t m = __ballot_sync(0xffffffffu, first);
            const uint32_t u = nv + __popc(m & (0xffffffffu >> (31 - lane)));
            if (valid) col[p] = u;
            if (first) tmp_cols[e0 + u - 1] = x;
            nv += __popc(m);
        }
        __syncwarp();
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) {
            const uint32_t j = lane + 32 * k;
            if (j < n) rank[e0 + j] = col[pos[k]] - 1;
        }
        if (lane == 0) nv_out[w] = nv;
        __syncwarp();  // shared buffers are reused by the next window
    }
    if (bad) atomicMax(&chk->bad, bad);
}

template <int VH, bool GBM = false>
__device__ __forceinline__ void bitmap_rank_window(const uint32_t* __restrict__ csr_rp,
                                                   const uint32_t* __restrict__ ci, uint64_t rows, uint64_t cols,
                                                   uint64_t w, uint4* bm4, uint4* pre4, uint32_t quads,
                                                   uint32_t* __restrict__ tmp_cols, uint32_t* __restrict__ rank,
                                                   uint32_t* __restrict__ nv_out, CheckOut* chk);

// Column spaces too wide for a shared-memory bitmap (R-MAT scale 23: 8.4 M
// columns).  Windows of up to kSortCap entries merge their VH sorted rows
// in shared memory; longer (hub) windows are ranked with a CTA-private
// bitmap in global memory (bscratch: 2 x quads uint4 per CTA), or -- when
// that would be larger than 2 x nnz keys -- merged in global scratch.
// Launched twice (kSortSplit): windows of up to kSortCapA entries with
// CAP = kSortCapA (half the shared memory, two CTAs per SM), then the rest
// with CAP = kSortCap; each launch skips the other's windows (n_min < n <=
// n_max) and has its own queue.
template <int VH, uint32_t CAP>
__global__ void __launch_bounds__(kBigThreads) window_sort_big(const uint32_t* __restrict__ csr_rp,
                                                               const uint32_t* __restrict__ ci, uint64_t rows,
                                                               uint64_t cols, uint64_t W,
                                                               uint64_t* __restrict__ scratch,
                                                               uint4* __restrict__ bscratch,
                                                               uint32_t* __restrict__ tmp_cols,
                                                               uint32_t* __restrict__ rank,
                                                               uint32_t* __restrict__ nv_out, CheckOut* chk,
                                                               const uint32_t* __restrict__ big, uint32_t n_min,
                                                               uint32_t n_max, uint32_t* queue) {
    extern __shared__ uint64_t smem_keys[];
    const uint32_t n_huge = chk->n_huge, n_big = chk->n_huge + chk->n_medium;
    const uint32_t quads = static_cast<uint32_t>((cols + 127) / 128);
    for (uint32_t i = cta_next(queue); i < n_big; i = cta_next(queue)) {
        const uint64_t w = big_window(big, W, n_huge, i);
        const uint32_t e0 = csr_rp[VH * w];
        const uint32_t n = csr_rp[min(VH * w + VH, rows)] - e0;
        if (n <= n_min || n > n_max) continue;  // the other launch's window (block-uniform)
        // separate inlined call sites, so that the shared-memory one compiles
        // to LDS/STS instead of generic loads and stores
        if (n <= CAP) {
            window_sort_rank<VH>(csr_rp, ci, rows, cols, w, smem_keys, smem_keys + CAP, tmp_cols, rank, nv_out,
                                 chk);
        } else if (bscratch) {
            uint4* bm4 = bscratch + 2ull * quads * blockIdx.x;
            bitmap_rank_window<VH, TCS_ENC_GBM_WARPSCAN>(csr_rp, ci, rows, cols, w, bm4, bm4 + quads, quads, tmp_cols,
                                                         rank, nv_out, chk);
        } else {
            uint64_t* a = scratch + 2ull * e0;  // window-private slice of a 2*nnz scratch
            window_sort_rank<VH>(csr_rp, ci, rows, cols, w, a, a + n, tmp_cols, rank, nv_out, chk);
        }
    }
}

// Bitmap ranking of one window by the whole CTA: set one bit per column in
// bm4 (quads x uint4, zeroed here), prefix-popcount into pre4, emit the
// window's sorted distinct columns to tmp_cols and each entry's rank.  bm4 /
// pre4 are shared memory (window_bitmap) or a CTA-private global slice
// (window_sort_big's hub windows when the column space exceeds shared
// memory: clearing and scanning cols/32 words in L2 beats three global
// merge passes over 10^4..10^5 entries).  The word arrays are walked as
// uint4 quads (words padded to a multiple of 4).
template <int VH, bool GBM>
__device__ __forceinline__ void bitmap_rank_window(const uint32_t* __restrict__ csr_rp,
                                                   const uint32_t* __restrict__ ci, uint64_t rows, uint64_t cols,
                                                   uint64_t w, uint4* bm4, uint4* pre4, uint32_t quads,
                                                   uint32_t* __restrict__ tmp_cols, uint32_t* __restrict__ rank,
                                                   uint32_t* __restrict__ nv_out, CheckOut* chk) {
    __shared__ uint32_t rb[VH + 1];
    const uint32_t* bm = reinterpret_cast<const uint32_t*>(bm4);
    const uint32_t* pre = reinterpret_cast<const uint32_t*>(pre4);
    const uint32_t nt = blockDim.x, qpt = (quads + nt - 1) / nt;
    const uint64_t r0 = VH * w;
    const uint32_t e0 = csr_rp[r0];
    const uint32_t n = csr_rp[min(r0 + VH, rows)] - e0;
    if (threadIdx.x <= VH) rb[threadIdx.x] = csr_rp[min(r0 + threadIdx.x, rows)] - e0;
    for (uint32_t i = threadIdx.x; i < quads; i += nt) bm4[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    // kBitmapU entries per thread in flight: a hub window (10^4..10^5
    // entries) is otherwise a chain of dependent-latency iterations.  The
    // first batch's columns stay in registers for the rank pass (a window of
    // up to kBitmapU * nt entries reads its columns once).
    const uint32_t lane = threadIdx.x & 31;
    uint32_t bad = 0;
    uint32_t keep[kBitmapU];
    // warp-uniform trip count (i0 - lane): the predecessor shuffle needs
    // every lane of the warp
    for (uint32_t i0 = threadIdx.x; i0 - lane < n; i0 += kBitmapU * nt) {
        uint32_t c[kBitmapU], cp0[kBitmapU];
#pragma unroll
        for (int u = 0; u < kBitmapU; ++u) {
            const uint32_t i = i0 + u * nt;
            c[u] = i < n ? __ldg(ci + e0 + i) : 0xFFFFFFFFu;
            // predecessor: lane - 1's column (consecutive lanes hold
            // consecutive entries), loaded only by lane 0
            cp0[u] = lane == 0 && i < n && i > 0 ? __ldg(ci + e0 + i - 1) : 0u;
        }
        if (kBitmapKeep && i0 == threadIdx.x) {
#pragma unroll
            for (int u = 0; u < kBitmapU; ++u) keep[u] = c[u];
        }
#pragma unroll
        for (int u = 0; u < kBitmapU; ++u) {
            const uint32_t i = i0 + u * nt;
            uint32_t cp = __shfl_up_sync(0xffffffffu, c[u], 1);
            if (lane == 0) cp = cp0[u];
            if (i >= n) continue;
            // check_col: a non-ascending pair is legal only across a row
            // boundary (rare, so the boundary test is off the common path)
            uint32_t b = c[u] >= cols ? 3u : 0u;
            if (i > 0 && cp >= c[u]) {
                bool row_start = false;
#pragma unroll
                for (int r = 1; r < VH; ++r) row_start |= (i == rb[r]);
                if (!row_start) b = 4u;
            }
            bad = max(bad, b);
            if (c[u] < cols) atomicOr(reinterpret_cast<uint32_t*>(bm4) + (c[u] >> 5), 1u << (c[u] & 31));
        }
    }
    if (bad) atomicMax(&chk->bad, bad);
    __syncthreads();
    uint32_t total;
    if constexpr (GBM) {
        // Global-memory bitmap (hub windows of wide column spaces, 10^5+
        // quads): a thread-contiguous run of quads would be one dependent
        // L2/DRAM latency per quad and uncoalesced (ncu, C5: 50% of
        // window_sort_big's stall samples).  Each warp scans a contiguous
        // range 32 quads at a time (coalesced, loads unrolled), with a warp
        // scan per iteration and a block scan of the warp totals.
        __shared__ uint32_t gbm_wsum[32];
        const uint32_t warp = threadIdx.x >> 5, nwarps = nt >> 5;
        const uint32_t per = ((quads + nwarps - 1) / nwarps + 31u) & ~31u;
        const uint32_t qa = min(quads, warp * per), qb = min(quads, qa + per);
        uint32_t wc = 0;
#pragma unroll 4
        for (uint32_t i = qa + lane; i < qb; i += 32) {
            const uint4 x = bm4[i];
            wc += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) wc += __shfl_xor_sync(0xffffffffu, wc, o);
        if (lane == 0) gbm_wsum[warp] = wc;
        __syncthreads();
        uint32_t carry = 0;
        total = 0;
        for (uint32_t j = 0; j < nwarps; ++j) {
            const uint32_t x = gbm_wsum[j];
            carry += j < warp ? x : 0u;
            total += x;
        }
        for (uint32_t i0 = qa; i0 < qb; i0 += 32) {
            const uint32_t i = i0 + lane;
            const uint4 x = i < qb ? bm4[i] : make_uint4(0, 0, 0, 0);
            const uint32_t c = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
            uint32_t inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= static_cast<uint32_t>(o)) inc += y;
            }
            const uint32_t p0 = carry + inc - c, p1 = p0 + __popc(x.x), p2 = p1 + __popc(x.y), p3 = p2 + __popc(x.z);
            if (i < qb) pre4[i] = make_uint4(p0, p1, p2, p3);
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    } else {
        // prefix popcount over this thread's contiguous run of quads
        const uint32_t q0 = min(quads, threadIdx.x * qpt), q1 = min(quads, q0 + qpt);
        uint32_t cnt = 0;
        for (uint32_t i = q0; i < q1; ++i) {
            const uint4 x = bm4[i];
            cnt += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
        }
        const uint32_t run = dev::block_exclusive_scan(cnt, &total);
        uint32_t p = run;
        for (uint32_t i = q0; i < q1; ++i) {
            const uint4 x = bm4[i];
            const uint32_t p0 = p, p1 = p0 + __popc(x.x), p2 = p1 + __popc(x.y), p3 = p2 + __popc(x.z);
            pre4[i] = make_uint4(p0, p1, p2, p3);
            p = p3 + __popc(x.w);
        }
    }
    if (threadIdx.x == 0) nv_out[w] = total;
    __syncthreads();
    // ranks, and the window's sorted distinct columns: every entry writes
    // its column to slot rank (entries sharing a column write the same
    // value), so every slot < total is written and no bit scan is needed
    for (uint32_t i0 = threadIdx.x; i0 < n; i0 += kBitmapU * nt) {
        uint32_t c[kBitmapU];
#pragma unroll
        for (int u = 0; u < kBitmapU; ++u) {
            const uint32_t i = i0 + u * nt;
            c[u] = kBitmapKeep && i0 == threadIdx.x ? keep[u] : i < n ? __ldg(ci + e0 + i) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < kBitmapU; ++u) {
            const uint32_t i = i0 + u * nt;
            if (i < n && c[u] < cols) {
                const uint32_t r = pre[c[u] >> 5] + __popc(bm[c[u] >> 5] & ((1u << (c[u] & 31)) - 1u));
                rank[e0 + i] = r;
                if (!kColsFromEntries) tmp_cols[e0 + r] = c[u];
            }
        }
    }
    __syncthreads();  // bitmap, prefix and rb are reused by the next window
}

// Bitmap ranking for windows with more than kSmallCap entries (column
// space within shared memory).
template <int VH>
__global__ void __launch_bounds__(kBitmapThreads, kBitmapMinBlocks) window_bitmap(const uint32_t* __restrict__ csr_rp,
                                                                const uint32_t* __restrict__ ci, uint64_t rows,
                                                                uint64_t cols, uint64_t W,
                                                                uint32_t* __restrict__ tmp_cols,
                                                                uint32_t* __restrict__ rank,
                                                                uint32_t* __restrict__ nv_out, CheckOut* chk,
                                                                const uint32_t* __restrict__ big) {
    extern __shared__ uint4 bm_smem4[];
    const uint32_t n_huge = chk->n_huge, n_big = chk->n_huge + chk->n_medium;
    const uint32_t quads = static_cast<uint32_t>((cols + 127) / 128);
    for (uint32_t bi = cta_next(&chk->next_bitmap); bi < n_big; bi = cta_next(&chk->next_bitmap))
        bitmap_rank_window<VH>(csr_rp, ci, rows, cols, big_window(big, W, n_huge, bi), bm_smem4, bm_smem4 + quads,
                               quads, tmp_cols, rank, nv_out, chk);
}

template <typename V>
__device__ __forceinline__ V store_cvt(float x);
template <>
__device__ __forceinline__ float store_cvt<float>(float x) { return x; }
template <>
__device__ __forceinline__ __half store_cvt<__half>(float x) { return __float2half_rn(x); }

// The value blocks of a window are contiguous ([8*rp[w], 8*rp[w+1])); they
// are assembled in shared memory a tile of kScatterTile vectors at a time
// (zero fill + scatter of the tile's entries) and written out with 16-byte
// coalesced stores -- every value byte hits global memory exactly once.
// Two launch shapes over the K0 size-class lists: small windows (at most
// kSmallCap entries, so at most kSmallCap vectors) get 128-thread CTAs with a
// kSmallCap-vector tile, many per SM -- a 512-thread CTA's barriers dominate
// on windows of a few hundred vectors (R-MAT: 10^6 windows of ~240); big
// windows get 512 threads and 4096-vector tiles.
#ifndef TCS_ENC_SCATTER_TILE
#define TCS_ENC_SCATTER_TILE 4096
#endif
#ifndef TCS_ENC_SCATTER_THREADS
#define TCS_ENC_SCATTER_THREADS 512
#endif
constexpr uint32_t kScatterTileBig = TCS_ENC_SCATTER_TILE;  // vectors per smem tile (multiple of k)
constexpr int kScatterThreadsBig = TCS_ENC_SCATTER_THREADS;
#ifndef TCS_ENC_SCATTER_MINB
#define TCS_ENC_SCATTER_MINB 3
#endif
constexpr int kScatterMinBlocksBig = TCS_ENC_SCATTER_MINB;  // 3 x 64 KB half tiles per SM
constexpr uint32_t kScatterTileSmall = kSmallCap;
constexpr int kScatterThreadsSmall = 128;
constexpr uint32_t kRangedTiles = 4;  // windows beyond this many tiles use per-row ranges
constexpr uint32_t kTileBatch = 63;   // tile boundaries searched at once (64 x VH threads)
constexpr int kScatterU = 8;          // entries in flight per thread (window_scatter)
#ifndef TCS_ENC_SCATTER_TINY_WARP
#define TCS_ENC_SCATTER_TINY_WARP 1
#endif
constexpr bool kScatterTinyByWarp = TCS_ENC_SCATTER_TINY_WARP;

// Tiles of each huge window (vectors / tile), exclusive prefix over the
// huge list (one CTA; the huge list is short) -> tile_off[0..n_huge], total
// in chk->huge_tiles.  The big scatter then hands out (window, tile) units,
// so a hub window's tiles are written by many CTAs at once instead of one
// CTA walking them in turn (its latency bounded the whole encode and, in the
// chunk pipeline of tcs_spmm_csr_host, every chunk).
__global__ void __launch_bounds__(1024) huge_tile_prefix(const uint32_t* __restrict__ rp,
                                                         const uint32_t* __restrict__ big, CheckOut* chk,
                                                         uint32_t tile, uint32_t* __restrict__ tile_off) {
    const uint32_t n = chk->n_huge;
    uint32_t carry = 0;
    for (uint32_t i0 = 0; i0 < n; i0 += blockDim.x) {
        const uint32_t i = i0 + threadIdx.x;
        uint32_t t = 0;
        if (i < n) {
            const uint32_t w = big[i];
            t = (rp[w + 1] - rp[w] + tile - 1) / tile;
        }
        uint32_t total;
        const uint32_t ex = dev::block_exclusive_scan(t, &total);
        if (i < n) tile_off[i] = carry + ex;
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        tile_off[n] = carry;
        chk->huge_tiles = carry;
    }
}

// Tiny windows (<= kTinyCap entries, so <= kTinyCap vectors; R-MAT's 10^6
// windows are mostly these): one warp per window, its value blocks
// assembled in a per-warp shared-memory tile, no CTA barriers.  A CTA per
// window (window_scatter) spent its time in three barriers and three
// dependent global latencies per window (C5: 2.9 ms for 10^6 windows).
// warps per CTA: as many per-warp tiles as fit 32 KB of static shared memory
template <int VH, typename V>
constexpr int scatter_warps() {
    return int(32768 / (kTinyCap * VH * sizeof(V))) < 8 ? int(32768 / (kTinyCap * VH * sizeof(V))) : 8;
}
template <int VH, typename V>
__global__ void __launch_bounds__(scatter_warps<VH, V>() * 32) window_scatter_warp(
    const uint32_t* __restrict__ csr_rp, const float* __restrict__ csr_vals, uint64_t rows, uint32_t k,
    const uint32_t* __restrict__ rp, const uint32_t* __restrict__ tmp_cols, const uint32_t* __restrict__ rank,
    uint32_t* __restrict__ out_ci, V* __restrict__ out_vals, const uint32_t* __restrict__ list, CheckOut* chk) {
    constexpr uint32_t kTileBytes = kTinyCap * VH * sizeof(V);
    constexpr int kScatterWarps = scatter_warps<VH, V>();
    __shared__ __align__(16) unsigned char tiles[kScatterWarps][kTileBytes];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* tile_b = tiles[wid];
    V* tile = reinterpret_cast<V*>(tile_b);
    const uint32_t n_tiny = chk->n_tiny;
    uint32_t tiny_flag = 0;
    for (uint32_t i = blockIdx.x * kScatterWarps + wid; i < n_tiny; i += gridDim.x * kScatterWarps) {
        const uint64_t w = list[i], r0 = VH * w;
        uint32_t b = 0;  // lane q <= VH: row boundary q (absolute entry index)
        if (lane <= VH) b = __ldg(csr_rp + min(r0 + lane, rows));
        const uint32_t base = __ldg(rp + w), nvw = __ldg(rp + w + 1) - base;
        const uint32_t e0 = __shfl_sync(0xffffffffu, b, 0), e1 = __shfl_sync(0xffffffffu, b, VH);
        const uint32_t n = e1 - e0;
        // loads first (column copy, ranks, values), then the tile
        constexpr uint32_t kPer = kTinyCap / 32;
        uint32_t cc[kPer], v[kPer];
        float x[kPer];
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            const uint32_t j = lane + 32 * u;
            cc[u] = j < nvw ? __ldg(tmp_cols + e0 + j) : 0u;
            v[u] = j < n ? __ldg(rank + e0 + j) : 0u;
            x[u] = j < n ? __ldg(csr_vals + e0 + j) : 0.f;
        }
        const uint32_t n16 = (VH * nvw * static_cast<uint32_t>(sizeof(V)) + 15) / 16;
        for (uint32_t j = lane; j < n16; j += 32) reinterpret_cast<uint4*>(tile_b)[j] = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            const uint32_t j = lane + 32 * u;
            if (j < nvw) out_ci[base + j] = cc[u];
        }
        uint32_t rbq[VH];  // row boundaries, in every lane (shuffled before any divergence)
#pragma unroll
        for (int q = 0; q < VH; ++q) rbq[q] = __shfl_sync(0xffffffffu, b, q);
        __syncwarp();
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            const uint32_t j = lane + 32 * u;
            if (j >= n || v[u] >= nvw) continue;  // (an invalid entry never leaves its window's tile)
            uint32_t r = 0;  // row of entry j: boundaries rb[1..VH-1] at or below e0 + j
#pragma unroll
            for (int q = 1; q < VH; ++q) r += (e0 + j >= rbq[q]) ? 1u : 0u;
            const uint32_t blk = v[u] / k, jj = v[u] - blk * k;
            const uint32_t width = min(k, nvw - blk * k);
            const V y = store_cvt<V>(x[u]);
            tile[blk * k * VH + r * width + jj] = y;
            if constexpr (sizeof(V) == 2)  // nonzero f32 that rounds to a binary16 zero
                if ((__float_as_uint(x[u]) & 0x7FFFFFFFu) && !(__half_as_ushort(y) & 0x7FFFu)) tiny_flag = 1;
        }
        __syncwarp();
        uint4* dst = reinterpret_cast<uint4*>(out_vals + static_cast<uint64_t>(VH) * base);  // 16-B aligned
        const uint32_t full16 = (VH * nvw * static_cast<uint32_t>(sizeof(V))) / 16;
        for (uint32_t j = lane; j < full16; j += 32) dst[j] = reinterpret_cast<const uint4*>(tile_b)[j];
        __syncwarp();  // the tile is reused by the warp's next window
    }
    if (tiny_flag) atomicOr(&chk->tiny, 1u);
}

template <int VH, typename V, int THREADS, uint32_t TILE>
__global__ void __launch_bounds__(THREADS, THREADS >= 512 ? kScatterMinBlocksBig : 8) window_scatter(const uint32_t* __restrict__ csr_rp,
                                                      const uint32_t* __restrict__ csr_ci,
                                                      const float* __restrict__ csr_vals, uint64_t rows, uint64_t W,
                                                      uint32_t k, const uint32_t* __restrict__ rp,
                                                      const uint32_t* __restrict__ tmp_cols,
                                                      const uint32_t* __restrict__ rank,
                                                      uint32_t* __restrict__ out_ci, V* __restrict__ out_vals,
                                                      const uint32_t* __restrict__ list, bool big, CheckOut* chk,
                                                      const uint32_t* __restrict__ tile_off) {
    extern __shared__ uint4 tile_raw[];
    const uint32_t ks = __ffs(k) - 1;  // log2 k
    // big list: units = (huge window, tile) pairs (huge_tile_prefix), then
    // the medium windows from the back of the list, dynamic queue; small
    // list: tiny windows from the front, small from the back, fixed stride
    const uint32_t n_front = big ? chk->n_huge : chk->n_tiny;
    const uint32_t n_huge_units = big ? chk->huge_tiles : 0u;
    const uint32_t n_units = big ? n_huge_units + chk->n_medium : n_front + chk->n_small;
    // small list: the tiny windows (front) belong to window_scatter_warp
    const uint32_t u_first = big || !kScatterTinyByWarp ? 0u : n_front;
    uint32_t* next = big ? &chk->next_scatter_big : nullptr;
    uint32_t* tiny = &chk->tiny;
    __shared__ uint32_t s_huge;
    V* tile = reinterpret_cast<V*>(tile_raw);
    __shared__ uint32_t rb[VH + 1];
    __shared__ uint32_t tb[kTileBatch + 1][VH];  // ranged: first entry of each row per tile boundary
    __shared__ uint32_t rlo[VH], roff[VH + 1];    // ranged: this tile's first entry per row, prefix
    constexpr uint32_t kTile = TILE * 8 / VH;  // vectors per smem tile
    // big list: dynamic queue (next != nullptr); small list: fixed stride
    for (uint32_t u = next ? cta_next(next) : u_first + blockIdx.x; u < n_units;
         u = next ? cta_next(next) : u + gridDim.x) {
        uint64_t w;
        uint32_t tile_lo = 0, tile_hi = 0xFFFFFFFFu;  // the unit's tiles of window w
        if (u < n_huge_units) {  // block-uniform
            if (threadIdx.x == 0) {  // huge window i: tile_off[i] <= u < tile_off[i + 1]
                uint32_t lo = 0, hi = n_front;
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) / 2;
                    if (tile_off[mid] <= u) lo = mid; else hi = mid;
                }
                s_huge = lo;
            }
            __syncthreads();
            const uint32_t i = s_huge;
            w = list[i];
            tile_lo = u - tile_off[i];
            tile_hi = tile_lo + 1;
        } else {
            w = big_window(list, W, n_front, big ? n_front + (u - n_huge_units) : u);
        }
        const uint64_t r0 = VH * w;
        if (threadIdx.x <= VH) rb[threadIdx.x] = csr_rp[min(r0 + threadIdx.x, rows)];
        const uint32_t base = rp[w], nvw = rp[w + 1] - base;
        __syncthreads();
        const uint32_t e0 = rb[0], e1 = rb[VH];
        const uint32_t v_lo = min(nvw, tile_lo * kTile);
        const uint32_t v_hi = uint64_t(tile_hi) * kTile < nvw ? tile_hi * kTile : nvw;
        // the column copy, 8 loads in flight per thread (one at a time it was
        // the kernel's top stall: a DRAM latency per 512 columns)
        for (uint32_t i0 = v_lo + threadIdx.x; !kColsFromEntries && i0 < v_hi; i0 += 8 * blockDim.x) {
            uint32_t cc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                cc[u] = i < v_hi ? __ldg(tmp_cols + e0 + i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                if (i < v_hi) out_ci[base + i] = cc[u];
            }
        }
        V* vals = out_vals + static_cast<uint64_t>(VH) * base;
        // block-uniform: a window of at most kRangedTiles tiles scans all of
        // its entries per tile and keeps those of the tile (cheap for few
        // tiles); longer (hub) windows find each tile's entries per row:
        // within a row the rank ascends with the column, so a tile's entries
        // are one contiguous range per row -- and the range boundaries of up
        // to kTileBatch tiles are binary-searched in parallel, one thread per
        // (tile boundary, row), instead of tile after tile.
        const bool ranged = nvw > kRangedTiles * kTile;
        for (uint32_t t0 = v_lo; t0 < v_hi; t0 += kTile) {
            const uint32_t tj = ((t0 - v_lo) / kTile) % kTileBatch;  // tile within its batch
            if (ranged && tj == 0) {
                __syncthreads();  // the previous batch's boundaries are no longer read
                for (uint32_t x = threadIdx.x; x < (kTileBatch + 1) * VH; x += blockDim.x) {
                    const uint32_t j = x / VH, r = x % VH;
                    const uint32_t key = min(nvw, t0 + j * kTile);
                    uint32_t lo = rb[r] - e0, hi = rb[r + 1] - e0;  // first entry of row r with rank >= key
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) / 2;
                        if (__ldg(rank + e0 + mid) < key) lo = mid + 1; else hi = mid;
                    }
                    tb[j][r] = e0 + lo;
                }
            }
            const uint32_t tn = min(kTile, nvw - t0);  // vectors in this tile
            const uint32_t n16 = (VH * tn * sizeof(V) + 15) / 16;
            for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) tile_raw[i] = make_uint4(0, 0, 0, 0);
            __syncthreads();
            if (ranged) {  // this tile's per-row entry ranges and their prefix
                if (threadIdx.x == 0) {
                    uint32_t acc = 0;
#pragma unroll
                    for (int q = 0; q < VH; ++q) {
                        rlo[q] = tb[tj][q];
                        roff[q] = acc;
                        acc += tb[tj + 1][q] - tb[tj][q];
                    }
                    roff[VH] = acc;
                }
                __syncthreads();
            }
            const uint32_t total = ranged ? roff[VH] : e1 - e0;
            // kScatterU entries in flight per thread (coalesced per sub-step)
            for (uint32_t i4 = 0; i4 < total; i4 += kScatterU * blockDim.x) {
                uint32_t v[kScatterU], e[kScatterU], c[kScatterU];
                float x[kScatterU];
#pragma unroll
                for (int u = 0; u < kScatterU; ++u) {
                    const uint32_t i = i4 + u * blockDim.x + threadIdx.x;
                    e[u] = 0xFFFFFFFFu;
                    if (i < total) {
                        if (!ranged) {
                            e[u] = e0 + i;
                        } else {
                            uint32_t q = 0;
#pragma unroll
                            for (int qq = 1; qq < VH; ++qq) q += (i >= roff[qq]) ? 1u : 0u;
                            e[u] = rlo[q] + (i - roff[q]);
                        }
                    }
                    v[u] = e[u] != 0xFFFFFFFFu ? __ldg(rank + e[u]) : 0u;
                    x[u] = e[u] != 0xFFFFFFFFu ? __ldg(csr_vals + e[u]) : 0.f;
                    c[u] = kColsFromEntries && e[u] != 0xFFFFFFFFu ? __ldg(csr_ci + e[u]) : 0u;
                }
#pragma unroll
                for (int u = 0; u < kScatterU; ++u) {
                    if (e[u] == 0xFFFFFFFFu || v[u] < t0 || v[u] >= t0 + tn) continue;
                    if (kColsFromEntries) out_ci[base + v[u]] = c[u];
                    uint32_t r = 0;
#pragma unroll
                    for (int q = 1; q < VH; ++q) r += (e[u] >= rb[q]) ? 1u : 0u;
                    const uint32_t b = v[u] >> ks, j = v[u] & (k - 1);  // k is 4 or 8
                    const uint32_t width = min(k, nvw - (b << ks));
                    const V y = store_cvt<V>(x[u]);
                    tile[((b << ks) - t0) * VH + r * width + j] = y;
                    if constexpr (sizeof(V) == 2) {  // nonzero f32 that rounds to a binary16 zero
                        if ((__float_as_uint(x[u]) & 0x7FFFFFFFu) && !(__half_as_ushort(y) & 0x7FFFu)) atomicOr(tiny, 1u);
                    }
                }
            }
            __syncthreads();
            uint4* dst = reinterpret_cast<uint4*>(vals + static_cast<uint64_t>(VH) * t0);  // 16-B aligned
            const uint32_t full16 = (VH * tn * sizeof(V)) / 16;
            for (uint32_t i = threadIdx.x; i < full16; i += blockDim.x) dst[i] = tile_raw[i];
            __syncthreads();
        }
    }
}

// Exact SDDMM liveness bytes (bit r of byte p: row r of stored vector p has
// a nonzero f32 CSR value, ref sddmm.hpp:131) for an F16 handle whose
// binary16 values lost a tiny nonzero (CheckOut::tiny).  One thread per CSR
// row; rare path, so bits are set with word atomics.
__global__ void exact_live_build(const uint32_t* __restrict__ csr_rp, const float* __restrict__ csr_vals,
                                 uint64_t rows, const uint32_t* __restrict__ rp, const uint32_t* __restrict__ rank,
                                 uint8_t* live) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t base = rp[r / 8], bit = 1u << (r % 8);
        for (uint32_t e = csr_rp[r]; e < csr_rp[r + 1]; ++e) {
            if (!(__float_as_uint(csr_vals[e]) & 0x7FFFFFFFu)) continue;
            const uint64_t p = uint64_t(base) + rank[e];
            atomicOr(reinterpret_cast<uint32_t*>(live + (p & ~uint64_t(3))), bit << (8 * (p & 3)));
        }
    }
}

// Value type V of a window_scatter instantiation (for the launch helper).
template <typename V>
V kern_value_type(void (*)(const uint32_t*, const uint32_t*, const float*, uint64_t, uint64_t, uint32_t, const uint32_t*,
                           const uint32_t*, const uint32_t*, uint32_t*, V*, const uint32_t*, bool, CheckOut*,
                           const uint32_t*));

const char* kBadMsg[] = {"", "row_ptr must be nondecreasing", "row_ptr exceeds nnz", "column index out of range",
                         "column indices must be strictly ascending within a row"};

}  // namespace
}  // namespace tcs

using namespace tcs;

namespace tcs {
namespace {

// async_chk == nullptr: the API encode (exact sizes; validation errors are
// thrown before it returns; three host round trips).  Otherwise the
// pipelined encode of tcs_spmm_csr_host: no host round trip at all -- the
// size-class kernels run on capacity grids and read their counts on the
// device, the ME-BCRS arrays are allocated for nv <= nnz, the work list is
// built with device-side counts (build_plan_async), and the validation code
// (CheckOut::bad) lands in the caller-owned, pre-zeroed async_chk block
// (encode_check_bytes() of device memory) for the caller to check once at
// the end -- no per-chunk memset or flag copy.
// The handle's num_vectors is then a capacity, and SDDMM liveness extras
// are not built (the pipeline only multiplies).
template <int VH>
void encode_impl(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype, tcs_mebcrs* out,
                 tcs_stream_t stream, void* async_chk = nullptr, uint64_t seg_nv = 0,
                 cudaEvent_t values_ready = nullptr) {
    {
        if (!csr || !out) fail(TCS_ERR_ARGUMENT, "null argument");
        if (precision != TCS_FP16 && precision != TCS_TF32) fail(TCS_ERR_ARGUMENT, "unknown precision");
        if (precision == TCS_TF32 && value_dtype != TCS_DTYPE_F32)
            fail(TCS_ERR_ARGUMENT, "TF32 ME-BCRS values must be stored as f32");
        if (value_dtype != TCS_DTYPE_F16 && value_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown dtype");
        if (!csr->row_ptr || (csr->nnz && (!csr->col_idx || !csr->values))) fail(TCS_ERR_ARGUMENT, "null CSR array");
        if (csr->nnz >= (1ull << 32)) fail(TCS_ERR_FORMAT, "nnz exceeds u32 row_ptr");
        cudaStream_t s = st(stream);
        const bool async = async_chk != nullptr;
        const uint64_t rows = csr->rows, W = (rows + VH - 1) / VH, nnz = csr->nnz, cols = csr->cols;
        const uint32_t k = precision == TCS_FP16 ? 8 : 4;
        const int sms = num_sms();

        tcs_mebcrs m{};
        m.rows = rows;
        m.cols = cols;
        m.vector_height = VH;
        m.k = k;
        m.precision = precision;
        m.value_dtype = value_dtype;
        m.num_windows = W;
        m.flags = TCS_MEBCRS_OWN_STRUCTURE | TCS_MEBCRS_OWN_VALUES;
        m.row_pointers = static_cast<uint32_t*>(dalloc((W + 1) * 4, s));
        struct Cleanup {
            tcs_mebcrs* m;
            cudaStream_t s;
            bool armed = true;
            ~Cleanup() {
                if (armed) {
                    dfree(m->row_pointers, s);
                    dfree(m->column_indices, s);
                    dfree(m->values, s);
                }
            }
        } cleanup{&m, s};

        uint32_t nv = 0;
        uint8_t* exact_live = nullptr;  // see CheckOut::tiny
        struct LiveCleanup {
            uint8_t*& p;
            cudaStream_t s;
            ~LiveCleanup() { dfree(p, s); }
        } live_cleanup{exact_live, s};
        if (W) {
            // K0: row_ptr invariants + size-class window lists
            DBuf chk, small_list(W * 4, s), big_list(W * 4, s);
            CheckOut* dchk = static_cast<CheckOut*>(async_chk);
            if (!async) {
                chk = DBuf(sizeof(CheckOut), s);
                TCS_CUDA(cudaMemsetAsync(chk.p, 0, sizeof(CheckOut), s));
                dchk = chk.as<CheckOut>();
            }
            DBuf nvw(W * 4, s);
            const int g0 = static_cast<int>(std::min<uint64_t>((W + 255) / 256, uint64_t(sms) * 8));
            window_stats<VH><<<g0, 256, 0, s>>>(csr->row_ptr, rows, W, nnz, dchk, small_list.as<uint32_t>(),
                                                big_list.as<uint32_t>(), async ? nvw.as<uint32_t>() : nullptr);
            TCS_LAUNCHED("window_stats");
            CheckOut h{};
            if (!async) {
                uint32_t ends[2] = {0, 0};
                TCS_CUDA(cudaMemcpyAsync(&h, dchk, sizeof(h), cudaMemcpyDeviceToHost, s));
                TCS_CUDA(cudaMemcpyAsync(&ends[0], csr->row_ptr, 4, cudaMemcpyDeviceToHost, s));
                TCS_CUDA(cudaMemcpyAsync(&ends[1], csr->row_ptr + rows, 4, cudaMemcpyDeviceToHost, s));
                TCS_CUDA(cudaStreamSynchronize(s));
                if (ends[0] != 0 || ends[1] != nnz) fail(TCS_ERR_FORMAT, "row_ptr endpoints inconsistent with nnz");
                if (h.bad) fail(TCS_ERR_FORMAT, kBadMsg[h.bad < 5 ? h.bad : 0]);
            } else {  // unknown: every class may hold every window
                const uint32_t w32 = static_cast<uint32_t>(std::min<uint64_t>(W, 0xFFFFFFFFu));
                h.n_tiny = h.n_small = h.n_medium = w32;
                h.n_huge = 0;
                h.max_window_entries = 0xFFFFFFFFu;
            }

            DBuf tmp_cols(std::max<uint64_t>(1, nnz) * 4, s), rank(std::max<uint64_t>(1, nnz) * 4, s);
            // (pipelined encode: window_stats zeroed nvw -- windows that fail
            // validation are in no list, so they scan as 0 vectors)
            const uint64_t n_big = uint64_t(h.n_medium) + h.n_huge;
            if (h.n_tiny) {
                const int gt = static_cast<int>(
                    std::min<uint64_t>((h.n_tiny + kTinyWarps - 1) / kTinyWarps, uint64_t(sms) * 8));
                window_sort_warp<VH><<<gt, kTinyWarps * 32, 0, s>>>(csr->row_ptr, csr->col_idx, rows, cols,
                                                                    tmp_cols.as<uint32_t>(), rank.as<uint32_t>(),
                                                                    nvw.as<uint32_t>(), dchk, small_list.as<uint32_t>());
                TCS_LAUNCHED("window_sort_warp");
            }
            if (h.n_small) {
                const int g1 = static_cast<int>(std::min<uint64_t>(h.n_small, uint64_t(sms) * 16));
                window_sort_small<VH><<<g1, kSmallThreads, 0, s>>>(csr->row_ptr, csr->col_idx, rows, cols, W,
                                                               tmp_cols.as<uint32_t>(), rank.as<uint32_t>(),
                                                               nvw.as<uint32_t>(), dchk, small_list.as<uint32_t>());
                TCS_LAUNCHED("window_sort_small");
            }
            if (n_big) {
                const uint64_t words = (cols + 31) / 32;
                if (words <= kBitmapMaxWords) {
                    const size_t smem = 2 * ((words + 3) / 4) * sizeof(uint4);
                    TCS_CUDA(cudaFuncSetAttribute(window_bitmap<VH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(std::max<size_t>(smem, 1))));
                    const int per_sm = std::max<int>(
                        1, std::min<int>(2048 / kBitmapThreads, int(200 * 1024 / std::max<size_t>(smem, 1))));
                    const int g2 = static_cast<int>(std::min<uint64_t>(n_big, uint64_t(sms) * per_sm));
                    window_bitmap<VH><<<g2, kBitmapThreads, smem, s>>>(csr->row_ptr, csr->col_idx, rows, cols, W,
                                                                   tmp_cols.as<uint32_t>(), rank.as<uint32_t>(),
                                                                   nvw.as<uint32_t>(), dchk, big_list.as<uint32_t>());
                    TCS_LAUNCHED("window_bitmap");
                } else {
                    auto sort_launch = [&](auto kern, uint32_t cap, uint32_t n_min, uint32_t n_max, uint32_t* queue,
                                           bool hubs) {
                        const size_t smem = 2 * size_t(cap) * sizeof(uint64_t);
                        TCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(smem)));
                        const int per_sm =
                            std::max<int>(1, std::min<int>(2048 / kBigThreads, int(220 * 1024 / smem)));
                        const int g2 = static_cast<int>(std::min<uint64_t>(n_big, uint64_t(sms) * per_sm));
                        // hub windows: a global bitmap per CTA, unless 2 x nnz merge keys are smaller
                        DBuf scratch, bscratch;
                        const uint64_t bm_bytes = uint64_t(g2) * 2 * ((cols + 127) / 128) * 16;
                        if (hubs && h.max_window_entries > cap) {
                            if (TCS_ENC_HUB_BITMAP && bm_bytes <= 2 * nnz * 8) bscratch = DBuf(bm_bytes, s);
                            else scratch = DBuf(2 * nnz * 8, s);
                        }
                        kern<<<g2, kBigThreads, smem, s>>>(csr->row_ptr, csr->col_idx, rows, cols, W,
                                                           scratch.as<uint64_t>(), bscratch.as<uint4>(),
                                                           tmp_cols.as<uint32_t>(), rank.as<uint32_t>(),
                                                           nvw.as<uint32_t>(), dchk, big_list.as<uint32_t>(), n_min,
                                                           n_max, queue);
                    };
                    if (kSortCapA) {
                        sort_launch(window_sort_big<VH, kSortCapA>, kSortCapA, 0, kSortCapA, &dchk->next_sort_big,
                                    false);
                        sort_launch(window_sort_big<VH, kSortCap>, kSortCap, kSortCapA, 0xFFFFFFFFu,
                                    &dchk->next_sort_big2, true);
                    } else {
                        sort_launch(window_sort_big<VH, kSortCap>, kSortCap, 0, 0xFFFFFFFFu, &dchk->next_sort_big,
                                    true);
                    }
                    TCS_LAUNCHED("window_sort_big");
                }
            }
            exclusive_scan_u32(nvw.as<uint32_t>(), m.row_pointers, W, s);
            if (!async) {
                TCS_CUDA(cudaMemcpyAsync(&nv, m.row_pointers + W, 4, cudaMemcpyDeviceToHost, s));
                TCS_CUDA(cudaMemcpyAsync(&h, dchk, sizeof(h), cudaMemcpyDeviceToHost, s));
                TCS_CUDA(cudaStreamSynchronize(s));
                if (h.bad) fail(TCS_ERR_FORMAT, kBadMsg[h.bad < 5 ? h.bad : 0]);
            } else {
                nv = static_cast<uint32_t>(nnz);  // capacity: nv <= nnz
            }
            m.num_vectors = nv;
            const size_t vw = value_dtype == TCS_DTYPE_F16 ? 2 : 4;
            m.column_indices = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, nv) * 4, s));
            m.values = dalloc(std::max<uint64_t>(1, uint64_t(VH) * nv) * vw, s);
            DBuf tile_off(W * 4 + 4, s);
            auto scatter = [&](auto kern, int threads, uint32_t tile, const uint32_t* list, bool big, uint64_t n) {
                if (!n) return;
                const size_t tile_smem = size_t(tile) * 8 * vw;
                const int per_sm = static_cast<int>(
                    std::max<size_t>(1, std::min<size_t>((200 * 1024) / tile_smem, 2048 / threads)));
                const int g3 = static_cast<int>(std::min<uint64_t>(n, uint64_t(sms) * per_sm));
                TCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(tile_smem)));
                kern<<<g3, threads, tile_smem, s>>>(csr->row_ptr, csr->col_idx, csr->values, rows, W, k, m.row_pointers,
                                                    tmp_cols.as<uint32_t>(), rank.as<uint32_t>(), m.column_indices,
                                                    static_cast<decltype(kern_value_type(kern))*>(m.values), list,
                                                    big, dchk, tile_off.as<uint32_t>());
            };
            // (window, tile) units of the huge windows for the big scatter
            if (n_big) {
                huge_tile_prefix<<<1, 1024, 0, s>>>(m.row_pointers, big_list.as<uint32_t>(), dchk,
                                                     kScatterTileBig * 8 / VH, tile_off.as<uint32_t>());
                TCS_LAUNCHED("huge_tile_prefix");
            }
            // the CSR values are read from here on (the pipeline uploads them
            // after the column indices the kernels above rank)
            if (values_ready) TCS_CUDA(cudaStreamWaitEvent(s, values_ready, 0));
            const uint64_t n_smalls = async ? W : uint64_t(h.n_tiny) + h.n_small;
            if (kScatterTinyByWarp && h.n_tiny) {  // tiny windows: one warp each
                auto gw = [&](int warps) {
                    return static_cast<int>(
                        std::min<uint64_t>((h.n_tiny + warps - 1) / warps, uint64_t(sms) * (64 / warps)));
                };
                constexpr int w16 = scatter_warps<VH, __half>(), w32 = scatter_warps<VH, float>();
                if (value_dtype == TCS_DTYPE_F16)
                    window_scatter_warp<VH, __half><<<gw(w16), w16 * 32, 0, s>>>(
                        csr->row_ptr, csr->values, rows, k, m.row_pointers, tmp_cols.as<uint32_t>(),
                        rank.as<uint32_t>(), m.column_indices, static_cast<__half*>(m.values),
                        small_list.as<uint32_t>(), dchk);
                else
                    window_scatter_warp<VH, float><<<gw(w32), w32 * 32, 0, s>>>(
                        csr->row_ptr, csr->values, rows, k, m.row_pointers, tmp_cols.as<uint32_t>(),
                        rank.as<uint32_t>(), m.column_indices, static_cast<float*>(m.values),
                        small_list.as<uint32_t>(), dchk);
                TCS_LAUNCHED("window_scatter_warp");
            }
            // big scatter units: with any huge window, as many CTAs as fit
            const uint64_t n_big_units = h.n_huge || async ? uint64_t(sms) * 64 : n_big;
            if (value_dtype == TCS_DTYPE_F16) {
                scatter(window_scatter<VH, __half, kScatterThreadsBig, kScatterTileBig>, kScatterThreadsBig,
                        kScatterTileBig, big_list.as<uint32_t>(), true, n_big ? n_big_units : 0);
                scatter(window_scatter<VH, __half, kScatterThreadsSmall, kScatterTileSmall>, kScatterThreadsSmall,
                        kScatterTileSmall, small_list.as<uint32_t>(), false, n_smalls);
            } else {
                scatter(window_scatter<VH, float, kScatterThreadsBig, kScatterTileBig>, kScatterThreadsBig,
                        kScatterTileBig, big_list.as<uint32_t>(), true, n_big ? n_big_units : 0);
                scatter(window_scatter<VH, float, kScatterThreadsSmall, kScatterTileSmall>, kScatterThreadsSmall,
                        kScatterTileSmall, small_list.as<uint32_t>(), false, n_smalls);
            }
            TCS_LAUNCHED("window_scatter");
            if (!async && value_dtype == TCS_DTYPE_F16 && VH == 8) {
                uint32_t tiny = 0;
                TCS_CUDA(cudaMemcpyAsync(&tiny, &dchk->tiny, 4, cudaMemcpyDeviceToHost, s));
                TCS_CUDA(cudaStreamSynchronize(s));
                if (tiny) {
                    exact_live = static_cast<uint8_t*>(dalloc(uint64_t(nv) + 16, s));
                    TCS_CUDA(cudaMemsetAsync(exact_live, 0, uint64_t(nv) + 16, s));
                    const int gl = static_cast<int>(std::min<uint64_t>((rows + 255) / 256, uint64_t(sms) * 8));
                    exact_live_build<<<gl, 256, 0, s>>>(csr->row_ptr, csr->values, rows, m.row_pointers,
                                                        rank.as<uint32_t>(), exact_live);
                    TCS_LAUNCHED("exact_live_build");
                }
            }
        } else {
            TCS_CUDA(cudaMemsetAsync(m.row_pointers, 0, 4, s));
            m.column_indices = static_cast<uint32_t*>(dalloc(4, s));
            m.values = dalloc(4, s);

        }
        cleanup.armed = false;
        *out = m;
        if (async) {
            out->plan = build_plan_async(out, nnz, seg_nv, s);
            return;
        }
        const tcs_status rc = tcs_mebcrs_prepare(out, stream);
        if (rc != TCS_OK) {
            const std::string msg = tcs_last_error();
            tcs_mebcrs_free(out, stream);
            fail(rc, msg);
        }
        if (exact_live) {  // the work list owns them from here
            Plan* plan = static_cast<Plan*>(out->plan);
            plan->exact_live = exact_live;
            plan->exact_live_src = out->values;
            exact_live = nullptr;
        }
    }
}

}  // namespace

const char* encode_bad_msg(uint32_t code) { return kBadMsg[code < 5 ? code : 0]; }
size_t encode_check_bytes() { return (sizeof(CheckOut) + 15) / 16 * 16; }
size_t encode_check_bad_offset() { return offsetof(CheckOut, bad); }

// The pipelined encode (see encode_impl): tcs_spmm_csr_host's chunks.
void encode_mebcrs_async(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype, tcs_mebcrs* out,
                         cudaStream_t s, void* check_dev, uint64_t seg_nv, cudaEvent_t values_ready) {
    encode_impl<8>(csr, precision, value_dtype, out, reinterpret_cast<tcs_stream_t>(s), check_dev, seg_nv,
                   values_ready);
}

}  // namespace tcs

extern "C" tcs_status tcs_mebcrs_encode(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype,
                                        tcs_mebcrs* out, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_mebcrs_encode"); encode_impl<8>(csr, precision, value_dtype, out, stream); });
}

extern "C" tcs_status tcs_mebcrs_encode_v(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype,
                                          uint32_t vector_height, tcs_mebcrs* out, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_mebcrs_encode_v");
        // ref partition.hpp:42-43
        if (vector_height == 8) encode_impl<8>(csr, precision, value_dtype, out, stream);
        else if (vector_height == 16) encode_impl<16>(csr, precision, value_dtype, out, stream);
        else fail(TCS_ERR_ARGUMENT, "vector height must be 8 or 16");
    });
}

extern "C" tcs_status tcs_mebcrs_encode_host(const tcs_csr* host_csr, tcs_precision precision,
                                             tcs_dtype value_dtype, tcs_mebcrs* out, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_mebcrs_encode_host");
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
