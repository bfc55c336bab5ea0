// Runtime plumbing behind the C-ABI: error state, stream-ordered memory,
// device-wide scan, the SpMM/SDDMM work-list planner, dtype/padding
// conversion, and the ME-BCRS handle lifecycle (upload/download/free).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "tcs_internal.cuh"

namespace tcs {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_last_error;
void set_last_error(const std::string& msg) { t_last_error = msg; }

// ----------------------------------------------------------------- memory
// cudaMallocAsync on the device's default pool with an unbounded release
// threshold: after warm-up, per-call workspaces are recycled without any
// driver allocation or implicit synchronisation.
static std::once_flag g_pool_once[64];

void* dalloc(size_t bytes, cudaStream_t s) {
    int dev = 0;
    TCS_CUDA(cudaGetDevice(&dev));
    std::call_once(g_pool_once[dev & 63], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? TCS_ERR_OOM : TCS_ERR_CUDA,
             std::string("cudaMallocAsync(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
    return p;
}

void dfree(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    TCS_CUDA(cudaGetDevice(&dev));
    if (!cached[dev & 63]) {
        int n = 0;
        TCS_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
        cached[dev & 63] = n;
    }
    return cached[dev & 63];
}

// ------------------------------------------------------------------- scan
namespace {
constexpr int kScanThreads = 256;
constexpr int kScanIpt = 8;
constexpr int kScanTile = kScanThreads * kScanIpt;

__global__ void __launch_bounds__(kScanThreads) scan_tiles(const uint32_t* __restrict__ in,
                                                           uint32_t* __restrict__ out,
                                                           uint32_t* __restrict__ tile_sums, uint64_t n) {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanIpt;
    uint32_t v[kScanIpt];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kScanIpt; ++i) {
        v[i] = base + i < n ? in[base + i] : 0u;
        sum += v[i];
    }
    uint32_t total;
    uint32_t run = dev::block_exclusive_scan(sum, &total);
#pragma unroll
    for (int i = 0; i < kScanIpt; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// Single block: exclusive scan of the tile sums in place; writes the grand
// total to *grand.
__global__ void __launch_bounds__(1024) scan_tile_sums(uint32_t* sums, uint64_t ntiles, uint32_t* grand) {
    uint32_t carry = 0;
    for (uint64_t b = 0; b < ntiles; b += blockDim.x) {
        const uint64_t i = b + threadIdx.x;
        const uint32_t v = i < ntiles ? sums[i] : 0u;
        uint32_t total;
        const uint32_t ex = dev::block_exclusive_scan(v, &total);
        if (i < ntiles) sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) *grand = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_add(uint32_t* __restrict__ out,
                                                         const uint32_t* __restrict__ tile_sums,
                                                         uint64_t n) {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
    const uint32_t add = tile_sums[blockIdx.x];
    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads)
        if (base + i < n) out[base + i] += add;
}
}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
    const uint64_t ntiles = std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile);
    DBuf sums(ntiles * sizeof(uint32_t), s);
    scan_tiles<<<ntiles, kScanThreads, 0, s>>>(in, out, sums.as<uint32_t>(), n);
    TCS_LAUNCHED("scan_tiles");
    scan_tile_sums<<<1, 1024, 0, s>>>(sums.as<uint32_t>(), ntiles, out + n);
    TCS_LAUNCHED("scan_tile_sums");
    if (ntiles > 1) {
        scan_add<<<ntiles, kScanThreads, 0, s>>>(out, sums.as<uint32_t>(), n);
        TCS_LAUNCHED("scan_add");
    }
}

// ------------------------------------------------------------------- plan
namespace {
struct PlanTotals {
    unsigned long long blocks_k;
    unsigned long long groups16;
    uint32_t max_nv;
    uint32_t pad;
};

__global__ void plan_count(const uint32_t* __restrict__ rp, uint64_t W, uint32_t seg, uint32_t k,
                           uint32_t* __restrict__ nslot, uint32_t* __restrict__ nsplit,
                           PlanTotals* __restrict__ tot) {
    unsigned long long blocks = 0, groups = 0;
    uint32_t mx = 0;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t nv = rp[w + 1] - rp[w];
        const uint32_t nseg = nv > seg ? (nv + seg - 1) / seg : 1u;
        nslot[w] = nseg > 1 ? nseg : 0u;
        nsplit[w] = nseg > 1 ? 1u : 0u;
        blocks += (nv + k - 1) / k;
        groups += (nv + 15) / 16;
        mx = max(mx, nv);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        blocks += __shfl_xor_sync(0xffffffffu, blocks, o);
        groups += __shfl_xor_sync(0xffffffffu, groups, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&tot->blocks_k, blocks);
        atomicAdd(&tot->groups16, groups);
        atomicMax(&tot->max_nv, mx);
    }
}

// Split windows' segments first (they are the longest items and should be
// dispatched first), then one item per remaining window (empty windows too:
// their item writes the zero rows).
// dcounts == nullptr: items from index 0 (the host read the counts).
// Otherwise the pipelined plan: items end at `cap`, and dcounts receives the
// claim start (cap - items) and the split-window count.
__global__ void plan_fill(const uint32_t* __restrict__ rp, uint64_t W, uint32_t seg,
                          const uint32_t* __restrict__ slot_off, const uint32_t* __restrict__ split_off,
                          WorkItem* __restrict__ items, SplitWindow* __restrict__ split, uint64_t cap,
                          uint32_t* __restrict__ dcounts) {
    const uint32_t n_slots = slot_off[W], n_split = split_off[W];
    const uint64_t off = dcounts ? cap - (n_slots + (W - n_split)) : 0;
    if (dcounts && blockIdx.x == 0 && threadIdx.x == 0) {
        dcounts[0] = static_cast<uint32_t>(off);
        dcounts[1] = n_split;
    }
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t nv = rp[w + 1] - rp[w];
        const uint32_t so = slot_off[w], sp = split_off[w];
        if (nv > seg) {
            const uint32_t nseg = (nv + seg - 1) / seg;
            for (uint32_t i = 0; i < nseg; ++i)
                items[off + so + i] = WorkItem{(uint32_t)w, i * seg, min(nv, (i + 1) * seg), so + i};
            split[sp] = SplitWindow{(uint32_t)w, so, nseg, 0};
        } else {
            items[off + n_slots + (w - sp)] = WorkItem{(uint32_t)w, 0, nv, kNoSlot};
        }
    }
}

// The whole pipelined work list of a small chunk (W <= kPlanSmallW) in one
// CTA: window counts, the two exclusive scans and the fill, one launch
// instead of eight (the tail chunks of tcs_spmm_csr_host are a chain of
// short dependent launches).  Same items, order and counts as plan_count +
// scans + plan_fill.
constexpr uint64_t kPlanSmallW = 32768;
__global__ void __launch_bounds__(1024) plan_async_small(const uint32_t* __restrict__ rp, uint64_t W, uint32_t seg,
                                                         uint32_t k, WorkItem* __restrict__ items,
                                                         SplitWindow* __restrict__ split, uint64_t cap,
                                                         uint32_t* __restrict__ dcounts) {
    __shared__ unsigned long long s_blocks;
    if (threadIdx.x == 0) s_blocks = 0;
    __syncthreads();
    uint32_t slots = 0, splits = 0;
    unsigned long long blocks = 0;
    for (uint64_t w = threadIdx.x; w < W; w += blockDim.x) {
        const uint32_t nv = rp[w + 1] - rp[w];
        if (nv > seg) {
            slots += (nv + seg - 1) / seg;
            splits += 1;
        }
        blocks += (nv + k - 1) / k;
    }
    atomicAdd(&s_blocks, blocks);
    uint32_t n_slots, n_split;
    dev::block_exclusive_scan(slots, &n_slots);
    __syncthreads();
    dev::block_exclusive_scan(splits, &n_split);
    __syncthreads();
    const uint64_t off = cap - (uint64_t(n_slots) + (W - n_split));
    if (threadIdx.x == 0) {
        dcounts[0] = static_cast<uint32_t>(off);
        dcounts[1] = n_split;
        *reinterpret_cast<unsigned long long*>(dcounts + 2) = s_blocks;
    }
    uint32_t carry_slot = 0, carry_split = 0;
    for (uint64_t base = 0; base < W; base += blockDim.x) {
        const uint64_t w = base + threadIdx.x;
        const uint32_t nv = w < W ? rp[w + 1] - rp[w] : 0u;
        const uint32_t nseg = nv > seg ? (nv + seg - 1) / seg : 0u;  // 0: not split
        uint32_t t_slot, t_split;
        const uint32_t so = carry_slot + dev::block_exclusive_scan(nseg, &t_slot);
        __syncthreads();
        const uint32_t sp = carry_split + dev::block_exclusive_scan(nseg ? 1u : 0u, &t_split);
        __syncthreads();
        if (w < W) {
            if (nseg) {
                for (uint32_t i = 0; i < nseg; ++i)
                    items[off + so + i] = WorkItem{(uint32_t)w, i * seg, min(nv, (i + 1) * seg), so + i};
                split[sp] = SplitWindow{(uint32_t)w, so, nseg, 0};
            } else {
                items[off + n_slots + (w - sp)] = WorkItem{(uint32_t)w, 0, nv, kNoSlot};
            }
        }
        carry_slot += t_slot;
        carry_split += t_split;
    }
}

__global__ void plan_blocks_out(const PlanTotals* __restrict__ tot, uint32_t* __restrict__ dcounts) {
    *reinterpret_cast<unsigned long long*>(dcounts + 2) = tot->blocks_k;
}
}  // namespace

// Shortest work item (vectors; a multiple of 16).  Small matrices split
// their windows down to this so that enough warps share the work.  32 or 64
// make C1 (4096^2, 65 k nnz) slower, 11.8 -> 22.6 / 17.7 us per graph-
// replayed SpMM: the split partials and their reduction cost more than the
// extra warps gain.
#ifndef TCS_PLAN_MIN_SEG
#define TCS_PLAN_MIN_SEG 256
#endif

// Segment length: enough items for ~64 per SM, bounded to [256, 16384]
// vectors and a multiple of 16 (SpMM/SDDMM step granularity).
static uint32_t plan_seg(uint64_t nv) {
    const uint64_t target = std::max<uint64_t>(1, nv / (uint64_t(num_sms()) * 64));
    return static_cast<uint32_t>(
        std::min<uint64_t>(16384, std::max<uint64_t>(TCS_PLAN_MIN_SEG, (target + 15) / 16 * 16)));
}

Plan* build_plan(const tcs_mebcrs* m, cudaStream_t s, uint32_t* max_nv, uint64_t* blocks_k,
                 uint64_t* groups16) {
    const uint64_t W = m->num_windows;
    const uint64_t nv = m->num_vectors;
    const uint32_t seg = plan_seg(nv);

    DBuf nslot((W + 1) * 4, s), nsplit((W + 1) * 4, s), slot_off((W + 1) * 4, s), split_off((W + 1) * 4, s);
    DBuf tot(sizeof(PlanTotals), s);
    TCS_CUDA(cudaMemsetAsync(tot.p, 0, sizeof(PlanTotals), s));
    const int grid = static_cast<int>(std::min<uint64_t>((W + 255) / 256 + 1, 4096));
    if (W) {
        plan_count<<<grid, 256, 0, s>>>(m->row_pointers, W, seg, m->k, nslot.as<uint32_t>(),
                                        nsplit.as<uint32_t>(), tot.as<PlanTotals>());
        TCS_LAUNCHED("plan_count");
    }
    exclusive_scan_u32(nslot.as<uint32_t>(), slot_off.as<uint32_t>(), W, s);
    exclusive_scan_u32(nsplit.as<uint32_t>(), split_off.as<uint32_t>(), W, s);
    PlanTotals h{};
    uint32_t n_slots = 0, n_split = 0;
    TCS_CUDA(cudaMemcpyAsync(&h, tot.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    TCS_CUDA(cudaMemcpyAsync(&n_slots, slot_off.as<uint32_t>() + W, 4, cudaMemcpyDeviceToHost, s));
    TCS_CUDA(cudaMemcpyAsync(&n_split, split_off.as<uint32_t>() + W, 4, cudaMemcpyDeviceToHost, s));
    TCS_CUDA(cudaStreamSynchronize(s));

    Plan* p = new Plan;
    p->seg = seg;
    p->n_slots = n_slots;
    p->n_split = n_split;
    p->n_items = n_slots + (W - n_split);
    p->items = static_cast<WorkItem*>(dalloc(std::max<uint64_t>(1, p->n_items) * sizeof(WorkItem), s));
    p->split = static_cast<SplitWindow*>(dalloc(std::max<uint64_t>(1, n_split) * sizeof(SplitWindow), s));
    if (W) {
        plan_fill<<<grid, 256, 0, s>>>(m->row_pointers, W, seg, slot_off.as<uint32_t>(), split_off.as<uint32_t>(),
                                       p->items, p->split, 0, nullptr);
        TCS_LAUNCHED("plan_fill");
    }
    if (max_nv) *max_nv = h.max_nv;
    if (blocks_k) *blocks_k = h.blocks_k;
    if (groups16) *groups16 = h.groups16;
    return p;
}

// The same work list without a host round trip (tcs_spmm_csr_host's
// chunks): the segment length comes from seg_nv (see below), the
// arrays are sized for the worst case (a split window has more than seg
// vectors, so split windows <= nv/seg and segments <= 2 nv/seg), and the
// real counts stay on the device (Plan::dcounts).
// seg_nv (0 = nv_cap): the vector count the segment length is sized for.
// A pipeline chunk uses its own: sized for the whole matrix, a small tail
// chunk's few hundred windows would each be walked by one warp (C3: 0.5 ms
// per tail-chunk SpMM instead of 0.04 ms + a 5 us split reduction).
Plan* build_plan_async(const tcs_mebcrs* m, uint64_t nv_cap, uint64_t seg_nv, cudaStream_t s) {
    const uint64_t W = m->num_windows;
    const uint32_t seg = plan_seg(std::max(nv_cap, seg_nv));
    const uint64_t split_cap = std::min<uint64_t>(W, nv_cap / seg);
    Plan* p = new Plan;
    p->seg = seg;
    p->n_split = split_cap;
    p->n_slots = nv_cap / seg + split_cap;
    p->n_items = p->n_slots + W;
    p->items = static_cast<WorkItem*>(dalloc(std::max<uint64_t>(1, p->n_items) * sizeof(WorkItem), s));
    p->split = static_cast<SplitWindow*>(dalloc(std::max<uint64_t>(1, split_cap) * sizeof(SplitWindow), s));
    p->dcounts = static_cast<uint32_t*>(dalloc(16, s));
    if (W && W <= kPlanSmallW) {
        plan_async_small<<<1, 1024, 0, s>>>(m->row_pointers, W, seg, m->k, p->items, p->split, p->n_items,
                                            p->dcounts);
        TCS_LAUNCHED("plan_async_small");
        return p;
    }
    TCS_CUDA(cudaMemsetAsync(p->dcounts, 0, 16, s));
    if (W) {
        DBuf nslot((W + 1) * 4, s), nsplit((W + 1) * 4, s), slot_off((W + 1) * 4, s), split_off((W + 1) * 4, s);
        DBuf tot(sizeof(PlanTotals), s);
        TCS_CUDA(cudaMemsetAsync(tot.p, 0, sizeof(PlanTotals), s));
        const int grid = static_cast<int>(std::min<uint64_t>((W + 255) / 256 + 1, 4096));
        plan_count<<<grid, 256, 0, s>>>(m->row_pointers, W, seg, m->k, nslot.as<uint32_t>(), nsplit.as<uint32_t>(),
                                        tot.as<PlanTotals>());
        TCS_LAUNCHED("plan_count");
        exclusive_scan_u32(nslot.as<uint32_t>(), slot_off.as<uint32_t>(), W, s);
        exclusive_scan_u32(nsplit.as<uint32_t>(), split_off.as<uint32_t>(), W, s);
        plan_fill<<<grid, 256, 0, s>>>(m->row_pointers, W, seg, slot_off.as<uint32_t>(), split_off.as<uint32_t>(),
                                       p->items, p->split, p->n_items, p->dcounts);
        TCS_LAUNCHED("plan_fill");
        plan_blocks_out<<<1, 1, 0, s>>>(tot.as<PlanTotals>(), p->dcounts);
        TCS_LAUNCHED("plan_blocks_out");
    }
    return p;
}

void free_plan(Plan* p, cudaStream_t s) {
    if (!p) return;
    dfree(p->dcounts, s);
    dfree(p->col_hot, s);
    dfree(p->ci_hot, s);
    dfree(p->items, s);
    dfree(p->split, s);
    dfree(p->live, s);
    dfree(p->exact_live, s);
    delete p;
}

// ------------------------------------------------------- pad / convert
namespace {
template <typename S, typename D>
__device__ __forceinline__ D cvt(S x);
template <> __device__ __forceinline__ float cvt<float, float>(float x) { return x; }
template <> __device__ __forceinline__ __half cvt<float, __half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ float cvt<__half, float>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ __half cvt<__half, __half>(__half x) { return x; }

template <typename S, typename D>
__global__ void pad_convert_kernel(const S* __restrict__ src, int64_t lds, D* __restrict__ dst, int64_t ldd,
                                   int64_t rows, int64_t cols, int64_t cols_pad) {
    const int64_t total = rows * cols_pad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols_pad, c = i % cols_pad;
        dst[r * ldd + c] = c < cols ? cvt<S, D>(src[r * lds + c]) : cvt<float, D>(0.0f);
    }
}
}  // namespace

void pad_convert(const void* src, tcs_dtype sdt, int64_t lds, void* dst, tcs_dtype ddt, int64_t ldd,
                 int64_t rows, int64_t cols, int64_t cols_pad, cudaStream_t s) {
    if (rows <= 0 || cols_pad <= 0) return;
    const int64_t total = rows * cols_pad;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, int64_t(num_sms()) * 16));
    if (sdt == TCS_DTYPE_F32 && ddt == TCS_DTYPE_F32)
        pad_convert_kernel<float, float><<<grid, 256, 0, s>>>((const float*)src, lds, (float*)dst, ldd, rows, cols, cols_pad);
    else if (sdt == TCS_DTYPE_F32 && ddt == TCS_DTYPE_F16)
        pad_convert_kernel<float, __half><<<grid, 256, 0, s>>>((const float*)src, lds, (__half*)dst, ldd, rows, cols, cols_pad);
    else if (sdt == TCS_DTYPE_F16 && ddt == TCS_DTYPE_F32)
        pad_convert_kernel<__half, float><<<grid, 256, 0, s>>>((const __half*)src, lds, (float*)dst, ldd, rows, cols, cols_pad);
    else
        pad_convert_kernel<__half, __half><<<grid, 256, 0, s>>>((const __half*)src, lds, (__half*)dst, ldd, rows, cols, cols_pad);
    TCS_LAUNCHED("pad_convert");
}

namespace {
__global__ void round_values_kernel(int precision, const float* __restrict__ in, float* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = precision == TCS_FP16 ? __half2float(__float2half_rn(in[i])) : __uint_as_float(dev::to_tf32(in[i]));
}
}  // namespace

void check_mebcrs(const tcs_mebcrs* m, bool any_height) {
    if (!m) fail(TCS_ERR_ARGUMENT, "null ME-BCRS handle");
    if (m->vector_height != 8 && !(any_height && m->vector_height == 16))
        fail(TCS_ERR_ARGUMENT, "ME-BCRS vector height must be 8");
    if (m->precision != TCS_FP16 && m->precision != TCS_TF32) fail(TCS_ERR_ARGUMENT, "unknown precision");
    if (m->k != (m->precision == TCS_FP16 ? 8u : 4u)) fail(TCS_ERR_FORMAT, "block width k does not match precision");
    if (m->precision == TCS_TF32 && m->value_dtype != TCS_DTYPE_F32)
        fail(TCS_ERR_ARGUMENT, "TF32 ME-BCRS values must be stored as f32");
    if (m->num_windows != (m->rows + m->vector_height - 1) / m->vector_height) fail(TCS_ERR_FORMAT, "row_pointers length must be numWindows+1");
    if (m->num_vectors >= (1ull << 32)) fail(TCS_ERR_FORMAT, "vector count exceeds u32 row pointers");
    if (!m->row_pointers) fail(TCS_ERR_ARGUMENT, "null row_pointers");
    if (m->num_vectors && (!m->column_indices || !m->values)) fail(TCS_ERR_ARGUMENT, "null ME-BCRS arrays");
}

void upload_mebcrs(uint64_t rows, uint64_t cols, tcs_precision precision, uint32_t vh, const uint32_t* row_pointers,
                   const uint32_t* column_indices, const float* values, tcs_mebcrs* out, cudaStream_t s) {
    if (!out || !row_pointers) fail(TCS_ERR_ARGUMENT, "null argument");
    if (precision != TCS_FP16 && precision != TCS_TF32) fail(TCS_ERR_ARGUMENT, "unknown precision");
    if (vh != 8 && vh != 16) fail(TCS_ERR_ARGUMENT, "vector height must be 8 or 16");
    tcs_mebcrs m{};
    m.rows = rows;
    m.cols = cols;
    m.vector_height = vh;
    m.k = precision == TCS_FP16 ? 8 : 4;
    m.precision = precision;
    m.value_dtype = TCS_DTYPE_F32;
    m.num_windows = (rows + vh - 1) / vh;
    m.num_vectors = row_pointers[m.num_windows];
    m.row_pointers = static_cast<uint32_t*>(dalloc((m.num_windows + 1) * 4, s));
    m.column_indices = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, m.num_vectors) * 4, s));
    m.values = dalloc(std::max<uint64_t>(1, uint64_t(vh) * m.num_vectors) * 4, s);
    m.flags = TCS_MEBCRS_OWN_STRUCTURE | TCS_MEBCRS_OWN_VALUES;
    TCS_CUDA(cudaMemcpyAsync(m.row_pointers, row_pointers, (m.num_windows + 1) * 4, cudaMemcpyHostToDevice, s));
    if (m.num_vectors) {
        TCS_CUDA(cudaMemcpyAsync(m.column_indices, column_indices, m.num_vectors * 4, cudaMemcpyHostToDevice, s));
        TCS_CUDA(cudaMemcpyAsync(m.values, values, uint64_t(vh) * m.num_vectors * 4, cudaMemcpyHostToDevice, s));
    }
    *out = m;
    const tcs_stream_t ts = reinterpret_cast<tcs_stream_t>(s);
    tcs_status rc = tcs_mebcrs_prepare(out, ts);
    if (rc != TCS_OK) {
        std::string msg = tcs_last_error();
        tcs_mebcrs_free(out, ts);
        fail(rc, msg);
    }
}

}  // namespace tcs

// ===================================================================== ABI
using namespace tcs;

extern "C" {

const char* tcs_version(void) { return "tcsparse-b200 0.1 (sm_100a)"; }
const char* tcs_last_error(void) { return t_last_error.c_str(); }
uint64_t tcs_launch_count(void) { return g_launches.load(); }

tcs_status tcs_round_values(tcs_precision precision, const float* in, float* out, uint64_t n, tcs_stream_t stream) {
    return guard([&] {
        if (precision != TCS_FP16 && precision != TCS_TF32) fail(TCS_ERR_ARGUMENT, "unknown precision");
        if (n == 0) return;
        if (!in || !out) fail(TCS_ERR_ARGUMENT, "null argument");
        const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 32));
        round_values_kernel<<<grid, 256, 0, st(stream)>>>(precision, in, out, n);
        TCS_LAUNCHED("round_values");
    });
}

tcs_status tcs_mebcrs_prepare(tcs_mebcrs* m, tcs_stream_t stream) {
    return guard([&] {
        check_mebcrs(m, true);
        cudaStream_t s = st(stream);
        uint8_t* exact = nullptr;  // exact liveness of these values survives a re-prepare
        if (m->plan && !(m->flags & TCS_MEBCRS_BORROWED_PLAN)) {
            Plan* old = static_cast<Plan*>(m->plan);
            if (old->exact_for(m->values)) std::swap(exact, old->exact_live);
            free_plan(old, s);
        }
        m->plan = nullptr;
        m->flags &= ~TCS_MEBCRS_BORROWED_PLAN;
        uint32_t mx = 0;
        uint64_t blocks = 0, groups = 0;
        m->plan = build_plan(m, s, &mx, &blocks, &groups);
        if (exact) {
            static_cast<Plan*>(m->plan)->exact_live = exact;
            static_cast<Plan*>(m->plan)->exact_live_src = m->values;
        }
        m->max_window_vectors = mx;
        m->num_blocks = blocks;
        m->num_groups16 = groups;
    });
}

tcs_status tcs_mebcrs_free(tcs_mebcrs* m, tcs_stream_t stream) {
    return guard([&] {
        if (!m) return;
        cudaStream_t s = st(stream);
        if (m->flags & TCS_MEBCRS_OWN_STRUCTURE) {
            dfree(m->row_pointers, s);
            dfree(m->column_indices, s);
        }
        // a liveness cache built from these values must not outlive them
        // (the allocator may hand the address to another handle of this plan)
        if (auto* p = static_cast<Plan*>(m->plan); p && p->live_src == m->values) p->live_src = nullptr;
        if (auto* p = static_cast<Plan*>(m->plan); p && p->exact_live_src == m->values) p->exact_live_src = nullptr;
        if (m->flags & TCS_MEBCRS_OWN_VALUES) dfree(m->values, s);
        if (!(m->flags & TCS_MEBCRS_BORROWED_PLAN)) free_plan(static_cast<Plan*>(m->plan), s);
        std::memset(m, 0, sizeof(*m));
    });
}

tcs_status tcs_mebcrs_download(const tcs_mebcrs* m, uint32_t* row_pointers, uint32_t* column_indices,
                               float* values, tcs_stream_t stream) {
    return guard([&] {
        check_mebcrs(m, true);
        cudaStream_t s = st(stream);
        if (row_pointers)
            TCS_CUDA(cudaMemcpyAsync(row_pointers, m->row_pointers, (m->num_windows + 1) * 4, cudaMemcpyDeviceToHost, s));
        if (column_indices && m->num_vectors)
            TCS_CUDA(cudaMemcpyAsync(column_indices, m->column_indices, m->num_vectors * 4, cudaMemcpyDeviceToHost, s));
        if (values && m->num_vectors) {
            const uint64_t n = uint64_t(m->vector_height) * m->num_vectors;
            if (m->value_dtype == TCS_DTYPE_F32) {
                TCS_CUDA(cudaMemcpyAsync(values, m->values, n * 4, cudaMemcpyDeviceToHost, s));
            } else {
                DBuf wide(n * 4, s);
                // 1-row view: treat the value array as a single row of n elements
                pad_convert(m->values, TCS_DTYPE_F16, (int64_t)n, wide.p, TCS_DTYPE_F32, (int64_t)n, 1, (int64_t)n,
                            (int64_t)n, s);
                TCS_CUDA(cudaMemcpyAsync(values, wide.p, n * 4, cudaMemcpyDeviceToHost, s));
            }
        }
        TCS_CUDA(cudaStreamSynchronize(s));
    });
}

tcs_status tcs_mebcrs_upload(uint64_t rows, uint64_t cols, tcs_precision precision, const uint32_t* row_pointers,
                             const uint32_t* column_indices, const float* values, tcs_mebcrs* out,
                             tcs_stream_t stream) {
    return guard([&] {
        upload_mebcrs(rows, cols, precision, 8, row_pointers, column_indices, values, out, st(stream));
    });
}

tcs_status tcs_mebcrs_validate(const tcs_mebcrs* m, tcs_stream_t stream) {
    return guard([&] {
        check_mebcrs(m, true);
        std::vector<uint32_t> rp(m->num_windows + 1), ci(m->num_vectors);
        cudaStream_t s = st(stream);
        TCS_CUDA(cudaMemcpyAsync(rp.data(), m->row_pointers, rp.size() * 4, cudaMemcpyDeviceToHost, s));
        if (!ci.empty())
            TCS_CUDA(cudaMemcpyAsync(ci.data(), m->column_indices, ci.size() * 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
        // ref mebcrs.hpp:58-77
        if (rp.front() != 0) fail(TCS_ERR_FORMAT, "row_pointers must start at 0");
        for (size_t w = 0; w + 1 < rp.size(); ++w)
            if (rp[w] > rp[w + 1]) fail(TCS_ERR_FORMAT, "row_pointers must be nondecreasing");
        if (rp.back() != ci.size()) fail(TCS_ERR_FORMAT, "row_pointers end must equal stored vector count");
        for (size_t w = 0; w + 1 < rp.size(); ++w)
            for (uint32_t p = rp[w]; p < rp[w + 1]; ++p) {
                if (ci[p] >= m->cols) fail(TCS_ERR_FORMAT, "column index out of range");
                if (p > rp[w] && ci[p - 1] >= ci[p]) fail(TCS_ERR_FORMAT, "column indices must ascend within a window");
            }
    });
}

}  // extern "C"
