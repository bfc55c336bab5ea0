// Internal helpers shared by the sm_100a kernels and the C-ABI glue.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "tcs/tcs.h"

namespace tcs {

// NVTX range over one C-ABI call (header-only NVTX v3: a no-op unless a
// tool such as ncu / nsys injects itself), so profiles group kernels by the
// entry point that launched them.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    tcs_status code;
    Error(tcs_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
extern std::atomic<uint64_t> g_launches;

[[noreturn]] inline void fail(tcs_status c, const std::string& m) { throw Error(c, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation) fail(TCS_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
        fail(TCS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define TCS_CUDA(x) ::tcs::cuda_check((x), #x)
// After every kernel launch: counts it and surfaces launch errors.
#define TCS_LAUNCHED(name)                                   \
    do {                                                     \
        ::tcs::g_launches.fetch_add(1, std::memory_order_relaxed); \
        ::tcs::cuda_check(cudaGetLastError(), name);         \
    } while (0)

// Launch with the programmatic-stream-serialization attribute (see
// pdl_wait / pdl_trigger below).  TCS_PDL=0: plain stream order (A/B knob).
#ifndef TCS_PDL
#define TCS_PDL 1
#endif
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = TCS_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TCS_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Runs `body`, mapping exceptions onto status codes (no exception crosses
// the C-ABI).
template <typename F>
tcs_status guard(F&& body) {
    try {
        body();
        set_last_error("");
        return TCS_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return TCS_ERR_OOM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return TCS_ERR_CUDA;
    }
}

// ------------------------------------------------- stream-ordered memory
void* dalloc(size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);
int num_sms();

// RAII device buffer (stream-ordered).
struct DBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(size_t bytes, cudaStream_t st) : p(dalloc(bytes, st)), s(st) {}
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
    DBuf& operator=(DBuf&& o) noexcept {
        reset();
        p = o.p; s = o.s; o.p = nullptr;
        return *this;
    }
    ~DBuf() { reset(); }
    void reset() {
        if (p) dfree(p, s);
        p = nullptr;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// ------------------------------------------------------------ scan / plan
// Exclusive prefix sum of n u32 values into out (n+1 entries, out[n] =
// total).  Totals must fit in u32 (the reference's u32 row pointers).
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s);

// Work list for SpMM / SDDMM: items of at most `seg` vectors (a multiple of
// 16) of one window.  Windows longer than `seg` are split; their partial
// SpMM sums are reduced in segment order (deterministic).
struct WorkItem {
    uint32_t window;
    uint32_t vbeg;  // window-relative vector range [vbeg, vend)
    uint32_t vend;
    uint32_t slot;  // partial-sum slot for split windows, else kNoSlot
};
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
struct SplitWindow {
    uint32_t window;
    uint32_t first_slot;
    uint32_t nseg;
    uint32_t pad;
};
struct Plan {
    uint32_t seg = 0;
    uint64_t n_items = 0;
    uint64_t n_slots = 0;
    uint64_t n_split = 0;
    WorkItem* items = nullptr;      // device
    SplitWindow* split = nullptr;   // device
    // SDDMM liveness bytes of the values at `live_src` (TCS_CFG_STATIC_MASK),
    // built on first use; rebuilt when a handle sharing this plan brings
    // other values.
    uint8_t* live = nullptr;        // device, num_vectors + 16
    const void* live_src = nullptr;
    // Exact liveness bytes of an F16 encode whose binary16 values lost a tiny
    // nonzero f32 value (encode.cu, CheckOut::tiny); valid for the values at
    // `exact_live_src` only.  Every liveness consumer prefers them.
    uint8_t* exact_live = nullptr;  // device, num_vectors + 16
    const void* exact_live_src = nullptr;
    const uint8_t* exact_for(const void* values) const {
        return exact_live && exact_live_src == values ? exact_live : nullptr;
    }
    // Pipelined plans (build_plan_async, no host round trip): n_items,
    // n_slots and n_split above are capacities.  The real items sit at the
    // END of `items`, so a persistent SpMM whose claim counters start at
    // dcounts[0] (= capacity - real items) walks exactly them; dcounts[1] is
    // the real number of split windows; dcounts[2..3] the u64 block count.
    uint32_t* dcounts = nullptr;  // device
    // Hot dense-operand rows (tcs_spmm when B does not fit in L2): bit c set
    // iff column c is among the most gathered columns whose B rows fit the
    // hot budget at `col_hot_rowbytes` per row; those gathers are issued
    // L2::evict_last, the rest evict_first.  Built on first use, kept.
    uint32_t* col_hot = nullptr;  // device, ceil(cols / 32) words
    uint32_t* ci_hot = nullptr;   // device, column indices with the hot bit in bit 31
    uint64_t col_hot_rowbytes = 0;
};
Plan* build_plan(const tcs_mebcrs* m, cudaStream_t s, uint32_t* max_nv, uint64_t* blocks_k,
                 uint64_t* groups16);
Plan* build_plan_async(const tcs_mebcrs* m, uint64_t nv_cap, uint64_t seg_nv, cudaStream_t s);
// check_dev: a caller-owned, zeroed block of encode_check_bytes() device
// bytes; its validation code sits at encode_check_bad_offset() (u32).
void encode_mebcrs_async(const tcs_csr* csr, tcs_precision precision, tcs_dtype value_dtype, tcs_mebcrs* out,
                         cudaStream_t s, void* check_dev, uint64_t seg_nv, cudaEvent_t values_ready);
const char* encode_bad_msg(uint32_t code);
size_t encode_check_bytes();
size_t encode_check_bad_offset();
void free_plan(Plan* p, cudaStream_t s);

// ------------------------------------------------------------ conversions
// dst[r][c] (ld_dst, dst dtype) = src[r][c] for c < cols, 0 for cols <= c < cols_pad.
void pad_convert(const void* src, tcs_dtype sdt, int64_t lds, void* dst, tcs_dtype ddt, int64_t ldd,
                 int64_t rows, int64_t cols, int64_t cols_pad, cudaStream_t s);

// vector height 8 only unless any_height (8 or 16: the 16x1 baseline layout).
void check_mebcrs(const tcs_mebcrs* m, bool any_height = false);
// Reference cost model (cost.cu).
void mebcrs_cost(const tcs_mebcrs* m, uint64_t nnz, int64_t n_cols, tcs_mapping mapping, tcs_cost* out, cudaStream_t s);
// Host arrays -> device handle (F32 values, vector height 8 or 16), prepared.
void upload_mebcrs(uint64_t rows, uint64_t cols, tcs_precision precision, uint32_t vh, const uint32_t* row_pointers,
                   const uint32_t* column_indices, const float* values, tcs_mebcrs* out, cudaStream_t s);

// TMA-gather + tcgen05 SpMM (spmm_tc05.cu); false = not applicable, nothing launched.
bool spmm_tc05(const tcs_mebcrs* A, const Plan* plan, const __half* B, int64_t ldb, int64_t b_rows, int64_t n,
               float* c, int64_t ldc, float* partial, int64_t ldp, cudaStream_t s);
inline cudaStream_t st(tcs_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// SDDMM pieces shared with the fused SDDMM -> row-softmax (sddmm.cu).
void sddmm_check(const tcs_mebcrs* mask, const void* a, tcs_dtype a_dtype, int64_t lda, int64_t a_rows, int64_t f_a,
                 const void* bt, tcs_dtype bt_dtype, int64_t ldbt, int64_t bt_rows, int64_t f_b, tcs_dtype out_dtype,
                 const tcs_kernel_config* cfg);
// Per-vector liveness bytes of a mask (bit r: row r's mask value != 0).
// mask_liveness caches them in the work list (TCS_CFG_STATIC_MASK);
// build_liveness writes nv + 16 bytes into caller memory.
const uint8_t* mask_liveness(const tcs_mebcrs* mask, Plan* plan, cudaStream_t s);
void build_liveness(const tcs_mebcrs* mask, uint8_t* live, cudaStream_t s);
void sddmm_launch(const tcs_mebcrs* mask, Plan* plan, const void* a, tcs_dtype a_dtype, int64_t lda,
                  int64_t a_rows, const void* bt, tcs_dtype bt_dtype, int64_t ldbt, int64_t bt_rows, int64_t F,
                  void* out_values, tcs_dtype out_dtype, float dead, bool static_mask, cudaStream_t s);

// AGNN aggregation pieces (softmax.cu / spmm.cu): per-row softmax
// statistics (m, 1/sum) of binary16 scores with dead slots -inf, and the
// SpMM that applies the softmax to its sparse operand in registers.
void softmax_rowstats(const tcs_mebcrs* S, const Plan* plan, float scale, float2* rowstat, cudaStream_t s);
void spmm_f16_softmax(const tcs_mebcrs* S, const Plan* plan, const float2* rowstat, float scale, const void* b,
                      tcs_dtype b_dtype, int64_t ldb, int64_t b_rows, int64_t n, float* c, int64_t ldc,
                      cudaStream_t s);

}  // namespace tcs

// ============================================================ device helpers
namespace tcs::dev {

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Work-item claiming for the persistent kernels.  Items are dealt
// round-robin to NS counters on separate 128-byte lines (item i to stripe
// i % NS); a warp starts on its block's stripe and moves on when that stripe
// runs dry.  Still one item per atomic -- the balance of a single counter --
// but the same-address atomics of ~1200 resident warps are spread over the
// stripes.  Every claimed list owns kClaimBytes of zeroed counters (room for
// kMaxClaimStripes).  Measured per kernel (profiles/r1s4_claim_stripes.txt):
// the C5 softmax statistics pass drops 1.55 -> 1.14 ms at NS = 8, the SDDMM
// gains ~1-2% at NS = 4, the C3 SpMM prefers the plain counter.
constexpr uint32_t kMaxClaimStripes = 8;
constexpr uint32_t kClaimStride = 32;  // u32 per stripe counter (128 B)
constexpr size_t kClaimBytes = size_t(kMaxClaimStripes) * kClaimStride * sizeof(uint32_t);
template <uint32_t NS>
struct StripedClaim {
    static_assert(NS >= 1 && NS <= kMaxClaimStripes, "stripe count");
    uint32_t stripe, tried = 0;
    __device__ __forceinline__ StripedClaim() : stripe(blockIdx.x % NS) {}
    __device__ __forceinline__ bool get(uint32_t* counters, uint64_t n_items, uint32_t& idx) {
        while (tried < NS) {
            uint32_t k = 0;
            if ((threadIdx.x & 31u) == 0) k = atomicAdd(counters + stripe * kClaimStride, 1u);
            k = __shfl_sync(0xffffffffu, k, 0);
            const uint64_t i = uint64_t(k) * NS + stripe;
            if (i < n_items) {
                idx = static_cast<uint32_t>(i);
                return true;
            }
            stripe = (stripe + 1) % NS;
            ++tried;
        }
        return false;
    }
};

// Plain single-counter claim (stripe 0 of a kClaimBytes block).
__device__ __forceinline__ uint32_t next_item(uint32_t* counter, uint32_t lane) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(counter, 1u);
    return __shfl_sync(0xffffffffu, i, 0);
}
// The claim counter of slab `slab`.
__device__ __forceinline__ uint32_t* slab_counter(uint32_t* counters, uint32_t slab) {
    return counters + static_cast<uint64_t>(slab) * (kClaimBytes / 4);
}

// Programmatic dependent launch.  A kernel launched with launch_pdl may be
// scheduled while the previous kernel on the stream is still draining (once
// that kernel has executed pdl_trigger, or at its exit); it must execute
// pdl_wait() -- which returns when the previous grid has completed and its
// memory is visible -- before it touches global memory.  Without the launch
// attribute both instructions are no-ops.  Used by the latency-bound small-
// list kernels, whose launch latency is then hidden behind their
// predecessor's tail (back-to-back calls, CUDA graphs).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// RNE fp32 -> tf32 (cvt.rn.tf32.f32, sm_90+); matches the reference's
// round_to_tf32 (ref precision.hpp:42-46; inf/NaN pass through).
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// D = A(16x16 f16, row) * B(16x8 f16, col) + D, fp32 accumulate.
__device__ __forceinline__ void mma_f16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                              uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// D = A(16x8 tf32, row) * B(8x8 tf32, col) + D.
__device__ __forceinline__ void mma_tf32_1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                              uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_lo(uint32_t x, uint32_t y) { return __byte_perm(x, y, 0x5410); }
__device__ __forceinline__ uint32_t pack_hi(uint32_t x, uint32_t y) { return __byte_perm(x, y, 0x7632); }

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
// Two f32 -> packed f16x2 with RNE (lo = a, hi = b).
__device__ __forceinline__ uint32_t f2_to_h2(float a, float b) { return h2_bits(__floats2half2_rn(a, b)); }

// Streaming (read-once) loads of the sparse arrays: keep them out of L1 so
// L1 holds the reused dense rows.
__device__ __forceinline__ uint32_t ld_stream_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// L2 prefetch of one line (the sparse value / column streams, a few steps
// ahead of their loads, so those hit L2 instead of waiting on DRAM).
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// L2 evict-first policy (createpolicy) for read-once streams, so they do not
// displace an L2-resident gathered operand.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint32_t ld_stream_ef_u32(const void* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ld_stream_u64(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_stream_u128(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
// Dense-row gathers: read-only path, L1-allocating (hub rows are reused).
__device__ __forceinline__ uint4 ld_gather_128(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_gather_32(const void* p) {
    uint32_t v;
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// The gather without L1 allocation (A/B knob TCS_GATHER_NA).
__device__ __forceinline__ uint4 ld_gather_128_na(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_gather_64(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
// The same gathers with an explicit L2 cache policy (createpolicy): hot
// dense-operand rows evict_last, cold ones evict_first (see Plan::col_hot).
__device__ __forceinline__ uint4 ld_gather_128_pol(const void* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ld_gather_64_pol(const void* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.b32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
template <int KIND>  // 0 evict_first, 1 evict_normal, 2 evict_unchanged
__device__ __forceinline__ uint64_t l2_cold_policy() {
    uint64_t pol;
    if constexpr (KIND == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else if constexpr (KIND == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_stream_f4(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d));
}

// Block-wide exclusive scan of one u32 per thread (blockDim.x a multiple of
// 32, <= 1024); returns the exclusive prefix, *total = block sum.  Contains
// __syncthreads: call from all threads of the block.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < nwarps ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t warp_prefix = warp ? warp_sums[warp - 1] : 0;
    *total = warp_sums[nwarps - 1];
    __syncthreads();
    return warp_prefix + x - v;
}

}  // namespace tcs::dev
