// Row-wise softmax over the ME-BCRS pattern: the middle stage of the AGNN
// attention layer (SDDMM -> row softmax -> SpMM, PAPER.md:685-712;
// BASELINE.json configs[4]).  The reference has no such operator
// (SPEC.md:368); the liveness rule is the reference SDDMM's sampling rule
// (a position is part of the pattern iff the mask value != 0, ref
// sddmm.hpp:131), so scores that happen to be 0 still take part.
//
//   out[pos] = exp(scale*x[pos] - max_r) / sum_r   over the live positions
//              of row r of the window; every other slot 0.
//
// Runs on the SpMM/SDDMM work list, so hub windows (R-MAT: 450 K vectors in
// one window) are spread over many warps:
//   K1 softmax_items   persistent warps; per item one online pass computes the
//                      per-row (max, sum exp) over the item's vectors: a full
//                      block is row-major (8 rows x K), so lane l streams row
//                      l%8 of block l/8 with one K-wide vector load and keeps
//                      scalar statistics for that row (xor-8/16 merged);
//                      an unsplit window is normalised in place right away,
//                      a split segment stores its 8 partials.
//   K2 softmax_combine per split window: merges the segments' partials.
//   K3 softmax_finish  writes the normalised values of split segments.
#include <algorithm>
#include <cfloat>
#include <type_traits>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

template <typename V>
__device__ __forceinline__ float ld_val(const V* p, uint64_t i);
template <>
__device__ __forceinline__ float ld_val<float>(const float* p, uint64_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ float ld_val<__half>(const __half* p, uint64_t i) { return __half2float(__ldg(p + i)); }

template <typename V>
__device__ __forceinline__ bool live_at(const V* m, uint64_t i);
template <>
__device__ __forceinline__ bool live_at<float>(const float* m, uint64_t i) {
    return (__float_as_uint(__ldg(m + i)) & 0x7FFFFFFFu) != 0u;
}
template <>
__device__ __forceinline__ bool live_at<__half>(const __half* m, uint64_t i) {
    return (__half_as_ushort(__ldg(m + i)) & 0x7FFFu) != 0u;
}

template <typename V>
__device__ __forceinline__ void st_val(V* p, uint64_t i, float x);
template <>
__device__ __forceinline__ void st_val<float>(float* p, uint64_t i, float x) { p[i] = x; }
template <>
__device__ __forceinline__ void st_val<__half>(__half* p, uint64_t i, float x) { p[i] = __float2half_rn(x); }

struct RowStat {
    float m, s;  // running max, sum of exp(x - m)
};

__device__ __forceinline__ void merge(float& m, float& s, float m2, float s2) {
    const float mm = fmaxf(m, m2);
    s = (m == -FLT_MAX ? 0.f : s * __expf(m - mm)) + (m2 == -FLT_MAX ? 0.f : s2 * __expf(m2 - mm));
    m = mm;
}

// ---- K-wide vector access to one block row (16-B / 8-B aligned: the block
// row starts at element 8*base + 8K*b + r*K)
template <int N>
__device__ __forceinline__ void ldv(const float* p, float (&x)[N]) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p + i));
        x[i] = t.x; x[i + 1] = t.y; x[i + 2] = t.z; x[i + 3] = t.w;
    }
}
template <int N>
__device__ __forceinline__ void ldv(const __half* p, float (&x)[N]) {
    if constexpr (N == 8) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
            x[2 * i] = f.x; x[2 * i + 1] = f.y;
        }
    } else {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
        const uint32_t w[2] = {t.x, t.y};
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
            x[2 * i] = f.x; x[2 * i + 1] = f.y;
        }
    }
}
template <int N>
__device__ __forceinline__ void ldlive(const float* p, bool (&l)[N]) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(p + i));
        l[i] = (t.x & 0x7FFFFFFFu) != 0; l[i + 1] = (t.y & 0x7FFFFFFFu) != 0;
        l[i + 2] = (t.z & 0x7FFFFFFFu) != 0; l[i + 3] = (t.w & 0x7FFFFFFFu) != 0;
    }
}
template <int N>
__device__ __forceinline__ void ldlive(const __half* p, bool (&l)[N]) {
    uint32_t w[N / 2];
    if constexpr (N == 8) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
        w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
    } else {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = t.x; w[1] = t.y;
    }
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
        l[2 * i] = (w[i] & 0x7FFFu) != 0;
        l[2 * i + 1] = (w[i] & 0x7FFF0000u) != 0;
    }
}
template <int N>
__device__ __forceinline__ void stv(float* p, const float (&y)[N]) {
#pragma unroll
    for (int i = 0; i < N; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(y[i], y[i + 1], y[i + 2], y[i + 3]);
}
template <int N>
__device__ __forceinline__ void stv(__half* p, const float (&y)[N]) {
    uint32_t w[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
        const __half2 h = __floats2half2_rn(y[2 * i], y[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    if constexpr (N == 8) *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    else *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
}


// Lane l owns row r = l % 8 of block (l / 8) of every group of 4 full blocks
// -- the K contiguous values of that block row -- so each lane's statistics
// belong to one row.  A narrow last block (width w < K, only at the end of
// a window) is taken by lanes 0..7, row = lane, values r*w .. r*w+w-1.
// Liveness of a block row: from the mask values, or -- VM = void, the fused
// SDDMM -> softmax whose dead slots hold -inf -- from the scores themselves.
template <uint32_t K, typename VM>
__device__ __forceinline__ void live_k(const VM* mask, uint64_t p, const float (&x)[K], bool (&l)[K]) {
    if constexpr (std::is_void_v<VM>) {
#pragma unroll
        for (uint32_t j = 0; j < K; ++j) l[j] = x[j] != -INFINITY;
    } else {
        ldlive<K>(mask + p, l);
    }
}
template <typename VM>
__device__ __forceinline__ bool live_1(const VM* mask, uint64_t p, float x) {
    if constexpr (std::is_void_v<VM>) return x != -INFINITY;
    else return live_at<VM>(mask, p);
}

// z = scale * x over a block row, -inf where not live.
template <uint32_t K, typename VS, typename VM>
__device__ __forceinline__ void block_z(const VS* scores, const VM* mask, uint64_t p, float scale, float (&z)[K]) {
    float x[K];
    bool l[K];
    ldv<K>(scores + p, x);
    live_k<K, VM>(mask, p, x, l);
#pragma unroll
    for (uint32_t j = 0; j < K; ++j) z[j] = l[j] ? scale * x[j] : -INFINITY;
}

// Adds n values (-inf = not live) to the running (m, s): one max over the
// values, at most one rescale, then branch-free exps (exp(-inf) = 0; m
// starts at -FLT_MAX, so no inf - inf arises).
template <uint32_t N>
__device__ __forceinline__ void add_values(float& m, float& s, const float (&z)[N]) {
    float bm = z[0];
#pragma unroll
    for (uint32_t j = 1; j < N; ++j) bm = fmaxf(bm, z[j]);
    if (bm > m) {
        s *= __expf(m - bm);
        m = bm;
    }
#pragma unroll
    for (uint32_t j = 0; j < N; ++j) s += __expf(z[j] - m);
}

template <uint32_t K, typename VS, typename VM>
__device__ __forceinline__ void row_stats(const VS* scores, const VM* mask, uint64_t vb, uint32_t v0, uint32_t v1,
                                          uint32_t lane, float scale, float& m, float& s) {
    const uint32_t r = lane & 7, bl = lane >> 3;
    const uint32_t b0 = v0 / K, nfull = (v1 - v0) / K, w = (v1 - v0) % K;
    m = -FLT_MAX;
    s = 0.f;
    // unrolled so that several block rows are in flight per lane (the loads
    // do not depend on the running (m, s)); 1.63 -> 1.56 ms on C5
#pragma unroll 4
    for (uint32_t b = b0 + bl; b < b0 + nfull; b += 4) {
        float z[K];
        block_z<K, VS, VM>(scores, mask, vb + 8ull * K * b + r * K, scale, z);
        add_values<K>(m, s, z);
    }
    if (w && lane < 8) {
        const uint64_t p = vb + 8ull * K * (b0 + nfull) + r * w;
        float z[K - 1];
#pragma unroll
        for (uint32_t j = 0; j < K - 1; ++j) {
            z[j] = -INFINITY;
            if (j < w) {
                const float x = ld_val<VS>(scores, p + j);
                if (live_1<VM>(mask, p + j, x)) z[j] = scale * x;
            }
        }
        add_values<K - 1>(m, s, z);
    }
    // merge the 4 lanes that own row r (lanes r, r+8, r+16, r+24)
#pragma unroll
    for (int o = 8; o <= 16; o <<= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
        merge(m, s, m2, s2);
    }
}

template <uint32_t K, typename VS, typename VM, typename VO>
__device__ __forceinline__ void row_write(const VS* scores, const VM* mask, VO* out, uint64_t vb, uint32_t v0,
                                          uint32_t v1, uint32_t lane, float scale, float m, float inv) {
    const uint32_t r = lane & 7, bl = lane >> 3;
    const uint32_t b0 = v0 / K, nfull = (v1 - v0) / K, w = (v1 - v0) % K;
    for (uint32_t b = b0 + bl; b < b0 + nfull; b += 4) {
        const uint64_t p = vb + 8ull * K * b + r * K;
        float z[K], y[K];
        block_z<K, VS, VM>(scores, mask, p, scale, z);
#pragma unroll
        for (uint32_t j = 0; j < K; ++j) y[j] = __expf(z[j] - m) * inv;  // not live: exp(-inf) = 0
        stv<K>(out + p, y);
    }
    if (w && lane < 8) {  // all loads before any store: no load-after-store round trips
        const uint64_t p = vb + 8ull * K * (b0 + nfull) + r * w;
        float x[K];
        bool l[K];
#pragma unroll
        for (uint32_t j = 0; j < K - 1; ++j) {
            x[j] = j < w ? ld_val<VS>(scores, p + j) : 0.f;
            l[j] = j < w && live_1<VM>(mask, p + j, x[j]);
        }
#pragma unroll
        for (uint32_t j = 0; j < K - 1; ++j)
            if (j < w) st_val<VO>(out, p + j, l[j] ? __expf(scale * x[j] - m) * inv : 0.f);
    }
}

template <uint32_t K, typename VS, typename VM, typename VO>
__global__ void __launch_bounds__(256) softmax_items(const WorkItem* __restrict__ items, uint64_t n_items,
                                                     uint32_t* counter, const uint32_t* __restrict__ rp,
                                                     const VS* scores, const VM* __restrict__ mask, VO* out,
                                                     float scale, RowStat* __restrict__ part) {
    const uint32_t lane = threadIdx.x & 31;
    dev::StripedClaim<8> claim;
    for (uint32_t idx; claim.get(counter, n_items, idx);) {
        const WorkItem it = items[idx];
        const uint64_t vb = 8ull * __ldg(rp + it.window);
        float m, s;
        row_stats<K, VS, VM>(scores, mask, vb, it.vbeg, it.vend, lane, scale, m, s);
        if (it.slot != kNoSlot) {  // segment of a split window: publish partials
            if (lane < 8) part[8ull * it.slot + lane] = RowStat{m, s};
            continue;
        }
        row_write<K, VS, VM, VO>(scores, mask, out, vb, it.vbeg, it.vend, lane, scale, m, s > 0.f ? 1.f / s : 0.f);
    }
}

// one thread per (split window, row): merge the segments' partials in place
// into the first segment's slot
__global__ void softmax_combine(const SplitWindow* __restrict__ split, uint64_t n_split, RowStat* __restrict__ part) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 8 * n_split;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const SplitWindow sw = split[i / 8];
        const uint32_t r = static_cast<uint32_t>(i % 8);
        float m = -FLT_MAX, s = 0.f;
        for (uint32_t q = 0; q < sw.nseg; ++q) {
            const RowStat x = part[8ull * (sw.first_slot + q) + r];
            merge(m, s, x.m, x.s);
        }
        part[8ull * sw.first_slot + r] = RowStat{m, s};
    }
}

template <uint32_t K, typename VS, typename VM, typename VO>
__global__ void __launch_bounds__(256) softmax_finish(const WorkItem* __restrict__ items, uint64_t n_slots,
                                                      const SplitWindow* __restrict__ split, uint64_t n_split,
                                                      const uint32_t* __restrict__ rp, const VS* scores,
                                                      const VM* __restrict__ mask, VO* out, float scale,
                                                      const RowStat* __restrict__ part) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    // split items occupy item indices [0, n_slots), slot == index
    for (uint64_t idx = w0; idx < n_slots; idx += nw) {
        const WorkItem it = items[idx];
        // first slot of this item's window: binary search the split list
        uint64_t lo = 0, hi = n_split;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (split[mid].first_slot <= it.slot) lo = mid;
            else hi = mid;
        }
        const uint32_t fs = split[lo].first_slot;
        const RowStat x = part[8ull * fs + (lane & 7)];
        const uint64_t vb = 8ull * __ldg(rp + it.window);
        row_write<K, VS, VM, VO>(scores, mask, out, vb, it.vbeg, it.vend, lane, scale, x.m, x.s > 0.f ? 1.f / x.s : 0.f);
    }
}

// ---- statistics only (the AGNN aggregation applies the softmax inside the
// SpMM, spmm_f16_softmax): per row (m, 1/sum), exactly the values
// softmax_items / softmax_finish normalise with.
template <uint32_t K, typename VS>
__global__ void __launch_bounds__(256) softmax_stats_items(const WorkItem* __restrict__ items, uint64_t n_items,
                                                           uint32_t* counter, const uint32_t* __restrict__ rp,
                                                           const VS* scores, float scale, float2* __restrict__ rowstat,
                                                           RowStat* __restrict__ part) {
    const uint32_t lane = threadIdx.x & 31;
    dev::StripedClaim<8> claim;
    for (uint32_t idx; claim.get(counter, n_items, idx);) {
        const WorkItem it = items[idx];
        const uint64_t vb = 8ull * __ldg(rp + it.window);
        float m, s;
        row_stats<K, VS, void>(scores, nullptr, vb, it.vbeg, it.vend, lane, scale, m, s);
        if (lane < 8) {
            if (it.slot != kNoSlot) part[8ull * it.slot + lane] = RowStat{m, s};
            else rowstat[8ull * it.window + lane] = make_float2(m, s > 0.f ? 1.f / s : 0.f);
        }
    }
}

__global__ void softmax_stats_combine(const SplitWindow* __restrict__ split, uint64_t n_split,
                                      const RowStat* __restrict__ part, float2* __restrict__ rowstat) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 8 * n_split;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const SplitWindow sw = split[i / 8];
        const uint32_t r = static_cast<uint32_t>(i % 8);
        float m = -FLT_MAX, s = 0.f;
        for (uint32_t q = 0; q < sw.nseg; ++q) {
            const RowStat x = part[8ull * (sw.first_slot + q) + r];
            merge(m, s, x.m, x.s);
        }
        rowstat[8ull * sw.window + r] = make_float2(m, s > 0.f ? 1.f / s : 0.f);
    }
}

// scores sv (structure of sc), mask values mv (nullptr with VM = void), out
// may alias sv.
template <uint32_t K, typename VS, typename VM, typename VO>
void run(const tcs_mebcrs* sc, const VS* sv, const VM* mv, VO* out, float scale, const Plan* plan, cudaStream_t s) {
    DBuf ctr(dev::kClaimBytes, s), part(std::max<uint64_t>(1, plan->n_slots) * 8 * sizeof(RowStat), s);
    TCS_CUDA(cudaMemsetAsync(ctr.p, 0, dev::kClaimBytes, s));
    const int grid = static_cast<int>(std::min<uint64_t>((plan->n_items + 7) / 8, uint64_t(num_sms()) * 8));
    softmax_items<K, VS, VM, VO><<<std::max(grid, 1), 256, 0, s>>>(plan->items, plan->n_items, ctr.as<uint32_t>(),
                                                                   sc->row_pointers, sv, mv, out, scale,
                                                                   part.as<RowStat>());
    TCS_LAUNCHED("softmax_items");
    if (plan->n_split) {
        softmax_combine<<<static_cast<int>(std::min<uint64_t>((8 * plan->n_split + 255) / 256, 1024)), 256, 0, s>>>(
            plan->split, plan->n_split, part.as<RowStat>());
        TCS_LAUNCHED("softmax_combine");
        const int g3 = static_cast<int>(std::min<uint64_t>((plan->n_slots + 7) / 8, uint64_t(num_sms()) * 8));
        softmax_finish<K, VS, VM, VO><<<std::max(g3, 1), 256, 0, s>>>(plan->items, plan->n_slots, plan->split,
                                                                      plan->n_split, sc->row_pointers, sv, mv, out,
                                                                      scale, part.as<RowStat>());
        TCS_LAUNCHED("softmax_finish");
    }
}

template <uint32_t K, typename VS, typename VM>
void run_o(const tcs_mebcrs* sc, const tcs_mebcrs* mk, void* out, tcs_dtype odt, float scale, const Plan* plan,
           cudaStream_t s) {
    const VS* sv = static_cast<const VS*>(sc->values);
    const VM* mv = static_cast<const VM*>(mk->values);
    if (odt == TCS_DTYPE_F32) run<K, VS, VM, float>(sc, sv, mv, static_cast<float*>(out), scale, plan, s);
    else run<K, VS, VM, __half>(sc, sv, mv, static_cast<__half*>(out), scale, plan, s);
}

template <uint32_t K>
void run_k(const tcs_mebcrs* sc, const tcs_mebcrs* mk, void* out, tcs_dtype odt, float scale, const Plan* plan,
           cudaStream_t s) {
    const bool s32 = sc->value_dtype == TCS_DTYPE_F32, m32 = mk->value_dtype == TCS_DTYPE_F32;
    if (s32 && m32) run_o<K, float, float>(sc, mk, out, odt, scale, plan, s);
    else if (s32) run_o<K, float, __half>(sc, mk, out, odt, scale, plan, s);
    else if (m32) run_o<K, __half, float>(sc, mk, out, odt, scale, plan, s);
    else run_o<K, __half, __half>(sc, mk, out, odt, scale, plan, s);
}

// Fused SDDMM -> row softmax: the scores come with dead slots = -inf, so
// the softmax passes read no mask (VM = void).
template <uint32_t K, typename VX>
void run_fused(const tcs_mebcrs* m, const void* x, void* out, tcs_dtype odt, float scale, const Plan* plan,
               cudaStream_t s) {
    const VX* xv = static_cast<const VX*>(x);
    if (odt == TCS_DTYPE_F32) run<K, VX, void, float>(m, xv, nullptr, static_cast<float*>(out), scale, plan, s);
    else run<K, VX, void, __half>(m, xv, nullptr, static_cast<__half*>(out), scale, plan, s);
}

}  // namespace

void softmax_rowstats(const tcs_mebcrs* S, const Plan* plan, float scale, float2* rowstat, cudaStream_t s) {
    if (!plan->n_items) return;
    DBuf ctr(dev::kClaimBytes, s), part(std::max<uint64_t>(1, plan->n_slots) * 8 * sizeof(RowStat), s);
    TCS_CUDA(cudaMemsetAsync(ctr.p, 0, dev::kClaimBytes, s));
    const int grid = static_cast<int>(std::min<uint64_t>((plan->n_items + 7) / 8, uint64_t(num_sms()) * 8));
    const __half* sv = static_cast<const __half*>(S->values);
    softmax_stats_items<8, __half><<<std::max(grid, 1), 256, 0, s>>>(plan->items, plan->n_items, ctr.as<uint32_t>(),
                                                                      S->row_pointers, sv, scale, rowstat,
                                                                      part.as<RowStat>());
    TCS_LAUNCHED("softmax_stats_items");
    if (plan->n_split) {
        softmax_stats_combine<<<static_cast<int>(std::min<uint64_t>((8 * plan->n_split + 255) / 256, 1024)), 256, 0,
                                s>>>(plan->split, plan->n_split, part.as<RowStat>(), rowstat);
        TCS_LAUNCHED("softmax_stats_combine");
    }
}

}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_mebcrs_row_softmax(const tcs_mebcrs* scores, const tcs_mebcrs* mask, float scale,
                                             tcs_mebcrs* out, tcs_dtype out_dtype, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_mebcrs_row_softmax");
        if (!out) fail(TCS_ERR_ARGUMENT, "null output");
        check_mebcrs(scores);
        check_mebcrs(mask);
        if (scores->rows != mask->rows || scores->cols != mask->cols || scores->num_vectors != mask->num_vectors ||
            scores->k != mask->k)
            fail(TCS_ERR_SHAPE, "scores and mask must share one ME-BCRS structure");
        if (out_dtype != TCS_DTYPE_F16 && out_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown output dtype");
        if (scores->precision == TCS_TF32 && out_dtype != TCS_DTYPE_F32)
            fail(TCS_ERR_ARGUMENT, "TF32 ME-BCRS values must be stored as f32");
        cudaStream_t s = st(stream);
        void* caller_values = out->values;
        tcs_mebcrs o = *scores;
        o.flags = o.plan ? TCS_MEBCRS_BORROWED_PLAN : 0u;  // structure and work list shared
        o.value_dtype = out_dtype;
        const size_t ow = out_dtype == TCS_DTYPE_F16 ? 2 : 4;
        if (caller_values) {
            o.values = caller_values;
        } else {
            o.values = dalloc(std::max<uint64_t>(1, 8 * scores->num_vectors) * ow, s);
            o.flags |= TCS_MEBCRS_OWN_VALUES;
        }
        if (scores->num_vectors && scores->num_windows) {
            const Plan* plan = static_cast<const Plan*>(scores->plan ? scores->plan : mask->plan);
            Plan* tmp = nullptr;
            if (!plan) plan = tmp = build_plan(scores, s, nullptr, nullptr, nullptr);
            struct G {
                Plan* p;
                cudaStream_t s;
                ~G() { free_plan(p, s); }
            } g{tmp, s};
            if (scores->k == 8) run_k<8>(scores, mask, o.values, out_dtype, scale, plan, s);
            else run_k<4>(scores, mask, o.values, out_dtype, scale, plan, s);
        }
        *out = o;
    });
}

extern "C" tcs_status tcs_sddmm_row_softmax(const tcs_mebcrs* mask, const void* a, tcs_dtype a_dtype, int64_t lda,
                                            int64_t a_rows, int64_t f_a, const void* bt, tcs_dtype bt_dtype,
                                            int64_t ldbt, int64_t bt_rows, int64_t f_b, float scale,
                                            tcs_dtype score_dtype, tcs_mebcrs* out, tcs_dtype out_dtype,
                                            const tcs_kernel_config* cfg, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_sddmm_row_softmax");
        if (!out) fail(TCS_ERR_ARGUMENT, "null output");
        sddmm_check(mask, a, a_dtype, lda, a_rows, f_a, bt, bt_dtype, ldbt, bt_rows, f_b, score_dtype, cfg);
        if (out_dtype != TCS_DTYPE_F16 && out_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown output dtype");
        if (mask->precision == TCS_TF32 && out_dtype != TCS_DTYPE_F32)
            fail(TCS_ERR_ARGUMENT, "TF32 ME-BCRS values must be stored as f32");
        cudaStream_t s = st(stream);
        const uint64_t nv = mask->num_vectors;
        void* caller_values = out->values;
        tcs_mebcrs o = *mask;
        o.flags = o.plan ? TCS_MEBCRS_BORROWED_PLAN : 0u;
        o.value_dtype = out_dtype;
        const size_t ow = out_dtype == TCS_DTYPE_F16 ? 2 : 4, xw = score_dtype == TCS_DTYPE_F16 ? 2 : 4;
        if (caller_values) {
            o.values = caller_values;
        } else {
            o.values = dalloc(std::max<uint64_t>(1, 8 * nv) * ow, s);
            o.flags |= TCS_MEBCRS_OWN_VALUES;
        }
        if (nv) {
            Plan* plan = static_cast<Plan*>(mask->plan);
            Plan* tmp_plan = nullptr;
            if (!plan) plan = tmp_plan = build_plan(mask, s, nullptr, nullptr, nullptr);
            struct PlanGuard {
                Plan* p;
                cudaStream_t s;
                ~PlanGuard() { free_plan(p, s); }
            } pg{tmp_plan, s};
            // the scores go to the output buffer when the dtypes agree (normalised in place)
            DBuf xbuf;
            void* x = o.values;
            if (score_dtype != out_dtype) {
                xbuf = DBuf(8 * nv * xw, s);
                x = xbuf.p;
            }
            sddmm_launch(mask, plan, a, a_dtype, lda, a_rows, bt, bt_dtype, ldbt, bt_rows, f_a, x, score_dtype,
                         -INFINITY, (cfg->flags & TCS_CFG_STATIC_MASK) && !tmp_plan, s);
            if (plan->n_items) {
                if (mask->k == 4) run_fused<4, float>(mask, x, o.values, out_dtype, scale, plan, s);
                else if (score_dtype == TCS_DTYPE_F32) run_fused<8, float>(mask, x, o.values, out_dtype, scale, plan, s);
                else run_fused<8, __half>(mask, x, o.values, out_dtype, scale, plan, s);
            }
        }
        *out = o;
    });
}

// AGNN aggregation (no reference counterpart):
//   C = row_softmax(scale * (Hn Hn^T) restricted to the mask's live slots) . Hc
// = tcs_sddmm_row_softmax(mask, Hn, Hn, scale, binary16 scores and P) then
// tcs_spmm(P, Hc), bit for bit, without materialising P: the SDDMM writes
// binary16 scores with dead slots -inf, a statistics pass computes each row's
// (max, 1/sum), and the SpMM applies the softmax to each sparse value in
// registers.
extern "C" tcs_status tcs_agnn_aggregate(const tcs_mebcrs* mask, const void* hn, tcs_dtype hn_dtype, int64_t ldhn,
                                         int64_t row0, int64_t rows, int64_t f, float scale, const void* hc,
                                         tcs_dtype hc_dtype, int64_t ldhc, int64_t n, float* c, int64_t ldc,
                                         const tcs_kernel_config* cfg, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_agnn_aggregate");
        if (row0 < 0 || !mask || row0 + static_cast<int64_t>(mask->rows) > static_cast<int64_t>(mask->cols))
            fail(TCS_ERR_SHAPE, "AGNN attention: mask rows [row0, row0 + rows) must be nodes of its columns");
        // the mask's row i is node row0 + i: A = Hn[row0 .. row0 + rows), Bt = Hn (all nodes)
        const size_t hw = hn_dtype == TCS_DTYPE_F16 ? 2 : 4;
        const void* hrows = static_cast<const char*>(hn) + static_cast<size_t>(row0) * ldhn * hw;
        sddmm_check(mask, hrows, hn_dtype, ldhn, rows, f, hn, hn_dtype, ldhn, static_cast<int64_t>(mask->cols), f,
                    TCS_DTYPE_F16, cfg);
        if (mask->precision != TCS_FP16) fail(TCS_ERR_ARGUMENT, "the fused AGNN aggregation runs in FP16");
        if (n < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        if (hc_dtype != TCS_DTYPE_F16 && hc_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown dtype");
        if (n > 0 && rows > 0 && (!hc || ldhc < n || !c || ldc < n)) fail(TCS_ERR_ARGUMENT, "bad dense buffer");
        cudaStream_t s = st(stream);
        const uint64_t nv = mask->num_vectors;
        if (n == 0 || rows == 0) return;
        if (!nv) {
            TCS_CUDA(cudaMemset2DAsync(c, ldc * 4, 0, n * 4, rows, s));
            return;
        }
        Plan* plan = static_cast<Plan*>(mask->plan);
        Plan* tmp_plan = nullptr;
        if (!plan) plan = tmp_plan = build_plan(mask, s, nullptr, nullptr, nullptr);
        struct PlanGuard {
            Plan* p;
            cudaStream_t s;
            ~PlanGuard() { free_plan(p, s); }
        } pg{tmp_plan, s};
        DBuf scores(8 * nv * 2, s), rowstat(8 * mask->num_windows * sizeof(float2), s);
        sddmm_launch(mask, plan, hrows, hn_dtype, ldhn, rows, hn, hn_dtype, ldhn, static_cast<int64_t>(mask->cols), f,
                     scores.p, TCS_DTYPE_F16, -INFINITY, (cfg->flags & TCS_CFG_STATIC_MASK) && !tmp_plan, s);
        tcs_mebcrs S = *mask;
        S.values = scores.p;
        S.value_dtype = TCS_DTYPE_F16;
        softmax_rowstats(&S, plan, scale, rowstat.as<float2>(), s);
        spmm_f16_softmax(&S, plan, rowstat.as<float2>(), scale, hc, hc_dtype, ldhc, static_cast<int64_t>(mask->cols),
                         n, c, ldc, s);
    });
}
