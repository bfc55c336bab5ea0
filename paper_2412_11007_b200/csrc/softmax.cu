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
// One warp per window (grid-stride): lane handles vectors v = lane + 32i;
// for each vector the 8 rows are visited in a static loop, so the per-row
// running max / sum stay in registers; three passes (max, sum, write) over
// the window's contiguous value region, warp-reduced per row.
#include <algorithm>
#include <cfloat>

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

template <uint32_t K, typename VS, typename VM, typename VO>
__global__ void __launch_bounds__(256) row_softmax_kernel(const uint32_t* __restrict__ rp, uint64_t W,
                                                          const VS* __restrict__ scores, const VM* __restrict__ mask,
                                                          VO* __restrict__ out, float scale) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    for (uint64_t w = warp0; w < W; w += nwarps) {
        const uint32_t base = rp[w], nvw = rp[w + 1] - base;
        if (nvw == 0) continue;
        const uint64_t vb = 8ull * base;
        auto pos = [&](uint32_t v, uint32_t r) -> uint64_t {
            const uint32_t b = v / K, width = min(K, nvw - b * K);
            return vb + 8ull * K * b + r * width + (v - b * K);
        };
        float mx[8], sm[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            mx[r] = -FLT_MAX;
            sm[r] = 0.f;
        }
        for (uint32_t v = lane; v < nvw; v += 32)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint64_t p = pos(v, r);
                if (live_at<VM>(mask, p)) mx[r] = fmaxf(mx[r], scale * ld_val<VS>(scores, p));
            }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int o = 16; o; o >>= 1) mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], o));
        for (uint32_t v = lane; v < nvw; v += 32)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint64_t p = pos(v, r);
                if (live_at<VM>(mask, p)) sm[r] += expf(scale * ld_val<VS>(scores, p) - mx[r]);
            }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int o = 16; o; o >>= 1) sm[r] += __shfl_xor_sync(0xffffffffu, sm[r], o);
            sm[r] = sm[r] > 0.f ? 1.f / sm[r] : 0.f;
        }
        for (uint32_t v = lane; v < nvw; v += 32)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint64_t p = pos(v, r);
                const float y = live_at<VM>(mask, p) ? expf(scale * ld_val<VS>(scores, p) - mx[r]) * sm[r] : 0.f;
                st_val<VO>(out, p, y);
            }
    }
}

template <uint32_t K, typename VS, typename VM>
void launch_out(const tcs_mebcrs* sc, const tcs_mebcrs* mk, void* out, tcs_dtype odt, float scale, cudaStream_t s) {
    const uint64_t W = sc->num_windows;
    const int grid = static_cast<int>(std::min<uint64_t>((W + 7) / 8, uint64_t(num_sms()) * 8));
    if (odt == TCS_DTYPE_F32)
        row_softmax_kernel<K, VS, VM, float><<<grid, 256, 0, s>>>(sc->row_pointers, W, static_cast<const VS*>(sc->values),
                                                                  static_cast<const VM*>(mk->values),
                                                                  static_cast<float*>(out), scale);
    else
        row_softmax_kernel<K, VS, VM, __half><<<grid, 256, 0, s>>>(sc->row_pointers, W,
                                                                   static_cast<const VS*>(sc->values),
                                                                   static_cast<const VM*>(mk->values),
                                                                   static_cast<__half*>(out), scale);
    TCS_LAUNCHED("row_softmax");
}

template <uint32_t K>
void launch_k(const tcs_mebcrs* sc, const tcs_mebcrs* mk, void* out, tcs_dtype odt, float scale, cudaStream_t s) {
    const bool s32 = sc->value_dtype == TCS_DTYPE_F32, m32 = mk->value_dtype == TCS_DTYPE_F32;
    if (s32 && m32) launch_out<K, float, float>(sc, mk, out, odt, scale, s);
    else if (s32) launch_out<K, float, __half>(sc, mk, out, odt, scale, s);
    else if (m32) launch_out<K, __half, float>(sc, mk, out, odt, scale, s);
    else launch_out<K, __half, __half>(sc, mk, out, odt, scale, s);
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_mebcrs_row_softmax(const tcs_mebcrs* scores, const tcs_mebcrs* mask, float scale,
                                             tcs_mebcrs* out, tcs_dtype out_dtype, tcs_stream_t stream) {
    return guard([&] {
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
            if (scores->k == 8) launch_k<8>(scores, mask, o.values, out_dtype, scale, s);
            else launch_k<4>(scores, mask, o.values, out_dtype, scale, s);
        }
        *out = o;
    });
}
