// Dense glue of the AGNN layer (§8(f1)): the input
// features feed both the SDDMM (row-normalised, cosine attention) and the
// SpMM (as they are), each in the kernels' operand dtype.  One streaming
// pass produces both instead of four framework elementwise kernels.
#include <algorithm>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

template <typename VO>
__device__ __forceinline__ void put(VO* p, float x) {
    if constexpr (std::is_same_v<VO, float>) *p = x;
    else *p = __float2half_rn(x);
}

// One warp per row: the row is read once (coalesced), its L2 norm reduced
// with shuffles, then both outputs written.
template <typename VO>
__global__ void __launch_bounds__(256) rows_normalize_kernel(const float* __restrict__ h, int64_t rows, int64_t f,
                                                             int64_t ldh, VO* __restrict__ hn, VO* __restrict__ hc,
                                                             int64_t ldo, float eps) {
    const uint32_t lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t r = w0; r < rows; r += nw) {
        const float* row = h + r * ldh;
        float ss = 0.f;
        for (int64_t c = lane; c < f; c += 32) {
            const float x = __ldg(row + c);
            ss = fmaf(x, x, ss);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        const float inv = 1.f / fmaxf(sqrtf(ss), eps);
        for (int64_t c = lane; c < f; c += 32) {
            const float x = __ldg(row + c);  // L1 hit
            if (hn) put<VO>(hn + r * ldo + c, x * inv);
            if (hc) put<VO>(hc + r * ldo + c, x);
        }
    }
}

// Vectorised form for f % 4 == 0 and 16-byte aligned rows (the common
// case: f = 32 in the C5 AGNN layer): S lanes per row with float4 loads
// (S = f/4 rounded up to a power of two, <= 32), 32/S rows per warp, two row
// groups in flight per iteration.  Each lane writes 4 outputs at once.
template <typename VO, int S>
__global__ void __launch_bounds__(256) rows_normalize_vec(const float* __restrict__ h, int64_t rows, int64_t f,
                                                          int64_t ldh, VO* __restrict__ hn, VO* __restrict__ hc,
                                                          int64_t ldo, float eps) {
    constexpr int RPW = 32 / S;  // rows per warp per group
    const uint32_t lane = threadIdx.x & 31, sub = lane % S, rw = lane / S;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const int64_t nq = f / 4;  // float4 per row
    auto store4 = [&](VO* dst, float4 v) {
        if constexpr (std::is_same_v<VO, float>) {
            *reinterpret_cast<float4*>(dst) = v;
        } else {
            const __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
            uint2 u;
            u.x = *reinterpret_cast<const uint32_t*>(&a);
            u.y = *reinterpret_cast<const uint32_t*>(&b);
            *reinterpret_cast<uint2*>(dst) = u;
        }
    };
    for (int64_t r0 = w0 * 2 * RPW; r0 < rows; r0 += nw * 2 * RPW) {
        float ss[2] = {0.f, 0.f};
        int64_t r[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            r[k] = r0 + k * RPW + rw;
            if (r[k] < rows)
                for (int64_t c = sub; c < nq; c += S) {
                    const float4 x = __ldg(reinterpret_cast<const float4*>(h + r[k] * ldh) + c);
                    ss[k] = fmaf(x.x, x.x, fmaf(x.y, x.y, fmaf(x.z, x.z, fmaf(x.w, x.w, ss[k]))));
                }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int o = S / 2; o >= 1; o >>= 1) ss[k] += __shfl_xor_sync(0xffffffffu, ss[k], o);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (r[k] >= rows) continue;
            const float inv = 1.f / fmaxf(sqrtf(ss[k]), eps);
            for (int64_t c = sub; c < nq; c += S) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(h + r[k] * ldh) + c);  // L1 hit
                if (hn) store4(hn + r[k] * ldo + 4 * c, make_float4(x.x * inv, x.y * inv, x.z * inv, x.w * inv));
                if (hc) store4(hc + r[k] * ldo + 4 * c, x);
            }
        }
    }
}

template <typename VO>
void launch_normalize(const float* h, int64_t rows, int64_t f, int64_t ldh, VO* hn, VO* hc, int64_t ldo, float eps,
                      cudaStream_t s) {
    const bool vec = f % 4 == 0 && ldh % 4 == 0 && ldo % 4 == 0 && (reinterpret_cast<uintptr_t>(h) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(hn) & 7) == 0 && (reinterpret_cast<uintptr_t>(hc) & 7) == 0 &&
                     (std::is_same_v<VO, __half> || ((reinterpret_cast<uintptr_t>(hn) | reinterpret_cast<uintptr_t>(hc)) & 15) == 0);
    if (!vec) {
        const int grid = static_cast<int>(std::min<int64_t>((rows + 7) / 8, int64_t(num_sms()) * 16));
        rows_normalize_kernel<VO><<<grid, 256, 0, s>>>(h, rows, f, ldh, hn, hc, ldo, eps);
        TCS_LAUNCHED("rows_normalize");
        return;
    }
    const int64_t q = f / 4;
    const int sl = q <= 1 ? 1 : q <= 2 ? 2 : q <= 4 ? 4 : q <= 8 ? 8 : q <= 16 ? 16 : 32;
    const int64_t rows_per_block = 8 * 2 * (32 / sl);
    const int grid = static_cast<int>(std::min<int64_t>((rows + rows_per_block - 1) / rows_per_block,
                                                        int64_t(num_sms()) * 16));
    switch (sl) {
        case 1: rows_normalize_vec<VO, 1><<<grid, 256, 0, s>>>(h, rows, f, ldh, hn, hc, ldo, eps); break;
        case 2: rows_normalize_vec<VO, 2><<<grid, 256, 0, s>>>(h, rows, f, ldh, hn, hc, ldo, eps); break;
        case 4: rows_normalize_vec<VO, 4><<<grid, 256, 0, s>>>(h, rows, f, ldh, hn, hc, ldo, eps); break;
        case 8: rows_normalize_vec<VO, 8><<<grid, 256, 0, s>>>(h, rows, f, ldh, hn, hc, ldo, eps); break;
        case 16: rows_normalize_vec<VO, 16><<<grid, 256, 0, s>>>(h, rows, f, ldh, hn, hc, ldo, eps); break;
        default: rows_normalize_vec<VO, 32><<<grid, 256, 0, s>>>(h, rows, f, ldh, hn, hc, ldo, eps); break;
    }
    TCS_LAUNCHED("rows_normalize_vec");
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_rows_normalize(const float* h, int64_t rows, int64_t f, int64_t ldh, void* hn, void* hc,
                                         int64_t ldo, tcs_dtype out_dtype, float eps, tcs_stream_t stream) {
    return guard([&] {
        if (rows < 0 || f < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        if (out_dtype != TCS_DTYPE_F16 && out_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown output dtype");
        if (rows == 0 || f == 0 || (!hn && !hc)) return;
        if (!h || ldh < f || ldo < f) fail(TCS_ERR_ARGUMENT, "bad operand / leading dimension");
        if (out_dtype == TCS_DTYPE_F16)
            launch_normalize<__half>(h, rows, f, ldh, static_cast<__half*>(hn), static_cast<__half*>(hc), ldo, eps,
                                     st(stream));
        else
            launch_normalize<float>(h, rows, f, ldh, static_cast<float*>(hn), static_cast<float*>(hc), ldo, eps,
                                    st(stream));
    });
}
