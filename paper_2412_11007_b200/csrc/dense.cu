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
        const int grid = static_cast<int>(std::min<int64_t>((rows + 7) / 8, int64_t(num_sms()) * 16));
        if (out_dtype == TCS_DTYPE_F16)
            rows_normalize_kernel<__half><<<grid, 256, 0, st(stream)>>>(h, rows, f, ldh, static_cast<__half*>(hn),
                                                                       static_cast<__half*>(hc), ldo, eps);
        else
            rows_normalize_kernel<float><<<grid, 256, 0, st(stream)>>>(h, rows, f, ldh, static_cast<float*>(hn),
                                                                      static_cast<float*>(hc), ldo, eps);
        TCS_LAUNCHED("rows_normalize");
    });
}
