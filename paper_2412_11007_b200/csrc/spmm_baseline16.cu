// Ablation baseline: SpMM over 16x1 vectors WITHOUT swap-and-transpose
// (ref spmm.hpp:187-257, spmm_baseline16; the paper's "16x1 TC block"
// comparison point).
//
// The sparse matrix is the 16-row-window ME-BCRS (tcs_mebcrs_encode_v with
// vector_height 16: windows of 16 rows, blocks 16 x k).  Each sparse block is
// the m=16 LEFT operand of a plain MMA and the gathered dense rows form the
// k x 8 right operand, so one instruction covers only 8 output features
// (the reference's shape.n = 8 tiles) against 16 for the swapped 8x1 path.
//
//   FP16: mma.sync.m16n8k16 (two k=8 storage blocks per instruction)
//   TF32: mma.sync.m16n8k8  (two k=4 blocks), operands RNE via cvt.rn.tf32
//
// The dense rows of a 16-vector (FP16) / 8-vector (TF32) step are gathered
// with coalesced 16-byte cp.async into a per-warp double-buffered shared
// tile (rows past the window's residue are zero-filled), and the B
// fragments are read with ldmatrix.trans (FP16) or conflict-free LDS
// (TF32) -- an equally engineered baseline, so the measured gap is the
// format/orientation, not the load path.  Work list, split-window partials
// and their segment-order reduction as in spmm.cu.
#include <algorithm>
#include <type_traits>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

using namespace dev;

constexpr int kWarps = 4;

struct B16Args {
    const WorkItem* items;
    uint64_t n_items;
    const uint32_t* rp;
    const uint32_t* ci;
    const void* vals;
    const void* B;  // feature-padded rows, 16-byte aligned
    int64_t ldb;
    float* C;
    int64_t ldc;
    uint64_t rows;
    int64_t N;
    float* partial;  // [slot][16][ldp]
    int64_t ldp;
    uint32_t* counter;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy; src_bytes 0 zero-fills the destination.
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// Sparse element (row r, window-relative vector v) of a 16-high window
// (ref mebcrs.hpp:46-56 with vector_height 16), 0 past the residue.
template <typename V>
__device__ __forceinline__ float b16_val(const V* vals, uint64_t vbase, uint32_t nvw, uint32_t k, uint32_t v,
                                         uint32_t r) {
    if (v >= nvw) return 0.f;
    const uint32_t b = v / k, j = v - b * k, width = min(k, nvw - b * k);
    const uint64_t off = vbase + 16ull * k * b + r * width + j;
    if constexpr (std::is_same<V, float>::value) return vals[off];
    else return __half2float(vals[off]);
}

// Epilogue shared by both precisions: acc[j] is the 16 x 8 tile of
// features feat0 + 8j (rows g, g+8; features 2t, 2t+1).
template <int NT>
__device__ __forceinline__ void b16_store(const B16Args& a, const WorkItem& it, int64_t feat0, uint32_t g, uint32_t t,
                                          const float (&acc)[NT][4]) {
    const bool split = it.slot != kNoSlot;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t r = g + 8 * h;
        const uint64_t row = 16ull * it.window + r;
        float* dst;
        int64_t lim;
        if (split) {
            dst = a.partial + (static_cast<uint64_t>(it.slot) * 16 + r) * a.ldp;
            lim = a.ldp;
        } else {
            if (row >= a.rows) continue;
            dst = a.C + row * a.ldc;
            lim = a.N;
        }
        const bool vec = split || ((a.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(a.C) & 7) == 0);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int64_t f = feat0 + 8 * j + 2 * t;
            if (vec && f + 2 <= lim) {
                *reinterpret_cast<float2*>(dst + f) = make_float2(acc[j][2 * h], acc[j][2 * h + 1]);
            } else {
                if (f < lim) dst[f] = acc[j][2 * h];
                if (f + 1 < lim) dst[f + 1] = acc[j][2 * h + 1];
            }
        }
    }
}

// ---------------------------------------------------------------- FP16
// Shared tile per warp and stage: 16 gathered rows x (8*NT halves + 8 pad).
template <int NT>
struct F16Tile {
    static constexpr int ROW = 8 * NT * 2 + 16;  // bytes; +16 keeps ldmatrix rows conflict-free
    static constexpr int BYTES = 16 * ROW;
};

template <int NT, bool VF32>
__global__ void __launch_bounds__(kWarps * 32, 4) spmm_b16_f16_kernel(const B16Args a) {
    using T = F16Tile<NT>;
    constexpr int CHUNKS = NT;  // 16-byte chunks per gathered row (8 halves each)
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t g = lane >> 2, t = lane & 3;
    unsigned char* tile = smem + warp * 2 * T::BYTES;
    const int64_t feat0 = static_cast<int64_t>(blockIdx.y) * 8 * NT;
    const __half* Bl = static_cast<const __half*>(a.B) + feat0;
    uint32_t* counter = a.counter + static_cast<uint64_t>(blockIdx.y) * (dev::kClaimBytes / 4);
    // ldmatrix row addresses: matrix m = lane/8 -> k rows (m&1)*8 + lane%8, features +8*(m>>1)
    const uint32_t ld_k = ((lane >> 3) & 1) * 8 + (lane & 7), ld_n = (lane >> 4) * 8;

    for (uint32_t idx = dev::next_item(counter, lane); idx < a.n_items; idx = dev::next_item(counter, lane)) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 16ull * base;
        const uint32_t vend = it.vend;

        float acc[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

        // gathers of step s into stage st: 16 rows x CHUNKS chunks over the warp
        auto issue = [&](uint32_t s, int stg) {
            const uint32_t colv = s + (lane & 15) < vend ? __ldg(ci + s + (lane & 15)) : 0u;
            const uint32_t dst0 = smem_u32(tile + stg * T::BYTES);
#pragma unroll
            for (int q = 0; q < (16 * CHUNKS + 31) / 32; ++q) {
                const int c = q * 32 + lane;
                if (16 * CHUNKS % 32 == 0 || c < 16 * CHUNKS) {
                    const int row = c / CHUNKS, ch = c % CHUNKS;
                    const uint32_t col = __shfl_sync(0xffffffffu, colv, row);
                    const bool live = s + row < vend;
                    cp16(dst0 + row * T::ROW + ch * 16, Bl + static_cast<uint64_t>(live ? col : 0) * a.ldb + ch * 8,
                         live ? 16u : 0u);
                }
            }
            cp_commit();
        };
        auto afrag = [&](uint32_t s, uint32_t (&af)[4]) {
            if (s + 16 <= vend) {  // two full-width k=8 blocks
                const uint64_t off = vbase + 8ull * 16 * (s / 8) + g * 8 + 2 * t;
                if constexpr (VF32) {
                    const float* fv = static_cast<const float*>(a.vals);
                    const uint2 x0 = ld_stream_u64(fv + off), x1 = ld_stream_u64(fv + off + 64);
                    const uint2 x2 = ld_stream_u64(fv + off + 128), x3 = ld_stream_u64(fv + off + 192);
                    af[0] = f2_to_h2(__uint_as_float(x0.x), __uint_as_float(x0.y));
                    af[1] = f2_to_h2(__uint_as_float(x1.x), __uint_as_float(x1.y));
                    af[2] = f2_to_h2(__uint_as_float(x2.x), __uint_as_float(x2.y));
                    af[3] = f2_to_h2(__uint_as_float(x3.x), __uint_as_float(x3.y));
                } else {
                    const __half* hv = static_cast<const __half*>(a.vals);
                    af[0] = ld_stream_u32(hv + off);
                    af[1] = ld_stream_u32(hv + off + 64);
                    af[2] = ld_stream_u32(hv + off + 128);
                    af[3] = ld_stream_u32(hv + off + 192);
                }
            } else {
                float e[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t v = s + 2 * t + (u & 1) + 8 * (u >> 2);
                    const uint32_t r = g + 8 * ((u >> 1) & 1);
                    e[u] = v < vend ? (VF32 ? b16_val(static_cast<const float*>(a.vals), vbase, nvw, 8, v, r)
                                            : b16_val(static_cast<const __half*>(a.vals), vbase, nvw, 8, v, r))
                                    : 0.f;
                }
                af[0] = f2_to_h2(e[0], e[1]);
                af[1] = f2_to_h2(e[2], e[3]);
                af[2] = f2_to_h2(e[4], e[5]);
                af[3] = f2_to_h2(e[6], e[7]);
            }
        };

        uint32_t s = it.vbeg;
        int stg = 0;
        if (s < vend) issue(s, 0);
        for (; s < vend; s += 16, stg ^= 1) {
            uint32_t af[4];
            afrag(s, af);
            if (s + 16 < vend) {
                issue(s + 16, stg ^ 1);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncwarp();
            const uint32_t tb = smem_u32(tile + stg * T::BYTES) + ld_k * T::ROW + ld_n * 2;
#pragma unroll
            for (int j = 0; j < NT; j += 2) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_trans(tb + j * 16, b0, b1, b2, b3);
                mma_f16_16816(acc[j], af[0], af[1], af[2], af[3], b0, b1);
                mma_f16_16816(acc[j + 1], af[0], af[1], af[2], af[3], b2, b3);
            }
            __syncwarp();  // stage stg is refilled two steps later
        }
        b16_store<NT>(a, it, feat0, g, t, acc);
    }
}

// ---------------------------------------------------------------- TF32
template <int NT>
struct Tf32Tile {
    static constexpr int ROW = 8 * NT * 4 + 32;  // bytes; +32 => lanes (g, t) hit distinct banks
    static constexpr int BYTES = 8 * ROW;
};

template <int NT>
__global__ void __launch_bounds__(kWarps * 32, 4) spmm_b16_tf32_kernel(const B16Args a) {
    using T = Tf32Tile<NT>;
    constexpr int CHUNKS = 2 * NT;  // 16-byte chunks per row (4 floats each)
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t g = lane >> 2, t = lane & 3;
    unsigned char* tile = smem + warp * 2 * T::BYTES;
    const int64_t feat0 = static_cast<int64_t>(blockIdx.y) * 8 * NT;
    const float* Bl = static_cast<const float*>(a.B) + feat0;
    const float* fv = static_cast<const float*>(a.vals);
    uint32_t* counter = a.counter + static_cast<uint64_t>(blockIdx.y) * (dev::kClaimBytes / 4);

    for (uint32_t idx = dev::next_item(counter, lane); idx < a.n_items; idx = dev::next_item(counter, lane)) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 16ull * base;
        const uint32_t vend = it.vend;

        float acc[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

        auto issue = [&](uint32_t s, int stg) {
            const uint32_t colv = s + (lane & 7) < vend ? __ldg(ci + s + (lane & 7)) : 0u;
            const uint32_t dst0 = smem_u32(tile + stg * T::BYTES);
#pragma unroll
            for (int q = 0; q < (8 * CHUNKS + 31) / 32; ++q) {
                const int c = q * 32 + lane;
                if (8 * CHUNKS % 32 == 0 || c < 8 * CHUNKS) {
                    const int row = c / CHUNKS, ch = c % CHUNKS;
                    const uint32_t col = __shfl_sync(0xffffffffu, colv, row);
                    const bool live = s + row < vend;
                    cp16(dst0 + row * T::ROW + ch * 16, Bl + static_cast<uint64_t>(live ? col : 0) * a.ldb + ch * 4,
                         live ? 16u : 0u);
                }
            }
            cp_commit();
        };

        uint32_t s = it.vbeg;
        int stg = 0;
        if (s < vend) issue(s, 0);
        for (; s < vend; s += 8, stg ^= 1) {
            uint32_t af[4];
            if (s + 8 <= vend) {  // two full k=4 blocks: (r, j) at 64 b + 4 r + j
                const uint64_t off = vbase + 64ull * (s / 4) + 4 * g + t;
                af[0] = to_tf32(__uint_as_float(ld_stream_u32(fv + off)));
                af[1] = to_tf32(__uint_as_float(ld_stream_u32(fv + off + 32)));
                af[2] = to_tf32(__uint_as_float(ld_stream_u32(fv + off + 64)));
                af[3] = to_tf32(__uint_as_float(ld_stream_u32(fv + off + 96)));
            } else {
                af[0] = to_tf32(s + t < vend ? b16_val(fv, vbase, nvw, 4, s + t, g) : 0.f);
                af[1] = to_tf32(s + t < vend ? b16_val(fv, vbase, nvw, 4, s + t, g + 8) : 0.f);
                af[2] = to_tf32(s + t + 4 < vend ? b16_val(fv, vbase, nvw, 4, s + t + 4, g) : 0.f);
                af[3] = to_tf32(s + t + 4 < vend ? b16_val(fv, vbase, nvw, 4, s + t + 4, g + 8) : 0.f);
            }
            if (s + 8 < vend) {
                issue(s + 8, stg ^ 1);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncwarp();
            const float* tb = reinterpret_cast<const float*>(tile + stg * T::BYTES);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const uint32_t b0 = to_tf32(tb[t * (T::ROW / 4) + 8 * j + g]);
                const uint32_t b1 = to_tf32(tb[(t + 4) * (T::ROW / 4) + 8 * j + g]);
                mma_tf32_1688(acc[j], af[0], af[1], af[2], af[3], b0, b1);
            }
            __syncwarp();
        }
        b16_store<NT>(a, it, feat0, g, t, acc);
    }
}

__global__ void __launch_bounds__(256) b16_reduce_split(const SplitWindow* __restrict__ split, uint64_t n_split,
                                                        const float* __restrict__ partial, int64_t ldp, float* C,
                                                        int64_t ldc, uint64_t rows, int64_t N) {
    for (uint64_t sw = blockIdx.x; sw < n_split; sw += gridDim.x) {
        const SplitWindow x = split[sw];
        for (int64_t e = threadIdx.x; e < 16 * N; e += blockDim.x) {
            const int64_t r = e / N, f = e - r * N;
            const uint64_t row = 16ull * x.window + r;
            if (row >= rows) continue;
            float acc = 0.f;
            for (uint32_t q = 0; q < x.nseg; ++q) acc += partial[((uint64_t)(x.first_slot + q) * 16 + r) * ldp + f];
            C[row * ldc + f] = acc;
        }
    }
}

template <typename K>
void launch_b16(K kernel, const B16Args& a, int slabs, size_t smem, cudaStream_t s, const char* name) {
    TCS_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const uint64_t per_slab = std::max<uint64_t>(1, uint64_t(num_sms()) * 4 / std::max(1, slabs));
    const uint64_t need = (a.n_items + kWarps - 1) / kWarps;
    const dim3 grid(static_cast<unsigned>(std::min(need, per_slab)), slabs);
    kernel<<<grid, kWarps * 32, smem, s>>>(a);
    TCS_LAUNCHED(name);
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_spmm_baseline16(const tcs_mebcrs* A, const void* b, tcs_dtype b_dtype, int64_t ldb,
                                          int64_t b_rows, int64_t n, float* c, int64_t ldc,
                                          const tcs_kernel_config* cfg, tcs_counters* counters,
                                          tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_baseline16");
        if (!cfg) fail(TCS_ERR_ARGUMENT, "null kernel config");
        // ref spmm.hpp:190-191
        if (cfg->vector_height != 16) fail(TCS_ERR_ARGUMENT, "baseline path requires vector height 16");
        check_mebcrs(A, true);
        if (A->vector_height != 16) fail(TCS_ERR_ARGUMENT, "baseline path needs a 16-row-window ME-BCRS");
        if (cfg->precision != A->precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded matrix");
        if (static_cast<int64_t>(A->cols) != b_rows) fail(TCS_ERR_SHAPE, "sparse cols must equal dense rows");
        if (n < 0 || b_rows < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        if (n > 0 && A->rows > 0 && (!c || ldc < n)) fail(TCS_ERR_ARGUMENT, "bad output buffer / ldc");
        if (n > 0 && b_rows > 0 && (!b || ldb < n)) fail(TCS_ERR_ARGUMENT, "bad dense buffer / ldb");
        if (b_dtype != TCS_DTYPE_F16 && b_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown dtype");
        if (A->precision == TCS_TF32 && b_dtype != TCS_DTYPE_F32)
            fail(TCS_ERR_ARGUMENT, "TF32 SpMM needs an f32 dense operand");
        if (counters) *counters = tcs_counters{};
        cudaStream_t s = st(stream);
        if (n == 0 || A->rows == 0) return;

        Plan* plan = static_cast<Plan*>(A->plan);
        Plan* tmp_plan = nullptr;
        if (!plan) plan = tmp_plan = build_plan(A, s, nullptr, nullptr, nullptr);
        struct PlanGuard {
            Plan* p;
            cudaStream_t s;
            ~PlanGuard() { free_plan(p, s); }
        } pg{tmp_plan, s};

        const int64_t npad = n <= 32 ? 32 : n <= 64 ? 64 : (n + 127) / 128 * 128;
        const int slab = npad <= 32 ? 32 : npad <= 64 ? 64 : 128;
        const tcs_dtype need = A->precision == TCS_FP16 ? TCS_DTYPE_F16 : TCS_DTYPE_F32;
        const int64_t align_elems = need == TCS_DTYPE_F16 ? 8 : 4;
        const bool direct = b_dtype == need && ldb % align_elems == 0 && ldb >= npad &&
                            (reinterpret_cast<uintptr_t>(b) & 15) == 0;
        DBuf bpad;
        const void* bp = b;
        int64_t bld = ldb;
        if (!direct) {
            bld = npad;
            bpad = DBuf(static_cast<size_t>(std::max<int64_t>(1, b_rows)) * npad * (need == TCS_DTYPE_F16 ? 2 : 4), s);
            pad_convert(b, b_dtype, ldb, bpad.p, need, npad, b_rows, n, npad, s);
            bp = bpad.p;
        }
        DBuf partial;
        if (plan->n_slots) partial = DBuf(plan->n_slots * 16 * npad * sizeof(float), s);
        const int slabs = static_cast<int>(npad / slab);
        DBuf ctr(slabs * dev::kClaimBytes, s);
        TCS_CUDA(cudaMemsetAsync(ctr.p, 0, slabs * dev::kClaimBytes, s));
        B16Args a{plan->items, plan->n_items, A->row_pointers, A->column_indices, A->values, bp, bld,
                  c, ldc, A->rows, n, partial.as<float>(), npad, ctr.as<uint32_t>()};
        if (plan->n_items) {
            if (A->precision == TCS_FP16) {
                const bool vf32 = A->value_dtype == TCS_DTYPE_F32;
                if (slab == 128) {
                    const size_t sm = kWarps * 2 * F16Tile<16>::BYTES;
                    vf32 ? launch_b16(spmm_b16_f16_kernel<16, true>, a, slabs, sm, s, "spmm_b16_f16<128,f32v>")
                         : launch_b16(spmm_b16_f16_kernel<16, false>, a, slabs, sm, s, "spmm_b16_f16<128>");
                } else if (slab == 64) {
                    const size_t sm = kWarps * 2 * F16Tile<8>::BYTES;
                    vf32 ? launch_b16(spmm_b16_f16_kernel<8, true>, a, slabs, sm, s, "spmm_b16_f16<64,f32v>")
                         : launch_b16(spmm_b16_f16_kernel<8, false>, a, slabs, sm, s, "spmm_b16_f16<64>");
                } else {
                    const size_t sm = kWarps * 2 * F16Tile<4>::BYTES;
                    vf32 ? launch_b16(spmm_b16_f16_kernel<4, true>, a, slabs, sm, s, "spmm_b16_f16<32,f32v>")
                         : launch_b16(spmm_b16_f16_kernel<4, false>, a, slabs, sm, s, "spmm_b16_f16<32>");
                }
            } else {
                if (slab == 128)
                    launch_b16(spmm_b16_tf32_kernel<16>, a, slabs, kWarps * 2 * Tf32Tile<16>::BYTES, s,
                               "spmm_b16_tf32<128>");
                else if (slab == 64)
                    launch_b16(spmm_b16_tf32_kernel<8>, a, slabs, kWarps * 2 * Tf32Tile<8>::BYTES, s,
                               "spmm_b16_tf32<64>");
                else
                    launch_b16(spmm_b16_tf32_kernel<4>, a, slabs, kWarps * 2 * Tf32Tile<4>::BYTES, s,
                               "spmm_b16_tf32<32>");
            }
        }
        if (plan->n_split) {
            const int grid = static_cast<int>(std::min<uint64_t>(plan->n_split, uint64_t(num_sms()) * 8));
            b16_reduce_split<<<grid, 256, 0, s>>>(plan->split, plan->n_split, partial.as<float>(), npad, c, ldc,
                                                  A->rows, n);
            TCS_LAUNCHED("b16_reduce_split");
        }
        // ref analysis.hpp:34-38 with Strategy::baseline16: blocks x ceil(N / 8)
        if (counters) counters->mma_invocations = A->num_blocks * ((n + 7) / 8);
        if (counters && (cfg->flags & TCS_CFG_COUNT_ACCESS)) {
            tcs_cost cost{};
            mebcrs_cost(A, 0, n, cfg->mapping, &cost, s);
            counters->transactions = cost.exec_transactions;
            counters->transaction_bytes = cost.exec_transaction_bytes;
            counters->useful_bytes = cost.exec_useful_bytes;
        }
    });
}

extern "C" tcs_status tcs_spmm_baseline16_csr_host(const tcs_csr* host_csr, const float* b, int64_t b_rows,
                                                   int64_t n, float* c, const tcs_kernel_config* cfg,
                                                   tcs_counters* counters, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_baseline16_csr_host");
        if (!host_csr || !cfg || !host_csr->row_ptr) fail(TCS_ERR_ARGUMENT, "null argument");
        // ref spmm.hpp:190-191, in its order
        if (cfg->vector_height != 16) fail(TCS_ERR_ARGUMENT, "baseline path requires vector height 16");
        if (static_cast<int64_t>(host_csr->cols) != b_rows) fail(TCS_ERR_SHAPE, "sparse cols must equal dense rows");
        if (n < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        cudaStream_t s = st(stream);
        const uint64_t rows = host_csr->rows, nnz = host_csr->nnz;
        DBuf rp((rows + 1) * 4, s), ci(std::max<uint64_t>(1, nnz) * 4, s), v(std::max<uint64_t>(1, nnz) * 4, s);
        TCS_CUDA(cudaMemcpyAsync(rp.p, host_csr->row_ptr, (rows + 1) * 4, cudaMemcpyHostToDevice, s));
        if (nnz) {
            TCS_CUDA(cudaMemcpyAsync(ci.p, host_csr->col_idx, nnz * 4, cudaMemcpyHostToDevice, s));
            TCS_CUDA(cudaMemcpyAsync(v.p, host_csr->values, nnz * 4, cudaMemcpyHostToDevice, s));
        }
        const tcs_csr d{rows, host_csr->cols, nnz, rp.as<uint32_t>(), ci.as<uint32_t>(), v.as<float>()};
        tcs_mebcrs m{};
        tcs_status rc = tcs_mebcrs_encode_v(&d, cfg->precision, TCS_DTYPE_F32, 16, &m, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        struct Free {
            tcs_mebcrs* m;
            tcs_stream_t s;
            ~Free() { tcs_mebcrs_free(m, s); }
        } fr{&m, stream};
        DBuf db(std::max<int64_t>(1, b_rows * n) * 4, s), dc(std::max<uint64_t>(1, rows * n) * 4, s);
        if (b_rows > 0 && n > 0) TCS_CUDA(cudaMemcpyAsync(db.p, b, b_rows * n * 4, cudaMemcpyHostToDevice, s));
        rc = tcs_spmm_baseline16(&m, db.p, TCS_DTYPE_F32, std::max<int64_t>(1, n), b_rows, n, dc.as<float>(),
                                 std::max<int64_t>(1, n), cfg, counters, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        if (rows > 0 && n > 0) TCS_CUDA(cudaMemcpyAsync(c, dc.p, rows * n * 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
    });
}
