// SpMM, FP16, Blackwell-native path: TMA gather4 -> SMEM -> tcgen05.mma ->
// TMEM -> registers -> C.  Same math as spmm.cu (swap-and-transpose,
// ref spmm.hpp:103-177): per 16-vector step of a window,
//
//   D[features x 8 rows] += A[features x 16 vectors] * S[16 vectors x 8 rows]
//
//   A: the 16 gathered dense rows, fetched by cp.async.bulk.tensor...gather4
//      (4 rows per instruction, box {64 features, 1 row}, 128-B swizzle)
//      straight from L2 into shared memory -- the gathers never touch the
//      L1/LSU data pipe that bounds the mma.sync kernel (ncu: one wavefront
//      per 32-B sector of L2-sourced LDG data).  MN-major SW128 operand.
//      Vectors past the window's nv_w get an out-of-range row index, which
//      TMA zero-fills (the reference's residue rule, ref spmm.hpp:40-45).
//   S: the two ME-BCRS k=8 blocks of the step, 256 contiguous bytes of the
//      value array = a K-major, no-swizzle UMMA operand (8 rows x 16 B core
//      matrices, LBO = 128 B); copied with one cp.async.bulk.  A narrow last
//      block (width < 8) is re-laid out with zero fill by the producer warp.
//   D: tcgen05.mma.cta_group::1.kind::f16, M = 64 features per instruction
//      (N = 8 needs M = 64), H instructions per step for 64*H features;
//      fp32 accumulators in TMEM, double buffered across work items.
//
// Warp roles (persistent CTA, one per SM): warp 0 = TMA producer, warp 1 =
// MMA issuer (one elected lane) + TMEM owner, warps 2-5 = epilogue
// (tcgen05.ld 32x32b, one TMEM sub-partition each).  smem ring of STAGES
// {A, S} stages with full/empty mbarriers; TMEM ring of 2 accumulators with
// full/empty mbarriers.  Layouts were validated on a B200 by
// tools/probe_tc05.cu.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

using namespace dev;

struct Tc05Args {
    const WorkItem* items;
    uint64_t n_items;
    const uint32_t* rp;
    const uint32_t* ci;
    const __half* vals;
    float* C;
    int64_t ldc;
    uint64_t rows;
    int64_t N;
    float* partial;
    int64_t ldp;
    uint32_t k_rows;  // rows of B (= sparse cols); row index k_rows is out of range -> zero fill
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t r0,
                                            int32_t r1, int32_t r2, int32_t r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// SMEM matrix descriptors (sm_100 UMMA format: start>>4 [0,14), LBO>>4
// [16,30), SBO>>4 [32,46), version 1 [46,48), layout [61,64)).
__device__ __forceinline__ uint64_t desc_a_mn_sw128(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_b_k_interleave(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           (1ull << 46);
}
// kind::f16 instruction descriptor: F32 accumulate, F16 A/B, A MN-major,
// B K-major, N = 8, M = 64.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 15) | ((8u >> 3) << 17) | ((64u >> 4) << 24);

template <int H>
struct Tc05Cfg {
    static constexpr int STAGES = H == 1 ? 48 : H == 2 ? 32 : 16;
    static constexpr int A_STAGE = H * 2048;  // H halves x 16 rows x 128 B
    static constexpr int S_STAGE = 256;
    static constexpr int TMEM_COLS = 16 * H <= 32 ? 32 : 64;  // 2 accumulators x 8H columns
    static constexpr size_t SMEM = 1024 + (size_t)STAGES * (A_STAGE + S_STAGE) + 1024;
};

constexpr int kThreads = 192;

template <int H>
__global__ void __launch_bounds__(kThreads, 1) spmm_tc05_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                  const Tc05Args a) {
    using Cfg = Tc05Cfg<H>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;                                 // STAGES x A_STAGE (1024-aligned)
    uint8_t* sS = base + (size_t)STAGES * Cfg::A_STAGE; // STAGES x 256
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base_sh;

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(Cfg::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_sh;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer warp
        uint32_t stage = 0, phase = 0;
        for (uint64_t idx = blockIdx.x; idx < a.n_items; idx += gridDim.x) {
            const WorkItem it = a.items[idx];
            const uint32_t base_v = __ldg(a.rp + it.window);
            const uint32_t nvw = __ldg(a.rp + it.window + 1) - base_v;
            const uint32_t* ci = a.ci + base_v;
            const __half* vals = a.vals + 8ull * base_v;
            const uint32_t vend = it.vend;
            // residue tile of the item's last step (narrow block or < 16 vectors)
            const uint32_t last = it.vbeg + ((vend - it.vbeg + 15) / 16 - 1) * 16;
            const bool partial_last = vend > it.vbeg && last + 16 > vend;
            __half res[4];
            if (partial_last) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t e = 4 * lane + q;  // tile element: kb*64 + r*8 + j
                    const uint32_t kb = e >> 6, r = (e >> 3) & 7, j = e & 7;
                    const uint32_t v = last + 8 * kb + j;
                    __half x = __float2half(0.f);
                    if (v < vend) {
                        const uint32_t b = v >> 3, width = min(8u, nvw - 8 * b);
                        x = vals[64ull * b + r * width + j];
                    }
                    res[q] = x;
                }
            }
            for (uint32_t c0 = it.vbeg; c0 < vend; c0 += 256) {
                uint32_t col[8];  // lane l: vectors c0 + l + 32 j
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t v = c0 + lane + 32 * j;
                    col[j] = v < vend ? __ldg(ci + v) : a.k_rows;
                }
#pragma unroll
                for (int st = 0; st < 16; ++st) {
                    const uint32_t s = c0 + 16 * st;
                    if (s >= vend) break;
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* dA = sA + (size_t)stage * Cfg::A_STAGE;
                    uint8_t* dS = sS + (size_t)stage * Cfg::S_STAGE;
                    const bool full_step = s + 16 <= vend;
                    if (!full_step) {
                        uint2 w;
                        w.x = (uint32_t)__half_as_ushort(res[0]) | ((uint32_t)__half_as_ushort(res[1]) << 16);
                        w.y = (uint32_t)__half_as_ushort(res[2]) | ((uint32_t)__half_as_ushort(res[3]) << 16);
                        *reinterpret_cast<uint2*>(dS + 8 * lane) = w;
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    __syncwarp();
                    // columns of this step: lanes (st&1)*16 + u, register st/2
                    const uint32_t mine = col[st >> 1];
                    const uint32_t srcl = ((st & 1) << 4) + 4 * (lane & 3);
                    const uint32_t r0 = __shfl_sync(0xffffffffu, mine, srcl + 0);
                    const uint32_t r1 = __shfl_sync(0xffffffffu, mine, srcl + 1);
                    const uint32_t r2 = __shfl_sync(0xffffffffu, mine, srcl + 2);
                    const uint32_t r3 = __shfl_sync(0xffffffffu, mine, srcl + 3);
                    if (lane == 0) mbar_expect_tx(&full[stage], H * 2048 + (full_step ? 256 : 0));
                    __syncwarp();
                    if (lane < 4) {
#pragma unroll
                        for (int h = 0; h < H; ++h)
                            tma_gather4(dA + h * 2048 + lane * 512, &tmap, &full[stage], 64 * h, (int32_t)r0,
                                        (int32_t)r1, (int32_t)r2, (int32_t)r3);
                    }
                    if (full_step && lane == 4) bulk_copy(dS, vals + 8ull * s, 256, &full[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------- MMA issuer warp
        uint32_t stage = 0, phase = 0, ab = 0, aphase = 0;
        for (uint64_t idx = blockIdx.x; idx < a.n_items; idx += gridDim.x) {
            const WorkItem it = a.items[idx];
            const uint32_t nsteps = (it.vend - it.vbeg + 15) / 16;
            mbar_wait(&acc_empty[ab], aphase ^ 1);
            tc_fence_after();
            const uint32_t d0 = tbase + ab * (8 * H);
            for (uint32_t stp = 0; stp < nsteps; ++stp) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t aaddr = smem_u32(sA + (size_t)stage * Cfg::A_STAGE);
                    const uint64_t bdesc = desc_b_k_interleave(smem_u32(sS + (size_t)stage * Cfg::S_STAGE));
#pragma unroll
                    for (int h = 0; h < H; ++h)
                        tc_mma_f16(d0 + 8 * h, desc_a_mn_sw128(aaddr + h * 2048), bdesc, kIdesc, stp > 0 ? 1u : 0u);
                    tc_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) {
                if (nsteps) tc_commit(&acc_full[ab]);
                else mbar_arrive(&acc_full[ab]);
            }
            __syncwarp();
            if (++ab == 2) {
                ab = 0;
                aphase ^= 1;
            }
        }
    } else {
        // -------------------------------------------------- epilogue warps
        const uint32_t q = warp & 3;  // TMEM sub-partition this warp may access
        uint32_t ab = 0, aphase = 0;
        for (uint64_t idx = blockIdx.x; idx < a.n_items; idx += gridDim.x) {
            const WorkItem it = a.items[idx];
            const bool any = it.vend > it.vbeg;
            mbar_wait(&acc_full[ab], aphase);
            tc_fence_after();
            uint32_t r[8 * H];
            if (any) {
                const uint32_t taddr = tbase + ((32 * q) << 16) + ab * (8 * H);
                if constexpr (H == 1) {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                                   "=r"(r[7])
                                 : "r"(taddr));
                } else {
#pragma unroll
                    for (int g = 0; g < H / 2; ++g)
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%"
                            "14,%15}, [%16];"
                            : "=r"(r[16 * g + 0]), "=r"(r[16 * g + 1]), "=r"(r[16 * g + 2]), "=r"(r[16 * g + 3]),
                              "=r"(r[16 * g + 4]), "=r"(r[16 * g + 5]), "=r"(r[16 * g + 6]), "=r"(r[16 * g + 7]),
                              "=r"(r[16 * g + 8]), "=r"(r[16 * g + 9]), "=r"(r[16 * g + 10]), "=r"(r[16 * g + 11]),
                              "=r"(r[16 * g + 12]), "=r"(r[16 * g + 13]), "=r"(r[16 * g + 14]), "=r"(r[16 * g + 15])
                            : "r"(taddr + 16 * g));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            } else {
#pragma unroll
                for (int i = 0; i < 8 * H; ++i) r[i] = 0u;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            if (++ab == 2) {
                ab = 0;
                aphase ^= 1;
            }
            // lane t < 16 holds feature row m = 16q + t of every 64-feature half
            if (lane < 16) {
                const uint32_t m = 16 * q + lane;
                const bool split = it.slot != kNoSlot;
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    const uint64_t row = 8ull * it.window + n;
                    float* dst;
                    int64_t lim;
                    if (split) {
                        dst = a.partial + (static_cast<uint64_t>(it.slot) * 8 + n) * a.ldp;
                        lim = a.ldp;
                    } else {
                        if (row >= a.rows) continue;
                        dst = a.C + row * a.ldc;
                        lim = a.N;
                    }
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        const int64_t f = 64 * h + m;
                        if (f < lim) dst[f] = __uint_as_float(r[8 * h + n]);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(Cfg::TMEM_COLS));
    }
}

// ------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

template <int H>
void launch_h(const CUtensorMap& map, const Tc05Args& a, cudaStream_t s) {
    using Cfg = Tc05Cfg<H>;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(spmm_tc05_kernel<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    });
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(a.n_items, (uint64_t)num_sms()));
    spmm_tc05_kernel<H><<<grid, kThreads, Cfg::SMEM, s>>>(map, a);
    TCS_LAUNCHED("spmm_tc05");
}

}  // namespace

// Returns false (nothing launched) when the operands do not fit this path.
bool spmm_tc05(const tcs_mebcrs* A, const Plan* plan, const __half* B, int64_t ldb, int64_t b_rows, int64_t n,
               float* c, int64_t ldc, float* partial, int64_t ldp, cudaStream_t s) {
    if (A->precision != TCS_FP16 || A->value_dtype != TCS_DTYPE_F16) return false;
    if (n <= 0 || n > 256 || (ldb % 8) != 0 || (reinterpret_cast<uintptr_t>(B) & 15) != 0) return false;
    if (b_rows <= 0 || b_rows >= (int64_t(1) << 31) - 1 || ldb < n) return false;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const int H = n <= 64 ? 1 : n <= 128 ? 2 : 4;
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)b_rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ldb * 2};
    const cuuint32_t box[2] = {64, 1};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(B), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    Tc05Args a{plan->items, plan->n_items, A->row_pointers, A->column_indices,
               static_cast<const __half*>(A->values), c, ldc, A->rows, n, partial, ldp,
               static_cast<uint32_t>(b_rows)};
    if (plan->n_items == 0) return true;
    if (H == 1) launch_h<1>(map, a, s);
    else if (H == 2) launch_h<2>(map, a, s);
    else launch_h<4>(map, a, s);
    return true;
}

}  // namespace tcs
