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
// Warp roles (persistent CTA, one per SM): warps 0-7 = TMA producers
// (steps dealt round-robin), warp 8 = MMA issuer (one elected lane) + TMEM
// owner, warps 9-12 = epilogue
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

// One accumulator tile (8H columns) of this warp's TMEM sub-partition.
template <int H>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[8 * H]) {
    if constexpr (H == 1) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else {
#pragma unroll
        for (int g = 0; g < H / 2; ++g)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(r[16 * g + 0]), "=r"(r[16 * g + 1]), "=r"(r[16 * g + 2]), "=r"(r[16 * g + 3]),
                  "=r"(r[16 * g + 4]), "=r"(r[16 * g + 5]), "=r"(r[16 * g + 6]), "=r"(r[16 * g + 7]),
                  "=r"(r[16 * g + 8]), "=r"(r[16 * g + 9]), "=r"(r[16 * g + 10]), "=r"(r[16 * g + 11]),
                  "=r"(r[16 * g + 12]), "=r"(r[16 * g + 13]), "=r"(r[16 * g + 14]), "=r"(r[16 * g + 15])
                : "r"(taddr + 16 * g));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Position in a CTA's step sequence: its work items blockIdx.x + i*gridDim.x
// in order, 16-vector steps each (items without vectors have no steps).
struct StepCursor {
    uint64_t idx;
    WorkItem it;
    uint32_t s, base_v, nvw;
    __device__ __forceinline__ bool load_item(const Tc05Args& a) {
        for (; idx < a.n_items; idx += gridDim.x) {
            it = a.items[idx];
            if (it.vend > it.vbeg) {
                base_v = __ldg(a.rp + it.window);
                nvw = __ldg(a.rp + it.window + 1) - base_v;
                s = it.vbeg;
                return true;
            }
        }
        return false;
    }
    __device__ __forceinline__ bool start(const Tc05Args& a) {
        idx = blockIdx.x;
        return load_item(a);
    }
    __device__ __forceinline__ bool advance(const Tc05Args& a) {
        s += 16;
        if (s < it.vend) return true;
        idx += gridDim.x;
        return load_item(a);
    }
    // lane j < 16: column index of vector s + j (row k_rows -> TMA zero fill past the item)
    __device__ __forceinline__ uint32_t cols(const Tc05Args& a, uint32_t lane) const {
        return lane < 16 && s + lane < it.vend ? __ldg(a.ci + base_v + s + lane) : a.k_rows;
    }
};

// Independent TMEM accumulators per work item: consecutive steps rotate
// over them.  One M=64, N=8, K=16 MMA into the same accumulator as its
// predecessor waits for it (~190 cycles per step measured with a single
// accumulator, which bound the kernel at one step per ~380 cycles per SM);
// kAcc chains overlap, and the epilogue adds the partial tiles in a fixed
// order (acc0 + acc1 + acc2 + acc3: deterministic).
constexpr int kAcc = 4;

template <int H>
struct Tc05Cfg {
    static constexpr int STAGES = H == 1 ? 48 : H == 2 ? 32 : 16;
    static constexpr int A_STAGE = H * 2048;  // H halves x 16 rows x 128 B
    static constexpr int S_STAGE = 256;
    // 2 items in flight x kAcc accumulators x 8H columns
    static constexpr int TMEM_COLS = 2 * kAcc * 8 * H <= 32 ? 32 : 2 * kAcc * 8 * H <= 64 ? 64
                                   : 2 * kAcc * 8 * H <= 128 ? 128 : 256;
    static constexpr size_t SMEM = 1024 + (size_t)STAGES * (A_STAGE + S_STAGE) + 1024;
};

constexpr int kProducers = 8;                 // TMA producer warps
constexpr int kThreads = 32 * (kProducers + 5);  // + MMA issuer + 4 epilogue warps

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
    if (warp == kProducers) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(Cfg::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_sh;

    if (warp < kProducers) {
        // ----------------------------------------------- TMA producer warps
        // The CTA's step sequence (its items blockIdx.x + i*gridDim.x in
        // order, 16-vector steps each) is dealt round-robin: producer p
        // issues global steps g = p, p + P, ...  into ring stage g % STAGES.
        // One producer warp is bound by its TMA issue latency at ~1.3 TB/s
        // (tools/gather_bench2.cu); eight saturate the TMA unit.  Each
        // producer's column indices are loaded three own steps ahead.
        StepCursor cur, pre;  // issue position; prefetch position (3 own steps ahead)
        bool ok = cur.start(a), ok_pre = pre.start(a);
        for (uint32_t k = 0; ok && k < warp; ++k) ok = cur.advance(a);
        for (uint32_t k = 0; ok_pre && k < warp; ++k) ok_pre = pre.advance(a);
        uint32_t c1 = 0, c2 = 0, c3 = 0;  // column indices of the next three own steps
        if (ok_pre) c1 = pre.cols(a, lane);
        for (int k = 0; ok_pre && k < kProducers; ++k) ok_pre = pre.advance(a);
        if (ok_pre) c2 = pre.cols(a, lane);
        for (int k = 0; ok_pre && k < kProducers; ++k) ok_pre = pre.advance(a);
        if (ok_pre) c3 = pre.cols(a, lane);
        uint32_t stage = warp, phase = 0;
        while (ok) {
            const uint32_t cs = cur.s, cvend = cur.it.vend, cbase = cur.base_v, cnvw = cur.nvw, ccol = c1;
            for (int k = 0; ok && k < kProducers; ++k) ok = cur.advance(a);
            c1 = c2;
            c2 = c3;
            for (int k = 0; ok_pre && k < kProducers; ++k) ok_pre = pre.advance(a);
            if (ok_pre) c3 = pre.cols(a, lane);  // in flight for three iterations
            const __half* vals = a.vals + 8ull * cbase;
            const bool full_step = cs + 16 <= cvend;
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* dA = sA + (size_t)stage * Cfg::A_STAGE;
            uint8_t* dS = sS + (size_t)stage * Cfg::S_STAGE;
            if (!full_step) {  // residue tile: zero fill past the window's last vector
                uint32_t w2[2];
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    uint32_t packed = 0;
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        const uint32_t e = 4 * lane + 2 * q2 + h2;  // tile element: kb*64 + r*8 + j
                        const uint32_t kb = e >> 6, r = (e >> 3) & 7, j = e & 7;
                        const uint32_t v = cs + 8 * kb + j;
                        uint32_t x = 0;
                        if (v < cvend) {
                            const uint32_t b = v >> 3, width = min(8u, cnvw - 8 * b);
                            x = __half_as_ushort(vals[64ull * b + r * width + j]);
                        }
                        packed |= x << (16 * h2);
                    }
                    w2[q2] = packed;
                }
                *reinterpret_cast<uint2*>(dS + 8 * lane) = make_uint2(w2[0], w2[1]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            __syncwarp();
            const uint32_t srcl = 4 * (lane & 3);
            const uint32_t r0 = __shfl_sync(0xffffffffu, ccol, srcl + 0);
            const uint32_t r1 = __shfl_sync(0xffffffffu, ccol, srcl + 1);
            const uint32_t r2 = __shfl_sync(0xffffffffu, ccol, srcl + 2);
            const uint32_t r3 = __shfl_sync(0xffffffffu, ccol, srcl + 3);
            if (lane == 0) mbar_expect_tx(&full[stage], H * 2048 + (full_step ? 256 : 0));
            __syncwarp();
            if (lane < 4) {
#pragma unroll
                for (int h = 0; h < H; ++h)
                    tma_gather4(dA + h * 2048 + lane * 512, &tmap, &full[stage], 64 * h, (int32_t)r0, (int32_t)r1,
                                (int32_t)r2, (int32_t)r3);
            }
            if (full_step && lane == 4) bulk_copy(dS, vals + 8ull * cs, 256, &full[stage]);
            stage += kProducers;
            if (stage >= STAGES) {
                stage -= STAGES;
                phase ^= 1;
            }
        }
    } else if (warp == kProducers) {
        // ------------------------------------------------- MMA issuer warp
        uint32_t stage = 0, phase = 0, ab = 0, aphase = 0;
        for (uint64_t idx = blockIdx.x; idx < a.n_items; idx += gridDim.x) {
            const WorkItem it = a.items[idx];
            const uint32_t nsteps = (it.vend - it.vbeg + 15) / 16;
            mbar_wait(&acc_empty[ab], aphase ^ 1);
            tc_fence_after();
            const uint32_t d0 = tbase + ab * (kAcc * 8 * H);
            for (uint32_t stp = 0; stp < nsteps; ++stp) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t aaddr = smem_u32(sA + (size_t)stage * Cfg::A_STAGE);
                    const uint64_t bdesc = desc_b_k_interleave(smem_u32(sS + (size_t)stage * Cfg::S_STAGE));
                    const uint32_t d = d0 + (stp % kAcc) * (8 * H);
#pragma unroll
                    for (int h = 0; h < H; ++h)
                        tc_mma_f16(d + 8 * h, desc_a_mn_sw128(aaddr + h * 2048), bdesc, kIdesc,
                                   stp >= kAcc ? 1u : 0u);
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
#pragma unroll
            for (int i = 0; i < 8 * H; ++i) r[i] = 0u;
            if (any) {
                const uint32_t used = min(static_cast<uint32_t>(kAcc), (it.vend - it.vbeg + 15) / 16);
                for (uint32_t j = 0; j < used; ++j) {
                    const uint32_t taddr = tbase + ((32 * q) << 16) + (ab * kAcc + j) * (8 * H);
                    uint32_t x[8 * H];
                    tmem_ld<H>(taddr, x);
#pragma unroll
                    for (int i = 0; i < 8 * H; ++i)
                        r[i] = j ? __float_as_uint(__uint_as_float(r[i]) + __uint_as_float(x[i])) : x[i];
                }
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
    if (warp == kProducers) {
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
