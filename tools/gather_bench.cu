// Microbenchmark (not product code): bandwidth of row gathers from an
// L2-resident dense matrix (233K x 128 fp16 rows of 256 B, random rows) with
// the gather mechanisms available on sm_100a.  Decides the SpMM design.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}

// --- 1: LDG.128 variants: each warp gathers 4 rows per instruction (8 lanes x 16 B per row)
template <int MODE>
__global__ void __launch_bounds__(256) ldg_kernel(const uint4* __restrict__ B, const uint32_t* __restrict__ idx, uint64_t nrows_total, uint4* sink) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint64_t g = warp * 32; g < nrows_total; g += nwarps * 32) {  // 32 rows per warp iteration
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t row = __ldg(idx + g + 4 * u + (lane >> 3));
            const uint4* p = B + (uint64_t)row * 16 + (lane & 7) + 8 * 0;
            if (MODE == 0) v[u] = __ldg(p);
            else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
            else asm volatile("ld.global.cg.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
        }
        // second half of each row (features 64..127)
        uint4 w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t row = __ldg(idx + g + 4 * u + (lane >> 3));
            const uint4* p = B + (uint64_t)row * 16 + (lane & 7) + 8;
            if (MODE == 0) w[u] = __ldg(p);
            else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w) : "l"(p));
            else asm volatile("ld.global.cg.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w) : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) { acc.x ^= v[u].x ^ w[u].x; acc.y ^= v[u].y ^ w[u].y; acc.z ^= v[u].z ^ w[u].z; acc.w ^= v[u].w ^ w[u].w; }
    }
    if (acc.x == 0x12345678u) sink[0] = acc;
}

// --- 2: TMA gather4 ring: P producer warps, 1 consumer warp (just releases stages)
template <int P, int STAGES, int MODE>  // MODE 0: gather4 box{64,1} SW128 (2 per 4 rows); 1: bulk 1D 256 B per row; 2: gather4 box{128,1} no swizzle
__global__ void __launch_bounds__(32 * (P + 1), 1) tma_kernel(const __grid_constant__ CUtensorMap tmap, const __half* B, const uint32_t* __restrict__ idx, uint64_t nrows_total) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    // stage = 16 rows x 256 B = 4 KB; stages distributed round-robin over producer warps
    const uint64_t nstages_total = nrows_total / 16;
    const uint64_t per_cta = (nstages_total + gridDim.x - 1) / gridDim.x;
    const uint64_t s0 = blockIdx.x * per_cta, s1 = min(nstages_total, s0 + per_cta);
    if (warp < P) {
        uint32_t k = 0;
        for (uint64_t s = s0 + warp; s < s1; s += P, ++k) {
            const uint32_t slot = (uint32_t)((s - s0) % STAGES);
            const uint32_t ph = (uint32_t)(((s - s0) / STAGES) & 1);
            mbar_wait(&empty[slot], ph ^ 1);
            const uint32_t myrow = lane < 16 ? __ldg(idx + s * 16 + lane) : 0u;
            uint8_t* dst = base + (size_t)slot * 4096;
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])), "r"(4096) : "memory");
            __syncwarp();
            if (MODE == 1) {
                if (lane < 16) {
                    const __half* src = B + (uint64_t)myrow * 128;
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(smem_u32(dst + lane * 256)), "l"(src), "r"(smem_u32(&full[slot])) : "memory");
                }
            } else {
                const uint32_t srcl = 4 * (lane & 3);
                const uint32_t r0 = __shfl_sync(0xffffffffu, myrow, srcl), r1 = __shfl_sync(0xffffffffu, myrow, srcl + 1), r2 = __shfl_sync(0xffffffffu, myrow, srcl + 2), r3 = __shfl_sync(0xffffffffu, myrow, srcl + 3);
                if (lane < 4) {
                    if (MODE == 0) {
                        for (int h = 0; h < 2; ++h)
                            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst + h * 2048 + lane * 512)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(smem_u32(&full[slot])), "r"(64 * h), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
                    } else {
                        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst + lane * 1024)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(smem_u32(&full[slot])), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
                    }
                }
            }
        }
    } else {
        for (uint64_t s = s0; s < s1; ++s) {
            const uint32_t slot = (uint32_t)((s - s0) % STAGES);
            const uint32_t ph = (uint32_t)(((s - s0) / STAGES) & 1);
            mbar_wait(&full[slot], ph);
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
            __syncwarp();
        }
    }
}

// --- 3: cp.async 16 B (LDGSTS) ring per warp
__global__ void __launch_bounds__(256) cpasync_kernel(const uint4* __restrict__ B, const uint32_t* __restrict__ idx, uint64_t nrows_total) {
    __shared__ __align__(16) uint4 buf[8][4][32][2];  // per warp 4 slots x (32 lanes x 2 x 16 B)
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    uint32_t it = 0;
    for (uint64_t g = warp * 4; g < nrows_total; g += nwarps * 4, ++it) {  // 4 rows x 256 B per iteration
        const uint32_t row = __ldg(idx + g + (lane >> 3));
        const uint4* p = B + (uint64_t)row * 16 + (lane & 7);
        uint4* d = &buf[wl][it & 3][lane][0];
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d)), "l"(p));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d + 1)), "l"(p + 8));
        asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 3;");
    }
    asm volatile("cp.async.wait_group 0;");
}

int main() {
    const int K = 232965, NC = 128;
    const uint64_t R = 1ull << 25;  // 32M row gathers = 8 GB
    __half* dB;
    uint32_t* didx;
    uint4* sink;
    CK(cudaMalloc(&dB, (size_t)K * NC * 2));
    CK(cudaMemset(dB, 1, (size_t)K * NC * 2));
    CK(cudaMalloc(&didx, R * 4));
    CK(cudaMalloc(&sink, 64));
    std::vector<uint32_t> h(R);
    uint64_t x = 88172645463325252ull;
    for (uint64_t i = 0; i < R; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)(x % K); }
    CK(cudaMemcpy(didx, h.data(), R * 4, cudaMemcpyHostToDevice));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto report = [&](const char* name, auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        printf("%-44s %8.3f ms  %8.1f GB/s\n", name, ms, R * 256.0 / ms / 1e6);
    };
    report("LDG.128 nc (L1 alloc)", [&] { ldg_kernel<0><<<sms * 8, 256>>>((const uint4*)dB, didx, R, sink); });
    report("LDG.128 nc L1::no_allocate", [&] { ldg_kernel<1><<<sms * 8, 256>>>((const uint4*)dB, didx, R, sink); });
    report("LDG.128 cg (L2 only)", [&] { ldg_kernel<2><<<sms * 8, 256>>>((const uint4*)dB, didx, R, sink); });
    report("cp.async.cg 16B -> smem", [&] { cpasync_kernel<<<sms * 8, 256>>>((const uint4*)dB, didx, R); });

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap t64, t128;
    cuuint64_t dims[2] = {(cuuint64_t)NC, (cuuint64_t)K};
    cuuint64_t strides[1] = {(cuuint64_t)NC * 2};
    cuuint32_t es[2] = {1, 1};
    cuuint32_t box64[2] = {64, 1}, box128[2] = {128, 1};
    CUresult r1 = ((EncodeTiled)fn)(&t64, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, dims, strides, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = ((EncodeTiled)fn)(&t128, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, dims, strides, box128, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor maps: %d %d\n", (int)r1, (int)r2);
    const size_t smem = 1024 + 32 * 4096;
#define TMA_CASE(P, MODE, MAP, NAME)                                                                             \
    {                                                                                                          \
        CK(cudaFuncSetAttribute(tma_kernel<P, 32, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        report(NAME, [&] { tma_kernel<P, 32, MODE><<<sms, 32 * (P + 1), smem>>>(MAP, dB, didx, R); });         \
    }
    TMA_CASE(1, 0, t64, "TMA gather4 {64,1} SW128, 1 producer warp");
    TMA_CASE(2, 0, t64, "TMA gather4 {64,1} SW128, 2 producer warps");
    TMA_CASE(4, 0, t64, "TMA gather4 {64,1} SW128, 4 producer warps");
    if (r2 == 0) {
        TMA_CASE(1, 2, t128, "TMA gather4 {128,1} no swizzle, 1 warp");
        TMA_CASE(4, 2, t128, "TMA gather4 {128,1} no swizzle, 4 warps");
    }
    TMA_CASE(1, 1, t64, "cp.async.bulk 256 B per row, 1 warp");
    TMA_CASE(4, 1, t64, "cp.async.bulk 256 B per row, 4 warps");
    return 0;
}
