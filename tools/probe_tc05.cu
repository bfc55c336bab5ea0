// Probe (not product code): validates on a B200 the layout assumptions of the
// TMA-gather + tcgen05 SpMM kernel:
//   1. cp.async.bulk.tensor.2d.tile::gather4 with a {64, 1} box and
//      SWIZZLE_128B writes 4 rows at 128-B stride, 16-B chunks XOR-swizzled
//      by smem address bits [7,10); out-of-range rows are zero-filled;
//   2. tcgen05.mma.kind::f16 M=64 N=8 K=16 with A = gathered rows (MN-major,
//      SW128) and B = two ME-BCRS k=8 blocks (K-major, no swizzle, LBO=128)
//      gives D^T = (sparse * dense)^T, read back with tcgen05.ld.32x32b.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe probe_tc05.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity));
}

template <int BOXROWS>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, const int* idx, const __half* spv, uint8_t* smem_dump,
                      float* out, int K) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    uint8_t* A0 = base;          // features 0..63 : 16 rows x 128 B
    uint8_t* A1 = base + 2048;   // features 64..127
    uint8_t* Bs = base + 4096;   // 256 B sparse tile
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base;
    if (tid == 0) {
        const uint32_t b0 = smem_u32(&bar[0]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0), "r"(4096 + 256));
        for (int h = 0; h < 2; ++h)
            for (int g = 0; g < 4; ++g) {
                uint8_t* dst = (h ? A1 : A0) + g * 512;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(b0), "r"(64 * h), "r"(idx[4 * g]),
                    "r"(idx[4 * g + 1]), "r"(idx[4 * g + 2]), "r"(idx[4 * g + 3])
                    : "memory");
            }
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                         smem_u32(Bs)),
                     "l"(spv), "r"(b0)
                     : "memory");
    }
    mbar_wait(smem_u32(&bar[0]), 0);
    for (int i = tid; i < 4096 + 256; i += blockDim.x) smem_dump[i] = base[i];
    __syncthreads();
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        // instruction descriptor: F32 accum, F16 A/B, A MN-major, B K-major, N=8, M=64
        const uint32_t idesc = (1u << 4) | (1u << 15) | ((8u >> 3) << 17) | ((64u >> 4) << 24);
        for (int h = 0; h < 2; ++h) {
            const uint32_t a_addr = smem_u32(h ? A1 : A0);
            const uint64_t adesc = (uint64_t)((a_addr >> 4) & 0x3FFF) | ((uint64_t)(8192 >> 4) << 16) |
                                   ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
            const uint32_t b_addr = smem_u32(Bs);
            const uint64_t bdesc = (uint64_t)((b_addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
                                   ((uint64_t)(256 >> 4) << 32) | (1ull << 46) | (0ull << 61);
            const uint32_t d = tbase + 8 * h;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar[1])));
    }
    mbar_wait(smem_u32(&bar[1]), 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[16];
    const uint32_t taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int lane = tid & 31;
    for (int c = 0; c < 16; ++c) out[(32 * (warp & 3) + lane) * 16 + c] = __uint_as_float(r[c]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase));
}

int main() {
    const int K = 64, NC = 128;
    std::vector<__half> hB(K * NC);
    std::vector<float> fB(K * NC);
    for (int i = 0; i < K * NC; ++i) {
        float v = (float)((i * 7 + 3) % 9 - 4);
        fB[i] = v;
        hB[i] = __float2half(v);
    }
    int hidx[16] = {5, 17, 2, 63, 40, 8, 8, 31, 12, 33, 50, 1, 0, K, K + 5, 22};  // two out-of-range rows
    std::vector<__half> hS(128);
    std::vector<float> fS(128);  // block-major: block b (k=8) rows r: values[b*64 + r*8 + j]
    for (int i = 0; i < 128; ++i) {
        float v = (float)((i * 5 + 1) % 7 - 3);
        fS[i] = v;
        hS[i] = __float2half(v);
    }
    __half *dB, *dS;
    int* didx;
    uint8_t* ddump;
    float* dout;
    CK(cudaMalloc(&dB, K * NC * 2));
    CK(cudaMalloc(&dS, 256));
    CK(cudaMalloc(&didx, 64));
    CK(cudaMalloc(&ddump, 4096 + 256));
    CK(cudaMalloc(&dout, 128 * 16 * 4));
    CK(cudaMemcpy(dB, hB.data(), K * NC * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dS, hS.data(), 256, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(didx, hidx, 64, cudaMemcpyHostToDevice));
    // idx must be readable from the kernel by value: copy into constant via kernel param array
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    int fails = 0;
    for (int boxrows : {1, 4}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)NC, (cuuint64_t)K};
        cuuint64_t strides[1] = {(cuuint64_t)NC * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)boxrows};
        cuuint32_t es[2] = {1, 1};
        CUresult rc = ((EncodeTiled)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("boxrows=%d encode rc=%d\n", boxrows, (int)rc);
        if (rc != 0) continue;
        CK(cudaMemset(ddump, 0xEE, 4096 + 256));
        CK(cudaMemset(dout, 0, 128 * 16 * 4));
        // host copy of idx is passed through device memory read in-kernel
        int* hidx_dev = didx;
        auto kern = boxrows == 1 ? probe<1> : probe<4>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
        // kernel reads idx[] from global: pass device pointer
        kern<<<1, 128, 16384>>>(tm, hidx_dev, dS, ddump, dout, K);
        cudaError_t e = cudaDeviceSynchronize();
        printf("  kernel: %s\n", cudaGetErrorString(e));
        if (e != cudaSuccess) { fails++; break; }
        std::vector<uint8_t> dump(4096 + 256);
        std::vector<float> out(128 * 16);
        CK(cudaMemcpy(dump.data(), ddump, dump.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
        // (1) swizzle check: row k of half h at h*2048 + k*128; 16B chunk c stored at chunk c ^ (k & 7)
        int bad_sw = 0, bad_unsw = 0;
        for (int h = 0; h < 2; ++h)
            for (int k = 0; k < 16; ++k)
                for (int c = 0; c < 8; ++c)
                    for (int e2 = 0; e2 < 8; ++e2) {
                        const int f = 64 * h + 8 * c + e2;
                        const float want = hidx[k] < K ? fB[hidx[k] * NC + f] : 0.f;
                        __half got_sw, got_un;
                        memcpy(&got_sw, &dump[h * 2048 + k * 128 + ((c ^ (k & 7)) * 16) + e2 * 2], 2);
                        memcpy(&got_un, &dump[h * 2048 + k * 128 + c * 16 + e2 * 2], 2);
                        bad_sw += __half2float(got_sw) != want;
                        bad_unsw += __half2float(got_un) != want;
                    }
        printf("  smem layout mismatches: swizzled-hypothesis=%d unswizzled=%d\n", bad_sw, bad_unsw);
        // (2) MMA check: D_h[m][n] = sum_k B[idx[k]][64h+m] * S[n][k]; S[n][k] = block k/8, value[(k/8)*64 + n*8 + k%8]
        int bad_mma = 0;
        for (int h = 0; h < 2; ++h)
            for (int m = 0; m < 64; ++m)
                for (int n = 0; n < 8; ++n) {
                    float want = 0;
                    for (int k = 0; k < 16; ++k) {
                        const float a = hidx[k] < K ? fB[hidx[k] * NC + 64 * h + m] : 0.f;
                        want += a * fS[(k / 8) * 64 + n * 8 + (k % 8)];
                    }
                    const int lane = 32 * (m / 16) + (m % 16);
                    const float got = out[lane * 16 + 8 * h + n];
                    if (got != want) {
                        if (bad_mma < 5) printf("    D%d[%d][%d] got %f want %f\n", h, m, n, got, want);
                        bad_mma++;
                    }
                }
        printf("  mma mismatches: %d\n", bad_mma);
        fails += (bad_sw != 0) + (bad_mma != 0);
    }
    printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
    return fails ? 1 : 0;
}
