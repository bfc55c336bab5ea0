// Microbenchmark (not product code), follow-up to gather_bench.cu: the TMA
// gather4 and LDGSTS rows there were limited by a dependent index load per
// stage (each producer waited one L2/DRAM round trip before every TMA
// issue).  Here the producers prefetch their row indices D stages ahead, so
// the measured rate is the TMA / LDGSTS engine's, not the index latency.
// Same workload: 32M random 256-byte row gathers from an L2-resident
// 233K x 128 fp16 matrix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_bench2 tools/gather_bench2.cu -lcuda
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

// P producer warps + 1 consumer warp per CTA, STAGES x 4 KB ring (16 rows of
// 256 B per stage).  MODE 0: gather4 box {64,1} SW128 (two per 4 rows);
// MODE 2: gather4 box {128,1} no swizzle (one per 4 rows).  A producer's lane
// j < 16 holds the row index of stage (its k-th + D) -- loaded D stages early.
template <int P, int STAGES, int MODE, int D>
__global__ void __launch_bounds__(32 * (P + 1), 1) tma_pf_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                 const uint32_t* __restrict__ idx, uint64_t nrows_total) {
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
    const uint64_t nstages_total = nrows_total / 16;
    const uint64_t per_cta = (nstages_total + gridDim.x - 1) / gridDim.x;
    const uint64_t s0 = blockIdx.x * per_cta, s1 = min(nstages_total, s0 + per_cta);
    if (warp < P) {
        uint32_t pre[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const uint64_t s = s0 + warp + uint64_t(d) * P;
            pre[d] = (lane < 16 && s < s1) ? __ldg(idx + s * 16 + lane) : 0u;
        }
        for (uint64_t s = s0 + warp; s < s1; s += uint64_t(D) * P) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const uint64_t sd = s + uint64_t(d) * P;
                if (sd >= s1) break;
                const uint32_t myrow = pre[d];
                const uint64_t sn = sd + uint64_t(D) * P;
                pre[d] = (lane < 16 && sn < s1) ? __ldg(idx + sn * 16 + lane) : 0u;
                const uint32_t slot = (uint32_t)((sd - s0) % STAGES);
                const uint32_t ph = (uint32_t)(((sd - s0) / STAGES) & 1);
                mbar_wait(&empty[slot], ph ^ 1);
                uint8_t* dst = base + (size_t)slot * 4096;
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])), "r"(4096) : "memory");
                __syncwarp();
                const uint32_t srcl = 4 * (lane & 3);
                const uint32_t r0 = __shfl_sync(0xffffffffu, myrow, srcl), r1 = __shfl_sync(0xffffffffu, myrow, srcl + 1),
                               r2 = __shfl_sync(0xffffffffu, myrow, srcl + 2), r3 = __shfl_sync(0xffffffffu, myrow, srcl + 3);
                if (lane < 4) {
                    if (MODE == 0) {
#pragma unroll
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

// LDGSTS (cp.async.cg 16 B) with indices prefetched 8 iterations ahead: each
// warp iteration gathers 4 rows x 256 B into a 4-slot ring.
__global__ void __launch_bounds__(256) cpasync_pf_kernel(const uint4* __restrict__ B, const uint32_t* __restrict__ idx,
                                                         uint64_t nrows_total) {
    __shared__ __align__(16) uint4 buf[8][4][32][2];
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    uint32_t it = 0;
    for (uint64_t g0 = warp * 32; g0 < nrows_total; g0 += nwarps * 32) {  // 32 rows: one index per lane
        const uint32_t mine = __ldg(idx + g0 + lane);
#pragma unroll
        for (int u = 0; u < 8; ++u, ++it) {
            const uint32_t row = __shfl_sync(0xffffffffu, mine, 4 * u + (lane >> 3));
            const uint4* p = B + (uint64_t)row * 16 + (lane & 7);
            uint4* d = &buf[wl][it & 3][lane][0];
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d)), "l"(p));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d + 1)), "l"(p + 8));
            asm volatile("cp.async.commit_group;");
            asm volatile("cp.async.wait_group 3;");
        }
    }
    asm volatile("cp.async.wait_group 0;");
}

// LDG.128 at the SpMM kernel's memory-level parallelism: 16 rows x 256 B
// (4 KB) in flight per warp, 4 warps x 4 CTAs per SM, plus the SHFL
// redistribution the mma.sync fragment needs (one SHFL per loaded register).
template <bool SHFL>
__global__ void __launch_bounds__(128, 4) ldg_spmm_like(const uint4* __restrict__ B, const uint32_t* __restrict__ idx,
                                                        uint64_t nrows_total, uint4* sink) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint32_t src = 8 * (lane & 3) + (lane >> 2);
    for (uint64_t g0 = warp * 32; g0 < nrows_total; g0 += nwarps * 32) {
        const uint32_t mine = __ldg(idx + g0 + lane);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t row = __shfl_sync(0xffffffffu, mine, 16 * h + 4 * u + (lane >> 3));
                const uint4* p = B + (uint64_t)row * 16 + (lane & 7);
                v[2 * u] = __ldg(p);
                v[2 * u + 1] = __ldg(p + 8);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                uint4 x = v[u];
                if (SHFL) {
                    x.x = __shfl_sync(0xffffffffu, x.x, src);
                    x.y = __shfl_sync(0xffffffffu, x.y, src);
                    x.z = __shfl_sync(0xffffffffu, x.z, src);
                    x.w = __shfl_sync(0xffffffffu, x.w, src);
                }
                acc.x ^= x.x; acc.y ^= x.y; acc.z ^= x.z; acc.w ^= x.w;
            }
        }
    }
    if (acc.x == 0x12345678u) sink[0] = acc;
}

// ldg_spmm_like + the SpMM kernel's arithmetic: PRMT pairs + HMMA m16n8k16
// per shuffled register quad (MMA), and the sparse-operand stream: VALS = 0
// none, 1 = 16 B of values per gathered row loaded right before use (read
// once with L1::no_allocate, as the ME-BCRS values are), 2 = the same loaded
// one 32-row iteration ahead.
template <bool MMA, int VALS>
__global__ void __launch_bounds__(128, 4) ldg_spmm_math(const uint4* __restrict__ B, const uint32_t* __restrict__ idx,
                                                        const uint2* __restrict__ vals, uint64_t nrows_total,
                                                        float* sink) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    float acc[8][4] = {};
    const uint32_t src = 8 * (lane & 3) + (lane >> 2);
    uint2 pre[2] = {make_uint2(0, 0), make_uint2(0, 0)};
    if (VALS == 2 && warp * 32 < nrows_total) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint2* pv = vals + (warp * 32 + 16 * h) * 2 + lane;
            asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0,%1}, [%2];" : "=r"(pre[h].x), "=r"(pre[h].y) : "l"(pv));
        }
    }
    for (uint64_t g0 = warp * 32; g0 < nrows_total; g0 += nwarps * 32) {
        const uint32_t mine = __ldg(idx + g0 + lane);
        uint2 cur[2] = {pre[0], pre[1]};
        if (VALS == 2 && g0 + nwarps * 32 < nrows_total) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint2* pv = vals + (g0 + nwarps * 32 + 16 * h) * 2 + lane;
                asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0,%1}, [%2];" : "=r"(pre[h].x), "=r"(pre[h].y) : "l"(pv));
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t row = __shfl_sync(0xffffffffu, mine, 16 * h + 4 * u + (lane >> 3));
                const uint4* p = B + (uint64_t)row * 16 + (lane & 7);
                v[2 * u] = __ldg(p);
                v[2 * u + 1] = __ldg(p + 8);
            }
            uint2 b = make_uint2(0x3c003c00u, 0x3c003c00u);
            if (VALS == 2) b = cur[h];
            if (VALS == 1) {
                const uint2* pv = vals + (g0 + 16 * h) * 2 + lane;
                asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0,%1}, [%2];" : "=r"(b.x), "=r"(b.y) : "l"(pv));
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t x[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint4 w = v[2 * u + c];
                        const uint32_t r = j == 0 ? w.x : j == 1 ? w.y : j == 2 ? w.z : w.w;
                        x[u] = __shfl_sync(0xffffffffu, r, src);
                    }
                    if (MMA) {
                        const uint32_t a0 = __byte_perm(x[0], x[1], 0x5410), a1 = __byte_perm(x[0], x[1], 0x7632);
                        const uint32_t a2 = __byte_perm(x[2], x[3], 0x5410), a3 = __byte_perm(x[2], x[3], 0x7632);
                        float* d = acc[4 * c + j];
                        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                                     : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b.x), "r"(b.y));
                    } else {
                        acc[4 * c + j][0] += __uint_as_float(x[0] ^ x[1] ^ x[2] ^ x[3] ^ b.x);
                    }
                }
        }
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    if (t == 1234.5f) sink[0] = t;
}

// Alternative fragment exchange: lane 4v + r loads 16 B (features 8r..8r+7)
// of vector v (a quarter-warp reads 2 rows x 64 B), then one movmatrix.trans
// per register yields the mma.sync A fragment (feature, vector pair).  Same
// bytes and the same 4 KB per warp in flight as ldg_spmm_like.
__global__ void __launch_bounds__(128, 4) ldg_movmatrix(const uint4* __restrict__ B, const uint32_t* __restrict__ idx,
                                                        uint64_t nrows_total, uint4* sink) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint64_t g0 = warp * 32; g0 < nrows_total; g0 += nwarps * 32) {
        const uint32_t mine = __ldg(idx + g0 + lane);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 2; ++u) {  // 8 vectors per u; 16 per h
                const uint32_t row = __shfl_sync(0xffffffffu, mine, 16 * h + 8 * u + (lane >> 2));
#pragma unroll
                for (int c = 0; c < 4; ++c)  // 4 x 32 features: lane r covers features 32c + 8r .. +7
                    v[4 * u + c] = __ldg(B + (uint64_t)row * 16 + 4 * c + (lane & 3));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                uint4 x = v[u];
                asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x.x));
                asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x.y));
                asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x.z));
                asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x.w));
                acc.x ^= x.x; acc.y ^= x.y; acc.z ^= x.z; acc.w ^= x.w;
            }
        }
    }
    if (acc.x == 0x12345678u) sink[0] = acc;
}

// Hybrid: per 32-row iteration a warp gathers 16 rows with LDG.128 + SHFL
// and the other 16 with TMA gather4 (box {64,1}, 128-B swizzle) into its
// own shared-memory slot, read back with ldmatrix.x4.trans (conflict-free
// under the swizzle).  TMA for iteration i+1 is issued before the LDG part
// of iteration i.  Tests whether moving half of the bytes off the LDG+SHFL
// path (2 L1 wavefronts per 128 B) onto TMA + ldmatrix (1 wavefront) lifts
// the per-SM ceiling.
__global__ void __launch_bounds__(128, 4) hybrid_kernel(const __grid_constant__ CUtensorMap tmap,
                                                        const uint4* __restrict__ B, const uint32_t* __restrict__ idx,
                                                        uint64_t nrows_total, uint4* sink) {
    __shared__ __align__(1024) uint8_t slots[4][2][4096];
    __shared__ __align__(8) uint64_t bar[4][2];
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[wl][0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[wl][1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const uint32_t src = 8 * (lane & 3) + (lane >> 2);
    uint4 acc = make_uint4(0, 0, 0, 0);
    auto issue = [&](uint64_t g, uint32_t slot, uint32_t rows_idx) {
        // rows_idx: lane j < 16 holds row index of TMA row j
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[wl][slot])), "r"(4096) : "memory");
        __syncwarp();
        const uint32_t srcl = 4 * (lane & 3);
        const uint32_t r0 = __shfl_sync(0xffffffffu, rows_idx, srcl), r1 = __shfl_sync(0xffffffffu, rows_idx, srcl + 1),
                       r2 = __shfl_sync(0xffffffffu, rows_idx, srcl + 2), r3 = __shfl_sync(0xffffffffu, rows_idx, srcl + 3);
        if (lane < 4) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(&slots[wl][slot][h * 2048 + lane * 512])), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(smem_u32(&bar[wl][slot])), "r"(64 * h), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
        }
    };
    uint64_t g0 = warp * 32;
    if (g0 >= nrows_total) return;
    uint32_t mine = __ldg(idx + g0 + lane);
    issue(g0, 0, __shfl_sync(0xffffffffu, mine, 16 + (lane & 15)));
    uint32_t it = 0;
    for (; g0 < nrows_total; g0 += nwarps * 32, ++it) {
        const uint64_t gn = g0 + nwarps * 32;
        const uint32_t next = gn < nrows_total ? __ldg(idx + gn + lane) : 0u;
        if (gn < nrows_total) issue(gn, (it + 1) & 1, __shfl_sync(0xffffffffu, next, 16 + (lane & 15)));
        // LDG + SHFL half: rows 0..15 of this iteration
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t row = __shfl_sync(0xffffffffu, mine, 4 * u + (lane >> 3));
            const uint4* p = B + (uint64_t)row * 16 + (lane & 7);
            v[2 * u] = __ldg(p);
            v[2 * u + 1] = __ldg(p + 8);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            uint4 x = v[u];
            x.x = __shfl_sync(0xffffffffu, x.x, src);
            x.y = __shfl_sync(0xffffffffu, x.y, src);
            x.z = __shfl_sync(0xffffffffu, x.z, src);
            x.w = __shfl_sync(0xffffffffu, x.w, src);
            acc.x ^= x.x; acc.y ^= x.y; acc.z ^= x.z; acc.w ^= x.w;
        }
        // TMA half: wait, then 8 x ldmatrix.x4.trans over the 4 KB slot
        const uint32_t slot = it & 1;
        mbar_wait(&bar[wl][slot], (it >> 1) & 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            // instruction i: half h = i/4, 16-B logical chunk pair; lane -> row (lane & 15), chunk 2*(i%4) + (lane >> 4)
            const uint32_t h = i >> 2, r = lane & 15, c = 2 * (i & 3) + (lane >> 4);
            const uint32_t addr = smem_u32(&slots[wl][slot][h * 2048 + r * 128 + ((c ^ (r & 7)) * 16)]);
            uint32_t a0, a1, a2, a3;
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(addr));
            acc.x ^= a0; acc.y ^= a1; acc.z ^= a2; acc.w ^= a3;
        }
        __syncwarp();
        mine = next;
    }
    if (acc.x == 0x12345678u) sink[0] = acc;
}

int main() {
    const int K = 232965, NC = 128;
    const uint64_t R = 1ull << 25;
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
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        printf("%-52s %8.3f ms  %8.1f GB/s\n", name, ms, R * 256.0 / ms / 1e6);
    };
    report("LDG.128, SpMM-like MLP (4 KB/warp, 16 warps/SM)", [&] { ldg_spmm_like<false><<<sms * 4, 128>>>((const uint4*)dB, didx, R, sink); });
    report("LDG.128 + SHFL, SpMM-like MLP", [&] { ldg_spmm_like<true><<<sms * 4, 128>>>((const uint4*)dB, didx, R, sink); });
    uint2* dvals;
    CK(cudaMalloc(&dvals, R * 16));
    CK(cudaMemset(dvals, 0, R * 16));
    report("LDG+SHFL (no MMA), same code shape", [&] { ldg_spmm_math<false, 0><<<sms * 4, 128>>>((const uint4*)dB, didx, dvals, R, (float*)sink); });
    report("LDG+SHFL + PRMT + HMMA", [&] { ldg_spmm_math<true, 0><<<sms * 4, 128>>>((const uint4*)dB, didx, dvals, R, (float*)sink); });
    report("LDG+SHFL + PRMT + HMMA + 16 B/row values, loaded at use", [&] { ldg_spmm_math<true, 1><<<sms * 4, 128>>>((const uint4*)dB, didx, dvals, R, (float*)sink); });
    report("LDG+SHFL + PRMT + HMMA + values one iteration ahead", [&] { ldg_spmm_math<true, 2><<<sms * 4, 128>>>((const uint4*)dB, didx, dvals, R, (float*)sink); });
    report("LDG.128 2 rows/quarter + movmatrix.trans", [&] { ldg_movmatrix<<<sms * 4, 128>>>((const uint4*)dB, didx, R, sink); });
    report("cp.async.cg 16B -> smem, idx prefetched", [&] { cpasync_pf_kernel<<<sms * 7, 256>>>((const uint4*)dB, didx, R); });

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap t64, t128;
    cuuint64_t dims[2] = {(cuuint64_t)NC, (cuuint64_t)K};
    cuuint64_t strides[1] = {(cuuint64_t)NC * 2};
    cuuint32_t es[2] = {1, 1};
    cuuint32_t box64[2] = {64, 1}, box128[2] = {128, 1};
    ((EncodeTiled)fn)(&t64, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, dims, strides, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    ((EncodeTiled)fn)(&t128, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, dims, strides, box128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    report("hybrid: 16 rows LDG+SHFL + 16 rows TMA->ldmatrix per warp", [&] { hybrid_kernel<<<sms * 4, 128>>>(t64, (const uint4*)dB, didx, R, sink); });
    const size_t smem = 1024 + 48 * 4096;
#define TMA_CASE(P, MODE, D, MAP, NAME)                                                                                  \
    {                                                                                                                    \
        CK(cudaFuncSetAttribute(tma_pf_kernel<P, 48, MODE, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        report(NAME, [&] { tma_pf_kernel<P, 48, MODE, D><<<sms, 32 * (P + 1), smem>>>(MAP, didx, R); });               \
    }
    TMA_CASE(1, 0, 8, t64, "TMA gather4 {64,1} SW128, 1 warp, idx 8 ahead");
    TMA_CASE(2, 0, 8, t64, "TMA gather4 {64,1} SW128, 2 warps, idx 8 ahead");
    TMA_CASE(4, 0, 8, t64, "TMA gather4 {64,1} SW128, 4 warps, idx 8 ahead");
    TMA_CASE(8, 0, 4, t64, "TMA gather4 {64,1} SW128, 8 warps, idx 4 ahead");
    TMA_CASE(1, 2, 8, t128, "TMA gather4 {128,1} no swizzle, 1 warp, idx 8 ahead");
    TMA_CASE(4, 2, 8, t128, "TMA gather4 {128,1} no swizzle, 4 warps, idx 8 ahead");
    TMA_CASE(8, 2, 4, t128, "TMA gather4 {128,1} no swizzle, 8 warps, idx 4 ahead");
    TMA_CASE(16, 2, 2, t128, "TMA gather4 {128,1} no swizzle, 16 warps, idx 2 ahead");
    TMA_CASE(24, 2, 2, t128, "TMA gather4 {128,1} no swizzle, 24 warps, idx 2 ahead");
    TMA_CASE(16, 0, 2, t64, "TMA gather4 {64,1} SW128, 16 warps, idx 2 ahead");
    return 0;
}
