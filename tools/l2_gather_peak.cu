// Hardware ceiling of the SpMM's dominant traffic: random 256-byte row
// gathers served by L2 (the dense operand of C3 FP16 N=128 is 60 MB and
// L2-resident).  Pure LDG.128 -- no shuffles, no MMA, no sparse stream --
// with each quarter-warp reading one 128-byte segment, swept over the
// memory-level parallelism (independent loads in flight per thread) and the
// resident warps per SM; the best rate is the L2 -> SM gather peak the bench
// divides by (roofline.l2_gather).  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_gather_peak tools/l2_gather_peak.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                      \
            return 1;                                                                          \
        }                                                                                      \
    } while (0)

// Each warp-iteration gathers UNR rows of 256 B per quarter-warp pair:
// quarter q of the warp reads segment (q & 1) of row idx[...] -- 4 quarters
// cover 2 rows per load instruction, UNR instructions in flight.
template <int UNR>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ table, const uint32_t* __restrict__ idx,
                                              uint64_t n_rows_per_warp, uint4* __restrict__ sink) {
    const uint32_t lane = threadIdx.x & 31, q = lane >> 3, l8 = lane & 7;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t* wi = idx + warp * n_rows_per_warp;
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint32_t nxt[UNR];  // row indices one iteration ahead (no dependent index load before a gather)
#pragma unroll
    for (int u = 0; u < UNR; ++u) nxt[u] = __ldg(wi + 2 * u + (q >> 1));
    for (uint64_t r = 0; r < n_rows_per_warp; r += 2 * UNR) {
        uint4 v[UNR];
        uint32_t cur[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) cur[u] = nxt[u];
        if (r + 2 * UNR < n_rows_per_warp) {
#pragma unroll
            for (int u = 0; u < UNR; ++u) nxt[u] = __ldg(wi + r + 2 * UNR + 2 * u + (q >> 1));
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint4* p = table + (uint64_t(cur[u]) * 16 + (q & 1) * 8 + l8);
            asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w;
        }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) sink[warp] = acc;  // keeps the loads alive
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t rows = 232965;  // C3's dense operand: 232,965 x 128 f16 = 59.6 MB
    const uint64_t n_rows_per_warp = 4096;
    uint4* table = nullptr;
    CK(cudaMalloc(&table, rows * 256));
    CK(cudaMemset(table, 1, rows * 256));
    uint4* sink = nullptr;
    const int max_blocks_per_sm = 8, warps_per_block = 8;
    const uint64_t max_warps = uint64_t(sms) * max_blocks_per_sm * warps_per_block;
    CK(cudaMalloc(&sink, max_warps * sizeof(uint4)));
    std::vector<uint32_t> h(max_warps * n_rows_per_warp);
    std::mt19937 g(2412);
    for (auto& x : h) x = g() % rows;
    uint32_t* idx = nullptr;
    CK(cudaMalloc(&idx, h.size() * 4));
    CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    double best = 0;
    int best_unr = 0, best_bps = 0;
    auto run = [&](auto kern, int unr, int bps) -> int {
        const int grid = sms * bps;
        for (int rep = 0; rep < 2; ++rep) kern<<<grid, 256>>>(table, idx, n_rows_per_warp, sink);
        CK(cudaEventRecord(a));
        const int reps = 5;
        for (int rep = 0; rep < reps; ++rep) kern<<<grid, 256>>>(table, idx, n_rows_per_warp, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double bytes = double(grid) * warps_per_block * n_rows_per_warp * 256.0 * reps;
        const double gbs = bytes / (ms * 1e-3) / 1e9;
        std::fprintf(stderr, "unroll %2d  blocks/SM %d  %.1f GB/s\n", unr, bps, gbs);
        if (gbs > best) best = gbs, best_unr = unr, best_bps = bps;
        return 0;
    };
    for (int bps : {2, 4, 6, 8}) {
        if (run(gather<2>, 2, bps) || run(gather<4>, 4, bps) || run(gather<8>, 8, bps)) return 1;
    }
    std::printf("{\"l2_gather_peak_gbs\": %.1f, \"unroll\": %d, \"blocks_per_sm\": %d, \"row_bytes\": 256, "
                "\"table_mb\": %.1f, \"pattern\": \"uniform random rows, LDG.128, quarter-warp per 128-B segment\"}\n",
                best, best_unr, best_bps, rows * 256 / 1e6);
    return 0;
}
