// Does the lane -> address layout of a 4-row LDG.128 gather change the
// L2 -> SM throughput?  Each load instruction reads 4 random rows x 128 B:
//   quarter: lane l reads row r[l >> 3], bytes 16 * (l & 7)   (one row per quarter-warp;
//            the SpMM kernels' layout, which then needs SHFLs to reach the MMA fragments)
//   tstride: lane l reads row r[l & 3],  bytes 16 * (l >> 2)  (lanes t, t+4, ... share a row;
//            the layout in which each lane loads its own m16n8k16 A-fragment data)
// Same memory-level parallelism and warps per SM for both.  Prints one line per
// (layout, unroll, blocks/SM) and a JSON summary.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_layout tools/gather_layout.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                             \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                 \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

// rows of 256 B; one instruction = 4 rows x one 128-B half (h alternates)
template <int UNR, bool TSTRIDE>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ table, const uint32_t* __restrict__ idx,
                                              uint64_t n_rows_per_warp, uint4* __restrict__ sink) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t sel = TSTRIDE ? (lane & 3) : (lane >> 3);  // which of the 4 rows
    const uint32_t seg = TSTRIDE ? (lane >> 2) : (lane & 7);  // 16-B segment within the 128-B half
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t* wi = idx + warp * n_rows_per_warp;
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint32_t nxt[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) nxt[u] = __ldg(wi + 4 * (u / 2) + sel);
    // UNR instructions per iteration: pairs (row quad, half 0/1)
    for (uint64_t r = 0; r < n_rows_per_warp; r += 2 * UNR) {
        uint4 v[UNR];
        uint32_t cur[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) cur[u] = nxt[u];
        if (r + 2 * UNR < n_rows_per_warp) {
#pragma unroll
            for (int u = 0; u < UNR; ++u) nxt[u] = __ldg(wi + r + 2 * UNR + 4 * (u / 2) + sel);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint4* p = table + (uint64_t(cur[u]) * 16 + (u & 1) * 8 + seg);
            asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w;
        }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) sink[warp] = acc;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t rows = 232965;  // C3's dense operand, N = 128 f16: 59.6 MB
    const uint64_t n_rows_per_warp = 4096;
    uint4* table = nullptr;
    CK(cudaMalloc(&table, rows * 256));
    CK(cudaMemset(table, 1, rows * 256));
    uint4* sink = nullptr;
    const int warps_per_block = 8;
    const uint64_t max_warps = uint64_t(sms) * 8 * warps_per_block;
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
    double best[2] = {0, 0};
    auto run = [&](auto kern, int layout, int unr, int bps) -> int {
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
        std::printf("%-8s unroll %2d  blocks/SM %d  %.1f GB/s\n", layout ? "tstride" : "quarter", unr, bps, gbs);
        if (gbs > best[layout]) best[layout] = gbs;
        return 0;
    };
    for (int bps : {2, 4, 6}) {
        if (run(gather<4, false>, 0, 4, bps) || run(gather<4, true>, 1, 4, bps)) return 1;
        if (run(gather<8, false>, 0, 8, bps) || run(gather<8, true>, 1, 8, bps)) return 1;
        if (run(gather<16, false>, 0, 16, bps) || run(gather<16, true>, 1, 16, bps)) return 1;
    }
    std::printf("{\"quarter_gbs\": %.1f, \"tstride_gbs\": %.1f}\n", best[0], best[1]);
    return 0;
}
