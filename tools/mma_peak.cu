// Legacy tensor-path (mma.sync -> HMMA) peak on this GPU: back-to-back
// m16n8k16 f16 -> f32 and m16n8k8 tf32 -> f32 MMAs with independent
// accumulator chains, every SM, CUDA events.  The SpMM's tensor-pipe
// fraction (bench.py roofline.tensor_pipe) is quoted against this figure.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_peak tools/mma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <bool TF32>
__global__ void __launch_bounds__(256) mma_loop(float* sink, unsigned seed) {
    unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b0 = a0 * 11u, b1 = a0 * 13u;
    float d[kChains][4] = {};
#pragma unroll 1
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if constexpr (TF32)
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            else
                asm volatile(
                    "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 12345.678f) sink[threadIdx.x] = s;  // keep the work
}

template <bool TF32>
double run(int sms, int blocks_per_sm) {
    float* sink;
    cudaMalloc(&sink, 1024 * sizeof(float));
    const int grid = sms * blocks_per_sm;
    mma_loop<TF32><<<grid, 256>>>(sink, 1u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        mma_loop<TF32><<<grid, 256>>>(sink, 2u + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double k = TF32 ? 8.0 : 16.0;
    const double flops = double(grid) * 8 /* warps */ * kIters * kChains * 2.0 * 16 * 8 * k;
    cudaFree(sink);
    return flops / (best * 1e-3) / 1e12;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    for (int bps : {1, 2, 4}) {
        const double f16 = run<false>(sms, bps), tf32 = run<true>(sms, bps);
        std::printf("mma.sync peak, %d SMs x %d CTAs of 8 warps, %d chains: f16 m16n8k16 %.1f TFLOP/s, "
                    "tf32 m16n8k8 %.1f TFLOP/s\n", sms, bps, kChains, f16, tf32);
    }
    std::printf("rc=%d\n", (int)cudaGetLastError());
    return 0;
}
