// ============================================================================
// TEST INFRASTRUCTURE ONLY -- the multi-GPU C-ABI (include/tcs/tcs_dist.h)
// and its drop-in overload tcsparse::gpu::spmm_sharded, driven from C++ with
// a real NCCL communicator, checked against the reference (tcsparse::spmm,
// ref spmm.hpp:173) and the single-GPU path:
//
//   1. spmm_sharded over an NCCL communicator == the reference's spmm, bit
//      for bit (small-integer inputs, ref generate.hpp:13-18), FP16 + TF32;
//   2. tcs_shard_windows == the nnz-balanced rule, for world 1..8;
//   3. window shards (world 3) encoded by tcs_mebcrs_encode_shard are the
//      matching slices of the whole-matrix encode, and their SpMMs,
//      concatenated, equal the whole-matrix tcs_spmm bit for bit;
//   4. tcs_spmm_sharded (B broadcast + grouped-broadcast exchange of C) ==
//      tcs_spmm;
//   5. error taxonomy: ARGUMENT for bad arguments, NCCL for a NULL/aborted
//      communicator, and a forced timeout aborts the communicator.
//
// One process holds every rank of the communicator (ncclCommInitAll over
// the visible GPUs: 1 on the test box, 8 on an HGX box).  Ranks beyond the
// first would need one thread each; the shard arithmetic of a world of N is
// exercised by (2)-(3) on any GPU count.
//
// Built by oracle/Makefile where the reference headers exist into
// oracle/_ref/dist_gpu (links libtcsparse_b200.so and libnccl); run on the
// GPU box by tests/test_gpu_dist_capi.py.
// ============================================================================
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tcsparse/gpu.hpp"
#include "tcsparse/tcsparse.hpp"

using namespace tcsparse;

namespace {

int failures = 0;
void report(const char* name, bool ok) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", name);
    if (!ok) ++failures;
}

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(2);                                                           \
        }                                                                           \
    } while (0)

template <typename T>
T* dup(const std::vector<T>& h) {
    T* d = nullptr;
    CK(cudaMalloc(&d, std::max<size_t>(1, h.size()) * sizeof(T)));
    if (!h.empty()) CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}
template <typename T>
std::vector<T> back(const T* d, size_t n) {
    std::vector<T> h(n);
    if (n) CK(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
    return h;
}

std::vector<uint64_t> rule_cuts(const CsrMatrix& m, int world) {
    const uint64_t W = (m.rows + 7) / 8, nnz = m.nnz();
    std::vector<uint64_t> c(world + 1);
    c[world] = W;
    for (int r = 1; r < world; ++r) {
        const uint64_t target = nnz * r / world;
        uint64_t w = 0;
        while (w < W && m.row_ptr[std::min<uint64_t>(8 * w, m.rows)] < target) ++w;
        c[r] = w;
    }
    return c;
}

bool bits_equal(const std::vector<float>& a, const std::vector<float>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0;
}

}  // namespace

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 1) {
        std::printf("no CUDA device\n");
        return 2;
    }
    ncclComm_t comm;
    int dev0 = 0;
    if (ncclCommInitAll(&comm, 1, &dev0) != ncclSuccess) {
        std::printf("ncclCommInitAll failed\n");
        return 2;
    }
    CK(cudaSetDevice(0));

    // 1. the drop-in overload against the reference
    {
        bool ok = true;
        for (int seed = 0; seed < 3 && ok; ++seed) {
            const CsrMatrix m = generate_random_sparse(517 + 64 * seed, 389 + 32 * seed, 0.02 + 0.03 * seed, 40 + seed);
            const DenseMatrix b = generate_random_dense(m.cols, 96 + 16 * seed, 50 + seed);
            for (Precision p : {Precision::fp16, Precision::tf32}) {
                const KernelConfig cfg{p, 8, ThreadMapping::coalesced};
                const SpmmResult want = spmm(encode_mebcrs(m, p), b, cfg);
                const SpmmResult got = gpu::spmm_sharded(m, b, cfg, comm, 0, 60000);
                ok = ok && got.output == want.output && got.counters.mma_invocations == want.counters.mma_invocations;
            }
        }
        report("spmm_sharded (NCCL comm) == reference spmm, bit-exact, FP16 + TF32", ok);
    }

    // a larger matrix with long windows for the C-ABI checks
    const CsrMatrix m = generate_random_sparse(2003, 1500, 0.05, 77);
    const DenseMatrix b = generate_random_dense(m.cols, 128, 78);
    const uint64_t rows = m.rows, cols = m.cols, n = 128;
    uint32_t* d_rp = dup(m.row_ptr);
    uint32_t* d_ci = dup(m.col_idx);
    float* d_v = dup(m.values);
    const tcs_csr dcsr{rows, cols, m.nnz(), d_rp, d_ci, d_v};
    std::vector<__half> bh(b.data.size());
    for (size_t i = 0; i < bh.size(); ++i) bh[i] = __float2half_rn(b.data[i]);
    __half* d_b = dup(bh);
    float* d_c = nullptr;
    CK(cudaMalloc(&d_c, rows * n * 4));
    const tcs_kernel_config kc{TCS_FP16, 8, TCS_MAP_COALESCED, 0};
    tcs_mebcrs whole{};
    bool enc_ok = tcs_mebcrs_encode(&dcsr, TCS_FP16, TCS_DTYPE_F16, &whole, nullptr) == TCS_OK;
    enc_ok = enc_ok && tcs_spmm(&whole, d_b, TCS_DTYPE_F16, n, cols, n, d_c, n, &kc, nullptr, nullptr) == TCS_OK;
    const std::vector<float> c_whole = back(d_c, rows * n);
    const auto rp_whole = back(whole.row_pointers, whole.num_windows + 1);
    const auto ci_whole = back(whole.column_indices, whole.num_vectors);
    const auto v_whole = back(static_cast<const __half*>(whole.values), 8 * whole.num_vectors);
    report("whole-matrix encode + spmm", enc_ok);

    // 2. cut rule
    {
        bool ok = true;
        for (int world = 1; world <= 8; ++world) {
            std::vector<uint64_t> cuts(world + 1);
            ok = ok && tcs_shard_windows(&dcsr, world, cuts.data(), nullptr) == TCS_OK && cuts == rule_cuts(m, world);
        }
        report("tcs_shard_windows == nnz-balanced rule, world 1..8", ok);
    }

    // 3. shards: slices of the whole encode, concatenated SpMM == whole SpMM
    {
        const int world = 3;
        std::vector<uint64_t> cuts(world + 1);
        bool ok = tcs_shard_windows(&dcsr, world, cuts.data(), nullptr) == TCS_OK;
        std::vector<float> c_cat;
        for (int r = 0; r < world && ok; ++r) {
            tcs_mebcrs sh{};
            ok = tcs_mebcrs_encode_shard(&dcsr, cuts[r], cuts[r + 1], TCS_FP16, TCS_DTYPE_F16, &sh, nullptr) == TCS_OK;
            if (!ok) break;
            const auto rp = back(sh.row_pointers, sh.num_windows + 1);
            const auto ci = back(sh.column_indices, sh.num_vectors);
            const auto v = back(static_cast<const __half*>(sh.values), 8 * sh.num_vectors);
            const uint32_t base = rp_whole[cuts[r]];
            for (size_t w = 0; w < rp.size(); ++w) ok = ok && rp[w] == rp_whole[cuts[r] + w] - base;
            ok = ok && std::memcmp(ci.data(), ci_whole.data() + base, ci.size() * 4) == 0;
            ok = ok && std::memcmp(v.data(), v_whole.data() + 8ull * base, v.size() * 2) == 0;
            float* d_cs = nullptr;
            CK(cudaMalloc(&d_cs, std::max<uint64_t>(1, sh.rows) * n * 4));
            ok = ok && tcs_spmm(&sh, d_b, TCS_DTYPE_F16, n, cols, n, d_cs, n, &kc, nullptr, nullptr) == TCS_OK;
            const auto part = back(d_cs, sh.rows * n);
            c_cat.insert(c_cat.end(), part.begin(), part.end());
            CK(cudaFree(d_cs));
            tcs_mebcrs_free(&sh, nullptr);
        }
        report("world-3 shards: encode slices bit-identical, concatenated SpMM == whole SpMM", ok && bits_equal(c_cat, c_whole));
    }

    // 4. tcs_spmm_sharded on the communicator
    tcs_dist d{};
    {
        bool ok = tcs_dist_init(&d, comm, 30000) == TCS_OK && d.world == 1 && d.rank == 0;
        std::vector<uint64_t> cuts(d.world + 1);
        ok = ok && tcs_shard_windows(&dcsr, d.world, cuts.data(), nullptr) == TCS_OK;
        tcs_mebcrs sh{};
        ok = ok && tcs_mebcrs_encode_shard(&dcsr, cuts[d.rank], cuts[d.rank + 1], TCS_FP16, TCS_DTYPE_F16, &sh, nullptr) == TCS_OK;
        CK(cudaMemset(d_c, 0xff, rows * n * 4));
        ok = ok && tcs_spmm_sharded(&d, cuts.data(), rows, &sh, d_b, TCS_DTYPE_F16, n, cols, n, 0,
                                    TCS_DIST_BROADCAST_B | TCS_DIST_ALLGATHER_C, d_c, n, &kc, nullptr, nullptr) == TCS_OK;
        report("tcs_spmm_sharded (broadcast B, exchange C) == tcs_spmm", ok && bits_equal(back(d_c, rows * n), c_whole));
        // errors
        std::vector<uint64_t> bad = cuts;
        bad[d.world] += 1;
        bool e_ok = tcs_spmm_sharded(&d, bad.data(), rows, &sh, d_b, TCS_DTYPE_F16, n, cols, n, 0, 0, d_c, n, &kc,
                                     nullptr, nullptr) == TCS_ERR_ARGUMENT;
        e_ok = e_ok && tcs_spmm_sharded(&d, cuts.data(), rows, &sh, d_b, TCS_DTYPE_F16, n, cols, n, 5, 0, d_c, n, &kc,
                                        nullptr, nullptr) == TCS_ERR_ARGUMENT;
        tcs_dist dnull = d;
        dnull.comm = nullptr;
        e_ok = e_ok && tcs_dist_broadcast(&dnull, d_b, 16, 0, nullptr) == TCS_ERR_NCCL;
        e_ok = e_ok && tcs_dist_init(&dnull, nullptr, 0) == TCS_ERR_ARGUMENT;
        e_ok = e_ok && tcs_dist_wait(&d, nullptr, 1000) == TCS_OK;
        report("error taxonomy (ARGUMENT / NCCL) and an idle wait", e_ok);
        tcs_mebcrs_free(&sh, nullptr);
    }

    // 5. a wait that cannot finish in time aborts the communicator
    {
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        // a long chain of SpMMs keeps the stream busy past a 1 ms timeout
        for (int i = 0; i < 400; ++i)
            tcs_spmm(&whole, d_b, TCS_DTYPE_F16, n, cols, n, d_c, n, &kc, nullptr, reinterpret_cast<tcs_stream_t>(s));
        const tcs_status rc = tcs_dist_wait(&d, reinterpret_cast<tcs_stream_t>(s), 1);
        const bool ok = (rc == TCS_ERR_NCCL && d.comm == nullptr) || rc == TCS_OK;  // OK only if the GPU outran 1 ms
        report("timeout -> TCS_ERR_NCCL + ncclCommAbort (comm cleared)", ok);
        CK(cudaStreamSynchronize(s));
        CK(cudaStreamDestroy(s));
        if (rc == TCS_OK) ncclCommDestroy(comm);
    }

    tcs_mebcrs_free(&whole, nullptr);
    CK(cudaFree(d_rp));
    CK(cudaFree(d_ci));
    CK(cudaFree(d_v));
    CK(cudaFree(d_b));
    CK(cudaFree(d_c));
    if (failures) {
        std::printf("%d multi-GPU C-ABI check(s) FAILED\n", failures);
        return 1;
    }
    std::printf("all multi-GPU C-ABI checks passed\n");
    return 0;
}
