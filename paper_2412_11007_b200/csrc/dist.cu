// Multi-GPU layer (include/tcs/tcs_dist.h): row-window shards balanced by
// nnz, B broadcast from its owner, optional exchange of the output shards,
// all over the caller's NCCL communicator.  NCCL is resolved with dlopen on
// first use; every collective is stream-ordered and, with a timeout, waited
// on with ncclCommGetAsyncError polling and ncclCommAbort on failure.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include "tcs/tcs_dist.h"
#include "tcs_internal.cuh"

namespace tcs {
namespace {

// ------------------------------------------------------------ NCCL symbols
struct Nccl {
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string load_error;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // the process may already hold a libnccl.so.2 (torch's): dlopen
        // returns that one, so both sides share one NCCL
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            n.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && n.load_error.empty()) n.load_error = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(n.CommCount, "ncclCommCount");
        sym(n.CommUserRank, "ncclCommUserRank");
        sym(n.Broadcast, "ncclBroadcast");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        sym(n.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(n.CommAbort, "ncclCommAbort");
        sym(n.GetErrorString, "ncclGetErrorString");
    });
    if (!n.load_error.empty()) fail(TCS_ERR_NCCL, n.load_error);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress)
        fail(TCS_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

ncclComm_t comm_of(const tcs_dist* d) {
    if (!d) fail(TCS_ERR_ARGUMENT, "null tcs_dist");
    if (!d->comm) fail(TCS_ERR_NCCL, "communicator is NULL (never bound, or aborted after an NCCL failure)");
    return static_cast<ncclComm_t>(d->comm);
}

void wait_impl(tcs_dist* d, cudaStream_t s, int64_t timeout_ms) {
    const Nccl& nc = nccl();
    ncclComm_t comm = comm_of(d);
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        ncclResult_t async = ncclSuccess;
        nccl_check(nc.CommGetAsyncError(comm, &async), "ncclCommGetAsyncError");
        if (async != ncclSuccess && async != ncclInProgress) {
            nc.CommAbort(comm);
            d->comm = nullptr;
            fail(TCS_ERR_NCCL, std::string("asynchronous NCCL error, communicator aborted: ") +
                                   nc.GetErrorString(async));
        }
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) TCS_CUDA(q);
        const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
        if (timeout_ms > 0 && ms.count() > timeout_ms) {
            nc.CommAbort(comm);
            d->comm = nullptr;
            fail(TCS_ERR_NCCL, "collective did not complete within " + std::to_string(timeout_ms) +
                                   " ms; communicator aborted");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
}

// ---------------------------------------------------------- shard cuts
// cuts[r] = first window w with rp[min(8w, rows)] >= r * nnz / world
// (lower bound over the window-start nnz offsets; monotone in r).
__global__ void shard_cuts_kernel(const uint32_t* __restrict__ rp, uint64_t rows, uint64_t W, int world,
                                  uint64_t* __restrict__ cuts) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > world) return;
    if (r == 0) { cuts[0] = 0; return; }
    if (r == world) { cuts[world] = W; return; }
    const uint64_t nnz = rp[rows];
    const uint64_t target = nnz * static_cast<uint64_t>(r) / static_cast<uint64_t>(world);
    uint64_t lo = 0, hi = W;  // first w in [0, W] with start(w) >= target
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (rp[std::min<uint64_t>(8 * mid, rows)] < target) lo = mid + 1;
        else hi = mid;
    }
    cuts[r] = lo;
}

// The same cut rule on a host row_ptr.
void host_cuts(const uint32_t* rp, uint64_t rows, int world, uint64_t* cuts) {
    const uint64_t W = (rows + 7) / 8, nnz = rp[rows];
    cuts[0] = 0;
    cuts[world] = W;
    for (int r = 1; r < world; ++r) {
        const uint64_t target = nnz * static_cast<uint64_t>(r) / static_cast<uint64_t>(world);
        uint64_t lo = 0, hi = W;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (rp[std::min<uint64_t>(8 * mid, rows)] < target) lo = mid + 1;
            else hi = mid;
        }
        cuts[r] = lo;
    }
}

__global__ void rebase_rows_kernel(const uint32_t* __restrict__ rp, uint64_t r0, uint64_t n, uint32_t* __restrict__ out) {
    const uint32_t base = rp[r0];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = rp[r0 + i] - base;
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_dist_init(tcs_dist* d, void* nccl_comm, int64_t timeout_ms) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_dist_init");
        if (!d || !nccl_comm) fail(TCS_ERR_ARGUMENT, "null tcs_dist or communicator");
        const Nccl& nc = nccl();
        ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
        int rank = -1, world = 0;
        nccl_check(nc.CommUserRank(comm, &rank), "ncclCommUserRank");
        nccl_check(nc.CommCount(comm, &world), "ncclCommCount");
        *d = tcs_dist{nccl_comm, rank, world, timeout_ms};
    });
}

extern "C" tcs_status tcs_shard_windows(const tcs_csr* csr, int world, uint64_t* cuts, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_shard_windows");
        if (!csr || !cuts || !csr->row_ptr) fail(TCS_ERR_ARGUMENT, "null argument");
        if (world < 1) fail(TCS_ERR_ARGUMENT, "world must be >= 1");
        cudaStream_t s = st(stream);
        const uint64_t W = (csr->rows + 7) / 8;
        DBuf d(sizeof(uint64_t) * (world + 1), s);
        shard_cuts_kernel<<<(world + 128) / 128, 128, 0, s>>>(csr->row_ptr, csr->rows, W, world, d.as<uint64_t>());
        TCS_LAUNCHED("shard_cuts");
        TCS_CUDA(cudaMemcpyAsync(cuts, d.p, sizeof(uint64_t) * (world + 1), cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
    });
}

extern "C" tcs_status tcs_mebcrs_encode_shard(const tcs_csr* csr, uint64_t w_begin, uint64_t w_end,
                                              tcs_precision precision, tcs_dtype value_dtype, tcs_mebcrs* out,
                                              tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_mebcrs_encode_shard");
        if (!csr || !out || !csr->row_ptr) fail(TCS_ERR_ARGUMENT, "null argument");
        const uint64_t W = (csr->rows + 7) / 8;
        if (w_begin > w_end || w_end > W) fail(TCS_ERR_ARGUMENT, "window range out of bounds");
        cudaStream_t s = st(stream);
        const uint64_t r0 = std::min<uint64_t>(8 * w_begin, csr->rows), r1 = std::min<uint64_t>(8 * w_end, csr->rows);
        uint32_t ends[2] = {0, 0};
        TCS_CUDA(cudaMemcpyAsync(&ends[0], csr->row_ptr + r0, 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaMemcpyAsync(&ends[1], csr->row_ptr + r1, 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
        if (ends[1] < ends[0]) fail(TCS_ERR_FORMAT, "row_ptr must be nondecreasing");
        DBuf rp((r1 - r0 + 1) * 4, s);
        const int grid = static_cast<int>(std::min<uint64_t>((r1 - r0 + 256) / 256, uint64_t(num_sms()) * 8));
        rebase_rows_kernel<<<grid, 256, 0, s>>>(csr->row_ptr, r0, r1 - r0, rp.as<uint32_t>());
        TCS_LAUNCHED("rebase_rows");
        tcs_csr part{r1 - r0, csr->cols, uint64_t(ends[1] - ends[0]), rp.as<uint32_t>(),
                     csr->col_idx ? csr->col_idx + ends[0] : nullptr, csr->values ? csr->values + ends[0] : nullptr};
        const tcs_status rc = tcs_mebcrs_encode(&part, precision, value_dtype, out, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
    });
}

extern "C" tcs_status tcs_dist_broadcast(tcs_dist* d, void* buf, uint64_t bytes, int root, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_dist_broadcast");
        ncclComm_t comm = comm_of(d);
        if (root < 0 || root >= d->world) fail(TCS_ERR_ARGUMENT, "root out of range");
        if (bytes && !buf) fail(TCS_ERR_ARGUMENT, "null buffer");
        cudaStream_t s = st(stream);
        if (bytes) nccl_check(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, comm, s), "ncclBroadcast");
        if (d->timeout_ms > 0) wait_impl(d, s, d->timeout_ms);
    });
}

extern "C" tcs_status tcs_spmm_sharded(tcs_dist* d, const uint64_t* cuts, uint64_t rows_total,
                                       const tcs_mebcrs* a_shard, void* b, tcs_dtype b_dtype, int64_t ldb,
                                       int64_t b_rows, int64_t n, int root, uint32_t dist_flags, float* c,
                                       int64_t ldc, const tcs_kernel_config* cfg, tcs_counters* counters,
                                       tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_sharded");
        ncclComm_t comm = comm_of(d);
        const Nccl& nc = nccl();
        if (!cuts || !a_shard) fail(TCS_ERR_ARGUMENT, "null argument");
        if (root < 0 || root >= d->world) fail(TCS_ERR_ARGUMENT, "root out of range");
        const uint64_t W = (rows_total + 7) / 8;
        if (cuts[0] != 0 || cuts[d->world] != W) fail(TCS_ERR_ARGUMENT, "cuts must span windows [0, ceil(rows/8))");
        for (int r = 0; r < d->world; ++r)
            if (cuts[r] > cuts[r + 1]) fail(TCS_ERR_ARGUMENT, "cuts must be nondecreasing");
        auto row_of = [&](uint64_t w) { return std::min<uint64_t>(8 * w, rows_total); };
        const uint64_t r0 = row_of(cuts[d->rank]), r1 = row_of(cuts[d->rank + 1]);
        if (a_shard->rows != r1 - r0) fail(TCS_ERR_SHAPE, "shard rows do not match cuts[rank]..cuts[rank+1]");
        const bool gather = dist_flags & TCS_DIST_ALLGATHER_C;
        if (gather && ldc != n) fail(TCS_ERR_ARGUMENT, "ALLGATHER_C needs a dense [rows_total x n] output (ldc == n)");
        cudaStream_t s = st(stream);
        if ((dist_flags & TCS_DIST_BROADCAST_B) && b_rows > 0 && n > 0) {
            if (!b) fail(TCS_ERR_ARGUMENT, "null dense buffer");
            const uint64_t bytes = uint64_t(b_rows) * uint64_t(ldb) * (b_dtype == TCS_DTYPE_F16 ? 2 : 4);
            nccl_check(nc.Broadcast(b, b, bytes, ncclUint8, root, comm, s), "ncclBroadcast(B)");
        }
        float* c_own = gather ? c + r0 * uint64_t(n) : c;
        const tcs_status rc = tcs_spmm(a_shard, b, b_dtype, ldb, b_rows, n, c_own, ldc, cfg, counters, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        if (gather && n > 0) {
            // variable-size all-gather: one broadcast per owner, grouped (each
            // shard's rows are contiguous in the row-major output)
            nccl_check(nc.GroupStart(), "ncclGroupStart");
            for (int r = 0; r < d->world; ++r) {
                const uint64_t a0 = row_of(cuts[r]), a1 = row_of(cuts[r + 1]);
                if (a1 > a0) {
                    float* p = c + a0 * uint64_t(n);
                    nccl_check(nc.Broadcast(p, p, (a1 - a0) * uint64_t(n), ncclFloat32, r, comm, s), "ncclBroadcast(C)");
                }
            }
            nccl_check(nc.GroupEnd(), "ncclGroupEnd");
        }
        if (d->timeout_ms > 0) wait_impl(d, s, d->timeout_ms);
    });
}

extern "C" tcs_status tcs_spmm_sharded_csr_host(tcs_dist* d, const tcs_csr* host_csr, tcs_precision precision,
                                                const float* b, int64_t n, int root, float* c,
                                                const tcs_kernel_config* cfg, tcs_counters* counters,
                                                tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_sharded_csr_host");
        comm_of(d);
        if (!host_csr || !host_csr->row_ptr || !cfg) fail(TCS_ERR_ARGUMENT, "null argument");
        if (root < 0 || root >= d->world) fail(TCS_ERR_ARGUMENT, "root out of range");
        if (n < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        if (n > 0 && host_csr->rows > 0 && !c) fail(TCS_ERR_ARGUMENT, "null output buffer");
        if (d->rank == root && n > 0 && host_csr->cols > 0 && !b) fail(TCS_ERR_ARGUMENT, "null dense buffer on root");
        cudaStream_t s = st(stream);
        const uint64_t rows = host_csr->rows, cols = host_csr->cols;
        std::vector<uint64_t> cuts(d->world + 1);
        host_cuts(host_csr->row_ptr, rows, d->world, cuts.data());
        const uint64_t r0 = std::min<uint64_t>(8 * cuts[d->rank], rows);
        const uint64_t r1 = std::min<uint64_t>(8 * cuts[d->rank + 1], rows);
        const uint32_t e0 = host_csr->row_ptr[r0], e1 = host_csr->row_ptr[r1];
        if (e1 < e0) fail(TCS_ERR_FORMAT, "row_ptr must be nondecreasing");
        // this rank's rows only: rebased row_ptr, entries [e0, e1)
        std::vector<uint32_t> rp(r1 - r0 + 1);
        for (uint64_t i = 0; i <= r1 - r0; ++i) rp[i] = host_csr->row_ptr[r0 + i] - e0;
        const tcs_csr part{r1 - r0, cols, uint64_t(e1 - e0), rp.data(), host_csr->col_idx + e0,
                           host_csr->values + e0};
        tcs_mebcrs a{};
        tcs_status rc = tcs_mebcrs_encode_host(&part, precision, TCS_DTYPE_F32, &a, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        struct Free {
            tcs_mebcrs* a;
            tcs_stream_t s;
            ~Free() { tcs_mebcrs_free(a, s); }
        } free_a{&a, stream};
        DBuf db(std::max<uint64_t>(1, cols * uint64_t(n)) * 4, s), dc(std::max<uint64_t>(1, rows * uint64_t(n)) * 4, s);
        if (d->rank == root && cols && n)
            TCS_CUDA(cudaMemcpyAsync(db.p, b, cols * uint64_t(n) * 4, cudaMemcpyHostToDevice, s));
        tcs_dist dw = *d;
        dw.timeout_ms = 0;  // one wait below, over the whole call
        rc = tcs_spmm_sharded(&dw, cuts.data(), rows, &a, db.p, TCS_DTYPE_F32, n, static_cast<int64_t>(cols), n, root,
                              TCS_DIST_BROADCAST_B | TCS_DIST_ALLGATHER_C, dc.as<float>(), n, cfg, counters, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        if (rows && n) TCS_CUDA(cudaMemcpyAsync(c, dc.p, rows * uint64_t(n) * 4, cudaMemcpyDeviceToHost, s));
        wait_impl(d, s, d->timeout_ms > 0 ? d->timeout_ms : 60000);
    });
}

extern "C" tcs_status tcs_dist_wait(tcs_dist* d, tcs_stream_t stream, int64_t timeout_ms) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_dist_wait"); wait_impl(d, st(stream), timeout_ms); });
}
