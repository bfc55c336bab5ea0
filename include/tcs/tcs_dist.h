/*
 * tcs_dist.h -- multi-GPU layer of the B200 FlashSparse hot path (C-ABI).
 *
 * One process per GPU.  The unit of work is the 8-row window: windows own
 * disjoint output rows (ref SPEC.md:364), so SpMM / SDDMM shard into
 * contiguous window ranges with no data-path collective.  The dense operand
 * B is broadcast once from its owner; the output shards stay local unless
 * the caller asks for the whole C on every rank (layers that chain).
 *
 * The reference has no communication layer (it is a single-threaded CPU
 * library); these entry points extend its API for the north star's 8-GPU
 * box.  The communicator is the caller's NCCL communicator (`ncclComm_t`,
 * passed as void*: e.g. the one torch.distributed created,
 * ProcessGroupNCCL._comm_ptr()).  libnccl.so.2 is resolved at run time
 * (dlopen) on the first call, so the library loads without NCCL.
 *
 * Failure handling: collectives are stream-ordered.  With timeout_ms > 0,
 * the sharded calls wait for their stream, polling ncclCommGetAsyncError;
 * an asynchronous NCCL error or the timeout aborts the communicator
 * (ncclCommAbort) and returns TCS_ERR_NCCL -- a dead peer cannot hang the
 * caller.  With timeout_ms == 0 they return as soon as the work is queued
 * and tcs_dist_wait does the polling.
 */
#ifndef TCS_TCS_DIST_H_
#define TCS_TCS_DIST_H_

#include "tcs/tcs.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tcs_dist {
    void* comm;         /* ncclComm_t; NULL once aborted                     */
    int rank;           /* this process's rank in comm (tcs_dist_init)      */
    int world;          /* ranks in comm                                    */
    int64_t timeout_ms; /* > 0: sharded calls wait and poll (see above)     */
} tcs_dist;

/* Binds a communicator: reads its rank and size.  ARGUMENT for a NULL
 * comm; NCCL when libnccl.so.2 cannot be loaded or the comm is invalid. */
tcs_status tcs_dist_init(tcs_dist* d, void* nccl_comm, int64_t timeout_ms);

/* Contiguous window ranges balanced by nnz (the north star's criterion):
 * cuts[0] = 0 <= cuts[1] <= ... <= cuts[world] = ceil(rows / 8); shard r
 * owns windows [cuts[r], cuts[r+1]), i.e. rows [8 cuts[r], min(8 cuts[r+1],
 * rows)).  cuts[r] is the first window whose starting nnz offset reaches
 * r * nnz / world.  csr is a DEVICE CSR; cuts is a host array of world + 1.
 * Synchronises. */
tcs_status tcs_shard_windows(const tcs_csr* csr, int world, uint64_t* cuts, tcs_stream_t stream);

/* CSR -> ME-BCRS of the rows of windows [w_begin, w_end) of a device CSR:
 * a standalone handle (row_pointers from 0, global column indices, so it
 * multiplies the whole B).  Its arrays equal the matching slice of
 * tcs_mebcrs_encode on the whole matrix bit for bit (row pointers rebased). */
tcs_status tcs_mebcrs_encode_shard(const tcs_csr* csr, uint64_t w_begin, uint64_t w_end, tcs_precision precision,
                                   tcs_dtype value_dtype, tcs_mebcrs* out, tcs_stream_t stream);

/* In-place broadcast of `bytes` bytes of device memory from `root`. */
tcs_status tcs_dist_broadcast(tcs_dist* d, void* buf, uint64_t bytes, int root, tcs_stream_t stream);

#define TCS_DIST_BROADCAST_B 0x1u /* broadcast b (b_rows x ldb elements) from root first   */
#define TCS_DIST_ALLGATHER_C 0x2u /* c is the whole [rows_total x n] output (ldc == n) on  */
                                  /* every rank: the shard computes its rows in place and  */
                                  /* the shards are exchanged (grouped broadcasts)          */

/* Sharded SpMM (ref spmm, spmm.hpp:173, over a row-window shard): this
 * rank's rows C[8 cuts[rank] ...] = A_shard * B, where a_shard came from
 * tcs_mebcrs_encode_shard(csr, cuts[rank], cuts[rank+1], ...).  cuts has
 * d->world + 1 entries (tcs_shard_windows); rows_total is the whole
 * matrix's row count.  Without TCS_DIST_ALLGATHER_C, c is the shard's own
 * [a_shard->rows x n] output (stride ldc).  Arguments, errors and counters
 * as tcs_spmm (the counters are the shard's); NCCL failures -> TCS_ERR_NCCL. */
tcs_status tcs_spmm_sharded(tcs_dist* d, const uint64_t* cuts, uint64_t rows_total, const tcs_mebcrs* a_shard,
                            void* b, tcs_dtype b_dtype, int64_t ldb, int64_t b_rows, int64_t n, int root,
                            uint32_t dist_flags, float* c, int64_t ldc, const tcs_kernel_config* cfg,
                            tcs_counters* counters, tcs_stream_t stream);

/* The multi-GPU form of tcs_spmm_csr_host (host buffers, value semantics):
 * every rank passes the same host CSR; rank `root` passes the host f32 B
 * [cols x n] (other ranks may pass NULL).  The windows are cut by nnz
 * (tcs_shard_windows' rule), each rank uploads and converts only its own
 * rows, B is broadcast from root, the shards are multiplied, exchanged, and
 * every rank receives the whole C [rows x n] (host f32).  Waits for
 * completion with the communicator's timeout (d->timeout_ms, or 60 s if
 * it is 0).  counters are this rank's shard's. */
tcs_status tcs_spmm_sharded_csr_host(tcs_dist* d, const tcs_csr* host_csr, tcs_precision precision, const float* b,
                                     int64_t n, int root, float* c, const tcs_kernel_config* cfg,
                                     tcs_counters* counters, tcs_stream_t stream);

/* Waits for `stream`, polling ncclCommGetAsyncError every ~100 us.  On an
 * NCCL error, or when timeout_ms (> 0) elapses first, aborts the
 * communicator (ncclCommAbort; d->comm becomes NULL) and returns
 * TCS_ERR_NCCL.  timeout_ms <= 0 waits without limit. */
tcs_status tcs_dist_wait(tcs_dist* d, tcs_stream_t stream, int64_t timeout_ms);

#ifdef __cplusplus
}
#endif

#endif /* TCS_TCS_DIST_H_ */
