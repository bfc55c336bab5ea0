// SpMM C = A_sparse * B over ME-BCRS with the FlashSparse 8x1
// swap-and-transpose strategy (ref spmm.hpp:103-177, mma.hpp:67-73):
//
//   C^T (features x 8 window rows) += B_gathered^T (features x vectors)
//                                     * A_block^T (vectors x 8 rows)
//
// so the 8-row sparse vectors are the n=8 MMA operand and the dense
// features fill m=16.  One warp owns one work item (<= plan.seg vectors of
// one window) and one feature slab (128/64/32 features).
//
// FP16: mma.sync.m16n8k16 consumes TWO reference k=8 blocks per instruction
// (storage k stays the reference k, instruction k=16).
// TF32: mma.sync.m16n8k8 consumes two k=4 blocks; operands are rounded
// RNE with cvt.rn.tf32.f32 (ref precision.hpp:42-46).
//
// Memory-efficient coalesced mapping (paper §3.3): the MMA's m dimension
// (features) is permuted so that lane (g = lane/4) owns FPL consecutive
// features of each gathered row: ONE 128-bit load per (lane, vector, chunk)
// feeds FPL/2 MMAs, 8 lanes cover 128 contiguous bytes of a B row, and the
// same permutation gives 128-bit fp32 stores of C.  The two vectors that
// share an A register (k = 2t, 2t+1) are packed with PRMT.
//
// Residue (ref spmm.hpp:40-45, paper §3.5): vector slots at or past the
// window's nv_w contribute zero registers and no loads are issued.
// Windows longer than plan.seg are split; partial sums are reduced in
// segment order by spmm_reduce_split (deterministic, no atomics).
#include <algorithm>
#include <cstring>
#include <memory>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

using namespace dev;

struct SpmmArgs {
    const WorkItem* items;
    uint64_t n_items;
    const uint32_t* rp;
    const uint32_t* ci;
    const void* vals;
    const void* B;   // feature-padded, 16-byte aligned rows
    int64_t ldb;
    float* C;
    int64_t ldc;
    uint64_t rows;
    int64_t N;
    float* partial;  // [slot][8][ldp]
    int64_t ldp;
    uint32_t* counter;  // per-slab claim counters, dev::kClaimBytes each (zeroed before launch)
    uint32_t slab0;     // first feature slab of this launch (slab = slab0 + blockIdx.y)
    // Softmax operand (SMX kernels, the AGNN aggregation): the sparse values
    // are binary16 scores x with dead slots -inf, and each is replaced by
    // exp(scale*x - m_r) * inv_r of its row r before the MMA -- the row
    // softmax of softmax.cu applied in registers instead of in memory.
    const float2* rowstat;  // per row (m, 1/sum), 8 * num_windows entries
    float scale;
};

// One binary16 score -> its softmax value, rounded as softmax.cu stores it
// (row_write: z = live ? scale*x : -inf; __expf(z - m) * inv; RNE to f16).
__device__ __forceinline__ uint32_t smx_h(uint32_t h, float scale, float m, float inv) {
    const float x = __half2float(__ushort_as_half(static_cast<unsigned short>(h)));
    const float z = x != -INFINITY ? scale * x : -INFINITY;
    return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(__expf(z - m) * inv)));
}
__device__ __forceinline__ uint32_t smx_h2(uint32_t w, float scale, float m, float inv) {
    return smx_h(w & 0xFFFFu, scale, m, inv) | (smx_h(w >> 16, scale, m, inv) << 16);
}
constexpr uint32_t kHalfNegInf = 0xFC00u;

constexpr int kWarps = 4;
// Resident CTAs per SM.  Narrow slabs (32 features: 64-byte gathers, few
// registers) need more warps in flight to cover DRAM-latency gathers when
// B does not fit in L2 (C5: 537 MB of B).
#ifndef TCS_SPMM_BPS_WIDE
#define TCS_SPMM_BPS_WIDE 8
#endif
constexpr int spmm_blocks(int nchunk, int fpl) { return nchunk * fpl <= 4 ? 8 : nchunk * fpl <= 8 ? TCS_SPMM_BPS_WIDE : 4; }
#ifndef TCS_SPMM_TF32_BPS_NARROW
#define TCS_SPMM_TF32_BPS_NARROW 8
#endif
#ifndef TCS_SPMM_TF32_BPS_WIDE
#define TCS_SPMM_TF32_BPS_WIDE 4
#endif
constexpr int tf32_blocks(int nchunk) { return nchunk <= 2 ? TCS_SPMM_TF32_BPS_NARROW : TCS_SPMM_TF32_BPS_WIDE; }
// Host pipeline of tcs_spmm_csr_host: at most this many equal window-range
// units (each of at least TCS_E2E_CHUNK_NNZ entries), the last one cut into
// halves TCS_E2E_TAIL_HALVINGS times.  Every chunk is two uploads (column
// indices, values) with ~12 us of copy overhead each, while only the last
// chunk's encode + SpMM + download is exposed after the last upload: few
// large units plus a geometric tail (4 + 6: 10 chunks) measured best
// (profiles/r2_e2e.txt).
#ifndef TCS_E2E_MAX_CHUNKS
#define TCS_E2E_MAX_CHUNKS 4
#endif
#ifndef TCS_E2E_DRAIN_LATE
#define TCS_E2E_DRAIN_LATE 0
#endif
#ifndef TCS_E2E_TAIL_HALVINGS
#define TCS_E2E_TAIL_HALVINGS 6
#endif
#ifndef TCS_E2E_CHUNK_NNZ
#define TCS_E2E_CHUNK_NNZ (1ull << 20)
#endif
#ifndef TCS_SPMM_DEEP32
#define TCS_SPMM_DEEP32 1
#endif
// TF32 SpMM on the 2.5-byte packed dense operand (spmm_tf32p_kernel) for
// feature slabs of 64 / 128; 0 = the f32-gather kernel everywhere.
#ifndef TCS_TF32_PACKED
#define TCS_TF32_PACKED 1
#endif
// Sparse-value stream of the packed TF32 kernel with an L2 evict-first
// policy (A/B knob).
#ifndef TCS_TF32P_EF
#define TCS_TF32P_EF 0
#endif
// Packed TF32, 128-feature slabs: a lane's two nibble words (chunks 0, 1)
// adjacent, one 8-byte load instead of two 4-byte loads per gathered row.
#ifndef TCS_TF32P_LO64
#define TCS_TF32P_LO64 1
#endif
// Hot-row L2 policy (see col_hot below; measured slower, off by default).
#ifndef TCS_HOT
#define TCS_HOT 0
#endif
// policy of the cold gathers under TCS_HOT: 0 evict_first, 1 evict_normal,
// 2 evict_unchanged
#ifndef TCS_HOT_COLD
#define TCS_HOT_COLD 0
#endif
// The FP16 (128-feature slabs) and packed-TF32 SpMM kernels prefetch the
// sparse-value and column-index streams into L2 this many vectors ahead of
// their loads (PF instances), when the dense operand fits comfortably in L2
// (<= TCS_PREFETCH_MAX_B_MB): the streamed lines then no longer wait on
// DRAM.  With a larger B the extra L2 traffic costs more than it hides
// (C3 N=256: +3-7%).  Measured in profiles/r2_prefetch.txt.
#ifndef TCS_PREFETCH_AHEAD
#define TCS_PREFETCH_AHEAD 64
#endif
#ifndef TCS_PREFETCH_F16
#define TCS_PREFETCH_F16 128
#endif
#ifndef TCS_PREFETCH_MAX_B_MB
#define TCS_PREFETCH_MAX_B_MB 80
#endif
// B-row gathers with L1::no_allocate (A/B knob; 0 = plain ld.global.nc).
#ifndef TCS_GATHER_NA
#define TCS_GATHER_NA 0
#endif
#ifndef TCS_SMALL_SLAB32
#define TCS_SMALL_SLAB32 1
#endif
// Feature slab of the TF32 kernel for N > 64 (experiment knob: 128 or 64).
#ifndef TCS_SPMM_SLAB_TF32
#define TCS_SPMM_SLAB_TF32 128
#endif
#ifndef TCS_SPMM_SLAB_F16
#define TCS_SPMM_SLAB_F16 128
#endif

// ------------------------------------------------------------- scheduling
// Persistent warps: each warp claims work items from its slab's striped
// counters (dev::StripedClaim: atomicAdd by lane 0, broadcast by shuffle)
// until the list is exhausted, so no warp slot idles behind a long item of a
// sibling warp.  Items are ordered longest-first by the planner (split-window
// segments lead); every stripe is a longest-first subsequence.

// Column indices of a 2-step (32-vector) window of the item, one per lane,
// loaded coalesced; slots pick theirs with a shuffle.
__device__ __forceinline__ uint32_t load_colpair(const uint32_t* __restrict__ ci, uint32_t s, uint32_t vend,
                                                 uint32_t lane) {
    return s + lane < vend ? ld_stream_u32(ci + s + lane) : 0u;
}
// HOT kernels read Plan::ci_hot, a copy of the column indices whose bit 31
// marks a hot column (columns are < 2^31; the gather masks it off and picks
// the L2 policy from it).
constexpr uint32_t kColMask = 0x7FFFFFFFu;

// ------------------------------------------------------------- FP16 path
//
// Gather mapping.  Loads are issued "quarter-warp coalesced": in load slot u
// (0..3) the 8 lanes of quarter q = lane/8 read ONE 128-byte segment (FPL
// features per lane) of vector  v(u, q) = 2q + (u & 1) + 8 (u >> 1)  of the
// 16-vector step -- one L1 wavefront per quarter, the pattern that reaches
// ~14 TB/s of L2 gather bandwidth on B200 (tools/gather_bench.cu).  The MMA
// fragment wants lane (g, t) = (lane/4, lane%4) to own vectors 2t, 2t+1,
// 2t+8, 2t+9 (k slots 0..3) at features FPL*g + [0, FPL): exactly what lane
// 8t + g loaded in slot u = k-slot, so one shuffle per register moves the
// data into place and the vector (k) order stays the identity -- the sparse
// fragment is the natural ME-BCRS pair at 8g + 2t.
// f32-stored values (VF32) of the 128-feature kernels stay raw in the step
// and are converted by f16_compute, so the conversion does not wait for the
// value loads at issue time (the TF32 lesson).  The narrower
// VF32 kernels keep converting at issue: two more registers per stage
// spill there.  (A/B knob.)
#ifndef TCS_VF32_DEFER
#define TCS_VF32_DEFER 1
#endif
template <bool VF32, int NCHUNK>
constexpr bool vf32_defer() { return VF32 && NCHUNK == 2 && TCS_VF32_DEFER; }

template <int NCHUNK, int FPL, bool VF32>
struct F16Step {
    static constexpr int NJ = FPL / 2;  // MMAs per chunk == u32 regs per (vector, chunk)
    static constexpr bool kDefer = vf32_defer<VF32, NCHUNK>();
    uint32_t L[4][NCHUNK][NJ];          // loader slots u = 0..3 (vector v(u, lane/8), features FPL*(lane%8))
    uint32_t b[kDefer ? 4 : 2];         // sparse fragment: rows g, vectors {2t,2t+1}, {2t+8,2t+9} (kDefer: raw f32)
};

// Vector held by MMA k slot u (0..3 = k 2t, 2t+1, 2t+8, 2t+9) of lane (g, t).
// Any bijection works if both operands use it; this one makes the sparse
// fragment the natural ME-BCRS pair at 8g + 2t of each k=8 block (placing
// vectors 4t..4t+3 instead, one 8-byte load per lane, measured 1.5% slower).
__device__ __forceinline__ uint32_t kslot_vec(uint32_t u, uint32_t t) { return 2 * t + (u & 1) + 8 * (u >> 1); }
__device__ __forceinline__ uint32_t loader_vec(uint32_t u, uint32_t q) { return kslot_vec(u, q); }

// Sparse fragment of a full 16-vector step: rows g, k slots of lane (g, t).
template <bool VF32>
__device__ __forceinline__ void load_sparse_full(const void* vals, uint64_t vbase, uint32_t s, uint32_t g, uint32_t t,
                                                 uint32_t& b0, uint32_t& b1) {
    const uint64_t off = vbase + 8ull * s + 8 * g + 2 * t;  // rows g, slots 2t..2t+1 of blocks s/8, s/8+1
    if constexpr (VF32) {
        const float* fv = static_cast<const float*>(vals);
        const uint2 x = ld_stream_u64(fv + off), y = ld_stream_u64(fv + off + 64);
        b0 = f2_to_h2(__uint_as_float(x.x), __uint_as_float(x.y));
        b1 = f2_to_h2(__uint_as_float(y.x), __uint_as_float(y.y));
    } else {
        const __half* hv = static_cast<const __half*>(vals);
        b0 = ld_stream_u32(hv + off);
        b1 = ld_stream_u32(hv + off + 64);
    }
}

template <bool VF32>
__device__ __forceinline__ uint32_t f16_val_general(const void* vals, uint64_t vbase, uint32_t nvw, uint32_t v,
                                                    uint32_t g) {
    if (v >= nvw) return 0u;
    const uint32_t b = v >> 3, j = v & 7u, width = min(8u, nvw - 8 * b);
    const uint64_t off = vbase + 64ull * b + g * width + j;
    if constexpr (VF32) {
        return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(static_cast<const float*>(vals)[off])));
    } else {
        return static_cast<uint32_t>(static_cast<const unsigned short*>(vals)[off]);
    }
}

// Issues the gathers + sparse-value loads of the 16-vector step at s.
// colpair holds the column indices of vectors [s - 16*half, +32).
// Sparse fragment (both k=8 blocks) of the 16-vector step at s into b:
// 0 past the item (-inf for a softmax operand, exp(-inf) = 0).
// Raw f32 fragment (kDefer steps): slots of the 16-vector step at s, 0 past the item.
__device__ __forceinline__ void f32_values_raw(const SpmmArgs& a, uint64_t vbase, uint32_t nvw, uint32_t vend,
                                               uint32_t s, uint32_t g, uint32_t t, uint32_t (&b)[4]) {
    const float* fv = static_cast<const float*>(a.vals);
    if (s + 16 <= vend) {
        const uint64_t off = vbase + 8ull * s + 8 * g + 2 * t;
        const uint2 x = ld_stream_u64(fv + off), y = ld_stream_u64(fv + off + 64);
        b[0] = x.x; b[1] = x.y; b[2] = y.x; b[3] = y.y;
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t v = s + kslot_vec(u, t);
            uint32_t x = 0u;
            if (v < vend && v < nvw) {
                const uint32_t blk = v >> 3, j = v & 7u, width = min(8u, nvw - 8 * blk);
                x = __float_as_uint(fv[vbase + 64ull * blk + g * width + j]);
            }
            b[u] = x;
        }
    }
}

template <bool VF32, bool SMX>
__device__ __forceinline__ void f16_values(const SpmmArgs& a, uint64_t vbase, uint32_t nvw, uint32_t vend, uint32_t s,
                                           uint32_t g, uint32_t t, uint32_t (&b)[2]) {
    if (s + 16 <= vend) {
        load_sparse_full<VF32>(a.vals, vbase, s, g, t, b[0], b[1]);
    } else {
        uint32_t e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t v = s + kslot_vec(u, t);
            e[u] = v < vend ? f16_val_general<VF32>(a.vals, vbase, nvw, v, g) : (SMX ? kHalfNegInf : 0u);
        }
        b[0] = e[0] | (e[1] << 16);
        b[1] = e[2] | (e[3] << 16);
    }
}

// Issues the gathers (and, with LOADV, the sparse-value loads) of the
// 16-vector step at s.  colpair holds the column indices of vectors
// [s - 16*half, +32).  (Loading the values two steps ahead instead, with
// their own register pair, measured 7% slower on C3: 2.61 -> 2.80 ms.)
// One gathered segment of a B row (HOT: with the row's L2 policy).
template <int FPL, bool HOT>
__device__ __forceinline__ void f16_gather(const __half* p, uint64_t pol, uint32_t (&dst)[FPL / 2]) {
    if constexpr (FPL == 8) {
        const uint4 x = HOT ? ld_gather_128_pol(p, pol) : TCS_GATHER_NA ? ld_gather_128_na(p) : ld_gather_128(p);
        dst[0] = x.x; dst[1] = x.y; dst[2] = x.z; dst[3] = x.w;
    } else {
        const uint2 x = HOT ? ld_gather_64_pol(p, pol) : ld_gather_64(p);
        dst[0] = x.x; dst[1] = x.y;
    }
}

template <int NCHUNK, int FPL, bool VF32, bool SMX = false, bool LOADV = true, bool HOT = false>
__device__ __forceinline__ void f16_issue(const SpmmArgs& a, const __half* __restrict__ Bl, uint64_t vbase,
                                          uint32_t nvw, uint32_t vend, uint32_t s, uint32_t g, uint32_t t, uint32_t q,
                                          uint32_t colpair, uint32_t half, F16Step<NCHUNK, FPL, VF32>& st,
                                          uint64_t pol_last = 0, uint64_t pol_first = 0) {
    constexpr int CHUNK = 8 * FPL;
    uint32_t col[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) col[u] = __shfl_sync(0xffffffffu, colpair, 16 * half + loader_vec(u, q));
    if (s + 16 <= vend) {
        // full step (warp-uniform): no predicates; both k=8 blocks are full width
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const __half* row = Bl + static_cast<uint64_t>(HOT ? col[u] & kColMask : col[u]) * a.ldb;
            const uint64_t pol = HOT && (col[u] >> 31) ? pol_last : pol_first;
#pragma unroll
            for (int c = 0; c < NCHUNK; ++c) f16_gather<FPL, HOT>(row + c * CHUNK, pol, st.L[u][c]);
        }
        if constexpr (LOADV) {
            if constexpr (F16Step<NCHUNK, FPL, VF32>::kDefer) f32_values_raw(a, vbase, nvw, vend, s, g, t, st.b);
            else load_sparse_full<VF32>(a.vals, vbase, s, g, t, st.b[0], st.b[1]);
        }
    } else {
        // residue step: vectors at or past vend contribute zero registers
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool ok = s + loader_vec(u, q) < vend;
            const __half* row = Bl + static_cast<uint64_t>(HOT ? col[u] & kColMask : col[u]) * a.ldb;
            const uint64_t pol = HOT && (col[u] >> 31) ? pol_last : pol_first;
#pragma unroll
            for (int c = 0; c < NCHUNK; ++c) {
                if (ok) {
                    f16_gather<FPL, HOT>(row + c * CHUNK, pol, st.L[u][c]);
                } else {
#pragma unroll
                    for (int j = 0; j < FPL / 2; ++j) st.L[u][c][j] = 0u;
                }
            }
        }
        if constexpr (LOADV) {
            if constexpr (F16Step<NCHUNK, FPL, VF32>::kDefer) f32_values_raw(a, vbase, nvw, vend, s, g, t, st.b);
            else f16_values<VF32, SMX>(a, vbase, nvw, vend, s, g, t, st.b);
        }
    }
}

template <int NCHUNK, int FPL, bool VF32, bool SMX = false>
__device__ __forceinline__ void f16_compute(const F16Step<NCHUNK, FPL, VF32>& st, float (&acc)[NCHUNK][FPL / 2][4],
                                            uint32_t src_lane, float scale = 0.f, float sm = 0.f, float sinv = 0.f) {
    uint32_t b0, b1;
    if constexpr (F16Step<NCHUNK, FPL, VF32>::kDefer) {
        static_assert(!SMX, "softmax operands are binary16");
        b0 = f2_to_h2(__uint_as_float(st.b[0]), __uint_as_float(st.b[1]));
        b1 = f2_to_h2(__uint_as_float(st.b[2]), __uint_as_float(st.b[3]));
    } else {
        b0 = st.b[0];
        b1 = st.b[1];
    }
    if constexpr (SMX) {  // applied here, when the values have landed
        b0 = smx_h2(b0, scale, sm, sinv);
        b1 = smx_h2(b1, scale, sm, sinv);
    }
#pragma unroll
    for (int c = 0; c < NCHUNK; ++c)
#pragma unroll
        for (int j = 0; j < FPL / 2; ++j) {
            // slot u of lane 8t+g = k-slot u of this lane (see the mapping note above)
            const uint32_t x0 = __shfl_sync(0xffffffffu, st.L[0][c][j], src_lane);
            const uint32_t x1 = __shfl_sync(0xffffffffu, st.L[1][c][j], src_lane);
            const uint32_t x2 = __shfl_sync(0xffffffffu, st.L[2][c][j], src_lane);
            const uint32_t x3 = __shfl_sync(0xffffffffu, st.L[3][c][j], src_lane);
            mma_f16_16816(acc[c][j], pack_lo(x0, x1), pack_hi(x0, x1), pack_lo(x2, x3), pack_hi(x2, x3), b0, b1);
        }
}

// Stores FPL consecutive features of one output row (row-major, stride ld).
template <int FPL>
__device__ __forceinline__ void store_row(float* __restrict__ dst, const float (&v)[FPL], int64_t feat,
                                          int64_t N, bool vec_ok) {
    if (vec_ok && feat + FPL <= N) {
#pragma unroll
        for (int q = 0; q < FPL; q += 4) st_stream_f4(dst + q, v[q], v[q + 1], v[q + 2], v[q + 3]);
    } else {
#pragma unroll
        for (int q = 0; q < FPL; ++q)
            if (feat + q < N) dst[q] = v[q];
    }
}

// Epilogue: lane holds window rows 2t, 2t+1 x features FPL*g + [0, FPL)
// of every chunk (accumulator layout, ref fragment.hpp:60-66).
template <int NCHUNK, int FPL>
__device__ __forceinline__ void f16_epilogue(const SpmmArgs& a, const WorkItem& it,
                                             const float (&acc)[NCHUNK][FPL / 2][4], int64_t feat0, uint32_t g,
                                             uint32_t t) {
    constexpr int NJ = FPL / 2, CHUNK = 8 * FPL;
    const bool split = it.slot != kNoSlot;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const uint32_t r = 2 * t + rr;
        const uint64_t row = 8ull * it.window + r;
        float* dst;
        bool vec_ok;
        if (split) {
            dst = a.partial + (static_cast<uint64_t>(it.slot) * 8 + r) * a.ldp;
            vec_ok = true;
        } else {
            if (row >= a.rows) continue;
            dst = a.C + row * a.ldc;
            vec_ok = (a.ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(a.C) & 15) == 0;
        }
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c) {
            float v[FPL];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                v[2 * j] = acc[c][j][rr];
                v[2 * j + 1] = acc[c][j][2 + rr];
            }
            const int64_t feat = feat0 + c * CHUNK + FPL * g;
            store_row<FPL>(dst + feat, v, feat, split ? a.ldp : a.N, vec_ok);
        }
    }
}

template <int NCHUNK, int FPL, bool VF32, bool SMX = false, bool HOT = false, bool PF = false>
__global__ void __launch_bounds__(kWarps * 32, spmm_blocks(NCHUNK, FPL)) spmm_f16_kernel(const SpmmArgs a) {
    constexpr int NJ = FPL / 2, CHUNK = 8 * FPL, SLAB = NCHUNK * CHUNK;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3;             // fragment coordinates
    const uint32_t q = lane >> 3, p = lane & 7;             // loader coordinates (quarter, lane in quarter)
    const uint32_t src_lane = 8 * t + g;                    // where this lane's fragment data was loaded
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * SLAB;
    const __half* Bl = static_cast<const __half*>(a.B) + feat0 + p * FPL;
    uint32_t* counter = dev::slab_counter(a.counter, a.slab0 + blockIdx.y);
    uint64_t pol_last = 0, pol_first = 0;
    if constexpr (HOT) {
        pol_last = l2_evict_last_policy();
        pol_first = l2_cold_policy<TCS_HOT_COLD>();
    }

    for (uint32_t idx = dev::next_item(counter, lane); idx < a.n_items; idx = dev::next_item(counter, lane)) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        const uint32_t vend = it.vend;
        float sm = 0.f, sinv = 0.f;  // softmax statistics of this lane's row g
        if constexpr (SMX) {
            const float2 st2 = a.rowstat[8ull * it.window + g];
            sm = st2.x;
            sinv = st2.y;
        }

        float acc[NCHUNK][NJ][4];
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[c][j][0] = acc[c][j][1] = acc[c][j][2] = acc[c][j][3] = 0.f;

        // Software pipeline: gathers one step ahead of the MMAs, column
        // indices (coalesced, 32 per load) two steps ahead of the gathers.
        F16Step<NCHUNK, FPL, VF32> sa, sb;
        uint32_t s = it.vbeg;
        if (s < vend) {
            uint32_t cp0 = load_colpair(ci, s, vend, lane);       // steps s, s+16
            uint32_t cp1 = load_colpair(ci, s + 32, vend, lane);  // steps s+32, s+48
            f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s, g, t, q, cp0, 0, sa, pol_last,
                                                         pol_first);
            for (;;) {
                if constexpr (PF && !VF32) {  // 32 vectors = 512 B of f16 values per iteration
                    const uint32_t pv = s + TCS_PREFETCH_F16;
                    if (lane < 4 && pv < vend && blockIdx.y == 0)
                        prefetch_l2(static_cast<const __half*>(a.vals) + vbase + 8ull * pv + 64 * lane);
                    if (lane == 4 && pv < vend && blockIdx.y == 0) prefetch_l2(ci + pv);
                }
                if (s + 16 < vend)
                    f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 16, g, t, q, cp0, 1, sb,
                                                                 pol_last, pol_first);
                f16_compute<NCHUNK, FPL, VF32, SMX>(sa, acc, src_lane, a.scale, sm, sinv);
                if (s + 16 >= vend) break;
                if (s + 32 < vend)
                    f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 32, g, t, q, cp1, 0, sa,
                                                                 pol_last, pol_first);
                cp0 = cp1;
                cp1 = load_colpair(ci, s + 64, vend, lane);
                f16_compute<NCHUNK, FPL, VF32, SMX>(sb, acc, src_lane, a.scale, sm, sinv);
                s += 32;
                if (s >= vend) break;
            }
        }

        f16_epilogue<NCHUNK, FPL>(a, it, acc, feat0, g, t);
    }
}

// Four-stage variant for narrow slabs (32 features: 64-byte rows, few
// registers per stage): three gather steps in flight while a fourth is
// multiplied, column indices four steps ahead.  (For 64-feature slabs, at 4
// CTAs/SM and 123 registers, it measured only 1% faster than the two-stage
// kernel at 8 CTAs/SM, so those keep the latter.)
#ifndef TCS_SPMM_DEEP_BPS
#define TCS_SPMM_DEEP_BPS 6
#endif
__device__ __forceinline__ uint32_t load_col16(const uint32_t* __restrict__ ci, uint32_t s, uint32_t vend,
                                               uint32_t lane) {
    return lane < 16 && s + lane < vend ? ld_stream_u32(ci + s + lane) : 0u;
}

template <int NCHUNK, int FPL, bool VF32, bool SMX, int BPS, bool HOT = false>
__global__ void __launch_bounds__(kWarps * 32, BPS) spmm_f16_kernel_deep(const SpmmArgs a) {
    constexpr int NJ = FPL / 2, CHUNK = 8 * FPL, SLAB = NCHUNK * CHUNK;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3;
    const uint32_t q = lane >> 3, p = lane & 7;
    const uint32_t src_lane = 8 * t + g;
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * SLAB;
    const __half* Bl = static_cast<const __half*>(a.B) + feat0 + p * FPL;
    uint32_t* counter = dev::slab_counter(a.counter, a.slab0 + blockIdx.y);
    uint64_t pol_last = 0, pol_first = 0;
    if constexpr (HOT) {
        pol_last = l2_evict_last_policy();
        pol_first = l2_cold_policy<TCS_HOT_COLD>();
    }
    dev::StripedClaim<1> claim;  // this loop form measured 7% faster than next_item here (C5 N=32)
    for (uint32_t idx; claim.get(counter, a.n_items, idx);) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        const uint32_t vend = it.vend;
        float sm = 0.f, sinv = 0.f;
        if constexpr (SMX) {
            const float2 st2 = a.rowstat[8ull * it.window + g];
            sm = st2.x;
            sinv = st2.y;
        }
        float acc[NCHUNK][NJ][4];
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[c][j][0] = acc[c][j][1] = acc[c][j][2] = acc[c][j][3] = 0.f;

        F16Step<NCHUNK, FPL, VF32> s0, s1, s2, s3;
        uint32_t s = it.vbeg;
        if (s < vend) {
            // loop-top invariant: s0/s1/s2 hold steps s, s+16, s+32 (issued);
            // c3 = columns of s+48, c0 of s+64, c1 of s+80, c2 of s+96
            uint32_t c0 = load_col16(ci, s, vend, lane), c1 = load_col16(ci, s + 16, vend, lane);
            uint32_t c2 = load_col16(ci, s + 32, vend, lane), c3 = load_col16(ci, s + 48, vend, lane);
            f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s, g, t, q, c0, 0, s0, pol_last, pol_first);
            c0 = load_col16(ci, s + 64, vend, lane);
            if (s + 16 < vend) f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 16, g, t, q, c1, 0, s1, pol_last, pol_first);
            c1 = load_col16(ci, s + 80, vend, lane);
            if (s + 32 < vend) f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 32, g, t, q, c2, 0, s2, pol_last, pol_first);
            c2 = load_col16(ci, s + 96, vend, lane);
            for (;;) {
                if (s + 48 < vend) f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 48, g, t, q, c3, 0, s3, pol_last, pol_first);
                c3 = load_col16(ci, s + 112, vend, lane);
                f16_compute<NCHUNK, FPL, VF32, SMX>(s0, acc, src_lane, a.scale, sm, sinv);
                if (s + 16 >= vend) break;
                if (s + 64 < vend) f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 64, g, t, q, c0, 0, s0, pol_last, pol_first);
                c0 = load_col16(ci, s + 128, vend, lane);
                f16_compute<NCHUNK, FPL, VF32, SMX>(s1, acc, src_lane, a.scale, sm, sinv);
                if (s + 32 >= vend) break;
                if (s + 80 < vend) f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 80, g, t, q, c1, 0, s1, pol_last, pol_first);
                c1 = load_col16(ci, s + 144, vend, lane);
                f16_compute<NCHUNK, FPL, VF32, SMX>(s2, acc, src_lane, a.scale, sm, sinv);
                if (s + 48 >= vend) break;
                if (s + 96 < vend) f16_issue<NCHUNK, FPL, VF32, SMX, true, HOT>(a, Bl, vbase, nvw, vend, s + 96, g, t, q, c2, 0, s2, pol_last, pol_first);
                c2 = load_col16(ci, s + 160, vend, lane);
                f16_compute<NCHUNK, FPL, VF32, SMX>(s3, acc, src_lane, a.scale, sm, sinv);
                s += 64;
                if (s >= vend) break;
            }
        }
        f16_epilogue<NCHUNK, FPL>(a, it, acc, feat0, g, t);
    }
}

// ------------------------------------------------- FP16, direct mapping
//
// The paper's "direct" thread mapping (ref access_pattern.hpp:79-95,
// ThreadMapping::direct), kept as the ablation of the memory-efficient
// mapping above: lane (g, t) loads exactly its own A-fragment elements,
// i.e. B[col(2t+dr)][16j + g + dc] for dr in {0,1}, dc in {0,8}, as single
// 2-byte loads -- 8 lanes of a quarter touch 16 bytes of a row per load and
// every B row is requested 2x as often (4 steps instead of 2 in the
// reference's transaction model).  Same MMA operands and k order as the
// coalesced kernel, hence bit-identical results (ref acceptance.cpp:103-104).
template <int NMMA, bool VF32>
__global__ void __launch_bounds__(kWarps * 32, 4) spmm_f16_direct_kernel(const SpmmArgs a) {
    constexpr int SLAB = 16 * NMMA;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3;
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * SLAB;
    const unsigned short* Bl = static_cast<const unsigned short*>(a.B) + feat0 + g;
    uint32_t* counter = dev::slab_counter(a.counter, a.slab0 + blockIdx.y);

    for (uint32_t idx = dev::next_item(counter, lane); idx < a.n_items; idx = dev::next_item(counter, lane)) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        const uint32_t vend = it.vend;

        float acc[NMMA][4];
#pragma unroll
        for (int j = 0; j < NMMA; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

        for (uint32_t s = it.vbeg; s < vend; s += 16) {
            const uint32_t colv = load_colpair(ci, s, vend, lane);
            uint32_t col[4];
            bool ok[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // k slots 2t, 2t+1, 2t+8, 2t+9 (vector order: kslot_vec)
                const uint32_t v = kslot_vec(u, t);
                col[u] = __shfl_sync(0xffffffffu, colv, v);
                ok[u] = s + v < vend;
            }
            uint32_t b0, b1;  // sparse fragment: rows g, vectors {2t, 2t+1}, {2t+8, 2t+9}
            if (s + 16 <= vend) {
                load_sparse_full<VF32>(a.vals, vbase, s, g, t, b0, b1);
            } else {
                uint32_t e[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t v = s + kslot_vec(u, t);
                    e[u] = v < vend ? f16_val_general<VF32>(a.vals, vbase, nvw, v, g) : 0u;
                }
                b0 = e[0] | (e[1] << 16);
                b1 = e[2] | (e[3] << 16);
            }
#pragma unroll
            for (int j = 0; j < NMMA; ++j) {
                uint32_t e[4][2];  // [k slot][feature g / g + 8]
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        e[u][h] = ok[u] ? __ldg(Bl + static_cast<uint64_t>(col[u]) * a.ldb + 16 * j + 8 * h) : 0u;
                mma_f16_16816(acc[j], e[0][0] | (e[1][0] << 16), e[0][1] | (e[1][1] << 16),
                              e[2][0] | (e[3][0] << 16), e[2][1] | (e[3][1] << 16), b0, b1);
            }
        }

        // accumulator (m = feature, n = window row): d0 (g, 2t), d1 (g, 2t+1), d2 (g+8, 2t), d3 (g+8, 2t+1)
        const bool split = it.slot != kNoSlot;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const uint32_t r = 2 * t + rr;
            const uint64_t row = 8ull * it.window + r;
            float* dst;
            int64_t lim;
            if (split) {
                dst = a.partial + (static_cast<uint64_t>(it.slot) * 8 + r) * a.ldp;
                lim = a.ldp;
            } else {
                if (row >= a.rows) continue;
                dst = a.C + row * a.ldc;
                lim = a.N;
            }
#pragma unroll
            for (int j = 0; j < NMMA; ++j) {
                const int64_t f = feat0 + 16 * j + g;
                if (f < lim) dst[f] = acc[j][rr];
                if (f + 8 < lim) dst[f + 8] = acc[j][2 + rr];
            }
        }
    }
}

// ------------------------------------------------------------- TF32 path
//
// Same scheme with m16n8k8.tf32: an 8-vector step; loader slot u (0, 1) of
// quarter q reads 128 B (32 features) of vector q + 4u; lane 8t + g then
// holds exactly the (vector t + 4u, features 4g..4g+3) fragment data of
// lane (g, t).  Operands are rounded RNE with cvt.rn.tf32.f32.
template <int NCHUNK>
struct Tf32Step {
    uint4 L[2][NCHUNK];  // loader slots: vector q + 4u, features 32c + 4p .. +3
    uint32_t b[2];       // sparse fragment: row g, vectors t, t+4 (raw f32 bits)
};

__device__ __forceinline__ float tf32_val_general(const float* vals, uint64_t vbase, uint32_t nvw, uint32_t v,
                                                  uint32_t g) {
    if (v >= nvw) return 0.f;
    const uint32_t b = v >> 2, j = v & 3u, width = min(4u, nvw - 4 * b);
    return __ldg(vals + vbase + 32ull * b + g * width + j);
}

// colquad holds the column indices of vectors [s - 8*sub, +32) (4 steps).
template <int NCHUNK>
__device__ __forceinline__ void tf32_issue(const SpmmArgs& a, const float* __restrict__ Bl, uint64_t vbase,
                                           uint32_t nvw, uint32_t vend, uint32_t s, uint32_t g, uint32_t t,
                                           uint32_t q, uint32_t colquad, uint32_t sub, Tf32Step<NCHUNK>& st) {
    const uint32_t c0 = __shfl_sync(0xffffffffu, colquad, 8 * sub + q);
    const uint32_t c1 = __shfl_sync(0xffffffffu, colquad, 8 * sub + q + 4);
    const float* fv = static_cast<const float*>(a.vals);
    float x0, x1;
    if (s + 8 <= vend) {
        const float* r0 = Bl + static_cast<uint64_t>(c0) * a.ldb;
        const float* r1 = Bl + static_cast<uint64_t>(c1) * a.ldb;
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c) {
            st.L[0][c] = ld_gather_128(r0 + c * 32);
            st.L[1][c] = ld_gather_128(r1 + c * 32);
        }
        const uint64_t off = vbase + 8ull * s + 4 * g + t;
        x0 = __uint_as_float(ld_stream_u32(fv + off));
        x1 = __uint_as_float(ld_stream_u32(fv + off + 32));
    } else {
        const bool ok0 = s + q < vend, ok1 = s + q + 4 < vend;
        const float* r0 = Bl + static_cast<uint64_t>(c0) * a.ldb;
        const float* r1 = Bl + static_cast<uint64_t>(c1) * a.ldb;
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c) {
            st.L[0][c] = ok0 ? ld_gather_128(r0 + c * 32) : make_uint4(0, 0, 0, 0);
            st.L[1][c] = ok1 ? ld_gather_128(r1 + c * 32) : make_uint4(0, 0, 0, 0);
        }
        x0 = s + t < vend ? tf32_val_general(fv, vbase, nvw, s + t, g) : 0.f;
        x1 = s + t + 4 < vend ? tf32_val_general(fv, vbase, nvw, s + t + 4, g) : 0.f;
    }
    // raw f32 bits: rounded to TF32 in the compute step, so the conversion
    // does not wait here for the value loads (ncu, C3 N=128: 57% of the
    // stall samples sat on this conversion, before the previous step's MMAs)
    st.b[0] = __float_as_uint(x0);
    st.b[1] = __float_as_uint(x1);
}

__device__ __forceinline__ uint4 shfl4(uint4 v, uint32_t src) {
    return make_uint4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                      __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}

template <int NCHUNK>
__device__ __forceinline__ void tf32_compute(const Tf32Step<NCHUNK>& st, float (&acc)[NCHUNK][2][4],
                                             uint32_t src_lane) {
    const uint32_t b0 = to_tf32(__uint_as_float(st.b[0])), b1 = to_tf32(__uint_as_float(st.b[1]));
#pragma unroll
    for (int c = 0; c < NCHUNK; ++c) {
        const uint4 x = shfl4(st.L[0][c], src_lane), y = shfl4(st.L[1][c], src_lane);
        mma_tf32_1688(acc[c][0], to_tf32(__uint_as_float(x.x)), to_tf32(__uint_as_float(x.y)),
                      to_tf32(__uint_as_float(y.x)), to_tf32(__uint_as_float(y.y)), b0, b1);
        mma_tf32_1688(acc[c][1], to_tf32(__uint_as_float(x.z)), to_tf32(__uint_as_float(x.w)),
                      to_tf32(__uint_as_float(y.z)), to_tf32(__uint_as_float(y.w)), b0, b1);
    }
}

// TF32 epilogue: lane holds rows 2t, 2t+1 x features 32c + 4g .. +3.
template <int NCHUNK>
__device__ __forceinline__ void tf32_epilogue(const SpmmArgs& a, const WorkItem& it, const float (&acc)[NCHUNK][2][4],
                                              int64_t feat0, uint32_t g, uint32_t t) {
    const bool split = it.slot != kNoSlot;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const uint32_t r = 2 * t + rr;
        const uint64_t row = 8ull * it.window + r;
        float* dst;
        bool vec_ok;
        if (split) {
            dst = a.partial + (static_cast<uint64_t>(it.slot) * 8 + r) * a.ldp;
            vec_ok = true;
        } else {
            if (row >= a.rows) continue;
            dst = a.C + row * a.ldc;
            vec_ok = (a.ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(a.C) & 15) == 0;
        }
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c) {
            const float v[4] = {acc[c][0][rr], acc[c][0][2 + rr], acc[c][1][rr], acc[c][1][2 + rr]};
            const int64_t feat = feat0 + c * 32 + 4 * g;
            store_row<4>(dst + feat, v, feat, split ? a.ldp : a.N, vec_ok);
        }
    }
}

template <int NCHUNK>
__global__ void __launch_bounds__(kWarps * 32, tf32_blocks(NCHUNK)) spmm_tf32_kernel(const SpmmArgs a) {
    constexpr int SLAB = NCHUNK * 32;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3;
    const uint32_t q = lane >> 3, p = lane & 7, src_lane = 8 * t + g;
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * SLAB;
    const float* Bl = static_cast<const float*>(a.B) + feat0 + 4 * p;
    uint32_t* counter = dev::slab_counter(a.counter, a.slab0 + blockIdx.y);

    for (uint32_t idx = dev::next_item(counter, lane); idx < a.n_items; idx = dev::next_item(counter, lane)) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        const uint32_t vend = it.vend;

        float acc[NCHUNK][2][4];
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[c][j][0] = acc[c][j][1] = acc[c][j][2] = acc[c][j][3] = 0.f;

        Tf32Step<NCHUNK> sa, sb;
        uint32_t s = it.vbeg;
        if (s < vend) {
            // colquad: 32 vectors = 4 steps; cur covers [s0, s0+32), nxt the next 32
            uint32_t s0 = s;
            uint32_t cur = load_colpair(ci, s0, vend, lane);
            uint32_t nxt = load_colpair(ci, s0 + 32, vend, lane);
            tf32_issue(a, Bl, vbase, nvw, vend, s, g, t, q, cur, 0, sa);
            for (;;) {
                // issue s + 8 into sb
                if (s + 8 < vend) {
                    const uint32_t sub = (s + 8 - s0) >> 3;
                    tf32_issue(a, Bl, vbase, nvw, vend, s + 8, g, t, q, sub < 4 ? cur : nxt, sub & 3, sb);
                }
                tf32_compute(sa, acc, src_lane);
                if (s + 8 >= vend) break;
                if (s + 16 < vend) {
                    uint32_t sub = (s + 16 - s0) >> 3;
                    if (sub >= 4) {  // advance the column window
                        s0 += 32;
                        cur = nxt;
                        nxt = load_colpair(ci, s0 + 32, vend, lane);
                        sub -= 4;
                    }
                    tf32_issue(a, Bl, vbase, nvw, vend, s + 16, g, t, q, cur, sub, sa);
                }
                tf32_compute(sb, acc, src_lane);
                s += 16;
                if (s >= vend) break;
            }
        }

        tf32_epilogue<NCHUNK>(a, it, acc, feat0, g, t);
    }
}

// ------------------------------------------------- TF32, packed operand
//
// The TF32 MMA reads only the top 19 bits of an operand (sign, exponent, 10
// mantissa bits), so the RNE-rounded dense operand is repacked once per call
// into 2.5 bytes per feature: the top 16 bits ("hi", one u16) and mantissa
// bits 10..12 below them ("lo", one nibble, stored as e << 1).  Per B row:
// [hi: 2*npad bytes][lo: npad/2 bytes] -- 320 B instead of 512 B at N = 128,
// so C3's 119 MB f32 operand becomes 75 MB and stays L2-resident, and each
// gathered row costs 2 + 1 loads and 10 shuffles per 128 features instead
// of 4 and 16.  Rebuilding an operand is one PRMT: the hi pair supplies the
// top two bytes, the nibble's byte the third (bits 13..15 = e; the low 13
// bits the MMA ignores are don't-care).  Bit-identical to the f32 path.
//
// Mapping: as the f32 TF32 kernel (loader slot u of quarter q reads vector
// q + 4u) but with 64-feature chunks, 8 features per lane: lane (g, t) gets,
// after the shuffle from lane 8t+g, features 8g..8g+7 of vectors t and t+4.
// M-tile j of a chunk holds feature 8g+2j in row g and 8g+2j+1 in row g+8,
// so the accumulator layout is the FP16 kernel's (f16_epilogue<., 8>).
// lo64: 128-feature slabs read both chunks' nibble words with one 8-byte
// load, so within a slab the word of (chunk c, lane p) sits at 8p + 4c.
__global__ void __launch_bounds__(256) tf32_pack_kernel(const float* __restrict__ b, int64_t ldb, int64_t rows,
                                                        int64_t n, int64_t npad, unsigned char* __restrict__ out,
                                                        int64_t lds, bool lo64) {
    const int64_t groups = npad / 8, total = rows * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / groups, f0 = (i - r * groups) * 8;
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = f0 + k < n ? to_tf32(b[r * ldb + f0 + k]) : 0u;
        uint4 hi;
        hi.x = (w[0] >> 16) | (w[1] & 0xFFFF0000u);
        hi.y = (w[2] >> 16) | (w[3] & 0xFFFF0000u);
        hi.z = (w[4] >> 16) | (w[5] & 0xFFFF0000u);
        hi.w = (w[6] >> 16) | (w[7] & 0xFFFF0000u);
        uint32_t lo = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) lo |= ((w[k] >> 13) & 7u) << (4 * k + 1);  // nibble k = e << 1
        unsigned char* row = out + r * lds;
        *reinterpret_cast<uint4*>(row + 2 * f0) = hi;
        const int64_t lo_off = lo64 ? (f0 / 128) * 64 + ((f0 % 64) / 8) * 8 + ((f0 % 128) / 64) * 4 : f0 / 2;
        *reinterpret_cast<uint32_t*>(row + 2 * npad + lo_off) = lo;
    }
}

// Operands of features 2j, 2j+1 from hi word h (pair j) and the nibble word
// L (S = L << 4): the odd feature's nibble is the high nibble of L's byte j,
// the even one's the high nibble of S's byte j.
template <int J>
__device__ __forceinline__ uint32_t tf32p_even(uint32_t h, uint32_t S) {
    return __byte_perm(h, S, 0x1000 | ((4 + J) << 4));
}
template <int J>
__device__ __forceinline__ uint32_t tf32p_odd(uint32_t h, uint32_t L) {
    return __byte_perm(h, L, 0x3200 | ((4 + J) << 4));
}

template <int NCHUNK>
struct Tf32PStep {
    uint4 H[2][NCHUNK];     // loader slots: vector q + 4u, hi of features 64c + 8p .. +7
    uint32_t L[2][NCHUNK];  // their nibbles
    uint32_t b[2];          // sparse fragment: row g, vectors t, t+4 (raw f32 bits)
};

template <int NCHUNK>
__device__ __forceinline__ void tf32p_issue(const SpmmArgs& a, const unsigned char* __restrict__ Bl,
                                            const unsigned char* __restrict__ Ll, uint64_t vbase, uint32_t nvw,
                                            uint32_t vend, uint32_t s, uint32_t g, uint32_t t, uint32_t q,
                                            uint32_t colquad, uint32_t sub, Tf32PStep<NCHUNK>& st) {
    const uint32_t c0 = __shfl_sync(0xffffffffu, colquad, 8 * sub + q);
    const uint32_t c1 = __shfl_sync(0xffffffffu, colquad, 8 * sub + q + 4);
    const float* fv = static_cast<const float*>(a.vals);
    const uint64_t o0 = static_cast<uint64_t>(c0) * a.ldb, o1 = static_cast<uint64_t>(c1) * a.ldb;
    float x0, x1;
    if (s + 8 <= vend) {
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c) {
            st.H[0][c] = TCS_GATHER_NA ? ld_gather_128_na(Bl + o0 + c * 128) : ld_gather_128(Bl + o0 + c * 128);
            st.H[1][c] = TCS_GATHER_NA ? ld_gather_128_na(Bl + o1 + c * 128) : ld_gather_128(Bl + o1 + c * 128);
        }
        if constexpr (NCHUNK == 2 && TCS_TF32P_LO64) {
            const uint2 l0 = ld_gather_64(Ll + o0), l1 = ld_gather_64(Ll + o1);
            st.L[0][0] = l0.x; st.L[0][1] = l0.y; st.L[1][0] = l1.x; st.L[1][1] = l1.y;
        } else {
#pragma unroll
            for (int c = 0; c < NCHUNK; ++c) {
                st.L[0][c] = ld_gather_32(Ll + o0 + c * 32);
                st.L[1][c] = ld_gather_32(Ll + o1 + c * 32);
            }
        }
        const uint64_t off = vbase + 8ull * s + 4 * g + t;
#if TCS_TF32P_EF
        const uint64_t pol = l2_evict_first_policy();
        x0 = __uint_as_float(ld_stream_ef_u32(fv + off, pol));
        x1 = __uint_as_float(ld_stream_ef_u32(fv + off + 32, pol));
#else
        x0 = __uint_as_float(ld_stream_u32(fv + off));
        x1 = __uint_as_float(ld_stream_u32(fv + off + 32));
#endif
    } else {
        const bool ok0 = s + q < vend, ok1 = s + q + 4 < vend;
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c) {
            st.H[0][c] = ok0 ? ld_gather_128(Bl + o0 + c * 128) : make_uint4(0, 0, 0, 0);
            st.H[1][c] = ok1 ? ld_gather_128(Bl + o1 + c * 128) : make_uint4(0, 0, 0, 0);
        }
        if constexpr (NCHUNK == 2 && TCS_TF32P_LO64) {
            const uint2 l0 = ok0 ? ld_gather_64(Ll + o0) : make_uint2(0, 0);
            const uint2 l1 = ok1 ? ld_gather_64(Ll + o1) : make_uint2(0, 0);
            st.L[0][0] = l0.x; st.L[0][1] = l0.y; st.L[1][0] = l1.x; st.L[1][1] = l1.y;
        } else {
#pragma unroll
            for (int c = 0; c < NCHUNK; ++c) {
                st.L[0][c] = ok0 ? ld_gather_32(Ll + o0 + c * 32) : 0u;
                st.L[1][c] = ok1 ? ld_gather_32(Ll + o1 + c * 32) : 0u;
            }
        }
        x0 = s + t < vend ? tf32_val_general(fv, vbase, nvw, s + t, g) : 0.f;
        x1 = s + t + 4 < vend ? tf32_val_general(fv, vbase, nvw, s + t + 4, g) : 0.f;
    }
    // raw f32 bits: rounded to TF32 in the compute step, so the conversion
    // does not wait here for the value loads (ncu, C3 N=128: 57% of the
    // stall samples sat on this conversion, before the previous step's MMAs)
    st.b[0] = __float_as_uint(x0);
    st.b[1] = __float_as_uint(x1);
}

template <int NCHUNK>
__device__ __forceinline__ void tf32p_compute(const Tf32PStep<NCHUNK>& st, float (&acc)[NCHUNK][4][4],
                                              uint32_t src_lane) {
    const uint32_t b0 = to_tf32(__uint_as_float(st.b[0])), b1 = to_tf32(__uint_as_float(st.b[1]));
#pragma unroll
    for (int c = 0; c < NCHUNK; ++c) {
        const uint4 x = shfl4(st.H[0][c], src_lane), y = shfl4(st.H[1][c], src_lane);
        const uint32_t lx = __shfl_sync(0xffffffffu, st.L[0][c], src_lane);
        const uint32_t ly = __shfl_sync(0xffffffffu, st.L[1][c], src_lane);
        const uint32_t sx = lx << 4, sy = ly << 4;
        mma_tf32_1688(acc[c][0], tf32p_even<0>(x.x, sx), tf32p_odd<0>(x.x, lx), tf32p_even<0>(y.x, sy),
                      tf32p_odd<0>(y.x, ly), b0, b1);
        mma_tf32_1688(acc[c][1], tf32p_even<1>(x.y, sx), tf32p_odd<1>(x.y, lx), tf32p_even<1>(y.y, sy),
                      tf32p_odd<1>(y.y, ly), b0, b1);
        mma_tf32_1688(acc[c][2], tf32p_even<2>(x.z, sx), tf32p_odd<2>(x.z, lx), tf32p_even<2>(y.z, sy),
                      tf32p_odd<2>(y.z, ly), b0, b1);
        mma_tf32_1688(acc[c][3], tf32p_even<3>(x.w, sx), tf32p_odd<3>(x.w, lx), tf32p_even<3>(y.w, sy),
                      tf32p_odd<3>(y.w, ly), b0, b1);
    }
}

// Resident CTAs per SM: 64-feature slabs (79 registers at 6, no spill)
// need the warps to cover DRAM latency (C3 N=64: 4.53 ms at 4, 3.60 at 6);
// 128-feature slabs keep their 126 registers (5 CTAs/SM spill: N=128 5.45
// -> 5.98 ms).  profiles/r2_tf32_packed.txt
#ifndef TCS_TF32P_BPS_WIDE
#define TCS_TF32P_BPS_WIDE 4
#endif
#ifndef TCS_TF32P_BPS_NARROW
#define TCS_TF32P_BPS_NARROW 6
#endif
constexpr int tf32p_blocks(int nchunk) { return nchunk == 1 ? TCS_TF32P_BPS_NARROW : TCS_TF32P_BPS_WIDE; }
// a.B = packed rows (tf32_pack_kernel), a.ldb = their stride in BYTES.
template <int NCHUNK, bool PF = false>
__global__ void __launch_bounds__(kWarps * 32, tf32p_blocks(NCHUNK)) spmm_tf32p_kernel(const SpmmArgs a) {
    constexpr int SLAB = NCHUNK * 64;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3;
    const uint32_t q = lane >> 3, p = lane & 7, src_lane = 8 * t + g;
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * SLAB;
    const unsigned char* Bl = static_cast<const unsigned char*>(a.B) + 2 * feat0 + 16 * p;
    const unsigned char* Ll = static_cast<const unsigned char*>(a.B) + 2 * a.ldp + feat0 / 2 +
                              (NCHUNK == 2 && TCS_TF32P_LO64 ? 8 : 4) * p;
    uint32_t* counter = dev::slab_counter(a.counter, a.slab0 + blockIdx.y);

    for (uint32_t idx = dev::next_item(counter, lane); idx < a.n_items; idx = dev::next_item(counter, lane)) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        const uint32_t vend = it.vend;

        float acc[NCHUNK][4][4];
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[c][j][0] = acc[c][j][1] = acc[c][j][2] = acc[c][j][3] = 0.f;

        Tf32PStep<NCHUNK> sa, sb;
        uint32_t s = it.vbeg;
        if (s < vend) {
            uint32_t s0 = s;
            uint32_t cur = load_colpair(ci, s0, vend, lane);
            uint32_t nxt = load_colpair(ci, s0 + 32, vend, lane);
            tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s, g, t, q, cur, 0, sa);
            for (;;) {
                if constexpr (PF) {  // 16 vectors = 512 B of f32 values per iteration
                    const uint32_t pv = s + TCS_PREFETCH_AHEAD;
                    if (lane < 4 && pv < vend && blockIdx.y == 0)  // one slab prefetches for all
                        prefetch_l2(static_cast<const float*>(a.vals) + vbase + 8ull * pv + 32 * lane);
                    if (lane == 4 && pv < vend && blockIdx.y == 0) prefetch_l2(ci + pv);
                }
                if (s + 8 < vend) {
                    const uint32_t sub = (s + 8 - s0) >> 3;
                    tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 8, g, t, q, sub < 4 ? cur : nxt, sub & 3, sb);
                }
                tf32p_compute(sa, acc, src_lane);
                if (s + 8 >= vend) break;
                if (s + 16 < vend) {
                    uint32_t sub = (s + 16 - s0) >> 3;
                    if (sub >= 4) {
                        s0 += 32;
                        cur = nxt;
                        nxt = load_colpair(ci, s0 + 32, vend, lane);
                        sub -= 4;
                    }
                    tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 16, g, t, q, cur, sub, sa);
                }
                tf32p_compute(sb, acc, src_lane);
                s += 16;
                if (s >= vend) break;
            }
        }
        f16_epilogue<NCHUNK, 8>(a, it, acc, feat0, g, t);
    }
}

// Four-stage packed TF32 kernel for 64-feature slabs: three 8-vector gather
// steps in flight while a fourth is multiplied (the two-stage kernel keeps
// one; TF32 was latency-bound there, ncu long-scoreboard 6.4 per issue at
// 16 warps/SM), column indices one 32-vector window ahead.
#ifndef TCS_TF32P_DEEP
#define TCS_TF32P_DEEP 0
#endif
#ifndef TCS_TF32P_DEEP_BPS
#define TCS_TF32P_DEEP_BPS 6
#endif
__global__ void __launch_bounds__(kWarps * 32, TCS_TF32P_DEEP_BPS) spmm_tf32p_deep(const SpmmArgs a) {
    constexpr int SLAB = 64;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3;
    const uint32_t q = lane >> 3, p = lane & 7, src_lane = 8 * t + g;
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * SLAB;
    const unsigned char* Bl = static_cast<const unsigned char*>(a.B) + 2 * feat0 + 16 * p;
    const unsigned char* Ll = static_cast<const unsigned char*>(a.B) + 2 * a.ldp + feat0 / 2 + 4 * p;
    uint32_t* counter = dev::slab_counter(a.counter, a.slab0 + blockIdx.y);
    for (uint32_t idx = dev::next_item(counter, lane); idx < a.n_items; idx = dev::next_item(counter, lane)) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        const uint32_t vend = it.vend;
        float acc[1][4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[0][j][0] = acc[0][j][1] = acc[0][j][2] = acc[0][j][3] = 0.f;
        Tf32PStep<1> s0, s1, s2, s3;
        uint32_t s = it.vbeg;
        if (s < vend) {
            // loop-top invariant: s0/s1/s2 hold steps s, s+8, s+16 (issued);
            // c0 = columns of [s, s+32), c1 = [s+32, s+64)
            uint32_t c0 = load_colpair(ci, s, vend, lane), c1 = load_colpair(ci, s + 32, vend, lane);
            tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s, g, t, q, c0, 0, s0);
            if (s + 8 < vend) tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 8, g, t, q, c0, 1, s1);
            if (s + 16 < vend) tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 16, g, t, q, c0, 2, s2);
            for (;;) {
                if (s + 24 < vend) tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 24, g, t, q, c0, 3, s3);
                const uint32_t c2 = load_colpair(ci, s + 64, vend, lane);
                tf32p_compute(s0, acc, src_lane);
                if (s + 8 >= vend) break;
                if (s + 32 < vend) tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 32, g, t, q, c1, 0, s0);
                tf32p_compute(s1, acc, src_lane);
                if (s + 16 >= vend) break;
                if (s + 40 < vend) tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 40, g, t, q, c1, 1, s1);
                tf32p_compute(s2, acc, src_lane);
                if (s + 24 >= vend) break;
                if (s + 48 < vend) tf32p_issue(a, Bl, Ll, vbase, nvw, vend, s + 48, g, t, q, c1, 2, s2);
                tf32p_compute(s3, acc, src_lane);
                s += 32;
                if (s >= vend) break;
                c0 = c1;
                c1 = c2;
            }
        }
        f16_epilogue<1, 8>(a, it, acc, feat0, g, t);
    }
}

// ------------------------------------------------ small lists: burst kernels
//
// BASELINE configs[0]/[1] (4096^2, 16 nnz/row: 512 windows of ~123 vectors)
// are latency-bound: one wave of warps, each walking its window through a
// chain of dependent loads (item -> row pointers -> column indices ->
// gathers), and the software pipeline of the persistent kernels never
// reaches steady state.  Here SPLIT warps of one CTA share an item, each
// takes a contiguous run of its steps and issues ALL of that run's gathers
// at once (up to MAXS steps per burst), so the chain is row pointers ->
// column indices -> gathers -> MMA; the partial accumulators are summed in
// shared memory in part order (deterministic).  With no split windows the
// plan's item i is window i (a.items == nullptr): one load less.
constexpr int kBurstRed = 8;  // accumulator floats per lane (32-feature slab)
// Resident CTAs per SM of the split burst kernels (73 registers: 4 FP16
// steps of 10 registers in flight without spilling; C1 at SPLIT = 2 is 4096
// warps, one wave at 7 x 4 x 148).
constexpr int kBurstBlocks = 7;
// Warps per CTA of the burst kernels (A/B knob: fewer, larger CTAs launch
// faster; the per-SM warp budget is the same).
#ifndef TCS_BURST_WARPS
#define TCS_BURST_WARPS 4
#endif
constexpr int kBW = TCS_BURST_WARPS;
#ifndef TCS_BURST_FORCE_SPLIT
#define TCS_BURST_FORCE_SPLIT 0
#endif

__device__ __forceinline__ WorkItem burst_item(const SpmmArgs& a, uint64_t idx, uint32_t& base, uint32_t& nvw) {
    WorkItem it;
    if (a.items) {
        it = a.items[idx];
        base = __ldg(a.rp + it.window);
        nvw = __ldg(a.rp + it.window + 1) - base;
    } else {
        base = __ldg(a.rp + idx);
        nvw = __ldg(a.rp + idx + 1) - base;
        it = WorkItem{static_cast<uint32_t>(idx), 0u, nvw, kNoSlot};
    }
    return it;
}

// Sums the SPLIT warps' accumulators of each item into part 0 (fixed order).
template <int SPLIT>
__device__ __forceinline__ void burst_reduce(float (&acc)[kBurstRed], uint32_t warp, uint32_t lane) {
    if constexpr (SPLIT > 1) {
        __shared__ float red[kBW][kBurstRed][32];
        if (warp % SPLIT)
#pragma unroll
            for (int j = 0; j < kBurstRed; ++j) red[warp][j][lane] = acc[j];
        __syncthreads();
        if (warp % SPLIT == 0)
#pragma unroll
            for (int p = 1; p < SPLIT; ++p)
#pragma unroll
                for (int j = 0; j < kBurstRed; ++j) acc[j] += red[warp + p][j][lane];
    }
}

template <bool VF32, int SPLIT, int MAXS, bool SMX = false>
__global__ void __launch_bounds__(kBW * 32, (SPLIT > 1 ? kBurstBlocks : 4) * kWarps / kBW) spmm_f16_burst(const SpmmArgs a) {
    static_assert(kBW % SPLIT == 0, "parts of an item share a CTA");
    constexpr int FPL = 4;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t g = lane >> 2, t = lane & 3, q = lane >> 3, p = lane & 7, src_lane = 8 * t + g;
    const uint32_t part = warp % SPLIT;
    const uint64_t idx = (static_cast<uint64_t>(blockIdx.x) * kBW + warp) / SPLIT;
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * 32;
    const __half* Bl = static_cast<const __half*>(a.B) + feat0 + p * FPL;
    pdl_trigger();  // the next small-list kernel may be scheduled now ...
    pdl_wait();     // ... and this one touches memory only after its predecessor completed
    const bool active = idx < a.n_items;  // every warp reaches the reduction barrier
    float acc[1][FPL / 2][4] = {};
    WorkItem it{};
    if (active) {
        uint32_t base, nvw;
        it = burst_item(a, idx, base, nvw);
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        float sm = 0.f, sinv = 0.f;  // softmax statistics of this lane's row g (SMX)
        if constexpr (SMX) {
            const float2 st2 = a.rowstat[8ull * it.window + g];
            sm = st2.x;
            sinv = st2.y;
        }
        const uint32_t steps = (it.vend - it.vbeg + 15) / 16, per = (steps + SPLIT - 1) / SPLIT;
        const uint32_t vend = min(it.vend, it.vbeg + 16 * per * (part + 1));
        for (uint32_t s0 = it.vbeg + 16 * per * part; s0 < vend; s0 += 16 * MAXS) {
            uint32_t cp[(MAXS + 1) / 2];
#pragma unroll
            for (int j = 0; j < (MAXS + 1) / 2; ++j) cp[j] = load_colpair(ci, s0 + 32 * j, vend, lane);
            F16Step<1, FPL, VF32> st[MAXS];
#pragma unroll
            for (int i = 0; i < MAXS; ++i)
                if (s0 + 16 * i < vend)
                    f16_issue<1, FPL, VF32, SMX>(a, Bl, vbase, nvw, vend, s0 + 16 * i, g, t, q, cp[i / 2], i & 1,
                                                 st[i]);
#pragma unroll
            for (int i = 0; i < MAXS; ++i)
                if (s0 + 16 * i < vend) f16_compute<1, FPL, VF32, SMX>(st[i], acc, src_lane, a.scale, sm, sinv);
        }
    }
    burst_reduce<SPLIT>(reinterpret_cast<float(&)[kBurstRed]>(acc), warp, lane);
    if (active && part == 0) f16_epilogue<1, FPL>(a, it, acc, feat0, g, t);
}

// TF32 (f32 gathers, 8-vector steps; the accumulator layout of
// tf32_epilogue<1>).
template <int SPLIT, int MAXS>
__global__ void __launch_bounds__(kBW * 32, (SPLIT > 1 ? kBurstBlocks : 4) * kWarps / kBW) spmm_tf32_burst(const SpmmArgs a) {
    static_assert(kBW % SPLIT == 0, "parts of an item share a CTA");
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t g = lane >> 2, t = lane & 3, q = lane >> 3, p = lane & 7, src_lane = 8 * t + g;
    const uint32_t part = warp % SPLIT;
    const uint64_t idx = (static_cast<uint64_t>(blockIdx.x) * kBW + warp) / SPLIT;
    const int64_t feat0 = static_cast<int64_t>(a.slab0 + blockIdx.y) * 32;
    const float* Bl = static_cast<const float*>(a.B) + feat0 + 4 * p;
    pdl_trigger();  // the next small-list kernel may be scheduled now ...
    pdl_wait();     // ... and this one touches memory only after its predecessor completed
    const bool active = idx < a.n_items;
    float acc[1][2][4] = {};
    WorkItem it{};
    if (active) {
        uint32_t base, nvw;
        it = burst_item(a, idx, base, nvw);
        const uint32_t* ci = a.ci + base;
        const uint64_t vbase = 8ull * base;
        const uint32_t steps = (it.vend - it.vbeg + 7) / 8, per = (steps + SPLIT - 1) / SPLIT;
        const uint32_t vend = min(it.vend, it.vbeg + 8 * per * (part + 1));
        for (uint32_t s0 = it.vbeg + 8 * per * part; s0 < vend; s0 += 8 * MAXS) {
            uint32_t cq[(MAXS + 3) / 4];
#pragma unroll
            for (int j = 0; j < (MAXS + 3) / 4; ++j) cq[j] = load_colpair(ci, s0 + 32 * j, vend, lane);
            Tf32Step<1> st[MAXS];
#pragma unroll
            for (int i = 0; i < MAXS; ++i)
                if (s0 + 8 * i < vend)
                    tf32_issue<1>(a, Bl, vbase, nvw, vend, s0 + 8 * i, g, t, q, cq[i / 4], i & 3, st[i]);
#pragma unroll
            for (int i = 0; i < MAXS; ++i)
                if (s0 + 8 * i < vend) tf32_compute<1>(st[i], acc, src_lane);
        }
    }
    burst_reduce<SPLIT>(reinterpret_cast<float(&)[kBurstRed]>(acc), warp, lane);
    if (active && part == 0) tf32_epilogue<1>(a, it, acc, feat0, g, t);
}

// Sums the segments of split windows in segment order (deterministic).
// n_split_dev (pipelined plans): the real count, on the device.  One CTA
// per split window, 4 features per thread, the segments' loads unrolled.
__global__ void __launch_bounds__(256) spmm_reduce_split(const SplitWindow* __restrict__ split, uint64_t n_split,
                                                         const float* __restrict__ partial, int64_t ldp, float* C,
                                                         int64_t ldc, uint64_t rows, int64_t N,
                                                         const uint32_t* __restrict__ n_split_dev = nullptr) {
    if (n_split_dev) n_split = *n_split_dev;
    const uint32_t q4 = static_cast<uint32_t>((N + 3) / 4);  // float4 groups per row (ldp % 4 == 0)
    for (uint64_t sw = blockIdx.x; sw < n_split; sw += gridDim.x) {
        const SplitWindow x = split[sw];
        for (uint32_t e = threadIdx.x; e < 8 * q4; e += blockDim.x) {
            const uint32_t r = e / q4, f = 4 * (e - r * q4);
            const uint64_t row = 8ull * x.window + r;
            if (row >= rows) continue;
            const float4* p = reinterpret_cast<const float4*>(partial + (uint64_t(x.first_slot) * 8 + r) * ldp + f);
            const uint64_t step = 2ull * ldp;  // one slot = 8 rows of ldp floats, in float4 units
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            uint32_t q = 0;
            for (; q + 4 <= x.nseg; q += 4) {
                const float4 a0 = p[(q + 0) * step], a1 = p[(q + 1) * step], a2 = p[(q + 2) * step],
                             a3 = p[(q + 3) * step];
                acc.x += a0.x; acc.y += a0.y; acc.z += a0.z; acc.w += a0.w;
                acc.x += a1.x; acc.y += a1.y; acc.z += a1.z; acc.w += a1.w;
                acc.x += a2.x; acc.y += a2.y; acc.z += a2.z; acc.w += a2.w;
                acc.x += a3.x; acc.y += a3.y; acc.z += a3.z; acc.w += a3.w;
            }
            for (; q < x.nseg; ++q) {
                const float4 a = p[q * step];
                acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
            }
            float* dst = C + row * ldc + f;
            const float v[4] = {acc.x, acc.y, acc.z, acc.w};
            for (int k = 0; k < 4 && f + k < N; ++k) dst[k] = v[k];
        }
    }
}

// Claim counters of a pipelined plan: every slab starts at the first real
// item (Plan::dcounts[0]; the list's real items end at its capacity).
__global__ void claim_init(uint32_t* __restrict__ counters, int slabs, const uint32_t* __restrict__ dcounts) {
    for (int i = threadIdx.x; i < slabs * int(dev::kClaimBytes / 4); i += blockDim.x)
        counters[i] = i % int(dev::kClaimBytes / 4) == 0 ? dcounts[0] : 0u;
}

// Persistent launch: `bps` CTAs (4 warps each) per SM, shared by the
// slabs; warps pull items from their slab's counter.
template <typename K>
void launch(K kernel, const SpmmArgs& a, int slabs, cudaStream_t s, const char* name, int bps = 4) {
    const uint64_t need = (a.n_items + kWarps - 1) / kWarps;
    const uint64_t per_slab = std::max<uint64_t>(1, uint64_t(num_sms()) * bps / std::max(1, slabs));
    const dim3 grid(static_cast<unsigned>(std::min(need, per_slab)), slabs);
    kernel<<<grid, kWarps * 32, 0, s>>>(a);
    TCS_LAUNCHED(name);
}

// ------------------------------------------- hot dense-operand rows (L2)
// When B does not fit in L2 (C4: 627 MB at N=128, C5: 537 MB at N=32) an
// LRU-like L2 keeps whatever was gathered last: ~25% hits on C4, although a
// power-law graph sends half its gathers to a few percent of the columns.
// The most-gathered columns whose rows fit TCS_HOT_BUDGET_MB are marked
// (Plan::col_hot, built once per handle from the column indices) and their
// gathers carry L2::evict_last, all others L2::evict_first.
#ifndef TCS_HOT_MIN_MB
#define TCS_HOT_MIN_MB 96
#endif
#ifndef TCS_HOT_BUDGET_MB
#define TCS_HOT_BUDGET_MB 64
#endif
constexpr int kHotBins = 4096;
constexpr uint64_t kPrefetchMaxB = uint64_t(TCS_PREFETCH_MAX_B_MB) << 20;

__global__ void col_count(const uint32_t* __restrict__ ci, uint64_t nv, uint32_t* __restrict__ cnt) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nv; p += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + ci[p], 1u);
}
__global__ void count_hist(const uint32_t* __restrict__ cnt, uint64_t cols, uint32_t* __restrict__ hist) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < cols; c += (uint64_t)gridDim.x * blockDim.x)
        if (cnt[c]) atomicAdd(hist + min(cnt[c], uint32_t(kHotBins - 1)), 1u);
}
__global__ void hot_bits(const uint32_t* __restrict__ cnt, uint64_t cols, uint32_t thr, uint32_t* __restrict__ bits) {
    const uint64_t words = (cols + 31) / 32;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t m = 0;
        for (uint32_t b = 0; b < 32 && 32 * w + b < cols; ++b) m |= uint32_t(cnt[32 * w + b] >= thr) << b;
        bits[w] = m;
    }
}

__global__ void mark_hot_cols(const uint32_t* __restrict__ ci, uint64_t nv, const uint32_t* __restrict__ bits,
                              uint32_t* __restrict__ out) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nv; p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = ci[p];
        out[p] = c | (((bits[c >> 5] >> (c & 31)) & 1u) << 31);
    }
}

// Plan::col_hot / Plan::ci_hot for rows of `rowbytes` (one host round trip,
// on first use); returns the marked column indices.
const uint32_t* col_hot(const tcs_mebcrs* A, Plan* plan, uint64_t rowbytes, cudaStream_t s) {
    if (plan->ci_hot && plan->col_hot_rowbytes == rowbytes) return plan->ci_hot;
    const uint64_t cols = A->cols, nv = A->num_vectors;
    DBuf cnt(std::max<uint64_t>(1, cols) * 4, s), hist(kHotBins * 4, s);
    TCS_CUDA(cudaMemsetAsync(cnt.p, 0, cols * 4, s));
    TCS_CUDA(cudaMemsetAsync(hist.p, 0, kHotBins * 4, s));
    const int sms = num_sms();
    col_count<<<sms * 8, 256, 0, s>>>(A->column_indices, nv, cnt.as<uint32_t>());
    TCS_LAUNCHED("col_count");
    count_hist<<<sms * 4, 256, 0, s>>>(cnt.as<uint32_t>(), cols, hist.as<uint32_t>());
    TCS_LAUNCHED("count_hist");
    std::vector<uint32_t> h(kHotBins);
    TCS_CUDA(cudaMemcpyAsync(h.data(), hist.p, kHotBins * 4, cudaMemcpyDeviceToHost, s));
    TCS_CUDA(cudaStreamSynchronize(s));
    // the largest set of most-gathered columns whose rows fit the budget
    const uint64_t budget = uint64_t(TCS_HOT_BUDGET_MB) << 20;
    uint32_t thr = kHotBins;  // nothing hot
    uint64_t rows = 0;
    for (int b = kHotBins - 1; b >= 2; --b) {  // a row gathered once gains nothing
        if ((rows + h[b]) * rowbytes > budget) break;
        rows += h[b];
        thr = b;
    }
    dfree(plan->col_hot, s);
    dfree(plan->ci_hot, s);
    plan->col_hot = static_cast<uint32_t*>(dalloc(((cols + 31) / 32) * 4 + 4, s));
    plan->ci_hot = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, nv) * 4, s));
    plan->col_hot_rowbytes = rowbytes;
    hot_bits<<<sms * 4, 256, 0, s>>>(cnt.as<uint32_t>(), cols, thr, plan->col_hot);
    TCS_LAUNCHED("hot_bits");
    mark_hot_cols<<<sms * 8, 256, 0, s>>>(A->column_indices, nv, plan->col_hot, plan->ci_hot);
    TCS_LAUNCHED("mark_hot_cols");
    return plan->ci_hot;
}

// Feature slab of one warp: 32 / 64 / 128.  Small item lists (BASELINE C1:
// 512 windows) leave most warp slots idle and each warp walks its window
// serially: 32-feature slabs give every window npad/32 warps (and the burst
// kernels below) while the whole launch still fits one wave.
int feature_slab(const Plan* plan, int64_t npad, tcs_precision prec, bool direct_map) {
    int slab = npad <= 32 ? 32 : npad <= 64 ? 64 : prec == TCS_FP16 ? TCS_SPMM_SLAB_F16 : TCS_SPMM_SLAB_TF32;
    if (npad > 32 && !direct_map && TCS_SMALL_SLAB32 && !plan->dcounts &&
        plan->n_items * uint64_t(npad / 32) <=
            uint64_t(num_sms()) * kWarps * (prec == TCS_FP16 ? TCS_SPMM_DEEP_BPS : tf32_blocks(1)))
        slab = 32;
    return slab;
}

// Burst kernels (above) for small lists: warps per item so that every
// (item, 32-feature slab) pair fits one wave; 0 = not a burst case.  Items
// are at most plan.seg vectors, so seg bounds the bursts per part.
#ifndef TCS_NO_BURST
#define TCS_NO_BURST 0
#endif
int burst_split(const Plan* plan, int slabs) {
    if (TCS_NO_BURST || plan->seg > 512) return 0;
    if (TCS_BURST_FORCE_SPLIT) return TCS_BURST_FORCE_SPLIT;
    const uint64_t w = plan->n_items * uint64_t(slabs), sms = uint64_t(num_sms());
    if (w * 4 <= sms * kBurstBlocks * kWarps) return 4;
    if (w * 2 <= sms * kBurstBlocks * kWarps) return 2;
    if (w <= sms * 4 * kWarps) return 1;
    return 0;
}

template <typename K>
void launch_burst(K kernel, const SpmmArgs& a, int split, int slabs, cudaStream_t s, const char* name) {
    const dim3 grid(static_cast<unsigned>((a.n_items * split + kBW - 1) / kBW), slabs);
    launch_pdl(kernel, grid, dim3(kBW * 32), 0, s, a);
    TCS_LAUNCHED(name);
}

}  // namespace

// C = softmax_rows(scale * S) . B for binary16 scores S whose dead slots are
// -inf (an SDDMM output with dead = -inf) and per-row statistics (m, 1/sum)
// from softmax_rowstats: the SpMM kernel applies the softmax to each sparse
// value in registers (SMX).  Same result, bit for bit, as normalising S into
// P with tcs_sddmm_row_softmax (binary16 P) and running tcs_spmm on P.
void spmm_f16_softmax(const tcs_mebcrs* S, const Plan* plan, const float2* rowstat, float scale, const void* b,
                      tcs_dtype b_dtype, int64_t ldb, int64_t b_rows, int64_t n, float* c, int64_t ldc,
                      cudaStream_t s) {
    if (n == 0 || S->rows == 0 || !plan->n_items) return;
    const int64_t npad = n <= 32 ? 32 : n <= 64 ? 64 : (n + 127) / 128 * 128;
    // the kernel choice of tcs_spmm on the same list (so the result equals
    // tcs_spmm on the materialised P bit for bit)
    const int slab = feature_slab(plan, npad, TCS_FP16, false);
    const bool direct = b_dtype == TCS_DTYPE_F16 && ldb % 8 == 0 && ldb >= npad &&
                        (reinterpret_cast<uintptr_t>(b) & 15) == 0;
    DBuf bpad;
    const void* bp = b;
    int64_t bld = ldb;
    if (!direct) {
        bld = npad;
        bpad = DBuf(static_cast<size_t>(std::max<int64_t>(1, b_rows)) * npad * 2, s);
        pad_convert(b, b_dtype, ldb, bpad.p, TCS_DTYPE_F16, npad, b_rows, n, npad, s);
        bp = bpad.p;
    }
    DBuf partial;
    if (plan->n_slots) partial = DBuf(plan->n_slots * 8 * npad * sizeof(float), s);
    const int slabs = static_cast<int>(npad / slab);
    if (const int split = slab == 32 ? burst_split(plan, slabs) : 0) {
        SpmmArgs a{plan->n_split ? plan->items : nullptr, plan->n_items, S->row_pointers, S->column_indices,
                   S->values, bp, bld, c, ldc, S->rows, n, partial.as<float>(), npad, nullptr, 0, rowstat, scale};
        if (split == 4) launch_burst(spmm_f16_burst<false, 4, 2, true>, a, 4, slabs, s, "spmm_f16_softmax_burst<4>");
        else if (split == 2) launch_burst(spmm_f16_burst<false, 2, 4, true>, a, 2, slabs, s, "spmm_f16_softmax_burst<2>");
        else launch_burst(spmm_f16_burst<false, 1, 8, true>, a, 1, slabs, s, "spmm_f16_softmax_burst<1>");
    } else {
    DBuf item_ctr(slabs * dev::kClaimBytes, s);
    TCS_CUDA(cudaMemsetAsync(item_ctr.p, 0, slabs * dev::kClaimBytes, s));
    SpmmArgs a{plan->items, plan->n_items, S->row_pointers, S->column_indices, S->values, bp, bld,
               c, ldc, S->rows, n, partial.as<float>(), npad, item_ctr.as<uint32_t>(), 0, rowstat, scale};
    if (slab == 128) launch(spmm_f16_kernel<2, 8, false, true>, a, slabs, s, "spmm_f16_softmax<128>");
    else if (slab == 64) launch(spmm_f16_kernel<1, 8, false, true>, a, slabs, s, "spmm_f16_softmax<64>", spmm_blocks(1, 8));
    else if (TCS_SPMM_DEEP32)
        launch(spmm_f16_kernel_deep<1, 4, false, true, TCS_SPMM_DEEP_BPS>, a, slabs, s, "spmm_f16_softmax_deep<32>",
               TCS_SPMM_DEEP_BPS);
    else launch(spmm_f16_kernel<1, 4, false, true>, a, slabs, s, "spmm_f16_softmax<32>", spmm_blocks(1, 4));
    }
    if (plan->n_split) {
        const int grid = static_cast<int>(std::min<uint64_t>(plan->n_split, uint64_t(num_sms()) * 8));
        spmm_reduce_split<<<grid, 256, 0, s>>>(plan->split, plan->n_split, partial.as<float>(), npad, c, ldc, S->rows,
                                              n);
        TCS_LAUNCHED("spmm_reduce_split");
    }
}

}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_spmm(const tcs_mebcrs* A, const void* b, tcs_dtype b_dtype, int64_t ldb, int64_t b_rows,
                               int64_t n, float* c, int64_t ldc, const tcs_kernel_config* cfg,
                               tcs_counters* counters, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm");
        if (!cfg) fail(TCS_ERR_ARGUMENT, "null kernel config");
        // ref spmm.hpp:106-109
        if (cfg->vector_height != 8) fail(TCS_ERR_ARGUMENT, "swap-and-transpose path requires vector height 8");
        check_mebcrs(A);
        if (cfg->precision != A->precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded matrix");
        if (static_cast<int64_t>(A->cols) != b_rows) fail(TCS_ERR_SHAPE, "sparse cols must equal dense rows");
        if (n < 0 || b_rows < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        if (n > 0 && A->rows > 0 && (!c || ldc < n)) fail(TCS_ERR_ARGUMENT, "bad output buffer / ldc");
        if (n > 0 && b_rows > 0 && (!b || ldb < n)) fail(TCS_ERR_ARGUMENT, "bad dense buffer / ldb");
        if (b_dtype != TCS_DTYPE_F16 && b_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown dtype");
        if (A->precision == TCS_TF32 && b_dtype != TCS_DTYPE_F32)
            fail(TCS_ERR_ARGUMENT, "TF32 SpMM needs an f32 dense operand");
        if (counters) {
            *counters = tcs_counters{};
        }
        cudaStream_t s = st(stream);
        if (n == 0 || A->rows == 0) return;

        Plan* plan = static_cast<Plan*>(A->plan);
        Plan* tmp_plan = nullptr;
        if (!plan) plan = tmp_plan = build_plan(A, s, nullptr, nullptr, nullptr);
        struct PlanGuard {
            Plan* p;
            cudaStream_t s;
            ~PlanGuard() { free_plan(p, s); }
        } pg{tmp_plan, s};

        // Feature padding: 32 / 64 / multiple of 128.
        const int64_t npad = n <= 32 ? 32 : n <= 64 ? 64 : (n + 127) / 128 * 128;
        const int slab = feature_slab(plan, npad, A->precision, cfg->mapping == TCS_MAP_DIRECT);
        const tcs_dtype need = A->precision == TCS_FP16 ? TCS_DTYPE_F16 : TCS_DTYPE_F32;
        const int64_t align_elems = need == TCS_DTYPE_F16 ? 8 : 4;
        const bool aligned = (reinterpret_cast<uintptr_t>(b) & 15) == 0;
        // Instruction path.  Default: warp mma.sync fed by quarter-warp-coalesced
        // LDG.128 gathers (measured faster on B200: 256-B row gathers are
        // TMA-op-rate bound, tools/gather_bench.cu).  tcgen05 + TMA gather4 on
        // request (FP16, binary16 values, N <= 256).
        const bool want_tc = A->precision == TCS_FP16 && A->value_dtype == TCS_DTYPE_F16 && n <= 256 &&
                             (cfg->flags & TCS_CFG_PATH_TCGEN05);
        if ((cfg->flags & TCS_CFG_PATH_TCGEN05) && !want_tc)
            fail(TCS_ERR_ARGUMENT, "tcgen05 path needs FP16 with binary16 values and N <= 256");
        // the TMA path reads B through a tensor map (OOB features zero-filled),
        // the mma.sync path needs rows padded to npad features
        const bool direct = b_dtype == need && ldb % align_elems == 0 && aligned && (want_tc || ldb >= npad);
        DBuf bpad;
        const void* bp = b;
        int64_t bld = ldb;
        if (!direct) {
            bld = npad;
            bpad = DBuf(static_cast<size_t>(std::max<int64_t>(1, b_rows)) * npad * (need == TCS_DTYPE_F16 ? 2 : 4), s);
            pad_convert(b, b_dtype, ldb, bpad.p, need, npad, b_rows, n, npad, s);
            bp = bpad.p;
        }
        DBuf partial;
        if (plan->n_slots) partial = DBuf(plan->n_slots * 8 * npad * sizeof(float), s);

        bool launched = false;
        if (want_tc)
            launched = spmm_tc05(A, plan, static_cast<const __half*>(bp), bld, b_rows, n, c, ldc, partial.as<float>(),
                                 npad, s);
        if (!launched && (cfg->flags & TCS_CFG_PATH_TCGEN05))
            fail(TCS_ERR_ARGUMENT, "tcgen05 path unavailable for these operands");
        if (!launched && bld < npad) {  // fall back to mma.sync: needs padded rows
            DBuf p2(static_cast<size_t>(std::max<int64_t>(1, b_rows)) * npad * 2, s);
            pad_convert(bp, TCS_DTYPE_F16, bld, p2.p, TCS_DTYPE_F16, npad, b_rows, n, npad, s);
            bpad = std::move(p2);
            bp = bpad.p;
            bld = npad;
        }
        const int slabs = static_cast<int>(npad / slab);
        const bool direct_map = cfg->mapping == TCS_MAP_DIRECT && A->precision == TCS_FP16;
        const int burst = plan->n_items && !launched && !direct_map && slab == 32 && !plan->dcounts
                              ? burst_split(plan, slabs) : 0;
        DBuf item_ctr;
        if (!launched && !burst && plan->n_items) {
            item_ctr = DBuf(slabs * dev::kClaimBytes, s);
            if (plan->dcounts) {
                claim_init<<<1, 256, 0, s>>>(item_ctr.as<uint32_t>(), slabs, plan->dcounts);
                TCS_LAUNCHED("claim_init");
            } else {
                TCS_CUDA(cudaMemsetAsync(item_ctr.p, 0, slabs * dev::kClaimBytes, s));
            }
        }
        SpmmArgs a{plan->items, plan->n_items, A->row_pointers, A->column_indices, A->values, bp, bld,
                   c, ldc, A->rows, n, partial.as<float>(), npad, item_ctr.as<uint32_t>()};
        if (plan->n_items && !launched && direct_map) {  // ablation: the paper's direct thread mapping
            const bool vf32 = A->value_dtype == TCS_DTYPE_F32;
            if (slab == 128)
                vf32 ? launch(spmm_f16_direct_kernel<8, true>, a, slabs, s, "spmm_f16_direct<128,f32v>")
                     : launch(spmm_f16_direct_kernel<8, false>, a, slabs, s, "spmm_f16_direct<128>");
            else if (slab == 64)
                vf32 ? launch(spmm_f16_direct_kernel<4, true>, a, slabs, s, "spmm_f16_direct<64,f32v>")
                     : launch(spmm_f16_direct_kernel<4, false>, a, slabs, s, "spmm_f16_direct<64>");
            else
                vf32 ? launch(spmm_f16_direct_kernel<2, true>, a, slabs, s, "spmm_f16_direct<32,f32v>")
                     : launch(spmm_f16_direct_kernel<2, false>, a, slabs, s, "spmm_f16_direct<32>");
        } else if (const int split = burst) {
            SpmmArgs ab = a;
            if (!plan->n_split) ab.items = nullptr;  // item i is window i
            ab.counter = nullptr;
            if (A->precision == TCS_FP16) {
                const bool vf32 = A->value_dtype == TCS_DTYPE_F32;
                if (split == 4)
                    vf32 ? launch_burst(spmm_f16_burst<true, 4, 2>, ab, 4, slabs, s, "spmm_f16_burst<4,f32v>")
                         : launch_burst(spmm_f16_burst<false, 4, 2>, ab, 4, slabs, s, "spmm_f16_burst<4>");
                else if (split == 2)
                    vf32 ? launch_burst(spmm_f16_burst<true, 2, 4>, ab, 2, slabs, s, "spmm_f16_burst<2,f32v>")
                         : launch_burst(spmm_f16_burst<false, 2, 4>, ab, 2, slabs, s, "spmm_f16_burst<2>");
                else
                    vf32 ? launch_burst(spmm_f16_burst<true, 1, 8>, ab, 1, slabs, s, "spmm_f16_burst<1,f32v>")
                         : launch_burst(spmm_f16_burst<false, 1, 8>, ab, 1, slabs, s, "spmm_f16_burst<1>");
            } else {
                if (split == 4) launch_burst(spmm_tf32_burst<4, 4>, ab, 4, slabs, s, "spmm_tf32_burst<4>");
                else if (split == 2) launch_burst(spmm_tf32_burst<2, 4>, ab, 2, slabs, s, "spmm_tf32_burst<2>");
                else launch_burst(spmm_tf32_burst<1, 8>, ab, 1, slabs, s, "spmm_tf32_burst<1>");
            }
        } else if (plan->n_items && !launched) {
            if (A->precision == TCS_FP16) {
                const bool vf32 = A->value_dtype == TCS_DTYPE_F32;
                const uint64_t b_bytes = uint64_t(b_rows) * npad * 2;  // the f16 operand as gathered
                // hot-row L2 policy: B larger than L2, binary16 values, a
                // plan with host-side counts (not a pipelined chunk)
                const bool hot = TCS_HOT && !vf32 && !plan->dcounts && (slab == 128 || slab == 32) &&
                                 uint64_t(b_rows) * npad * 2 > (uint64_t(TCS_HOT_MIN_MB) << 20);
                if (hot) a.ci = col_hot(A, plan, uint64_t(npad) * 2, s);
                if (hot && slab == 128)
                    launch(spmm_f16_kernel<2, 8, false, false, true>, a, slabs, s, "spmm_f16_hot<128>");
                else if (hot)
                    launch(spmm_f16_kernel_deep<1, 4, false, false, TCS_SPMM_DEEP_BPS, true>, a, slabs, s,
                           "spmm_f16_deep_hot<32>", TCS_SPMM_DEEP_BPS);
                else if (slab == 128 && !vf32 && TCS_PREFETCH_F16 > 0 && b_bytes <= kPrefetchMaxB)
                    launch(spmm_f16_kernel<2, 8, false, false, false, true>, a, slabs, s, "spmm_f16_pf<128>");
                else if (slab == 128)
                    vf32 ? launch(spmm_f16_kernel<2, 8, true>, a, slabs, s, "spmm_f16<128,f32v>")
                         : launch(spmm_f16_kernel<2, 8, false>, a, slabs, s, "spmm_f16<128>");
                else if (slab == 64 && !vf32 && TCS_PREFETCH_F16 > 0 && b_bytes <= kPrefetchMaxB)
                    launch(spmm_f16_kernel<1, 8, false, false, false, true>, a, slabs, s, "spmm_f16_pf<64>",
                           spmm_blocks(1, 8));
                else if (slab == 64)
                    vf32 ? launch(spmm_f16_kernel<1, 8, true>, a, slabs, s, "spmm_f16<64,f32v>", spmm_blocks(1, 8))
                         : launch(spmm_f16_kernel<1, 8, false>, a, slabs, s, "spmm_f16<64>", spmm_blocks(1, 8));
                else if (TCS_SPMM_DEEP32)
                    vf32 ? launch(spmm_f16_kernel_deep<1, 4, true, false, TCS_SPMM_DEEP_BPS>, a, slabs, s, "spmm_f16_deep<32,f32v>", TCS_SPMM_DEEP_BPS)
                         : launch(spmm_f16_kernel_deep<1, 4, false, false, TCS_SPMM_DEEP_BPS>, a, slabs, s, "spmm_f16_deep<32>", TCS_SPMM_DEEP_BPS);
                else
                    vf32 ? launch(spmm_f16_kernel<1, 4, true>, a, slabs, s, "spmm_f16<32,f32v>", spmm_blocks(1, 4))
                         : launch(spmm_f16_kernel<1, 4, false>, a, slabs, s, "spmm_f16<32>", spmm_blocks(1, 4));
            } else if (TCS_TF32_PACKED && slab >= 64 && !(cfg->flags & TCS_CFG_TF32_F32_GATHER)) {
                // dense operand repacked to 2.5 B per feature (see tf32_pack_kernel)
                const int64_t lds = npad * 5 / 2;
                DBuf packed(static_cast<size_t>(std::max<int64_t>(1, b_rows)) * lds, s);
                if (b_rows > 0) {
                    const int64_t total = b_rows * (npad / 8);
                    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, int64_t(num_sms()) * 16));
                    tf32_pack_kernel<<<grid, 256, 0, s>>>(static_cast<const float*>(bp), bld, b_rows, n, npad,
                                                          packed.as<unsigned char>(), lds,
                                                          slab == 128 && TCS_TF32P_LO64);
                    TCS_LAUNCHED("tf32_pack");
                }
                SpmmArgs ap = a;
                ap.B = packed.p;
                ap.ldb = lds;  // bytes
                const bool pf = TCS_PREFETCH_AHEAD > 0 && uint64_t(b_rows) * lds <= kPrefetchMaxB;
                if (slab == 128 && pf)
                    launch(spmm_tf32p_kernel<2, true>, ap, slabs, s, "spmm_tf32p_pf<128>", tf32p_blocks(2));
                else if (slab == 128) launch(spmm_tf32p_kernel<2>, ap, slabs, s, "spmm_tf32p<128>", tf32p_blocks(2));
                else if (pf && !TCS_TF32P_DEEP)
                    launch(spmm_tf32p_kernel<1, true>, ap, slabs, s, "spmm_tf32p_pf<64>", tf32p_blocks(1));
                else if (TCS_TF32P_DEEP)
                    launch(spmm_tf32p_deep, ap, slabs, s, "spmm_tf32p_deep<64>", TCS_TF32P_DEEP_BPS);
                else launch(spmm_tf32p_kernel<1>, ap, slabs, s, "spmm_tf32p<64>", tf32p_blocks(1));
            } else {
                if (slab == 128) launch(spmm_tf32_kernel<4>, a, slabs, s, "spmm_tf32<128>");
                else if (slab == 64) launch(spmm_tf32_kernel<2>, a, slabs, s, "spmm_tf32<64>", tf32_blocks(2));
                else launch(spmm_tf32_kernel<1>, a, slabs, s, "spmm_tf32<32>", tf32_blocks(1));
            }
        }
        if (plan->n_split) {
            const int grid = static_cast<int>(std::min<uint64_t>(plan->n_split, uint64_t(num_sms()) * 8));
            spmm_reduce_split<<<grid, 256, 0, s>>>(plan->split, plan->n_split, partial.as<float>(), npad, c, ldc,
                                                  A->rows, n, plan->dcounts ? plan->dcounts + 1 : nullptr);
            TCS_LAUNCHED("spmm_reduce_split");
        }
        if (counters) counters->mma_invocations = A->num_blocks * ((n + 15) / 16);  // ref analysis.hpp:34-38
        if (counters && (cfg->flags & TCS_CFG_COUNT_ACCESS)) {
            tcs_cost cost{};
            mebcrs_cost(A, 0, n, cfg->mapping, &cost, s);
            counters->transactions = cost.exec_transactions;
            counters->transaction_bytes = cost.exec_transaction_bytes;
            counters->useful_bytes = cost.exec_useful_bytes;
        }
    });
}

extern "C" tcs_status tcs_spmm_host(uint64_t rows, uint64_t cols, tcs_precision precision,
                                    const uint32_t* row_pointers, const uint32_t* column_indices, const float* values,
                                    const float* b, int64_t b_rows, int64_t n, float* c,
                                    const tcs_kernel_config* cfg, tcs_counters* counters, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_host");
        if (!cfg) fail(TCS_ERR_ARGUMENT, "null kernel config");
        if (cfg->vector_height != 8) fail(TCS_ERR_ARGUMENT, "swap-and-transpose path requires vector height 8");
        if (cfg->precision != precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded matrix");
        if (static_cast<int64_t>(cols) != b_rows) fail(TCS_ERR_SHAPE, "sparse cols must equal dense rows");
        cudaStream_t s = st(stream);
        tcs_mebcrs m{};
        tcs_status rc = tcs_mebcrs_upload(rows, cols, precision, row_pointers, column_indices, values, &m, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        struct Free {
            tcs_mebcrs* m;
            tcs_stream_t s;
            ~Free() { tcs_mebcrs_free(m, s); }
        } fr{&m, stream};
        DBuf db(std::max<int64_t>(1, b_rows * n) * 4, s), dc(std::max<uint64_t>(1, rows * n) * 4, s);
        if (b_rows > 0 && n > 0) TCS_CUDA(cudaMemcpyAsync(db.p, b, b_rows * n * 4, cudaMemcpyHostToDevice, s));
        rc = tcs_spmm(&m, db.p, TCS_DTYPE_F32, n, b_rows, n, dc.as<float>(), n, cfg, counters, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        if (rows > 0 && n > 0) TCS_CUDA(cudaMemcpyAsync(c, dc.p, rows * n * 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
    });
}

namespace tcs {
namespace {
__global__ void rebase_u32(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, uint64_t n, uint32_t sub) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] - sub;
}

// Compute streams the chunks alternate over.  Two (chunk i's SpMM running
// while the host waits in chunk i+1's encode) measured no faster than one on
// C3: each chunk's encode + SpMM starts when it lands and the tail is the
// last chunk's work either way.
// Compute streams of the pipeline: chunk i runs on stream i % S, so the
// small tail chunks (whose latency is mostly their largest window's) overlap.
#ifndef TCS_E2E_STREAMS
#define TCS_E2E_STREAMS 2
#endif
struct Streams {
    cudaStream_t copy = nullptr, drain = nullptr;
    cudaStream_t compute[TCS_E2E_STREAMS] = {};
    Streams() {
        TCS_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
        for (auto& c : compute) TCS_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
        TCS_CUDA(cudaStreamCreateWithFlags(&drain, cudaStreamNonBlocking));
    }
    ~Streams() {
        cudaStreamDestroy(copy);
        for (auto& c : compute) cudaStreamDestroy(c);
        cudaStreamDestroy(drain);
    }
};
// The pipeline's side streams, created once per host thread and device
// (stream creation costs tens of microseconds of host time per call).
Streams& thread_streams() {
    static thread_local std::unique_ptr<Streams> per_dev[64];
    int dev = 0;
    TCS_CUDA(cudaGetDevice(&dev));
    auto& p = per_dev[dev & 63];
    if (p) {  // a device reset since the last call invalidates the handles
        const cudaError_t e = cudaStreamQuery(p->copy);
        if (e != cudaSuccess && e != cudaErrorNotReady) {
            cudaGetLastError();
            p.reset();  // the handles died with the old context (their destroy calls just fail)
            cudaGetLastError();
        }
    }
    if (!p) p = std::make_unique<Streams>();
    return *p;
}
// TCS_E2E_TRACE=1 (environment): the host pipeline below prints when each
// chunk landed / was multiplied / was drained (diagnostics).
bool e2e_trace() {
    static const bool on = [] {
        const char* v = std::getenv("TCS_E2E_TRACE");
        return v && v[0] == '1';
    }();
    return on;
}
struct Event {
    cudaEvent_t e = nullptr;
    Event() { TCS_CUDA(cudaEventCreateWithFlags(&e, e2e_trace() ? cudaEventDefault : cudaEventDisableTiming)); }
    ~Event() { cudaEventDestroy(e); }
    void record(cudaStream_t s) { TCS_CUDA(cudaEventRecord(e, s)); }
    void wait_on(cudaStream_t s) { TCS_CUDA(cudaStreamWaitEvent(s, e, 0)); }
};
}  // namespace
}  // namespace tcs

// The reference CLI pipeline (encode_mebcrs + spmm) from host buffers,
// pipelined over window-range chunks: the copy stream uploads B then the
// chunks' CSR slices back to back at link speed; the compute stream converts
// and multiplies chunk i as soon as it has landed (conversion synchronises
// the compute stream only, uploads keep flowing); the drain stream copies
// each chunk's C rows back as soon as they are final.  Chunks are disjoint
// row ranges, so the result is identical to a single encode + spmm.
extern "C" tcs_status tcs_spmm_csr_host(const tcs_csr* host_csr, tcs_precision precision, const float* b, int64_t n,
                                        float* c, const tcs_kernel_config* cfg, tcs_counters* counters,
                                        tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_spmm_csr_host");
        if (!host_csr || !cfg || !host_csr->row_ptr) fail(TCS_ERR_ARGUMENT, "null argument");
        if (cfg->vector_height != 8) fail(TCS_ERR_ARGUMENT, "swap-and-transpose path requires vector height 8");
        if (cfg->precision != precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded matrix");
        if (n < 0) fail(TCS_ERR_SHAPE, "negative dimension");
        if (counters) *counters = tcs_counters{};
        cudaStream_t s = st(stream);
        const uint64_t rows = host_csr->rows, nnz = host_csr->nnz, W = (rows + 7) / 8;
        const int64_t b_rows = static_cast<int64_t>(host_csr->cols);
        const uint32_t* hrp = host_csr->row_ptr;
        if (hrp[0] != 0 || hrp[rows] != nnz) fail(TCS_ERR_FORMAT, "row_ptr endpoints inconsistent with nnz");
        if (rows == 0 || n == 0) {
            for (uint64_t r = 0; r < rows; ++r)
                if (hrp[r + 1] < hrp[r]) fail(TCS_ERR_FORMAT, "row_ptr must be nondecreasing");
            return;
        }
        const uint64_t max_chunks = TCS_E2E_MAX_CHUNKS + TCS_E2E_TAIL_HALVINGS + 1;

        // device buffers, allocated in `stream` order before the fork
        const bool f16 = precision == TCS_FP16;
        DBuf d_rp_all((rows + 1) * 4, s), d_rp((rows + max_chunks) * 4, s), d_ci(std::max<uint64_t>(1, nnz) * 4, s),
            d_v(std::max<uint64_t>(1, nnz) * 4, s), d_b32(std::max<int64_t>(1, b_rows * n) * 4, s),
            d_c(rows * n * 4, s);
        DBuf d_b16;
        if (f16) d_b16 = DBuf(std::max<int64_t>(1, b_rows * n) * 2, s);
        // pipelined chunks (no host round trip per chunk) unless the tcgen05
        // path is requested (its launcher sizes the work list on the host)
        const bool pipelined = !(cfg->flags & TCS_CFG_PATH_TCGEN05);
        // per-chunk encode validation blocks, zeroed once
        const size_t chk_bytes = encode_check_bytes();
        DBuf d_checks(max_chunks * chk_bytes, s), d_blocks(max_chunks * 8, s);
        TCS_CUDA(cudaMemsetAsync(d_checks.p, 0, max_chunks * chk_bytes, s));
        Streams& ss = thread_streams();
        // On any exit (an error in a later chunk included) the side streams'
        // queued copies and kernels finish before the buffers above are
        // released in `stream` order and before control returns to the
        // caller (the drain stream writes into the caller's host C).
        struct Join {
            Streams& ss;
            bool joined = false;
            ~Join() {
                if (joined) return;
                cudaStreamSynchronize(ss.copy);
                for (auto c : ss.compute) cudaStreamSynchronize(c);
                cudaStreamSynchronize(ss.drain);
            }
        } join{ss};
        Event forked;
        forked.record(s);
        forked.wait_on(ss.copy);
        for (auto c : ss.compute) forked.wait_on(c);
        forked.wait_on(ss.drain);

        // B first: its upload hides the host work below
        if (b_rows > 0) TCS_CUDA(cudaMemcpyAsync(d_b32.p, b, b_rows * n * 4, cudaMemcpyHostToDevice, ss.copy));
        Event b_ready;
        b_ready.record(ss.copy);

        // row_ptr is validated here, on the host (the chunk cuts and copies
        // depend on it); column indices are validated by the chunk encodes
        for (uint64_t r = 0; r < rows; ++r)
            if (hrp[r + 1] < hrp[r]) fail(TCS_ERR_FORMAT, "row_ptr must be nondecreasing");

        // Chunk cut points: windows at nnz quantiles (host row_ptr).  The
        // encode of a chunk needs no host round trip (encode_mebcrs_async),
        // so every chunk's work is queued up front and runs as soon as its
        // upload lands; only the last chunk's encode + SpMM + download is
        // exposed after the last upload, so the last unit of work is cut
        // into halves: 1/2, 1/4, ..., 1/2^T, 1/2^T of a unit.
        const uint64_t units = std::max<uint64_t>(
            1, std::min<uint64_t>({TCS_E2E_MAX_CHUNKS, W, nnz / (TCS_E2E_CHUNK_NNZ) + 1}));
        const int tail = units > 1 && W > units + TCS_E2E_TAIL_HALVINGS ? TCS_E2E_TAIL_HALVINGS : 0;
        std::vector<double> frac;  // cumulative nnz fraction at each cut
        for (uint64_t i = 1; i < units; ++i) frac.push_back(double(i) / units);
        for (int h = 1; h <= tail; ++h) frac.push_back((units - std::ldexp(1.0, -h)) / units);
        const uint64_t nchunks = frac.size() + 1;
        std::vector<uint64_t> wcut(nchunks + 1, 0);
        for (uint64_t i = 1; i < nchunks; ++i) {
            const uint64_t target = static_cast<uint64_t>(frac[i - 1] * double(nnz));
            uint64_t lo = wcut[i - 1], hi = W;  // first window whose start >= target
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if (hrp[std::min(rows, 8 * mid)] < target) lo = mid + 1;
                else hi = mid;
            }
            wcut[i] = lo;
        }
        wcut[nchunks] = W;

        // row_ptr in one copy; per chunk its column indices, then its values
        // (the chunk's ranking kernels need only the former)
        std::vector<Event> cols_in(nchunks), landed(nchunks), done(nchunks), encoded(e2e_trace() ? nchunks : 0);
        TCS_CUDA(cudaMemcpyAsync(d_rp_all.p, hrp, (rows + 1) * 4, cudaMemcpyHostToDevice, ss.copy));
        for (uint64_t i = 0; i < nchunks; ++i) {
            const uint64_t r0 = std::min(rows, 8 * wcut[i]), r1 = std::min(rows, 8 * wcut[i + 1]);
            const uint64_t e0 = hrp[r0], e1 = hrp[r1];
            if (e1 > e0)
                TCS_CUDA(cudaMemcpyAsync(d_ci.as<uint32_t>() + e0, host_csr->col_idx + e0, (e1 - e0) * 4,
                                         cudaMemcpyHostToDevice, ss.copy));
            cols_in[i].record(ss.copy);
            if (e1 > e0)
                TCS_CUDA(cudaMemcpyAsync(d_v.as<float>() + e0, host_csr->values + e0, (e1 - e0) * 4,
                                         cudaMemcpyHostToDevice, ss.copy));
            landed[i].record(ss.copy);
        }
        // dense operand in the kernel's storage type, once
        b_ready.wait_on(ss.compute[0]);
        const void* bdev = d_b32.p;
        tcs_dtype bdt = TCS_DTYPE_F32;
        if (f16) {
            pad_convert(d_b32.p, TCS_DTYPE_F32, n, d_b16.p, TCS_DTYPE_F16, n, b_rows, n, n, ss.compute[0]);
            bdev = d_b16.p;
            bdt = TCS_DTYPE_F16;
        }
        Event b_conv;
        b_conv.record(ss.compute[0]);
        for (int q = 1; q < TCS_E2E_STREAMS; ++q) b_conv.wait_on(ss.compute[q]);
        for (uint64_t i = 0; i < nchunks; ++i) {
            const uint64_t r0 = std::min(rows, 8 * wcut[i]), r1 = std::min(rows, 8 * wcut[i + 1]);
            const uint64_t e0 = hrp[r0], e1 = hrp[r1];
            cudaStream_t cs = ss.compute[i % TCS_E2E_STREAMS];
            tcs_stream_t ks = reinterpret_cast<tcs_stream_t>(cs);
            cols_in[i].wait_on(cs);
            uint32_t* rp_i = d_rp.as<uint32_t>() + r0 + i;  // the chunk's row_ptr, rebased to 0
            rebase_u32<<<static_cast<unsigned>(std::min<uint64_t>((r1 - r0 + 256) / 256, 1024)), 256, 0, cs>>>(
                d_rp_all.as<uint32_t>() + r0, rp_i, r1 - r0 + 1, static_cast<uint32_t>(e0));
            TCS_LAUNCHED("rebase_u32");
            tcs_csr chunk{r1 - r0, host_csr->cols, e1 - e0, rp_i, d_ci.as<uint32_t>() + e0, d_v.as<float>() + e0};
            tcs_mebcrs m{};
            tcs_status rc = TCS_OK;
            if (pipelined) {
                encode_mebcrs_async(&chunk, precision, f16 ? TCS_DTYPE_F16 : TCS_DTYPE_F32, &m, cs,
                                    d_checks.as<unsigned char>() + i * chk_bytes, 0, landed[i].e);
            } else {
                landed[i].wait_on(cs);
                rc = tcs_mebcrs_encode(&chunk, precision, f16 ? TCS_DTYPE_F16 : TCS_DTYPE_F32, &m, ks);
                if (rc != TCS_OK) fail(rc, tcs_last_error());
            }
            if (e2e_trace()) encoded[i].record(cs);
            tcs_counters cn{};
            rc = tcs_spmm(&m, bdev, bdt, n, b_rows, n, d_c.as<float>() + r0 * n, n, cfg, counters ? &cn : nullptr, ks);
            if (rc == TCS_OK && pipelined && counters)  // this chunk's k-block count, read once at the end
                rc = cudaMemcpyAsync(d_blocks.as<uint64_t>() + i, static_cast<Plan*>(m.plan)->dcounts + 2, 8,
                                     cudaMemcpyDeviceToDevice, cs) == cudaSuccess ? TCS_OK : TCS_ERR_CUDA;
            tcs_mebcrs_free(&m, ks);
            if (rc != TCS_OK) fail(rc, tcs_last_error());
            if (counters && !pipelined) counters->mma_invocations += cn.mma_invocations;
            done[i].record(cs);
            done[i].wait_on(ss.drain);
            if (TCS_E2E_DRAIN_LATE) landed[nchunks - 1].wait_on(ss.drain);  // diagnostic: downloads after all uploads
            TCS_CUDA(cudaMemcpyAsync(c + r0 * n, d_c.as<float>() + r0 * n, (r1 - r0) * n * 4, cudaMemcpyDeviceToHost,
                                     ss.drain));
        }
        Event joined_copy, joined_drain;
        Event joined_compute[TCS_E2E_STREAMS];
        if (e2e_trace()) {
            std::vector<Event> drained(1);
            drained[0].record(ss.drain);
            TCS_CUDA(cudaStreamSynchronize(ss.drain));
            for (auto c : ss.compute) TCS_CUDA(cudaStreamSynchronize(c));
            auto ms = [&](const Event& x) {
                float t = 0.f;
                cudaEventElapsedTime(&t, forked.e, x.e);
                return t;
            };
            std::fprintf(stderr, "[tcs e2e] %llu chunks, B landed %.3f ms\n", (unsigned long long)nchunks, ms(b_ready));
            for (uint64_t i = 0; i < nchunks; ++i)
                std::fprintf(stderr, "[tcs e2e] chunk %llu: landed %.3f  encoded %.3f  computed %.3f\n",
                             (unsigned long long)i, ms(landed[i]), ms(encoded[i]), ms(done[i]));
            std::fprintf(stderr, "[tcs e2e] drained %.3f ms\n", ms(drained[0]));
        }
        joined_copy.record(ss.copy);
        for (int q = 0; q < TCS_E2E_STREAMS; ++q) joined_compute[q].record(ss.compute[q]);
        joined_drain.record(ss.drain);
        joined_copy.wait_on(s);
        for (auto& e : joined_compute) e.wait_on(s);
        joined_drain.wait_on(s);
        join.joined = true;
        std::vector<unsigned char> checks(nchunks * chk_bytes, 0);
        std::vector<uint64_t> blocks(nchunks, 0);
        if (pipelined) {
            TCS_CUDA(cudaMemcpyAsync(checks.data(), d_checks.p, nchunks * chk_bytes, cudaMemcpyDeviceToHost, s));
            if (counters)
                TCS_CUDA(cudaMemcpyAsync(blocks.data(), d_blocks.p, nchunks * 8, cudaMemcpyDeviceToHost, s));
        }
        TCS_CUDA(cudaStreamSynchronize(s));
        for (uint64_t i = 0; i < nchunks; ++i) {  // the first invalid chunk's validation code (encode.cu kBadMsg)
            uint32_t bad = 0;
            std::memcpy(&bad, checks.data() + i * chk_bytes + encode_check_bad_offset(), 4);
            if (bad) fail(TCS_ERR_FORMAT, encode_bad_msg(bad));
        }
        if (counters && pipelined)
            for (uint64_t i = 0; i < nchunks; ++i) counters->mma_invocations += blocks[i] * ((n + 15) / 16);
    });
}
