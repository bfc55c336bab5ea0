// SDDMM over the ME-BCRS mask with the same 8x1 granularity
// (ref sddmm.hpp:84-136, paper §3.4):
//
//   acc^T (16 vectors x 8 window rows) += Bt_gathered (16 vectors x K)
//                                         * A_window^T (K x 8 rows)
//
// i.e. the sampled B columns are the m=16 operand and the window's 8 A rows
// the n=8 operand -- the orientation of ref sddmm.hpp:107-120.  One warp owns
// one work item (<= plan.seg vectors of one window); each group of 16
// consecutive vectors (ref :104) is one accumulator tile.
//
// The inner (feature) dimension is permuted identically in both operands so
// every lane reads 16 contiguous bytes per gathered row (FP16: features
// 8t..8t+7 feed two m16n8k16 MMAs; TF32: 4t..4t+3 feed two m16n8k8 MMAs).
// Features are zero-padded (0*0 adds exactly 0, as the reference's padded
// K tiles, ref :110-118).
//
// Write-back follows Algorithm 1 (ref sddmm.hpp:28-63): accumulator element
// (vector v, row r) lands at 8*(rp[w]+b*k) + r*width_b + v%k, b = v/k; it is
// written only where the mask's stored value is != 0 (ref :131) and every
// other slot of the output blocks is 0.
#include <algorithm>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

using namespace dev;

#ifndef TCS_SDDMM_BPS1
#define TCS_SDDMM_BPS1 4
#endif
#ifndef TCS_SDDMM_NSC4
#define TCS_SDDMM_NSC4 1
#endif

struct SddmmArgs {
    const WorkItem* items;
    uint64_t n_items;
    const uint32_t* rp;
    const uint32_t* ci;
    const void* mask;   // mask values (F16 or F32)
    const void* A;      // [rows][lda], feature padded
    int64_t lda;
    const void* Bt;     // [cols][ldbt], feature padded
    int64_t ldbt;
    void* out;          // output values (F16 or F32)
    uint64_t rows;
    int passes;         // feature passes of NSC super-chunks
    uint32_t k;         // storage block width (8 / 4)
    uint32_t* counter;  // claim counters, dev::kClaimBytes (zeroed before launch)
    float dead;         // value of stored slots whose mask value is 0: 0, or -inf for the fused softmax
    const uint8_t* live;  // per-vector liveness bytes (bit r: row r's mask value != 0), mask mode kLive
    uint32_t sub;         // warps per work item (burst kernel only; 1 otherwise)
};

// Mask modes (template parameter MM): how a slot's liveness is read.
constexpr int kMaskF16 = 0;   // the mask's binary16 values
constexpr int kMaskF32 = 1;   // the mask's binary32 values
constexpr int kLive = 2;      // one liveness byte per stored vector (TCS_CFG_STATIC_MASK)

constexpr int kWarps = 4;
constexpr int kRing = 4;  // column-index batches staged per warp
// Resident CTAs per SM (sets the register budget): 4 (128 registers) for
// single-pass inner dimensions, 3 when two super-chunks are double-buffered.
template <int NSC>
constexpr int kMinBlocks = NSC == 1 ? TCS_SDDMM_BPS1 : 3;
// Groups per double-buffered batch: the register budget of a batch is about
// constant (NSC * D super-chunk tiles).
template <int NSC>
constexpr int kBatchGroups = NSC == 1 ? 4 : NSC == 2 ? 2 : 1;

// Storage position of accumulator element q (vector g or g+8, row 2t or
// 2t+1) of the group at s.  K (storage block width) is a compile-time
// constant.  Full groups use Algorithm 1's offsets (ref sddmm.hpp:28-33):
// inside the 16-vector group's 128 contiguous values, vector v / row r sits
// at 8K*(v/K) + K*r + v%K; a narrow last block uses its block_width
// (ref sddmm.hpp:125-130).
template <uint32_t K>
__device__ __forceinline__ uint64_t acc_pos(uint64_t vbase, uint32_t nvw, uint32_t s, bool full, uint32_t g,
                                            uint32_t t, int q) {
    const uint32_t vl = g + (q >= 2 ? 8u : 0u);  // vector within the group
    const uint32_t r = 2 * t + (q & 1);
    if (full) return vbase + 8ull * s + 8 * K * (vl / K) + K * r + (vl % K);
    const uint32_t v = s + vl;
    const uint32_t b = v / K, j = v % K, width = min(K, nvw - b * K);
    return vbase + 8ull * b * K + r * width + j;
}

// Liveness bits of the mask values at the group's 4 accumulator positions
// (nonzero magnitude == the reference's `mask.values[pos] != 0`; -0.0 is not
// live, ref sddmm.hpp:131).  Issued one group ahead of use.
// Mask words per group and lane: 4 f32 or 4 packed f16 values.
template <int MM>
constexpr int kMaskWords = MM == kMaskF32 ? 4 : MM == kMaskF16 ? 2 : 1;

template <uint32_t K, int MM>
__device__ __forceinline__ void mask_prefetch(const SddmmArgs& a, uint64_t vbase, uint32_t nvw, uint32_t vend,
                                              uint32_t s, uint32_t g, uint32_t t,
                                              uint32_t (&mk)[kMaskWords<MM>]) {
    const bool full = s + 16 <= vend;
#pragma unroll
    for (int w = 0; w < kMaskWords<MM>; ++w) mk[w] = 0u;
    if constexpr (MM == kLive) {  // bytes of vectors g (bits 0-7) and g + 8 (bits 8-15)
        const uint8_t* lv = a.live + vbase / 8;
        if (s + g < vend) mk[0] = __ldg(lv + s + g);
        if (s + g + 8 < vend) mk[0] |= static_cast<uint32_t>(__ldg(lv + s + g + 8)) << 8;
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t v = s + g + (q >= 2 ? 8u : 0u);
            if (v < vend) {
                const uint64_t pos = acc_pos<K>(vbase, nvw, s, full, g, t, q);
                // raw bits only: the liveness test happens at store time, so the
                // load stays in flight until then
                if constexpr (MM == kMaskF32) mk[q] = __float_as_uint(__ldg(static_cast<const float*>(a.mask) + pos));
                else mk[q >> 1] |= static_cast<uint32_t>(__ldg(static_cast<const unsigned short*>(a.mask) + pos))
                                   << (16 * (q & 1));
            }
        }
    }
}

// Liveness bits (bit q) of lane (g,t)'s accumulator elements from the two
// liveness bytes of vectors g (b0) and g + 8 (b1): rows 2t, 2t+1.
__device__ __forceinline__ uint32_t live_bits(uint32_t b0, uint32_t b1, uint32_t t) {
    return ((b0 >> (2 * t)) & 3u) | (((b1 >> (2 * t)) & 3u) << 2);
}

// Output values are written once and not re-read by this kernel: streaming
// (evict-first) stores keep L2 for the gathered rows and the mask stream
// (C3 F=32 1.345 -> 1.29 ms, C5 4.30 -> 4.17 ms; profiles/r1s4_sddmm_stream_stores.txt).
// TCS_SDDMM_STREAM_OUT=0 restores plain stores (A/B knob).
#ifndef TCS_SDDMM_STREAM_OUT
#define TCS_SDDMM_STREAM_OUT 1
#endif
template <bool OF32>
__device__ __forceinline__ void out_store(void* out, uint64_t pos, float v) {
#if TCS_SDDMM_STREAM_OUT
    if constexpr (OF32) __stcs(static_cast<float*>(out) + pos, v);
    else __stcs(reinterpret_cast<unsigned short*>(out) + pos, __half_as_ushort(__float2half_rn(v)));
#else
    if constexpr (OF32) static_cast<float*>(out)[pos] = v;
    else static_cast<__half*>(out)[pos] = __float2half_rn(v);
#endif
}

// Liveness bits (bit q) of lane (g,t)'s accumulator elements in a general
// group; elements past the item's last vector are not live.
template <int MM>
__device__ __forceinline__ uint32_t slow_live(const uint32_t (&mk)[kMaskWords<MM>], uint32_t s, uint32_t vend,
                                              uint32_t g, uint32_t t) {
    uint32_t bits = 0;
    if constexpr (MM == kLive) {
        bits = live_bits(mk[0] & 0xFFu, mk[0] >> 8, t);  // bytes past vend were left 0
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t v = s + g + (q >= 2 ? 8u : 0u);
            const bool live = v < vend && (MM == kMaskF32 ? (mk[q] & 0x7FFFFFFFu) != 0u
                                                          : ((mk[q >> 1] >> (16 * (q & 1))) & 0x7FFFu) != 0u);
            bits |= static_cast<uint32_t>(live) << q;
        }
    }
    return bits;
}

// Writes the 16x8 accumulator tile of the general group starting at s:
// live elements get their value, the other stored slots `dead`.
template <uint32_t K, bool OF32>
__device__ __forceinline__ void sddmm_store(void* out, const float (&acc)[4], uint32_t live, float dead,
                                            uint64_t vbase, uint32_t nvw, uint32_t vend, uint32_t s, uint32_t g,
                                            uint32_t t) {
    const bool full = s + 16 <= vend;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t v = s + g + (q >= 2 ? 8u : 0u);
        if (v >= vend) continue;
        out_store<OF32>(out, acc_pos<K>(vbase, nvw, s, full, g, t, q), (live >> q) & 1u ? acc[q] : dead);
    }
}

// ---- full groups (all 16 vectors inside full-width blocks): the group's
// 128 output/mask slots are contiguous; accumulator element q of lane (g,t)
// sits at slot full_pos(g,t,q) of them.
template <uint32_t K>
__device__ __forceinline__ uint32_t full_pos(uint32_t g, uint32_t t, int q) {
    if constexpr (K == 8) return 64u * (q >> 1) + 16u * t + 8u * (q & 1) + g;
    else return 32u * (g >> 2) + 64u * (q >> 1) + 8u * t + 4u * (q & 1) + (g & 3);
}

// Liveness bits (bit q) of lane (g,t)'s accumulator elements, read from the
// group's 128 mask values staged in shared memory.
template <uint32_t K, int MM>
__device__ __forceinline__ uint32_t ring_live(const unsigned char* m, uint32_t g, uint32_t t) {
    uint32_t bits = 0;
    if constexpr (MM == kLive) {
        bits = live_bits(m[g], m[g + 8], t);  // m: the group's 16 liveness bytes
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t p = full_pos<K>(g, t, q);
            const bool live = MM == kMaskF32 ? (reinterpret_cast<const uint32_t*>(m)[p] & 0x7FFFFFFFu) != 0u
                                             : (reinterpret_cast<const unsigned short*>(m)[p] & 0x7FFFu) != 0u;
            bits |= static_cast<uint32_t>(live) << q;
        }
    }
    return bits;
}

template <uint32_t K, bool OF32>
__device__ __forceinline__ void full_store(void* out, uint64_t slot0, const float (&acc)[4], uint32_t live,
                                           float dead, uint32_t g, uint32_t t) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
        out_store<OF32>(out, slot0 + full_pos<K>(g, t, q), (live >> q) & 1u ? acc[q] : dead);
}

// Bytes of one ring slot: BV column indices + BV*8 mask values, or BV
// liveness bytes + one spare word (they are copied as aligned 4-byte words).
template <int NSC, int MM>
constexpr uint32_t ring_slot_bytes() {
    constexpr uint32_t BV = 16u * kBatchGroups<NSC>;
    return MM == kLive ? (BV * 4u + BV + 4u + 15u) / 16u * 16u : BV * (4u + 8u * (MM == kMaskF32 ? 4u : 2u));
}

// ---------------------------------------------------------------- FP16
template <int NSC>
struct F16Tile {
    uint4 q0[NSC], q1[NSC];  // Bt rows of vectors g, g+8 (the window's A row g is hoisted per item)
};

template <int NSC>
__device__ __forceinline__ void f16_tile_load(const SddmmArgs& a, uint32_t c0, bool ok0, uint32_t c1, bool ok1,
                                              int pass, uint32_t t, F16Tile<NSC>& x) {
    const __half* bt = static_cast<const __half*>(a.Bt);
#pragma unroll
    for (int sc = 0; sc < NSC; ++sc) {
        const int64_t f = (static_cast<int64_t>(pass) * NSC + sc) * 32 + 8 * t;
        x.q0[sc] = ok0 ? ld_gather_128(bt + static_cast<uint64_t>(c0) * a.ldbt + f) : make_uint4(0, 0, 0, 0);
        x.q1[sc] = ok1 ? ld_gather_128(bt + static_cast<uint64_t>(c1) * a.ldbt + f) : make_uint4(0, 0, 0, 0);
    }
}

// A row g of the window, features of pass `pass` (same K permutation as the tiles).
template <int NSC, typename Elem>
__device__ __forceinline__ void arow_load(const Elem* __restrict__ arow, bool ok, int pass, uint32_t t,
                                          uint4 (&ar)[NSC]) {
    constexpr int SC = sizeof(Elem) == 2 ? 32 : 16;  // features per super-chunk
    constexpr int PER_LANE = sizeof(Elem) == 2 ? 8 : 4;
#pragma unroll
    for (int sc = 0; sc < NSC; ++sc) {
        const int64_t f = (static_cast<int64_t>(pass) * NSC + sc) * SC + PER_LANE * t;
        ar[sc] = ok ? ld_gather_128(arow + f) : make_uint4(0, 0, 0, 0);
    }
}

template <int NSC>
__device__ __forceinline__ void f16_tile_mma(const F16Tile<NSC>& x, const uint4 (&ar)[NSC], float (&acc)[4]) {
#pragma unroll
    for (int sc = 0; sc < NSC; ++sc) {
        // chunk 0: k = {2t,2t+1} <-> features 8t+0,1 ; k = {2t+8,2t+9} <-> 8t+2,3
        mma_f16_16816(acc, x.q0[sc].x, x.q1[sc].x, x.q0[sc].y, x.q1[sc].y, ar[sc].x, ar[sc].y);
        // chunk 1: features 8t+4,5 and 8t+6,7
        mma_f16_16816(acc, x.q0[sc].z, x.q1[sc].z, x.q0[sc].w, x.q1[sc].w, ar[sc].z, ar[sc].w);
    }
}

// ---------------------------------------------------------------- TF32
template <int NSC>
struct Tf32Tile {
    uint4 q0[NSC], q1[NSC];  // 4 f32 features each
};

template <int NSC>
__device__ __forceinline__ void tf32_tile_load(const SddmmArgs& a, uint32_t c0, bool ok0, uint32_t c1, bool ok1,
                                               int pass, uint32_t t, Tf32Tile<NSC>& x) {
    const float* bt = static_cast<const float*>(a.Bt);
#pragma unroll
    for (int sc = 0; sc < NSC; ++sc) {
        const int64_t f = (static_cast<int64_t>(pass) * NSC + sc) * 16 + 4 * t;
        x.q0[sc] = ok0 ? ld_gather_128(bt + static_cast<uint64_t>(c0) * a.ldbt + f) : make_uint4(0, 0, 0, 0);
        x.q1[sc] = ok1 ? ld_gather_128(bt + static_cast<uint64_t>(c1) * a.ldbt + f) : make_uint4(0, 0, 0, 0);
    }
}

__device__ __forceinline__ uint32_t tf(uint32_t bits) { return to_tf32(__uint_as_float(bits)); }

template <int NSC>
__device__ __forceinline__ void tf32_tile_mma(const Tf32Tile<NSC>& x, const uint4 (&ar)[NSC], float (&acc)[4]) {
#pragma unroll
    for (int sc = 0; sc < NSC; ++sc) {
        // chunk 0: k = t <-> feature 4t, k = t+4 <-> 4t+1 ; chunk 1: 4t+2, 4t+3
        mma_tf32_1688(acc, tf(x.q0[sc].x), tf(x.q1[sc].x), tf(x.q0[sc].y), tf(x.q1[sc].y), tf(ar[sc].x),
                      tf(ar[sc].y));
        mma_tf32_1688(acc, tf(x.q0[sc].z), tf(x.q1[sc].z), tf(x.q0[sc].w), tf(x.q1[sc].w), tf(ar[sc].z),
                      tf(ar[sc].w));
    }
}

// One kernel body for both precisions; Tile/loader/mma chosen by TF32.
template <bool TF32, int NSC, int MM, bool OF32>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks<NSC>) sddmm_kernel(const SddmmArgs a) {
    using Elem = typename std::conditional<TF32, float, __half>::type;
    using Tile = typename std::conditional<TF32, Tf32Tile<NSC>, F16Tile<NSC>>::type;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t g = lane >> 2, t = lane & 3;
    extern __shared__ __align__(16) unsigned char ring_all[];  // per-warp ring, see below
    // persistent warps pulling work items (dev::StripedClaim)
    dev::StripedClaim<4> claim;
    for (uint32_t idx; claim.get(a.counter, a.n_items, idx);) {
    const WorkItem it = a.items[idx];
    const uint32_t base = __ldg(a.rp + it.window);
    const uint32_t nvw = __ldg(a.rp + it.window + 1) - base;
    const uint32_t* ci = a.ci + base;
    const uint64_t vbase = 8ull * base;
    const uint32_t vbeg = it.vbeg, vend = it.vend;
    const uint64_t arow_i = 8ull * it.window + g;
    const bool arow_ok = arow_i < a.rows;
    const Elem* arow = static_cast<const Elem*>(a.A) + (arow_ok ? arow_i : 0) * a.lda;

    auto load = [&](uint32_t s, const uint32_t (&c)[2], int pass, Tile& x) {
        if constexpr (TF32)
            tf32_tile_load<NSC>(a, c[0], s + g < vend, c[1], s + g + 8 < vend, pass, t, x);
        else
            f16_tile_load<NSC>(a, c[0], s + g < vend, c[1], s + g + 8 < vend, pass, t, x);
    };
    auto mma = [&](const Tile& x, const uint4 (&ar)[NSC], float (&acc)[4]) {
        if constexpr (TF32) tf32_tile_mma<NSC>(x, ar, acc);
        else f16_tile_mma<NSC>(x, ar, acc);
    };
    uint4 ar0[NSC];  // A row g, pass 0: shared by every group of the item
    arow_load<NSC>(arow, arow_ok, 0, t, ar0);
    auto cols = [&](uint32_t s, uint32_t (&c)[2]) {
        c[0] = s + g < vend ? __ldg(ci + s + g) : 0u;
        c[1] = s + g + 8 < vend ? __ldg(ci + s + g + 8) : 0u;
    };
    // one group: prefetched pass 0 + (rare) extra passes loaded in place
    constexpr int MW = kMaskWords<MM>;
    auto group = [&](uint32_t s, const uint32_t (&c)[2], const Tile& x0, const uint32_t (&mk)[MW]) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        mma(x0, ar0, acc);
        if constexpr (NSC > 1) {  // NSC == 1 <=> the inner dimension fits one pass
            for (int p = 1; p < a.passes; ++p) {
                Tile x;
                uint4 arp[NSC];
                load(s, c, p, x);
                arow_load<NSC>(arow, arow_ok, p, t, arp);
                mma(x, arp, acc);
            }
        }
        const uint32_t live = slow_live<MM>(mk, s, vend, g, t);
        sddmm_store<TF32 ? 4u : 8u, OF32>(a.out, acc, live, a.dead, vbase, nvw, vend, s, g, t);
    };

    // Double-buffered batches of D groups (16*D vectors): the gathers of
    // batch i+1 are in flight while batch i is consumed.  A per-warp
    // shared-memory ring, filled by cp.async RING-1 batches ahead, stages
    // each batch's column indices (so no gather waits on a dependent global
    // load) and, for a full batch, its 128*D contiguous mask values (the
    // DRAM-streamed operand gets the deepest prefetch).  A batch whose
    // vectors all lie in full-width blocks takes the predicate-free path
    // (liveness bits read from the ring, fixed store offsets); only the last
    // batch of a window takes the general one.
    constexpr int D = kBatchGroups<NSC>;
    constexpr uint32_t BV = 16 * D;
    constexpr uint32_t MSZ = MM == kMaskF32 ? 4 : 2;
    constexpr uint32_t SLOT = ring_slot_bytes<NSC, MM>();
    unsigned char* wring = ring_all + warp * kRing * SLOT;
    auto ring_cols = [&](uint32_t slot) { return reinterpret_cast<uint32_t*>(wring + slot * SLOT); };
    auto ring_mask = [&](uint32_t slot) { return wring + slot * SLOT + BV * 4; };
    auto prefetch_cols = [&](uint32_t sb, uint32_t slot) {
        __syncwarp();  // every lane is done reading this slot
        uint32_t* rc = ring_cols(slot);
#pragma unroll
        for (uint32_t i = lane; i < BV && sb < vend; i += 32) {
            const uint32_t v = min(sb + i, vend - 1);  // clamp: stays inside the item's columns
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(rc + i))),
                         "l"(ci + v)
                         : "memory");
        }
        if (sb + BV <= vend) {
            if constexpr (MM == kLive) {
                // the batch's BV liveness bytes, as the aligned words covering them
                const uint8_t* src = a.live + vbase / 8 + sb;
                const uint32_t* w0 = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(src) & ~uintptr_t(3));
                unsigned char* dst = ring_mask(slot);
                if (lane <= BV / 4)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                     static_cast<uint32_t>(__cvta_generic_to_shared(dst + 4 * lane))),
                                 "l"(w0 + lane)
                                 : "memory");
            } else {
                const unsigned char* src = static_cast<const unsigned char*>(a.mask) + (vbase + 8ull * sb) * MSZ;
                unsigned char* dst = ring_mask(slot);
#pragma unroll
                for (uint32_t c = lane; c < BV * 8 * MSZ / 16; c += 32)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     static_cast<uint32_t>(__cvta_generic_to_shared(dst + 16 * c))),
                                 "l"(src + 16 * c)
                                 : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // Full batches: predicate-free loads, liveness from the ring.
    auto issue_full = [&](uint32_t sb, uint32_t slot, Tile (&x)[D], uint32_t (&live)[D], uint32_t (&cg)[D][2]) {
        const uint32_t* rc = ring_cols(slot);
#pragma unroll
        for (int d = 0; d < D; ++d) {
            cg[d][0] = rc[16 * d + g];
            cg[d][1] = rc[16 * d + g + 8];
            if constexpr (TF32) tf32_tile_load<NSC>(a, cg[d][0], true, cg[d][1], true, 0, t, x[d]);
            else f16_tile_load<NSC>(a, cg[d][0], true, cg[d][1], true, 0, t, x[d]);
            if constexpr (MM == kLive)
                live[d] = ring_live<TF32 ? 4u : 8u, MM>(ring_mask(slot) + ((vbase / 8 + sb) & 3u) + 16u * d, g, t);
            else
                live[d] = ring_live<TF32 ? 4u : 8u, MM>(ring_mask(slot) + 128u * d * MSZ, g, t);
        }
    };
    auto consume_full = [&](uint32_t sb, const Tile (&x)[D], const uint32_t (&live)[D], const uint32_t (&cg)[D][2]) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const uint32_t s = sb + 16 * d;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            mma(x[d], ar0, acc);
            if constexpr (NSC > 1) {
                for (int p = 1; p < a.passes; ++p) {
                    Tile xp;
                    uint4 arp[NSC];
                    load(s, cg[d], p, xp);
                    arow_load<NSC>(arow, arow_ok, p, t, arp);
                    mma(xp, arp, acc);
                }
            }
            full_store<TF32 ? 4u : 8u, OF32>(a.out, vbase + 8ull * s, acc, live[d], a.dead, g, t);
        }
    };

    const uint32_t s0 = vbeg;
    if (s0 < vend) {
        const uint32_t nf = (vend - s0) / BV;  // full batches; at most one partial batch follows
        uint32_t pb = 0;                       // next batch to prefetch
        for (int r = 0; r < kRing - 1; ++r, ++pb) prefetch_cols(s0 + pb * BV, pb % kRing);
        auto ring_next = [&]() {  // prefetch one more batch, wait for batch ib
            prefetch_cols(s0 + pb * BV, pb % kRing);
            ++pb;
            asm volatile("cp.async.wait_group %0;" ::"n"(kRing - 1) : "memory");
            __syncwarp();
        };
        if (nf) {  // double-buffered full batches: batch i+1 in flight while i is consumed
            Tile ta[D], tb[D];
            uint32_t la[D], lb[D], ga[D][2], gb[D][2];
            ring_next();
            issue_full(s0, 0, ta, la, ga);
            for (uint32_t i = 0;;) {
                if (i + 1 < nf) {
                    ring_next();
                    issue_full(s0 + (i + 1) * BV, (i + 1) % kRing, tb, lb, gb);
                }
                consume_full(s0 + i * BV, ta, la, ga);
                if (++i >= nf) break;
                if (i + 1 < nf) {
                    ring_next();
                    issue_full(s0 + (i + 1) * BV, (i + 1) % kRing, ta, la, ga);
                }
                consume_full(s0 + i * BV, tb, lb, gb);
                if (++i >= nf) break;
            }
        }
        if (s0 + nf * BV < vend) {  // the window's last, partial batch: general path
            ring_next();
            const uint32_t sb = s0 + nf * BV;
            const uint32_t* rc = ring_cols(nf % kRing);
            Tile x[D];
            uint32_t mk[D][MW], cg[D][2];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const uint32_t s = sb + 16 * d;
                cg[d][0] = rc[16 * d + g];
                cg[d][1] = rc[16 * d + g + 8];
                if (s < vend) {
                    load(s, cg[d], 0, x[d]);
                    mask_prefetch<TF32 ? 4u : 8u, MM>(a, vbase, nvw, vend, s, g, t, mk[d]);
                }
            }
#pragma unroll
            for (int d = 0; d < D; ++d)
                if (sb + 16 * d < vend) group(sb + 16 * d, cg[d], x[d], mk[d]);
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");  // no ring write outlives the item
        __syncwarp();
    }
    }  // work items
}

// Small lists (BASELINE configs[1]: 512 windows of ~123 vectors) are
// latency-bound: one wave, and the ring pipeline above never reaches steady
// state.  Here `sub` warps share an item, each taking a run of its 16-vector
// groups and issuing all loads of up to G groups at once, so the chain is
// row pointers -> column indices (+ mask values) -> gathers -> MMA -> store.
// Single pass only (FP16 K <= 32*NSC, TF32 K <= 16*NSC).  With no split
// windows item i is window i (a.items == nullptr).
constexpr int kBurstBlocks = 8;
// groups per burst of the single-super-chunk SDDMM burst kernel (A/B knob)
#ifndef TCS_SDDMM_BURST_G
#define TCS_SDDMM_BURST_G 2
#endif
#ifndef TCS_BURST_WARPS
#define TCS_BURST_WARPS 4
#endif
constexpr int kBW = TCS_BURST_WARPS;  // warps per CTA of the burst kernel
// most warps sharing one item (A/B knob)
#ifndef TCS_SDDMM_BURST_SUB
#define TCS_SDDMM_BURST_SUB 16
#endif
template <bool TF32, int NSC, int MM, bool OF32, int G>
__global__ void __launch_bounds__(kBW * 32, kBurstBlocks * kWarps / kBW) sddmm_burst(const SddmmArgs a) {
    using Elem = typename std::conditional<TF32, float, __half>::type;
    using Tile = typename std::conditional<TF32, Tf32Tile<NSC>, F16Tile<NSC>>::type;
    constexpr uint32_t K = TF32 ? 4u : 8u;
    constexpr int MW = kMaskWords<MM>;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kBW + (threadIdx.x >> 5);
    const uint64_t idx = gw / a.sub;
    const uint32_t part = static_cast<uint32_t>(gw % a.sub);
    pdl_trigger();  // see dev::pdl_wait: launched with launch_pdl
    pdl_wait();
    if (idx >= a.n_items) return;
    WorkItem it;
    uint32_t base, nvw;
    if (a.items) {
        it = a.items[idx];
        base = __ldg(a.rp + it.window);
        nvw = __ldg(a.rp + it.window + 1) - base;
    } else {
        base = __ldg(a.rp + idx);
        nvw = __ldg(a.rp + idx + 1) - base;
        it = WorkItem{static_cast<uint32_t>(idx), 0u, nvw, kNoSlot};
    }
    const uint64_t arow_i = 8ull * it.window + g;
    const bool arow_ok = arow_i < a.rows;
    uint4 ar0[NSC];
    arow_load<NSC>(static_cast<const Elem*>(a.A) + (arow_ok ? arow_i : 0) * a.lda, arow_ok, 0, t, ar0);
    const uint32_t* ci = a.ci + base;
    const uint64_t vbase = 8ull * base;
    const uint32_t run = ((it.vend - it.vbeg + a.sub - 1) / a.sub + 15u) & ~15u;
    const uint32_t vbeg = min(it.vend, it.vbeg + part * run);
    const uint32_t vend = min(it.vend, vbeg + run);
    for (uint32_t s0 = vbeg; s0 < vend; s0 += 16 * G) {
        uint32_t c[G][2];
        Tile x[G];
        uint32_t mk[G][MW];
#pragma unroll
        for (int d = 0; d < G; ++d) {
            const uint32_t s = s0 + 16 * d;
            c[d][0] = s + g < vend ? __ldg(ci + s + g) : 0u;
            c[d][1] = s + g + 8 < vend ? __ldg(ci + s + g + 8) : 0u;
            if (s < vend) mask_prefetch<K, MM>(a, vbase, nvw, vend, s, g, t, mk[d]);
        }
#pragma unroll
        for (int d = 0; d < G; ++d) {
            const uint32_t s = s0 + 16 * d;
            if (s >= vend) continue;
            if constexpr (TF32) tf32_tile_load<NSC>(a, c[d][0], s + g < vend, c[d][1], s + g + 8 < vend, 0, t, x[d]);
            else f16_tile_load<NSC>(a, c[d][0], s + g < vend, c[d][1], s + g + 8 < vend, 0, t, x[d]);
        }
#pragma unroll
        for (int d = 0; d < G; ++d) {
            const uint32_t s = s0 + 16 * d;
            if (s >= vend) continue;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            if constexpr (TF32) tf32_tile_mma<NSC>(x[d], ar0, acc);
            else f16_tile_mma<NSC>(x[d], ar0, acc);
            sddmm_store<K, OF32>(a.out, acc, slow_live<MM>(mk[d], s, vend, g, t), a.dead, vbase, nvw, vend, s, g, t);
        }
    }
}

template <bool TF32, int NSC, int G>
void launch_sddmm_burst(const SddmmArgs& a, bool mf32, bool of32, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((a.n_items * a.sub + kBW - 1) / kBW));
    const dim3 block(kBW * 32);
    if (a.live) {
        if (of32) launch_pdl(sddmm_burst<TF32, NSC, kLive, true, G>, grid, block, 0, s, a);
        else launch_pdl(sddmm_burst<TF32, NSC, kLive, false, G>, grid, block, 0, s, a);
    } else if (mf32 && of32) launch_pdl(sddmm_burst<TF32, NSC, kMaskF32, true, G>, grid, block, 0, s, a);
    else if (mf32) launch_pdl(sddmm_burst<TF32, NSC, kMaskF32, false, G>, grid, block, 0, s, a);
    else if (of32) launch_pdl(sddmm_burst<TF32, NSC, kMaskF16, true, G>, grid, block, 0, s, a);
    else launch_pdl(sddmm_burst<TF32, NSC, kMaskF16, false, G>, grid, block, 0, s, a);
    TCS_LAUNCHED(TF32 ? "sddmm_tf32_burst" : "sddmm_f16_burst");
}

template <bool TF32, int NSC>
void launch_sddmm(const SddmmArgs& a, bool mf32, bool of32, cudaStream_t s) {
    const uint64_t need = (a.n_items + kWarps - 1) / kWarps;
    const dim3 grid(static_cast<unsigned>(std::min<uint64_t>(need, uint64_t(num_sms()) * kMinBlocks<NSC>)));
    const size_t sm32 = kWarps * kRing * ring_slot_bytes<NSC, kMaskF32>();
    const size_t sm16 = kWarps * kRing * ring_slot_bytes<NSC, kMaskF16>();
    const size_t sml = kWarps * kRing * ring_slot_bytes<NSC, kLive>();
    if (a.live) {
        if (of32) sddmm_kernel<TF32, NSC, kLive, true><<<grid, kWarps * 32, sml, s>>>(a);
        else sddmm_kernel<TF32, NSC, kLive, false><<<grid, kWarps * 32, sml, s>>>(a);
    } else if (mf32 && of32) sddmm_kernel<TF32, NSC, kMaskF32, true><<<grid, kWarps * 32, sm32, s>>>(a);
    else if (mf32) sddmm_kernel<TF32, NSC, kMaskF32, false><<<grid, kWarps * 32, sm32, s>>>(a);
    else if (of32) sddmm_kernel<TF32, NSC, kMaskF16, true><<<grid, kWarps * 32, sm16, s>>>(a);
    else sddmm_kernel<TF32, NSC, kMaskF16, false><<<grid, kWarps * 32, sm16, s>>>(a);
    TCS_LAUNCHED(TF32 ? "sddmm_tf32" : "sddmm_f16");
}

// Liveness byte of every stored vector (bit r = row r's stored value is
// nonzero; -0.0 is not live, ref sddmm.hpp:131), one thread per vector.
template <typename V>
__global__ void live_build(const uint32_t* __restrict__ rp, uint64_t W, const V* __restrict__ vals, uint64_t nv,
                           uint32_t k, uint8_t* __restrict__ live) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nv; p += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = W;  // window: rp[lo] <= p < rp[lo + 1]
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (rp[mid] <= p) lo = mid; else hi = mid;
        }
        const uint32_t base = rp[lo], j = static_cast<uint32_t>(p - base), nvw = rp[lo + 1] - base;
        const uint32_t b = j / k, jj = j % k, width = min(k, nvw - b * k);
        const uint64_t off = 8ull * (base + b * k) + jj;
        uint32_t bits = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const V x = vals[off + r * width];
            const bool nz = sizeof(V) == 2 ? (static_cast<uint32_t>(x) & 0x7FFFu) != 0u
                                           : (static_cast<uint32_t>(x) & 0x7FFFFFFFu) != 0u;
            bits |= static_cast<uint32_t>(nz) << r;
        }
        live[p] = static_cast<uint8_t>(bits);
    }
}

}  // namespace

// Validation shared by tcs_sddmm and tcs_sddmm_row_softmax (ref sddmm.hpp:86-90).
void sddmm_check(const tcs_mebcrs* mask, const void* a, tcs_dtype a_dtype, int64_t lda, int64_t a_rows, int64_t f_a,
                 const void* bt, tcs_dtype bt_dtype, int64_t ldbt, int64_t bt_rows, int64_t f_b, tcs_dtype out_dtype,
                 const tcs_kernel_config* cfg) {
    if (!cfg) fail(TCS_ERR_ARGUMENT, "null argument");
    check_mebcrs(mask);
    if (cfg->precision != mask->precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded mask");
    if (cfg->vector_height != 8) fail(TCS_ERR_ARGUMENT, "SDDMM requires vector height 8");
    if (a_rows != static_cast<int64_t>(mask->rows)) fail(TCS_ERR_SHAPE, "A rows must equal mask rows");
    if (bt_rows != static_cast<int64_t>(mask->cols)) fail(TCS_ERR_SHAPE, "B cols must equal mask cols");
    if (f_a != f_b) fail(TCS_ERR_SHAPE, "inner dimensions of A and B must agree");
    if (f_a < 0) fail(TCS_ERR_SHAPE, "negative inner dimension");
    if (out_dtype != TCS_DTYPE_F16 && out_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "unknown output dtype");
    if ((a_rows && f_a && (!a || lda < f_a)) || (bt_rows && f_b && (!bt || ldbt < f_b)))
        fail(TCS_ERR_ARGUMENT, "bad dense operand / leading dimension");
    const bool tf32 = mask->precision == TCS_TF32;
    if (tf32 && (a_dtype != TCS_DTYPE_F32 || bt_dtype != TCS_DTYPE_F32))
        fail(TCS_ERR_ARGUMENT, "TF32 SDDMM needs f32 dense operands");
    if (tf32 && out_dtype != TCS_DTYPE_F32) fail(TCS_ERR_ARGUMENT, "TF32 ME-BCRS values must be stored as f32");
}

// Runs the SDDMM of `mask` into out_values (8*nv values of out_dtype).
// `dead`: the value of stored slots whose mask value is 0 (0 for tcs_sddmm,
// -inf for the fused softmax, which then needs no mask re-read).
// Liveness bytes of the mask's current values, cached in its work list
// (TCS_CFG_STATIC_MASK: the caller guarantees the values do not change
// between calls that reuse the cache).
const uint8_t* mask_liveness(const tcs_mebcrs* mask, Plan* plan, cudaStream_t s) {
    if (const uint8_t* ex = plan->exact_for(mask->values)) return ex;
    if (plan->live && plan->live_src == mask->values) return plan->live;
    if (!plan->live) plan->live = static_cast<uint8_t*>(dalloc(mask->num_vectors + 16, s));
    build_liveness(mask, plan->live, s);
    plan->live_src = mask->values;
    return plan->live;
}

// live[p] for every stored vector p (nv + 16 bytes; the 16 past nv zeroed).
void build_liveness(const tcs_mebcrs* mask, uint8_t* live, cudaStream_t s) {
    const uint64_t nv = mask->num_vectors;
    if (const Plan* plan = static_cast<const Plan*>(mask->plan); plan && plan->exact_for(mask->values)) {
        TCS_CUDA(cudaMemcpyAsync(live, plan->exact_live, nv + 16, cudaMemcpyDeviceToDevice, s));
        return;
    }
    TCS_CUDA(cudaMemsetAsync(live + nv, 0, 16, s));
    if (!nv) return;
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((nv + 255) / 256, uint64_t(num_sms()) * 16)));
    if (mask->value_dtype == TCS_DTYPE_F16)
        live_build<unsigned short><<<grid, 256, 0, s>>>(mask->row_pointers, mask->num_windows,
                                                        static_cast<const unsigned short*>(mask->values), nv, mask->k,
                                                        live);
    else
        live_build<uint32_t><<<grid, 256, 0, s>>>(mask->row_pointers, mask->num_windows,
                                                  static_cast<const uint32_t*>(mask->values), nv, mask->k, live);
    TCS_LAUNCHED("sddmm_live_build");
}

void sddmm_launch(const tcs_mebcrs* mask, Plan* plan, const void* a, tcs_dtype a_dtype, int64_t lda,
                  int64_t a_rows, const void* bt, tcs_dtype bt_dtype, int64_t ldbt, int64_t bt_rows, int64_t F,
                  void* out_values, tcs_dtype out_dtype, float dead, bool static_mask, cudaStream_t s) {
    const uint64_t nv = mask->num_vectors;
    const size_t ow = out_dtype == TCS_DTYPE_F16 ? 2 : 4;
    if (!nv) return;
    if (F == 0 && dead == 0.f) {
        TCS_CUDA(cudaMemsetAsync(out_values, 0, 8 * nv * ow, s));
        return;
    }
    const bool tf32 = mask->precision == TCS_TF32;
    // feature padding: super-chunk = 32 (FP16) / 16 (TF32) features
    const int64_t sc = tf32 ? 16 : 32;
    int64_t fpad = std::max<int64_t>(1, (F + sc - 1) / sc) * sc;
    // NSC super-chunks per pass (double-buffered in registers); wider inner
    // dimensions take several passes.
    // (Every pass after the first loads and multiplies without prefetch, so
    // wide inner dimensions use 4 super-chunks per pass: FP16 F <= 128 and
    // TF32 F <= 64 in one pass.)
    int nsc = 1;
    if (fpad > 2 * sc && TCS_SDDMM_NSC4) {
        nsc = 4;
        fpad = (F + 4 * sc - 1) / (4 * sc) * (4 * sc);
    } else if (fpad > sc) {
        nsc = 2;
        fpad = (F + 2 * sc - 1) / (2 * sc) * (2 * sc);
    }
    const tcs_dtype need = tf32 ? TCS_DTYPE_F32 : TCS_DTYPE_F16;
    const int64_t al = tf32 ? 4 : 8;
    auto prep = [&](const void* src, tcs_dtype dt, int64_t ld, int64_t nrows, DBuf& buf,
                    int64_t& out_ld) -> const void* {
        if (F > 0 && dt == need && ld >= fpad && ld % al == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            out_ld = ld;
            return src;
        }
        out_ld = fpad;
        buf = DBuf(std::max<int64_t>(1, nrows) * fpad * (tf32 ? 4 : 2), s);
        pad_convert(src, dt, ld, buf.p, need, fpad, nrows, F, fpad, s);
        return buf.p;
    };
    DBuf abuf, bbuf;
    int64_t alda = 0, bldb = 0;
    const void* ap = prep(a, a_dtype, lda, a_rows, abuf, alda);
    const void* bp = prep(bt, bt_dtype, ldbt, bt_rows, bbuf, bldb);
    const bool mf32 = mask->value_dtype == TCS_DTYPE_F32, of32 = out_dtype == TCS_DTYPE_F32;
    if (!plan->n_items) return;
#ifndef TCS_NO_BURST
    // small single-pass lists: the burst kernel, `sub` warps per item, one wave
    const uint64_t burst_cap = uint64_t(num_sms()) * kBurstBlocks * kWarps;
    if (fpad == nsc * sc && nsc <= 2 && plan->seg <= 512 && plan->n_items <= burst_cap) {
        SddmmArgs b{plan->n_split ? plan->items : nullptr, plan->n_items, mask->row_pointers, mask->column_indices,
                    mask->values, ap, alda, bp, bldb, out_values, mask->rows, 1, mask->k, nullptr, dead, nullptr,
                    static_cast<uint32_t>(std::min<uint64_t>(TCS_SDDMM_BURST_SUB, burst_cap / plan->n_items))};
        if (static_mask) b.live = mask_liveness(mask, plan, s);
        else if (const uint8_t* ex = plan->exact_for(mask->values)) b.live = ex;
        if (tf32) {
            if (nsc == 1) launch_sddmm_burst<true, 1, TCS_SDDMM_BURST_G>(b, mf32, of32, s);
            else launch_sddmm_burst<true, 2, 1>(b, mf32, of32, s);
        } else {
            if (nsc == 1) launch_sddmm_burst<false, 1, TCS_SDDMM_BURST_G>(b, mf32, of32, s);
            else launch_sddmm_burst<false, 2, 1>(b, mf32, of32, s);
        }
        return;
    }
#endif
    DBuf item_ctr(dev::kClaimBytes, s);
    TCS_CUDA(cudaMemsetAsync(item_ctr.p, 0, dev::kClaimBytes, s));
    SddmmArgs args{plan->items, plan->n_items, mask->row_pointers, mask->column_indices, mask->values,
                   ap, alda, bp, bldb, out_values, mask->rows,
                   static_cast<int>(fpad / (nsc * sc)), mask->k, item_ctr.as<uint32_t>(), dead, nullptr, 1};
    if (static_mask) args.live = mask_liveness(mask, plan, s);
    // binary16 values that lost a tiny nonzero: the exact bytes decide (ref :131)
    else if (const uint8_t* ex = plan->exact_for(mask->values)) args.live = ex;
    if (tf32) {
        if (nsc == 1) launch_sddmm<true, 1>(args, mf32, of32, s);
        else if (nsc == 2) launch_sddmm<true, 2>(args, mf32, of32, s);
        else launch_sddmm<true, 4>(args, mf32, of32, s);
    } else {
        if (nsc == 1) launch_sddmm<false, 1>(args, mf32, of32, s);
        else if (nsc == 2) launch_sddmm<false, 2>(args, mf32, of32, s);
        else launch_sddmm<false, 4>(args, mf32, of32, s);
    }
}

}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_sddmm(const tcs_mebcrs* mask, const void* a, tcs_dtype a_dtype, int64_t lda,
                                int64_t a_rows, int64_t f_a, const void* bt, tcs_dtype bt_dtype, int64_t ldbt,
                                int64_t bt_rows, int64_t f_b, tcs_mebcrs* out, tcs_dtype out_dtype,
                                const tcs_kernel_config* cfg, tcs_counters* counters, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_sddmm");
        if (!out) fail(TCS_ERR_ARGUMENT, "null argument");
        sddmm_check(mask, a, a_dtype, lda, a_rows, f_a, bt, bt_dtype, ldbt, bt_rows, f_b, out_dtype, cfg);
        cudaStream_t s = st(stream);
        // output: the mask's structure, fresh values
        const size_t ow = out_dtype == TCS_DTYPE_F16 ? 2 : 4;
        void* caller_values = out->values;
        tcs_mebcrs o = *mask;
        o.flags = o.plan ? TCS_MEBCRS_BORROWED_PLAN : 0u;  // structure and work list shared
        o.value_dtype = out_dtype;
        if (caller_values) {
            o.values = caller_values;
        } else {
            o.values = dalloc(std::max<uint64_t>(1, 8 * mask->num_vectors) * ow, s);
            o.flags |= TCS_MEBCRS_OWN_VALUES;
        }
        if (counters) *counters = tcs_counters{};
        if (mask->num_vectors) {
            Plan* plan = static_cast<Plan*>(mask->plan);
            Plan* tmp_plan = nullptr;
            if (!plan && f_a > 0) plan = tmp_plan = build_plan(mask, s, nullptr, nullptr, nullptr);
            struct PlanGuard {
                Plan* p;
                cudaStream_t s;
                ~PlanGuard() { free_plan(p, s); }
            } pg{tmp_plan, s};
            // a temporary plan cannot keep a liveness cache
            const bool static_mask = (cfg->flags & TCS_CFG_STATIC_MASK) && !tmp_plan;
            sddmm_launch(mask, plan, a, a_dtype, lda, a_rows, bt, bt_dtype, ldbt, bt_rows, f_a, o.values, out_dtype,
                         0.f, static_mask, s);
        }
        // ref sddmm.hpp:121: one MMA per (16-vector group, k-step)
        if (counters) counters->mma_invocations = mask->num_groups16 * ((f_a + mask->k - 1) / mask->k);
        *out = o;
    });
}

extern "C" tcs_status tcs_sddmm_host(uint64_t rows, uint64_t cols, tcs_precision precision,
                                     const uint32_t* row_pointers, const uint32_t* column_indices,
                                     const float* mask_values, const float* a, int64_t a_rows, int64_t f_a,
                                     const float* bt, int64_t bt_rows, int64_t f_b, float* out_values,
                                     const tcs_kernel_config* cfg, tcs_counters* counters, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_sddmm_host");
        if (!cfg) fail(TCS_ERR_ARGUMENT, "null kernel config");
        if (cfg->precision != precision) fail(TCS_ERR_ARGUMENT, "config precision must match the encoded mask");
        if (a_rows != static_cast<int64_t>(rows)) fail(TCS_ERR_SHAPE, "A rows must equal mask rows");
        if (bt_rows != static_cast<int64_t>(cols)) fail(TCS_ERR_SHAPE, "B cols must equal mask cols");
        if (f_a != f_b) fail(TCS_ERR_SHAPE, "inner dimensions of A and B must agree");
        cudaStream_t s = st(stream);
        tcs_mebcrs m{};
        tcs_status rc = tcs_mebcrs_upload(rows, cols, precision, row_pointers, column_indices, mask_values, &m, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        struct Free {
            tcs_mebcrs* m;
            tcs_stream_t s;
            ~Free() { tcs_mebcrs_free(m, s); }
        } fr{&m, stream};
        DBuf da(std::max<int64_t>(1, a_rows * f_a) * 4, s), db(std::max<int64_t>(1, bt_rows * f_b) * 4, s);
        if (a_rows > 0 && f_a > 0) TCS_CUDA(cudaMemcpyAsync(da.p, a, a_rows * f_a * 4, cudaMemcpyHostToDevice, s));
        if (bt_rows > 0 && f_b > 0) TCS_CUDA(cudaMemcpyAsync(db.p, bt, bt_rows * f_b * 4, cudaMemcpyHostToDevice, s));
        tcs_mebcrs o{};
        rc = tcs_sddmm(&m, da.p, TCS_DTYPE_F32, std::max<int64_t>(1, f_a), a_rows, f_a, db.p, TCS_DTYPE_F32,
                       std::max<int64_t>(1, f_b), bt_rows, f_b, &o, TCS_DTYPE_F32, cfg, counters, stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        if (m.num_vectors)
            TCS_CUDA(cudaMemcpyAsync(out_values, o.values, 8 * m.num_vectors * 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
        tcs_mebcrs_free(&o, stream);
    });
}
