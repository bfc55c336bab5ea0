// Fused AGNN attention (BASELINE.json configs[4]; no
// reference counterpart):
//
//   out[i] = sum_j softmax_j( scale * cos(h_{row0+i}, h_j) ) * h_j
//
// over the live (i, j) of an ME-BCRS mask (live = mask value != 0, the
// reference SDDMM's sampling rule, sddmm.hpp:131).  tcs_agnn_aggregate runs
// this as SDDMM -> statistics -> softmax-applying SpMM, which gathers every
// neighbour row twice and writes and re-reads binary16 scores.  Here one
// warp per work item gathers each neighbour row ONCE and uses it for both
// products, flash-attention style:
//
//   per 16-vector step of the window (rows g = 0..7 of the window):
//     S (8 x 16)   = Hi (8 x F) . Hj^T          m16n8k16, rows 8..15 zero
//     online softmax per row (running max m, sum l; log2 domain)
//     O (8 x F)   += P (8 x 16) . Hj (16 x F)   m16n8k16, P straight from
//                                                 S's accumulator registers
//
// Gather layout: lane (g, t) loads 16 contiguous bytes (features
// 32c + 8t .. +7) of vectors g and g + 8 -- 4 lanes per 64-byte row.  The
// score contraction runs over a permuted feature order (the same
// permutation for Hi and Hj), so those loads ARE the B fragments.  The
// aggregation needs Hj transposed (vectors along k): one movmatrix.trans
// per 8x8 block, after which lane (g, t) accumulates features
// 32c + 8t .. +7 of row g -- two float4 stores in the epilogue.
//
// Scores use the node's inverse norms (rn, computed here from h):
// scale * rn_i * rn_j * <h_i, h_j>.  Split windows (the work list's hub
// segments) store unnormalised partials (O, m, l) merged in segment order by
// agnn_combine (deterministic).
#include <algorithm>
#include <cmath>

#include "tcs_internal.cuh"

namespace tcs {
namespace {
using namespace dev;

#ifndef TCS_AGNN_BPS
#define TCS_AGNN_BPS 6
#endif
constexpr int kAgnnWarps = 4;
// CTAs per SM: F = 32 fits 80 registers; F = 64 needs ~110.
constexpr int agnn_bps(int nc) { return nc == 1 ? TCS_AGNN_BPS : 4; }
constexpr float kLog2e = 1.4426950408889634f;

struct AttendArgs {
    const WorkItem* items;
    uint64_t n_items;
    uint32_t* counter;
    const uint32_t* rp;
    const uint32_t* ci;
    const uint8_t* live;  // per-vector liveness bytes
    const __half* h;      // nodes x ldh, f16
    int64_t ldh;
    const float* rn;      // per-node inverse norm
    int64_t row0;         // mask row i is node row0 + i
    uint64_t rows;        // mask rows
    float scale2;         // scale * log2(e)
    float* out;
    int64_t ldo;
    float* partial;       // n_slots x 8 x F (unnormalised O of split segments)
    float2* pstat;        // n_slots x 8 (m, l) in log2 units
};

__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int NC>
struct AttStep {
    uint4 h[2][NC];  // vectors g (half 0) and g + 8 (half 1), features 32c + 8t .. +7
    float rn[2];     // inverse norms of those two vectors
    uint32_t live[2];  // their liveness bytes
    uint32_t ok;       // bit hf: vector of half hf is inside the item (else h / live count as 0)
};

// cols: column indices of vectors [s0, s0 + 32) of the window, one per lane.
template <int NC>
__device__ __forceinline__ void att_issue(const AttendArgs& a, uint32_t base, uint32_t vend, uint32_t s, uint32_t s0,
                                          uint32_t cols, uint32_t lane, AttStep<NC>& st) {
    const uint32_t g = lane >> 2, t = lane & 3, off = s - s0;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
        const uint32_t v = s + 8 * hf + g;
        const uint32_t col = __shfl_sync(0xffffffffu, cols, off + 8 * hf + g);
        const bool ok = v < vend;
        // Unconditional loads (past the item: column 0's row, slot s -- both
        // in bounds); att_compute zeroes them by `ok`.  Selecting the zero
        // here made the issue wait for its own loads (ncu, C5: 24% of the
        // stall samples on that select), before the previous step's MMAs.
        const __half* r = a.h + static_cast<uint64_t>(ok ? col : 0u) * a.ldh + 8 * t;
#pragma unroll
        for (int c = 0; c < NC; ++c) st.h[hf][c] = ld_gather_128(r + 32 * c);
        st.rn[hf] = __ldg(a.rn + (ok ? col : 0u));
        st.live[hf] = static_cast<uint32_t>(__ldg(a.live + base + (ok ? v : s)));
        if (hf == 0) st.ok = ok ? 1u : 0u;
        else st.ok |= ok ? 2u : 0u;
    }
}

__device__ __forceinline__ uint32_t comp(const uint4& v, int k) {
    return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

// Scores of one step, zero C (no accumulator materialisation).
__device__ __forceinline__ void mma_f16_16816_z(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%10,%10,%10};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
}

// Swap form (vectors on M): lane (g, t) owns vectors g, g + 8 and rows
// 2t, 2t + 1 of the window.
//   S^T (16 vec x 8 rows) = Hj (16 x F) . Hi^T      A = gathered rows, B = Hi
//   O^T (F x 8 rows)     += Hj^T (F x 16) . P^T     A = movmatrix(Hj), B = movmatrix(P^T)
// m, l: running max (log2 units) and lane-partial sum of rows 2t, 2t + 1.
// o[c][q]: features phi(c, 2q + j, g) = 32c + 8(g >> 1) + 2(2q + j) + (g & 1),
// j = 0 (o[0], o[1]) and 1 (o[2], o[3]); o[.][.][e & 1] is row 2t + (e & 1).
template <int NC>
__device__ __forceinline__ void att_compute(const AttStep<NC>& st, const uint4 (&hi)[NC], const float (&qs)[2],
                                            uint32_t lane, float (&m)[2], float (&l)[2], float (&o)[NC][2][4]) {
    const uint32_t t = lane & 3;
    const bool ok0 = st.ok & 1u, ok1 = st.ok & 2u;
    uint4 h0[NC], h1[NC];  // vectors past the item contribute zero rows
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        h0[c] = ok0 ? st.h[0][c] : make_uint4(0, 0, 0, 0);
        h1[c] = ok1 ? st.h[1][c] : make_uint4(0, 0, 0, 0);
    }
    const uint32_t lv[2] = {ok0 ? st.live[0] : 0u, ok1 ? st.live[1] : 0u};
    float acc[4];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const uint4 &x = h0[c], &y = h1[c];
        if (c == 0) mma_f16_16816_z(acc, x.x, y.x, x.y, y.y, hi[c].x, hi[c].y);
        else mma_f16_16816(acc, x.x, y.x, x.y, y.y, hi[c].x, hi[c].y);
        mma_f16_16816(acc, x.z, y.z, x.w, y.w, hi[c].z, hi[c].w);
    }
    // acc: (vector g, row 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)
    float z[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int hf = e >> 1, r = e & 1;
        const bool live = (lv[hf] >> (2 * t + r)) & 1u;
        z[e] = live ? acc[e] * qs[r] * st.rn[hf] : -INFINITY;
    }
    float mx[2] = {fmaxf(z[0], z[2]), fmaxf(z[1], z[3])};
#pragma unroll
    for (int o2 = 4; o2 <= 16; o2 <<= 1) {
        mx[0] = fmaxf(mx[0], __shfl_xor_sync(0xffffffffu, mx[0], o2));
        mx[1] = fmaxf(mx[1], __shfl_xor_sync(0xffffffffu, mx[1], o2));
    }
    float alpha[2], mref[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const float mn = fmaxf(m[r], mx[r]);
        // no early exit (the MMAs are warp-collective): a row with no live
        // slot yet keeps m = -inf and gets p = 0
        mref[r] = mn == -INFINITY ? 0.f : mn;
        alpha[r] = fast_exp2(m[r] - mref[r]);  // m = -inf -> 0
        m[r] = mn;
    }
    float p[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = fast_exp2(z[e] - mref[e & 1]);
    l[0] = l[0] * alpha[0] + (p[0] + p[2]);
    l[1] = l[1] * alpha[1] + (p[1] + p[3]);
    // P^T as the B operand: k = vectors 2t, 2t+1 (b0) and 2t+8, 2t+9 (b1), n = row g
    const uint32_t b0 = movtrans(f2_to_h2(p[0], p[1])), b1 = movtrans(f2_to_h2(p[2], p[3]));
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            float (&d)[4] = o[c][q];
            d[0] *= alpha[0];
            d[1] *= alpha[1];
            d[2] *= alpha[0];
            d[3] *= alpha[1];
            mma_f16_16816(d, movtrans(comp(h0[c], 2 * q)), movtrans(comp(h0[c], 2 * q + 1)),
                          movtrans(comp(h1[c], 2 * q)), movtrans(comp(h1[c], 2 * q + 1)), b0, b1);
        }
}

template <int NC>
__global__ void __launch_bounds__(kAgnnWarps * 32, agnn_bps(NC)) agnn_attend_kernel(const AttendArgs a) {
    constexpr int F = 32 * NC;
    const uint32_t lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    dev::StripedClaim<8> claim;
    for (uint32_t idx; claim.get(a.counter, a.n_items, idx);) {
        const WorkItem it = a.items[idx];
        const uint32_t base = __ldg(a.rp + it.window);
        const uint32_t* ci = a.ci + base;
        const uint32_t vend = it.vend;
        const uint64_t row_g = 8ull * it.window + g;  // Hi operand row
        const bool g_ok = row_g < a.rows;
        const int64_t node_g = a.row0 + static_cast<int64_t>(g_ok ? row_g : 0);
        uint4 hi[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c)
            hi[c] = g_ok ? ld_gather_128(a.h + node_g * a.ldh + 32 * c + 8 * t) : make_uint4(0, 0, 0, 0);
        float qs[2];  // scale * log2(e) / |h_i| of rows 2t, 2t + 1
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const uint64_t row = 8ull * it.window + 2 * t + r;
            qs[r] = row < a.rows ? a.scale2 * __ldg(a.rn + a.row0 + static_cast<int64_t>(row)) : 0.f;
        }

        float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
        float o[NC][2][4];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int q = 0; q < 2; ++q) o[c][q][0] = o[c][q][1] = o[c][q][2] = o[c][q][3] = 0.f;

        uint32_t s = it.vbeg;
        if (s < vend) {
            AttStep<NC> sa, sb;
            uint32_t s0 = s;
            uint32_t cur = s0 + lane < vend ? ld_stream_u32(ci + s0 + lane) : 0u;
            uint32_t nxt = s0 + 32 + lane < vend ? ld_stream_u32(ci + s0 + 32 + lane) : 0u;
            att_issue<NC>(a, base, vend, s, s0, cur, lane, sa);
            for (;;) {  // invariant: s == s0, cur = columns of steps s and s + 16
                if (s + 16 < vend) att_issue<NC>(a, base, vend, s + 16, s0, cur, lane, sb);
                att_compute<NC>(sa, hi, qs, lane, m, l, o);
                if (s + 16 >= vend) break;
                if (s + 32 < vend) {  // advance the column window by 32
                    s0 += 32;
                    cur = nxt;
                    nxt = s0 + 32 + lane < vend ? ld_stream_u32(ci + s0 + 32 + lane) : 0u;
                    att_issue<NC>(a, base, vend, s + 32, s0, cur, lane, sa);
                }
                att_compute<NC>(sb, hi, qs, lane, m, l, o);
                s += 32;
                if (s >= vend) break;
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int o2 = 4; o2 <= 16; o2 <<= 1) l[r] += __shfl_xor_sync(0xffffffffu, l[r], o2);
        const bool split = it.slot != kNoSlot;
        if (split && g == 0) {
#pragma unroll
            for (int r = 0; r < 2; ++r)
                a.pstat[static_cast<uint64_t>(it.slot) * 8 + 2 * t + r] = make_float2(m[r], l[r]);
        }
        // Lanes g and g ^ 1 hold the even / odd features of the same 8-feature
        // group: swap halves so that each writes 4 contiguous features of its
        // rows (even g: group + 0..3, odd g: group + 4..7).
        const bool odd = g & 1;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const uint64_t row = 8ull * it.window + 2 * t + r;
            float* dst;
            float inv = 1.f;
            if (split) {
                dst = a.partial + (static_cast<uint64_t>(it.slot) * 8 + 2 * t + r) * F;
            } else {
                dst = a.out + row * a.ldo;
                inv = l[r] > 0.f ? 1.f / l[r] : 0.f;
            }
            const bool ok = split || row < a.rows;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                // own values at features 2k + (g & 1), k = 0..3: o[c][k >> 1][2 (k & 1) + r]
                const float v0 = o[c][0][r], v1 = o[c][0][2 + r], v2 = o[c][1][r], v3 = o[c][1][2 + r];
                // even lane keeps k = 0, 1 and receives the odd lane's k = 0, 1
                const float s0v = odd ? v0 : v2, s1v = odd ? v1 : v3;
                const float r0v = __shfl_xor_sync(0xffffffffu, s0v, 4);
                const float r1v = __shfl_xor_sync(0xffffffffu, s1v, 4);
                float4 out;
                if (!odd) out = make_float4(v0 * inv, r0v * inv, v1 * inv, r1v * inv);
                else out = make_float4(r0v * inv, v2 * inv, r1v * inv, v3 * inv);
                if (ok) *reinterpret_cast<float4*>(dst + 32 * c + 8 * (g >> 1) + 4 * odd) = out;
            }
        }
    }
}

// Split windows: merge the segments' (O, m, l) in segment order.
__global__ void __launch_bounds__(256) agnn_combine(const SplitWindow* __restrict__ split, uint64_t n_split,
                                                    const float* __restrict__ partial,
                                                    const float2* __restrict__ pstat, int64_t F, uint64_t rows,
                                                    float* out, int64_t ldo) {
    for (uint64_t sw = blockIdx.x; sw < n_split; sw += gridDim.x) {
        const SplitWindow x = split[sw];
        for (int64_t e = threadIdx.x; e < 8 * F; e += blockDim.x) {
            const int64_t r = e / F, f = e - r * F;
            const uint64_t row = 8ull * x.window + r;
            if (row >= rows) continue;
            float m = -INFINITY;
            for (uint32_t q = 0; q < x.nseg; ++q) m = fmaxf(m, pstat[(uint64_t)(x.first_slot + q) * 8 + r].x);
            float acc = 0.f, l = 0.f;
            if (m != -INFINITY)
                for (uint32_t q = 0; q < x.nseg; ++q) {
                    const uint64_t slot = x.first_slot + q;
                    const float2 st = pstat[slot * 8 + r];
                    const float w = st.x == -INFINITY ? 0.f : exp2f(st.x - m);
                    l += w * st.y;
                    acc += w * partial[(slot * 8 + r) * F + f];
                }
            out[row * ldo + f] = l > 0.f ? acc / l : 0.f;
        }
    }
}

// rn[j] = 1 / max(||h_j||, eps) from the f16 rows; F / 8 lanes per row.
template <int LPR>
__global__ void __launch_bounds__(256) inv_norms(const __half* __restrict__ h, int64_t nodes, int64_t ldh, float eps,
                                                 float* __restrict__ rn) {
    constexpr int RPW = 32 / LPR;
    const uint32_t lane = threadIdx.x & 31, sub = lane % LPR;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t r0 = w0 * RPW; r0 < nodes; r0 += nw * RPW) {
        const int64_t r = r0 + lane / LPR;
        float ss = 0.f;
        if (r < nodes) {
            const uint4 v = ld_stream_u128(h + r * ldh + 8 * sub);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
                ss = fmaf(f2.x, f2.x, fmaf(f2.y, f2.y, ss));
            }
        }
#pragma unroll
        for (int o = LPR / 2; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (r < nodes && sub == 0) rn[r] = 1.f / fmaxf(sqrtf(ss), eps);
    }
}

}  // namespace
}  // namespace tcs

using namespace tcs;

extern "C" tcs_status tcs_agnn_attend(const tcs_mebcrs* mask, const void* h, tcs_dtype h_dtype, int64_t ldh,
                                      int64_t row0, int64_t f, float scale, float eps, float* c, int64_t ldc,
                                      const tcs_kernel_config* cfg, tcs_stream_t stream) {
    return guard([&] {
        NvtxRange nvtx_range("tcs_agnn_attend");
        if (!mask || !cfg) fail(TCS_ERR_ARGUMENT, "null argument");
        check_mebcrs(mask);
        if (cfg->vector_height != 8) fail(TCS_ERR_ARGUMENT, "swap-and-transpose path requires vector height 8");
        if (h_dtype != TCS_DTYPE_F16) fail(TCS_ERR_ARGUMENT, "fused AGNN attention gathers f16 features");
        if (f != 32 && f != 64) fail(TCS_ERR_SHAPE, "fused AGNN attention supports F = 32 or 64");
        const int64_t nodes = static_cast<int64_t>(mask->cols);
        if (row0 < 0 || row0 + static_cast<int64_t>(mask->rows) > nodes)
            fail(TCS_ERR_SHAPE, "AGNN attention: mask rows [row0, row0 + rows) must be nodes of its columns");
        if (!(eps > 0.f)) fail(TCS_ERR_ARGUMENT, "eps must be positive");
        const uint64_t rows = mask->rows;
        if (rows == 0) return;
        if (!h || !c || ldh < f || ldc < f || ldh % 8 || ldc % 4 || (reinterpret_cast<uintptr_t>(h) & 15) ||
            (reinterpret_cast<uintptr_t>(c) & 15))
            fail(TCS_ERR_ARGUMENT, "bad dense buffer (16-byte aligned rows required)");
        cudaStream_t s = st(stream);
        const uint64_t nv = mask->num_vectors;
        if (!nv) {
            TCS_CUDA(cudaMemset2DAsync(c, ldc * 4, 0, f * 4, rows, s));
            return;
        }
        Plan* plan = static_cast<Plan*>(mask->plan);
        Plan* tmp_plan = nullptr;
        if (!plan) plan = tmp_plan = build_plan(mask, s, nullptr, nullptr, nullptr);
        struct PlanGuard {
            Plan* p;
            cudaStream_t s;
            ~PlanGuard() { free_plan(p, s); }
        } pg{tmp_plan, s};
        DBuf live_tmp;
        const uint8_t* live;
        if ((cfg->flags & TCS_CFG_STATIC_MASK) && !tmp_plan) {
            live = mask_liveness(mask, plan, s);
        } else {
            live_tmp = DBuf(nv + 16, s);
            build_liveness(mask, live_tmp.as<uint8_t>(), s);
            live = live_tmp.as<uint8_t>();
        }
        DBuf rn(nodes * sizeof(float), s);
        {
            const __half* hh = static_cast<const __half*>(h);
            const int lpr = static_cast<int>(f / 8);
            const int grid = static_cast<int>(std::max<int64_t>(
                1, std::min<int64_t>((nodes * lpr + 255) / 256, int64_t(num_sms()) * 16)));
            if (lpr == 4) inv_norms<4><<<grid, 256, 0, s>>>(hh, nodes, ldh, eps, rn.as<float>());
            else inv_norms<8><<<grid, 256, 0, s>>>(hh, nodes, ldh, eps, rn.as<float>());
            TCS_LAUNCHED("agnn_inv_norms");
        }
        DBuf partial, pstat;
        if (plan->n_slots) {
            partial = DBuf(plan->n_slots * 8 * f * sizeof(float), s);
            pstat = DBuf(plan->n_slots * 8 * sizeof(float2), s);
        }
        DBuf ctr(dev::kClaimBytes, s);
        TCS_CUDA(cudaMemsetAsync(ctr.p, 0, dev::kClaimBytes, s));
        AttendArgs a{plan->items, plan->n_items, ctr.as<uint32_t>(), mask->row_pointers, mask->column_indices, live,
                     static_cast<const __half*>(h), ldh, rn.as<float>(), row0, rows, scale * kLog2e, c, ldc,
                     partial.as<float>(), pstat.as<float2>()};
        const uint64_t need = (plan->n_items + kAgnnWarps - 1) / kAgnnWarps;
        const int grid = static_cast<int>(
            std::max<uint64_t>(1, std::min<uint64_t>(need, uint64_t(num_sms()) * agnn_bps(f == 32 ? 1 : 2))));
        if (f == 32) agnn_attend_kernel<1><<<grid, kAgnnWarps * 32, 0, s>>>(a);
        else agnn_attend_kernel<2><<<grid, kAgnnWarps * 32, 0, s>>>(a);
        TCS_LAUNCHED("agnn_attend");
        if (plan->n_split) {
            const int g2 = static_cast<int>(std::min<uint64_t>(plan->n_split, 4096));
            agnn_combine<<<g2, 256, 0, s>>>(plan->split, plan->n_split, partial.as<float>(), pstat.as<float2>(), f,
                                            rows, c, ldc);
            TCS_LAUNCHED("agnn_combine");
        }
    });
}
