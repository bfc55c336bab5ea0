// ============================================================================
// TEST INFRASTRUCTURE ONLY -- CPU oracle for the FlashSparse hot path.
//
// This file is a CPU restatement of the reference algorithm
// (/root/reference/proj/include/tcsparse, "the reference") for the path
// CSR -> ME-BCRS -> SpMM / SDDMM.  It is the *checker*: only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs may load it.  The product library (libtcsparse_b200.so) never links,
// loads or calls it, and has no CPU fallback.
//
// Parity pinning: tests/test_oracle.py checks every function here against
// (a) the golden vectors in tests/golden/ that were produced by the
// reference itself (oracle/_ref, built from the reference headers by
// oracle/Makefile) and (b) the reference's own known-answer tests
// (tests/test_formats.cpp, tests/test_tcu_emu.cpp, tests/test_kernels.cpp).
//
// Numerics: every product rnd(a)*rnd(b) of two 11-bit significands is exact
// in binary32, so the reference's sequential fp32 accumulation in ascending
// vector / feature order (inc/mma.hpp:47-61) is reproduced by a plain ordered
// loop.  Built with -ffp-contract=off as a safeguard for everything else.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---- precision (inc/precision.hpp:29-68) ----------------------------------
inline uint32_t f2u(float x) { uint32_t u; std::memcpy(&u, &x, 4); return u; }
inline float u2f(uint32_t u) { float x; std::memcpy(&x, &u, 4); return x; }

// RNE from a 24-bit to an 11-bit significand (inc/precision.hpp:34-37).
inline uint32_t rne13(uint32_t bits) {
    bits += 0xFFFu + ((bits >> 13) & 1u);
    return bits & ~0x1FFFu;
}

// inc/precision.hpp:42-46
inline float rnd_tf32(float x) {
    const uint32_t b = f2u(x);
    if ((b & 0x7F800000u) == 0x7F800000u) return x;
    return u2f(rne13(b));
}

// inc/precision.hpp:51-64
inline float rnd_fp16(float x) {
    const uint32_t b = f2u(x);
    const uint32_t sign = b & 0x80000000u, mag = b & 0x7FFFFFFFu;
    if (mag >= 0x7F800000u) return x;
    if (mag >= 0x477FF000u) return u2f(sign | 0x7F800000u);
    if (mag >= 0x38800000u) return u2f(sign | rne13(mag));
    return std::nearbyintf(x * 0x1p24f) * 0x1p-24f;
}

inline float rnd(float x, int precision) { return precision == 0 ? rnd_fp16(x) : rnd_tf32(x); }

// ---- generators (inc/generate.hpp:13-76) ----------------------------------
inline float small_int_value(std::mt19937& g) {           // generate.hpp:15-18
    const uint32_t m = g() % 8u;
    return static_cast<float>(m < 4 ? static_cast<int>(m) - 4 : static_cast<int>(m) - 3);
}
inline float uniform_real_value(std::mt19937& g) {        // generate.hpp:20-22
    return static_cast<float>(g()) * 0x1p-31f - 1.0f;
}

}  // namespace

extern "C" {

float orc_round_fp16(float x) { return rnd_fp16(x); }
float orc_round_tf32(float x) { return rnd_tf32(x); }

void orc_free(void* p) { std::free(p); }

// Vectorised round_to_precision (inc/precision.hpp:66-68).
void orc_round_array(int precision, const float* in, float* out, uint64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < static_cast<int64_t>(n); ++i) out[i] = rnd(in[i], precision);
}

// generate_random_sparse / _real (generate.hpp:29-59).  Returns nnz; the
// three arrays are malloc'd and released with orc_free.  Returns -1 on an
// argument error (the reference throws ArgumentError).
int64_t orc_generate_random_sparse(uint64_t rows, uint64_t cols, double density, uint64_t seed,
                                   int real, uint32_t** row_ptr, uint32_t** col_idx,
                                   float** values) {
    if (rows == 0 || cols == 0) return -1;
    if (!(density > 0.0) || density > 1.0) return -1;
    std::mt19937 gen(static_cast<uint32_t>(seed));
    const auto threshold = static_cast<uint64_t>(std::llround(density * 4294967296.0));
    std::vector<uint32_t> rp(rows + 1, 0), ci;
    std::vector<float> v;
    ci.reserve(static_cast<size_t>(rows * cols * density * 1.1) + 16);
    v.reserve(ci.capacity());
    for (uint64_t r = 0; r < rows; ++r) {
        for (uint64_t c = 0; c < cols; ++c) {
            if (static_cast<uint64_t>(gen()) < threshold) {
                ci.push_back(static_cast<uint32_t>(c));
                v.push_back(small_int_value(gen));
            }
        }
        rp[r + 1] = static_cast<uint32_t>(ci.size());
    }
    if (real) {  // generate.hpp:55-59
        std::mt19937 g2(static_cast<uint32_t>(seed ^ 0x9e3779b9u));
        for (auto& x : v) x = uniform_real_value(g2);
    }
    const size_t nnz = ci.size();
    *row_ptr = static_cast<uint32_t*>(std::malloc(4 * (rows + 1)));
    *col_idx = static_cast<uint32_t*>(std::malloc(4 * (nnz ? nnz : 1)));
    *values = static_cast<float*>(std::malloc(4 * (nnz ? nnz : 1)));
    std::memcpy(*row_ptr, rp.data(), 4 * (rows + 1));
    if (nnz) {
        std::memcpy(*col_idx, ci.data(), 4 * nnz);
        std::memcpy(*values, v.data(), 4 * nnz);
    }
    return static_cast<int64_t>(nnz);
}

// generate_random_dense / _real (generate.hpp:62-76); out has rows*cols floats.
void orc_generate_random_dense(uint64_t rows, uint64_t cols, uint64_t seed, int real, float* out) {
    std::mt19937 gen(static_cast<uint32_t>(seed));
    const uint64_t n = rows * cols;
    if (real)
        for (uint64_t i = 0; i < n; ++i) out[i] = uniform_real_value(gen);
    else
        for (uint64_t i = 0; i < n; ++i) out[i] = small_int_value(gen);
}

// ---- ME-BCRS encode, phase 1: partition (inc/partition.hpp:40-66) ----------
// Computes row_pointers (num_windows+1 entries, inc/mebcrs.hpp:89-95) and
// returns the stored vector count nv.  Windows are 8 rows; the union of the
// rows' column sets, ascending, is the window's vector list.
// vh = vector height (8; 16 for the baseline16 layout, partition.hpp:42).
int64_t orc_mebcrs_row_pointers_v(uint64_t rows, uint64_t vh, const uint32_t* row_ptr, const uint32_t* col_idx,
                                  uint32_t* out_rp) {
    const uint64_t W = (rows + vh - 1) / vh;
    std::vector<uint32_t> counts(W, 0);
#pragma omp parallel
    {
        std::vector<uint32_t> merged;
#pragma omp for schedule(dynamic, 64)
        for (int64_t w = 0; w < static_cast<int64_t>(W); ++w) {
            merged.clear();
            const uint64_t r0 = vh * w, r1 = std::min<uint64_t>(rows, r0 + vh);
            merged.insert(merged.end(), col_idx + row_ptr[r0], col_idx + row_ptr[r1]);
            std::sort(merged.begin(), merged.end());
            counts[w] = static_cast<uint32_t>(std::unique(merged.begin(), merged.end()) - merged.begin());
        }
    }
    uint64_t acc = 0;
    out_rp[0] = 0;
    for (uint64_t w = 0; w < W; ++w) {
        acc += counts[w];
        out_rp[w + 1] = static_cast<uint32_t>(acc);
    }
    return static_cast<int64_t>(acc);
}
int64_t orc_mebcrs_row_pointers(uint64_t rows, const uint32_t* row_ptr, const uint32_t* col_idx, uint32_t* out_rp) {
    return orc_mebcrs_row_pointers_v(rows, 8, row_ptr, col_idx, out_rp);
}

// ---- ME-BCRS encode, phase 2: column_indices + values ----------------------
// inc/mebcrs.hpp:86-112 without the O(rows*cols) to_dense (:97): each CSR
// entry lands at values[8*(rp[w]+b*k) + r*width_b + j] where its column is
// the (b*k+j)-th vector of window w and width_b = min(k, nv_w - b*k)
// (block_width, inc/mebcrs.hpp:46-51).  Every other slot stays 0.
void orc_mebcrs_fill_v(uint64_t rows, uint64_t vh, const uint32_t* row_ptr, const uint32_t* col_idx,
                       const float* values, uint32_t k, const uint32_t* rp, uint32_t* out_ci, float* out_values) {
    const uint64_t W = (rows + vh - 1) / vh;
    std::memset(out_values, 0, sizeof(float) * vh * rp[W]);
#pragma omp parallel
    {
        std::vector<uint32_t> merged;
#pragma omp for schedule(dynamic, 64)
        for (int64_t w = 0; w < static_cast<int64_t>(W); ++w) {
            merged.clear();
            const uint64_t r0 = vh * w, r1 = std::min<uint64_t>(rows, r0 + vh);
            merged.insert(merged.end(), col_idx + row_ptr[r0], col_idx + row_ptr[r1]);
            std::sort(merged.begin(), merged.end());
            merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
            const uint64_t base = rp[w], nvw = merged.size();
            std::copy(merged.begin(), merged.end(), out_ci + base);
            for (uint64_t r = r0; r < r1; ++r) {
                for (uint64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
                    const uint64_t v = std::lower_bound(merged.begin(), merged.end(), col_idx[p]) - merged.begin();
                    const uint64_t b = v / k, j = v % k;
                    const uint64_t width = std::min<uint64_t>(k, nvw - b * k);
                    out_values[vh * (base + b * k) + (r - r0) * width + j] = values[p];
                }
            }
        }
    }
}
void orc_mebcrs_fill(uint64_t rows, const uint32_t* row_ptr, const uint32_t* col_idx, const float* values,
                     uint32_t k, const uint32_t* rp, uint32_t* out_ci, float* out_values) {
    orc_mebcrs_fill_v(rows, 8, row_ptr, col_idx, values, k, rp, out_ci, out_values);
}

// ---- decode (inc/mebcrs.hpp:118-138): ME-BCRS -> dense, zeros dropped ------
// Writes a dense rows x cols matrix (test sizes only).
void orc_mebcrs_to_dense(uint64_t rows, uint64_t cols, uint32_t k, const uint32_t* rp,
                         const uint32_t* ci, const float* vals, float* dense) {
    const uint64_t W = (rows + 7) / 8;
    std::memset(dense, 0, sizeof(float) * rows * cols);
    for (uint64_t w = 0; w < W; ++w) {
        const uint64_t nvw = rp[w + 1] - rp[w];
        for (uint64_t v = 0; v < nvw; ++v) {
            const uint64_t b = v / k, j = v % k, width = std::min<uint64_t>(k, nvw - b * k);
            for (uint64_t r = 0; r < 8 && 8 * w + r < rows; ++r) {
                const float x = vals[8 * (rp[w] + b * k) + r * width + j];
                if (x != 0.0f) dense[(8 * w + r) * cols + ci[rp[w] + v]] = x;
            }
        }
    }
}

// ---- SpMM (inc/spmm.hpp:103-177) -------------------------------------------
// C[i][n] = sum over the window's vectors v, ascending, of
//           rnd(A_blk[r][v]) * rnd(B[ci[v]][n])   (sequential binary32)
// which is what spmm_swapped computes: blocks in order (:128), each block's
// k products in order inside mma (:55-57), residue slots contributing 0*0
// (:59-74).  `strict` = 1 also visits stored zero fill (matters only for
// non-finite B, 0*inf = NaN); strict = 0 visits the stored vector values
// only.  Empty windows leave rows at 0 (:128).  C is rows x N row-major.
// vh 16: spmm_baseline16 (inc/spmm.hpp:187-257) -- the same sequential
// ascending-vector sum over 16-row windows ("same numerical contract").
void orc_spmm_v(uint64_t rows, uint64_t vh, uint32_t k, int precision, const uint32_t* rp, const uint32_t* ci,
                const float* vals, const float* B, uint64_t ldb, uint64_t N, float* C, uint64_t ldc, int strict) {
    const int64_t W = static_cast<int64_t>((rows + vh - 1) / vh);
#pragma omp parallel
    {
        std::vector<float> acc(N), brow(N);
#pragma omp for schedule(dynamic, 16)
        for (int64_t w = 0; w < W; ++w) {
            const uint64_t nvw = rp[w + 1] - rp[w];
            for (uint64_t r = 0; r < vh && vh * w + r < rows; ++r) {
                std::fill(acc.begin(), acc.end(), 0.0f);
                for (uint64_t v = 0; v < nvw; ++v) {
                    const uint64_t b = v / k, j = v % k, width = std::min<uint64_t>(k, nvw - b * k);
                    const float a = vals[vh * (rp[w] + b * k) + r * width + j];
                    if (a == 0.0f && !strict) continue;
                    const float ar = rnd(a, precision);
                    const float* brp = B + static_cast<uint64_t>(ci[rp[w] + v]) * ldb;
                    for (uint64_t n = 0; n < N; ++n) acc[n] += ar * rnd(brp[n], precision);
                }
                std::copy(acc.begin(), acc.end(), C + (vh * w + r) * ldc);
            }
        }
    }
}
void orc_spmm(uint64_t rows, uint32_t k, int precision, const uint32_t* rp, const uint32_t* ci, const float* vals,
              const float* B, uint64_t ldb, uint64_t N, float* C, uint64_t ldc, int strict) {
    orc_spmm_v(rows, 8, k, precision, rp, ci, vals, B, ldb, N, C, ldc, strict);
}

// ---- SDDMM (inc/sddmm.hpp:84-136) ------------------------------------------
// out[pos] = sum_l rnd(A[i][l]) * rnd(Bt[c][l]), l ascending (the K loop of
// :106-122 accumulates tile after tile, each tile sequential in l), written
// only where mask[pos] != 0 (:131); all other slots of the output blocks are
// 0 (:99-100).  rp/ci are shared with the mask.
void orc_sddmm(uint64_t rows, uint32_t k, int precision, const uint32_t* rp, const uint32_t* ci,
               const float* mask_vals, const float* A, uint64_t lda, const float* Bt, uint64_t ldbt,
               uint64_t F, float* out_vals) {
    const int64_t W = static_cast<int64_t>((rows + 7) / 8);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t w = 0; w < W; ++w) {
        const uint64_t nvw = rp[w + 1] - rp[w];
        for (uint64_t v = 0; v < nvw; ++v) {
            const uint64_t b = v / k, j = v % k, width = std::min<uint64_t>(k, nvw - b * k);
            const float* bt = Bt + static_cast<uint64_t>(ci[rp[w] + v]) * ldbt;
            for (uint64_t r = 0; r < 8; ++r) {
                const uint64_t pos = 8 * (rp[w] + b * k) + r * width + j;
                float acc = 0.0f;
                if (8 * w + r < rows && mask_vals[pos] != 0.0f) {
                    const float* a = A + (8 * w + r) * lda;
                    for (uint64_t l = 0; l < F; ++l) acc += rnd(a[l], precision) * rnd(bt[l], precision);
                }
                out_vals[pos] = acc;
            }
        }
    }
}

// ---- CSR-form restatements for full-size parity (BASELINE configs 3-5) ----
// The reference needs an O(M*K) dense copy to encode (inc/mebcrs.hpp:97),
// so at C3-C5 sizes the oracle computes the same sums straight from the CSR:
//
// SpMM (inc/spmm.hpp:126-163): C[r][n] = sum over the row's stored vectors
// in ascending column order of rnd(a)*rnd(B[c][n]), accumulated sequentially
// in fp32 (mma.hpp:55-57, block after block).  The zero fill and residue
// slots of a window add +-0 and change nothing (orc_spmm_v with strict = 0
// skips them the same way), so the ascending CSR row loop is the same
// sequence of additions.  B is rounded once up front (rnd is a pure function
// of the element).  Rows `sel[i]` (all rows if sel is null) -> C row i.
void orc_spmm_csr_rows(uint64_t rows, int precision, const uint32_t* row_ptr, const uint32_t* col_idx,
                       const float* vals, const float* B, uint64_t b_rows, uint64_t ldb, uint64_t N,
                       const uint64_t* sel, uint64_t n_sel, float* C, uint64_t ldc) {
    std::vector<float> Br(b_rows * N);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < static_cast<int64_t>(b_rows); ++i)
        for (uint64_t n = 0; n < N; ++n) Br[i * N + n] = rnd(B[i * ldb + n], precision);
    const int64_t cnt = static_cast<int64_t>(sel ? n_sel : rows);
#pragma omp parallel
    {
        std::vector<float> acc(N);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < cnt; ++i) {
            const uint64_t r = sel ? sel[i] : static_cast<uint64_t>(i);
            std::fill(acc.begin(), acc.end(), 0.0f);
            for (uint32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
                if (vals[e] == 0.0f) continue;
                const float a = rnd(vals[e], precision);
                const float* brp = Br.data() + static_cast<uint64_t>(col_idx[e]) * N;
                for (uint64_t n = 0; n < N; ++n) acc[n] += a * brp[n];
            }
            std::copy(acc.begin(), acc.end(), C + i * ldc);
        }
    }
}

// SDDMM (inc/sddmm.hpp:102-132) per CSR entry of the selected rows, in CSR
// order: dot[e] = sum_l rnd(A[r][l]) * rnd(Bt[c][l]) (l ascending) where the
// f32 value is nonzero (:131), else 0; pos[e] = the entry's slot in the
// ME-BCRS value array 8*(rp[w]+b*k) + (r%8)*width_b + j (inc/mebcrs.hpp:46-56)
// for the window's vector list (rp, ci) -- the vector index j of column c is
// found by a merge of the ascending row and window lists.  Entries are
// written at offsets eoff[i] + (e - row_ptr[r]) (eoff: prefix of the
// selected rows' lengths).
void orc_sddmm_csr_rows(uint64_t rows, int precision, uint32_t k, const uint32_t* row_ptr, const uint32_t* col_idx,
                        const float* vals, const uint32_t* rp, const uint32_t* ci, const float* A, uint64_t lda,
                        const float* Bt, uint64_t ldbt, uint64_t F, const uint64_t* sel, uint64_t n_sel,
                        const uint64_t* eoff, float* dot, uint64_t* pos) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < static_cast<int64_t>(n_sel); ++i) {
        const uint64_t r = sel[i], w = r / 8;
        const uint32_t base = rp ? rp[w] : 0, nvw = rp ? rp[w + 1] - base : 0;
        uint32_t j = 0;
        for (uint32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
            const uint32_t c = col_idx[e];
            const uint64_t o = eoff[i] + (e - row_ptr[r]);
            if (rp) {  // rp == null: dot products only (the CPU-baseline timing)
                while (j < nvw && ci[base + j] < c) ++j;
                if (j >= nvw || ci[base + j] != c) {  // not a vector of the window: an encoding error
                    pos[o] = ~0ull;
                    dot[o] = 0.0f;
                    continue;
                }
                const uint32_t b = j / k, jj = j % k, width = std::min(k, nvw - b * k);
                pos[o] = 8ull * (base + b * k) + (r % 8) * width + jj;
            }
            float acc = 0.0f;
            if (vals[e] != 0.0f) {
                const float* a = A + r * lda;
                const float* bt = Bt + static_cast<uint64_t>(c) * ldbt;
                for (uint64_t l = 0; l < F; ++l) acc += rnd(a[l], precision) * rnd(bt[l], precision);
            }
            dot[o] = acc;
        }
    }
}

// count_mma (inc/analysis.hpp:34-38) for the swap8 strategy:
//   sum_w ceil(nv_w / k) * ceil(N / 16).
uint64_t orc_count_mma_spmm(uint64_t W, const uint32_t* rp, uint32_t k, uint64_t N) {
    uint64_t blocks = 0;
    for (uint64_t w = 0; w < W; ++w) blocks += (rp[w + 1] - rp[w] + k - 1) / k;
    return blocks * ((N + 15) / 16);
}

// SDDMM invocation count (inc/sddmm.hpp:102-121): sum_w ceil(nv_w/16) * ceil(F/k).
uint64_t orc_count_mma_sddmm(uint64_t W, const uint32_t* rp, uint32_t k, uint64_t F) {
    uint64_t groups = 0;
    for (uint64_t w = 0; w < W; ++w) groups += (rp[w + 1] - rp[w] + 15) / 16;
    return groups * ((F + k - 1) / k);
}

// Raw std::mt19937 draws, so tests can replay the reference tests' seeded
// size / value sequences (e.g. tests/acceptance.cpp:90-96).
void orc_mt19937(uint32_t seed, uint64_t n, uint32_t* out) {
    std::mt19937 g(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = g();
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

}  // extern "C"
