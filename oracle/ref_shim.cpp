// ============================================================================
// TEST INFRASTRUCTURE ONLY -- C-ABI shim over the *unmodified* reference
// headers (/root/reference/proj/include/tcsparse).  oracle/Makefile compiles
// this file against the reference sources where they lie and writes the
// result to oracle/_ref/libtcsref.so (git-ignored; it travels to the GPU box
// as a prebuilt file).  It is used to (1) generate the golden vectors under
// tests/golden/, (2) pin the restatement in oracle/oracle.cpp, and (3) time
// the reference's own CPU path in bench.py (--impl reference / cpu_baseline).
// No reference source is copied into this repository.
// ============================================================================
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <vector>

#include <sstream>
#include <string>

#include "tcsparse/cli.hpp"
#include "tcsparse/tcsparse.hpp"

using namespace tcsparse;

namespace {

template <typename T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

CsrMatrix make_csr(uint64_t rows, uint64_t cols, const uint32_t* rp, const uint32_t* ci,
                   const float* vals) {
    CsrMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.row_ptr.assign(rp, rp + rows + 1);
    const uint64_t nnz = rp[rows];
    m.col_idx.assign(ci, ci + nnz);
    m.values.assign(vals, vals + nnz);
    return m;
}

MeBcrsMatrix make_me(uint64_t rows, uint64_t cols, int precision, const uint32_t* rp,
                     const uint32_t* ci, const float* vals) {
    MeBcrsMatrix me;
    const Precision p = static_cast<Precision>(precision);
    const MmaShape s = shape_for(p);
    me.rows = rows;
    me.cols = cols;
    me.vector_height = s.n;
    me.k = s.k;
    me.precision = p;
    const uint64_t W = (rows + 7) / 8;
    me.row_pointers.assign(rp, rp + W + 1);
    const uint64_t nv = rp[W];
    me.column_indices.assign(ci, ci + nv);
    me.values.assign(vals, vals + 8 * nv);
    return me;
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }
float ref_round_fp16(float x) { return round_to_fp16(x); }
float ref_round_tf32(float x) { return round_to_tf32(x); }

int64_t ref_generate_random_sparse(uint64_t rows, uint64_t cols, double density, uint64_t seed,
                                   int real, uint32_t** rp, uint32_t** ci, float** vals) {
    try {
        const CsrMatrix m = real ? generate_random_sparse_real(rows, cols, density, seed)
                                 : generate_random_sparse(rows, cols, density, seed);
        *rp = dup(m.row_ptr);
        *ci = dup(m.col_idx);
        *vals = dup(m.values);
        return static_cast<int64_t>(m.nnz());
    } catch (const std::exception&) {
        return -1;
    }
}

void ref_generate_random_dense(uint64_t rows, uint64_t cols, uint64_t seed, int real, float* out) {
    const DenseMatrix d = real ? generate_random_dense_real(rows, cols, seed)
                               : generate_random_dense(rows, cols, seed);
    std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
}

// encode_mebcrs (inc/mebcrs.hpp:80). Returns nv, or -1 on error.
int64_t ref_encode_mebcrs(uint64_t rows, uint64_t cols, const uint32_t* rp, const uint32_t* ci,
                          const float* vals, int precision, uint32_t** out_rp, uint32_t** out_ci,
                          float** out_vals) {
    try {
        const MeBcrsMatrix me = encode_mebcrs(make_csr(rows, cols, rp, ci, vals),
                                              static_cast<Precision>(precision));
        *out_rp = dup(me.row_pointers);
        *out_ci = dup(me.column_indices);
        *out_vals = dup(me.values);
        return static_cast<int64_t>(me.column_indices.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// decode_mebcrs (inc/mebcrs.hpp:118). Returns nnz, or -1 (FormatError).
int64_t ref_decode_mebcrs(uint64_t rows, uint64_t cols, int precision, const uint32_t* rp,
                          const uint32_t* ci, const float* vals, uint32_t** out_rp,
                          uint32_t** out_ci, float** out_vals) {
    try {
        const CsrMatrix m = decode_mebcrs(make_me(rows, cols, precision, rp, ci, vals));
        *out_rp = dup(m.row_ptr);
        *out_ci = dup(m.col_idx);
        *out_vals = dup(m.values);
        return static_cast<int64_t>(m.nnz());
    } catch (const std::exception&) {
        return -1;
    }
}

// spmm(MeBcrsMatrix) (inc/spmm.hpp:173). C is rows x N. Returns 0, or
// 1 = ArgumentError, 2 = ShapeError, 3 = other.
int ref_spmm(uint64_t rows, uint64_t cols, int precision, const uint32_t* rp, const uint32_t* ci,
             const float* vals, const float* B, uint64_t b_rows, uint64_t N, int cfg_precision,
             uint64_t vector_height, int mapping, float* C, uint64_t* mma_invocations) {
    try {
        DenseMatrix b(b_rows, N);
        std::memcpy(b.data.data(), B, sizeof(float) * b_rows * N);
        const KernelConfig cfg{static_cast<Precision>(cfg_precision), vector_height,
                               static_cast<ThreadMapping>(mapping)};
        const SpmmResult res = spmm(make_me(rows, cols, precision, rp, ci, vals), b, cfg);
        std::memcpy(C, res.output.data.data(), sizeof(float) * rows * N);
        if (mma_invocations) *mma_invocations = res.counters.mma_invocations;
        return 0;
    } catch (const ArgumentError&) {
        return 1;
    } catch (const ShapeError&) {
        return 2;
    } catch (const std::exception&) {
        return 3;
    }
}

// encode_srbcrs (inc/srbcrs.hpp:40-72). Returns the padded vector count, or -1.
int64_t ref_encode_srbcrs(uint64_t rows, uint64_t cols, const uint32_t* rp, const uint32_t* ci, const float* vals,
                          int precision, uint32_t** out_pairs, uint32_t** out_ci, float** out_vals) {
    try {
        const SrBcrsMatrix sr = encode_srbcrs(make_csr(rows, cols, rp, ci, vals), static_cast<Precision>(precision));
        *out_pairs = dup(sr.row_pointer_pairs);
        *out_ci = dup(sr.column_indices);
        *out_vals = dup(sr.values);
        return static_cast<int64_t>(sr.column_indices.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// spmm(SrBcrsMatrix) (inc/spmm.hpp:181-185) on arrays from ref_encode_srbcrs.
int ref_spmm_srbcrs(uint64_t rows, uint64_t cols, int precision, const uint32_t* pairs, const uint32_t* ci,
                    const float* vals, const float* B, uint64_t b_rows, uint64_t N, int cfg_precision, float* C,
                    uint64_t* mma_invocations) {
    try {
        SrBcrsMatrix sr;
        const Precision p = static_cast<Precision>(precision);
        sr.rows = rows;
        sr.cols = cols;
        sr.vector_height = 8;
        sr.k = shape_for(p).k;
        sr.precision = p;
        const uint64_t W = (rows + 7) / 8;
        sr.row_pointer_pairs.assign(pairs, pairs + 2 * W);
        const uint64_t P = W ? pairs[2 * W - 1] : 0;
        sr.column_indices.assign(ci, ci + P);
        sr.values.assign(vals, vals + 8 * P);
        DenseMatrix b(b_rows, N);
        std::memcpy(b.data.data(), B, sizeof(float) * b_rows * N);
        const SpmmResult res = spmm(sr, b, KernelConfig{static_cast<Precision>(cfg_precision), 8,
                                                        ThreadMapping::coalesced});
        std::memcpy(C, res.output.data.data(), sizeof(float) * rows * N);
        if (mma_invocations) *mma_invocations = res.counters.mma_invocations;
        return 0;
    } catch (const ArgumentError&) {
        return 1;
    } catch (const ShapeError&) {
        return 2;
    } catch (const std::exception&) {
        return 3;
    }
}

// sddmm (inc/sddmm.hpp:84). out_vals has 8*nv floats.
int ref_sddmm(uint64_t rows, uint64_t cols, int precision, const uint32_t* rp, const uint32_t* ci,
              const float* mask_vals, const float* A, uint64_t a_rows, const float* Bt,
              uint64_t bt_rows, uint64_t F_a, uint64_t F_b, int cfg_precision, float* out_vals,
              uint64_t* mma_invocations) {
    try {
        SddmmOperands ops;
        ops.mask = make_me(rows, cols, precision, rp, ci, mask_vals);
        ops.a = DenseMatrix(a_rows, F_a);
        std::memcpy(ops.a.data.data(), A, sizeof(float) * a_rows * F_a);
        ops.b_t = DenseMatrix(bt_rows, F_b);
        std::memcpy(ops.b_t.data.data(), Bt, sizeof(float) * bt_rows * F_b);
        const KernelConfig cfg{static_cast<Precision>(cfg_precision), 8, ThreadMapping::coalesced};
        const SddmmResult res = sddmm(ops, cfg);
        std::memcpy(out_vals, res.output.values.data(), sizeof(float) * res.output.values.size());
        if (mma_invocations) *mma_invocations = res.counters.mma_invocations;
        return 0;
    } catch (const ArgumentError&) {
        return 1;
    } catch (const ShapeError&) {
        return 2;
    } catch (const std::exception&) {
        return 3;
    }
}

// partition_windows (inc/partition.hpp:40-66) at any vector height, as
// CSR-style row pointers + concatenated window column lists.  Returns nv.
int64_t ref_partition_windows(uint64_t rows, uint64_t cols, const uint32_t* rp, const uint32_t* ci,
                              const float* vals, uint64_t vector_height, uint64_t k, uint32_t** out_rp,
                              uint32_t** out_ci) {
    try {
        const WindowPartition part = partition_windows(make_csr(rows, cols, rp, ci, vals), vector_height, k);
        std::vector<uint32_t> prp(1, 0), pci;
        for (const auto& w : part.windows) {
            pci.insert(pci.end(), w.begin(), w.end());
            prp.push_back(static_cast<uint32_t>(pci.size()));
        }
        *out_rp = dup(prp);
        *out_ci = dup(pci);
        return static_cast<int64_t>(pci.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// spmm_baseline16 (inc/spmm.hpp:187-257).  Returns 0 / 1 ArgumentError /
// 2 ShapeError / 3 other.
int ref_spmm_baseline16(uint64_t rows, uint64_t cols, const uint32_t* rp, const uint32_t* ci, const float* vals,
                        const float* B, uint64_t b_rows, uint64_t N, int precision, uint64_t vector_height,
                        float* C, uint64_t* mma_invocations) {
    try {
        DenseMatrix b(b_rows, N);
        std::memcpy(b.data.data(), B, sizeof(float) * b_rows * N);
        const KernelConfig cfg{static_cast<Precision>(precision), vector_height, ThreadMapping::coalesced};
        const SpmmResult res = spmm_baseline16(make_csr(rows, cols, rp, ci, vals), b, cfg);
        std::memcpy(C, res.output.data.data(), sizeof(float) * rows * N);
        if (mma_invocations) *mma_invocations = res.counters.mma_invocations;
        return 0;
    } catch (const ArgumentError&) {
        return 1;
    } catch (const ShapeError&) {
        return 2;
    } catch (const std::exception&) {
        return 3;
    }
}

// ---- the reference CLI (inc/cli.hpp:104-358), stdout/stderr captured ----
static char* dup_str(const std::string& x) {
    char* p = static_cast<char*>(std::malloc(x.size() + 1));
    std::memcpy(p, x.c_str(), x.size() + 1);
    return p;
}

// cmd: 0 convert, 1 spmm, 2 sddmm, 3 stats, 4 bench.  n_list has n_count
// entries (spmm/sddmm/bench use the last).  Returns the exit code.
int ref_cli(int cmd, const char* input, const char* dir, const char* output, int precision, int mapping,
            const uint64_t* n_list, int n_count, uint64_t vector_height, uint64_t seed, int verify, int real,
            int json, char** out_text, char** err_text) {
    std::ostringstream out, err;
    int rc = -1;
    try {
        const Precision p = static_cast<Precision>(precision);
        const ThreadMapping m = mapping == 0 ? ThreadMapping::direct : ThreadMapping::coalesced;
        std::vector<std::size_t> ns(n_list, n_list + n_count);
        switch (cmd) {
            case 0: {
                cli::ConvertOptions o;
                o.input = input;
                o.output = output;
                o.precision = p;
                rc = cli::run_convert(o, out, err);
                break;
            }
            case 1: {
                cli::SpmmOptions o;
                o.input = input;
                if (!ns.empty()) o.n = ns.back();
                o.precision = p;
                o.vector_height = vector_height;
                o.mapping = m;
                o.seed = seed;
                o.verify = verify;
                o.real_values = real;
                rc = cli::run_spmm(o, out, err);
                break;
            }
            case 2: {
                cli::SddmmOptions o;
                o.input = input;
                if (!ns.empty()) o.n = ns.back();
                o.precision = p;
                o.seed = seed;
                o.verify = verify;
                o.real_values = real;
                o.output = output;
                rc = cli::run_sddmm(o, out, err);
                break;
            }
            case 3: {
                cli::StatsOptions o;
                o.input = input;
                o.dir = dir;
                if (!ns.empty()) o.n_list = ns;
                o.mapping = m;
                o.format = json ? ReportFormat::json : ReportFormat::csv;
                o.output = output;
                rc = cli::run_stats(o, out, err);
                break;
            }
            case 4: {
                cli::BenchOptions o;
                o.input = input;
                o.dir = dir;
                if (!ns.empty()) o.n = ns.back();
                o.seed = seed;
                o.mapping = m;
                o.output = output;
                rc = cli::run_bench(o, out, err);
                break;
            }
        }
    } catch (const std::exception& e) {
        err << "exception: " << e.what() << "\n";
        rc = -2;
    }
    *out_text = dup_str(out.str());
    *err_text = dup_str(err.str());
    return rc;
}

// parse_matrix_market (inc/matrix_market.hpp:28-94) of an in-memory text.
// Returns nnz, or -1 with *err_text = the ParseError message.
int64_t ref_parse_matrix_market(const char* text, uint64_t len, uint64_t* rows, uint64_t* cols, uint32_t** rp,
                                uint32_t** ci, float** vals, char** err_text) {
    *err_text = nullptr;
    try {
        std::istringstream in(std::string(text, len));
        const CsrMatrix m = parse_matrix_market(in);
        *rows = m.rows;
        *cols = m.cols;
        *rp = dup(m.row_ptr);
        *ci = dup(m.col_idx);
        *vals = dup(m.values);
        return static_cast<int64_t>(m.nnz());
    } catch (const std::exception& e) {
        *err_text = dup_str(e.what());
        return -1;
    }
}

// read_mebcrs (inc/container_io.hpp:70-91) of a file; returns nv or -1 with
// the FormatError message.
int64_t ref_read_mebcrs(const char* path, uint64_t* rows, uint64_t* cols, int* precision, uint32_t** rp,
                        uint32_t** ci, float** vals, char** err_text) {
    *err_text = nullptr;
    try {
        std::ifstream in(path, std::ios::binary);
        const MeBcrsMatrix m = read_mebcrs(in);
        *rows = m.rows;
        *cols = m.cols;
        *precision = static_cast<int>(m.precision);
        *rp = dup(m.row_pointers);
        *ci = dup(m.column_indices);
        *vals = dup(m.values);
        return static_cast<int64_t>(m.column_indices.size());
    } catch (const std::exception& e) {
        *err_text = dup_str(e.what());
        return -1;
    }
}

uint64_t ref_sddmm_output_offsets(uint64_t lane, int kind) {
    return sddmm_output_offsets(lane, kind == 0 ? SubBlockKind::b8x8 : SubBlockKind::b8x4);
}

// ---- timed reference pipelines for bench.py's CPU baseline -----------------
// The reference CLI's pipelines (inc/cli.hpp:162-200 spmm, :205-240 sddmm):
// encode_mebcrs then spmm / sddmm on a CSR row slice, against a dense
// operand built once (ref_dense_new) so that the shim's own copies stay out
// of the measurement.  Returns the seconds spent inside the reference calls,
// or a negative value on error.
void* ref_dense_new(uint64_t rows, uint64_t cols, const float* data) {
    auto* d = new DenseMatrix(rows, cols);
    std::memcpy(d->data.data(), data, sizeof(float) * rows * cols);
    return d;
}
void ref_dense_free(void* d) { delete static_cast<DenseMatrix*>(d); }

double ref_time_encode_spmm(uint64_t rows, uint64_t cols, const uint32_t* rp, const uint32_t* ci,
                            const float* vals, int precision, const void* dense, float* C) {
    try {
        const CsrMatrix m = make_csr(rows, cols, rp, ci, vals);
        const DenseMatrix& b = *static_cast<const DenseMatrix*>(dense);
        const Precision p = static_cast<Precision>(precision);
        const auto t0 = std::chrono::steady_clock::now();
        const MeBcrsMatrix me = encode_mebcrs(m, p);
        const SpmmResult res = spmm(me, b, KernelConfig{p, 8, ThreadMapping::coalesced});
        const auto t1 = std::chrono::steady_clock::now();
        std::memcpy(C, res.output.data.data(), sizeof(float) * rows * b.cols);
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception&) {
        return -1.0;
    }
}

double ref_time_encode_sddmm(uint64_t rows, uint64_t cols, const uint32_t* rp, const uint32_t* ci,
                             const float* vals, int precision, const float* A, uint64_t F, const void* bt_dense,
                             float* out_vals, uint64_t out_cap) {
    try {
        const CsrMatrix m = make_csr(rows, cols, rp, ci, vals);
        const Precision p = static_cast<Precision>(precision);
        SddmmOperands ops;
        ops.a = DenseMatrix(rows, F);
        std::memcpy(ops.a.data.data(), A, sizeof(float) * rows * F);
        ops.b_t = *static_cast<const DenseMatrix*>(bt_dense);
        const auto t0 = std::chrono::steady_clock::now();
        ops.mask = encode_mebcrs(m, p);
        const SddmmResult res = sddmm(ops, KernelConfig{p, 8, ThreadMapping::coalesced});
        const auto t1 = std::chrono::steady_clock::now();
        const uint64_t n = std::min<uint64_t>(out_cap, res.output.values.size());
        std::memcpy(out_vals, res.output.values.data(), sizeof(float) * n);
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception&) {
        return -1.0;
    }
}

}  // extern "C"
