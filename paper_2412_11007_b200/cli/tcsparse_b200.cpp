// tcsparse-b200 -- the reference's command-line front end (ref
// proj/tools/tcsparse.cpp + inc/cli.hpp) on the B200 path: every matrix is
// parsed through tcs_matrix_market_read (GPU CSR assembly), converted and
// multiplied by the sm_100a kernels, and the structural counters come from
// the GPU cost model (tcs_mebcrs_cost).  Subcommands, options, report
// formats, verification rules and exit codes follow the reference so that
// outputs can be diffed byte for byte (tests/test_gpu_cli.py does).
//
//   convert --input A.mtx [--output A.mebc] [--precision fp16|tf32]
//   spmm    --input A.mtx [--n 128] [--vector 8|16] [--seed 1] [--verify] [--real]
//           [--precision ..] [--mapping direct|coalesced]
//   sddmm   --input M.mtx [--n 32] [--seed 1] [--output O.mebc] [--verify] [--real] [--precision ..]
//   stats   (--input A.mtx | --dir D) [--n N]... [--mapping ..] [--format csv|json] [--output F]
//   bench   (--input A.mtx | --dir D) [--n 128] [--seed 1] [--mapping ..] [--output F]
//
// The dense operands come from the reference's generators (ref
// generate.hpp:13-22, 62-76: raw std::mt19937 draws), restated below.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "tcs/tcs.h"

namespace {

// Exit codes (ref cli.hpp:23-26).
constexpr int kExitOk = 0, kExitPartial = 1, kExitInputError = 2, kExitVerifyFailed = 3, kExitDevice = 4;
constexpr double kRealTolFp16 = 1e-2, kRealTolTf32 = 1e-3;  // ref cli.hpp:30-31

struct DeviceError {
    std::string what;
};
struct InputError {  // ParseError / unreadable input
    std::string what;
};

void check(tcs_status s) {
    if (s == TCS_OK) return;
    if (s == TCS_ERR_PARSE) throw InputError{tcs_last_error()};
    throw DeviceError{tcs_last_error()};
}

const char* prec_name(tcs_precision p) { return p == TCS_FP16 ? "fp16" : "tf32"; }
const char* map_name(tcs_mapping m) { return m == TCS_MAP_DIRECT ? "direct" : "coalesced"; }

// ------------------------------------------------ ref generate.hpp restated
float small_int_value(std::mt19937& g) {
    const uint32_t m = g() % 8u;
    return static_cast<float>(m < 4 ? static_cast<int>(m) - 4 : static_cast<int>(m) - 3);
}
float uniform_real_value(std::mt19937& g) { return static_cast<float>(g()) * 0x1p-31f - 1.0f; }

struct Dense {
    uint64_t rows = 0, cols = 0;
    std::vector<float> data;
};
Dense generate_dense(uint64_t rows, uint64_t cols, uint64_t seed, bool real) {
    std::mt19937 g(static_cast<uint32_t>(seed));
    Dense d{rows, cols, std::vector<float>(rows * cols)};
    for (auto& v : d.data) v = real ? uniform_real_value(g) : small_int_value(g);
    return d;
}

// ------------------------------------------------------------ host CSR
struct Csr {
    tcs_csr m{};
    Csr() = default;
    Csr(const Csr&) = delete;
    ~Csr() { tcs_csr_free_host(&m); }
};

void load_matrix_market(const std::string& path, Csr& out) { check(tcs_matrix_market_read(path.c_str(), &out.m, nullptr)); }

struct Handle {
    tcs_mebcrs h{};
    Handle() = default;
    Handle(const Handle&) = delete;
    ~Handle() { tcs_mebcrs_free(&h, nullptr); }
};

// Device buffer for the operands this tool stages itself.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) throw DeviceError{"cudaMalloc failed"};
    }
    DevBuf(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFree(p); }
    void up(const void* src, size_t bytes) {
        if (bytes && cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
            throw DeviceError{"cudaMemcpy H2D failed"};
    }
    void down(void* dst, size_t bytes) const {
        if (bytes && cudaMemcpy(dst, p, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
            throw DeviceError{"cudaMemcpy D2H failed"};
    }
};

void encode_any(const Csr& c, tcs_precision p, uint32_t vh, Handle& out) {
    if (vh == 8) {
        check(tcs_mebcrs_encode_host(&c.m, p, TCS_DTYPE_F32, &out.h, nullptr));
        return;
    }
    DevBuf rp((c.m.rows + 1) * 4), ci(c.m.nnz * 4), v(c.m.nnz * 4);
    rp.up(c.m.row_ptr, (c.m.rows + 1) * 4);
    ci.up(c.m.col_idx, c.m.nnz * 4);
    v.up(c.m.values, c.m.nnz * 4);
    const tcs_csr d{c.m.rows, c.m.cols, c.m.nnz, static_cast<uint32_t*>(rp.p), static_cast<uint32_t*>(ci.p),
                    static_cast<float*>(v.p)};
    check(tcs_mebcrs_encode_v(&d, p, TCS_DTYPE_F32, vh, &out.h, nullptr));
}

// C = A * B on the GPU (swap8 or baseline16), host result + counters.
std::vector<float> run_spmm_gpu(const Handle& a, const Dense& b, tcs_precision p, uint32_t vh, tcs_mapping mapping,
                                tcs_counters& cnt) {
    DevBuf db(b.data.size() * 4), dc(a.h.rows * b.cols * 4);
    db.up(b.data.data(), b.data.size() * 4);
    const tcs_kernel_config cfg{p, vh, mapping, TCS_CFG_COUNT_ACCESS};
    if (vh == 8)
        check(tcs_spmm(&a.h, db.p, TCS_DTYPE_F32, static_cast<int64_t>(b.cols), static_cast<int64_t>(b.rows),
                       static_cast<int64_t>(b.cols), static_cast<float*>(dc.p), static_cast<int64_t>(b.cols), &cfg,
                       &cnt, nullptr));
    else
        check(tcs_spmm_baseline16(&a.h, db.p, TCS_DTYPE_F32, static_cast<int64_t>(b.cols),
                                  static_cast<int64_t>(b.rows), static_cast<int64_t>(b.cols),
                                  static_cast<float*>(dc.p), static_cast<int64_t>(b.cols), &cfg, &cnt, nullptr));
    std::vector<float> out(a.h.rows * b.cols);
    dc.down(out.data(), out.size() * 4);
    return out;
}

// ref cli.hpp:42-53 (dense_matmul_reference) on the CSR: same ascending-l
// order and zero skipping, so the doubles are identical.
std::vector<double> matmul_reference(const Csr& a, const Dense& b) {
    std::vector<double> out(a.m.rows * b.cols, 0.0);
    for (uint64_t i = 0; i < a.m.rows; ++i)
        for (uint64_t p = a.m.row_ptr[i]; p < a.m.row_ptr[i + 1]; ++p) {
            const double av = a.m.values[p];
            if (av == 0.0) continue;
            const float* br = b.data.data() + static_cast<uint64_t>(a.m.col_idx[p]) * b.cols;
            double* o = out.data() + i * b.cols;
            for (uint64_t j = 0; j < b.cols; ++j) o[j] += av * static_cast<double>(br[j]);
        }
    return out;
}

struct Verify {
    bool exact = true, within_tol = true;
    double max_abs_diff = 0.0;
};
// ref cli.hpp:61-72
Verify compare(const std::vector<float>& got, const std::vector<double>& want, double tol) {
    Verify v;
    for (size_t i = 0; i < got.size(); ++i) {
        const double diff = std::abs(static_cast<double>(got[i]) - want[i]);
        v.max_abs_diff = std::max(v.max_abs_diff, diff);
        if (diff != 0.0) v.exact = false;
        if (diff > tol * std::max(1.0, std::abs(want[i]))) v.within_tol = false;
    }
    return v;
}

// ref cli.hpp:74-89
std::vector<std::string> collect_inputs(const std::string& input, const std::string& dir, std::ostream& err) {
    std::vector<std::string> files;
    if (!input.empty()) {
        files.push_back(input);
    } else {
        std::error_code ec;
        for (const auto& e : std::filesystem::directory_iterator(dir, ec))
            if (e.is_regular_file() && e.path().extension() == ".mtx") files.push_back(e.path().string());
        if (ec) err << "error: cannot read directory '" << dir << "'\n";
        std::sort(files.begin(), files.end());
    }
    return files;
}
std::string matrix_id(const std::string& path) { return std::filesystem::path(path).stem().string(); }
void write_text(const std::string& path, const std::string& text, std::ostream& out) {
    if (path.empty()) {
        out << text;
        return;
    }
    std::ofstream f(path, std::ios::binary);
    f << text;
}

// ------------------------------------------------------------- commands
struct Opts {
    std::string input, output, dir, format = "csv";
    tcs_precision precision = TCS_FP16;
    tcs_mapping mapping = TCS_MAP_COALESCED;
    std::vector<uint64_t> n_list;
    uint64_t vector = 8, seed = 1;
    bool verify = false, real = false;
};

// ref cli.hpp:104-148
int run_convert(const Opts& o, std::ostream& out, std::ostream& err) {
    Csr csr;
    try {
        load_matrix_market(o.input, csr);
    } catch (const InputError& e) {
        err << "error: " << o.input << ": " << e.what << "\n";
        return kExitInputError;
    }
    Handle me;
    encode_any(csr, o.precision, 8, me);
    if (!o.output.empty()) {
        const tcs_status s = tcs_mebcrs_write(o.output.c_str(), &me.h, nullptr);
        if (s == TCS_ERR_IO) {
            err << "error: cannot open output '" << o.output << "'\n";
            return kExitInputError;
        }
        check(s);
    }
    tcs_cost cost{};
    check(tcs_mebcrs_cost(&me.h, csr.m.nnz, 0, TCS_MAP_COALESCED, &cost, nullptr));
    const uint64_t vw = o.precision == TCS_FP16 ? 2 : 4;
    const uint64_t me_ptr = (me.h.num_windows + 1) * 4, sr_ptr = 2 * me.h.num_windows * 4;
    out << "matrix: " << csr.m.rows << "x" << csr.m.cols << " nnz=" << csr.m.nnz << "\n";
    out << "stored vectors: " << me.h.num_vectors << " (padded: " << cost.padded_vectors << ")\n";
    out << "pointer bytes: me=" << me_ptr << " sr=" << sr_ptr << "\n";
    out << "footprint bytes (" << prec_name(o.precision) << ", " << vw << "-byte values): me=" << cost.footprint_me
        << " sr=" << cost.footprint_sr << " reduction="
        << (cost.footprint_sr == 0 ? 0.0
                                   : 1.0 - static_cast<double>(cost.footprint_me) /
                                               static_cast<double>(cost.footprint_sr))
        << "\n";
    return kExitOk;
}

// ref cli.hpp:164-213
int run_spmm(const Opts& o, std::ostream& out, std::ostream& err) {
    Csr csr;
    try {
        load_matrix_market(o.input, csr);
    } catch (const InputError& e) {
        err << "error: " << o.input << ": " << e.what << "\n";
        return kExitInputError;
    }
    const uint64_t n = o.n_list.empty() ? 128 : o.n_list.back();
    const Dense dense = generate_dense(csr.m.cols, n, o.seed, o.real);
    Handle a;
    const uint32_t vh = o.vector == 8 ? 8 : 16;
    encode_any(csr, o.precision, vh, a);
    tcs_counters cnt{};
    const std::vector<float> got = run_spmm_gpu(a, dense, o.precision, vh, o.mapping, cnt);
    out << "spmm vector=" << o.vector << " precision=" << prec_name(o.precision) << " mapping=" << map_name(o.mapping)
        << " n=" << n << "\n";
    out << "mma=" << cnt.mma_invocations << " transactions=" << cnt.transactions
        << " transaction_bytes=" << cnt.transaction_bytes << " useful_bytes=" << cnt.useful_bytes << "\n";
    if (o.verify) {
        const auto want = matmul_reference(csr, dense);
        const double tol = o.precision == TCS_FP16 ? kRealTolFp16 : kRealTolTf32;
        const Verify v = compare(got, want, tol);
        if (o.real ? !v.within_tol : !v.exact) {
            err << "verification FAILED: max_abs_diff=" << v.max_abs_diff << "\n";
            return kExitVerifyFailed;
        }
        out << (v.exact ? "verify: exact match\n"
                        : "verify: within tolerance, max_abs_diff=" + std::to_string(v.max_abs_diff) + "\n");
    }
    return kExitOk;
}

// ref cli.hpp:225-271
int run_sddmm(const Opts& o, std::ostream& out, std::ostream& err) {
    Csr csr;
    try {
        load_matrix_market(o.input, csr);
    } catch (const InputError& e) {
        err << "error: " << o.input << ": " << e.what << "\n";
        return kExitInputError;
    }
    const uint64_t n = o.n_list.empty() ? 32 : o.n_list.back();
    Handle mask;
    encode_any(csr, o.precision, 8, mask);
    const Dense A = generate_dense(csr.m.rows, n, o.seed, o.real);
    const Dense Bt = generate_dense(csr.m.cols, n, o.seed + 1, o.real);
    DevBuf da(A.data.size() * 4), db(Bt.data.size() * 4), dv(8 * mask.h.num_vectors * 4);
    da.up(A.data.data(), A.data.size() * 4);
    db.up(Bt.data.data(), Bt.data.size() * 4);
    Handle res;
    res.h.values = dv.p;  // caller-owned output values
    const tcs_kernel_config cfg{o.precision, 8, TCS_MAP_COALESCED, 0};
    tcs_counters cnt{};
    check(tcs_sddmm(&mask.h, da.p, TCS_DTYPE_F32, static_cast<int64_t>(n), static_cast<int64_t>(A.rows),
                    static_cast<int64_t>(n), db.p, TCS_DTYPE_F32, static_cast<int64_t>(n),
                    static_cast<int64_t>(Bt.rows), static_cast<int64_t>(n), &res.h, TCS_DTYPE_F32, &cfg, &cnt,
                    nullptr));
    out << "sddmm precision=" << prec_name(o.precision) << " k=" << n << " sampled=" << csr.m.nnz << "\n";
    out << "mma=" << cnt.mma_invocations << "\n";
    if (o.verify) {
        const uint64_t W = mask.h.num_windows, nv = mask.h.num_vectors;
        std::vector<uint32_t> rp(W + 1), ci(nv);
        std::vector<float> vals(8 * nv);
        check(tcs_mebcrs_download(&mask.h, rp.data(), ci.data(), nullptr, nullptr));
        dv.down(vals.data(), vals.size() * 4);
        const uint64_t k = mask.h.k;
        const double tol = o.precision == TCS_FP16 ? kRealTolFp16 : kRealTolTf32;
        double max_diff = 0.0;
        bool ok = true;
        for (uint64_t r = 0; ok && r < csr.m.rows; ++r) {
            const uint64_t w = r / 8, base = rp[w], nvw = rp[w + 1] - base;
            for (uint64_t p = csr.m.row_ptr[r]; p < csr.m.row_ptr[r + 1]; ++p) {
                const uint32_t col = csr.m.col_idx[p];
                double dot = 0.0;
                for (uint64_t l = 0; l < n; ++l)
                    dot += static_cast<double>(A.data[r * n + l]) * static_cast<double>(Bt.data[col * n + l]);
                // sampled value at (r, col): decode_mebcrs drops zeros, so 0 reads as 0
                const uint64_t v = std::lower_bound(ci.begin() + base, ci.begin() + base + nvw, col) - ci.begin() - base;
                const uint64_t b = v / k, j = v % k, width = std::min<uint64_t>(k, nvw - b * k);
                const float got = vals[8 * (base + b * k) + (r % 8) * width + j];
                const double diff = std::abs(static_cast<double>(got != 0.0f ? got : 0.0f) - dot);
                max_diff = std::max(max_diff, diff);
                if (o.real ? diff > tol * std::max(1.0, std::abs(dot)) : diff != 0.0) {
                    ok = false;
                    break;
                }
            }
        }
        if (!ok) {
            err << "verification FAILED: max_abs_diff=" << max_diff << "\n";
            return kExitVerifyFailed;
        }
        out << "verify: ok, max_abs_diff=" << max_diff << "\n";
    }
    if (!o.output.empty()) {
        const tcs_status s = tcs_mebcrs_write(o.output.c_str(), &res.h, nullptr);
        if (s == TCS_ERR_IO) {
            err << "error: cannot open output '" << o.output << "'\n";
            return kExitInputError;
        }
        check(s);
    }
    res.h.values = nullptr;  // owned by dv
    return kExitOk;
}

// ---------------------------------------------------------------- stats
struct Record {
    uint64_t vh, n;
    tcs_precision p;
    tcs_cost c;
};
struct Report {
    std::string id;
    uint64_t rows, cols, nnz;
    std::vector<Record> recs;
};

// ref analyze_matrix (analysis.hpp:188-226): N outer, then v8/fp16, v8/tf32, v16/fp16, v16/tf32.
Report analyze(const std::string& id, const Csr& csr, const std::vector<uint64_t>& n_list, tcs_mapping mapping) {
    Report rep{id, csr.m.rows, csr.m.cols, csr.m.nnz, {}};
    Handle h[2][2];
    for (int vi = 0; vi < 2; ++vi)
        for (int pi = 0; pi < 2; ++pi) encode_any(csr, static_cast<tcs_precision>(pi), vi ? 16 : 8, h[vi][pi]);
    for (const uint64_t n : n_list)
        for (int vi = 0; vi < 2; ++vi)
            for (int pi = 0; pi < 2; ++pi) {
                Record r{vi ? 16u : 8u, n, static_cast<tcs_precision>(pi), {}};
                check(tcs_mebcrs_cost(&h[vi][pi].h, csr.m.nnz, static_cast<int64_t>(n), mapping, &r.c, nullptr));
                rep.recs.push_back(r);
            }
    return rep;
}

std::string json_escape(const std::string& s) {
    std::string o;
    for (const unsigned char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    o += buf;
                } else {
                    o += static_cast<char>(c);
                }
        }
    }
    return o;
}

// ref emit_report (analysis.hpp:233-266): CSV, or ordered JSON dumped with indent 2.
std::string emit_report(const std::vector<Report>& reps, const std::string& format) {
    std::ostringstream out;
    if (format == "csv") {
        out << "matrix_id,rows,cols,nnz,vector_height,precision,n_cols,mma_count,zero_fill,"
               "access_bytes,transactions,footprint_me,footprint_sr\n";
        for (const auto& rep : reps)
            for (const auto& r : rep.recs)
                out << rep.id << "," << rep.rows << "," << rep.cols << "," << rep.nnz << "," << r.vh << ","
                    << prec_name(r.p) << "," << r.n << "," << r.c.mma_count << "," << r.c.zero_fill << ","
                    << r.c.access_bytes << "," << r.c.transactions << "," << r.c.footprint_me << ","
                    << r.c.footprint_sr << "\n";
        return out.str();
    }
    if (reps.empty()) return "[]\n";
    out << "[\n";
    for (size_t i = 0; i < reps.size(); ++i) {
        const auto& rep = reps[i];
        out << "  {\n    \"matrix_id\": \"" << json_escape(rep.id) << "\",\n    \"rows\": " << rep.rows
            << ",\n    \"cols\": " << rep.cols << ",\n    \"nnz\": " << rep.nnz << ",\n    \"records\": ";
        if (rep.recs.empty()) {
            out << "[]\n";
        } else {
            out << "[\n";
            for (size_t j = 0; j < rep.recs.size(); ++j) {
                const auto& r = rep.recs[j];
                out << "      {\n        \"vector_height\": " << r.vh << ",\n        \"precision\": \""
                    << prec_name(r.p) << "\",\n        \"n_cols\": " << r.n << ",\n        \"mma_count\": "
                    << r.c.mma_count << ",\n        \"zero_fill\": " << r.c.zero_fill
                    << ",\n        \"nonzero_count\": " << rep.nnz << ",\n        \"access_bytes\": "
                    << r.c.access_bytes << ",\n        \"transactions\": " << r.c.transactions
                    << ",\n        \"footprint_me\": " << r.c.footprint_me << ",\n        \"footprint_sr\": "
                    << r.c.footprint_sr << "\n      }" << (j + 1 < rep.recs.size() ? ",\n" : "\n");
            }
            out << "    ]\n";
        }
        out << "  }" << (i + 1 < reps.size() ? ",\n" : "\n");
    }
    out << "]\n";
    return out.str();
}

// ref cli.hpp:286-302
int run_stats(const Opts& o, std::ostream& out, std::ostream& err) {
    const auto files = collect_inputs(o.input, o.dir, err);
    const std::vector<uint64_t> n_list = o.n_list.empty() ? std::vector<uint64_t>{128} : o.n_list;
    std::vector<Report> reps;
    size_t failed = 0;
    for (const auto& path : files) {
        try {
            Csr csr;
            load_matrix_market(path, csr);
            reps.push_back(analyze(matrix_id(path), csr, n_list, o.mapping));
        } catch (const InputError& e) {
            err << "skipping " << path << ": " << e.what << "\n";
            ++failed;
        }
    }
    write_text(o.output, emit_report(reps, o.format), out);
    if (reps.empty() || failed > 0) return kExitPartial;
    return kExitOk;
}

// ref cli.hpp:318-358
int run_bench(const Opts& o, std::ostream& out, std::ostream& err) {
    const auto files = collect_inputs(o.input, o.dir, err);
    const uint64_t n = o.n_list.empty() ? 128 : o.n_list.back();
    std::ostringstream csv;
    csv << "matrix_id,precision,n_cols,mma_swap8,mma_baseline16,mma_swap8_analytic,"
           "mma_baseline16_analytic,transactions_swap8,transaction_bytes_swap8,verified\n";
    size_t processed = 0;
    bool verify_failed = false;
    for (const auto& path : files) {
        Csr csr;
        try {
            load_matrix_market(path, csr);
        } catch (const InputError& e) {
            err << "skipping " << path << ": " << e.what << "\n";
            continue;
        }
        ++processed;
        const Dense dense = generate_dense(csr.m.cols, n, o.seed, false);
        const auto want = matmul_reference(csr, dense);
        for (const tcs_precision p : {TCS_FP16, TCS_TF32}) {
            Handle a8, a16;
            encode_any(csr, p, 8, a8);
            encode_any(csr, p, 16, a16);
            tcs_counters c8{}, c16{};
            const auto g8 = run_spmm_gpu(a8, dense, p, 8, o.mapping, c8);
            const auto g16 = run_spmm_gpu(a16, dense, p, 16, o.mapping, c16);
            tcs_cost k8{}, k16{};
            check(tcs_mebcrs_cost(&a8.h, csr.m.nnz, static_cast<int64_t>(n), o.mapping, &k8, nullptr));
            check(tcs_mebcrs_cost(&a16.h, csr.m.nnz, static_cast<int64_t>(n), o.mapping, &k16, nullptr));
            const bool ok = compare(g8, want, 0).exact && compare(g16, want, 0).exact;
            verify_failed = verify_failed || !ok;
            csv << matrix_id(path) << "," << prec_name(p) << "," << n << "," << c8.mma_invocations << ","
                << c16.mma_invocations << "," << k8.mma_count << "," << k16.mma_count << "," << c8.transactions << ","
                << c8.transaction_bytes << "," << (ok ? "yes" : "no") << "\n";
        }
    }
    write_text(o.output, csv.str(), out);
    if (verify_failed) return kExitVerifyFailed;
    if (processed == 0) return kExitPartial;
    return kExitOk;
}

int usage(std::ostream& err) {
    err << "usage: tcsparse-b200 {convert|spmm|sddmm|stats|bench} [options]  (see the header of this tool)\n";
    return kExitInputError;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage(std::cerr);
    const std::string cmd = argv[1];
    Opts o;
    std::string prec = "fp16", mapping = "coalesced";
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i], val;
        const auto eq = a.find('=');
        bool has_val = false;
        if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = a.substr(eq + 1);
            a = a.substr(0, eq);
            has_val = true;
        }
        auto next = [&]() -> std::string {
            if (has_val) return val;
            if (i + 1 >= argc) throw std::runtime_error(a + " needs a value");
            return argv[++i];
        };
        try {
            if (a == "--input") o.input = next();
            else if (a == "--output") o.output = next();
            else if (a == "--dir") o.dir = next();
            else if (a == "--precision") prec = next();
            else if (a == "--mapping") mapping = next();
            else if (a == "--format") o.format = next();
            else if (a == "--vector") o.vector = std::stoull(next());
            else if (a == "--seed") o.seed = std::stoull(next());
            else if (a == "--n") {
                o.n_list.push_back(std::stoull(next()));
                while (!has_val && i + 1 < argc && argv[i + 1][0] != '-') o.n_list.push_back(std::stoull(argv[++i]));
            } else if (a == "--verify") o.verify = true;
            else if (a == "--real") o.real = true;
            else {
                std::cerr << "error: unknown option " << a << "\n";
                return usage(std::cerr);
            }
        } catch (const std::exception& e) {
            std::cerr << "error: " << e.what() << "\n";
            return usage(std::cerr);
        }
    }
    if (prec != "fp16" && prec != "tf32") return usage(std::cerr);
    if (mapping != "direct" && mapping != "coalesced") return usage(std::cerr);
    if (o.format != "csv" && o.format != "json") return usage(std::cerr);
    if (o.vector != 8 && o.vector != 16) return usage(std::cerr);
    o.precision = prec == "fp16" ? TCS_FP16 : TCS_TF32;
    o.mapping = mapping == "direct" ? TCS_MAP_DIRECT : TCS_MAP_COALESCED;
    try {
        if (cmd == "convert" || cmd == "spmm" || cmd == "sddmm") {
            if (o.input.empty()) {
                std::cerr << "error: --input is required\n";
                return kExitInputError;
            }
            if (cmd == "convert") return run_convert(o, std::cout, std::cerr);
            if (cmd == "spmm") return run_spmm(o, std::cout, std::cerr);
            return run_sddmm(o, std::cout, std::cerr);
        }
        if (cmd == "stats" || cmd == "bench") {
            if (o.input.empty() && o.dir.empty()) {
                std::cerr << "error: " << cmd << " needs --input or --dir\n";
                return kExitInputError;
            }
            return cmd == "stats" ? run_stats(o, std::cout, std::cerr) : run_bench(o, std::cout, std::cerr);
        }
    } catch (const DeviceError& e) {
        std::cerr << "error: device: " << e.what << "\n";
        return kExitDevice;
    } catch (const InputError& e) {
        std::cerr << "error: " << e.what << "\n";
        return kExitInputError;
    }
    return usage(std::cerr);
}
