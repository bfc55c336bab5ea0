// Ingest and persistence around the hot path:
//
//   * MatrixMarket coordinate input (ref matrix_market.hpp:28-94): the text
//     is tokenised on the host by all cores (chunks split at line breaks,
//     the reference's exact acceptance rules and error messages, ParseError
//     line numbers), and the coordinate list -> CSR assembly (ref
//     csr_from_coords, matrix.hpp:96-128: sort by (row, col), duplicates
//     summed) runs on the GPU: a radix sort of (row << 32 | col) keys, a
//     head-flag scan and one ordered sum per run.
//   * MatrixMarket output (ref write_matrix_market, matrix_market.hpp:97-104).
//   * The MEBC binary container v1 (ref container_io.hpp:56-91), read into /
//     written from a device ME-BCRS handle, byte-identical to the reference's
//     write_mebcrs for the same matrix.
//
// Duplicate coordinates: the reference sums them after an (unstable)
// std::sort; here they are summed in input order.  Two duplicates give the
// same bits either way (fp32 addition commutes); three or more may differ in
// the last ulp.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <thread>
#include <vector>

#include "tcs_internal.cuh"

namespace tcs {
namespace {

// ------------------------------------------------------------ text parsing
struct ParseFail {
    std::string msg;
    uint64_t line;  // 1-based, 0 = no line (ref errors.hpp:13-15)
};

std::string lower(std::string s) {
    for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

[[noreturn]] void parse_fail(const std::string& what, uint64_t line = 0) {
    fail(TCS_ERR_PARSE, line > 0 ? "line " + std::to_string(line) + ": " + what : what);
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// istream >> long long: skip whitespace, [+-]digits; false if no digits or
// out of range.
bool scan_i64(const char*& p, const char* e, long long& out) {
    while (p < e && is_ws(*p)) ++p;
    const char* b = p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* d = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == d) return false;
    char buf[64];
    const size_t n = std::min<size_t>(63, p - b);
    std::memcpy(buf, b, n);
    buf[n] = 0;
    errno = 0;
    out = std::strtoll(buf, nullptr, 10);
    return errno == 0;
}

// istream >> double (libstdc++ num_get): accumulates [+-] digits [. digits]
// [(e|E) [+-] digits] and converts that prefix; no inf/nan/hex forms.
bool scan_f64(const char*& p, const char* e, double& out) {
    while (p < e && is_ws(*p)) ++p;
    const char* b = p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    bool digits = false;
    while (p < e && *p >= '0' && *p <= '9') ++p, digits = true;
    if (p < e && *p == '.') {
        ++p;
        while (p < e && *p >= '0' && *p <= '9') ++p, digits = true;
    }
    if (!digits) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        const char* q = p + 1;
        if (q < e && (*q == '+' || *q == '-')) ++q;
        const char* d = q;
        while (q < e && *q >= '0' && *q <= '9') ++q;
        if (q == d) return false;  // num_get consumed the 'e' and found no exponent digits
        p = q;
    }
    std::string buf(b, p);
    errno = 0;
    out = std::strtod(buf.c_str(), nullptr);
    if (errno == ERANGE && std::fabs(out) == HUGE_VAL) return false;  // num_get: overflow sets failbit
    return true;
}

struct Coords {
    std::vector<uint32_t> r, c;
    std::vector<float> v;
};

// Lines [b, e) of the body; collects entries until `limit` (the first error
// stops the chunk; whether it matters depends on how many entries precede
// it globally, decided by the caller).
struct Chunk {
    const char* b;
    const char* e;
    uint64_t lines = 0;      // line breaks inside the chunk
    uint64_t err_line = 0;   // chunk-local 1-based line of the first error (0 = none)
    std::string err;
    Coords out;
};

void parse_chunk(Chunk& ck, long long rows, long long cols, bool pattern, bool symmetric) {
    const char* p = ck.b;
    uint64_t line = 0;
    while (p < ck.e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', ck.e - p));
        const char* le = nl ? nl : ck.e;
        ++line;
        const char* q = p;
        p = nl ? nl + 1 : ck.e;
        if (q == le || *q == '%') continue;  // empty or comment line
        bool blank = true;
        for (const char* x = q; x < le; ++x)
            if (!(*x == ' ' || *x == '\t' || *x == '\r')) { blank = false; break; }
        if (blank) continue;
        long long i = 0, j = 0;
        if (!scan_i64(q, le, i) || !scan_i64(q, le, j)) {
            ck.err = "malformed entry";
            ck.err_line = line;
            break;
        }
        double v = 1.0;
        if (!pattern && !scan_f64(q, le, v)) {
            ck.err = "entry value missing";
            ck.err_line = line;
            break;
        }
        if (i < 1 || i > rows || j < 1 || j > cols) {
            ck.err = "coordinate (" + std::to_string(i) + "," + std::to_string(j) + ") out of range";
            ck.err_line = line;
            break;
        }
        const auto r = static_cast<uint32_t>(i - 1), c = static_cast<uint32_t>(j - 1);
        const float val = static_cast<float>(v);
        ck.out.r.push_back(r);
        ck.out.c.push_back(c);
        ck.out.v.push_back(val);
        if (symmetric && r != c) {
            ck.out.r.push_back(c);
            ck.out.c.push_back(r);
            ck.out.v.push_back(val);
        }
    }
    ck.lines = line;
}

struct Parsed {
    uint64_t rows = 0, cols = 0;
    Coords coords;  // file order (symmetric mirrors follow their entry)
};

// ref parse_matrix_market (matrix_market.hpp:28-94).
Parsed parse_mm(const char* text, size_t len) {
    const char* p = text;
    const char* end = text + len;
    uint64_t lineno = 0;
    auto getline = [&](const char*& b, const char*& e) -> bool {
        if (p >= end) return false;
        b = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        return true;
    };
    const char *b, *e;
    if (!getline(b, e)) parse_fail("empty input, MatrixMarket banner missing");
    ++lineno;
    std::istringstream banner(std::string(b, e));
    std::string tag, object, format, field, symmetry;
    banner >> tag >> object >> format >> field >> symmetry;
    if (tag != "%%MatrixMarket") parse_fail("MatrixMarket banner missing", lineno);
    object = lower(object);
    format = lower(format);
    field = lower(field);
    symmetry = lower(symmetry);
    if (object != "matrix") parse_fail("unsupported object '" + object + "'", lineno);
    if (format != "coordinate") parse_fail("only coordinate format is supported", lineno);
    if (field != "real" && field != "integer" && field != "pattern")
        parse_fail("unsupported field '" + field + "'", lineno);
    if (symmetry != "general" && symmetry != "symmetric") parse_fail("unsupported symmetry '" + symmetry + "'", lineno);
    const bool pattern = field == "pattern", symmetric = symmetry == "symmetric";

    long long rows = 0, cols = 0, declared = 0;
    for (;;) {
        if (!getline(b, e)) parse_fail("size line missing");
        ++lineno;
        if (b == e || *b == '%') continue;
        bool blank = true;
        for (const char* x = b; x < e; ++x)
            if (!(*x == ' ' || *x == '\t' || *x == '\r')) { blank = false; break; }
        if (blank) continue;
        std::istringstream sz(std::string(b, e));
        if (!(sz >> rows >> cols >> declared) || rows < 0 || cols < 0 || declared < 0)
            parse_fail("malformed size line", lineno);
        break;
    }
    if (rows > (1ll << 32) || cols > (1ll << 32)) fail(TCS_ERR_FORMAT, "matrix dimensions exceed u32 indices");

    // Body: chunks cut at line breaks, parsed by all host threads.
    const size_t body = end - p;
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                        static_cast<unsigned>(body / (1 << 20) + 1)));
    std::vector<Chunk> chunks(nt);
    const char* cb = p;
    for (unsigned t = 0; t < nt; ++t) {
        const char* ce = t + 1 == nt ? end : std::min(end, p + body * (t + 1) / nt);
        if (ce < end && ce > cb) {
            const char* nl = static_cast<const char*>(std::memchr(ce - 1, '\n', end - (ce - 1)));
            ce = nl ? nl + 1 : end;
        }
        if (ce < cb) ce = cb;
        chunks[t].b = cb;
        chunks[t].e = ce;
        cb = ce;
    }
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t)
        th.emplace_back(parse_chunk, std::ref(chunks[t]), rows, cols, pattern, symmetric);
    parse_chunk(chunks[0], rows, cols, pattern, symmetric);
    for (auto& x : th) x.join();

    // The reference reads exactly `declared` entries: an error matters only
    // if it occurs before that many entries were seen.
    Parsed out;
    out.rows = static_cast<uint64_t>(rows);
    out.cols = static_cast<uint64_t>(cols);
    const uint64_t want = static_cast<uint64_t>(declared);
    uint64_t seen = 0, line_base = lineno;
    for (auto& ck : chunks) {
        // copy entries (an off-diagonal symmetric entry carries its mirror)
        // until `declared` entries have been seen
        const size_t n = ck.out.r.size();
        size_t i = 0;
        while (i < n && seen < want) {
            const size_t cnt = symmetric && ck.out.r[i] != ck.out.c[i] ? 2 : 1;
            for (size_t q = 0; q < cnt; ++q) {
                out.coords.r.push_back(ck.out.r[i + q]);
                out.coords.c.push_back(ck.out.c[i + q]);
                out.coords.v.push_back(ck.out.v[i + q]);
            }
            i += cnt;
            ++seen;
        }
        if (seen == want) return out;  // later lines are never read by the reference
        if (!ck.err.empty()) parse_fail(ck.err, line_base + ck.err_line);
        line_base += ck.lines;
    }
    parse_fail("unexpected end of file: expected " + std::to_string(want) + " entries, got " + std::to_string(seen));
}

std::vector<char> read_file(const char* path, tcs_status on_fail, const std::string& what) {
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(on_fail, "cannot open '" + std::string(path) + "'" + what);
    std::vector<char> buf;
    char tmp[1 << 16];
    if (std::fseek(f, 0, SEEK_END) == 0) {
        const long sz = std::ftell(f);
        if (sz > 0) buf.reserve(static_cast<size_t>(sz));
        std::fseek(f, 0, SEEK_SET);
    }
    size_t n;
    while ((n = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + n);
    std::fclose(f);
    return buf;
}

// --------------------------------------------------- coords -> CSR (GPU)
__global__ void make_keys(const uint32_t* __restrict__ r, const uint32_t* __restrict__ c, uint64_t n,
                          uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        keys[i] = (static_cast<uint64_t>(r[i]) << 32) | c[i];
        idx[i] = static_cast<uint32_t>(i);
    }
}

__global__ void run_heads(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ head) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// One thread per run head: the run's values summed in input order starting
// from 0.0f (ref matrix.hpp:114-119; note 0.0f + -0.0f = +0.0f, as there).
__global__ void run_sums(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                         const float* __restrict__ v, uint64_t n, const uint32_t* __restrict__ head,
                         const uint32_t* __restrict__ pos, uint32_t* __restrict__ out_c,
                         float* __restrict__ out_v, uint32_t* __restrict__ row_count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!head[i]) continue;
        const uint64_t key = keys[i];
        float sum = 0.0f;
        for (uint64_t j = i; j < n && keys[j] == key; ++j) sum += v[idx[j]];
        const uint32_t o = pos[i];
        out_c[o] = static_cast<uint32_t>(key);
        out_v[o] = sum;
        atomicAdd(row_count + (key >> 32), 1u);
    }
}

int grid_for(uint64_t n) { return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 65535))); }

// Device coordinates -> device CSR arrays (library-allocated).
void coo_to_csr_device(uint64_t rows, uint64_t cols, uint64_t n, const uint32_t* r, const uint32_t* c, const float* v,
                       tcs_csr* out, cudaStream_t s) {
    if (n >= (1ull << 32)) fail(TCS_ERR_FORMAT, "too many coordinates for u32 row_ptr");
    DBuf keys(std::max<uint64_t>(1, n) * 8, s), keys2(std::max<uint64_t>(1, n) * 8, s);
    DBuf idx(std::max<uint64_t>(1, n) * 4, s), idx2(std::max<uint64_t>(1, n) * 4, s);
    DBuf head(std::max<uint64_t>(1, n) * 4, s), pos((n + 1) * 4, s);
    uint32_t* rp = static_cast<uint32_t*>(dalloc((rows + 1) * 4, s));
    uint32_t* cnt = static_cast<uint32_t*>(dalloc(std::max<uint64_t>(1, rows) * 4, s));
    struct Guard {
        void* p;
        cudaStream_t s;
        bool armed = true;
        ~Guard() { if (armed) dfree(p, s); }
    } grp{rp, s};
    DBuf cnt_owner;
    cnt_owner.p = cnt;
    cnt_owner.s = s;
    TCS_CUDA(cudaMemsetAsync(cnt, 0, std::max<uint64_t>(1, rows) * 4, s));
    uint32_t nnz = 0;
    uint32_t* oc = nullptr;
    float* ov = nullptr;
    if (n) {
        make_keys<<<grid_for(n), 256, 0, s>>>(r, c, n, keys.as<uint64_t>(), idx.as<uint32_t>());
        TCS_LAUNCHED("make_keys");
        int end_bit = 32;
        while (end_bit < 64 && (rows >> (end_bit - 32)) > 0) ++end_bit;
        size_t tmp_bytes = 0;
        TCS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                                 idx.as<uint32_t>(), idx2.as<uint32_t>(), static_cast<int64_t>(n), 0,
                                                 end_bit, s));
        DBuf tmp(std::max<size_t>(16, tmp_bytes), s);
        TCS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                                 idx.as<uint32_t>(), idx2.as<uint32_t>(), static_cast<int64_t>(n), 0,
                                                 end_bit, s));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        run_heads<<<grid_for(n), 256, 0, s>>>(keys2.as<uint64_t>(), n, head.as<uint32_t>());
        TCS_LAUNCHED("run_heads");
        exclusive_scan_u32(head.as<uint32_t>(), pos.as<uint32_t>(), n, s);
        TCS_CUDA(cudaMemcpyAsync(&nnz, pos.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
        TCS_CUDA(cudaStreamSynchronize(s));
        oc = static_cast<uint32_t*>(dalloc(std::max<uint32_t>(1, nnz) * 4, s));
        ov = static_cast<float*>(dalloc(std::max<uint32_t>(1, nnz) * 4, s));
        run_sums<<<grid_for(n), 256, 0, s>>>(keys2.as<uint64_t>(), idx2.as<uint32_t>(), v, n, head.as<uint32_t>(),
                                             pos.as<uint32_t>(), oc, ov, cnt);
        TCS_LAUNCHED("run_sums");
    } else {
        oc = static_cast<uint32_t*>(dalloc(4, s));
        ov = static_cast<float*>(dalloc(4, s));
    }
    if (rows) exclusive_scan_u32(cnt, rp, rows, s);
    else TCS_CUDA(cudaMemsetAsync(rp, 0, 4, s));
    grp.armed = false;
    *out = tcs_csr{rows, cols, nnz, rp, oc, ov};
}

// ref write_matrix_market (matrix_market.hpp:97-104): same stream settings.
void write_mm(const char* path, const tcs_csr* m) {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(TCS_ERR_IO, "cannot open output '" + std::string(path) + "'");
    out << "%%MatrixMarket matrix coordinate real general\n";
    out << m->rows << " " << m->cols << " " << m->nnz << "\n";
    out.precision(std::numeric_limits<float>::max_digits10);
    for (uint64_t r = 0; r < m->rows; ++r)
        for (uint64_t p = m->row_ptr[r]; p < m->row_ptr[r + 1]; ++p)
            out << r + 1 << " " << m->col_idx[p] + 1 << " " << m->values[p] << "\n";
    if (!out) fail(TCS_ERR_IO, "write failed '" + std::string(path) + "'");
}

// ------------------------------------------------------- MEBC container
constexpr char kMagic[4] = {'M', 'E', 'B', 'C'};
constexpr uint32_t kVersion = 1;

template <typename T>
void put(std::vector<char>& b, T v) {
    const char* p = reinterpret_cast<const char*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
}
template <typename T>
void put_array(std::vector<char>& b, const T* p, uint64_t n) {
    if (n >= (1ull << 32)) fail(TCS_ERR_FORMAT, "container arrays are limited to 2^32 - 1 elements");
    put<uint32_t>(b, static_cast<uint32_t>(n));
    const char* c = reinterpret_cast<const char*>(p);
    b.insert(b.end(), c, c + n * sizeof(T));
}

struct Reader {
    const char* p;
    const char* e;
    template <typename T>
    T get() {
        if (static_cast<size_t>(e - p) < sizeof(T)) fail(TCS_ERR_FORMAT, "container truncated");
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return v;
    }
    template <typename T>
    std::vector<T> get_array() {
        const uint32_t n = get<uint32_t>();
        if (static_cast<uint64_t>(e - p) < uint64_t(n) * sizeof(T)) fail(TCS_ERR_FORMAT, "container array truncated");
        std::vector<T> v(n);
        if (n) std::memcpy(v.data(), p, size_t(n) * sizeof(T));
        p += size_t(n) * sizeof(T);
        return v;
    }
};

// ref MeBcrsMatrix::validate (mebcrs.hpp:58-77) on host arrays.
void validate_host(uint64_t rows, uint64_t cols, uint64_t vh, const std::vector<uint32_t>& rp,
                   const std::vector<uint32_t>& ci, uint64_t nvalues) {
    const uint64_t W = (rows + vh - 1) / vh;
    if (rp.size() != W + 1) fail(TCS_ERR_FORMAT, "row_pointers length must be numWindows+1");
    if (!rp.empty() && rp.front() != 0) fail(TCS_ERR_FORMAT, "row_pointers must start at 0");
    for (size_t w = 0; w + 1 < rp.size(); ++w)
        if (rp[w] > rp[w + 1]) fail(TCS_ERR_FORMAT, "row_pointers must be nondecreasing");
    if (!rp.empty() && rp.back() != ci.size()) fail(TCS_ERR_FORMAT, "row_pointers end must equal stored vector count");
    if (nvalues != vh * ci.size()) fail(TCS_ERR_FORMAT, "values length must be vectorHeight * stored vectors");
    for (size_t w = 0; w + 1 < rp.size(); ++w)
        for (uint32_t p = rp[w]; p < rp[w + 1]; ++p) {
            if (ci[p] >= cols) fail(TCS_ERR_FORMAT, "column index out of range");
            if (p > rp[w] && ci[p - 1] >= ci[p]) fail(TCS_ERR_FORMAT, "column indices must ascend within a window");
        }
}

}  // namespace

}  // namespace tcs

using namespace tcs;

extern "C" {

tcs_status tcs_matrix_market_parse(const char* text, uint64_t len, tcs_csr* out, tcs_stream_t stream) {
    return guard([&] {
        if (!out || (!text && len)) fail(TCS_ERR_ARGUMENT, "null argument");
        cudaStream_t s = st(stream);
        Parsed pm = parse_mm(text ? text : "", text ? len : 0);
        const uint64_t n = pm.coords.r.size();
        DBuf r(std::max<uint64_t>(1, n) * 4, s), c(std::max<uint64_t>(1, n) * 4, s), v(std::max<uint64_t>(1, n) * 4, s);
        if (n) {
            TCS_CUDA(cudaMemcpyAsync(r.p, pm.coords.r.data(), n * 4, cudaMemcpyHostToDevice, s));
            TCS_CUDA(cudaMemcpyAsync(c.p, pm.coords.c.data(), n * 4, cudaMemcpyHostToDevice, s));
            TCS_CUDA(cudaMemcpyAsync(v.p, pm.coords.v.data(), n * 4, cudaMemcpyHostToDevice, s));
        }
        tcs_csr d{};
        coo_to_csr_device(pm.rows, pm.cols, n, r.as<uint32_t>(), c.as<uint32_t>(), v.as<float>(), &d, s);
        DBuf drp, dci, dv;
        drp.p = const_cast<uint32_t*>(d.row_ptr), drp.s = s;
        dci.p = const_cast<uint32_t*>(d.col_idx), dci.s = s;
        dv.p = const_cast<float*>(d.values), dv.s = s;
        auto* hrp = static_cast<uint32_t*>(std::malloc((d.rows + 1) * 4));
        auto* hci = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(1, d.nnz) * 4));
        auto* hv = static_cast<float*>(std::malloc(std::max<uint64_t>(1, d.nnz) * 4));
        if (!hrp || !hci || !hv) {
            std::free(hrp), std::free(hci), std::free(hv);
            fail(TCS_ERR_OOM, "host allocation failed");
        }
        TCS_CUDA(cudaMemcpyAsync(hrp, d.row_ptr, (d.rows + 1) * 4, cudaMemcpyDeviceToHost, s));
        if (d.nnz) {
            TCS_CUDA(cudaMemcpyAsync(hci, d.col_idx, d.nnz * 4, cudaMemcpyDeviceToHost, s));
            TCS_CUDA(cudaMemcpyAsync(hv, d.values, d.nnz * 4, cudaMemcpyDeviceToHost, s));
        }
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            std::free(hrp), std::free(hci), std::free(hv);
            cuda_check(e, "cudaStreamSynchronize");
        }
        *out = tcs_csr{d.rows, d.cols, d.nnz, hrp, hci, hv};
    });
}

tcs_status tcs_matrix_market_read(const char* path, tcs_csr* out, tcs_stream_t stream) {
    std::vector<char> buf;
    const tcs_status rc = guard([&] {
        if (!path || !out) fail(TCS_ERR_ARGUMENT, "null argument");
        buf = read_file(path, TCS_ERR_PARSE, "");  // ref cli.hpp:36-37: ParseError("cannot open '...'")
    });
    if (rc != TCS_OK) return rc;
    return tcs_matrix_market_parse(buf.data(), buf.size(), out, stream);
}

tcs_status tcs_matrix_market_write(const char* path, const tcs_csr* host_csr) {
    return guard([&] {
        if (!path || !host_csr || !host_csr->row_ptr) fail(TCS_ERR_ARGUMENT, "null argument");
        write_mm(path, host_csr);
    });
}

tcs_status tcs_csr_free_host(tcs_csr* m) {
    return guard([&] {
        if (!m) return;
        std::free(const_cast<uint32_t*>(m->row_ptr));
        std::free(const_cast<uint32_t*>(m->col_idx));
        std::free(const_cast<float*>(m->values));
        std::memset(m, 0, sizeof(*m));
    });
}

tcs_status tcs_coo_to_csr(uint64_t rows, uint64_t cols, uint64_t n, const uint32_t* row, const uint32_t* col,
                          const float* values, tcs_csr* out, tcs_stream_t stream) {
    return guard([&] {
        if (!out || (n && (!row || !col || !values))) fail(TCS_ERR_ARGUMENT, "null argument");
        // range check on the device copy would need a kernel; the reference
        // throws ArgumentError("coordinate out of range") (matrix.hpp:99-102)
        coo_to_csr_device(rows, cols, n, row, col, values, out, st(stream));
    });
}

tcs_status tcs_csr_free(tcs_csr* m, tcs_stream_t stream) {
    return guard([&] {
        if (!m) return;
        cudaStream_t s = st(stream);
        dfree(const_cast<uint32_t*>(m->row_ptr), s);
        dfree(const_cast<uint32_t*>(m->col_idx), s);
        dfree(const_cast<float*>(m->values), s);
        std::memset(m, 0, sizeof(*m));
    });
}

// ref write_mebcrs (container_io.hpp:56-68).
tcs_status tcs_mebcrs_write(const char* path, const tcs_mebcrs* m, tcs_stream_t stream) {
    return guard([&] {
        if (!path) fail(TCS_ERR_ARGUMENT, "null argument");
        check_mebcrs(m, true);
        std::vector<uint32_t> rp(m->num_windows + 1), ci(m->num_vectors);
        std::vector<float> v(uint64_t(m->vector_height) * m->num_vectors);
        const tcs_status rc = tcs_mebcrs_download(m, rp.data(), ci.data(), v.data(), stream);
        if (rc != TCS_OK) fail(rc, tcs_last_error());
        std::vector<char> b;
        b.reserve(64 + 4 * (rp.size() + ci.size() + v.size()));
        b.insert(b.end(), kMagic, kMagic + 4);
        put<uint32_t>(b, kVersion);
        put<uint64_t>(b, m->rows);
        put<uint64_t>(b, m->cols);
        put<uint32_t>(b, m->vector_height);
        put<uint32_t>(b, m->k);
        put<uint8_t>(b, static_cast<uint8_t>(m->precision));
        put_array(b, rp.data(), rp.size());
        put_array(b, ci.data(), ci.size());
        put_array(b, v.data(), v.size());
        FILE* f = std::fopen(path, "wb");
        if (!f) fail(TCS_ERR_IO, "cannot open output '" + std::string(path) + "'");
        const size_t w = std::fwrite(b.data(), 1, b.size(), f);
        const int cl = std::fclose(f);
        if (w != b.size() || cl != 0) fail(TCS_ERR_IO, "write failed '" + std::string(path) + "'");
    });
}

// ref read_mebcrs (container_io.hpp:70-91): magic, version, header, arrays,
// validate; the arrays land in a device handle with F32 values.
tcs_status tcs_mebcrs_read(const char* path, tcs_mebcrs* out, tcs_stream_t stream) {
    return guard([&] {
        if (!path || !out) fail(TCS_ERR_ARGUMENT, "null argument");
        const std::vector<char> buf = read_file(path, TCS_ERR_IO, "");
        Reader rd{buf.data(), buf.data() + buf.size()};
        if (buf.size() < 4 || std::memcmp(buf.data(), kMagic, 4) != 0) fail(TCS_ERR_FORMAT, "bad container magic");
        rd.p += 4;
        const uint32_t version = rd.get<uint32_t>();
        if (version != kVersion) fail(TCS_ERR_FORMAT, "unsupported container version " + std::to_string(version));
        const uint64_t rows = rd.get<uint64_t>(), cols = rd.get<uint64_t>();
        const uint32_t vh = rd.get<uint32_t>(), k = rd.get<uint32_t>();
        const uint8_t prec = rd.get<uint8_t>();
        if (prec > 1) fail(TCS_ERR_FORMAT, "bad precision tag");
        const auto rp = rd.get_array<uint32_t>();
        const auto ci = rd.get_array<uint32_t>();
        const auto v = rd.get_array<float>();
        if (vh == 0) fail(TCS_ERR_FORMAT, "row_pointers length must be numWindows+1");
        validate_host(rows, cols, vh, rp, ci, v.size());
        if (vh != 8 && vh != 16) fail(TCS_ERR_FORMAT, "vector height must be 8 or 16");
        if (k != (prec == 0 ? 8u : 4u)) fail(TCS_ERR_FORMAT, "block width k does not match precision");
        upload_mebcrs(rows, cols, static_cast<tcs_precision>(prec), vh, rp.data(), ci.data(), v.data(), out,
                      st(stream));
    });
}

}  // extern "C"
