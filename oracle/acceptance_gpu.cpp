// ============================================================================
// TEST INFRASTRUCTURE ONLY -- replay of the reference's acceptance criteria
// 2, 3, 6 and 7 (tests/acceptance.cpp:89-131, 178-273) with the GPU
// drop-in (tcsparse::gpu::*, include/tcsparse/gpu.hpp) substituted for the
// reference functions, same mt19937 seeds and generators.  Every GPU result
// must equal BOTH the reference function's result and the reference tests'
// independent oracle (tests/oracles.hpp).  This proves the drop-in claim:
// reference-API code switches by changing the namespace qualifier.
//
// Built by oracle/Makefile where /root/reference exists (it includes the
// reference headers and tests/oracles.hpp where they lie) into
// oracle/_ref/acceptance_gpu, linked against libtcsparse_b200.so; run on the
// GPU box by tests/test_gpu_dropin.py.
// ============================================================================
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "oracles.hpp"
#include "tcsparse/gpu.hpp"
#include "tcsparse/tcsparse.hpp"

using namespace tcsparse;

namespace {

int failures = 0;

void report(int idx, const char* name, bool ok) {
    std::printf("[%s] criterion %d (gpu drop-in): %s\n", ok ? "PASS" : "FAIL", idx, name);
    if (!ok) ++failures;
}

bool same_me(const MeBcrsMatrix& a, const MeBcrsMatrix& b) {
    return a.rows == b.rows && a.cols == b.cols && a.k == b.k && a.precision == b.precision &&
           a.row_pointers == b.row_pointers && a.column_indices == b.column_indices && a.values == b.values;
}

bool criterion2() {  // tests/acceptance.cpp:89-110
    std::mt19937 gen(7);
    for (int i = 0; i < 200; ++i) {
        const std::size_t rows = (i % 25 == 0) ? 512 : 16 + gen() % 30 * 8;
        const std::size_t cols = (i % 25 == 12) ? 512 : 16 + gen() % 30 * 8;
        const double density = 0.005 + (gen() % 1000) / 1000.0 * 0.295;
        const CsrMatrix m = generate_random_sparse(rows, cols, density, 1000 + i);
        const DenseMatrix dense = generate_random_dense(cols, 32, 2000 + i);
        const DenseMatrix want = oracles::dense_product(to_dense(m), dense);
        for (Precision p : {Precision::fp16, Precision::tf32}) {
            const MeBcrsMatrix me = gpu::encode_mebcrs(m, p);
            if (!same_me(me, encode_mebcrs(m, p))) return false;
            for (ThreadMapping mode : {ThreadMapping::direct, ThreadMapping::coalesced}) {
                const SpmmResult r = gpu::spmm(me, dense, {p, 8, mode});
                if (r.output != want) return false;
                // every counter in the reference's units (ref spmm.hpp:144-151)
                const KernelCounters rc = spmm(me, dense, {p, 8, mode}).counters;
                if (r.counters.mma_invocations != rc.mma_invocations || r.counters.transactions != rc.transactions ||
                    r.counters.transaction_bytes != rc.transaction_bytes || r.counters.useful_bytes != rc.useful_bytes)
                    return false;
            }
            // tests/acceptance.cpp:105 -- the 16x1 baseline on the CSR
            const SpmmResult b16 = gpu::spmm_baseline16(m, dense, {p, 16, ThreadMapping::coalesced});
            if (b16.output != want) return false;
            const KernelCounters rb = spmm_baseline16(m, dense, {p, 16, ThreadMapping::coalesced}).counters;
            if (b16.counters.mma_invocations != rb.mma_invocations || b16.counters.transactions != rb.transactions ||
                b16.counters.transaction_bytes != rb.transaction_bytes || b16.counters.useful_bytes != rb.useful_bytes)
                return false;
        }
    }
    return true;
}

bool criterion3() {  // tests/acceptance.cpp:114-131
    std::vector<Coord> coords;
    for (std::uint32_t i = 0; i < 16; ++i) coords.push_back({i, i, 1.0f});
    const CsrMatrix m = csr_from_coords(16, 16, coords);
    const DenseMatrix dense = generate_random_dense(16, 16, 42);
    const SpmmResult r = gpu::spmm(gpu::encode_mebcrs(m, Precision::fp16), dense,
                                   {Precision::fp16, 8, ThreadMapping::coalesced});
    return r.counters.mma_invocations == 2 && r.output == dense;
}

bool criterion6() {  // tests/acceptance.cpp:178-236
    std::mt19937 gen(11);
    for (int i = 0; i < 100; ++i) {
        const std::size_t m_rows = 8 + gen() % 7 * 8;
        const std::size_t n_cols = 8 + gen() % 7 * 8;
        const std::size_t inner = 4 + gen() % 29;
        const double density = 0.05 + (gen() % 100) / 400.0;
        const CsrMatrix mask = generate_random_sparse(m_rows, n_cols, density, 3000 + i);
        const DenseMatrix a = generate_random_dense(m_rows, inner, 4000 + i);
        const DenseMatrix b_t = generate_random_dense(n_cols, inner, 5000 + i);
        const Precision p = i % 2 ? Precision::fp16 : Precision::tf32;
        const SddmmOperands ops{gpu::encode_mebcrs(mask, p), a, b_t};
        const SddmmResult g = gpu::sddmm(ops, {p, 8, ThreadMapping::coalesced});
        const SddmmResult r = sddmm(ops, {p, 8, ThreadMapping::coalesced});
        if (!same_me(g.output, r.output)) return false;
        if (g.counters.mma_invocations != r.counters.mma_invocations) return false;
        const DenseMatrix d = generate_random_dense(n_cols, 16, 6000 + i);
        const SpmmResult chained = gpu::spmm(g.output, d, {p, 8, ThreadMapping::coalesced});
        if (chained.output != spmm(r.output, d, {p, 8, ThreadMapping::coalesced}).output) return false;
    }
    return true;
}

bool criterion7() {  // tests/acceptance.cpp:240-273 (its value draws; reference + oracle compared)
    std::mt19937 gen(13);
    for (int i = 0; i < 20; ++i) {
        std::vector<Coord> coords;
        const std::size_t windows = 2 + gen() % 4;
        for (std::size_t w = 0; w < windows; ++w) {
            const std::size_t count = 1 + 8 * (gen() % 3);
            for (std::size_t c = 0; c < count; ++c) {
                const auto val = static_cast<float>(1 + gen() % 4) * (gen() % 2 ? 1.0f : -1.0f);
                coords.push_back({static_cast<std::uint32_t>(8 * w + c % 8), static_cast<std::uint32_t>(c), val});
            }
        }
        const CsrMatrix m = csr_from_coords(8 * windows, 24, coords);
        const DenseMatrix dense = generate_random_dense(24, 24, 7000 + i);
        const DenseMatrix want = oracles::dense_product(to_dense(m), dense);
        for (Precision p : {Precision::fp16, Precision::tf32}) {
            const MeBcrsMatrix me = gpu::encode_mebcrs(m, p);
            if (!same_me(me, encode_mebcrs(m, p))) return false;
            const auto me_out = gpu::spmm(me, dense, {p, 8, ThreadMapping::coalesced});
            if (me_out.output != want) return false;
            // padded baseline format (tests/acceptance.cpp:264-267)
            const SrBcrsMatrix sr = gpu::encode_srbcrs(m, p);
            const SrBcrsMatrix sr_ref = encode_srbcrs(m, p);
            if (sr.row_pointer_pairs != sr_ref.row_pointer_pairs || sr.column_indices != sr_ref.column_indices ||
                sr.values != sr_ref.values)
                return false;
            if (gpu::decode_srbcrs(sr) != decode_srbcrs(sr_ref)) return false;
            const auto sr_out = gpu::spmm(sr, dense, {p, 8, ThreadMapping::coalesced});
            if (sr_out.output != me_out.output) return false;
            if (sr_out.counters.mma_invocations != spmm(sr_ref, dense, {p, 8, ThreadMapping::coalesced}).counters.mma_invocations)
                return false;
            if (decode_mebcrs(me) != m) return false;
            if (gpu::decode_mebcrs(me) != m) return false;  // GPU decode round trip
        }
    }
    return true;
}

bool errors() {  // tests/test_kernels.cpp:127-137, 303-312
    std::vector<Coord> coords;
    for (std::uint32_t i = 0; i < 8; ++i) coords.push_back({i, i, 1.0f});
    const MeBcrsMatrix me = gpu::encode_mebcrs(csr_from_coords(8, 8, coords), Precision::fp16);
    const DenseMatrix dense = generate_random_dense(8, 16, 1);
    auto throws = [](auto&& f, auto tag) {
        try {
            f();
        } catch (const decltype(tag)&) {
            return true;
        } catch (...) {
            return false;
        }
        return false;
    };
    bool ok = throws([&] { gpu::spmm(me, dense, {Precision::fp16, 16, ThreadMapping::direct}); }, ArgumentError(""));
    ok = ok && throws([&] { gpu::spmm(me, dense, {Precision::tf32, 8, ThreadMapping::direct}); }, ArgumentError(""));
    ok = ok && throws([&] { gpu::spmm(me, generate_random_dense(9, 16, 1), {Precision::fp16, 8, ThreadMapping::direct}); },
                      ShapeError(""));
    SddmmOperands ops{gpu::encode_mebcrs(generate_random_sparse(16, 16, 0.2, 81), Precision::fp16),
                      generate_random_dense(16, 8, 1), generate_random_dense(16, 8, 2)};
    ok = ok && throws([&] { gpu::sddmm(ops, {Precision::tf32, 8, ThreadMapping::coalesced}); }, ArgumentError(""));
    ops.a = generate_random_dense(15, 8, 1);
    ok = ok && throws([&] { gpu::sddmm(ops, {Precision::fp16, 8, ThreadMapping::coalesced}); }, ShapeError(""));
    return ok;
}

}  // namespace

int main() {
    report(2, "gpu spmm == reference spmm == dense oracle (200 matrices, both precisions/mappings)", criterion2());
    report(3, "scenario matrix: 2 MMAs on the swapped path", criterion3());
    report(6, "gpu sddmm == reference sddmm, and feeds spmm", criterion6());
    report(7, "residue blocks: gpu encode/spmm (ME-BCRS and SR-BCRS) == reference, decode round-trips", criterion7());
    report(0, "reference exception taxonomy through the C-ABI", errors());
    std::printf(failures ? "%d drop-in criteria FAILED\n" : "all drop-in criteria passed\n", failures);
    return failures ? 1 : 0;
}
