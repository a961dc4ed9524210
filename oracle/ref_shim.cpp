// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).  Built by
// oracle/Makefile into oracle/_ref/libspqr_ref.so straight from the sources
// where they lie (/root/reference/proj/include), with the declaration-only
// Eigen stand-in in oracle/eigen_shim.  No reference source is copied here;
// this file only includes the headers and marshals arguments.
//
// The namespace is renamed (spqr -> spqr_ref) so the reference can never be
// confused with, or link against, the product's own spqr:: symbols.
#define spqr spqr_ref
#include "spqr/kernel.hpp"
#undef spqr

#include <cstring>
#include <thread>
#include <vector>

namespace R = spqr_ref;

namespace {
struct Handle {
    R::SpqrTensor t;
    R::TilePlan plan;
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const R::Error& e) {
        return 1 + static_cast<int>(e.code());
    } catch (...) {
        return 1000;
    }
}
}  // namespace

extern "C" {

int ref_decode(const uint8_t* bytes, size_t n, void** out) {
    *out = nullptr;
    return guard([&] {
        auto* h = new Handle;
        try {
            h->t = R::decode(std::span<const uint8_t>(bytes, n));  // format.hpp:354
            h->plan = R::build_tile_plan(h->t);                   // kernel.hpp:54
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void ref_free(void* h) { delete static_cast<Handle*>(h); }

int ref_encode(void* hv, uint8_t* out, size_t cap, size_t* len) {
    return guard([&] {
        auto b = R::encode(static_cast<Handle*>(hv)->t);  // format.hpp:269
        *len = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    });
}

int ref_dequantize_full(void* hv, float* out) {
    return guard([&] {
        R::DenseTensor w = R::dequantize_full(static_cast<Handle*>(hv)->t);  // kernel.hpp:17
        std::memcpy(out, w.data().data(), w.size() * sizeof(float));
    });
}

int ref_matvec(void* hv, const float* x, float* y) {
    return guard([&] {
        auto* h = static_cast<Handle*>(hv);
        auto v = R::matvec(h->t, std::span<const float>(x, h->t.cols), h->plan);  // kernel.hpp:89
        std::memcpy(y, v.data(), v.size() * sizeof(float));
    });
}

int ref_matvec_naive(void* hv, const float* x, float* y) {
    return guard([&] {
        auto* h = static_cast<Handle*>(hv);
        auto v = R::matvec_naive(h->t, std::span<const float>(x, h->t.cols));  // kernel.hpp:131
        std::memcpy(y, v.data(), v.size() * sizeof(float));
    });
}

// Rows [r0, r1) of a decoded reference tensor as an independent reference
// tensor (same columns, permutation and flags; statistics of the band's
// beta2-groups; outliers rebased), with its own TilePlan.  Built from the
// reference's own types (format.hpp:32-67, solver.hpp:66-142) so the CPU
// baseline never touches the product library.  r0 must be beta2-aligned.
int ref_slice_rows(void* hv, uint32_t r0, uint32_t r1, void** out) {
    *out = nullptr;
    return guard([&] {
        const R::SpqrTensor& s = static_cast<Handle*>(hv)->t;
        if (r0 >= r1 || r1 > s.rows || r0 % s.beta2 != 0)
            R::fail(R::Errc::config_invalid, "band must be non-empty, in range and beta2-aligned");
        auto* h = new Handle;
        R::SpqrTensor& t = h->t;
        const uint32_t m = r1 - r0, n = s.cols;
        t.rows = m; t.cols = n; t.weight_bits = s.weight_bits; t.scale_bits = s.scale_bits;
        t.zero_bits = s.zero_bits; t.beta1 = s.beta1; t.beta2 = s.beta2; t.act_order = s.act_order;
        t.integer_zero = s.integer_zero; t.full_range_sign = s.full_range_sign;
        t.outliers_enabled = s.outliers_enabled; t.tau = s.tau; t.lambda_rel = s.lambda_rel;
        t.permutation = s.permutation;
        t.codes.rows = m; t.codes.cols = n; t.codes.bits = s.codes.bits;
        t.codes.codes.assign(s.codes.codes.begin() + static_cast<size_t>(r0) * n,
                             s.codes.codes.begin() + static_cast<size_t>(r1) * n);
        t.stats = s.stats;
        t.stats.rows = m;
        const uint32_t g0 = r0 / s.beta2, g1 = (r1 + s.beta2 - 1) / s.beta2;
        for (auto& b : t.stats.blocks) {
            auto cut = [&](auto& v) {
                if (!v.empty()) v.assign(v.begin() + r0, v.begin() + r1);
            };
            cut(b.scale_codes); cut(b.zero_codes); cut(b.raw_scales); cut(b.raw_zeros);
            if (!b.groups.empty()) b.groups.assign(b.groups.begin() + g0, b.groups.begin() + g1);
        }
        t.outliers.rows = m; t.outliers.cols = n;
        for (const auto& o : s.outliers.items)
            if (o.row >= r0 && o.row < r1) t.outliers.items.push_back(R::Outlier{o.row - r0, o.col, o.value16});
        h->plan = R::build_tile_plan(t);  // kernel.hpp:54
        *out = h;
    });
}

// Row-band harness for the multi-core CPU baseline: each band is an
// independent reference tensor; `nthreads` threads call the reference's own
// matvec(t, x, plan) on disjoint bands.  The reference code is unmodified.
int ref_matvec_bands(void** hs, int nbands, const float* x, float* y, int nthreads) {
    std::vector<size_t> off(nbands + 1, 0);
    for (int b = 0; b < nbands; ++b) off[b + 1] = off[b] + static_cast<Handle*>(hs[b])->t.rows;
    std::vector<int> rc(nbands, 0);
    auto work = [&](int tid) {
        for (int b = tid; b < nbands; b += nthreads) rc[b] = ref_matvec(hs[b], x, y + off[b]);
    };
    std::vector<std::thread> th;
    for (int i = 1; i < nthreads; ++i) th.emplace_back(work, i);
    work(0);
    for (auto& t : th) t.join();
    for (int v : rc)
        if (v) return v;
    return 0;
}

int ref_bench_matvec(void* hv, const float* x, int repeats, double* out3) {
    return guard([&] {
        auto* h = static_cast<Handle*>(hv);
        auto r = R::bench_matvec(h->t, std::span<const float>(x, h->t.cols), repeats);  // kernel.hpp:185
        out3[0] = r.tiled_ns_per_op;
        out3[1] = r.naive_ns_per_op;
        out3[2] = r.dense_ns_per_op;
    });
}

int ref_estimate_avg_bits(int bw, int bs, int bz, uint32_t b1, uint32_t b2, double ro, double* out5) {
    return guard([&] {
        auto e = R::estimate_avg_bits(bw, bs, bz, b1, b2, ro);  // format.hpp:531
        out5[0] = e.avg_bits; out5[1] = e.base; out5[2] = e.first_level;
        out5[3] = e.second_level; out5[4] = e.outliers;
    });
}

int ref_measure_actual_bits(void* hv, double* out3) {
    return guard([&] {
        auto mb = R::measure_actual_bits(static_cast<Handle*>(hv)->t);  // format.hpp:550
        out3[0] = mb.bits_per_param; out3[1] = mb.per_outlier_bits;
        out3[2] = static_cast<double>(mb.payload_bytes);
    });
}

size_t ref_payload_bytes(uint32_t rows, uint32_t cols, int wb, int sb, int zb, uint32_t b1,
                         uint32_t b2, uint32_t nnz, int has_perm) {
    R::LayoutSpec ls;
    ls.rows = rows; ls.cols = cols; ls.weight_bits = wb; ls.scale_bits = sb; ls.zero_bits = zb;
    ls.beta1 = b1; ls.beta2 = b2; ls.outlier_count = nnz; ls.has_permutation = has_perm != 0;
    return R::stream_payload_bytes(ls);  // layout.hpp:47
}

uint16_t ref_fp16_from_float(float f) { return R::fp16_from_float(f); }
float ref_fp16_to_float(uint16_t h) { return R::fp16_to_float(h); }

// Build a reference SpqrTensor from flat arrays (same layout as the C oracle's
// oracle_from_arrays) so tests can encode synthetic tensors with the reference.
int ref_from_arrays(uint32_t rows, uint32_t cols, int wb, int sb, int zb, uint32_t b1, uint32_t b2,
                    uint16_t flags, float tau, float lambda_rel, const uint32_t* order,
                    const uint8_t* codes, const uint8_t* scodes, const uint8_t* zcodes,
                    const float* raw_s, const float* raw_z, const uint16_t* scal, uint32_t nnz,
                    const uint32_t* orow, const uint32_t* ocol, const uint16_t* oval, void** out) {
    *out = nullptr;
    return guard([&] {
        auto* h = new Handle;
        R::SpqrTensor& t = h->t;
        t.rows = rows; t.cols = cols; t.weight_bits = wb; t.scale_bits = sb; t.zero_bits = zb;
        t.beta1 = b1; t.beta2 = b2;
        t.act_order = flags & R::fformat::kFlagActOrder;
        t.integer_zero = flags & R::fformat::kFlagIntegerZero;
        t.full_range_sign = flags & R::fformat::kFlagFullRangeSign;
        t.outliers_enabled = flags & R::fformat::kFlagOutliersEnabled;
        t.tau = tau; t.lambda_rel = lambda_rel;
        if (order) {
            t.permutation = R::Permutation::from_order(std::vector<uint32_t>(order, order + cols));
        } else {
            t.permutation = R::Permutation::identity(cols);
        }
        t.codes.rows = rows; t.codes.cols = cols; t.codes.bits = wb;
        t.codes.codes.assign(codes, codes + static_cast<size_t>(rows) * cols);
        const uint32_t NB = (cols + b1 - 1) / b1, NG = (rows + b2 - 1) / b2;
        t.stats.rows = rows; t.stats.cols = cols; t.stats.beta1 = b1; t.stats.beta2 = b2;
        t.stats.scale_bits = sb; t.stats.zero_bits = zb;
        t.stats.blocks.resize(NB);
        const bool anyq = sb != R::kRawStatsBits || zb != R::kRawStatsBits;
        for (uint32_t k = 0; k < NB; ++k) {
            R::BlockStats& b = t.stats.blocks[k];
            const size_t o = static_cast<size_t>(k) * rows;
            if (sb != R::kRawStatsBits) b.scale_codes.assign(scodes + o, scodes + o + rows);
            else b.raw_scales.assign(raw_s + o, raw_s + o + rows);
            if (zb != R::kRawStatsBits) b.zero_codes.assign(zcodes + o, zcodes + o + rows);
            else b.raw_zeros.assign(raw_z + o, raw_z + o + rows);
            if (anyq) {
                b.groups.resize(NG);
                for (uint32_t g = 0; g < NG; ++g) {
                    const uint16_t* s = scal + (static_cast<size_t>(k) * NG + g) * 4;
                    b.groups[g].scale_s = s[0]; b.groups[g].scale_z = s[1];
                    b.groups[g].zero_s = s[2]; b.groups[g].zero_z = s[3];
                }
            }
        }
        t.outliers.rows = rows; t.outliers.cols = cols;
        t.outliers.items.resize(nnz);
        for (uint32_t i = 0; i < nnz; ++i) t.outliers.items[i] = R::Outlier{orow[i], ocol[i], oval[i]};
        h->plan = R::build_tile_plan(t);
        *out = h;
    });
}

}  // extern "C"
