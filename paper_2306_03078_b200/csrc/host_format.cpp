// host_format.cpp -- the .spqr wire format on the host: validation, decode,
// encode, size model, bit budgets, row slicing, and their C ABI entry points.
//
// Behavioural contract (the reference, /root/reference/proj/include/spqr):
//   size model ............ layout.hpp:14-77
//   encode ................ format.hpp:269-352 (validate_tensor_for_encode :219-265)
//   decode ................ format.hpp:354-500 (same checks, order and Errc)
//   save/load ............. format.hpp:502-517
//   estimate/measure bits . format.hpp:531-557
// Parity: tests/test_format.py checks every entry point byte-for-byte against
// the reference compiled into oracle/_ref and the golden fixtures.
#include <algorithm>
#include <fstream>
#include <numeric>

#include "internal.hpp"

namespace spqr {

// ------------------------------------------------------------------ types --
Permutation Permutation::identity(std::uint32_t n) {
    Permutation p;
    p.order.resize(n);
    std::iota(p.order.begin(), p.order.end(), 0u);
    p.inverse = p.order;
    return p;
}

Permutation Permutation::from_order(std::vector<std::uint32_t> order) {
    Permutation p;
    const std::uint32_t n = static_cast<std::uint32_t>(order.size());
    p.inverse.assign(n, UINT32_MAX);
    for (std::uint32_t k = 0; k < n; ++k) {
        const std::uint32_t src = order[k];
        if (src >= n || p.inverse[src] != UINT32_MAX)
            fail(Errc::config_invalid, "order is not a bijection");
        p.inverse[src] = k;
    }
    p.order = std::move(order);
    return p;
}

bool Permutation::is_identity() const {
    for (std::uint32_t k = 0; k < order.size(); ++k)
        if (order[k] != k) return false;
    return true;
}

double OutlierSet::rate() const {
    if (rows == 0 || cols == 0) return 0.0;
    return static_cast<double>(items.size()) / (static_cast<double>(rows) * cols);
}

void OutlierSet::validate() const {
    for (std::size_t i = 1; i < items.size(); ++i)
        if (!(items[i - 1] < items[i]))
            fail(Errc::corrupt_csr, "outliers must be strictly sorted by (row, col)");
    for (const Outlier& o : items)
        if (o.row >= rows || o.col >= cols) fail(Errc::corrupt_csr, "outlier out of bounds");
    if (rate() > kOutlierRateCap)
        fail(Errc::outlier_budget_exceeded,
             "outlier rate " + std::to_string(rate()) + " exceeds sanity cap");
}

float BilevelStats::scale_at(std::uint32_t block, std::uint32_t row) const {
    const BlockStats& b = blocks[block];
    if (scale_bits == kRawStatsBits) return b.raw_scales[row];
    const StatGroupScalars& g = b.groups[row / beta2];
    return stat_dequant(g.scale_s, g.scale_z, b.scale_codes[row]);
}

float BilevelStats::zero_at(std::uint32_t block, std::uint32_t row) const {
    const BlockStats& b = blocks[block];
    if (zero_bits == kRawStatsBits) return b.raw_zeros[row];
    const StatGroupScalars& g = b.groups[row / beta2];
    return stat_dequant(g.zero_s, g.zero_z, b.zero_codes[row]);
}

DenseTensor::DenseTensor(std::uint32_t rows, std::uint32_t cols)
    : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows) * cols, 0.0f) {
    if (rows == 0 || cols == 0) fail(Errc::shape_mismatch, "tensor dimensions must be >= 1");
}

DenseTensor::DenseTensor(std::uint32_t rows, std::uint32_t cols, std::vector<float> values)
    : rows_(rows), cols_(cols), data_(std::move(values)) {
    if (rows == 0 || cols == 0) fail(Errc::shape_mismatch, "tensor dimensions must be >= 1");
    if (data_.size() != static_cast<std::size_t>(rows) * cols)
        fail(Errc::shape_mismatch, "payload size does not match dimensions");
}

LayoutSpec SpqrTensor::layout() const {
    LayoutSpec ls;
    ls.rows = rows;
    ls.cols = cols;
    ls.weight_bits = weight_bits;
    ls.scale_bits = scale_bits;
    ls.zero_bits = zero_bits;
    ls.beta1 = beta1;
    ls.beta2 = beta2;
    ls.outlier_count = static_cast<std::uint32_t>(outliers.items.size());
    ls.has_permutation = has_permutation();
    return ls;
}

// ------------------------------------------------------------- size model --
std::size_t packed_field_bytes(std::size_t count, int bits) {
    return (count * static_cast<std::size_t>(bits) + 7) / 8;
}

std::size_t group_record_bytes(const LayoutSpec& ls, std::uint32_t gr, std::uint32_t bw) {
    auto side = [gr](int bits) {
        return bits <= 8 ? 4 + packed_field_bytes(gr, bits) : 4 * static_cast<std::size_t>(gr);
    };
    return side(ls.scale_bits) + side(ls.zero_bits) +
           packed_field_bytes(static_cast<std::size_t>(gr) * bw, ls.weight_bits);
}

// Closed form: at most two distinct block widths and two group heights.
std::size_t stream_payload_bytes(const LayoutSpec& ls) {
    const std::uint32_t nb_full = ls.cols / ls.beta1, last_w = ls.cols % ls.beta1;
    const std::uint32_t ng_full = ls.rows / ls.beta2, last_r = ls.rows % ls.beta2;
    auto column = [&](std::uint32_t bw) {
        std::size_t b = static_cast<std::size_t>(ng_full) * group_record_bytes(ls, ls.beta2, bw);
        if (last_r) b += group_record_bytes(ls, last_r, bw);
        return b;
    };
    std::size_t bytes = static_cast<std::size_t>(nb_full) * column(ls.beta1);
    if (last_w) bytes += column(last_w);
    if (ls.has_permutation) bytes += 4 * static_cast<std::size_t>(ls.cols);
    bytes += 4 * (static_cast<std::size_t>(ls.rows) + 1);
    bytes += 4 * static_cast<std::size_t>(ls.outlier_count);
    return bytes;
}

double measured_bits_per_param(const LayoutSpec& ls) {
    return 8.0 * static_cast<double>(stream_payload_bytes(ls)) /
           (static_cast<double>(ls.rows) * static_cast<double>(ls.cols));
}

double per_outlier_bits(const LayoutSpec& ls) {
    if (ls.outlier_count == 0) return 0.0;
    return 32.0 + 32.0 * (static_cast<double>(ls.rows) + 1.0) / ls.outlier_count;
}

BitsEstimate estimate_avg_bits(int b_w, int b_s, int b_z, std::uint32_t beta1,
                               std::uint32_t beta2, double r_o) {
    if (b_w < 1 || b_s < 1 || b_z < 1 || beta1 < 1 || beta2 < 1 || r_o < 0.0)
        fail(Errc::config_invalid, "estimate parameters must be positive");
    BitsEstimate e;
    e.base = b_w;
    e.first_level = static_cast<double>(b_s + b_z) / beta1;
    e.second_level = 64.0 / (static_cast<double>(beta1) * beta2);
    e.outliers = 32.0 * r_o;
    e.avg_bits = e.base + e.first_level + e.second_level + e.outliers;
    return e;
}

MeasuredBits measure_actual_bits(const SpqrTensor& t) {
    const LayoutSpec ls = t.layout();
    return MeasuredBits{measured_bits_per_param(ls), per_outlier_bits(ls), stream_payload_bytes(ls)};
}

// ------------------------------------------------------------ bit fields --
namespace detail {

void unpack_bits(const std::uint8_t* src, std::uint8_t* dst, std::size_t count, int bits) {
    const std::uint32_t mask = (1u << bits) - 1u;
    std::uint64_t acc = 0;
    int have = 0;
    for (std::size_t i = 0; i < count; ++i) {
        if (have < bits) {
            acc |= static_cast<std::uint64_t>(*src++) << have;
            have += 8;
        }
        dst[i] = static_cast<std::uint8_t>(acc & mask);
        acc >>= bits;
        have -= bits;
    }
}

void pack_bits(const std::uint8_t* src, std::size_t count, int bits, std::vector<std::uint8_t>& out) {
    std::uint64_t acc = 0;
    int have = 0;
    for (std::size_t i = 0; i < count; ++i) {
        acc |= static_cast<std::uint64_t>(src[i]) << have;
        have += bits;
        while (have >= 8) {
            out.push_back(static_cast<std::uint8_t>(acc));
            acc >>= 8;
            have -= 8;
        }
    }
    if (have > 0) out.push_back(static_cast<std::uint8_t>(acc));
}

// ------------------------------------------------------------ StreamView --
std::size_t StreamView::record_bytes(std::uint32_t gr, std::uint32_t bw) const {
    auto side = [gr](int bits) {
        return bits <= 8 ? 4 + packed_field_bytes(gr, bits) : 4 * static_cast<std::size_t>(gr);
    };
    return side(sb) + side(zb) + packed_field_bytes(static_cast<std::size_t>(gr) * bw, wb);
}

std::size_t StreamView::record_offset(std::uint32_t k, std::uint32_t g) const {
    return rec_off + static_cast<std::size_t>(k) * col_block_bytes +
           static_cast<std::size_t>(g) * record_bytes(b2, block_width(k));
}

std::uint32_t StreamView::order(std::uint32_t k) const {
    return perm_flag ? load_u32(base + perm_off + 4u * k) : k;
}

namespace {
// Header fields + derived offsets; `check` applies decode's header checks.
void read_header(StreamView& v, const std::uint8_t* bytes) {
    v.flags = StreamView::load_u16(bytes + 6);
    v.rows = StreamView::load_u32(bytes + 8);
    v.cols = StreamView::load_u32(bytes + 12);
    v.wb = bytes[16];
    v.sb = bytes[17];
    v.zb = bytes[18];
    v.b1 = StreamView::load_u32(bytes + 20);
    v.b2 = StreamView::load_u32(bytes + 24);
    v.nnz = StreamView::load_u32(bytes + 28);
    std::memcpy(&v.tau, bytes + 32, 4);
    std::memcpy(&v.lambda_rel, bytes + 36, 4);
    v.perm_flag = (v.flags & fformat::kFlagPermutation) != 0;
}

std::size_t expected_bytes(const StreamView& v) {
    LayoutSpec ls;
    ls.rows = v.rows; ls.cols = v.cols; ls.weight_bits = v.wb; ls.scale_bits = v.sb;
    ls.zero_bits = v.zb; ls.beta1 = v.b1; ls.beta2 = v.b2; ls.outlier_count = v.nnz;
    ls.has_permutation = v.perm_flag;
    return kSpqrHeaderBytes + stream_payload_bytes(ls);
}

void compute_offsets(StreamView& v) {
    v.nblocks = (v.cols + v.b1 - 1) / v.b1;
    v.ngroups = (v.rows + v.b2 - 1) / v.b2;
    v.perm_off = kSpqrHeaderBytes;
    v.rec_off = v.perm_off + (v.perm_flag ? 4 * static_cast<std::size_t>(v.cols) : 0);
    v.col_block_bytes = static_cast<std::size_t>(v.ngroups - 1) * v.record_bytes(v.b2, v.b1) +
                        v.record_bytes(v.group_rows(v.ngroups - 1), v.b1);
    std::size_t rec_total = static_cast<std::size_t>(v.nblocks - 1) * v.col_block_bytes;
    const std::uint32_t bwl = v.block_width(v.nblocks - 1);
    rec_total += static_cast<std::size_t>(v.ngroups - 1) * v.record_bytes(v.b2, bwl) +
                 v.record_bytes(v.group_rows(v.ngroups - 1), bwl);
    v.csr_off = v.rec_off + rec_total;
    v.ent_off = v.csr_off + 4 * (static_cast<std::size_t>(v.rows) + 1);
}
}  // namespace

StreamView geometry_from_prefix(const std::uint8_t* prefix, std::size_t len) {
    StreamView v;
    v.base = prefix;
    read_header(v, prefix);
    v.nbytes = expected_bytes(v);
    compute_offsets(v);
    if (len < v.rec_off) fail(Errc::malformed_stream, "prefix truncated");
    if (v.perm_flag) {
        bool ident = true;
        for (std::uint32_t k = 0; k < v.cols && ident; ++k) ident = v.order(k) == k;
        v.has_permutation = !ident;
    }
    return v;
}

StreamView parse_stream(const std::uint8_t* bytes, std::size_t n) {
    StreamView v;
    v.base = bytes;
    v.nbytes = n;
    if (n < kSpqrHeaderBytes) fail(Errc::malformed_stream, "stream truncated");
    if (std::memcmp(bytes, kSpqrMagic, 4) != 0) fail(Errc::malformed_stream, "bad magic");
    const std::uint16_t version = StreamView::load_u16(bytes + 4);
    if (version != kSpqrVersion) fail(Errc::version_unsupported, "version " + std::to_string(version));
    read_header(v, bytes);
    if (v.rows == 0 || v.cols == 0) fail(Errc::malformed_stream, "zero dimension");
    if (v.wb < 1 || v.wb > 8) fail(Errc::malformed_stream, "bad weight bits");
    auto stat_ok = [](int b) { return (b >= 1 && b <= 8) || b == kRawStatsBits; };
    if (!stat_ok(v.sb) || !stat_ok(v.zb)) fail(Errc::malformed_stream, "bad statistic bits");
    if (v.b1 < 1 || v.b2 < 1) fail(Errc::malformed_stream, "bad group sizes");
    if (v.nnz > 0 && v.cols > 0xffffu)
        fail(Errc::malformed_stream, "outliers present but columns exceed u16 range");
    if (n != expected_bytes(v)) fail(Errc::malformed_stream, "stream length does not match header");
    compute_offsets(v);

    // permutation: must be a bijection (hessian.hpp:27-39 via format.hpp:400-410)
    if (v.perm_flag) {
        std::vector<std::uint8_t> seen(v.cols, 0);
        bool ident = true;
        for (std::uint32_t k = 0; k < v.cols; ++k) {
            const std::uint32_t s = v.order(k);
            if (s >= v.cols || seen[s]) fail(Errc::malformed_stream, "permutation is not a bijection");
            seen[s] = 1;
            ident &= (s == k);
        }
        v.has_permutation = !ident;
    }

    // records: only the second-level scale sign is checked (format.hpp:448-449)
    if (v.sb != kRawStatsBits) {
        for (std::uint32_t k = 0; k < v.nblocks; ++k)
            for (std::uint32_t g = 0; g < v.ngroups; ++g)
                if (fp16_to_float(StreamView::load_u16(bytes + v.record_offset(k, g))) < 0.0f)
                    fail(Errc::malformed_stream, "negative second-level scale");
    }

    // CSR (format.hpp:475-497)
    if (v.row_start(0) != 0) fail(Errc::corrupt_csr, "row starts must begin at 0");
    for (std::uint32_t r = 0; r < v.rows; ++r)
        if (v.row_start(r + 1) < v.row_start(r)) fail(Errc::corrupt_csr, "row starts decrease");
    if (v.row_start(v.rows) != v.nnz) fail(Errc::corrupt_csr, "row starts do not sum to outlier count");
    for (std::uint32_t r = 0; r < v.rows; ++r) {
        const std::uint32_t e0 = v.row_start(r), e1 = v.row_start(r + 1);
        for (std::uint32_t i = e0; i < e1; ++i) {
            const std::uint16_t c = v.ent_col(i);
            if (c >= v.cols) fail(Errc::corrupt_csr, "outlier column out of range");
            if (i > e0 && v.ent_col(i - 1) >= c)
                fail(Errc::corrupt_csr, "outlier columns must increase within a row");
        }
    }
    return v;
}

// error plumbing
thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
int status_of(const Error& e) { return 1 + static_cast<int>(e.code()); }

}  // namespace detail

// ---------------------------------------------------------------- decode --
SpqrTensor decode(std::span<const std::uint8_t> bytes) {
    const detail::StreamView v = detail::parse_stream(bytes.data(), bytes.size());
    SpqrTensor t;
    t.rows = v.rows; t.cols = v.cols;
    t.weight_bits = v.wb; t.scale_bits = v.sb; t.zero_bits = v.zb;
    t.beta1 = v.b1; t.beta2 = v.b2;
    t.act_order = v.flags & fformat::kFlagActOrder;
    t.integer_zero = v.flags & fformat::kFlagIntegerZero;
    t.full_range_sign = v.flags & fformat::kFlagFullRangeSign;
    t.outliers_enabled = v.flags & fformat::kFlagOutliersEnabled;
    t.tau = v.tau; t.lambda_rel = v.lambda_rel;
    if (v.perm_flag) {
        std::vector<std::uint32_t> order(v.cols);
        for (std::uint32_t k = 0; k < v.cols; ++k) order[k] = v.order(k);
        t.permutation = Permutation::from_order(std::move(order));
    } else {
        t.permutation = Permutation::identity(v.cols);
    }
    t.codes.rows = v.rows; t.codes.cols = v.cols; t.codes.bits = v.wb;
    t.codes.codes.assign(static_cast<std::size_t>(v.rows) * v.cols, 0);
    BilevelStats& st = t.stats;
    st.rows = v.rows; st.cols = v.cols; st.beta1 = v.b1; st.beta2 = v.b2;
    st.scale_bits = v.sb; st.zero_bits = v.zb;
    st.blocks.resize(v.nblocks);
    const bool any_q = v.sb != kRawStatsBits || v.zb != kRawStatsBits;
    std::vector<std::uint8_t> wbuf;
    for (std::uint32_t k = 0; k < v.nblocks; ++k) {
        BlockStats& bs = st.blocks[k];
        const std::uint32_t c0 = k * v.b1, bw = v.block_width(k);
        if (any_q) bs.groups.resize(v.ngroups);
        (v.sb != kRawStatsBits ? (void)bs.scale_codes.resize(v.rows) : (void)bs.raw_scales.resize(v.rows));
        (v.zb != kRawStatsBits ? (void)bs.zero_codes.resize(v.rows) : (void)bs.raw_zeros.resize(v.rows));
        for (std::uint32_t g = 0; g < v.ngroups; ++g) {
            const std::uint32_t r0 = g * v.b2, gr = v.group_rows(g);
            const std::uint8_t* p = v.base + v.record_offset(k, g);
            if (v.sb != kRawStatsBits) {
                bs.groups[g].scale_s = detail::StreamView::load_u16(p);
                bs.groups[g].scale_z = detail::StreamView::load_u16(p + 2);
                p += 4;
            }
            if (v.zb != kRawStatsBits) {
                bs.groups[g].zero_s = detail::StreamView::load_u16(p);
                bs.groups[g].zero_z = detail::StreamView::load_u16(p + 2);
                p += 4;
            }
            if (v.sb != kRawStatsBits) {
                detail::unpack_bits(p, bs.scale_codes.data() + r0, gr, v.sb);
                p += packed_field_bytes(gr, v.sb);
            } else {
                std::memcpy(bs.raw_scales.data() + r0, p, 4u * gr);
                p += 4u * gr;
            }
            if (v.zb != kRawStatsBits) {
                detail::unpack_bits(p, bs.zero_codes.data() + r0, gr, v.zb);
                p += packed_field_bytes(gr, v.zb);
            } else {
                std::memcpy(bs.raw_zeros.data() + r0, p, 4u * gr);
                p += 4u * gr;
            }
            wbuf.resize(static_cast<std::size_t>(gr) * bw);
            detail::unpack_bits(p, wbuf.data(), wbuf.size(), v.wb);
            for (std::uint32_t r = 0; r < gr; ++r)
                std::memcpy(t.codes.codes.data() + static_cast<std::size_t>(r0 + r) * v.cols + c0,
                            wbuf.data() + static_cast<std::size_t>(r) * bw, bw);
        }
    }
    t.outliers.rows = v.rows;
    t.outliers.cols = v.cols;
    t.outliers.items.reserve(v.nnz);
    for (std::uint32_t r = 0; r < v.rows; ++r)
        for (std::uint32_t i = v.row_start(r); i < v.row_start(r + 1); ++i)
            t.outliers.items.push_back(Outlier{r, v.ent_col(i), v.ent_val(i)});
    return t;
}

// ---------------------------------------------------------------- encode --
namespace {

void put16(std::vector<std::uint8_t>& o, std::uint16_t v) {
    o.push_back(static_cast<std::uint8_t>(v));
    o.push_back(static_cast<std::uint8_t>(v >> 8));
}
void put32(std::vector<std::uint8_t>& o, std::uint32_t v) {
    for (int s = 0; s < 32; s += 8) o.push_back(static_cast<std::uint8_t>(v >> s));
}

void validate_for_encode(const SpqrTensor& t) {  // format.hpp:219-265
    if (t.rows == 0 || t.cols == 0) fail(Errc::shape_mismatch, "empty tensor");
    if (t.weight_bits < 1 || t.weight_bits > 8) fail(Errc::shape_mismatch, "bad weight bits");
    auto stat_ok = [](int b) { return (b >= 1 && b <= 8) || b == kRawStatsBits; };
    if (!stat_ok(t.scale_bits) || !stat_ok(t.zero_bits)) fail(Errc::shape_mismatch, "bad statistic bits");
    if (t.beta1 < 1 || t.beta2 < 1) fail(Errc::shape_mismatch, "bad group sizes");
    if (t.codes.rows != t.rows || t.codes.cols != t.cols || t.codes.bits != t.weight_bits)
        fail(Errc::shape_mismatch, "code matrix does not match header");
    if (t.codes.codes.size() != static_cast<std::size_t>(t.rows) * t.cols)
        fail(Errc::shape_mismatch, "code payload size mismatch");
    const std::uint32_t maxq = max_code(t.weight_bits);
    if (std::any_of(t.codes.codes.begin(), t.codes.codes.end(), [maxq](std::uint8_t c) { return c > maxq; }))
        fail(Errc::shape_mismatch, "weight code out of range");
    const BilevelStats& s = t.stats;
    if (s.rows != t.rows || s.cols != t.cols || s.beta1 != t.beta1 || s.beta2 != t.beta2 ||
        s.scale_bits != t.scale_bits || s.zero_bits != t.zero_bits)
        fail(Errc::shape_mismatch, "statistics do not match header");
    const std::uint32_t nb = (t.cols + t.beta1 - 1) / t.beta1, ng = (t.rows + t.beta2 - 1) / t.beta2;
    if (s.blocks.size() != nb) fail(Errc::shape_mismatch, "block count mismatch");
    const bool any_q = t.scale_bits != kRawStatsBits || t.zero_bits != kRawStatsBits;
    for (const BlockStats& b : s.blocks) {
        if (t.scale_bits == kRawStatsBits ? b.raw_scales.size() != t.rows : b.scale_codes.size() != t.rows)
            fail(Errc::shape_mismatch, t.scale_bits == kRawStatsBits ? "raw scale size" : "scale code size");
        if (t.zero_bits == kRawStatsBits ? b.raw_zeros.size() != t.rows : b.zero_codes.size() != t.rows)
            fail(Errc::shape_mismatch, t.zero_bits == kRawStatsBits ? "raw zero size" : "zero code size");
        if (any_q && b.groups.size() != ng) fail(Errc::shape_mismatch, "stat group count mismatch");
    }
    if (t.outliers.rows != t.rows || t.outliers.cols != t.cols)
        fail(Errc::shape_mismatch, "outlier set does not match header");
    t.outliers.validate();
    if (!t.outliers.items.empty() && t.cols > 0xffffu)
        fail(Errc::column_index_overflow, "outliers need column indices < 65536");
    if (t.has_permutation() && t.permutation.size() != t.cols)
        fail(Errc::shape_mismatch, "permutation size mismatch");
}

}  // namespace

std::vector<std::uint8_t> encode(const SpqrTensor& t) {
    validate_for_encode(t);
    std::vector<std::uint8_t> out;
    out.reserve(kSpqrHeaderBytes + stream_payload_bytes(t.layout()));
    const bool perm = t.has_permutation();
    std::uint16_t flags = (perm ? fformat::kFlagPermutation : 0) |
                          (t.act_order ? fformat::kFlagActOrder : 0) |
                          (t.integer_zero ? fformat::kFlagIntegerZero : 0) |
                          (t.full_range_sign ? fformat::kFlagFullRangeSign : 0) |
                          (t.outliers_enabled ? fformat::kFlagOutliersEnabled : 0);
    out.insert(out.end(), kSpqrMagic, kSpqrMagic + 4);
    put16(out, kSpqrVersion);
    put16(out, flags);
    put32(out, t.rows);
    put32(out, t.cols);
    out.push_back(static_cast<std::uint8_t>(t.weight_bits));
    out.push_back(static_cast<std::uint8_t>(t.scale_bits));
    out.push_back(static_cast<std::uint8_t>(t.zero_bits));
    out.push_back(0);
    put32(out, t.beta1);
    put32(out, t.beta2);
    put32(out, static_cast<std::uint32_t>(t.outliers.items.size()));
    put32(out, std::bit_cast<std::uint32_t>(t.tau));
    put32(out, std::bit_cast<std::uint32_t>(t.lambda_rel));
    out.resize(out.size() + 8, 0);
    if (perm)
        for (std::uint32_t k : t.permutation.order) put32(out, k);

    const std::uint32_t nb = t.stats.block_count(), ng = t.stats.group_count();
    std::vector<std::uint8_t> tile;
    for (std::uint32_t k = 0; k < nb; ++k) {
        const std::uint32_t c0 = k * t.beta1, bw = std::min(t.beta1, t.cols - c0);
        const BlockStats& bs = t.stats.blocks[k];
        for (std::uint32_t g = 0; g < ng; ++g) {
            const std::uint32_t r0 = g * t.beta2, gr = std::min(t.beta2, t.rows - r0);
            if (t.scale_bits != kRawStatsBits) { put16(out, bs.groups[g].scale_s); put16(out, bs.groups[g].scale_z); }
            if (t.zero_bits != kRawStatsBits) { put16(out, bs.groups[g].zero_s); put16(out, bs.groups[g].zero_z); }
            if (t.scale_bits != kRawStatsBits) detail::pack_bits(bs.scale_codes.data() + r0, gr, t.scale_bits, out);
            else for (std::uint32_t r = r0; r < r0 + gr; ++r) put32(out, std::bit_cast<std::uint32_t>(bs.raw_scales[r]));
            if (t.zero_bits != kRawStatsBits) detail::pack_bits(bs.zero_codes.data() + r0, gr, t.zero_bits, out);
            else for (std::uint32_t r = r0; r < r0 + gr; ++r) put32(out, std::bit_cast<std::uint32_t>(bs.raw_zeros[r]));
            tile.resize(static_cast<std::size_t>(gr) * bw);
            for (std::uint32_t r = 0; r < gr; ++r)
                std::memcpy(tile.data() + static_cast<std::size_t>(r) * bw,
                            t.codes.codes.data() + static_cast<std::size_t>(r0 + r) * t.cols + c0, bw);
            detail::pack_bits(tile.data(), tile.size(), t.weight_bits, out);
        }
    }
    // CSR: cumulative row counts, then (u16 col, u16 value) pairs
    put32(out, 0);
    std::size_t item = 0;
    for (std::uint32_t r = 0; r < t.rows; ++r) {
        while (item < t.outliers.items.size() && t.outliers.items[item].row == r) ++item;
        put32(out, static_cast<std::uint32_t>(item));
    }
    for (const Outlier& o : t.outliers.items) {
        put16(out, static_cast<std::uint16_t>(o.col));
        put16(out, o.value16);
    }
    return out;
}

void save_spqr(const SpqrTensor& t, const std::filesystem::path& path) {
    const std::vector<std::uint8_t> bytes = encode(t);
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) fail(Errc::io_failure, "cannot open " + path.string() + " for writing");
    os.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!os) fail(Errc::io_failure, "write failed for " + path.string());
}

SpqrTensor load_spqr(const std::filesystem::path& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) fail(Errc::missing_file, "cannot open " + path.string());
    std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    return decode(bytes);
}

// ------------------------------------------------------------ slice rows --
std::vector<std::uint8_t> slice_rows(std::span<const std::uint8_t> stream, std::uint32_t r0,
                                     std::uint32_t r1) {
    const detail::StreamView v = detail::parse_stream(stream.data(), stream.size());
    if (r0 >= r1 || r1 > v.rows) fail(Errc::shape_mismatch, "row band out of range");
    if (r0 % v.b2 != 0 && r0 != 0)
        fail(Errc::config_invalid, "row band must start on a beta2 group boundary");
    const std::uint32_t m = r1 - r0, g0 = r0 / v.b2, g1 = (r1 + v.b2 - 1) / v.b2;
    if (r1 != v.rows && r1 % v.b2 != 0)
        fail(Errc::config_invalid, "row band must end on a beta2 group boundary");
    const std::uint32_t e0 = v.row_start(r0), e1 = v.row_start(r1);
    std::vector<std::uint8_t> out(stream.begin(), stream.begin() + kSpqrHeaderBytes);
    std::memcpy(out.data() + 8, &m, 4);
    const std::uint32_t nnz = e1 - e0;
    std::memcpy(out.data() + 28, &nnz, 4);
    if (v.perm_flag) out.insert(out.end(), stream.begin() + v.perm_off, stream.begin() + v.rec_off);
    for (std::uint32_t k = 0; k < v.nblocks; ++k) {
        const std::size_t a = v.record_offset(k, g0);
        const std::size_t b = (g1 == v.ngroups) ? (k + 1 < v.nblocks ? v.record_offset(k + 1, 0) : v.csr_off)
                                                : v.record_offset(k, g1);
        out.insert(out.end(), stream.begin() + a, stream.begin() + b);
    }
    for (std::uint32_t r = r0; r <= r1; ++r) put32(out, v.row_start(r) - e0);
    out.insert(out.end(), stream.begin() + v.ent_off + 4u * e0, stream.begin() + v.ent_off + 4u * e1);
    return out;
}

}  // namespace spqr

// ================================================================ C ABI ====
using spqr::detail::guard;

namespace {

spqr::SpqrTensor tensor_from_arrays(const spqr_tensor_arrays& a) {
    using namespace spqr;
    SpqrTensor t;
    t.rows = a.rows; t.cols = a.cols;
    t.weight_bits = a.weight_bits; t.scale_bits = a.scale_bits; t.zero_bits = a.zero_bits;
    t.beta1 = a.beta1; t.beta2 = a.beta2;
    t.act_order = a.flags & fformat::kFlagActOrder;
    t.integer_zero = a.flags & fformat::kFlagIntegerZero;
    t.full_range_sign = a.flags & fformat::kFlagFullRangeSign;
    t.outliers_enabled = a.flags & fformat::kFlagOutliersEnabled;
    t.tau = a.tau; t.lambda_rel = a.lambda_rel;
    if (t.rows == 0 || t.cols == 0 || t.beta1 == 0 || t.beta2 == 0)
        fail(Errc::shape_mismatch, "empty tensor");
    t.permutation = a.order ? Permutation::from_order(std::vector<std::uint32_t>(a.order, a.order + a.cols))
                            : Permutation::identity(a.cols);
    const std::size_t mn = static_cast<std::size_t>(a.rows) * a.cols;
    t.codes.rows = a.rows; t.codes.cols = a.cols; t.codes.bits = a.weight_bits;
    t.codes.codes.assign(a.codes, a.codes + mn);
    BilevelStats& s = t.stats;
    s.rows = a.rows; s.cols = a.cols; s.beta1 = a.beta1; s.beta2 = a.beta2;
    s.scale_bits = a.scale_bits; s.zero_bits = a.zero_bits;
    const std::uint32_t nb = s.block_count(), ng = s.group_count();
    const bool any_q = a.scale_bits != kRawStatsBits || a.zero_bits != kRawStatsBits;
    s.blocks.resize(nb);
    for (std::uint32_t k = 0; k < nb; ++k) {
        BlockStats& b = s.blocks[k];
        const std::size_t o = static_cast<std::size_t>(k) * a.rows;
        if (a.scale_bits == kRawStatsBits) b.raw_scales.assign(a.raw_scales + o, a.raw_scales + o + a.rows);
        else b.scale_codes.assign(a.scale_codes + o, a.scale_codes + o + a.rows);
        if (a.zero_bits == kRawStatsBits) b.raw_zeros.assign(a.raw_zeros + o, a.raw_zeros + o + a.rows);
        else b.zero_codes.assign(a.zero_codes + o, a.zero_codes + o + a.rows);
        if (any_q) {
            b.groups.resize(ng);
            for (std::uint32_t g = 0; g < ng; ++g) {
                const std::uint16_t* p = a.group_scalars + (static_cast<std::size_t>(k) * ng + g) * 4;
                b.groups[g] = StatGroupScalars{p[0], p[1], p[2], p[3]};
            }
        }
    }
    t.outliers.rows = a.rows; t.outliers.cols = a.cols;
    t.outliers.items.resize(a.outlier_count);
    for (std::uint32_t i = 0; i < a.outlier_count; ++i)
        t.outliers.items[i] = Outlier{a.outlier_rows[i], a.outlier_cols[i], a.outlier_vals[i]};
    return t;
}

void fill_info(const spqr::detail::StreamView& v, spqr_layer_info* info) {
    std::memset(info, 0, sizeof(*info));
    info->rows = v.rows; info->cols = v.cols;
    info->weight_bits = v.wb; info->scale_bits = v.sb; info->zero_bits = v.zb;
    info->beta1 = v.b1; info->beta2 = v.b2; info->outlier_count = v.nnz;
    info->flags = v.flags; info->has_permutation = v.has_permutation;
    info->tau = v.tau; info->lambda_rel = v.lambda_rel;
    info->payload_bytes = v.nbytes - spqr::kSpqrHeaderBytes;
    info->fast_path = spqr::detail::tiled_supported(v);
    info->device = -1;
}

int copy_out(const std::vector<std::uint8_t>& b, std::uint8_t* out, std::size_t cap, std::size_t* len) {
    if (len) *len = b.size();
    if (!out || cap < b.size()) {
        spqr::detail::set_last_error("buffer too small");
        return SPQR_E_BUFFER_TOO_SMALL;
    }
    std::memcpy(out, b.data(), b.size());
    return SPQR_OK;
}

}  // namespace

extern "C" {

const char* spqr_last_error(void) { return spqr::detail::g_last_error.c_str(); }
const char* spqr_version(void) { return "spqr-b200 0.1 (tiled layout v1, sm_100a)"; }

int spqr_stream_validate(const uint8_t* stream, size_t nbytes, spqr_layer_info* info) {
    return guard([&] { fill_info(spqr::detail::parse_stream(stream, nbytes), info); });
}

int spqr_decode_arrays(const uint8_t* stream, size_t nbytes, spqr_tensor_arrays* o) {
    return guard([&] {
        const spqr::SpqrTensor t = spqr::decode(std::span<const std::uint8_t>(stream, nbytes));
        o->rows = t.rows; o->cols = t.cols; o->weight_bits = t.weight_bits;
        o->scale_bits = t.scale_bits; o->zero_bits = t.zero_bits; o->beta1 = t.beta1; o->beta2 = t.beta2;
        o->flags = (t.act_order ? 2u : 0u) | (t.integer_zero ? 4u : 0u) | (t.full_range_sign ? 8u : 0u) |
                   (t.outliers_enabled ? 16u : 0u) | (t.has_permutation() ? 1u : 0u);
        o->tau = t.tau; o->lambda_rel = t.lambda_rel;
        if (o->order) std::memcpy(o->order, t.permutation.order.data(), 4ull * t.cols);
        if (o->codes) std::memcpy(o->codes, t.codes.codes.data(), t.codes.codes.size());
        const std::uint32_t nb = t.stats.block_count(), ng = t.stats.group_count();
        for (std::uint32_t k = 0; k < nb; ++k) {
            const spqr::BlockStats& b = t.stats.blocks[k];
            const std::size_t off = static_cast<std::size_t>(k) * t.rows;
            if (o->scale_codes && !b.scale_codes.empty()) std::memcpy(o->scale_codes + off, b.scale_codes.data(), t.rows);
            if (o->zero_codes && !b.zero_codes.empty()) std::memcpy(o->zero_codes + off, b.zero_codes.data(), t.rows);
            if (o->raw_scales && !b.raw_scales.empty()) std::memcpy(o->raw_scales + off, b.raw_scales.data(), 4ull * t.rows);
            if (o->raw_zeros && !b.raw_zeros.empty()) std::memcpy(o->raw_zeros + off, b.raw_zeros.data(), 4ull * t.rows);
            if (o->group_scalars && !b.groups.empty())
                for (std::uint32_t g = 0; g < ng; ++g) {
                    std::uint16_t* p = o->group_scalars + (static_cast<std::size_t>(k) * ng + g) * 4;
                    p[0] = b.groups[g].scale_s; p[1] = b.groups[g].scale_z;
                    p[2] = b.groups[g].zero_s; p[3] = b.groups[g].zero_z;
                }
        }
        o->outlier_count = static_cast<std::uint32_t>(t.outliers.items.size());
        for (std::size_t i = 0; i < t.outliers.items.size(); ++i) {
            if (o->outlier_rows) o->outlier_rows[i] = t.outliers.items[i].row;
            if (o->outlier_cols) o->outlier_cols[i] = t.outliers.items[i].col;
            if (o->outlier_vals) o->outlier_vals[i] = t.outliers.items[i].value16;
        }
    });
}

int spqr_encode_arrays(const spqr_tensor_arrays* a, uint8_t* out, size_t cap, size_t* len) {
    int rc = SPQR_OK;
    int g = guard([&] { rc = copy_out(spqr::encode(tensor_from_arrays(*a)), out, cap, len); });
    return g ? g : rc;
}

uint64_t spqr_payload_bytes(const spqr_layout_spec* s) {
    spqr::LayoutSpec ls;
    ls.rows = s->rows; ls.cols = s->cols; ls.weight_bits = s->weight_bits;
    ls.scale_bits = s->scale_bits; ls.zero_bits = s->zero_bits; ls.beta1 = s->beta1;
    ls.beta2 = s->beta2; ls.outlier_count = s->outlier_count; ls.has_permutation = s->has_permutation;
    return spqr::stream_payload_bytes(ls);
}

int spqr_estimate_avg_bits(int b_w, int b_s, int b_z, uint32_t beta1, uint32_t beta2, double r_o,
                           double* out5) {
    return guard([&] {
        const spqr::BitsEstimate e = spqr::estimate_avg_bits(b_w, b_s, b_z, beta1, beta2, r_o);
        out5[0] = e.avg_bits; out5[1] = e.base; out5[2] = e.first_level;
        out5[3] = e.second_level; out5[4] = e.outliers;
    });
}

int spqr_measure_actual_bits(const uint8_t* stream, size_t nbytes, double* out3) {
    return guard([&] {
        const spqr::detail::StreamView v = spqr::detail::parse_stream(stream, nbytes);
        spqr::LayoutSpec ls;
        ls.rows = v.rows; ls.cols = v.cols; ls.weight_bits = v.wb; ls.scale_bits = v.sb;
        ls.zero_bits = v.zb; ls.beta1 = v.b1; ls.beta2 = v.b2; ls.outlier_count = v.nnz;
        ls.has_permutation = v.has_permutation;
        out3[0] = spqr::measured_bits_per_param(ls);
        out3[1] = spqr::per_outlier_bits(ls);
        out3[2] = static_cast<double>(spqr::stream_payload_bytes(ls));
    });
}

int spqr_stream_slice_rows(const uint8_t* stream, size_t nbytes, uint32_t r0, uint32_t r1,
                           uint8_t* out, size_t cap, size_t* len) {
    int rc = SPQR_OK;
    int g = guard([&] {
        rc = copy_out(spqr::slice_rows(std::span<const std::uint8_t>(stream, nbytes), r0, r1), out, cap, len);
    });
    return g ? g : rc;
}

int spqr_transcode_roundtrip_host(const uint8_t* stream, size_t nbytes, uint8_t* out, size_t cap,
                                  size_t* len) {
    int rc = SPQR_OK;
    int g = guard([&] {
        const spqr::detail::StreamView v = spqr::detail::parse_stream(stream, nbytes);
        if (!spqr::detail::tiled_supported(v))
            spqr::fail(spqr::Errc::config_invalid, "layer is outside the tiled fast-path geometry");
        const spqr::detail::TiledHost t = spqr::detail::transcode_to_tiled(v, 0);
        rc = copy_out(spqr::detail::tiled_to_stream(v, t, 0), out, cap, len);
    });
    return g ? g : rc;
}

int spqr_debug_tiled_host(const uint8_t* stream, size_t nbytes, uint32_t* dims4, uint8_t* cells,
                          uint32_t* cell_off, uint32_t* entries) {
    return guard([&] {
        const spqr::detail::StreamView v = spqr::detail::parse_stream(stream, nbytes);
        if (!spqr::detail::tiled_supported(v))
            spqr::fail(spqr::Errc::config_invalid, "layer is outside the tiled fast-path geometry");
        const spqr::detail::TiledHost t = spqr::detail::transcode_to_tiled(v, 0);
        dims4[0] = t.Gn; dims4[1] = t.Pn; dims4[2] = t.cell_bytes;
        dims4[3] = static_cast<std::uint32_t>(t.cells.size());
        if (cells) std::memcpy(cells, t.cells.data(), t.cells.size());
        if (cell_off) std::memcpy(cell_off, t.cell_off.data(), 4 * t.cell_off.size());
        (void)entries;
    });
}

}  // extern "C"
