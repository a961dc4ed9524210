// spqr/types.hpp -- the data types of the SpQR decode path (drop-in API).
//
// Field names follow the reference so existing callers compile unchanged:
//   CodeMatrix, max_code, dequant_value, stat_dequant ... quantizer.hpp:34-67
//   LayoutSpec ........................................... layout.hpp:18-28
//   Permutation .......................................... hessian.hpp:14-48
//   Outlier, OutlierSet, StatGroupScalars, BlockStats,
//   BilevelStats ......................................... solver.hpp:66-142
//   DenseTensor .......................................... tensor.hpp:30-66
//   SpqrTensor ........................................... format.hpp:32-67
// The arithmetic in dequant_value / stat_dequant is the binary32 contract the
// GPU kernels reproduce bit-for-bit.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "spqr/common.hpp"

namespace spqr {

inline constexpr int kRawStatsBits = 16;
inline constexpr double kOutlierRateCap = 0.05;

inline std::uint32_t max_code(int bits) { return (1u << bits) - 1u; }

// W = s * (code - z) in binary32: two roundings, never contracted (the library
// is built with -ffp-contract=off).
inline float dequant_value(float s, float z, std::uint32_t code) {
    return s * (static_cast<float>(code) - z);
}
inline float stat_dequant(std::uint16_t s16, std::uint16_t z16, std::uint32_t code) {
    return dequant_value(fp16_to_float(s16), fp16_to_float(z16), code);
}

struct CodeMatrix {
    std::uint32_t rows = 0, cols = 0;
    int bits = 0;
    std::vector<std::uint8_t> codes;  // row-major, one code per byte
    std::uint8_t operator()(std::uint32_t r, std::uint32_t c) const {
        return codes[static_cast<std::size_t>(r) * cols + c];
    }
};

struct LayoutSpec {
    std::uint32_t rows = 0, cols = 0;
    int weight_bits = 0, scale_bits = 0, zero_bits = 0;
    std::uint32_t beta1 = 0, beta2 = 0;
    std::uint32_t outlier_count = 0;
    bool has_permutation = false;
};

struct Permutation {
    std::vector<std::uint32_t> order;    // order[k]: source column at solve position k
    std::vector<std::uint32_t> inverse;  // inverse[order[k]] == k

    static Permutation identity(std::uint32_t n);
    static Permutation from_order(std::vector<std::uint32_t> order);  // throws config_invalid
    bool is_identity() const;
    std::uint32_t size() const { return static_cast<std::uint32_t>(order.size()); }
};

struct Outlier {
    std::uint32_t row = 0;
    std::uint32_t col = 0;      // solve-order column
    std::uint16_t value16 = 0;  // binary16 correction added on top of the in-place code
    friend bool operator<(const Outlier& a, const Outlier& b) {
        return a.row != b.row ? a.row < b.row : a.col < b.col;
    }
};

struct OutlierSet {
    std::uint32_t rows = 0, cols = 0;
    std::vector<Outlier> items;  // strictly sorted by (row, col)
    double rate() const;
    void validate() const;  // corrupt_csr / outlier_budget_exceeded
};

struct StatGroupScalars {
    std::uint16_t scale_s = 0x3c00, scale_z = 0x0000;  // identity defaults (1.0, 0.0)
    std::uint16_t zero_s = 0x3c00, zero_z = 0x0000;
};

struct BlockStats {
    std::vector<std::uint8_t> scale_codes, zero_codes;  // m each when bits <= 8
    std::vector<StatGroupScalars> groups;               // ceil(m/beta2) when any side quantized
    std::vector<float> raw_scales, raw_zeros;           // m each when bits == 16
};

struct BilevelStats {
    std::uint32_t rows = 0, cols = 0, beta1 = 0, beta2 = 0;
    int scale_bits = 0, zero_bits = 0;
    std::vector<BlockStats> blocks;

    std::uint32_t block_count() const { return (cols + beta1 - 1) / beta1; }
    std::uint32_t group_count() const { return (rows + beta2 - 1) / beta2; }
    float scale_at(std::uint32_t block, std::uint32_t row) const;
    float zero_at(std::uint32_t block, std::uint32_t row) const;
};

class DenseTensor {
public:
    DenseTensor() = default;
    DenseTensor(std::uint32_t rows, std::uint32_t cols);
    DenseTensor(std::uint32_t rows, std::uint32_t cols, std::vector<float> values);
    std::uint32_t rows() const { return rows_; }
    std::uint32_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    float operator()(std::uint32_t r, std::uint32_t c) const {
        return data_[static_cast<std::size_t>(r) * cols_ + c];
    }
    float& operator()(std::uint32_t r, std::uint32_t c) {
        return data_[static_cast<std::size_t>(r) * cols_ + c];
    }
    const std::vector<float>& data() const { return data_; }
    std::vector<float>& data() { return data_; }
    bool operator==(const DenseTensor& o) const = default;

private:
    std::uint32_t rows_ = 0, cols_ = 0;
    std::vector<float> data_;
};

struct SpqrTensor {
    std::uint32_t rows = 0, cols = 0;
    int weight_bits = 0, scale_bits = 0, zero_bits = 0;
    std::uint32_t beta1 = 0, beta2 = 0;
    bool act_order = false, integer_zero = false, full_range_sign = true, outliers_enabled = true;
    float tau = 0.0f, lambda_rel = 0.0f;
    Permutation permutation;
    CodeMatrix codes;
    BilevelStats stats;
    OutlierSet outliers;

    bool has_permutation() const { return !permutation.is_identity(); }
    LayoutSpec layout() const;
};

}  // namespace spqr
