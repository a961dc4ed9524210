// spqr/format.hpp -- the .spqr wire format: size model, encode/decode,
// file I/O and bit-budget reports (drop-in API).
//
// Replaces, name for name:
//   kSpqrHeaderBytes, packed_field_bytes, group_record_bytes,
//   stream_payload_bytes, measured_bits_per_param, per_outlier_bits .. layout.hpp:12-77
//   kSpqrMagic, kSpqrVersion, fformat::kFlag* ........................ format.hpp:18-27
//   encode / decode / save_spqr / load_spqr .......................... format.hpp:269-517
//   BitsEstimate / estimate_avg_bits / MeasuredBits /
//   measure_actual_bits ............................................... format.hpp:523-557
// plus slice_rows (row bands for the row-sharded multi-GPU wrapper).
#pragma once

#include <cstdint>
#include <filesystem>
#include <span>
#include <vector>

#include "spqr/types.hpp"

namespace spqr {

inline constexpr std::size_t kSpqrHeaderBytes = 48;
inline constexpr char kSpqrMagic[4] = {'S', 'P', 'Q', 'R'};
inline constexpr std::uint16_t kSpqrVersion = 1;

namespace fformat {
inline constexpr std::uint16_t kFlagPermutation = 1u << 0;
inline constexpr std::uint16_t kFlagActOrder = 1u << 1;
inline constexpr std::uint16_t kFlagIntegerZero = 1u << 2;
inline constexpr std::uint16_t kFlagFullRangeSign = 1u << 3;
inline constexpr std::uint16_t kFlagOutliersEnabled = 1u << 4;
}  // namespace fformat

std::size_t packed_field_bytes(std::size_t count, int bits);
std::size_t group_record_bytes(const LayoutSpec& ls, std::uint32_t rows_in_group,
                               std::uint32_t cols_in_block);
std::size_t stream_payload_bytes(const LayoutSpec& ls);
double measured_bits_per_param(const LayoutSpec& ls);
double per_outlier_bits(const LayoutSpec& ls);

std::vector<std::uint8_t> encode(const SpqrTensor& t);
SpqrTensor decode(std::span<const std::uint8_t> bytes);
void save_spqr(const SpqrTensor& t, const std::filesystem::path& path);
SpqrTensor load_spqr(const std::filesystem::path& path);

struct BitsEstimate {
    double avg_bits = 0.0, base = 0.0, first_level = 0.0, second_level = 0.0, outliers = 0.0;
};
BitsEstimate estimate_avg_bits(int b_w, int b_s, int b_z, std::uint32_t beta1,
                               std::uint32_t beta2, double r_o);

struct MeasuredBits {
    double bits_per_param = 0.0, per_outlier_bits = 0.0;
    std::size_t payload_bytes = 0;
};
MeasuredBits measure_actual_bits(const SpqrTensor& t);

// Rows [r0, r1) of a stream as a standalone valid stream (rebased CSR).
std::vector<std::uint8_t> slice_rows(std::span<const std::uint8_t> stream, std::uint32_t r0,
                                     std::uint32_t r1);

}  // namespace spqr
