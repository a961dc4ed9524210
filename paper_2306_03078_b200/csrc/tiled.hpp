// tiled.hpp -- geometry of the HBM "tiled planes" layout of a fast-path layer.
// Shared by the host transcoder (transcode.cpp) and the CUDA kernels.
//
// Fast path: beta1, beta2 multiples of 16 (stored as repeated 16 x 16
// tiles), weight_bits in {2,3,4}, scale/zero bits in {2,3,4} (equal).  The layer is cut into CELLS of 32 rows x 256 columns (a row-group
// pair x a 16-block panel); cell (G, P) is stored contiguously at
// (G * Pn + P) * cell_bytes, cells in row-major order, so a warp streaming a
// contiguous cell range streams contiguous bytes.  A cell is two UNITS (one
// per 16-row group), each unit =
//
//   [codes  : 32 lanes x 16*BW bytes ]  lane L's A-fragment codes for the 16
//                                       m16n8k16 MMAs of the unit (2 super-
//                                       tiles x 8 blocks), in "containers"
//   [stats  : 32 lanes x (BS+BZ) bytes] lane L's 16 statistics codes as two
//                                       streams (rows g / g+8), see below
//   [scalars: 16 blocks x 8 bytes     ]  binary16 {scale_s, scale_z, zero_s, zero_z}
//
// unit_bytes = 512*BW + 32*(BS+BZ) + 128 = 16 group records of the stream
// (1856 B = 16 x 116 B at 3/3/3): the layout adds no bytes.  Rows / columns
// beyond the layer are zero padding (m -> multiple of 32, n -> of 256).
//
// Lane L = 4g + t holds, for MMA mu = 8h + j (block 16P + 8h + j):
//   A register r = 2*kh + rho : rows g + 8*rho, columns 2t + 8*kh + {0,1}
// (the m16n8k16 row-major A fragment).  A "container" of CW 32-bit words
// carries NPAIR (lo, hi) code pairs: lo codes form a 16*CW-bit stream in the
// low halves of the words, hi codes in the high halves; pair i sits at bit
// BW*i of both streams.  Pair i of container c is
//   rho = i / (NPAIR/2),  q = i % (NPAIR/2),  m = q / 2,  kh = q % 2,
//   mu = MPC*c + m.
// The kernel turns a pair into an f16x2 A register with ONE LOP3 mask: the
// codes land at bit offset p(q) of a window of the stream, i.e. as binary16
// subnormals worth code * 2^(p-24); the x operand is pre-scaled by 2^-p per
// column (xprep), so the product is exact and p cancels.
//
// Statistics (BS = BZ, the fast path): lane L = 4g + t holds 8 code pairs
// j = 4*kind + 2h + b (kind 0 = scale code, 1 = zero code; block 8h + 2t + b),
// the code of row g in a "lo" stream and that of row g + 8 in a "hi" stream,
// pair j at stream bit BS*j.  Like the weight containers, the lane's field
// interleaves the two streams per 16-bit word half -- word w = lo bytes
// 2w, 2w+1 | hi bytes 2w, 2w+1 (a 3-byte stream ends in the 2-byte word
// lo byte 2 | hi byte 2) -- so ONE LOP3 of a 16-bit window turns pair j into
// an f16x2 register holding both rows' codes as binary16 subnormals worth
// code * 2^(p-24), p = (BS*j) mod 8 (stat_p), which the kernel feeds straight
// to mixed-precision FMAs (fma.rn.f32.f16): the stat_dequant of a whole
// (row, block) pair without an int->float conversion.
//
// Outliers are re-bucketed per cell: offsets u32[cells+1] and entries u32
//   value16 | (col & 255) << 16 | (row - 32G) << 24
// sorted by (cell, row, col) -- 4 bytes per outlier like the stream.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define SPQR_HD __host__ __device__ __forceinline__
#else
#define SPQR_HD inline
#endif

namespace spqr_tiled {

inline constexpr std::uint32_t kCellRows = 32;
inline constexpr std::uint32_t kCellCols = 256;
inline constexpr std::uint32_t kUnitRows = 16;
inline constexpr std::uint32_t kScalarBytes = 128;

// The layout itself is defined for any bs, bz in [1, 8]; the kernel is
// instantiated for the statistic widths below (others use the raw-stream
// kernels, which are generic).
// Group sizes: any beta1, beta2 that are multiples of 16 -- a 16 x 16 tile of
// the layout then lies inside one stream record, whose statistics and scalars
// the loader repeats in every tile it covers (the kernels see beta1 = beta2 =
// 16; the stream / export keep the true groups).
SPQR_HD constexpr bool supported(int bw, int bs, int bz, std::uint32_t b1, std::uint32_t b2) {
    return b1 >= 16 && b1 % 16 == 0 && b2 >= 16 && b2 % 16 == 0 && (bw == 2 || bw == 3 || bw == 4) && bs == bz &&
           bs >= 2 && bs <= 4;
}
SPQR_HD constexpr int words_per_container(int bw) { return bw == 3 ? 3 : 1; }
SPQR_HD constexpr int mmas_per_container(int bw) { return bw == 3 ? 4 : (bw == 4 ? 1 : 2); }
SPQR_HD constexpr int pairs_per_container(int bw) { return 16 * words_per_container(bw) / bw; }
SPQR_HD constexpr int containers_per_unit(int bw) { return 16 / mmas_per_container(bw); }
SPQR_HD constexpr std::uint32_t code_bytes(int bw) { return 512u * bw; }
SPQR_HD constexpr std::uint32_t stat_bytes(int bs, int bz) { return 32u * (bs + bz); }
SPQR_HD constexpr std::uint32_t unit_bytes(int bw, int bs, int bz) {
    return code_bytes(bw) + stat_bytes(bs, bz) + kScalarBytes;
}
SPQR_HD constexpr std::uint32_t cell_bytes(int bw, int bs, int bz) { return 2u * unit_bytes(bw, bs, bz); }

// Pair i of a container starts at stream bit BW*i; the kernel reads it through
// the 16-bit window starting at byte floor(BW*i/8), where it sits at bit
// p = (BW*i) mod 8 (p + BW - 1 <= 9 keeps it inside the binary16 mantissa).
// p depends only on the pair class q = i % (NPAIR/2) = 2m + kh, so both rows of
// an MMA column pair share it: it is the per-column x pre-scale exponent.
SPQR_HD constexpr int prescale_p(int bw, int q) { return (bw * q) & 7; }

// Column (block k, column cc in block) -> pre-scale exponent.
SPQR_HD constexpr int column_prescale(int bw, std::uint32_t k, std::uint32_t cc) {
    const int m = static_cast<int>(k % 8) % mmas_per_container(bw);
    const int kh = static_cast<int>(cc / 8);
    return prescale_p(bw, 2 * m + kh);
}

// x operands of one 256-column panel, built by the kernel in shared memory.
// x modes: 0 = one fp16 column, 1 = one fp32 column as fp16 hi + lo parts,
// 2 = two fp16 batch columns (the second column's operands after the first's).
//   [B rows : 16 blocks x 16 f16  ] fp16(x 2^(e - p_c - p_s(block))), natural
//                                    column order (ldmatrix rows of B^T)
//   [XX     : 16 f32              ] -2^(-p_z(block)) sum_c B_c 2^p_c
//   [SC     : 2 f32 (+ 8 B pad)   ] 2^(48 - e) as a product of two normal floats
//   [xp     : 256 f16 | 256 f32 | 2 x 256 f16] x in solve order (outlier products)
//   [B lo   : 16 x 16 f16         ] mode 1: fp16(residual of B); mode 2: column 1's B rows
//   [XX1, SC1: 16 f32, 2 f32 + pad] mode 2: column 1's
// e = the panel's power-of-two scale (max |x| 2^e in [2^14, 2^15)), p_c = the
// column's code pre-scale, p_s / p_z = the pre-scales of the block's scale /
// zero code pairs (stat_p).
inline constexpr std::uint32_t kPanelFragBytes = 512;
inline constexpr std::uint32_t kPanelXXOff = 512;
inline constexpr std::uint32_t kPanelSCOff = 576;
inline constexpr std::uint32_t kPanelXPOff = 592;
SPQR_HD constexpr std::uint32_t panel_xp_bytes(int xm) { return xm == 0 ? 512u : 1024u; }
SPQR_HD constexpr std::uint32_t panel_lo_off(int xm) { return kPanelXPOff + panel_xp_bytes(xm); }
SPQR_HD constexpr std::uint32_t panel_xx1_off(int xm) { return panel_lo_off(xm) + kPanelFragBytes; }
SPQR_HD constexpr std::uint32_t panel_sc1_off(int xm) { return panel_xx1_off(xm) + 64u; }
SPQR_HD constexpr std::uint32_t panel_bytes(int xm) {
    return xm == 0 ? kPanelXPOff + 512u : (xm == 1 ? panel_lo_off(1) + kPanelFragBytes : panel_sc1_off(2) + 16u);
}

// Statistics pair geometry (BS bits per code): stream bit, window byte and
// the code's bit offset inside its 16-bit window.
SPQR_HD constexpr int stat_pair(int kind, int h, int b) { return 4 * kind + 2 * h + b; }
SPQR_HD constexpr int stat_window(int bs, int j) { return (bs * j) >> 3; }
SPQR_HD constexpr int stat_p(int bs, int j) { return (bs * j) & 7; }
// Logical byte f of a lane's statistics field -> (stream: 0 lo / 1 hi, stream byte).
SPQR_HD constexpr int stat_field_stream(int bs, int f) {
    return f < 4 * (bs / 2) ? (f & 3) >> 1 : (f - 4 * (bs / 2));
}
SPQR_HD constexpr int stat_field_byte(int bs, int f) {
    return f < 4 * (bs / 2) ? 2 * (f >> 2) + (f & 1) : bs - 1;
}

// Byte b of lane L's statistics field inside the unit's stats area.  A
// 6-byte field (3/3-bit statistics) is split into a 4-byte plane and a 2-byte
// plane so that a lane reads it with two aligned loads; other widths are
// lane-contiguous.
SPQR_HD constexpr std::uint32_t stat_byte_offset(int lane, int b, int sb) {
    return (sb > 4 && sb < 8)
               ? (b < 4 ? 4u * lane + b : 128u + static_cast<std::uint32_t>(sb - 4) * lane + (b - 4))
               : static_cast<std::uint32_t>(sb * lane + b);
}

// Entry packing of the per-cell outlier lists.
SPQR_HD constexpr std::uint32_t pack_entry(std::uint32_t local_row, std::uint32_t col_in_cell,
                                           std::uint16_t v) {
    return static_cast<std::uint32_t>(v) | ((col_in_cell & 255u) << 16) | (local_row << 24);
}

}  // namespace spqr_tiled
