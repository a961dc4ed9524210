// internal.hpp -- host-side internals shared by the library's translation units.
#pragma once

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "spqr/format.hpp"
#include "spqr/types.hpp"
#include "spqr_cuda.h"

namespace spqr::detail {

// Validated view over a .spqr stream (no codes materialised).  parse_stream()
// applies decode's checks (format.hpp:354-500) in the same order with the
// same Errc codes.
struct StreamView {
    const std::uint8_t* base = nullptr;
    std::size_t nbytes = 0;
    std::uint32_t rows = 0, cols = 0;
    int wb = 0, sb = 0, zb = 0;
    std::uint32_t b1 = 0, b2 = 0, nnz = 0;
    std::uint16_t flags = 0;
    float tau = 0.0f, lambda_rel = 0.0f;
    bool perm_flag = false;      // permutation section present in the stream
    bool has_permutation = false;  // ... and not the identity (SpqrTensor::has_permutation)
    std::uint32_t nblocks = 0, ngroups = 0;
    std::size_t perm_off = 0, rec_off = 0, csr_off = 0, ent_off = 0;
    std::size_t col_block_bytes = 0;  // bytes of one full-width column block of records

    std::uint32_t block_width(std::uint32_t k) const { return k + 1 < nblocks ? b1 : cols - k * b1; }
    std::uint32_t group_rows(std::uint32_t g) const { return g + 1 < ngroups ? b2 : rows - g * b2; }
    std::size_t record_bytes(std::uint32_t gr, std::uint32_t bw) const;
    std::size_t record_offset(std::uint32_t k, std::uint32_t g) const;
    std::uint32_t order(std::uint32_t k) const;  // permutation (identity when absent)
    std::uint32_t row_start(std::uint32_t r) const { return load_u32(base + csr_off + 4u * r); }
    std::uint16_t ent_col(std::uint32_t i) const { return load_u16(base + ent_off + 4u * i); }
    std::uint16_t ent_val(std::uint32_t i) const { return load_u16(base + ent_off + 4u * i + 2); }

    static std::uint32_t load_u32(const std::uint8_t* p) {
        std::uint32_t v;
        std::memcpy(&v, p, 4);
        return v;
    }
    static std::uint16_t load_u16(const std::uint8_t* p) {
        std::uint16_t v;
        std::memcpy(&v, p, 2);
        return v;
    }
};

StreamView parse_stream(const std::uint8_t* bytes, std::size_t n);
// Geometry only, from the header + permutation prefix of a stream whose
// payload was validated earlier (no payload access).
StreamView geometry_from_prefix(const std::uint8_t* prefix, std::size_t len);

// LSB-first packed field reader / writer (byte-padded fields).
void unpack_bits(const std::uint8_t* src, std::uint8_t* dst, std::size_t count, int bits);
void pack_bits(const std::uint8_t* src, std::size_t count, int bits, std::vector<std::uint8_t>& out);

// ---- tiled device layout (transcode.cpp) --------------------------------
struct TiledHost {
    std::uint32_t Gn = 0, Pn = 0;       // cell grid
    std::uint32_t cell_bytes = 0;
    std::vector<std::uint8_t> prefix;     // stream header + permutation section
    std::vector<std::uint8_t> cells;      // cell records: cell_bytes + entries (16-B padded)
    std::vector<std::uint32_t> cell_off;  // byte offset of record q, Gn*Pn+1 entries
};
bool tiled_supported(const StreamView& v);
TiledHost transcode_to_tiled(const StreamView& v, int threads);
// Inverse: rebuild the stream bytes (header fields and permutation from `hdr`).
std::vector<std::uint8_t> tiled_to_stream(const StreamView& hdr, const TiledHost& t, int threads);

// ---- C ABI error plumbing -------------------------------------------------
void set_last_error(const std::string& msg);
int status_of(const Error& e);

template <class F>
int guard(F&& f) {
    try {
        set_last_error("");
        f();
        return SPQR_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return status_of(e);
    } catch (const std::bad_alloc&) {
        set_last_error("IoFailure: host allocation failed");
        return SPQR_E_IO_FAILURE;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SPQR_E_CUDA;
    }
}

}  // namespace spqr::detail
