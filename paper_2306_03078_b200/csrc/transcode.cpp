// transcode.cpp -- stream <-> tiled HBM layout (see tiled.hpp for the layout).
//
// The stream stores group records column-block-major (format.hpp:300-333):
// record (k, g) for all row groups of block k, then block k+1.  The GPU wants
// a 32-row strip to stream contiguously with every lane's MMA fragment in one
// 16-byte-aligned slice, so the loader re-lays the records once at load time.
// The transform is lossless (tiled_to_stream is its inverse; tests check the
// round trip byte-for-byte) and adds no bytes beyond zero padding of ragged
// edges.  Parallel over row-group pairs with std::thread.
#include <algorithm>
#include <thread>

#include "internal.hpp"
#include "tiled.hpp"

namespace spqr::detail {

namespace T = spqr_tiled;

bool tiled_supported(const StreamView& v) { return T::supported(v.wb, v.sb, v.zb, v.b1, v.b2); }

namespace {

// Dense staging of one unit (16 rows x 256 columns = 16 blocks).
struct UnitStage {
    std::uint8_t codes[16][256];
    std::uint8_t scode[16][16];  // [block][row]
    std::uint8_t zcode[16][16];
    std::uint16_t scal[16][4];
};

template <class F>
void parallel_for(std::uint32_t n, int threads, F&& f) {
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    threads = static_cast<int>(std::min<std::uint32_t>(threads, std::max(1u, n)));
    if (threads <= 1) {
        for (std::uint32_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    for (int w = 0; w < threads; ++w)
        th.emplace_back([&, w] {
            for (std::uint32_t i = w; i < n; i += threads) f(i);
        });
    for (auto& t : th) t.join();
}

// The 16 x 16 window at (row ro, column co) of stream record (k, g) -> stage
// block `blk` (beta1, beta2 multiples of 16: statistics and scalars of a wider
// group / block repeat in every unit / tiled block they cover).
void load_record(const StreamView& v, std::uint32_t k, std::uint32_t g, std::uint32_t ro, std::uint32_t co, int blk,
                 UnitStage& u, std::vector<std::uint8_t>& tmp) {
    const std::uint32_t gr = v.group_rows(g), bw = v.block_width(k);
    if (ro >= gr || co >= bw) return;
    const std::uint8_t* p = v.base + v.record_offset(k, g);
    for (int i = 0; i < 4; ++i) u.scal[blk][i] = StreamView::load_u16(p + 2 * i);
    p += 8;
    tmp.resize(static_cast<std::size_t>(gr) * bw + 2 * gr);
    std::uint8_t *sc = tmp.data(), *zc = sc + gr, *w = zc + gr;
    unpack_bits(p, sc, gr, v.sb);
    p += packed_field_bytes(gr, v.sb);
    unpack_bits(p, zc, gr, v.zb);
    p += packed_field_bytes(gr, v.zb);
    unpack_bits(p, w, static_cast<std::size_t>(gr) * bw, v.wb);
    const std::uint32_t nr = std::min(16u, gr - ro), nc = std::min(16u, bw - co);
    for (std::uint32_t r = 0; r < nr; ++r) {
        u.scode[blk][r] = sc[ro + r];
        u.zcode[blk][r] = zc[ro + r];
        std::memcpy(&u.codes[r][16 * blk], w + static_cast<std::size_t>(ro + r) * bw + co, nc);
    }
}

template <int BW>
void pack_unit_codes(const UnitStage& u, std::uint8_t* dst) {
    constexpr int CW = T::words_per_container(BW), MPC = T::mmas_per_container(BW);
    constexpr int NP = T::pairs_per_container(BW), CPU = T::containers_per_unit(BW);
    for (int L = 0; L < 32; ++L) {
        const int g = L >> 2, t = L & 3;
        std::uint8_t* lane = dst + L * 16 * BW;
        for (int c = 0; c < CPU; ++c) {
            std::uint64_t lo = 0, hi = 0;
            for (int i = 0; i < NP; ++i) {
                const int rho = i / (NP / 2), q = i % (NP / 2), m = q / 2, kh = q % 2;
                const int mu = MPC * c + m, blk = mu;  // mu = 8h + j = block within unit
                const int row = g + 8 * rho, col = 16 * blk + 2 * t + 8 * kh;
                lo |= static_cast<std::uint64_t>(u.codes[row][col]) << (BW * i);
                hi |= static_cast<std::uint64_t>(u.codes[row][col + 1]) << (BW * i);
            }
            for (int w = 0; w < CW; ++w) {
                const std::uint32_t word = static_cast<std::uint32_t>((lo >> (16 * w)) & 0xffffu) |
                                           (static_cast<std::uint32_t>((hi >> (16 * w)) & 0xffffu) << 16);
                std::memcpy(lane + 4 * (CW * c + w), &word, 4);
            }
        }
    }
}

template <int BW>
void unpack_unit_codes(const std::uint8_t* src, UnitStage& u) {
    constexpr int CW = T::words_per_container(BW), MPC = T::mmas_per_container(BW);
    constexpr int NP = T::pairs_per_container(BW), CPU = T::containers_per_unit(BW);
    constexpr std::uint64_t mask = (1u << BW) - 1u;
    for (int L = 0; L < 32; ++L) {
        const int g = L >> 2, t = L & 3;
        const std::uint8_t* lane = src + L * 16 * BW;
        for (int c = 0; c < CPU; ++c) {
            std::uint64_t lo = 0, hi = 0;
            for (int w = 0; w < CW; ++w) {
                std::uint32_t word;
                std::memcpy(&word, lane + 4 * (CW * c + w), 4);
                lo |= static_cast<std::uint64_t>(word & 0xffffu) << (16 * w);
                hi |= static_cast<std::uint64_t>(word >> 16) << (16 * w);
            }
            for (int i = 0; i < NP; ++i) {
                const int rho = i / (NP / 2), q = i % (NP / 2), m = q / 2, kh = q % 2;
                const int blk = MPC * c + m;
                const int row = g + 8 * rho, col = 16 * blk + 2 * t + 8 * kh;
                u.codes[row][col] = static_cast<std::uint8_t>((lo >> (BW * i)) & mask);
                u.codes[row][col + 1] = static_cast<std::uint8_t>((hi >> (BW * i)) & mask);
            }
        }
    }
}

// Lane statistics (tiled.hpp): pair j = 4*kind + 2h + b of block 8h + 2t + b,
// row g in the lo stream, row g + 8 in the hi stream, at stream bit bs*j.
void pack_unit_stats(const UnitStage& u, int bs, int bz, std::uint8_t* dst) {
    const int sbytes = bs + bz;
    for (int L = 0; L < 32; ++L) {
        const int g = L >> 2, t = L & 3;
        std::uint32_t st[2] = {0, 0};  // lo / hi streams (8 * bs <= 32 bits)
        for (int j = 0; j < 8; ++j) {
            const int kind = j >> 2, h = (j >> 1) & 1, b = j & 1, blk = 8 * h + 2 * t + b;
            for (int rho = 0; rho < 2; ++rho) {
                const std::uint32_t code = kind ? u.zcode[blk][g + 8 * rho] : u.scode[blk][g + 8 * rho];
                st[rho] |= code << (bs * j);
            }
        }
        for (int f = 0; f < sbytes; ++f)
            dst[T::stat_byte_offset(L, f, sbytes)] = static_cast<std::uint8_t>(
                st[T::stat_field_stream(bs, f)] >> (8 * T::stat_field_byte(bs, f)));
    }
}

void unpack_unit_stats(const std::uint8_t* src, int bs, int bz, UnitStage& u) {
    const int sbytes = bs + bz;
    const std::uint32_t mask = (1u << bs) - 1u;
    for (int L = 0; L < 32; ++L) {
        const int g = L >> 2, t = L & 3;
        std::uint32_t st[2] = {0, 0};
        for (int f = 0; f < sbytes; ++f)
            st[T::stat_field_stream(bs, f)] |= static_cast<std::uint32_t>(src[T::stat_byte_offset(L, f, sbytes)])
                                               << (8 * T::stat_field_byte(bs, f));
        for (int j = 0; j < 8; ++j) {
            const int kind = j >> 2, h = (j >> 1) & 1, b = j & 1, blk = 8 * h + 2 * t + b;
            for (int rho = 0; rho < 2; ++rho) {
                const auto code = static_cast<std::uint8_t>((st[rho] >> (bs * j)) & mask);
                (kind ? u.zcode : u.scode)[blk][g + 8 * rho] = code;
            }
        }
    }
}

void pack_unit(const UnitStage& u, int bw, int bs, int bz, std::uint8_t* dst) {
    switch (bw) {
        case 2: pack_unit_codes<2>(u, dst); break;
        case 3: pack_unit_codes<3>(u, dst); break;
        default: pack_unit_codes<4>(u, dst); break;
    }
    pack_unit_stats(u, bs, bz, dst + T::code_bytes(bw));
    std::memcpy(dst + T::code_bytes(bw) + T::stat_bytes(bs, bz), u.scal, T::kScalarBytes);
}

void unpack_unit(const std::uint8_t* src, int bw, int bs, int bz, UnitStage& u) {
    switch (bw) {
        case 2: unpack_unit_codes<2>(src, u); break;
        case 3: unpack_unit_codes<3>(src, u); break;
        default: unpack_unit_codes<4>(src, u); break;
    }
    unpack_unit_stats(src + T::code_bytes(bw), bs, bz, u);
    std::memcpy(u.scal, src + T::code_bytes(bw) + T::stat_bytes(bs, bz), T::kScalarBytes);
}

}  // namespace

TiledHost transcode_to_tiled(const StreamView& v, int threads) {
    if (!tiled_supported(v)) fail(Errc::config_invalid, "layer outside the tiled geometry");
    TiledHost t;
    t.Gn = (v.rows + 31) / 32;
    t.Pn = (v.cols + 255) / 256;
    t.cell_bytes = T::cell_bytes(v.wb, v.sb, v.zb);
    t.prefix.assign(v.base, v.base + v.rec_off);
    const std::size_t ncell = static_cast<std::size_t>(t.Gn) * t.Pn;
    const std::uint32_t ub = T::unit_bytes(v.wb, v.sb, v.zb);

    // outliers per cell -> record sizes: cell bytes + entries padded to 16 B
    std::vector<std::uint32_t> cnt(ncell, 0);
    for (std::uint32_t r = 0; r < v.rows; ++r)
        for (std::uint32_t i = v.row_start(r); i < v.row_start(r + 1); ++i)
            cnt[static_cast<std::size_t>(r / 32) * t.Pn + v.ent_col(i) / 256]++;
    t.cell_off.assign(ncell + 1, 0);
    std::uint64_t total = 0;
    for (std::size_t q = 0; q < ncell; ++q) {
        t.cell_off[q] = static_cast<std::uint32_t>(total);
        total += t.cell_bytes + 16ull * ((cnt[q] + 3) / 4);
        if (total > 0xfffffff0ull) fail(Errc::config_invalid, "layer too large for 32-bit record offsets");
    }
    t.cell_off[ncell] = static_cast<std::uint32_t>(total);
    t.cells.assign(total, 0xff);  // entry padding = 0xffffffff sentinels (row 255)
    // entries in (row, col) order within each cell
    std::vector<std::uint32_t> cursor(ncell);
    for (std::size_t q = 0; q < ncell; ++q) cursor[q] = t.cell_off[q] + t.cell_bytes;
    for (std::uint32_t r = 0; r < v.rows; ++r)  // rows ascending, cols ascending -> order kept
        for (std::uint32_t i = v.row_start(r); i < v.row_start(r + 1); ++i) {
            const std::uint32_t c = v.ent_col(i);
            const std::size_t q = static_cast<std::size_t>(r / 32) * t.Pn + c / 256;
            const std::uint32_t e = T::pack_entry(r % 32, c % 256, v.ent_val(i));
            std::memcpy(t.cells.data() + cursor[q], &e, 4);
            cursor[q] += 4;
        }

    parallel_for(t.Gn, threads, [&](std::uint32_t G) {
        UnitStage u;
        std::vector<std::uint8_t> tmp;
        for (std::uint32_t P = 0; P < t.Pn; ++P) {
            for (int rg = 0; rg < 2; ++rg) {
                std::memset(&u, 0, sizeof(u));
                const std::uint32_t r0u = 32 * G + 16 * rg, gg = r0u / v.b2;
                if (gg < v.ngroups)
                    for (int blk = 0; blk < 16; ++blk) {
                        const std::uint32_t c0 = 256 * P + 16 * blk, k = c0 / v.b1;
                        if (k < v.nblocks) load_record(v, k, gg, r0u - gg * v.b2, c0 - k * v.b1, blk, u, tmp);
                    }
                pack_unit(u, v.wb, v.sb, v.zb,
                          t.cells.data() + t.cell_off[static_cast<std::size_t>(G) * t.Pn + P] + rg * ub);
            }
        }
    });
    return t;
}

std::vector<std::uint8_t> tiled_to_stream(const StreamView& hdr, const TiledHost& t, int threads) {
    // geometry from the header prefix (the layer keeps header + permutation)
    const StreamView& v = hdr;
    const std::uint32_t ub = T::unit_bytes(v.wb, v.sb, v.zb);
    std::vector<std::uint8_t> out(t.prefix);
    out.resize(v.csr_off, 0);
    std::uint8_t* recs = out.data();
    // 1. every unit back into dense per-row arrays (16-column blocks)
    const std::uint32_t n16 = 16 * t.Pn, mpad = 32 * t.Gn, npad = 256 * t.Pn;
    std::vector<std::uint8_t> codes(static_cast<std::size_t>(mpad) * npad), scode(static_cast<std::size_t>(n16) * mpad),
        zcode(static_cast<std::size_t>(n16) * mpad);
    std::vector<std::uint16_t> scal(static_cast<std::size_t>(n16) * (mpad / 16) * 4);
    parallel_for(t.Gn, threads, [&](std::uint32_t G) {
        UnitStage u;
        for (std::uint32_t P = 0; P < t.Pn; ++P)
            for (int rg = 0; rg < 2; ++rg) {
                unpack_unit(t.cells.data() + t.cell_off[static_cast<std::size_t>(G) * t.Pn + P] + rg * ub,
                            v.wb, v.sb, v.zb, u);
                const std::uint32_t r0 = 32 * G + 16 * rg;
                for (int r = 0; r < 16; ++r)
                    std::memcpy(&codes[static_cast<std::size_t>(r0 + r) * npad + 256 * P], u.codes[r], 256);
                for (int blk = 0; blk < 16; ++blk) {
                    const std::size_t kb = 16 * P + blk;
                    std::memcpy(&scode[kb * mpad + r0], u.scode[blk], 16);
                    std::memcpy(&zcode[kb * mpad + r0], u.zcode[blk], 16);
                    std::memcpy(&scal[(kb * (mpad / 16) + r0 / 16) * 4], u.scal[blk], 8);
                }
            }
    });
    // 2. every stream record (k, g) from the first tiled block / unit it covers
    parallel_for(v.ngroups, threads, [&](std::uint32_t gg) {
        std::vector<std::uint8_t> buf, w;
        const std::uint32_t gr = v.group_rows(gg), r0 = gg * v.b2;
        for (std::uint32_t k = 0; k < v.nblocks; ++k) {
            const std::uint32_t bw = v.block_width(k), c0 = k * v.b1, kb = c0 / 16;
            buf.clear();
            const std::uint16_t* sc = &scal[(static_cast<std::size_t>(kb) * (mpad / 16) + r0 / 16) * 4];
            for (int i = 0; i < 4; ++i) {
                buf.push_back(static_cast<std::uint8_t>(sc[i]));
                buf.push_back(static_cast<std::uint8_t>(sc[i] >> 8));
            }
            pack_bits(&scode[static_cast<std::size_t>(kb) * mpad + r0], gr, v.sb, buf);
            pack_bits(&zcode[static_cast<std::size_t>(kb) * mpad + r0], gr, v.zb, buf);
            w.resize(static_cast<std::size_t>(gr) * bw);
            for (std::uint32_t r = 0; r < gr; ++r)
                std::memcpy(&w[static_cast<std::size_t>(r) * bw], &codes[static_cast<std::size_t>(r0 + r) * npad + c0], bw);
            pack_bits(w.data(), w.size(), v.wb, buf);
            std::memcpy(recs + v.record_offset(k, gg), buf.data(), buf.size());
        }
    });
    // CSR: per row, walk the row's cells left to right
    std::vector<std::uint32_t> rs(v.rows + 1, 0);
    std::vector<std::uint8_t> ent;
    ent.reserve(4ull * v.nnz);
    for (std::uint32_t r = 0; r < v.rows; ++r) {
        const std::uint32_t G = r / 32, lr = r % 32;
        for (std::uint32_t P = 0; P < t.Pn; ++P) {
            const std::size_t q = static_cast<std::size_t>(G) * t.Pn + P;
            for (std::uint32_t b = t.cell_off[q] + t.cell_bytes; b < t.cell_off[q + 1]; b += 4) {
                std::uint32_t e;
                std::memcpy(&e, t.cells.data() + b, 4);
                if ((e >> 24) != lr) continue;  // other row, or 0xffffffff padding
                const std::uint16_t col = static_cast<std::uint16_t>(256 * P + ((e >> 16) & 255u));
                ent.push_back(static_cast<std::uint8_t>(col));
                ent.push_back(static_cast<std::uint8_t>(col >> 8));
                ent.push_back(static_cast<std::uint8_t>(e));
                ent.push_back(static_cast<std::uint8_t>(e >> 8));
            }
        }
        rs[r + 1] = static_cast<std::uint32_t>(ent.size() / 4);
    }
    for (std::uint32_t r = 0; r <= v.rows; ++r)
        for (int b = 0; b < 4; ++b) out.push_back(static_cast<std::uint8_t>(rs[r] >> (8 * b)));
    out.insert(out.end(), ent.begin(), ent.end());
    return out;
}

}  // namespace spqr::detail
