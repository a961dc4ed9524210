// transcode_dev.cuh -- the loader's stream -> tiled-layout transform on the
// GPU (K0 of SURVEY §8f), byte-identical to transcode.cpp's host version.
// Included by kernels.cuh (namespace spqr_dev).
//
// Reference anchor: the stream is decode()'s input (format.hpp:354-500: record
// (k, g) of column block k, row group g at rec_off + k*col_block_bytes +
// g*record_bytes; [S_s Z_s S_z Z_z] u16, packed scale codes, packed zero codes,
// packed weight codes row-major in the tile; CSR row_starts + (u16 col, u16
// value) entries).  The host validates the stream (parse_stream) and uploads
// it; these kernels re-lay it into cells (tiled.hpp):
//   tc_entries<true>   per cell: outlier count  -> host prefix -> cell_off
//   tc_units           per unit (warp): lane-fragment codes, lane statistics,
//                      block scalars
//   tc_entries<false>  per cell (warp): the cell's entries in (row, col) order
//                      + 0xffffffff padding to 16 B
// One warp per unit / cell, no atomics: the output is deterministic.

// Field offsets of record (k, gg).
struct RecFields {
    std::uint64_t o, s, z, w;  // record start, scale codes, zero codes, weight codes
    std::uint32_t bw, gr;      // block width, group rows
};
__device__ __forceinline__ RecFields rec_fields(const RawGeom& geo, std::uint32_t k, std::uint32_t gg) {
    RecFields f;
    f.bw = geo.block_width(k);
    f.gr = geo.group_rows(gg);
    f.o = geo.record_offset(k, gg);
    f.s = f.o + 8;
    f.z = f.s + RawGeom::packed(f.gr, geo.sb);
    f.w = f.z + RawGeom::packed(f.gr, geo.zb);
    return f;
}

template <int BW>
__global__ void __launch_bounds__(256) tc_units(const RawGeom geo, std::uint32_t Gn, std::uint32_t Pn,
                                                const std::uint32_t* __restrict__ cell_off, std::uint8_t* cells) {
    constexpr int CW = T::words_per_container(BW), MPC = T::mmas_per_container(BW);
    constexpr int NP = T::pairs_per_container(BW), CPU = T::containers_per_unit(BW);
    const std::uint32_t U = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    if (U >= 2u * Gn * Pn) return;
    const std::uint32_t q = U >> 1, rg = U & 1u;
    const std::uint32_t G = q / Pn, P = q - G * Pn;
    // beta1, beta2 multiples of 16: the unit's 16 rows lie in stream row group
    // gg at row offset ro, tiled block blk (16 columns) in stream column
    // block k at column offset co; statistics and scalars of wider groups /
    // blocks repeat in every unit / tiled block they cover
    const std::uint32_t r0u = 32u * G + 16u * rg;
    const std::uint32_t gg = r0u / geo.b2, ro = r0u - gg * geo.b2;
    auto kblk = [&](std::uint32_t blk, std::uint32_t& co) {
        const std::uint32_t c0 = 256u * P + 16u * blk, k = c0 / geo.b1;
        co = c0 - k * geo.b1;
        return k;
    };
    const int bs = geo.sb, bz = geo.zb;
    const std::uint32_t ub = T::unit_bytes(BW, bs, bz);
    std::uint8_t* dst = cells + cell_off[q] + rg * ub;
    const bool gvalid = gg < geo.ngroups;

    // weight codes: lane L's containers (tiled.hpp)
#pragma unroll 1
    for (int c = 0; c < CPU; ++c) {
        std::uint64_t lo = 0, hi = 0;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const int rho = i / (NP / 2), qq = i % (NP / 2), m = qq / 2, kh = qq % 2;
            const int blk = MPC * c + m;
            std::uint32_t co;
            const std::uint32_t k = kblk(blk, co);
            const std::uint32_t row = ro + g + 8 * rho, col = co + 2 * t + 8 * kh;  // within record (k, gg)
            std::uint32_t c0 = 0, c1 = 0;
            if (gvalid && k < geo.nblocks) {
                const RecFields f = rec_fields(geo, k, gg);
                if (row < f.gr) {
                    if (col < f.bw) c0 = geo.bits_at(f.w, static_cast<std::uint64_t>(row) * f.bw + col, BW);
                    if (col + 1 < f.bw) c1 = geo.bits_at(f.w, static_cast<std::uint64_t>(row) * f.bw + col + 1, BW);
                }
            }
            lo |= static_cast<std::uint64_t>(c0) << (BW * i);
            hi |= static_cast<std::uint64_t>(c1) << (BW * i);
        }
#pragma unroll
        for (int w = 0; w < CW; ++w) {
            const std::uint32_t word = static_cast<std::uint32_t>((lo >> (16 * w)) & 0xffffu) |
                                       (static_cast<std::uint32_t>((hi >> (16 * w)) & 0xffffu) << 16);
            reinterpret_cast<std::uint32_t*>(dst + lane * 16 * BW)[CW * c + w] = word;
        }
    }
    // lane statistics (tiled.hpp): pair j = 4*kind + 2h + b, rows g / g + 8 in
    // the lo / hi stream at stream bit bs*j
    {
        std::uint32_t st[2] = {0, 0};
#pragma unroll 1
        for (int j = 0; j < 8; ++j) {
            const int kind = j >> 2, h = (j >> 1) & 1, b = j & 1;
            std::uint32_t co;
            const std::uint32_t k = kblk(8 * h + 2 * t + b, co);
            RecFields f{};
            const bool kv = gvalid && k < geo.nblocks && co < geo.block_width(k);
            if (kv) f = rec_fields(geo, k, gg);
#pragma unroll
            for (int rho = 0; rho < 2; ++rho) {
                const std::uint32_t row = ro + g + 8 * rho;
                std::uint32_t code = 0;
                if (kv && row < f.gr) code = kind ? geo.bits_at(f.z, row, bz) : geo.bits_at(f.s, row, bs);
                st[rho] |= code << (bs * j);
            }
        }
        const int sbytes = bs + bz;
        std::uint8_t* sd = dst + T::code_bytes(BW);
        for (int f = 0; f < sbytes; ++f)
            sd[T::stat_byte_offset(lane, f, sbytes)] =
                static_cast<std::uint8_t>(st[T::stat_field_stream(bs, f)] >> (8 * T::stat_field_byte(bs, f)));
    }
    // block scalars {S_s, Z_s, S_z, Z_z}
    if (lane < 16) {
        std::uint32_t co;
        const std::uint32_t k = kblk(lane, co);
        std::uint32_t w0 = 0, w1 = 0;
        if (gvalid && k < geo.nblocks && co < geo.block_width(k)) {
            const std::uint64_t o = geo.record_offset(k, gg);
            w0 = geo.u32(o);
            w1 = geo.u32(o + 4);
        }
        std::uint32_t* sd = reinterpret_cast<std::uint32_t*>(dst + T::code_bytes(BW) + T::stat_bytes(bs, bz) + 8 * lane);
        sd[0] = w0;
        sd[1] = w1;
    }
}

// Per cell (one warp): lane = local row.  COUNT: number of entries of the
// cell -> cnt[q].  Else: the entries in (row, col) order at the cell's
// record tail, padded with 0xffffffff to a multiple of 4 entries.
template <bool COUNT>
__global__ void __launch_bounds__(256) tc_entries(const RawGeom geo, std::uint32_t Gn, std::uint32_t Pn,
                                                  std::uint32_t cell_bytes, const std::uint32_t* __restrict__ cell_off,
                                                  std::uint8_t* cells, std::uint32_t* cnt) {
    const std::uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= Gn * Pn) return;
    const std::uint32_t G = q / Pn, P = q - G * Pn;
    const std::uint32_t r = 32u * G + lane;
    std::uint32_t lo = 0, hi = 0;
    if (r < geo.rows) {
        const std::uint32_t rs = geo.u32(geo.csr_off + 4ull * r), re = geo.u32(geo.csr_off + 4ull * (r + 1));
        auto col_at = [&](std::uint32_t i) { return geo.u16(geo.ent_off + 4ull * i); };
        auto lower = [&](std::uint32_t c) {  // first entry of the row with col >= c
            std::uint32_t a = rs, b = re;
            while (a < b) {
                const std::uint32_t mid = (a + b) >> 1;
                if (col_at(mid) < c) a = mid + 1; else b = mid;
            }
            return a;
        };
        lo = lower(256u * P);
        hi = lower(256u * P + 256u);
    }
    const std::uint32_t n = hi - lo;
    std::uint32_t incl = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const std::uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
    }
    const std::uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if constexpr (COUNT) {
        if (lane == 0) cnt[q] = total;
    } else {
        std::uint32_t* ent = reinterpret_cast<std::uint32_t*>(cells + cell_off[q] + cell_bytes);
        const std::uint32_t off = incl - n;
        for (std::uint32_t j = 0; j < n; ++j) {
            const std::uint32_t i = lo + j;
            const std::uint32_t col = geo.u16(geo.ent_off + 4ull * i), val = geo.u16(geo.ent_off + 4ull * i + 2);
            ent[off + j] = T::pack_entry(static_cast<std::uint32_t>(lane), col & 255u, static_cast<std::uint16_t>(val));
        }
        const std::uint32_t padded = (total + 3u) & ~3u;
        for (std::uint32_t i = total + lane; i < padded; i += 32) ent[i] = 0xffffffffu;
    }
}
