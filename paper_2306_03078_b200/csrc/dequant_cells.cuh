// dequant_cells.cuh -- bit-exact dequantize_full (kernel.hpp:17-25) straight
// from the tiled cell records (tiled.hpp), so a fast-path layer needs no raw
// stream copy in HBM.  Included by kernels.cuh (namespace spqr_dev).
//
// Reference semantics: reconstruct_solve_order (solver.hpp:345-362) -- per
// (block k, row r): s = stat_dequant(S_s, Z_s, scale code), z likewise
// (quantizer.hpp:65-67: S * (float(code) - Z), binary32), W = s * (q - z)
// (dequant_value, quantizer.hpp:60-62), then "+= fp16_to_float(v)" per
// outlier as a separate binary32 add -- and the column un-permute of
// dequantize_full, out(r, order[k]) = solve(r, k).  The same __fmul_rn /
// __fsub_rn / __fadd_rn sequence as dequant_raw, so the two agree bit for bit.
//
// One warp per unit (16 rows x 256 columns): lane (g, t) decodes the 8
// statistic code pairs of its lane field into (s, z) for rows g, g + 8 of
// blocks 8h + 2t + b and publishes them in a per-warp shared table; then it
// walks its A-fragment code pairs (the batch-1 layout: one LOP3-style mask of
// a window per pair, the code at bit offset p) and writes W two columns at a
// time.  The warp then adds the cell's outliers of its 16 rows in place.
// Write-bound: 4*m*n bytes out, the stream payload in.

template <int BW, int BS>
__global__ void __launch_bounds__(256) dequant_cells(const std::uint8_t* __restrict__ cells,
                                                     const std::uint32_t* __restrict__ cell_off, std::uint32_t Gn,
                                                     std::uint32_t Pn, std::uint32_t m, std::uint32_t n,
                                                     const std::uint32_t* __restrict__ order, float* __restrict__ w) {
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BS);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BS);
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr std::uint32_t SMASK = (1u << BS) - 1u;
    __shared__ float2 tab[8][16][17];  // per warp: (s, z) by [row in unit][block] (+1: bank spread)

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // unit index
    if (gw >= 2u * Gn * Pn) return;
    const std::uint32_t q = gw >> 1, ui = gw & 1u;
    const std::uint32_t Gq = q / Pn, Pq = q - Gq * Pn;
    const std::uint32_t r0 = __ldg(cell_off + q), r1 = __ldg(cell_off + q + 1);
    const std::uint8_t* unit = cells + r0 + ui * UNIT;
    const int g = lane >> 2, t = lane & 3;

    // code words first: their loads are in flight while the statistics decode
    std::uint32_t cw[G::LANE_WORDS];
#pragma unroll
    for (int i = 0; i < G::LANE_WORDS / 4; ++i) {
        const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(unit + lane * 16 * BW) + i);
        cw[4 * i] = w4.x;
        cw[4 * i + 1] = w4.y;
        cw[4 * i + 2] = w4.z;
        cw[4 * i + 3] = w4.w;
    }
    // this lane's first outlier entries (cells hold ~1 % outliers: one or two per lane)
    const std::uint32_t cnt = (r1 - r0 - CELL) / 4u;
    const std::uint32_t* ent = reinterpret_cast<const std::uint32_t*>(cells + r0 + CELL);
    constexpr int kE = 2;
    std::uint32_t e0[kE];
#pragma unroll
    for (int j = 0; j < kE; ++j) {
        const std::uint32_t i = static_cast<std::uint32_t>(lane) + 32u * j;
        e0[j] = i < cnt ? __ldg(ent + i) : 0xffffffffu;
    }

    // ---- statistics: this lane's 8 code pairs -> (s, z) of rows g, g + 8
    std::uint32_t sw[2];
    {
        const std::uint8_t* stats = unit + CODEB;
        if constexpr (BS == 3) {
            sw[0] = __ldg(reinterpret_cast<const std::uint32_t*>(stats) + lane);
            sw[1] = __byte_perm(__ldg(reinterpret_cast<const std::uint16_t*>(stats + 128) + lane), 0u, 0x4140);
        } else if constexpr (BS == 2) {
            sw[0] = __ldg(reinterpret_cast<const std::uint32_t*>(stats) + lane);
            sw[1] = 0u;
        } else {
            const uint2 v2 = __ldg(reinterpret_cast<const uint2*>(stats) + lane);
            sw[0] = v2.x;
            sw[1] = v2.y;
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int kk = 8 * h + 2 * t + b;
            const uint2 sc = __ldg(reinterpret_cast<const uint2*>(unit + CODEB + STATB) + kk);  // {S_s|Z_s, S_z|Z_z}
            float v[2][2];  // [kind][rho]
#pragma unroll
            for (int kind = 0; kind < 2; ++kind) {
                const int j = T::stat_pair(kind, h, b);
                const std::uint32_t win = window<2>(sw, T::stat_window(BS, j));
                const int p = T::stat_p(BS, j);
                const std::uint32_t SZ = kind ? sc.y : sc.x;
                const float S = h2f_bits(SZ & 0xffffu), Z = h2f_bits(SZ >> 16);
                v[kind][0] = __fmul_rn(S, __fsub_rn(static_cast<float>((win >> p) & SMASK), Z));
                v[kind][1] = __fmul_rn(S, __fsub_rn(static_cast<float>((win >> (16 + p)) & SMASK), Z));
            }
            tab[warp][g][kk] = make_float2(v[0][0], v[1][0]);
            tab[warp][g + 8][kk] = make_float2(v[0][1], v[1][1]);
        }
    __syncwarp();

    // ---- codes: A-fragment pairs -> W
    const std::uint32_t rowb = 32u * Gq + 16u * ui + static_cast<std::uint32_t>(g);
    const bool vec = order == nullptr && (n & 1u) == 0u;
#pragma unroll
    for (int mu = 0; mu < 16; ++mu) {
        const int cidx = mu / G::MPC, mm = mu % G::MPC;
        const std::uint32_t* wc = cw + G::CW * cidx;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
            const int i = rho * (G::NP / 2) + qq;
            const int B = (BW * i) >> 3, pb = (BW * i) & 7;
            const std::uint32_t win = window<G::CW>(wc, B);
            const float2 sz = tab[warp][g + 8 * rho][mu];
            const float v0 = __fmul_rn(sz.x, __fsub_rn(static_cast<float>((win >> pb) & MASK), sz.y));
            const float v1 = __fmul_rn(sz.x, __fsub_rn(static_cast<float>((win >> (16 + pb)) & MASK), sz.y));
            const std::uint32_t row = rowb + 8u * rho;
            const std::uint32_t col = 256u * Pq + 16u * mu + 2u * t + 8u * kh;
            if (row >= m) continue;
            float* wr = w + static_cast<std::uint64_t>(row) * n;
            if (vec && col + 1u < n) {
                *reinterpret_cast<float2*>(wr + col) = make_float2(v0, v1);
            } else {
                if (col < n) wr[order ? __ldg(order + col) : col] = v0;
                if (col + 1u < n) wr[order ? __ldg(order + col + 1u) : col + 1u] = v1;
            }
        }
    }
    __syncwarp();  // this warp's W stores before the outlier read-modify-writes

    // ---- outliers of this unit's 16 rows: a separate binary32 add (solver.hpp:360).
    // The lane's first kE entries: every old value is loaded before any add is
    // stored (latency once, not per entry) unless two of them hit the same
    // weight (then in entry order); the rest, rare, one at a time.
    auto target = [&](std::uint32_t e) -> float* {
        const std::uint32_t lr = e >> 24;  // 255: padding
        if ((lr >> 4) != ui) return nullptr;
        const std::uint32_t row = 32u * Gq + lr, col = 256u * Pq + ((e >> 16) & 255u);
        if (row >= m || col >= n) return nullptr;
        return w + static_cast<std::uint64_t>(row) * n + (order ? __ldg(order + col) : col);
    };
    float* pw[kE];
    float old[kE];
#pragma unroll
    for (int j = 0; j < kE; ++j) pw[j] = target(e0[j]);
    if (pw[0] != nullptr && pw[0] == pw[1]) {
        *pw[0] = __fadd_rn(*pw[0], h2f_bits(e0[0] & 0xffffu));
        *pw[1] = __fadd_rn(*pw[1], h2f_bits(e0[1] & 0xffffu));
    } else {
#pragma unroll
        for (int j = 0; j < kE; ++j) old[j] = pw[j] ? *pw[j] : 0.f;
#pragma unroll
        for (int j = 0; j < kE; ++j)
            if (pw[j]) *pw[j] = __fadd_rn(old[j], h2f_bits(e0[j] & 0xffffu));
    }
    for (std::uint32_t i = static_cast<std::uint32_t>(lane) + 32u * kE; i < cnt; i += 32u) {
        float* p = target(__ldg(ent + i));
        if (p) *p = __fadd_rn(*p, h2f_bits(__ldg(ent + i) & 0xffffu));
    }
}
