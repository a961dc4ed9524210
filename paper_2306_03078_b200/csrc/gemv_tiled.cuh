// gemv_tiled.cuh -- the fused SpQR decode-GEMV + CSR outlier merge (sm_100a).
// Included by kernels.cuh (inside namespace spqr_dev).
//
// Reference semantics: matvec(t, x, plan), kernel.hpp:89-124 --
//   y[r] = sum_k  s(k,r) * sum_{c in k} (q(r,c) - z(k,r)) * x[c]  +  sum_outliers v * x[col]
// computed here as, per (row, 16-column block k),
//   s*2^(24-e_k) * ( C + z * XX_k ),   C = sum_c (q_c 2^(p_c-24)) (x_c 2^(e_k-p_c))
// where C comes from an m16n8k16 f16 MMA with binary16-subnormal code operands
// (exact products, fp32 accumulate) and XX_k = -2^-24 sum_c x_c 2^e_k (xprep).
//
// Work: a persistent grid, one CTA per SM, NW warps per CTA; warp k streams a
// contiguous range of 32x256 cells (host-balanced by bytes incl. outliers)
// through its own TMA ring (cp.async.bulk + mbarrier, NSLOT cells in flight).
// Each slot receives the cell, the panel's prepared x operands and the cell's
// outlier entries, so the inner loop touches only shared memory and registers.
// MMA j of super-tile h routes block 8h+j to output column j by zeroing the B
// fragment in every lane but those with g == j, so the 8 MMAs of a super-tile
// accumulate into one C and each lane ends up holding 4 distinct
// (row, block) dot products -- one statistics decode per 16 weights.
// Outliers of a cell are merged by their row's owner lane (lane = local row).
// Rows split between warps are combined deterministically by the last arriving
// warp in warp order; every y row is written exactly once.

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

// code -> (2^23 + code) as float bits; fadd2 with -2^23 makes it exact.
__device__ __forceinline__ float magic_code(std::uint32_t v) { return __int_as_float(0x4B000000u | v); }

// Lane statistics field (SB bytes at 2-byte alignment) as two 32-bit words:
// s = bits [0, 32), z = bits [8*BS, 8*BS + 32) (all zero codes, aligned at 0).
template <int BS, int BZ>
__device__ __forceinline__ void load_stats(const std::uint8_t* p, std::uint32_t& s, std::uint32_t& z) {
    std::uint64_t v[2];
    load_stat_bits<BS + BZ>(p, v);
    s = static_cast<std::uint32_t>(v[0]);
    const int sh = 8 * BS;  // < 64
    z = static_cast<std::uint32_t>(v[0] >> sh);
    if constexpr (8 * BS + 8 * BZ > 64) z |= static_cast<std::uint32_t>(v[1] << (64 - sh));
}

template <int BW, int BS, int BZ, bool XLO, int NW, int NSLOT>
__global__ void __launch_bounds__(NW * 32, 1) gemv_tiled(const TiledParams p) {
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BZ);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BZ);
    constexpr std::uint32_t PANEL = T::panel_bytes(XLO);
    constexpr std::uint32_t O_FRAG = CELL, O_SC = CELL + T::kPanelFragBytes;
    constexpr std::uint32_t O_XP = O_SC + T::kPanelScBytes, O_LO = O_XP + T::kPanelXpBytes;
    constexpr std::uint32_t O_ENT = CELL + PANEL;
    constexpr int SB = BS + BZ;
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr float kMagic = 8388608.0f;

    extern __shared__ __align__(128) std::uint8_t smem[];
    __shared__ std::uint64_t bars[NW][NSLOT];
    __shared__ std::uint32_t slot_e[NW][NSLOT][2];
    __shared__ std::uint32_t heads[NW][32];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const std::uint32_t wk = blockIdx.x * NW + warp;
    const std::uint32_t q0 = p.warp_start[wk], q1 = p.warp_start[wk + 1];
    std::uint8_t* ring = smem + static_cast<std::size_t>(warp) * NSLOT * p.slot_bytes;

    if (lane == 0) {
        for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[warp][s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (q0 >= q1) {
        pdl_wait();
        return;
    }

    // per-cell outlier offsets, 32 cells at a time across the lanes
    std::uint32_t off_base = q0;
    std::uint32_t off_lane = (q0 + lane <= q1) ? __ldg(p.cell_off + q0 + lane) : 0u;
    auto cell_offset = [&](std::uint32_t q) -> std::uint32_t {  // monotone q, whole warp
        if (q >= off_base + 32) {
            off_base = q;
            off_lane = (q + lane <= q1) ? __ldg(p.cell_off + q + lane) : 0u;
        }
        return __shfl_sync(0xffffffffu, off_lane, static_cast<int>(q - off_base));
    };
    // Panel of cell q = q % Pn, tracked incrementally for the issue pointer.
    // weights + outlier entries of cell q into `slot` (arms the barrier for the
    // whole slot including the x panel, which issue_x adds)
    auto issue_w = [&](std::uint32_t q, int slot) {
        const std::uint32_t e0 = cell_offset(q), e1 = cell_offset(q + 1);
        if (lane == 0) {
            slot_e[warp][slot][0] = e0;
            slot_e[warp][slot][1] = e1;
            std::uint8_t* dst = ring + static_cast<std::size_t>(slot) * p.slot_bytes;
            std::uint32_t nb = 0, a0 = 0;
            if (e1 > e0) {
                a0 = (e0 * 4u) & ~15u;
                nb = min(((e1 * 4u + 15u) & ~15u) - a0, p.ent_cap_bytes);
            }
            std::uint64_t* bar = &bars[warp][slot];
            fence_proxy_async();
            mbar_expect_tx(bar, CELL + PANEL + nb);
            bulk_g2s(dst, p.cells + static_cast<std::size_t>(q) * CELL, CELL, bar);
            if (nb) bulk_g2s(dst + O_ENT, reinterpret_cast<const std::uint8_t*>(p.ent) + a0, nb, bar);
        }
    };
    // x operands of panel P (written by the preceding xprep kernel)
    auto issue_x = [&](std::uint32_t P, int slot) {
        if (lane == 0) {
            std::uint8_t* dst = ring + static_cast<std::size_t>(slot) * p.slot_bytes;
            std::uint64_t* bar = &bars[warp][slot];
            bulk_g2s(dst + O_FRAG, reinterpret_cast<const std::uint8_t*>(p.xfrag) + 512u * P, 512u, bar);
            bulk_g2s(dst + O_SC, reinterpret_cast<const std::uint8_t*>(p.xsc) + 128u * P, 128u, bar);
            bulk_g2s(dst + O_XP, reinterpret_cast<const std::uint8_t*>(p.xp) + 1024u * P, 1024u, bar);
            if constexpr (XLO)
                bulk_g2s(dst + O_LO, reinterpret_cast<const std::uint8_t*>(p.xlo) + 512u * P, 512u, bar);
        }
    };

    const std::uint32_t ncell = q1 - q0;
    // weights stream while the preceding xprep kernel is still running (PDL)
#pragma unroll 1
    for (int s = 0; s < NSLOT; ++s)
        if (static_cast<std::uint32_t>(s) < ncell) issue_w(q0 + s, s);
    pdl_wait();  // xprep has completed: x, partials and y are ours from here on
    {
        std::uint32_t Pi = q0 % p.Pn;
#pragma unroll 1
        for (int s = 0; s < NSLOT; ++s) {
            if (static_cast<std::uint32_t>(s) < ncell) issue_x(Pi, s);
            Pi = (Pi + 1 == p.Pn) ? 0u : Pi + 1;
        }
    }

    float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // [unit] = rows (g, g+8)
    float oacc = 0.f;  // outliers of local row `lane`
    std::uint32_t Gc = q0 / p.Pn, P = q0 - Gc * p.Pn;
    const std::uint32_t Gq0 = Gc;

    auto flush = [&](std::uint32_t Gf, bool whole) {
        float v[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            float a = acc[u].x, b = acc[u].y;
            a += __shfl_xor_sync(0xffffffffu, a, 1);
            b += __shfl_xor_sync(0xffffffffu, b, 1);
            a += __shfl_xor_sync(0xffffffffu, a, 2);
            b += __shfl_xor_sync(0xffffffffu, b, 2);
            v[u][0] = a;
            v[u][1] = b;
        }
        // lane R owns local row R = 16u + 8rho + gg; the value sits in lane 4gg
        const int R = lane, u = R >> 4, rho = (R >> 3) & 1, gg = R & 7;
        float mine = 0.f;
#pragma unroll
        for (int uu = 0; uu < 2; ++uu)
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const float o = __shfl_sync(0xffffffffu, v[uu][rr], gg * 4);
                if (uu == u && rr == rho) mine = o;
            }
        mine += oacc;
        oacc = 0.f;
        acc[0] = acc[1] = make_float2(0.f, 0.f);
        const std::uint32_t row = 32u * Gf + R;
        if (whole) {
            if (row < p.m) p.y[row] = mine;
            return;
        }
        const std::uint32_t side = (Gf == Gq0) ? 0u : 1u;
        p.partial[(wk * 2 + side) * 32 + R] = mine;
        __threadfence();
        __syncwarp();
        std::uint32_t prev = 0;
        if (lane == 0) prev = atomicAdd(p.counters + Gf, 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == __ldg(p.wcnt + Gf) - 1) {  // last contributor reduces in warp order
            __threadfence();
            float sum = 0.f;
            const std::uint32_t k1 = __ldg(p.wlast + Gf);
            for (std::uint32_t k = __ldg(p.wfirst + Gf); k <= k1; ++k) {
                const std::uint32_t s0 = __ldg(p.warp_start + k);
                if (s0 == __ldg(p.warp_start + k + 1)) continue;  // idle warp
                const std::uint32_t sk = (s0 / p.Pn == Gf) ? 0u : 1u;
                sum += __ldcg(p.partial + (k * 2 + sk) * 32 + R);
            }
            if (row < p.m) p.y[row] = sum;
            if (lane == 0) p.counters[Gf] = 0;
        }
    };

#pragma unroll 1
    for (std::uint32_t it = 0; it < ncell; ++it) {
        const std::uint32_t q = q0 + it;
        const int slot = static_cast<int>(it % NSLOT);
        const std::uint32_t phase = (it / NSLOT) & 1u;

        mbar_wait(&bars[warp][slot], phase);
        const std::uint8_t* cell = ring + static_cast<std::size_t>(slot) * p.slot_bytes;
        const std::uint32_t e0 = slot_e[warp][slot][0], e1 = slot_e[warp][slot][1];

        // x operands of this panel (shared by both units)
        uint2 xf[2], xl[2];
        float4 xs[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            xf[h] = reinterpret_cast<const uint2*>(cell + O_FRAG)[(8 * h + g) * 4 + t];
            if constexpr (XLO) xl[h] = reinterpret_cast<const uint2*>(cell + O_LO)[(8 * h + g) * 4 + t];
            xs[h] = reinterpret_cast<const float4*>(cell + O_SC)[4 * h + t];
        }

        // lane data of both units
        std::uint32_t cw[2][G::LANE_WORDS];
        std::uint32_t ss[2], zz[2];
        uint4 sc[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const std::uint8_t* unit = cell + u * UNIT;
#pragma unroll
            for (int i = 0; i < G::LANE_WORDS / 4; ++i) {
                const uint4 v = reinterpret_cast<const uint4*>(unit + lane * 16 * BW)[i];
                cw[u][4 * i] = v.x;
                cw[u][4 * i + 1] = v.y;
                cw[u][4 * i + 2] = v.z;
                cw[u][4 * i + 3] = v.w;
            }
            load_stats<BS, BZ>(unit + CODEB + lane * SB, ss[u], zz[u]);
            sc[u][0] = *reinterpret_cast<const uint4*>(unit + CODEB + STATB + (2 * t) * 8);
            sc[u][1] = *reinterpret_cast<const uint4*>(unit + CODEB + STATB + (8 + 2 * t) * 8);
        }

#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float c[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int mu = 8 * h + j, cidx = mu / G::MPC, mm = mu % G::MPC;
                const bool mine = (g == j);
                const std::uint32_t b0 = mine ? xf[h].x : 0u, b1 = mine ? xf[h].y : 0u;
                std::uint32_t l0 = 0, l1 = 0;
                if constexpr (XLO) {
                    l0 = mine ? xl[h].x : 0u;
                    l1 = mine ? xl[h].y : 0u;
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {  // two independent MMA chains
                    const std::uint32_t* w = cw[u] + G::CW * cidx;
                    std::uint32_t a[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
                        const int i = rho * (G::NP / 2) + qq;
                        const int B = (BW * i) >> 3, pp = (BW * i) & 7;
                        a[r] = window<G::CW>(w, B) & ((MASK << pp) * 0x00010001u);
                    }
                    mma16816(c[u], a, b0, b1);
                    if constexpr (XLO) mma16816(c[u], a, l0, l1);
                }
            }
            // epilogue: lane holds D(row g+8rho, block 8h+2t+bs) in c[u][2rho+bs]
#pragma unroll
            for (int bs = 0; bs < 2; ++bs) {
                const float scb = bs ? xs[h].z : xs[h].x, xxb = bs ? xs[h].w : xs[h].y;
                const int e0i = 4 * h + 2 * bs;  // entries eps = e0i + rho
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const std::uint32_t w01 = bs ? sc[u][h].z : sc[u][h].x;  // scale_s | scale_z
                    const std::uint32_t w23 = bs ? sc[u][h].w : sc[u][h].y;  // zero_s  | zero_z
                    const float2 S = __half22float2(*reinterpret_cast<const __half2*>(&w01));
                    const float2 Z = __half22float2(*reinterpret_cast<const __half2*>(&w23));
                    const float A1 = S.x * scb, A0 = -A1 * S.y, B0 = -Z.x * Z.y;
                    constexpr std::uint32_t SM = (1u << BS) - 1u, ZM = (1u << BZ) - 1u;
                    const float2 cs = fadd2(make_float2(magic_code((ss[u] >> (e0i * BS)) & SM),
                                                        magic_code((ss[u] >> ((e0i + 1) * BS)) & SM)),
                                            make_float2(-kMagic, -kMagic));
                    const float2 cz = fadd2(make_float2(magic_code((zz[u] >> (e0i * BZ)) & ZM),
                                                        magic_code((zz[u] >> ((e0i + 1) * BZ)) & ZM)),
                                            make_float2(-kMagic, -kMagic));
                    const float2 shat = ffma2(make_float2(A1, A1), cs, make_float2(A0, A0));
                    const float2 zhat = ffma2(make_float2(Z.x, Z.x), cz, make_float2(B0, B0));
                    const float2 tt = ffma2(zhat, make_float2(xxb, xxb), make_float2(c[u][bs], c[u][2 + bs]));
                    acc[u] = ffma2(shat, tt, acc[u]);
                }
            }
        }

        // outliers: lane R accumulates the entries of local row R (column order)
        const std::uint32_t cnt = e1 - e0;
        if (cnt) {
            const std::uint32_t lead = e0 * 4u - ((e0 * 4u) & ~15u);
            const std::uint32_t* es = reinterpret_cast<const std::uint32_t*>(cell + O_ENT + lead);
            const std::uint32_t got = min(((e1 * 4u + 15u) & ~15u) - (e0 * 4u - lead), p.ent_cap_bytes);
            const std::uint32_t in_smem = got > lead ? (got - lead) / 4u : 0u;
            const float* xpanel = reinterpret_cast<const float*>(cell + O_XP);
            auto merge = [&](auto entry) {
                heads[warp][lane] = cnt;
                __syncwarp();
                int last = -1;
#pragma unroll 1
                for (std::uint32_t base = 0; base < cnt; base += 32) {
                    const std::uint32_t i = base + lane;
                    const int r = i < cnt ? static_cast<int>(entry(i) >> 24) : 64;
                    int rp = __shfl_up_sync(0xffffffffu, r, 1);
                    if (lane == 0) rp = last;
                    if (i < cnt && r != rp) heads[warp][r] = i;
                    last = __shfl_sync(0xffffffffu, r, 31);
                }
                __syncwarp();
                std::uint32_t st = heads[warp][lane];
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {  // suffix minimum: first entry with row >= lane
                    const std::uint32_t o = __shfl_down_sync(0xffffffffu, st, d);
                    if (lane + d < 32) st = min(st, o);
                }
                std::uint32_t en = __shfl_down_sync(0xffffffffu, st, 1);
                if (lane == 31) en = cnt;
                std::uint32_t i = st;
                for (; i + 1 < en; i += 2) {
                    const std::uint32_t ea = entry(i), eb = entry(i + 1);
                    oacc = fmaf(h2f_bits(ea & 0xffffu), xpanel[(ea >> 16) & 255u], oacc);
                    oacc = fmaf(h2f_bits(eb & 0xffffu), xpanel[(eb >> 16) & 255u], oacc);
                }
                if (i < en) {
                    const std::uint32_t ea = entry(i);
                    oacc = fmaf(h2f_bits(ea & 0xffffu), xpanel[(ea >> 16) & 255u], oacc);
                }
            };
            if (cnt <= in_smem)
                merge([&](std::uint32_t i) { return es[i]; });
            else
                merge([&](std::uint32_t i) { return i < in_smem ? es[i] : __ldg(p.ent + e0 + i); });
        }

        __syncwarp();
        if (it + NSLOT < ncell) {
            issue_w(q + NSLOT, slot);
            std::uint32_t Pn_ = P + NSLOT;
            while (Pn_ >= p.Pn) Pn_ -= p.Pn;
            issue_x(Pn_, slot);
        }
        if (++P == p.Pn) {
            flush(Gc, Gc * p.Pn >= q0);
            P = 0;
            ++Gc;
        }
    }
    if (P != 0) flush(Gc, false);  // range ended inside row-group pair Gc
}
