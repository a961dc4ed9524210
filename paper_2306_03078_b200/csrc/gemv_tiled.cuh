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
// contiguous range of cell records (32x256 weights + that cell's outliers,
// host-balanced by bytes) through its own TMA ring (cp.async.bulk + mbarrier,
// NSLOT records in flight).  Each slot also receives the panel's prepared x
// operands, so the inner loop touches only shared memory and registers.
// MMA j of super-tile h routes block 8h+j to output column j by zeroing the B
// fragment in every lane but those with g == j, so the 8 MMAs of a super-tile
// accumulate into one C and each lane ends up holding 4 distinct
// (row, block) dot products -- one statistics decode per 16 weights.
// Outliers of a cell are merged by their row's owner lane (lane = local row).
// Rows split between warps are combined by the last arriving warp in warp
// order; every y row is written exactly once.

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
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

// The issue-rate budget is set by the ALU pipe (LOP3/SHF/SEL/PRMT issue at
// half rate per SMSP); the helpers below move what they can to the FMA pipe.

// w >> s as IMAD.HI (FMA pipe) instead of SHF (ALU pipe); s in [1, 31].
__device__ __forceinline__ std::uint32_t shr_fma(std::uint32_t w, int s) {
    std::uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(1u << (32 - s)));
    return r;
}
// a * m for m in {0, 1}: the B-fragment lane mask as IMAD (FMA pipe), not SEL.
__device__ __forceinline__ std::uint32_t mask01(std::uint32_t a, std::uint32_t m) {
    std::uint32_t r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(m));
    return r;
}
// ((w >> shift) & M) | 2^23-pattern: the code as the float 2^23 + code with
// ONE LOP3 (the exponent pattern lives in a register: LOP3 takes a single
// immediate).  `shift` is a compile-time constant after unrolling.
template <std::uint32_t M>
__device__ __forceinline__ float magic_field_rt(std::uint32_t w, int shift, std::uint32_t magic) {
    std::uint32_t r;
    const std::uint32_t x = shift ? shr_fma(w, shift) : w;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(x), "n"(M), "r"(magic));
    return __uint_as_float(r);
}

// Lane statistics field (tiled.hpp stat_byte_offset) as two 32-bit words:
// s = bits [0, 32) (scale codes), z = bits [8*BS, 8*BS + 32) (zero codes).
template <int BS, int BZ>
__device__ __forceinline__ void load_stats(const std::uint8_t* stats, int lane, std::uint32_t& s, std::uint32_t& z) {
    constexpr int SB = BS + BZ;
    if constexpr (SB > 4 && SB < 8) {  // 4-byte plane + (SB-4)-byte plane
        static_assert(SB == 6, "only 3/3-bit statistics use the split planes on the fast path");
        const std::uint32_t w0 = reinterpret_cast<const std::uint32_t*>(stats)[lane];
        const std::uint32_t w1 = reinterpret_cast<const std::uint16_t*>(stats + 128)[lane];
        s = w0;
        z = __funnelshift_r(w0, w1, 8 * BS);
    } else {
        std::uint64_t v[2];
        load_stat_bits<SB>(stats + lane * SB, v);
        s = static_cast<std::uint32_t>(v[0]);
        const int sh = 8 * BS;  // < 64
        z = static_cast<std::uint32_t>(v[0] >> sh);
        if constexpr (8 * BS + 8 * BZ > 64) z |= static_cast<std::uint32_t>(v[1] << (64 - sh));
    }
}

#ifdef SPQR_TIMELINE
// tools-only instrumentation (tools/timeline_dev.py): per warp %globaltimer at
// entry, after the PDL wait, first cell staged, loop end, exit.
__device__ unsigned long long g_timeline[148 * 32 * 8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SPQR_TL(k) \
    if (lane == 0 && wk < 148 * 32) g_timeline[8 * wk + (k)] = gtime();
#else
#define SPQR_TL(k)
#endif

template <int BW, int BS, int BZ, bool XLO, int NW, int NSLOT>
__global__ void __launch_bounds__(NW * 32, 1) gemv_tiled(const TiledParams p) {
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BZ);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BZ);
    constexpr std::uint32_t PANEL = T::panel_bytes(XLO);
    constexpr std::uint32_t O_FRAG = 0, O_SC = T::kPanelFragBytes, O_XP = O_SC + T::kPanelScBytes;
    constexpr std::uint32_t O_LO = O_XP + 256u * (XLO ? 4u : 2u);
    constexpr std::uint32_t O_REC = PANEL;  // cell record follows the panel in a slot
    constexpr int SB = BS + BZ;
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr std::uint32_t SMASK = (1u << BS) - 1u, ZMASK = (1u << BZ) - 1u;
    constexpr float kMagic = 8388608.0f;

    extern __shared__ __align__(128) std::uint8_t smem[];
    __shared__ std::uint64_t bars[NW][NSLOT];
    __shared__ std::uint32_t slot_r[NW][NSLOT][2];  // record byte range of the slot's cell
    __shared__ float rowsum[NW][32];                 // outlier row sums of a cell (zero between cells)
    __shared__ __align__(16) std::uint32_t zrow[NW][4];  // 16 zero bytes: masked ldmatrix rows

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const std::uint32_t wk = blockIdx.x * NW + warp;
    const std::uint32_t q0 = p.warp_start[wk], q1 = p.warp_start[wk + 1];
    std::uint8_t* ring = smem + static_cast<std::size_t>(warp) * NSLOT * p.slot_bytes;
    SPQR_TL(0)

    // the next layer's xprep may launch now; it reads x only after this grid
    // has completed (its griddepcontrol.wait), so the tails of consecutive
    // layers overlap
    pdl_launch();
    if (lane == 0) {
        for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[warp][s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (q0 >= q1) {
        pdl_wait();
        return;
    }

    // TMA issue state, lane 0 only: record offsets of the next cell to issue
    // (r0, r1) and the one after (prefetched a full cell ahead), its panel.
    const std::uint32_t ncell = q1 - q0;
    std::uint32_t i_q = q0, i_r0 = 0, i_r1 = 0, i_nx = 0, i_P = 0;
    std::uint32_t Gc = q0 / p.Pn, P = q0 - Gc * p.Pn;
    if (lane == 0) {
        i_r0 = __ldg(p.cell_off + q0);
        i_r1 = __ldg(p.cell_off + q0 + 1);
        i_nx = (q0 + 2 <= q1) ? __ldg(p.cell_off + q0 + 2) : 0u;
        i_P = P;
    }
    auto issue_rec = [&](int slot) {  // lane 0: cell i_q -> slot, arms the barrier for record + panel
        slot_r[warp][slot][0] = i_r0;
        slot_r[warp][slot][1] = i_r1;
        const std::uint32_t nb = min(i_r1 - i_r0, p.rec_cap_bytes);
        std::uint64_t* bar = &bars[warp][slot];
        mbar_expect_tx(bar, PANEL + nb);
        bulk_g2s(ring + static_cast<std::size_t>(slot) * p.slot_bytes + O_REC, p.cells + i_r0, nb, bar);
        ++i_q;
        i_r0 = i_r1;
        i_r1 = i_nx;
        i_nx = (i_q + 2 <= q1) ? __ldg(p.cell_off + i_q + 2) : 0u;
    };
    auto issue_x = [&](int slot) {  // lane 0: x operands of panel i_P (written by xprep)
        bulk_g2s(ring + static_cast<std::size_t>(slot) * p.slot_bytes, p.xpanel + PANEL * i_P, PANEL,
                 &bars[warp][slot]);
        i_P = (i_P + 1 == p.Pn) ? 0u : i_P + 1;
    };

    // weights stream while the preceding xprep kernel is still running (PDL)
    if (lane == 0) {
#pragma unroll 1
        for (int s = 0; s < NSLOT; ++s)
            if (static_cast<std::uint32_t>(s) < ncell) issue_rec(s);
    }
    pdl_wait();  // xprep has completed: x panels, partials and y are ours from here on
    SPQR_TL(1)
    if (lane == 0) {
#pragma unroll 1
        for (int s = 0; s < NSLOT; ++s)
            if (static_cast<std::uint32_t>(s) < ncell) issue_x(s);
    }

    float2 acc[2][2];  // [unit][rho] = (block 2t, block 2t+1) partials of row g + 8 rho
#pragma unroll
    for (int u = 0; u < 2; ++u) acc[u][0] = acc[u][1] = make_float2(0.f, 0.f);
    const std::uint32_t Gq0 = Gc;
    const std::uint32_t magic = 0x4B000000u;
    // ldmatrix row addresses for the masked B operand: MMA j of a super-tile
    // routes block j to output column j, so B^T row n is block j's x when
    // n == j and zero otherwise.  Call c loads MMAs 2c, 2c+1 (x4: k halves).
    // Lane (lm, lr) = (lane / 8, lane % 8) addresses row lr of matrix lm; it
    // carries data only in the call whose MMA j + lm/2 == lr, i.e. j == jact,
    // and then always the same 16 bytes of the panel (block 8h + lr, k half
    // lm % 2), at a fixed lane offset -- the per-call offset 256h is an
    // immediate, so the zero row is pre-biased by -256h.
    const int lm = lane >> 3, lr = lane & 7;
    const int jact = lr - (lm >> 1);
    const std::uint32_t lane_off = O_FRAG + 32u * lr + 16u * (lm & 1);
    const std::uint32_t zero_sa = smem_u32(&zrow[warp][0]);
    const std::uint32_t zb[2] = {zero_sa, zero_sa - 256u};
    const std::uint32_t zl[2] = {zero_sa - (O_LO - O_FRAG), zero_sa - 256u - (O_LO - O_FRAG)};
    if (lane < 4) zrow[warp][lane] = 0u;
    rowsum[warp][lane] = 0.f;
    __syncwarp();
#ifdef SPQR_TIMELINE
    std::uint32_t r_last_cnt = 0;
#endif
    float orow_reg = 0.f;  // outlier sum of local row `lane` (current row-group pair)

    auto flush = [&](std::uint32_t Gf, bool whole) {
        float v[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                float a = acc[u][r].x + acc[u][r].y;
                a += __shfl_xor_sync(0xffffffffu, a, 1);
                a += __shfl_xor_sync(0xffffffffu, a, 2);
                v[u][r] = a;
                acc[u][r] = make_float2(0.f, 0.f);
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
        mine += orow_reg;
        orow_reg = 0.f;
        const std::uint32_t row = 32u * Gf + R;
        if (whole) {
            if (row < p.m) p.y[row] = mine;
            return;
        }
        // split row-group pair: contributor slot = pbase[G] + this warp's ordinal
        const uint2 gm = __ldg(reinterpret_cast<const uint2*>(p.gmap) + Gf);  // {pbase, count}
        const std::uint32_t ord = __ldg(p.wmap + 2 * wk + ((Gf == Gq0) ? 0u : 1u));
        p.partial[(gm.x + ord) * 32 + R] = mine;
        __syncwarp();
        std::uint32_t prev = 0;
        if (lane == 0) {  // release our partial, acquire the others'
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.counters + Gf) : "memory");
        }
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == gm.y - 1) {  // last contributor: reduce in contributor (warp) order
            __syncwarp();
            float sum = 0.f;
            const float* src = p.partial + gm.x * 32 + R;
            std::uint32_t j = 0;
            for (; j + 4 <= gm.y; j += 4) {
                const float a = __ldcg(src + 32 * j), b = __ldcg(src + 32 * (j + 1));
                const float c = __ldcg(src + 32 * (j + 2)), d = __ldcg(src + 32 * (j + 3));
                sum += a;
                sum += b;
                sum += c;
                sum += d;
            }
            for (; j < gm.y; ++j) sum += __ldcg(src + 32 * j);
            if (row < p.m) p.y[row] = sum;
            if (lane == 0) p.counters[Gf] = 0;
        }
    };

#pragma unroll 1
    for (std::uint32_t it = 0; it < ncell; ++it) {
        const int slot = static_cast<int>(it % NSLOT);
        const std::uint32_t phase = (it / NSLOT) & 1u;

        mbar_wait(&bars[warp][slot], phase);
#ifdef SPQR_TIMELINE
        if (it == 0) SPQR_TL(2)
#endif
        const std::uint8_t* sl = ring + static_cast<std::size_t>(slot) * p.slot_bytes;
        const std::uint8_t* cell = sl + O_REC;
        const std::uint32_t r0 = slot_r[warp][slot][0], r1 = slot_r[warp][slot][1];

        // x operands of this panel (shared by both units)
        float4 xs[2];  // {SC(2t), SC(2t+1), XX(2t), XX(2t+1)} of super-tile h
#pragma unroll
        for (int h = 0; h < 2; ++h) xs[h] = reinterpret_cast<const float4*>(sl + O_SC)[4 * h + t];
        const std::uint32_t lane_sa = smem_u32(sl) + lane_off;

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
            load_stats<BS, BZ>(unit + CODEB, lane, ss[u], zz[u]);
            sc[u][0] = *reinterpret_cast<const uint4*>(unit + CODEB + STATB + (2 * t) * 8);
            sc[u][1] = *reinterpret_cast<const uint4*>(unit + CODEB + STATB + (8 + 2 * t) * 8);
        }

        // 4 independent MMA chains (super-tile h x unit u), interleaved
        std::uint32_t bfr[2][4], lfr[2][4];
        float cc[2][2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int i = 0; i < 4; ++i) cc[h][u][i] = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int mu = 8 * h + j, cidx = mu / G::MPC, mm = mu % G::MPC;
                // B fragments of MMAs (2c, 2c+1), c = j/2, fetched at the even j
                std::uint32_t bq[4], lq[4];
                if ((j & 1) == 0) {
                    const bool act = jact == j;
                    ldsm_x4((act ? lane_sa : zb[h]) + 256u * h, bq);  // constant offset folds into LDSM
                    if constexpr (XLO) ldsm_x4((act ? lane_sa : zl[h]) + (256u * h + (O_LO - O_FRAG)), lq);
                    bfr[h][0] = bq[0]; bfr[h][1] = bq[1]; bfr[h][2] = bq[2]; bfr[h][3] = bq[3];
                    if constexpr (XLO) {
                        lfr[h][0] = lq[0]; lfr[h][1] = lq[1]; lfr[h][2] = lq[2]; lfr[h][3] = lq[3];
                    }
                }
                const std::uint32_t b0 = bfr[h][2 * (j & 1)], b1 = bfr[h][2 * (j & 1) + 1];
                std::uint32_t l0 = 0, l1 = 0;
                if constexpr (XLO) {
                    l0 = lfr[h][2 * (j & 1)];
                    l1 = lfr[h][2 * (j & 1) + 1];
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const std::uint32_t* w = cw[u] + G::CW * cidx;
                    std::uint32_t a[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
                        const int i = rho * (G::NP / 2) + qq;
                        const int B = (BW * i) >> 3, pp = (BW * i) & 7;
                        a[r] = window<G::CW>(w, B) & ((MASK << pp) * 0x00010001u);
                    }
                    mma16816(cc[h][u], a, b0, b1);
                    if constexpr (XLO) mma16816(cc[h][u], a, l0, l1);
                }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float (&c)[2][4] = cc[h];
            // epilogue: lane holds D(row g+8rho, block 8h+2t+bs) in c[u][2rho+bs];
            // everything is paired over bs = (block 2t, block 2t+1)
            const float2 SC = make_float2(xs[h].x, xs[h].y), XX = make_float2(xs[h].z, xs[h].w);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint4 s4 = sc[u][h];  // {scale_s|scale_z, zero_s|zero_z} x 2 blocks
                const __half2 s0 = u32_as_h2(s4.x), z0 = u32_as_h2(s4.y), s1 = u32_as_h2(s4.z), z1 = u32_as_h2(s4.w);
                const float2 Ss = make_float2(__low2float(s0), __low2float(s1));
                const float2 Zs = make_float2(__high2float(s0), __high2float(s1));
                const float2 Sz = make_float2(__low2float(z0), __low2float(z1));
                const float2 Zz = make_float2(-__high2float(z0), -__high2float(z1));
                const float2 A1 = fmul2(Ss, SC);                             // s_s * 2^(24-e)
                const float2 A0 = fmul2(A1, make_float2(-Zs.x, -Zs.y));      // -s_s z_s 2^(24-e)
                const float2 B0 = fmul2(Sz, Zz);                             // -z_s z_z
#pragma unroll
                for (int rho = 0; rho < 2; ++rho) {
                    const int e0i = 4 * h + rho, e1i = 4 * h + 2 + rho;  // eps of (bs=0, bs=1)
                    const float2 cs = fadd2(make_float2(magic_field_rt<SMASK>(ss[u], e0i * BS, magic),
                                                        magic_field_rt<SMASK>(ss[u], e1i * BS, magic)),
                                            make_float2(-kMagic, -kMagic));
                    const float2 cz = fadd2(make_float2(magic_field_rt<ZMASK>(zz[u], e0i * BZ, magic),
                                                        magic_field_rt<ZMASK>(zz[u], e1i * BZ, magic)),
                                            make_float2(-kMagic, -kMagic));
                    const float2 shat = ffma2(A1, cs, A0);
                    const float2 zhat = ffma2(Sz, cz, B0);
                    const float2 tt = ffma2(zhat, XX, make_float2(c[u][2 * rho], c[u][2 * rho + 1]));
                    acc[u][rho] = ffma2(shat, tt, acc[u][rho]);
                }
            }
        }

        // outliers: entries (row, col, value) of this cell, sorted by (row, col),
        // 0xffffffff padding (row 255).  Chunks of 128 entries, 4 consecutive
        // per lane (one 16-byte load): products, a segmented inclusive scan by
        // row (in-lane, then across lanes by the lanes' last row), and the
        // last entry of each row in the chunk adds the row total to rowsum.
        // Chunks run in order, so the sums are deterministic.  Entries beyond
        // the staged part of the record are read from global memory.
        const std::uint32_t cnt = (r1 - r0 - CELL) / 4u;
#ifdef SPQR_TIMELINE
        r_last_cnt += cnt;
#endif
        if (cnt) {
            const std::uint32_t nfast = (min(r1 - r0, p.rec_cap_bytes) - CELL) / 4u;
            const std::uint32_t* es = reinterpret_cast<const std::uint32_t*>(cell + CELL);  // in our slot
            const std::uint32_t* eg = reinterpret_cast<const std::uint32_t*>(p.cells + r0 + CELL) + nfast;
            float* rs = rowsum[warp];
            auto chunk = [&](const std::uint32_t* src, std::uint32_t i0, std::uint32_t lim, bool first) {
                uint4 ev = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                if (i0 < lim) ev = *reinterpret_cast<const uint4*>(src + i0);  // lim % 4 == 0
                const std::uint32_t e[4] = {ev.x, ev.y, ev.z, ev.w};
                std::uint32_t k[4];
                float sv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    k[j] = e[j] >> 24;
                    const std::uint32_t c = (e[j] >> 16) & 255u;
                    float xv;
                    if constexpr (XLO)
                        xv = reinterpret_cast<const float*>(sl + O_XP)[c];
                    else
                        xv = __half2float(reinterpret_cast<const __half*>(sl + O_XP)[c]);
                    sv[j] = h2f_bits(e[j] & 0xffffu) * xv;
                }
                bool same[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    same[j] = k[j + 1] == k[j];
                    if (same[j]) sv[j + 1] += sv[j];
                }
                // across lanes: segments of equal last-row keys (sorted => contiguous)
                const std::uint32_t K = k[3];
                const std::uint32_t pK = __shfl_up_sync(0xffffffffu, K, 1);
                const bool head = lane == 0 || pK != K;
                const std::uint32_t heads = __ballot_sync(0xffffffffu, head) & (0xffffffffu >> (31 - lane));
                const int seg0 = 31 - __clz(heads);
                float V = sv[3];
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const float o = __shfl_up_sync(0xffffffffu, V, d);
                    if (lane - d >= seg0) V += o;
                }
                float cin = __shfl_up_sync(0xffffffffu, V, 1);
                if (lane == 0 || pK != k[0]) cin = 0.f;
                const std::uint32_t nk0 = __shfl_down_sync(0xffffffffu, k[0], 1);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool tail = (j < 3) ? !same[j] : (lane == 31 || nk0 != k[3]);
                    if (tail && k[j] < 32u) {
                        const float tot = (k[j] == k[0]) ? sv[j] + cin : sv[j];
                        if (first)
                            rs[k[j]] = tot;
                        else
                            rs[k[j]] += tot;
                    }
                }
            };
            chunk(es, 4u * lane, nfast, true);
#pragma unroll 1
            for (std::uint32_t base = 128; base < nfast; base += 128) {
                __syncwarp();
                chunk(es, base + 4u * lane, nfast, false);
            }
#pragma unroll 1
            for (std::uint32_t base = nfast; base < cnt; base += 128) {  // rare: record larger than the slot
                __syncwarp();
                chunk(eg, base - nfast + 4u * lane, cnt - nfast, false);  // eg starts at entry nfast
            }
            __syncwarp();
            orow_reg += rs[lane];
            rs[lane] = 0.f;
        }

        __syncwarp();  // every lane is done with the slot
        if (lane == 0 && it + NSLOT < ncell) {
            issue_rec(slot);
            issue_x(slot);
        }
        if (++P == p.Pn) {
            flush(Gc, Gc * p.Pn >= q0);
            P = 0;
            ++Gc;
        }
    }
    SPQR_TL(3)
#ifdef SPQR_TIMELINE
    if (lane == 0) {
        unsigned smid;
        asm("mov.u32 %0, %smid;" : "=r"(smid));
        g_timeline[8 * wk + 5] = ncell;
        g_timeline[8 * wk + 6] = smid;
        g_timeline[8 * wk + 7] = r_last_cnt;
    }
#endif
    if (P != 0) flush(Gc, false);  // range ended inside row-group pair Gc
    SPQR_TL(4)
}
