// gemv_cta.cuh -- the fused SpQR decode-GEMV + CSR outlier merge, v14
// (sm_100a).  Included by kernels.cuh (inside namespace spqr_dev).
//
// Reference semantics: matvec(t, x, plan), kernel.hpp:89-124 (x gather through
// the permutation :93-98, per-tile dequant :100-111, CSR slices :112-120) --
//   y[r] = sum_k  s(k,r) * sum_{c in k} (q(r,c) - z(k,r)) * x[c]  +  sum_outliers v * x[col]
// The first-level statistics are stat_dequant (quantizer.hpp:65-67) of 3-bit
// codes under binary16 second-level scalars (solver.hpp:129-141).
//
// Per (row, 16-column block k) of a cell, in registers:
//   C      = sum_c (q_c 2^(p_c-24)) B_c                   m16n8k16 f16 MMA, exact products
//   s'     = S_s * (cs 2^(p_s-24)) - S_s Z_s 2^(p_s-24)    one fma.rn.f32.f16 (FHFMA)
//   z'     = S_z * (cz 2^(p_z-24)) - S_z Z_z 2^(p_z-24)    one FHFMA
//   acc   += s' * (C + z' XX_k)                            two packed f32x2 FMAs per 2 blocks
// with B_c = x_c 2^(e - p_c - p_s(k)) (fp16) and XX_k = -2^(-p_z(k)) sum_c B_c 2^p_c,
// so s'(C + z' XX) = 2^(e-48) s (sum_c (q_c - z) x_c): one power of two per
// panel (SC = 2^(48-e)) turns a cell's row sums into y.  The statistic codes
// arrive as binary16 subnormals straight from one LOP3 of their lane field
// (tiled.hpp), the -S Z 2^(p-24) terms come from a per-warp table each lane
// fills one entry of, so a (row, block) costs ~4 instructions.
//
// Structure (one CTA per SM, NC warps):
//  * the host cuts the cell sequence (row-major 32x256 cells) into contiguous
//    byte-balanced ranges, one per CTA (more only when a range's row-sum array
//    would not fit shared memory);
//  * warps take cells dynamically (a shared ticket counter) and hold one
//    ticket of lookahead whose record copy (cp.async.bulk, mbarrier) is in
//    flight while the current cell computes; the first records go out before
//    the preceding kernel has finished (PDL: weights do not depend on it);
//  * x panels (gather through the permutation, per-panel power-of-two scale,
//    per-column pre-scales, block sums) are built after the PDL wait: once
//    per CTA into shared memory when all Pn panels fit (SHX), else per cell;
//  * per cell the warp writes 32 row sums (MMA part + outliers) to a per-CTA
//    array and counts the cell against its row-group pair; the warp that
//    completes a pair adds its cells in cell order and writes y.  A pair
//    shared with the neighbouring range (ranges hold >= Pn cells, so at most
//    two share a pair) is finished by whichever side completes second: both
//    store their partial rows to a global slot, the second arriver (atomic
//    ticket) adds first-side + last-side and resets the ticket -- no CTA ever
//    waits for another, so launches need not be co-resident.
//  * GATHER = true (row-sharded decode, gather.cu): every y row is also stored
//    into the other ranks' full-y buffers; the grid's last CTA bumps this
//    rank's round counter on every rank and waits until every rank's counter
//    reached the round (the all-gather's wait, fused: no second launch).
// Every reduction order is fixed by the partition, not by the schedule, so y
// is bitwise reproducible run to run.

constexpr int kQFirst = 161;
constexpr int kMaxPeers = 7;  // 8 ranks per node
struct CtaParams {
    const std::uint8_t* cells;        // cell records
    const std::uint32_t* cell_off;    // [ncell+1]
    const std::uint32_t* cta_start;   // [nvcta+1] first cell of each range
    const void* x;                    // this batch column, original column order (f16 or f32)
    const std::uint32_t* order;       // solve position -> source column, or null
    float* y;                         // [m] this batch column
    float* xpart;                     // [nvcta+1][2][32] partial rows of pairs shared by two ranges
    std::uint32_t* xcnt;              // [nvcta+1] arrivals per shared pair (zero between launches)
    std::uint32_t m, n, Pn, Gn, nvcta;
    std::uint32_t pn_magic;           // q / Pn == umulhi(q, pn_magic) for every cell index q
    std::uint32_t rec_cap, slot_bytes;
    std::uint32_t pan_off, part_off, off_off, gd_off, part_cap;
    std::uint32_t x_vec;              // x is 16-B aligned and not permuted: vector loads
    const uint2* first_rec;           // [grid][NC] {r0, r1}: record of warp w's first cell (r0 == r1: none)
    // cta_start[0 .. grid] by value (grid < kQFirst): the first range's bounds
    // come from the parameter bank, not from HBM while the preceding kernel
    // saturates it
    std::uint32_t q_first[kQFirst];
    // Fused all-gather (row-sharded decode): every final y row
    // is also stored into the full-y buffers of the npeer other ranks (P2P /
    // NVLink addresses from CUDA IPC) at row_base + row; after the grid's last
    // y store the last CTA to finish bumps this rank's counter on every rank
    // (pflags[j][rank], world entries including itself).  npeer == 0 and
    // pflags == null: a plain matvec.
    float* ypeer[kMaxPeers];
    std::uint32_t* pflags[kMaxPeers + 1];
    std::uint32_t* done_ctr;          // CTAs finished this round (last one resets it)
    std::uint32_t npeer, nflag, row_base, rank;
    // Before storing round R into peer j's y, a CTA waits until peer j's band
    // kernel of round R has started (started[j] >= R in this rank's block,
    // posted by j): everything peer j's stream ordered before that kernel --
    // its consumers of y from round R-1 -- is then complete, so a rank running
    // one round ahead never overwrites rows a peer is still reading.
    const std::uint32_t* round;       // this rank's completed rounds (the grid's last CTA advances it)
    const std::uint32_t* started;     // [world] in this rank's block: peer j's latest started round
};
constexpr std::uint32_t kGatherStartedWord = 32;  // started[] at byte 128 of a gather block

__device__ __forceinline__ void bar_sync_named(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ std::uint32_t pack_h2_rn(float lo, float hi) {
    std::uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// a * b + c with a = half HA of a2, b = half HB of b2 (binary16), c and the
// result binary32: one FHFMA (mixed-precision fma.rn.f32.f16, sm_100); the
// product of two binary16 values is exact, so the result is rounded once.
template <int HA, int HB>
__device__ __forceinline__ float fhfma(std::uint32_t a2, std::uint32_t b2, float c) {
    float d;
    if constexpr (HA == 0 && HB == 0)
        asm("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
            "fma.rn.f32.f16 %0, al, bl, %3;\n\t}"
            : "=f"(d) : "r"(a2), "r"(b2), "f"(c));
    else if constexpr (HA == 0 && HB == 1)
        asm("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
            "fma.rn.f32.f16 %0, al, bh, %3;\n\t}"
            : "=f"(d) : "r"(a2), "r"(b2), "f"(c));
    else if constexpr (HA == 1 && HB == 0)
        asm("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
            "fma.rn.f32.f16 %0, ah, bl, %3;\n\t}"
            : "=f"(d) : "r"(a2), "r"(b2), "f"(c));
    else
        asm("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
            "fma.rn.f32.f16 %0, ah, bh, %3;\n\t}"
            : "=f"(d) : "r"(a2), "r"(b2), "f"(c));
    return d;
}
__device__ __forceinline__ float pow2f(int k) {  // 2^k for k in [-126, 127]
    return __uint_as_float(static_cast<std::uint32_t>(127 + k) << 23);
}

// Pre-scales of a panel column (block kk of the panel, column cc in the block):
// the weight code's (p_c) and the block's scale / zero code pairs' (p_s, p_z).
template <int BW, int BS>
__device__ __forceinline__ void column_scales(std::uint32_t kk, std::uint32_t cc, int& pc, int& ps, int& pz) {
    pc = T::column_prescale(BW, kk, cc);
    const int h = static_cast<int>((kk >> 3) & 1u), b = static_cast<int>(kk & 1u);
    ps = T::stat_p(BS, T::stat_pair(0, h, b));
    pz = T::stat_p(BS, T::stat_pair(1, h, b));
}

// One lane's share of a cell's x panel: columns 8*lane .. 8*lane+7 of panel P
// (block kk = lane/2, half hf = lane%2).  load_x fetches them (through the
// permutation, zero beyond n); build_panel writes the panel (tiled.hpp).
// x modes (template XM): 0 = fp16 x, one column; 1 = fp32 x, one column as
// fp16 hi + lo parts sharing each MMA; 2 = fp16 x, two batch columns sharing
// each MMA (the batch-2 pass: every weight decoded once for both columns).
template <int XM>
struct XLane {
    std::uint32_t w[XM ? 8 : 4];  // fp16 pairs (mode 2: column 0 then column 1), or fp32 bit patterns
};

__device__ __forceinline__ void load_x_f16(const CtaParams& p, const void* xs, std::uint32_t c0, std::uint32_t* w) {
    if (p.x_vec && c0 + 8u <= p.n) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(static_cast<const __half*>(xs) + c0));
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
        std::uint32_t h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const std::uint32_t c = c0 + i;
            h[i] = 0;
            if (c < p.n) h[i] = __ldg(static_cast<const unsigned short*>(xs) + (p.order ? __ldg(p.order + c) : c));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = h[2 * i] | (h[2 * i + 1] << 16);
    }
}

template <int XM>
__device__ __forceinline__ XLane<XM> load_x(const CtaParams& p, std::uint32_t P, int lane) {
    XLane<XM> r;
    const std::uint32_t c0 = 256u * P + 8u * static_cast<std::uint32_t>(lane);
    if constexpr (XM == 0) {
        load_x_f16(p, p.x, c0, r.w);
    } else if constexpr (XM == 2) {  // batch columns 0 and 1 (x is batch x n)
        load_x_f16(p, p.x, c0, r.w);
        load_x_f16(p, static_cast<const __half*>(p.x) + p.n, c0, r.w + 4);
    } else {
        if (p.x_vec && c0 + 8u <= p.n) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(static_cast<const float*>(p.x) + c0));
            const uint4 b = __ldg(reinterpret_cast<const uint4*>(static_cast<const float*>(p.x) + c0 + 4));
            r.w[0] = a.x; r.w[1] = a.y; r.w[2] = a.z; r.w[3] = a.w;
            r.w[4] = b.x; r.w[5] = b.y; r.w[6] = b.z; r.w[7] = b.w;
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const std::uint32_t c = c0 + i;
                r.w[i] = 0;
                if (c < p.n) r.w[i] = __ldg(static_cast<const unsigned*>(p.x) + (p.order ? __ldg(p.order + c) : c));
            }
        }
    }
    return r;
}

// One column's panel operands (B rows at o_frag, XX, SC, x in solve order at
// o_xp; XLO: fp32 x, its residual B rows at o_lo).
template <int BW, int BS, bool XLO>
__device__ __forceinline__ void build_col(const std::uint32_t* xw, int lane, std::uint8_t* pan, std::uint32_t o_frag,
                                          std::uint32_t o_xx, std::uint32_t o_sc, std::uint32_t o_xp,
                                          std::uint32_t o_lo) {
    const std::uint32_t kk = static_cast<std::uint32_t>(lane) >> 1, cc = 8u * (lane & 1);
    int pc, ps, pz;
    column_scales<BW, BS>(kk, cc, pc, ps, pz);
    float f[8];
    if constexpr (!XLO) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 v = __half22float2(u32_as_h2(xw[i]));
            f[2 * i] = v.x;
            f[2 * i + 1] = v.y;
        }
        *reinterpret_cast<uint4*>(pan + o_xp + 16u * lane) = make_uint4(xw[0], xw[1], xw[2], xw[3]);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(xw[i]);
        uint4* xp = reinterpret_cast<uint4*>(pan + o_xp + 32u * lane);
        xp[0] = make_uint4(xw[0], xw[1], xw[2], xw[3]);
        xp[1] = make_uint4(xw[4], xw[5], xw[6], xw[7]);
    }
    // the panel's scale: max |x| 2^e in [2^14, 2^15)
    float mx = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) mx = fmaxf(mx, fabsf(f[i]));
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    int e = 0;
    if (mx > 0.f && mx < INFINITY) {
        const std::uint32_t eb = __float_as_uint(mx) >> 23;
        int E = static_cast<int>(eb) - 126;  // mx = m 2^E, m in [0.5, 1)
        if (XLO && eb == 0u) frexpf(mx, &E);  // fp32 subnormal max
        e = 15 - E;
    }
    // B = x 2^(e - pc - ps): fp16 x keeps e - pc - ps in [-15, 38]; fp32 x may
    // need two factors at the ends of the exponent range
    const int k = e - pc - ps;
    const int k1 = k < -126 ? -126 : (k > 127 ? 127 : k), k2 = k - k1;
    const float sc1 = pow2f(k1), sc2 = pow2f(k2 < -126 ? -126 : (k2 > 127 ? 127 : k2));
    float s[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] = XLO ? (f[i] * sc1) * sc2 : f[i] * sc1;
    std::uint32_t hv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) hv[i] = pack_h2_rn(s[2 * i], s[2 * i + 1]);
    *reinterpret_cast<uint4*>(pan + o_frag + 16u * lane) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    float eff[8];
    if constexpr (XLO) {
        std::uint32_t lv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 hh = __half22float2(u32_as_h2(hv[i]));
            lv[i] = pack_h2_rn(s[2 * i] - hh.x, s[2 * i + 1] - hh.y);
            const float2 l = __half22float2(u32_as_h2(lv[i]));
            eff[2 * i] = hh.x + l.x;
            eff[2 * i + 1] = hh.y + l.y;
        }
        *reinterpret_cast<uint4*>(pan + o_lo + 16u * lane) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 hh = __half22float2(u32_as_h2(hv[i]));
            eff[2 * i] = hh.x;
            eff[2 * i + 1] = hh.y;
        }
    }
    // XX_k = -2^(-pz) sum_c B_c 2^pc (exact power-of-two factors; fixed order)
    float X = ((eff[0] + eff[1]) + (eff[2] + eff[3])) + ((eff[4] + eff[5]) + (eff[6] + eff[7]));
    X *= pow2f(pc - pz);
    X += __shfl_xor_sync(0xffffffffu, X, 1);
    if ((lane & 1) == 0) reinterpret_cast<float*>(pan + o_xx)[kk] = -X;
    if (lane == 0) {  // y = R 2^(48 - e): as two normal factors
        const int q = 48 - e;
        const int q1 = q < -126 ? -126 : (q > 127 ? 127 : q);
        reinterpret_cast<float*>(pan + o_sc)[0] = pow2f(q1);
        reinterpret_cast<float*>(pan + o_sc)[1] = pow2f(q - q1);
    }
}

template <int BW, int BS, int XM>
__device__ __forceinline__ void build_panel(const XLane<XM>& xl, int lane, std::uint8_t* pan) {
    constexpr std::uint32_t O_XX = T::kPanelXXOff, O_SC = T::kPanelSCOff, O_XP = T::kPanelXPOff;
    constexpr std::uint32_t O_LO = T::panel_lo_off(XM);
    if constexpr (XM == 2) {
        build_col<BW, BS, false>(xl.w, lane, pan, 0, O_XX, O_SC, O_XP, 0);
        build_col<BW, BS, false>(xl.w + 4, lane, pan, O_LO, T::panel_xx1_off(2), T::panel_sc1_off(2), O_XP + 512u, 0);
    } else {
        build_col<BW, BS, XM == 1>(xl.w, lane, pan, 0, O_XX, O_SC, O_XP, O_LO);
    }
}

// SHX: the CTA prepares all Pn x panels once (shared memory) instead of each
// warp preparing its cell's panel -- for layers whose panels fit.
template <int BW, int BS, int BZ, int XM, int NC, bool SHX, bool GATHER = false>
__global__ void __launch_bounds__(NC * 32, 1) gemv_cta(const CtaParams p) {
    static_assert(BS == BZ, "fast path: scale and zero codes share the statistic width");
    static_assert(!(GATHER && XM == 2), "the fused gather is batch 1");
    constexpr bool XLO = XM == 1;
    constexpr int NCOL = XM == 2 ? 2 : 1;  // batch columns of one launch
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BZ);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BZ);
    constexpr std::uint32_t PANEL = T::panel_bytes(XM);
    constexpr std::uint32_t O_FRAG = 0, O_XX = T::kPanelXXOff, O_SC = T::kPanelSCOff, O_XP = T::kPanelXPOff;
    constexpr std::uint32_t O_LO = T::panel_lo_off(XM);
    constexpr std::uint32_t O_XX1 = T::panel_xx1_off(2), O_SC1 = T::panel_sc1_off(2);  // mode 2: column 1
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr std::uint32_t SMASK = (1u << BS) - 1u;
    constexpr int NT = NC * 32;

    extern __shared__ __align__(128) std::uint8_t smem[];
    __shared__ std::uint64_t full[NC][2];
    __shared__ std::uint64_t coff_bar;               // the first range's record offsets have landed
    __shared__ std::uint32_t slot_r[NC][2][2];       // record byte range of the slot's cell
    __shared__ std::uint32_t tick[2];                // per-range ticket counters (by range parity)
    __shared__ volatile std::uint32_t pflag[64];     // SHX: x panel built
    __shared__ float rowsum[NC][NCOL][32];           // outlier row sums of a cell (zero between cells)
    __shared__ __align__(16) float coef[NC][2][32];  // -S Z 2^(p-24) per (unit, block, kind)
    __shared__ __align__(16) std::uint32_t zrow[NC][4];  // 16 zero bytes: masked ldmatrix rows

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ std::uint32_t g_round, g_round_ok, g_peers_ok;  // GATHER: this launch's round; peers have started it
    auto wait_peers = [&]() {  // (GATHER) until every peer's band kernel of this round has started
        if (lane == 0) {
            while (*reinterpret_cast<volatile std::uint32_t*>(&g_round_ok) == 0u) {
            }
            const unsigned long long t0 = globaltimer();
            for (std::uint32_t j = 0; j < p.nflag; ++j) {
                if (j == p.rank) continue;
                for (std::uint32_t it = 0;; ++it) {
                    std::uint32_t v;
                    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p.started + j) : "memory");
                    if (static_cast<int>(v - g_round) >= 0) break;
                    if ((it & 1023u) == 1023u && globaltimer() - t0 > 20000000000ull) __trap();  // dead peer
                }
            }
            *reinterpret_cast<volatile std::uint32_t*>(&g_peers_ok) = 1u;
        }
        __syncwarp();
    };
    auto put_y = [&](std::uint32_t row, float v) {
        p.y[row] = v;
        if constexpr (GATHER) {
            if (p.npeer && *reinterpret_cast<volatile std::uint32_t*>(&g_peers_ok) == 0u) wait_peers();
            for (std::uint32_t j = 0; j < p.npeer; ++j) p.ypeer[j][p.row_base + row] = v;
        }
    };
#ifdef SPQR_TIMELINE
    const std::uint32_t wk = blockIdx.x * 16u + static_cast<std::uint32_t>(warp);
    unsigned long long tl_wait = 0, tl_panels = 0;
    std::uint32_t tl_cnt = 0;
#endif
    SPQR_TL(0)

    if (lane == 0) {
        mbar_init(&full[warp][0], 1);
        mbar_init(&full[warp][1], 1);
        if (warp == 0) mbar_init(&coff_bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x == 0) {
        tick[0] = tick[1] = NC;  // ticket w < NC is warp w's first cell
        if constexpr (GATHER) g_round_ok = g_peers_ok = 0u;
    }
    if (threadIdx.x < 64) pflag[threadIdx.x] = 0u;
    for (int c = 0; c < NCOL; ++c) rowsum[warp][c][lane] = 0.f;
    if (lane < 4) zrow[warp][lane] = 0u;
    // lane 0: bulk copy of a cell's record bytes (up to the slot's capacity)
    auto copy_rec = [&](std::uint8_t* dst, std::uint32_t r0, std::uint32_t r1, std::uint64_t* bar) {
        const std::uint32_t nb = min(r1 - r0, p.rec_cap);
        mbar_expect_tx(bar, nb);
        bulk_g2s(dst, p.cells + r0, nb, bar);
    };
    std::uint32_t* const coff_base = reinterpret_cast<std::uint32_t*>(smem + p.off_off);
    std::uint32_t* coff = coff_base;
    std::uint32_t* gdone = reinterpret_cast<std::uint32_t*>(smem + p.gd_off);  // finished cells per pair
    for (std::uint32_t i = threadIdx.x; i <= p.part_cap; i += NT) gdone[i] = 0;  // whole capacity
    // Shared state is ready at this barrier, and no global load precedes it: a
    // CTA that becomes resident late reaches the PDL wait without a round trip.
    __syncthreads();
    // the first record of this warp's first ticket goes out first, its offsets
    // from the plan's per-CTA table
    if (blockIdx.x < p.nvcta && lane == 0) {
        const uint2 r = __ldg(p.first_rec + blockIdx.x * NC + warp);
        if (r.y > r.x) {
            slot_r[warp][0][0] = r.x;
            slot_r[warp][0][1] = r.y;
            copy_rec(smem + static_cast<std::size_t>(warp) * 2u * p.slot_bytes, r.x, r.y, &full[warp][0]);
        }
    }
    // record offsets of the range: the first range's arrive by one bulk copy
    // (16-B aligned superset; cell_off is padded), waited on only where used;
    // later ranges load them after a barrier
    auto range_setup = [&](std::uint32_t v) {
        const std::uint32_t q0 = __ldg(p.cta_start + v), q1 = __ldg(p.cta_start + v + 1);
        coff = coff_base;
        for (std::uint32_t i = threadIdx.x; i <= q1 - q0; i += NT) {
            coff[i] = __ldg(p.cell_off + q0 + i);
            gdone[i] = 0;
        }
    };
    auto range_bounds = [&](std::uint32_t v, std::uint32_t& q0, std::uint32_t& q1) {
        if (v == blockIdx.x && gridDim.x < static_cast<unsigned>(kQFirst)) {
            q0 = p.q_first[v];
            q1 = p.q_first[v + 1];
        } else {
            q0 = __ldg(p.cta_start + v);
            q1 = __ldg(p.cta_start + v + 1);
        }
    };
    if (blockIdx.x < p.nvcta) {
        std::uint32_t q0, q1;
        range_bounds(blockIdx.x, q0, q1);
        const std::uint32_t qa = q0 & ~3u, qb = (q1 + 4u) & ~3u;
        coff = coff_base + (q0 - qa);
        if (threadIdx.x == 0) {  // the thread that initialised coff_bar
            mbar_expect_tx(&coff_bar, 4u * (qb - qa));
            bulk_g2s(coff_base, p.cell_off + qa, 4u * (qb - qa), &coff_bar);
        }
    }
    // the next kernel in the stream may be scheduled now; it reads what we
    // write only after this grid has completed (its griddepcontrol.wait)
    pdl_launch();

    // ----------------------------------------------------------- consumers --
    const int g = lane >> 2, t = lane & 3;
    std::uint8_t* const pan_base = smem + p.pan_off;
    std::uint8_t* pan = SHX ? pan_base : pan_base + static_cast<std::uint32_t>(warp) * PANEL;
    float* part_base = reinterpret_cast<float*>(smem + p.part_off);
    // ldmatrix row addresses for the masked B operand: MMA j of a super-tile
    // routes block j to output column j, so B^T row n is block j's x when
    // n == j and zero otherwise.  Call c loads MMAs 2c, 2c+1 (x4: k halves).
    // Lane (lm, lr) addresses row lr of matrix lm; it carries data only in
    // the call whose MMA j + lm/2 == lr, and then always the same 16 bytes of
    // the panel (block 8h + lr, k half lm % 2) -- the per-call offset 256h is
    // an immediate, so the zero row is pre-biased by -256h.
    const int lm = lane >> 3, lr = lane & 7;
    const int jact = lr - (lm >> 1);
    const std::uint32_t lane_off = O_FRAG + 32u * lr + 16u * (lm & 1);
    const std::uint32_t zero_sa = smem_u32(&zrow[warp][0]);
    const std::uint32_t zb[2] = {zero_sa, zero_sa - 256u};
    // fp32 x: in the MMA of slot s of a half super-tile (blocks 8h + 2s + par),
    // B row 2s is the block's hi fragment and row 2s + 1 its lo fragment; this
    // lane addresses row lr, active in the call of slot lr / 2
    const int jact2 = (lr >> 1) - (lm >> 1);
    const std::uint32_t hl_off = ((lr & 1) ? O_LO : O_FRAG) + 64u * static_cast<std::uint32_t>(lr >> 1) + 16u * (lm & 1);
    // this lane's entry of the -S Z 2^(p-24) table: block kb = lane/2 of the
    // unit, kind = lane % 2; consumers (t, h) read {cS(b0), cS(b1), cZ(b0), cZ(b1)}
    const int kb = lane >> 1, kind = lane & 1;
    const std::uint32_t coef_src = CODEB + STATB + 8u * static_cast<std::uint32_t>(kb) + 4u * kind;
    const int coef_ix = 16 * (kb >> 3) + 4 * ((kb >> 1) & 3) + 2 * kind + (kb & 1);
    const float coef_mul = -pow2f(T::stat_p(BS, T::stat_pair(kind, kb >> 3, kb & 1)) - 24);

    std::uint8_t* ring = smem + static_cast<std::size_t>(warp) * 2u * p.slot_bytes;
    // lane 0: copy the record of cell k into slot sl (offsets from coff)
    auto issue = [&](std::uint32_t k, std::uint32_t sl) {
        if (lane == 0) {
            mbar_wait(&coff_bar, 0);  // immediate after the first range's offsets landed
            const std::uint32_t r0 = coff[k], r1 = coff[k + 1];
            slot_r[warp][sl][0] = r0;
            slot_r[warp][sl][1] = r1;
            copy_rec(ring + sl * p.slot_bytes, r0, r1, &full[warp][sl]);
        }
    };
    std::uint32_t nit = 0;  // cells this warp has taken (slot nit & 1, phase (nit >> 1) & 1)

    std::uint32_t it = 0;
    bool waited = false;
#pragma unroll 1
    for (std::uint32_t v = blockIdx.x; v < p.nvcta; v += gridDim.x, ++it) {
        std::uint32_t q0, q1;
        range_bounds(v, q0, q1);
        const std::uint32_t nc = q1 - q0;
        float* part = part_base;
        const std::uint32_t Ga = p.Pn == 1u ? q0 : __umulhi(q0, p.pn_magic);
        auto pair_of = [&](std::uint32_t k) {
            const std::uint32_t q = q0 + k;
            return p.Pn == 1u ? q : __umulhi(q, p.pn_magic);
        };
        auto grab = [&]() {
            std::uint32_t k = 0;
            if (lane == 0) k = atomicAdd(&tick[it & 1u], 1u);
            return __shfl_sync(0xffffffffu, k, 0);
        };
        auto panel_of = [&](std::uint32_t k) {
            const std::uint32_t q = q0 + k;
            return p.Pn == 1u ? 0u : q - __umulhi(q, p.pn_magic) * p.Pn;
        };
        // one ticket of lookahead: the next cell's record copy and x loads are
        // in flight while this cell computes.  Warp w's first ticket is w.
        std::uint32_t tk = static_cast<std::uint32_t>(warp);
        if (tk < nc && waited) issue(tk, nit & 1u);  // (the first range's went out in the prologue)
        // SHX: panel index i = warp + NC j covers panel (P0 + i) mod Pn; j = 0 is the
        // panel of this warp's first cell.  Each warp builds its panels right
        // after the PDL wait; readers check pflag instead of a CTA barrier.
        const std::uint32_t P0 = panel_of(0);
        auto panel_at = [&](std::uint32_t i) {
            std::uint32_t P = P0 + i;
            return P >= p.Pn ? P - p.Pn : P;
        };
        auto publish = [&](std::uint32_t P, const XLane<XM>& xv) {
            build_panel<BW, BS, XM>(xv, lane, pan_base + P * PANEL);
            __syncwarp();
            __threadfence_block();
            if (lane == 0) pflag[P] = 1u;
        };
        if (!waited) {
            pdl_wait();  // the preceding kernel has completed: x, y and the partial slots are ours
            waited = true;
            if constexpr (GATHER) {
                if (threadIdx.x == 0) {  // (the other warps go on: only peer stores need the round)
                    const std::uint32_t r = *p.round + 1u;  // the previous round's grid has completed
                    if (blockIdx.x == 0) {  // announce: this rank's band kernel of round r runs
                        if (p.nflag > 1) {
                            for (std::uint32_t j = 0; j < p.nflag; ++j)
                                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.pflags[j] + kGatherStartedWord + p.rank),
                                             "r"(r) : "memory");
                        } else {  // world 1: no other observer than this GPU
                            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.pflags[0] + kGatherStartedWord + p.rank),
                                         "r"(r) : "memory");
                        }
                    }
                    g_round = r;
                    __threadfence_block();
                    *reinterpret_cast<volatile std::uint32_t*>(&g_round_ok) = 1u;
                }
            }
            SPQR_TL(1)
            if constexpr (SHX) {  // own panels (<= 3), the first cell's first; every x load
                                  // is in flight before the first build; no CTA barrier
                const std::uint32_t i0 = warp, i1 = warp + NC, i2 = warp + 2 * NC;
                XLane<XM> xa{}, xb{}, xc{};
                if (i0 < p.Pn) xa = load_x<XM>(p, panel_at(i0), lane);
                if (i1 < p.Pn) xb = load_x<XM>(p, panel_at(i1), lane);
                if (i2 < p.Pn) xc = load_x<XM>(p, panel_at(i2), lane);
                if (i0 < p.Pn) publish(panel_at(i0), xa);
                if (i1 < p.Pn) publish(panel_at(i1), xb);
                if (i2 < p.Pn) publish(panel_at(i2), xc);
#pragma unroll 1
                for (std::uint32_t i = warp + 3 * NC; i < p.Pn; i += NC) publish(panel_at(i), load_x<XM>(p, panel_at(i), lane));
            }
#ifdef SPQR_TIMELINE
            tl_panels = gtime();
#endif
        }
        XLane<XM> xl{};
        if (!SHX && tk < nc) xl = load_x<XM>(p, panel_of(tk), lane);
#pragma unroll 1
        while (tk < nc) {
            const std::uint32_t tn = grab();
            XLane<XM> xn{};
            if (tn < nc) {
                issue(tn, (nit + 1u) & 1u);
                if constexpr (!SHX) xn = load_x<XM>(p, panel_of(tn), lane);
            }
            const std::uint32_t slot = nit & 1u;
            const std::uint32_t ck = tk;  // this ticket's cell (range index)

            if constexpr (SHX) {
                const std::uint32_t P = panel_of(ck);
                pan = pan_base + P * PANEL;
                if (pflag[P] == 0u) {
                    while (pflag[P] == 0u) {
                    }
                }
                __threadfence_block();
            } else {
                build_panel<BW, BS, XM>(xl, lane, pan);
                __syncwarp();
            }
            const std::uint32_t lane_sa = smem_u32(pan) + lane_off;
            const std::uint32_t hl_sa = smem_u32(pan) + hl_off;  // fp32 x
#ifdef SPQR_TIMELINE
            const unsigned long long tw0 = gtime();
#endif
            mbar_wait(&full[warp][slot], (nit >> 1) & 1u);
#ifdef SPQR_TIMELINE
            if (tl_cnt == 0) SPQR_TL(2)
            tl_wait = tw0;  // start of the latest cell (after its panel)
            ++tl_cnt;
#endif
            const std::uint8_t* cell = ring + slot * p.slot_bytes;
            const std::uint32_t r0 = slot_r[warp][slot][0], r1 = slot_r[warp][slot][1];

            // ---- this lane's entry of the -S Z 2^(p-24) table, both units
            {
                const std::uint32_t w0 = *reinterpret_cast<const std::uint32_t*>(cell + coef_src);
                const std::uint32_t w1 = *reinterpret_cast<const std::uint32_t*>(cell + UNIT + coef_src);
                coef[warp][0][coef_ix] = fhfma<0, 1>(w0, w0, 0.f) * coef_mul;
                coef[warp][1][coef_ix] = fhfma<0, 1>(w1, w1, 0.f) * coef_mul;
            }
            // ---- lane statistics words of both units (tiled.hpp): W0 = lo bytes
            // 0,1 | hi bytes 0,1, W1 = lo bytes 2,3 | hi bytes 2,3
            std::uint32_t sw[2][2];
#pragma unroll
            for (int ui = 0; ui < 2; ++ui) {
                const std::uint8_t* stats = cell + ui * UNIT + CODEB;
                if constexpr (BS == 3) {
                    sw[ui][0] = reinterpret_cast<const std::uint32_t*>(stats)[lane];
                    const std::uint32_t u16 = reinterpret_cast<const std::uint16_t*>(stats + 128)[lane];
                    sw[ui][1] = __byte_perm(u16, 0u, 0x4140);
                } else if constexpr (BS == 2) {
                    sw[ui][0] = reinterpret_cast<const std::uint32_t*>(stats)[lane];
                    sw[ui][1] = 0u;
                } else {
                    const uint2 v2 = reinterpret_cast<const uint2*>(stats)[lane];
                    sw[ui][0] = v2.x;
                    sw[ui][1] = v2.y;
                }
            }
            // pair j of unit ui as an f16x2 of subnormals code 2^(p-24) (rows g, g+8)
            auto stat_pair = [&](int ui, int j) -> std::uint32_t {
                const int B = T::stat_window(BS, j), pb = T::stat_p(BS, j);
                return window<2>(sw[ui], B) & ((SMASK << pb) * 0x00010001u);
            };

            // lane data of the units: code words
            std::uint32_t cw[2][XM ? 1 : G::LANE_WORDS];
            if constexpr (XM == 0) {
#pragma unroll
                for (int ui = 0; ui < 2; ++ui) {
                    const std::uint8_t* unit = cell + ui * UNIT;
#pragma unroll
                    for (int i = 0; i < G::LANE_WORDS / 4; ++i) {
                        const uint4 w4 = reinterpret_cast<const uint4*>(unit + lane * 16 * BW)[i];
                        cw[ui][4 * i] = w4.x;
                        cw[ui][4 * i + 1] = w4.y;
                        cw[ui][4 * i + 2] = w4.z;
                        cw[ui][4 * i + 3] = w4.w;
                    }
                }
            }
            __syncwarp();  // the coefficient table is complete

            // epilogue of super-tile h: acc += s' (C + z' XX)
            float2 acc[NCOL][2][2];  // [column][unit][rho] = (block 2t, block 2t+1) partials of row g + 8 rho
#pragma unroll
            for (int c = 0; c < NCOL; ++c)
#pragma unroll
                for (int ui = 0; ui < 2; ++ui) acc[c][ui][0] = acc[c][ui][1] = make_float2(0.f, 0.f);
            auto epilogue = [&](auto HC, const float (&c)[2][4], int col) {
                constexpr int h = decltype(HC)::value;
                const float2 xx = *reinterpret_cast<const float2*>(pan + (col ? O_XX1 : O_XX) + 4u * (8u * h + 2u * t));
#pragma unroll
                for (int ui = 0; ui < 2; ++ui) {
                    // {S_s|Z_s, S_z|Z_z} of blocks 8h + 2t and 8h + 2t + 1
                    const uint4 s4 = *reinterpret_cast<const uint4*>(cell + ui * UNIT + CODEB + STATB + (8 * h + 2 * t) * 8);
                    const float4 cf = *reinterpret_cast<const float4*>(&coef[warp][ui][16 * h + 4 * t]);
                    const std::uint32_t rs0 = stat_pair(ui, T::stat_pair(0, h, 0));
                    const std::uint32_t rs1 = stat_pair(ui, T::stat_pair(0, h, 1));
                    const std::uint32_t rz0 = stat_pair(ui, T::stat_pair(1, h, 0));
                    const std::uint32_t rz1 = stat_pair(ui, T::stat_pair(1, h, 1));
                    {  // rho = 0: row g
                        const float2 sh = make_float2(fhfma<0, 0>(s4.x, rs0, cf.x), fhfma<0, 0>(s4.z, rs1, cf.y));
                        const float2 zh = make_float2(fhfma<0, 0>(s4.y, rz0, cf.z), fhfma<0, 0>(s4.w, rz1, cf.w));
                        const float2 tt = ffma2(zh, xx, make_float2(c[ui][0], c[ui][1]));
                        acc[col][ui][0] = ffma2(sh, tt, acc[col][ui][0]);
                    }
                    {  // rho = 1: row g + 8
                        const float2 sh = make_float2(fhfma<0, 1>(s4.x, rs0, cf.x), fhfma<0, 1>(s4.z, rs1, cf.y));
                        const float2 zh = make_float2(fhfma<0, 1>(s4.y, rz0, cf.z), fhfma<0, 1>(s4.w, rz1, cf.w));
                        const float2 tt = ffma2(zh, xx, make_float2(c[ui][2], c[ui][3]));
                        acc[col][ui][1] = ffma2(sh, tt, acc[col][ui][1]);
                    }
                }
            };
            // A fragments of MMA (super-tile h, block j) of unit ui from code words w
            auto afrag = [&](const std::uint32_t* cwu, int h, int j, std::uint32_t (&a)[4]) {
                const int mu = 8 * h + j, cidx = mu / G::MPC, mm = mu % G::MPC;
                const std::uint32_t* w = cwu + G::CW * cidx;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
                    const int i = rho * (G::NP / 2) + qq;
                    const int B = (BW * i) >> 3, pb = (BW * i) & 7;
                    a[r] = window<G::CW>(w, B) & ((MASK << pb) * 0x00010001u);
                }
            };
            if constexpr (XM == 0) {
                // 4 independent MMA chains (super-tile h x unit), interleaved
                std::uint32_t bfr[2][4];
                float cc[2][2][4];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int ui = 0; ui < 2; ++ui)
#pragma unroll
                        for (int i = 0; i < 4; ++i) cc[h][ui][i] = 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if ((j & 1) == 0) {
                            const bool act = jact == j;
                            ldsm_x4((act ? lane_sa : zb[h]) + 256u * h, bfr[h]);
                        }
                        const std::uint32_t b0 = bfr[h][2 * (j & 1)], b1 = bfr[h][2 * (j & 1) + 1];
#pragma unroll
                        for (int ui = 0; ui < 2; ++ui) {
                            std::uint32_t a[4];
                            afrag(cw[ui], h, j, a);
                            mma16816(cc[h][ui], a, b0, b1);
                        }
                    }
                }
                epilogue(std::integral_constant<int, 0>{}, cc[0], 0);
                epilogue(std::integral_constant<int, 1>{}, cc[1], 0);
            } else {
                // fp32 x = hi + lo, both f16, sharing one MMA: super-tile h
                // runs as its even blocks then its odd blocks (parity par);
                // the MMA of block 8h + 2s + par routes the hi part to
                // output column 2s and the lo part to 2s + 1, so lane (g, t)
                // gets hi and lo of block 8h + 2t + par side by side -- the
                // (row, block) pairs whose statistics it holds -- and adds
                // them in-lane: 32 MMAs per cell as for f16 x, no shuffles.
                auto half = [&](auto HC) {
                    constexpr int h = decltype(HC)::value;
                    constexpr int W0 = G::CW * (8 * h / G::MPC), W1 = G::CW * ((8 * h + 7) / G::MPC + 1);
                    static_assert(W0 % 2 == 0 && W1 % 2 == 0, "code words of a super-tile: 8 B aligned");
                    std::uint32_t cwh[2][G::LANE_WORDS];
#pragma unroll
                    for (int ui = 0; ui < 2; ++ui) {
                        const std::uint8_t* unit = cell + ui * UNIT;
#pragma unroll
                        for (int i = W0; i < W1; i += 2) {
                            const uint2 w2 = reinterpret_cast<const uint2*>(unit + lane * 16 * BW)[i / 2];
                            cwh[ui][i] = w2.x;
                            cwh[ui][i + 1] = w2.y;
                        }
                    }
                    float d[2][2][4];  // [parity][unit]: {hi, lo} of block 8h + 2t + par, rows g / g + 8
#pragma unroll
                    for (int par = 0; par < 2; ++par)
#pragma unroll
                        for (int ui = 0; ui < 2; ++ui)
#pragma unroll
                            for (int i = 0; i < 4; ++i) d[par][ui][i] = 0.f;
#pragma unroll
                    for (int par = 0; par < 2; ++par) {
#pragma unroll
                        for (int c2 = 0; c2 < 2; ++c2) {  // slots s = 2 c2, 2 c2 + 1
                            std::uint32_t bq[4];
                            ldsm_x4(jact2 == 2 * c2 ? hl_sa + 256u * h + 32u * par : zero_sa, bq);
#pragma unroll
                            for (int m2 = 0; m2 < 2; ++m2) {
                                const int j = 2 * (2 * c2 + m2) + par;  // block 8h + j
#pragma unroll
                                for (int ui = 0; ui < 2; ++ui) {
                                    std::uint32_t a[4];
                                    afrag(cwh[ui], h, j, a);
                                    mma16816(d[par][ui], a, bq[2 * m2], bq[2 * m2 + 1]);
                                }
                            }
                        }
                    }
                    if constexpr (XLO) {
                        float ch[2][4];  // the f16 layout: (g, 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)
#pragma unroll
                        for (int ui = 0; ui < 2; ++ui) {
                            ch[ui][0] = d[0][ui][0] + d[0][ui][1];
                            ch[ui][1] = d[1][ui][0] + d[1][ui][1];
                            ch[ui][2] = d[0][ui][2] + d[0][ui][3];
                            ch[ui][3] = d[1][ui][2] + d[1][ui][3];
                        }
                        epilogue(HC, ch, 0);
                    } else {  // two batch columns: slot 2s carries column 0, 2s + 1 column 1
                        float c0[2][4], c1[2][4];
#pragma unroll
                        for (int ui = 0; ui < 2; ++ui) {
                            c0[ui][0] = d[0][ui][0]; c0[ui][1] = d[1][ui][0]; c0[ui][2] = d[0][ui][2]; c0[ui][3] = d[1][ui][2];
                            c1[ui][0] = d[0][ui][1]; c1[ui][1] = d[1][ui][1]; c1[ui][2] = d[0][ui][3]; c1[ui][3] = d[1][ui][3];
                        }
                        epilogue(HC, c0, 0);
                        epilogue(HC, c1, 1);
                    }
                };
                half(std::integral_constant<int, 0>{});
                half(std::integral_constant<int, 1>{});
            }

            // outliers: entries (row, col, value) of this cell, sorted by (row,
            // col), 0xffffffff padding (row 255).  Chunks of 128 entries, 4
            // consecutive per lane (one 16-byte load): products, a segmented
            // inclusive scan by row, and the last entry of each row in the
            // chunk adds the row total to rowsum.  Chunks run in order, so the
            // sums are deterministic.  Entries beyond the staged part of the
            // record are read from global memory.
            const std::uint32_t cnt = (r1 - r0 - CELL) / 4u;
            if (cnt) {
                const std::uint32_t nfast = (min(r1 - r0, p.rec_cap) - CELL) / 4u;
                const std::uint32_t* es = reinterpret_cast<const std::uint32_t*>(cell + CELL);
                const std::uint32_t* eg = reinterpret_cast<const std::uint32_t*>(p.cells + r0 + CELL) + nfast;
                auto chunk = [&](const std::uint32_t* src, std::uint32_t i0, std::uint32_t lim, bool first) {
                    uint4 ev = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                    if (i0 < lim) ev = *reinterpret_cast<const uint4*>(src + i0);  // lim % 4 == 0
                    const std::uint32_t e[4] = {ev.x, ev.y, ev.z, ev.w};
                    std::uint32_t k[4];
                    float sv[NCOL][4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        k[j] = e[j] >> 24;
                        const std::uint32_t c = __byte_perm(e[j], 0u, 0x4442);  // col: byte 2
                        if constexpr (XLO) {
                            sv[0][j] = h2f_bits(e[j] & 0xffffu) * reinterpret_cast<const float*>(pan + O_XP)[c];
                        } else {
#pragma unroll
                            for (int cl = 0; cl < NCOL; ++cl) {
                                const std::uint32_t xv = reinterpret_cast<const unsigned short*>(pan + O_XP + 512u * cl)[c];
                                sv[cl][j] = fhfma<0, 0>(e[j], xv, 0.f);  // v * x, exact
                            }
                        }
                    }
                    bool same[3];
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        same[j] = k[j + 1] == k[j];
#pragma unroll
                        for (int cl = 0; cl < NCOL; ++cl)
                            if (same[j]) sv[cl][j + 1] += sv[cl][j];
                    }
                    const std::uint32_t K = k[3];
                    const std::uint32_t pK = __shfl_up_sync(0xffffffffu, K, 1);
                    const bool head = lane == 0 || pK != K;
                    const std::uint32_t heads = __ballot_sync(0xffffffffu, head) & (0xffffffffu >> (31 - lane));
                    const int seg0 = 31 - __clz(heads);
                    const std::uint32_t nk0 = __shfl_down_sync(0xffffffffu, k[0], 1);
#pragma unroll
                    for (int cl = 0; cl < NCOL; ++cl) {
                        float V = sv[cl][3];
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const float o = __shfl_up_sync(0xffffffffu, V, d);
                            if (lane - d >= seg0) V += o;
                        }
                        float cin = __shfl_up_sync(0xffffffffu, V, 1);
                        if (lane == 0 || pK != k[0]) cin = 0.f;
                        float* rs = rowsum[warp][cl];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const bool tail = (j < 3) ? !same[j] : (lane == 31 || nk0 != k[3]);
                            if (tail && k[j] < 32u) {
                                const float tot = (k[j] == k[0]) ? sv[cl][j] + cin : sv[cl][j];
                                if (first)
                                    rs[k[j]] = tot;
                                else
                                    rs[k[j]] += tot;
                            }
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
                    chunk(eg, base - nfast + 4u * lane, cnt - nfast, false);
                }
            }

            // the cell's row sums.  Lane (g, t) holds partials of rows
            // 16u + 8rho + g over its blocks; a transpose-add across the quad
            // gives each row one lane: row = 16 (t >> 1) + 8 (t & 1) + g.
            float* prow = part + ck * (32u * NCOL);
#pragma unroll
            for (int cl = 0; cl < NCOL; ++cl) {
                const float a0 = acc[cl][0][0].x + acc[cl][0][0].y, a1 = acc[cl][0][1].x + acc[cl][0][1].y;
                const float a2 = acc[cl][1][0].x + acc[cl][1][0].y, a3 = acc[cl][1][1].x + acc[cl][1][1].y;
                const bool o1 = t & 1, o2 = t & 2;
                const float k0 = o1 ? a1 : a0, k1 = o1 ? a3 : a2;  // combos (t&1), (t&1)+2
                const float s0 = o1 ? a0 : a1, s1 = o1 ? a2 : a3;
                const float b0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 1);
                const float b1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 1);
                const float keep = o2 ? b1 : b0, send = o2 ? b0 : b1;
                const float R = keep + __shfl_xor_sync(0xffffffffu, send, 2);
                const int row = 16 * (t >> 1) + 8 * (t & 1) + g;
                const float2 sc = *reinterpret_cast<const float2*>(pan + (cl ? O_SC1 : O_SC));
                const float Rs = XLO ? (R * sc.x) * sc.y : R * sc.x;
                __syncwarp();
                if (cnt) {
                    prow[32 * cl + row] = Rs + rowsum[warp][cl][row];
                    rowsum[warp][cl][row] = 0.f;
                } else {
                    prow[32 * cl + row] = Rs;
                }
            }

            // count the cell against its pair; the warp that completes the
            // pair reduces it (row = lane, cells in order) and writes y
            const std::uint32_t Gq = pair_of(ck);
            const std::uint32_t cs = Gq * p.Pn, ce = cs + p.Pn;
            const std::uint32_t a = max(cs, q0), b = min(ce, q1);
            __threadfence_block();  // this cell's row sums before the count
            std::uint32_t done = 0;
            if (lane == 0) done = atomicAdd(&gdone[Gq - Ga], 1u) + 1u;
            done = __shfl_sync(0xffffffffu, done, 0);
            if (done == b - a) {
                __threadfence_block();
#pragma unroll
                for (int cl = 0; cl < NCOL; ++cl) {
                float sum = 0.f;
                const float* src = part + (a - q0) * (32u * NCOL) + 32u * cl + lane;
#pragma unroll 4
                for (std::uint32_t qq = a; qq < b; ++qq, src += 32 * NCOL) sum += *src;
                const std::uint32_t row = 32u * Gq + lane;
                if (a == cs && b == ce) {  // the pair is ours alone
                    if (row < p.m) put_y(cl * p.m + row, sum);
                } else {
                    // shared with the neighbouring range: the second side to
                    // finish adds first-side + last-side (threadFenceReduction)
                    const std::uint32_t side = a != cs ? 1u : 0u;  // 1: we hold the pair's last cells
                    const std::uint32_t bx = side ? v : v + 1u;    // boundary below range bx
                    float* slot = p.xpart + ((2u * bx + side) * NCOL + cl) * 32u;
                    __stcg(slot + lane, sum);
                    __threadfence();
                    __syncwarp();
                    std::uint32_t prev = 0;
                    if (lane == 0) prev = atomicAdd(p.xcnt + NCOL * bx + cl, 1u);
                    prev = __shfl_sync(0xffffffffu, prev, 0);
                    if (prev == 1u) {
                        __threadfence();
                        const float other = __ldcg(p.xpart + ((2u * bx + (side ^ 1u)) * NCOL + cl) * 32u + lane);
                        if (row < p.m) put_y(cl * p.m + row, side ? other + sum : sum + other);
                        if (lane == 0) p.xcnt[NCOL * bx + cl] = 0u;  // ready for the next launch
                    }
                }
                }
            }
            __syncwarp();  // every lane is done with the slot before it is refilled
            tk = tn;
            xl = xn;
            ++nit;
        }
        SPQR_TL(3)
        if (v + gridDim.x < p.nvcta) {  // this CTA has another range
            bar_sync_named(1, NT);
            if (threadIdx.x == 0) tick[it & 1u] = NC;
            range_setup(v + gridDim.x);
            bar_sync_named(1, NT);
        }
    }
#ifdef SPQR_TIMELINE
    SPQR_TL(4)
    if (lane == 0) {
        g_timeline[8 * wk + 5] = tl_cnt;   // cells this warp processed
        g_timeline[8 * wk + 6] = tl_wait;  // start of its last cell
        unsigned smid;
        asm("mov.u32 %0, %smid;" : "=r"(smid));
        g_timeline[8 * wk + 7] = 1000u + smid;
    }
#endif
    if constexpr (GATHER) {  // fused all-gather: signal the round to every rank
        __syncthreads();        // every y store of this CTA precedes thread 0's release
        if (threadIdx.x == 0) {
            // A CTA that stored into peers' memory (NVLink) drains those
            // stores system-wide itself (a GPU-scope release need not wait
            // for remote acknowledgements); then a GPU-scope acq_rel counter,
            // and the grid's last CTA -- which has observed every CTA's
            // release -- fences system-wide and bumps the ranks' round counters
            if (p.npeer) __threadfence_system();
            std::uint32_t prev;
            asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.done_ctr) : "memory");
            if (prev == gridDim.x - 1u) {  // the grid's last CTA: acquire every CTA's release
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                *p.done_ctr = 0u;
                // (the CTAs' peer stores were fenced system-wide before their
                // release; the sys-scope release below is cumulative over them)
                if (p.nflag > 1) {
                    for (std::uint32_t j = 0; j < p.nflag; ++j)
                        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.pflags[j] + p.rank) : "memory");
                } else {  // world 1: GPU scope (the next kernel in this stream is the only reader)
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.pflags[0] + p.rank) : "memory");
                }
                // the gather's wait, fused: this CTA (and so the grid) completes
                // once every rank's counter reached this round -- y is then whole
                // for whatever the stream runs next; the round advances here
                const std::uint32_t* flags = p.pflags[p.rank];
                const unsigned long long t0 = globaltimer();
                for (std::uint32_t j = 0; j < p.nflag; ++j)
                    for (std::uint32_t it = 0; j != p.rank; ++it) {  // (our own counter: bumped just above)
                        std::uint32_t v;
                        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + j) : "memory");
                        if (static_cast<int>(v - g_round) >= 0) break;
                        if ((it & 1023u) == 1023u && globaltimer() - t0 > 20000000000ull) __trap();  // dead peer
                    }
                *const_cast<std::uint32_t*>(p.round) = g_round;
            }
        }
    }
}

// The GATHER = true instantiations live in gather.cu (compiled in parallel
// with capi.cu); the single-GPU kernels carry none of the gather code.
cudaError_t launch_cta_gather(int bw, int bsz, bool xlo, bool shx, const CtaParams& p, std::uint32_t grid,
                              std::uint32_t smem, int nc, std::uint32_t smem_limit, cudaStream_t st);
