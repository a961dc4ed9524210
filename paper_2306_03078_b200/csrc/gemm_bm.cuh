// gemm_bm.cuh -- exact batched SpQR decode with the batch in the MMA's M
// dimension (exact mode, batch 9..32).  Included by kernels.cuh (namespace
// spqr_dev) after gemm_ex.cuh; instantiated in gemm_ex.cu.
//
// Reference semantics: matvec(t, x, plan) (kernel.hpp:89-124) per batch
// column, y[r] = sum_k s(k,r) sum_{c in k} (q(r,c) - z(k,r)) x[c] + sum v x[col].
// One mma.sync.m16n8k16 per (16 batch columns, 16-column block, 8 rows):
//   A = x 2^(e - p_c)  (fp16, batch x k: one ldmatrix.x4 per block from the
//                       panel's x tile, shared by every row of the CTA)
//   B = the codes      the batch-1 A-fragment registers ARE m16n8k16 B
//                      fragments (lane (g, t): row g, columns 2t + {0,1}, 8 +
//                      2t + {0,1}) -- binary16 subnormals q 2^(p-24) from ONE
//                      LOP3 per pair: exact products
//   acc += s (C - z X_k 2^-24)   per (row, block) in fp32 registers, s and z
//                      the stat_dequant values from a per-warp table
//   O  += V X          the outliers: fp16 v 2^p_c scattered into a zeroed,
//                      padded per-warp tile, ldmatrix'ed as B fragments, MMAs
//                      into one accumulator per tile (exact products)
//   y = (2^24 acc + O) 2^-e
// fp32 rounding only, as the batch-1 kernel.  No tensor memory, no hand-off
// warp: the 16 warps of a CTA each own 16 rows x 8 blocks (half a panel) of
// the 128-row tile and run the whole pipeline on them; they share only the x
// tile ring (bulk copies, issued by warp 0 ahead), each cell row's record
// slots, and at a tile's end the two halves of a row group add up (fixed
// order, through shared memory).
//
// Work unit: (128-row tile T, 256-column panel P) ranges and partial slots as
// gemm_tc / gemm_ex (TcPlan).

// x tile of a panel (xprep_bm, bytes):
//   BX f16 [N batch x 256 k]: K-major core matrices (k/8) 16N + (n/8) 128 + (n%8) 16 + (k%8) 2
//   XZ fp32 [16 blocks][N/16 tiles][8 g][2]: (X 2^-24 of batch 16m + g, of 16m + g + 8), X = sum_c x 2^e
__host__ __device__ constexpr std::uint32_t bm_xbytes(std::uint32_t N) { return 512u * N + 64u * N; }
constexpr std::uint32_t kBmOStride = 144;  // outlier tile row stride (128 + 16: ldmatrix rows conflict-free)
constexpr std::uint32_t kBmOTile = 16u * kBmOStride;
constexpr std::uint32_t kBmTab = 8u * 16u * 8u;  // per warp: [block of its half][row pair] float4 {s(2i), s(2i+1), -z(2i), -z(2i+1)}
constexpr std::uint32_t kBmRecSlots = 3;
constexpr int kBmWarps = 16;
__host__ __device__ constexpr std::uint32_t bm_nx(std::uint32_t N) { return N == 16 ? 4u : 3u; }
// per warp outlier tile + table, and the halves' exchange (8 row groups x 32 lanes x N/2 floats)
__host__ __device__ constexpr std::uint32_t bm_fixed_smem(std::uint32_t N) {
    return kBmWarps * (kBmOTile + kBmTab) + 8u * 32u * (N / 2u) * 4u;
}

// an outlier entry (value16 | col << 16 | local row << 24) as quarter << 30 |
// byte offset in the warp's padded quarter tile << 16 | fp16(v 2^p_c)
template <int BW>
__device__ __forceinline__ std::uint32_t bm_outlier_item(std::uint32_t en) {
    const std::uint32_t col = (en >> 16) & 255u, lr = (en >> 24) & 15u;
    const int pc = T::column_prescale(BW, col >> 4, col & 15u);
    const float vv = h2f_bits(en & 0xffffu) * __uint_as_float(static_cast<std::uint32_t>(127 + pc) << 23);
    const std::uint32_t off = lr * kBmOStride + (col & 63u) * 2u;
    return ((col >> 6) << 30) | (off << 16) | __half_as_ushort(__float2half_rn(vv));
}

static __global__ void __launch_bounds__(256) xprep_bm(const void* __restrict__ x, int x_f16, std::uint32_t n,
                                                       std::uint32_t B, std::uint32_t N, std::uint32_t Pn,
                                                       const std::uint32_t* __restrict__ order,
                                                       std::uint8_t* __restrict__ out, float* __restrict__ escale,
                                                       int bw) {
    pdl_launch();
    pdl_wait();
    __shared__ float red[8];
    const std::uint32_t nn = blockIdx.x;
    const bool live = nn < B;
    const std::size_t col0 = static_cast<std::size_t>(nn) * n;
    auto ld = [&](std::uint32_t c) -> float {
        return x_f16 ? __half2float(__ldg(static_cast<const __half*>(x) + col0 + c))
                     : __ldg(static_cast<const float*>(x) + col0 + c);
    };
    float mx = 0.f;
    if (live) {
        const bool vec = (reinterpret_cast<std::uintptr_t>(x) & 15u) == 0 && (n * (x_f16 ? 2u : 4u)) % 16u == 0;
        if (vec) {  // 16-B loads, four in flight per thread
            const uint4* xv = reinterpret_cast<const uint4*>(static_cast<const std::uint8_t*>(x) + col0 * (x_f16 ? 2u : 4u));
            const std::uint32_t nv = n * (x_f16 ? 2u : 4u) / 16u;
#pragma unroll 4
            for (std::uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
                const uint4 w = __ldg(xv + i);
                const std::uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (x_f16) {
                        const __half2 h = u32_as_h2(ws[j]);
                        mx = fmaxf(mx, fmaxf(fabsf(__low2float(h)), fabsf(__high2float(h))));
                    } else {
                        mx = fmaxf(mx, fabsf(__uint_as_float(ws[j])));
                    }
                }
            }
        } else {
#pragma unroll 4
            for (std::uint32_t c = threadIdx.x; c < n; c += blockDim.x) mx = fmaxf(mx, fabsf(ld(c)));
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) mx = fmaxf(mx, red[i]);
    int e = 0;
    if (mx > 0.f && mx <= 3.4e38f) e = min(max(14 - ilogbf(mx), -126), 126);
    const float sc = __uint_as_float(static_cast<std::uint32_t>(127 + e) << 23);
    if (threadIdx.x == 0 && blockIdx.y == 0) escale[nn] = __uint_as_float(static_cast<std::uint32_t>(127 - e) << 23);
    const int mpc = T::mmas_per_container(bw);
    const std::uint32_t nb = 16u * Pn;
    const std::uint32_t ncol = (nn >> 3) * 128u + (nn & 7u) * 16u;
    const std::uint32_t xzi = ((nn >> 4) * 8u + (nn & 7u)) * 2u + ((nn >> 3) & 1u);  // float index in a block's XZ
    for (std::uint32_t k = blockIdx.y * blockDim.x + threadIdx.x; k < nb; k += gridDim.y * blockDim.x) {
        float v[16];
        float X = 0.f;
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) {
            const std::uint32_t c = 16u * k + cc;
            float val = 0.f;
            if (live && c < n) val = ld(order ? __ldg(order + c) : c) * sc;
            v[cc] = val;
            X += val;
        }
        std::uint8_t* base = out + static_cast<std::size_t>(k >> 4) * bm_xbytes(N);
        const std::uint32_t kb = k & 15u;  // block in the panel
        const int m_ = static_cast<int>(k & 7u) % mpc;
        const float ps0 = __uint_as_float(static_cast<std::uint32_t>(127 - T::prescale_p(bw, 2 * m_)) << 23);
        const float ps1 = __uint_as_float(static_cast<std::uint32_t>(127 - T::prescale_p(bw, 2 * m_ + 1)) << 23);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            std::uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                w[q] = pack_h2_rn(v[8 * hf + 2 * q] * (hf ? ps1 : ps0), v[8 * hf + 2 * q + 1] * (hf ? ps1 : ps0));
            *reinterpret_cast<uint4*>(base + (2u * kb + hf) * 16u * N + ncol) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        reinterpret_cast<float*>(base + 512u * N)[kb * N + xzi] = X * 5.9604644775390625e-8f;  // X 2^-24
    }
}

template <int BW, int BS, int MT>
__global__ void __launch_bounds__(kBmWarps * 32, 1) gemm_bm(const ExParams p) {
    static_assert(kBmWarps == 16, "warp roles: 4 cell rows x 2 units x 2 block halves");
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BS);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BS);
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr std::uint32_t SMASK = (1u << BS) - 1u;
    constexpr float kMagic = 8388608.0f;
    constexpr std::uint32_t N = 16u * MT;
    constexpr std::uint32_t NX = bm_nx(N);
    constexpr std::uint32_t XB = bm_xbytes(N);
    constexpr std::uint32_t NS = kBmRecSlots;

    extern __shared__ __align__(128) std::uint8_t smem[];  // [NX][XB] x tiles, per warp outlier tile + table, records
    __shared__ std::uint64_t rec_full[4][NS], rec_empty[4][NS], x_full[NX], x_free[NX];
    __shared__ std::uint32_t slot_r[4][NS][3];  // record byte range, first entry of unit 1

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ci = warp & 3, uu = (warp >> 2) & 1, hh = warp >> 3;  // cell row, unit, block half
    const int g = lane >> 2, t = lane & 3;
    std::uint8_t* xbuf = smem;
    std::uint8_t* otile = smem + NX * XB + static_cast<std::uint32_t>(warp) * kBmOTile;
    float* tab = reinterpret_cast<float*>(smem + NX * XB + kBmWarps * kBmOTile + static_cast<std::uint32_t>(warp) * kBmTab);
    // table index of (block b, row r): pair (b, r / 2) at float4 b * 8 + r / 2, s at component r % 2, -z at 2 + r % 2
    auto tix = [](int b, int r) { return (b * 8 + (r >> 1)) * 4 + (r & 1); };
    float* xch = reinterpret_cast<float*>(smem + NX * XB + kBmWarps * (kBmOTile + kBmTab)) +
                 static_cast<std::uint32_t>(warp & 7) * 32u * (N / 2u);  // this row group's exchange
    std::uint8_t* recs = smem + NX * XB + bm_fixed_smem(N);
    std::uint8_t* ring = recs + static_cast<std::uint32_t>(ci) * NS * p.slot_bytes;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i)
            for (std::uint32_t k = 0; k < NS; ++k) {
                mbar_init(&rec_full[i][k], 1);
                mbar_init(&rec_empty[i][k], 4);  // the cell row's four warps
            }
        for (std::uint32_t b = 0; b < NX; ++b) {
            mbar_init(&x_full[b], 1);
            mbar_init(&x_free[b], kBmWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch();
    const std::uint32_t v = blockIdx.x;
    const std::uint32_t u0 = __ldg(p.cta_start + v), u1 = __ldg(p.cta_start + v + 1);
    auto tile_of = [&](std::uint32_t u) { return p.Pn == 1u ? u : __umulhi(u, p.pn_magic); };
    auto cell_of = [&](std::uint32_t u, std::uint32_t& q) {
        const std::uint32_t T_ = tile_of(u), P = u - T_ * p.Pn;
        const std::uint32_t Gq = 4u * T_ + static_cast<std::uint32_t>(ci);
        q = Gq * p.Pn + P;
        return Gq < p.Gn;
    };
    // records of this cell row: cell u is record u - u0, slot (u - u0) % NS, two cells ahead
    std::uint32_t nr0 = 0, nr1 = 0, nsp = 0;
    auto load_off = [&](std::uint32_t u) {
        std::uint32_t q;
        if (uu == 0 && hh == 0 && lane == 0 && u < u1 && cell_of(u, q)) {
            nr0 = __ldg(p.cell_off + q);
            nr1 = __ldg(p.cell_off + q + 1);
            nsp = __ldg(p.usplit + q);
        }
    };
    auto issue_rec = [&](std::uint32_t u) {
        std::uint32_t q;
        if (uu == 0 && hh == 0 && lane == 0 && u < u1 && cell_of(u, q)) {
            const std::uint32_t k = u - u0, sl = k % NS;
            if (k >= NS) mbar_wait(&rec_empty[ci][sl], ((k / NS) - 1u) & 1u);
            slot_r[ci][sl][0] = nr0;
            slot_r[ci][sl][1] = nr1;
            slot_r[ci][sl][2] = nsp;
            const std::uint32_t nb = min(nr1 - nr0, p.rec_cap);
            mbar_expect_tx(&rec_full[ci][sl], nb);
            bulk_g2s(ring + sl * p.slot_bytes, p.cells + nr0, nb, &rec_full[ci][sl]);
        }
    };
    // x tile of unit u (warp 0): buffer (u - u0) % NX once every warp is done with its previous unit
    auto issue_x = [&](std::uint32_t u) {
        if (warp == 0 && u < u1) {
            const std::uint32_t k = u - u0, bx = k % NX;
            if (k >= NX) mbar_wait(&x_free[bx], ((k / NX) - 1u) & 1u);
            if (lane == 0) {
                const std::uint32_t P = u - tile_of(u) * p.Pn;
                mbar_expect_tx(&x_full[bx], XB);
                bulk_g2s(xbuf + bx * XB, p.xpanels + static_cast<std::size_t>(P) * XB, XB, &x_full[bx]);
            }
            __syncwarp();
        }
    };
    load_off(u0);
    issue_rec(u0);
    load_off(u0 + 1);
    issue_rec(u0 + 1);
    load_off(u0 + 2);
    if (warp == 0) {
        pdl_wait();  // xprep_bm has completed
        for (std::uint32_t u = u0; u < u0 + NX - 1 && u < u1; ++u) issue_x(u);
    }
    pdl_wait();  // y, partial slots and counters are ours

    const std::uint32_t magic = 0x4B000000u;
    __align__(8) float acc[MT][2][4];  // [batch tile][8-row tile][C fragment]
    float oacc[MT][2][4];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[m][nt][i] = oacc[m][nt][i] = 0.f;
    // ldmatrix row address offsets: A (x) matrix mi = lane / 8: batch group mi & 1, k core mi >> 1;
    // outlier B: matrix mi: row group mi >> 1 ... (rows 0-7: k halves 0, 1; rows 8-15: k halves 0, 1)
    const std::uint32_t a_off = ((lane >> 4) & 1u) * 16u * N + ((lane >> 3) & 1u) * 128u + (lane & 7u) * 16u;
    const std::uint32_t o_off = (((lane >> 4) & 1u) * 8u + (lane & 7u)) * kBmOStride + ((lane >> 3) & 1u) * 16u;

#pragma unroll 1
    for (std::uint32_t u = u0; u < u1; ++u) {
        std::uint32_t q;
        const bool have = cell_of(u, q);
        if (have) {
            issue_rec(u + 2);
            load_off(u + 3);
        }
        issue_x(u + NX - 1);
        const std::uint32_t k = u - u0, sl = k % NS, bx = k % NX;
        const std::uint32_t T_ = tile_of(u), P = u - T_ * p.Pn;
        std::uint32_t cw[G::LANE_WORDS];
        std::uint32_t oit[4];
        std::uint32_t obeg = 0, oend = 0, onf = 0, oc0 = 0;
        bool ofast = true;
        const std::uint8_t* unit = ring + sl * p.slot_bytes + uu * UNIT;
        const std::uint32_t* ees = reinterpret_cast<const std::uint32_t*>(ring + sl * p.slot_bytes + CELL);
        if (have) {
            mbar_wait(&rec_full[ci][sl], (k / NS) & 1u);
            // statistics -> the warp's table [block][row] {s, -z} (stat_dequant, binary32)
            std::uint32_t st[2];
            load_stat_streams<BS>(unit + CODEB, lane, st);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h != hh) continue;  // this warp's half of the blocks
                const uint4 s4 = *reinterpret_cast<const uint4*>(unit + CODEB + STATB + (8 * h + 2 * t) * 8);
                const float2 Ss = make_float2(h2f_bits(s4.x & 0xffffu), h2f_bits(s4.z & 0xffffu));
                const float2 Zs = make_float2(h2f_bits(s4.x >> 16), h2f_bits(s4.z >> 16));
                const float2 Sz = make_float2(h2f_bits(s4.y & 0xffffu), h2f_bits(s4.w & 0xffffu));
                const float2 Zz = make_float2(h2f_bits(s4.y >> 16), h2f_bits(s4.w >> 16));
#pragma unroll
                for (int rho = 0; rho < 2; ++rho) {
                    const int j0 = T::stat_pair(0, h, 0), j1 = T::stat_pair(0, h, 1);
                    const float2 cs = fadd2(make_float2(magic_field_rt<SMASK>(st[rho], j0 * BS, magic),
                                                        magic_field_rt<SMASK>(st[rho], j1 * BS, magic)),
                                            make_float2(-kMagic, -kMagic));
                    const float2 cz = fadd2(make_float2(magic_field_rt<SMASK>(st[rho], (j0 + 4) * BS, magic),
                                                        magic_field_rt<SMASK>(st[rho], (j1 + 4) * BS, magic)),
                                            make_float2(-kMagic, -kMagic));
                    const int row = g + 8 * rho, b0 = 2 * t;  // block 8h + b0 of the panel
                    tab[tix(b0, row)] = __fmul_rn(Ss.x, __fsub_rn(cs.x, Zs.x));
                    tab[tix(b0, row) + 2] = -__fmul_rn(Sz.x, __fsub_rn(cz.x, Zz.x));
                    tab[tix(b0 + 1, row)] = __fmul_rn(Ss.y, __fsub_rn(cs.y, Zs.y));
                    tab[tix(b0 + 1, row) + 2] = -__fmul_rn(Sz.y, __fsub_rn(cz.y, Zz.y));
                }
            }
#pragma unroll
            for (int i = 0; i < G::LANE_WORDS / 4; ++i) {
                const uint4 w4 = reinterpret_cast<const uint4*>(unit + lane * 16 * BW)[i];
                cw[4 * i] = w4.x;
                cw[4 * i + 1] = w4.y;
                cw[4 * i + 2] = w4.z;
                cw[4 * i + 3] = w4.w;
            }
            // this unit's outliers: [obeg, oend) of the cell's (row, col)-sorted list, counted by ballots,
            // up to 128 precomputed per lane as quarter << 30 | tile offset << 16 | fp16(v 2^p_c)
            const std::uint32_t c0 = slot_r[ci][sl][0], c1 = slot_r[ci][sl][1];
            const std::uint32_t cnt = (c1 - c0 - CELL) / 4u;
            onf = (min(c1 - c0, p.rec_cap) - CELL) / 4u;
            oc0 = c0;
            obeg = uu == 0 ? 0u : slot_r[ci][sl][2] & 0xFFFFu;
            oend = uu == 0 ? slot_r[ci][sl][2] & 0xFFFFu : slot_r[ci][sl][2] >> 16;
            (void)cnt;
            ofast = oend - obeg <= 128u;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const std::uint32_t i = obeg + lane + 32u * j;
                oit[j] = 0xFFFFFFFFu;
                if (ofast && i < oend) {
                    const std::uint32_t en = ex_entry(ees, onf, p.cells, oc0, CELL, i);
                    if (((en >> 23) & 1u) == static_cast<std::uint32_t>(hh)) oit[j] = bm_outlier_item<BW>(en);  // this half (col >> 7)
                }
            }
            __syncwarp();  // the table is complete
        }
        mbar_wait(&x_full[bx], (k / NX) & 1u);
        const std::uint8_t* xt = xbuf + bx * XB;
        const std::uint32_t xs = smem_u32(xt);
        const float* xz = reinterpret_cast<const float*>(xt + 512u * N);
        auto half = [&](auto HC) {
#pragma unroll
        for (int Qi = 0; Qi < 2; ++Qi) {
            constexpr int H = decltype(HC)::value;
            const int Q = 2 * H + Qi;
            // outlier tile of this quarter: zero, scatter
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const std::uint32_t c = static_cast<std::uint32_t>(lane + 32 * j);  // 16 rows x 8 chunks of 16 B
                *reinterpret_cast<uint4*>(otile + (c >> 3) * kBmOStride + (c & 7u) * 16u) = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
            if (ofast) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (oit[j] != 0xFFFFFFFFu && (oit[j] >> 30) == static_cast<std::uint32_t>(Q))
                        *reinterpret_cast<unsigned short*>(otile + ((oit[j] >> 16) & 0x3FFFu)) =
                            static_cast<unsigned short>(oit[j] & 0xFFFFu);
            } else {
#pragma unroll 1
                for (std::uint32_t i = obeg + lane; i < oend; i += 32u) {
                    const std::uint32_t it = bm_outlier_item<BW>(ex_entry(ees, onf, p.cells, oc0, CELL, i));
                    if ((it >> 30) == static_cast<std::uint32_t>(Q))
                        *reinterpret_cast<unsigned short*>(otile + ((it >> 16) & 0x3FFFu)) =
                            static_cast<unsigned short>(it & 0xFFFFu);
                }
            }
            __syncwarp();
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int blk = 4 * Q + jj, tb = 4 * Qi + jj;  // block of the panel, of this half
                // B fragments of the codes (the batch-1 A-fragment registers): rows g (tile 0), g + 8 (tile 1)
                const int mu = blk, cidx = mu / G::MPC, mm = mu % G::MPC;
                const std::uint32_t* w = cw + G::CW * cidx;
                std::uint32_t a[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
                    const int i = rho * (G::NP / 2) + qq;
                    const int Bq = (BW * i) >> 3, pb = (BW * i) & 7;
                    a[r] = window<G::CW>(w, Bq) & ((MASK << pb) * 0x00010001u);
                }
                // outlier B fragments: rows 0-7 (k 0-7, 8-15), rows 8-15 (k 0-7, 8-15)
                std::uint32_t ob[4];
                ldsm_x4(smem_u32(otile) + o_off + static_cast<std::uint32_t>(jj) * 32u, ob);
                // s and -z of rows 2t, 2t + 1 (tile 0) and 8 + 2t, 9 + 2t (tile 1)
                const float4 tz0 = *reinterpret_cast<const float4*>(&tab[(tb * 8 + t) * 4]);      // rows 2t, 2t+1
                const float4 tz1 = *reinterpret_cast<const float4*>(&tab[(tb * 8 + 4 + t) * 4]);  // rows 8+2t, 9+2t
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    std::uint32_t xa[4];
                    ldsm_x4(xs + a_off + static_cast<std::uint32_t>(2 * blk) * 16u * N + static_cast<std::uint32_t>(m) * 256u, xa);
                    const float2 X2 = *reinterpret_cast<const float2*>(xz + blk * N + (m * 8 + g) * 2);  // batch 16m+g, +8
                    float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
                    mma16816(c0, xa, a[0], a[2]);
                    mma16816(c1, xa, a[1], a[3]);
                    mma16816(oacc[m][0], xa, ob[0], ob[1]);
                    mma16816(oacc[m][1], xa, ob[2], ob[3]);
                    // C (batch g / g + 8) x (rows 2t, 2t + 1): acc += s (C - z X), register-adjacent pairs
                    const float2 xg = make_float2(X2.x, X2.x), xh = make_float2(X2.y, X2.y);
                    const float2 s0 = make_float2(tz0.x, tz0.y), z0 = make_float2(tz0.z, tz0.w);
                    const float2 s1 = make_float2(tz1.x, tz1.y), z1 = make_float2(tz1.z, tz1.w);
                    float2* a0 = reinterpret_cast<float2*>(acc[m][0]);
                    float2* a1 = reinterpret_cast<float2*>(acc[m][1]);
                    a0[0] = ffma2(s0, ffma2(z0, xg, make_float2(c0[0], c0[1])), a0[0]);
                    a0[1] = ffma2(s0, ffma2(z0, xh, make_float2(c0[2], c0[3])), a0[1]);
                    a1[0] = ffma2(s1, ffma2(z1, xg, make_float2(c1[0], c1[1])), a1[0]);
                    a1[1] = ffma2(s1, ffma2(z1, xh, make_float2(c1[2], c1[3])), a1[1]);
                }
            }
        }
        };
        if (have) {
            if (hh == 0) half(std::integral_constant<int, 0>{});
            else half(std::integral_constant<int, 1>{});
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&x_free[bx]);
        if (have) {
            if (lane == 0) mbar_arrive(&rec_empty[ci][sl]);
        }
        if (u + 1 == u1 || P + 1 == p.Pn) {
            // tile end: y[batch][row] = (2^24 acc + O) 2^-e; lane: batches 16m + g (+8), rows 8nt + 2t (+1)
            float val[MT][2][4];
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int i = 0; i < 4; ++i) val[m][nt][i] = fmaf(acc[m][nt][i], 16777216.0f, oacc[m][nt][i]);
            // the two block halves of the row group: half 1 hands its sums to half 0 (fixed order)
            if (hh == 1) {
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
                        *reinterpret_cast<float4*>(xch + ((m * 2 + nt) * 32 + lane) * 4) =
                            make_float4(val[m][nt][0], val[m][nt][1], val[m][nt][2], val[m][nt][3]);
            }
            bar_sync_named(1 + (warp & 7), 64);
            if (hh == 0) {
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        const float4 o = *reinterpret_cast<const float4*>(xch + ((m * 2 + nt) * 32 + lane) * 4);
                        val[m][nt][0] += o.x;
                        val[m][nt][1] += o.y;
                        val[m][nt][2] += o.z;
                        val[m][nt][3] += o.w;
                    }
            }
            bar_sync_named(1 + (warp & 7), 64);  // the exchange is free again
            if (hh == 0) {
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[m][nt][i] = val[m][nt][i];
            }
            if (hh == 1) {
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[m][nt][i] = oacc[m][nt][i] = 0.f;
            }
        }
        if (hh == 0 && (u + 1 == u1 || P + 1 == p.Pn)) {
            const std::uint32_t rowu = 32u * static_cast<std::uint32_t>(ci) + 16u * static_cast<std::uint32_t>(uu);
            const std::uint32_t ua = u0 > T_ * p.Pn ? u0 : T_ * p.Pn;
            const bool whole = ua == T_ * p.Pn && u + 1 == (T_ + 1) * p.Pn;
            auto bcol_of = [&](int m, int i) { return static_cast<std::uint32_t>(16 * m + g + 8 * (i >> 1)); };
            auto rowl_of = [&](int nt, int i) { return rowu + static_cast<std::uint32_t>(8 * nt + 2 * t + (i & 1)); };
            float (&val)[MT][2][4] = acc;  // the halves' sum
            if (whole) {
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const std::uint32_t bcol = bcol_of(m, i), row = 128u * T_ + rowl_of(nt, i);
                            if (bcol < p.B && row < p.m)
                                p.y[static_cast<std::size_t>(bcol) * p.m + row] = val[m][nt][i] * __ldg(p.escale + bcol);
                        }
            } else {
                const uint2 gm = __ldg(reinterpret_cast<const uint2*>(p.gmap) + T_);
                const std::uint32_t ord = __ldg(p.cmap + 2u * v + (T_ == tile_of(u0) ? 0u : 1u));
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            __stcg(p.partial + (static_cast<std::size_t>(gm.x + ord) * N + bcol_of(m, i)) * 128u + rowl_of(nt, i),
                                   val[m][nt][i]);
                std::uint32_t prev = 0;
                __syncwarp();
                if (lane == 0)
                    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;"
                                 : "=r"(prev)
                                 : "l"(p.counters + 16u * T_ + static_cast<std::uint32_t>(warp & 7))
                                 : "memory");
                prev = __shfl_sync(0xffffffffu, prev, 0);
                __syncwarp();
                if (prev == gm.y - 1u) {  // last contributor: add the partial tiles in range order
#pragma unroll
                    for (int m = 0; m < MT; ++m)
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const std::uint32_t bcol = bcol_of(m, i), row = 128u * T_ + rowl_of(nt, i);
                                float sum = 0.f;
                                for (std::uint32_t j = 0; j < gm.y; ++j)
                                    sum += __ldcg(p.partial + (static_cast<std::size_t>(gm.x + j) * N + bcol) * 128u + rowl_of(nt, i));
                                if (bcol < p.B && row < p.m) p.y[static_cast<std::size_t>(bcol) * p.m + row] = sum * __ldg(p.escale + bcol);
                            }
                    if (lane == 0) p.counters[16u * T_ + static_cast<std::uint32_t>(warp & 7)] = 0;
                }
            }
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[m][nt][i] = oacc[m][nt][i] = 0.f;
        }
    }
}

// gemm_ex.cu: the instantiations (bw, bs in {2, 3, 4}; batch tiles 1, 2).
cudaError_t launch_gemm_bm(int bw, int bs, int mt, const ExParams& p, std::uint32_t smem, std::uint32_t smem_limit,
                           cudaStream_t st);
