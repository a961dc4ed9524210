// gemm_ex.cuh -- batched SpQR decode on the tcgen05 tensor cores with EXACT
// weight codes (batch >= 2).  Included by kernels.cuh (namespace spqr_dev);
// instantiated in gemm_ex.cu.
//
// Reference semantics: matvec(t, x, plan) (kernel.hpp:89-124) per batch
// column, y[r] = sum_k s(k,r) sum_{c in k} (q(r,c) - z(k,r)) x[c] + sum v x[col],
// s and z the stat_dequant values (quantizer.hpp:65-67, solver.hpp:129-141).
// Unlike the dequant-to-fp16 kernel (gemm_tc.cuh) no weight is ever rounded:
//
//   D_k  = Q_k X_k                 tcgen05.mma kind::f16, A = the 3-bit codes as
//                                  binary16 subnormals q 2^(p-24) (ONE mask per
//                                  code pair, tiled.hpp), B = x 2^(e - p_c): exact
//                                  products, one fp32 accumulator per 16-column
//                                  block k (a TMEM slot ring)
//   acc += s_k D_k                 the epilogue warps, packed f32x2 FMAs: the
//                                  per-(row, block) first-level scale in fp32
//   O   += V X + (-s z)(sum_c x)   one unscaled accumulator per 128-row tile:
//                                  the outliers (fp16 v 2^p_c, exact) through
//                                  kind::f16 and the zero-point terms through
//                                  kind::tf32 with hi/lo splits of both factors
//   y    = (2^24 acc + O) 2^-e     e: per batch column, max |x| 2^e in [2^14, 2^15)
//
// so the result carries fp32 rounding only (tolerance 1e-5 relative like the
// batch-1 kernel, not the 1e-3 of fp16 weights).
//
// Work unit: (128-row tile T = 4 cell rows, 256-column panel P) as in gemm_tc,
// cut into four 64-column STAGES (4 blocks each); CTA ranges, split tiles and
// partial slots are gemm_tc's (TcPlan).  Warps:
//   * 8 producer warps (cell row ci = w % 4, unit uu = w / 4): stream the
//     cell records (cp.async.bulk, two slots per cell row), decode the unit's
//     statistics once per cell, and per stage write the code tile (stmatrix,
//     K-major core matrices), the s table, the -s z tf32 tile and the outlier
//     tile (zeroed, then the cell's entries of this (unit, stage) scattered);
//   * 8 epilogue warps (TMEM lane quarter w % 4, column half): per stage read
//     the block accumulators (tcgen05.ld) and fold them into registers with
//     the s table; at a tile's end add O and write y (or a partial slot);
//   * 1 control warp: TMEM (512 columns: a 3-slot ring of 128-column block
//     accumulators + two O buffers), the x tiles of each stage (bulk copy of
//     xprep_ex's layout), the MMAs and their commits.

struct ExParams {
    const std::uint8_t* cells;      // cell records (batch-1 layout)
    const std::uint32_t* cell_off;  // [ncell+1]
    const std::uint32_t* cta_start; // [nv+1] first unit (T * Pn + P) of each range
    const std::uint32_t* gmap;      // [Tn][2] {partial slot base, contributing ranges}
    const std::uint32_t* cmap;      // [nv][2] ordinal of the range in its first / last tile
    const std::uint8_t* xpanels;    // [4 Pn][xb] x tiles per stage (xprep_ex)
    const float* escale;            // [N] 2^-e per batch column
    float* y;                       // [B][m]
    float* partial;                 // [slots][N][128]
    std::uint32_t* counters;        // [Tn][16], zero between launches
    std::uint32_t m, Pn, Gn, Tn, nv, B, N;
    std::uint32_t rec_cap, slot_bytes, pn_magic;
    std::uint32_t na;           // stage buffers (2 or 3)
    std::uint32_t lo;           // fp32 x: lo tiles present
    std::uint32_t xb;           // bytes of one stage's x tiles
    std::uint32_t stage_bytes;  // one stage buffer
};

// Stage buffer layout (bytes).  K-major core matrices (8 rows x 16 B):
//   codes / outliers (f16, 128 rows x 64 columns): (k/8) 2048 + (r/8) 128 + (r%8) 16 + (k%8) 2
//   -s z (tf32, 128 rows x 8: blocks 0-3 hi, then lo): (kk/4) 2048 + (r/8) 128 + (r%8) 16 + (kk%4) 4
//   s table: fp32 [128 rows][4 blocks]
//   x tiles (xprep_ex): BX f16 [N x 64] ((k/8) 16N + (n/8) 128 + (n%8) 16 + (k%8) 2),
//   BL (fp32 x: residual), BZ two tf32 tiles [N x 8] ((kk/4) 16N + (n/8) 128 + (n%8) 16 + (kk%4) 4):
//   tile 0 = {Xhi(blocks 0-3), Xhi(0-3)}, tile 1 = {Xlo(0-3), 0}
constexpr std::uint32_t kExOffAC = 0, kExOffAO = 16384, kExOffAZ = 32768, kExOffS = 36864, kExOffX = 38912;
constexpr std::uint32_t kExStaticMax = 1024;
constexpr int kExProd = 8, kExEpi = 8;
constexpr int kExThreads = 32 * (kExProd + kExEpi + 1);
__host__ __device__ constexpr std::uint32_t ex_xbytes(std::uint32_t N, bool lo) { return (lo ? 256u : 128u) * N + 64u * N; }
__host__ __device__ constexpr std::uint32_t ex_stage_bytes(std::uint32_t N, bool lo) {
    return (kExOffX + ex_xbytes(N, lo) + 127u) & ~127u;
}

namespace tc {
__device__ __forceinline__ void mma_tf32(std::uint32_t d_tmem, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                         std::uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 32 lanes x NE consecutive 32-bit columns (no wait: tcgen05.wait::ld separately)
template <int NE>
__device__ __forceinline__ void ld_cols(std::uint32_t taddr, float (&v)[NE]) {
    std::uint32_t r[NE];
    if constexpr (NE == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else if constexpr (NE == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else {
        static_assert(NE == 32, "ld_cols: 8, 16 or 32 columns");
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float tf32_rna(float v) {
    std::uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}
}  // namespace tc

// x tiles of every stage for batch column blockIdx.x (< N; zero beyond B):
// the column's power-of-two scale e first (block max), then per 16-column
// block k: BX = fp16(x 2^(e - p_c)) (+ BL = fp16 residual for fp32 x), and the
// block sum X = sum_c x 2^e split into tf32 hi / lo in the BZ tiles.
static __global__ void __launch_bounds__(1024) xprep_ex(const void* __restrict__ x, int x_f16, std::uint32_t n,
                                                        std::uint32_t B, std::uint32_t N, std::uint32_t Pn,
                                                        const std::uint32_t* __restrict__ order,
                                                        std::uint8_t* __restrict__ out, float* __restrict__ escale,
                                                        std::uint32_t xb, std::uint32_t lo, int bw) {
    pdl_launch();
    pdl_wait();
    __shared__ float red[32];
    const std::uint32_t nn = blockIdx.x;
    const bool live = nn < B;
    auto ld = [&](std::uint32_t c) -> float {
        const std::size_t off = static_cast<std::size_t>(nn) * n + c;
        return x_f16 ? __half2float(__ldg(static_cast<const __half*>(x) + off)) : __ldg(static_cast<const float*>(x) + off);
    };
    float mx = 0.f;
    if (live)
        for (std::uint32_t c = threadIdx.x; c < n; c += blockDim.x) mx = fmaxf(mx, fabsf(ld(c)));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    int e = 0;
    if (mx > 0.f && mx <= 3.4e38f) e = min(max(14 - ilogbf(mx), -126), 126);
    const float sc = __uint_as_float(static_cast<std::uint32_t>(127 + e) << 23);
    if (threadIdx.x == 0) escale[nn] = __uint_as_float(static_cast<std::uint32_t>(127 - e) << 23);
    const int mpc = T::mmas_per_container(bw);
    const std::uint32_t nb = 16u * Pn;
    const std::uint32_t ncol = (nn >> 3) * 128u + (nn & 7u) * 16u;
    for (std::uint32_t k = threadIdx.x; k < nb; k += blockDim.x) {
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
        std::uint8_t* base = out + static_cast<std::size_t>(k >> 2) * xb;
        const std::uint32_t bl = k & 3u;
        const int m_ = static_cast<int>(k & 7u) % mpc;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int pc = T::prescale_p(bw, 2 * m_ + hf);
            const float ps = __uint_as_float(static_cast<std::uint32_t>(127 - pc) << 23);
            std::uint32_t w[4], wl[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float a = v[8 * hf + 2 * q] * ps, b = v[8 * hf + 2 * q + 1] * ps;
                w[q] = pack_h2_rn(a, b);
                const __half2 h = u32_as_h2(w[q]);
                wl[q] = pack_h2_rn(a - __low2float(h), b - __high2float(h));
            }
            const std::uint32_t o = (2u * bl + hf) * 16u * N + ncol;
            *reinterpret_cast<uint4*>(base + o) = make_uint4(w[0], w[1], w[2], w[3]);
            if (lo) *reinterpret_cast<uint4*>(base + 128u * N + o) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
        }
        const float xh = tc::tf32_rna(X), xl = X - xh;
        std::uint8_t* bz = base + (lo ? 256u : 128u) * N;
        auto at = [&](std::uint32_t t, std::uint32_t kk) {
            return reinterpret_cast<float*>(bz + t * 32u * N + (kk >> 2) * 16u * N + ncol + (kk & 3u) * 4u);
        };
        *at(0, bl) = xh;
        *at(0, 4 + bl) = xh;
        *at(1, bl) = xl;
        *at(1, 4 + bl) = 0.f;
    }
}

template <int BW, int BS, int NE>
__global__ void __launch_bounds__(kExThreads, 1) gemm_ex(const ExParams p) {
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BS);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BS);
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr std::uint32_t SMASK = (1u << BS) - 1u;
    constexpr float kMagic = 8388608.0f;
    constexpr std::uint32_t KC_A = 2048u;
    constexpr std::uint32_t N = 2 * NE < 16 ? 16u : 2u * NE;  // MMA N
    constexpr int SBK = 128 / static_cast<int>(N) >= 4 ? 4 : 128 / static_cast<int>(N);  // blocks per TMEM slot
    constexpr int SPS = 4 / SBK;                                                            // slots per stage
    constexpr std::uint32_t O_COL = 384u;
    constexpr int CTRL = kExProd + kExEpi;

    extern __shared__ __align__(128) std::uint8_t smem[];
    __shared__ std::uint64_t rec_full[4][2], rec_empty[4][2], a_full[3], a_free[3], b_full[3], s_free[3], d_full[3],
        d_free[3], o_full[2], o_free[2];
    __shared__ std::uint32_t slot_r[4][2][2];
    __shared__ std::uint32_t tmem_base;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::uint32_t NA = p.na;
    std::uint8_t* recs = smem + NA * p.stage_bytes;  // [4 cell rows][2][slot_bytes]
    auto stage_buf = [&](std::uint32_t b) { return smem + b * p.stage_bytes; };

    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i)
            for (int k = 0; k < 2; ++k) {
                mbar_init(&rec_full[i][k], 1);
                mbar_init(&rec_empty[i][k], 2);  // the two producer warps of the cell row
            }
        for (int b = 0; b < 3; ++b) {
            mbar_init(&a_full[b], kExProd);
            mbar_init(&a_free[b], 1);
            mbar_init(&b_full[b], 1);
            mbar_init(&s_free[b], kExEpi);
            mbar_init(&d_full[b], 1);
            mbar_init(&d_free[b], kExEpi);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&o_full[b], 1);
            mbar_init(&o_free[b], kExEpi);
        }
        fence_mbar_init();
    }
    if (warp == CTRL) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    pdl_launch();
    const std::uint32_t tmem = tmem_base;
    const std::uint32_t v = blockIdx.x;
    const std::uint32_t u0 = __ldg(p.cta_start + v), u1 = __ldg(p.cta_start + v + 1);
    const std::uint32_t nst = 4u * (u1 - u0);  // stages of this range
    auto tile_of = [&](std::uint32_t u) { return p.Pn == 1u ? u : __umulhi(u, p.pn_magic); };

    if (warp == CTRL) {
        // ------------------------------------------------------------ control --
        if (lane == 0) {
            pdl_wait();  // xprep_ex has completed
            const std::uint32_t idesc_h = (1u << 4) | ((N >> 3) << 17) | ((128u >> 4) << 24);  // f16 x f16 -> f32
            const std::uint32_t idesc_t = idesc_h | (2u << 7) | (2u << 10);                    // tf32 x tf32 -> f32
            auto issue_b = [&](std::uint32_t s) {  // x tiles of stage s into its buffer
                const std::uint32_t b = s % NA;
                if (s >= NA) mbar_wait(&a_free[b], ((s / NA) - 1u) & 1u);
                const std::uint32_t u = u0 + (s >> 2), P = u - tile_of(u) * p.Pn;
                mbar_expect_tx(&b_full[b], p.xb);
                bulk_g2s(stage_buf(b) + kExOffX, p.xpanels + static_cast<std::size_t>(4u * P + (s & 3u)) * p.xb, p.xb,
                         &b_full[b]);
            };
            for (std::uint32_t s = 0; s + 1 < NA && s < nst; ++s) issue_b(s);
            std::uint32_t tile_i = 0, dslot = 0;
            const std::uint32_t lo = p.lo;
#pragma unroll 1
            for (std::uint32_t s = 0; s < nst; ++s) {
                const std::uint32_t b = s % NA, nb = s / NA;
                const std::uint32_t u = u0 + (s >> 2), P = u - tile_of(u) * p.Pn, Q = s & 3u;
                const bool first = Q == 0 && (s == 0 || P == 0);
                const bool last = Q == 3 && (u + 1 == u1 || P + 1 == p.Pn);
                mbar_wait(&a_full[b], nb & 1u);
                mbar_wait(&b_full[b], nb & 1u);
                if (first && tile_i >= 2) mbar_wait(&o_free[tile_i & 1u], ((tile_i >> 1) - 1u) & 1u);
                tc::fence_after();
                const std::uint32_t base = smem_u32(stage_buf(b));
                const std::uint32_t ac = base + kExOffAC, ao = base + kExOffAO, az = base + kExOffAZ;
                const std::uint32_t bx = base + kExOffX, bl = bx + 128u * N, bz = bx + (lo ? 256u : 128u) * N;
#pragma unroll
                for (int sl = 0; sl < SPS; ++sl) {
                    const std::uint32_t r = dslot % 3u;
                    if (dslot >= 3) {
                        mbar_wait(&d_free[r], ((dslot / 3u) - 1u) & 1u);
                        tc::fence_after();
                    }
#pragma unroll
                    for (int j = 0; j < SBK; ++j) {
                        const std::uint32_t blk = static_cast<std::uint32_t>(sl * SBK + j);
                        const std::uint32_t d = tmem + r * 128u + static_cast<std::uint32_t>(j) * N;
                        const std::uint64_t da = tc::smem_desc(ac + blk * 2u * KC_A, KC_A, 128u);
                        tc::mma_f16(d, da, tc::smem_desc(bx + blk * 32u * N, 16u * N, 128u), idesc_h, 0u);
                        if (lo) tc::mma_f16(d, da, tc::smem_desc(bl + blk * 32u * N, 16u * N, 128u), idesc_h, 1u);
                    }
                    tc::commit(&d_full[r]);
                    ++dslot;
                }
                const std::uint32_t o = tmem + O_COL + (tile_i & 1u) * N;
#pragma unroll
                for (std::uint32_t blk = 0; blk < 4; ++blk) {
                    const std::uint64_t da = tc::smem_desc(ao + blk * 2u * KC_A, KC_A, 128u);
                    tc::mma_f16(o, da, tc::smem_desc(bx + blk * 32u * N, 16u * N, 128u), idesc_h,
                                (first && blk == 0) ? 0u : 1u);
                    if (lo) tc::mma_f16(o, da, tc::smem_desc(bl + blk * 32u * N, 16u * N, 128u), idesc_h, 1u);
                }
                const std::uint64_t dz = tc::smem_desc(az, KC_A, 128u);
                tc::mma_tf32(o, dz, tc::smem_desc(bz, 16u * N, 128u), idesc_t, 1u);
                tc::mma_tf32(o, dz, tc::smem_desc(bz + 32u * N, 16u * N, 128u), idesc_t, 1u);
                tc::commit(&a_free[b]);  // stage buffer b (A, s table readers aside, x) free once these complete
                if (last) {
                    tc::commit(&o_full[tile_i & 1u]);
                    ++tile_i;
                }
                if (s + NA - 1 < nst) issue_b(s + NA - 1);
            }
        }
        __syncwarp();
    } else if (warp < kExProd) {
        // ---------------------------------------------------------- producers --
        const int ci = warp & 3, uu = warp >> 2;
        const int g = lane >> 2, t = lane & 3;
        std::uint8_t* ring = recs + static_cast<std::uint32_t>(ci) * 2u * p.slot_bytes;
        auto cell_of = [&](std::uint32_t u, std::uint32_t& q) {
            const std::uint32_t T_ = tile_of(u), P = u - T_ * p.Pn;
            const std::uint32_t Gq = 4u * T_ + static_cast<std::uint32_t>(ci);
            q = Gq * p.Pn + P;
            return Gq < p.Gn;
        };
        std::uint32_t nr0 = 0, nr1 = 0;
        auto load_off = [&](std::uint32_t u) {
            std::uint32_t q;
            if (uu == 0 && lane == 0 && u < u1 && cell_of(u, q)) {
                nr0 = __ldg(p.cell_off + q);
                nr1 = __ldg(p.cell_off + q + 1);
            }
        };
        auto issue = [&](std::uint32_t u, std::uint32_t k) {
            std::uint32_t q;
            if (uu == 0 && lane == 0 && cell_of(u, q)) {
                const std::uint32_t sl = k & 1u;
                if (k >= 2) mbar_wait(&rec_empty[ci][sl], ((k >> 1) - 1u) & 1u);
                slot_r[ci][sl][0] = nr0;
                slot_r[ci][sl][1] = nr1;
                const std::uint32_t nb = min(nr1 - nr0, p.rec_cap);
                mbar_expect_tx(&rec_full[ci][sl], nb);
                bulk_g2s(ring + sl * p.slot_bytes, p.cells + nr0, nb, &rec_full[ci][sl]);
            }
        };
        const std::uint32_t magic = 0x4B000000u;
        const std::uint32_t mq = static_cast<std::uint32_t>(lane >> 3);
        const std::uint32_t a_row = (mq >> 1) * KC_A + (4u * ci + 2u * uu + (mq & 1u)) * 128u + (lane & 7) * 16u;
        std::uint32_t k = 0;
        load_off(u0);
        if (u0 < u1) issue(u0, 0);
        load_off(u0 + 1);
#pragma unroll 1
        for (std::uint32_t u = u0; u < u1; ++u) {
            std::uint32_t q;
            const bool have = cell_of(u, q);
            if (have && u + 1 < u1) {
                issue(u + 1, k + 1);
                load_off(u + 2);
            }
            const std::uint32_t sl = k & 1u;
            const std::uint8_t* cell = ring + sl * p.slot_bytes;
            const std::uint8_t* unit = cell + uu * UNIT;
            std::uint32_t r0 = 0, r1 = 0;
            // per lane: rows g + 8 rho, blocks 8h + 2t + {0, 1}: s and the tf32 hi / lo of -s z
            float2 sv[2][2], zh[2][2], zl[2][2];
            std::uint32_t cw[G::LANE_WORDS];
            if (have) {
                mbar_wait(&rec_full[ci][sl], (k >> 1) & 1u);
                r0 = slot_r[ci][sl][0];
                r1 = slot_r[ci][sl][1];
                std::uint32_t st[2];
                load_stat_streams<BS>(unit + CODEB, lane, st);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
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
                        // stat_dequant, binary32 (quantizer.hpp:65-67)
                        const float s0 = __fmul_rn(Ss.x, __fsub_rn(cs.x, Zs.x)), s1 = __fmul_rn(Ss.y, __fsub_rn(cs.y, Zs.y));
                        const float z0 = __fmul_rn(Sz.x, __fsub_rn(cz.x, Zz.x)), z1 = __fmul_rn(Sz.y, __fsub_rn(cz.y, Zz.y));
                        const float n0 = -__fmul_rn(s0, z0), n1 = -__fmul_rn(s1, z1);
                        const float h0 = tc::tf32_rna(n0), h1 = tc::tf32_rna(n1);
                        sv[h][rho] = make_float2(s0, s1);
                        zh[h][rho] = make_float2(h0, h1);
                        zl[h][rho] = make_float2(n0 - h0, n1 - h1);
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
            }
            const std::uint32_t cnt = have ? (r1 - r0 - CELL) / 4u : 0u;
            const std::uint32_t nfast = have ? (min(r1 - r0, p.rec_cap) - CELL) / 4u : 0u;
            const std::uint32_t* es = reinterpret_cast<const std::uint32_t*>(cell + CELL);
            const std::uint32_t* eg = reinterpret_cast<const std::uint32_t*>(p.cells + r0 + CELL);
#pragma unroll
            for (int Q = 0; Q < 4; ++Q) {
                const std::uint32_t s = 4u * (u - u0) + Q;
                const std::uint32_t b = s % NA, nb = s / NA;
                if (nb) {
                    mbar_wait(&a_free[b], (nb - 1u) & 1u);
                    mbar_wait(&s_free[b], (nb - 1u) & 1u);
                }
                std::uint8_t* sb = stage_buf(b);
                if (have) {
                    // codes of blocks 4Q .. 4Q+3 of the unit: binary16 subnormals q 2^(p-24)
                    const std::uint32_t row_sa = smem_u32(sb + kExOffAC) + a_row;
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int mu = 4 * Q + jj, cidx = mu / G::MPC, mm = mu % G::MPC;
                        const std::uint32_t* w = cw + G::CW * cidx;
                        std::uint32_t a[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
                            const int i = rho * (G::NP / 2) + qq;
                            const int Bq = (BW * i) >> 3, pb = (BW * i) & 7;
                            a[r] = window<G::CW>(w, Bq) & ((MASK << pb) * 0x00010001u);
                        }
                        tc::stsm_x4(row_sa + 2u * jj * KC_A, a[0], a[1], a[2], a[3]);
                    }
                    // s table and -s z (tf32 hi in kk = block, lo in kk = 4 + block)
                    if ((t >> 1) == (Q & 1)) {
                        const int h = Q >> 1;
                        const std::uint32_t bl0 = 2u * (t & 1);
#pragma unroll
                        for (int rho = 0; rho < 2; ++rho) {
                            const std::uint32_t row = 32u * ci + 16u * uu + g + 8u * rho;
                            *reinterpret_cast<float2*>(sb + kExOffS + row * 16u + bl0 * 4u) = sv[h][rho];
                            std::uint8_t* zr = sb + kExOffAZ + (row >> 3) * 128u + (row & 7u) * 16u + bl0 * 4u;
                            *reinterpret_cast<float2*>(zr) = zh[h][rho];
                            *reinterpret_cast<float2*>(zr + KC_A) = zl[h][rho];
                        }
                    }
                    // outlier tile of this unit: zero, then this stage's entries (v 2^p_c, exact)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const std::uint32_t c = static_cast<std::uint32_t>(lane + 32 * j);
                        const std::uint32_t cm = c >> 3;
                        *reinterpret_cast<uint4*>(sb + kExOffAO + (cm >> 1) * KC_A +
                                                  (4u * ci + 2u * uu + (cm & 1u)) * 128u + (c & 7u) * 16u) =
                            make_uint4(0, 0, 0, 0);
                    }
                    __syncwarp();
#pragma unroll 1
                    for (std::uint32_t i = lane; i < cnt; i += 32u) {
                        const std::uint32_t e = i < nfast ? es[i] : __ldg(eg + i);
                        const std::uint32_t lr = e >> 24, col = (e >> 16) & 255u;
                        if ((lr >> 4) == static_cast<std::uint32_t>(uu) && (col >> 6) == static_cast<std::uint32_t>(Q)) {
                            const std::uint32_t row = 32u * ci + lr, kk = col & 63u;
                            const int pc = T::column_prescale(BW, col >> 4, col & 15u);
                            const float vv = h2f_bits(e & 0xffffu) * __uint_as_float(static_cast<std::uint32_t>(127 + pc) << 23);
                            const unsigned short hb = __half_as_ushort(__float2half_rn(vv));
                            const std::uint32_t sa = smem_u32(sb + kExOffAO) + (kk >> 3) * KC_A + (row >> 3) * 128u +
                                                     (row & 7u) * 16u + (kk & 7u) * 2u;
                            asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa), "h"(hb));
                        }
                    }
                }
                fence_proxy_async();  // generic-proxy smem writes -> tensor core reads
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[b]);
            }
            if (have) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&rec_empty[ci][sl]);
                ++k;
            }
        }
    } else {
        // ----------------------------------------------------------- epilogue --
        const int e = warp - kExProd;
        const std::uint32_t qe = static_cast<std::uint32_t>(warp & 3), ch = static_cast<std::uint32_t>(e >> 2);
        const std::uint32_t row_l = 32u * qe + lane;
        const std::uint32_t ta = tmem + ((32u * qe) << 16) + ch * NE;
        pdl_wait();  // y, partial slots and counters are ours; escale is written
        float acc[NE];
#pragma unroll
        for (int i = 0; i < NE; ++i) acc[i] = 0.f;
        std::uint32_t dslot = 0, tile_i = 0;
#pragma unroll 1
        for (std::uint32_t s = 0; s < nst; ++s) {
            const std::uint32_t b = s % NA, nb = s / NA;
            const std::uint32_t u = u0 + (s >> 2), T_ = tile_of(u), P = u - T_ * p.Pn;
            mbar_wait(&a_full[b], nb & 1u);
            const float4 s4 = *reinterpret_cast<const float4*>(stage_buf(b) + kExOffS + row_l * 16u);
            const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[b]);
#pragma unroll
            for (int sl = 0; sl < SPS; ++sl) {
                const std::uint32_t r = dslot % 3u;
                mbar_wait(&d_full[r], (dslot / 3u) & 1u);
                tc::fence_after();
                // the slot's blocks in groups of LB (<= 32 accumulator registers in flight)
                constexpr int LB = SBK * NE <= 32 ? SBK : 1;
#pragma unroll
                for (int j0 = 0; j0 < SBK; j0 += LB) {
                    float d[LB][NE];
#pragma unroll
                    for (int j = 0; j < LB; ++j)
                        tc::ld_cols<NE>(ta + r * 128u + static_cast<std::uint32_t>(j0 + j) * N, d[j]);
                    tc::wait_ld();
                    if (j0 + LB == SBK) {
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&d_free[r]);
                    }
#pragma unroll
                    for (int j = 0; j < LB; ++j) {
                        const float2 s2 = make_float2(sv[sl * SBK + j0 + j], sv[sl * SBK + j0 + j]);
#pragma unroll
                        for (int i = 0; i < NE; i += 2) {
                            const float2 a2 =
                                ffma2(s2, make_float2(d[j][i], d[j][i + 1]), make_float2(acc[i], acc[i + 1]));
                            acc[i] = a2.x;
                            acc[i + 1] = a2.y;
                        }
                    }
                }
                ++dslot;
            }
            if ((s & 3u) == 3u && (u + 1 == u1 || P + 1 == p.Pn)) {
                // tile end: y = (2^24 acc + O) 2^-e
                const std::uint32_t ob = tile_i & 1u;
                mbar_wait(&o_full[ob], (tile_i >> 1) & 1u);
                tc::fence_after();
                float o[NE];
                tc::ld_cols<NE>(ta + O_COL + ob * N, o);
                tc::wait_ld();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&o_free[ob]);
#pragma unroll
                for (int i = 0; i < NE; ++i) {
                    o[i] = fmaf(acc[i], 16777216.0f, o[i]);
                    acc[i] = 0.f;
                }
                const std::uint32_t row = 128u * T_ + row_l;
                const std::uint32_t ua = u0 > T_ * p.Pn ? u0 : T_ * p.Pn;
                const bool whole = ua == T_ * p.Pn && u + 1 == (T_ + 1) * p.Pn;
                if (whole) {
#pragma unroll
                    for (int i = 0; i < NE; ++i) {
                        const std::uint32_t bcol = ch * NE + i;
                        if (bcol < p.B && row < p.m) p.y[static_cast<std::size_t>(bcol) * p.m + row] = o[i] * __ldg(p.escale + bcol);
                    }
                } else {
                    const uint2 gm = __ldg(reinterpret_cast<const uint2*>(p.gmap) + T_);
                    const std::uint32_t ord = __ldg(p.cmap + 2u * v + (T_ == tile_of(u0) ? 0u : 1u));
#pragma unroll
                    for (int i = 0; i < NE; ++i)
                        __stcg(p.partial + (static_cast<std::size_t>(gm.x + ord) * N + ch * NE + i) * 128u + row_l, o[i]);
                    std::uint32_t prev = 0;
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;"
                                     : "=r"(prev)
                                     : "l"(p.counters + 16u * T_ + static_cast<std::uint32_t>(e))
                                     : "memory");
                    prev = __shfl_sync(0xffffffffu, prev, 0);
                    __syncwarp();
                    if (prev == gm.y - 1u) {  // last contributor: add the partial tiles in range order
#pragma unroll 1
                        for (std::uint32_t i = 0; i < NE; ++i) {
                            const std::uint32_t bcol = ch * NE + i;
                            if (bcol >= p.B) break;
                            float sum = 0.f;
                            for (std::uint32_t j = 0; j < gm.y; ++j)
                                sum += __ldcg(p.partial + (static_cast<std::size_t>(gm.x + j) * N + bcol) * 128u + row_l);
                            if (row < p.m) p.y[static_cast<std::size_t>(bcol) * p.m + row] = sum * __ldg(p.escale + bcol);
                        }
                        if (lane == 0) p.counters[16u * T_ + static_cast<std::uint32_t>(e)] = 0;
                    }
                }
                ++tile_i;
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == CTRL) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// gemm_ex.cu: the instantiations (bw, bs in {2, 3, 4}; ne in {8, 16, 32}).
cudaError_t launch_gemm_ex(int bw, int bs, int ne, const ExParams& p, std::uint32_t smem, std::uint32_t smem_limit,
                           cudaStream_t st);
