// gemm_ex.cuh -- batched SpQR decode on the tcgen05 tensor cores with EXACT
// weight codes (batch >= 2).  Included by kernels.cuh (namespace spqr_dev);
// instantiated in gemm_ex.cu.
//
// Reference semantics: matvec(t, x, plan) (kernel.hpp:89-124) per batch
// column, y[r] = sum_k s(k,r) sum_{c in k} (q(r,c) - z(k,r)) x[c] + sum v x[col],
// s and z the stat_dequant values (quantizer.hpp:65-67, solver.hpp:129-141).
// Unlike the dequant-to-fp16 kernel (gemm_tc.cuh) no weight is ever rounded:
//
//   D_k  = Q_k X_k         tcgen05.mma kind::f16, A in TMEM: the codes as
//                          binary16 subnormals q 2^(p-24) (ONE mask per code
//                          pair, tiled.hpp; tcgen05.st straight from the
//                          registers), B = x 2^(e - p_c): exact products, one
//                          fp32 accumulator per 16-column block k
//   acc += (2^24 s_k) D_k  fp32, in the registers of the warp that owns the rows
//   O   += V X + (-s z) X_sum   one unscaled accumulator per tile: the outliers
//                          (kind::f16, A = fp16 v 2^p_c scattered into a zeroed
//                          shared tile: exact products) and the zero-point
//                          terms (kind::tf32, A = hi / lo of -s z per (row,
//                          block) in TMEM, B = hi / lo of the block sums
//                          X_sum = sum_c x 2^e)
//   y    = (acc + O) 2^-e  e: per batch column, max |x| 2^e in [2^14, 2^15)
//
// so the result carries fp32 rounding only (the batch-1 kernel's 1e-5, not
// the 1e-3 of fp16 weights).
//
// Work unit: (128-row tile T = 4 cell rows, 256-column panel P) as in gemm_tc,
// cut into four 64-column STAGES (4 blocks each); CTA ranges, split tiles and
// partial slots are gemm_tc's (TcPlan).  Warps:
//   * 8 workers, warp w = cell row ci = w % 4, unit uu = w / 4: the 16 rows
//     32 ci + 16 uu of the tile, TMEM lanes of its own quarter.  Per stage a
//     worker decodes (once per cell) and stores its code tile and -s z tile
//     into TMEM, then folds the PREVIOUS stage's block accumulators of its
//     rows into registers (tcgen05.ld in the same fragment layout, the s
//     values by shuffles from the lanes that decoded them); at a tile's end
//     it adds O and writes y (or a partial slot).  The outlier tile of its
//     rows is zeroed and scattered in shared memory while it produces.
//     Warp 0 also streams each stage's x tiles (bulk copies, NX - 2 stages
//     ahead), the first warp of a cell row the cell records (two ahead).
//   * 1 control warp: TMEM allocation and the MMAs (the whole warp runs the
//     loop so the operands stay warp-uniform; small MMAs issued from one lane
//     with per-lane operands cost ~3x, tools/umma_bench.cu).

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
    std::uint32_t lo;  // fp32 x: residual tiles present
    std::uint32_t xb;  // bytes of one stage's x tiles
    const std::uint32_t* usplit;  // [ncell] (gemm_bm) first outlier entry of rows 16.. | end of the real entries << 16
};

// Per cell: the index of the first outlier entry of the second unit (local
// rows >= 16) in its (row, col)-sorted list and the end of the real entries
// (before the 16-B padding, row 255) -- computed once at load.
static __global__ void cell_unit_split(const std::uint8_t* __restrict__ cells, const std::uint32_t* __restrict__ off,
                                       std::uint32_t ncell, std::uint32_t cell_bytes, std::uint32_t* __restrict__ out) {
    const std::uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ncell) return;
    const std::uint32_t r0 = off[q], cnt = (off[q + 1] - r0 - cell_bytes) / 4u;
    const std::uint32_t* e = reinterpret_cast<const std::uint32_t*>(cells + r0 + cell_bytes);
    auto lower = [&](std::uint32_t key) {
        std::uint32_t lo = 0, hi = cnt;
        while (lo < hi) {
            const std::uint32_t mid = (lo + hi) >> 1;
            if ((e[mid] >> 24) < key) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    out[q] = lower(16u) | (lower(32u) << 16);
}

// TMEM code tile of a stage (tcgen05.st in the batch-1 register layout):
// column 2t + w of a block holds the codes of columns 8w + 2t + {0, 1}, so the
// x tile uses the column order K' = 4t + 2w + h within each block.
// x tiles of a stage (xprep_ex, bytes):
//   BX  f16 [N x 64 K'] K-major core matrices: (k/8) 16N + (n/8) 128 + (n%8) 16 + (k%8) 2
//   BL  (fp32 x) the fp16 residuals, same layout
//   BZ  two tf32 [N x 8] tiles, (kk/4) 16N + (n/8) 128 + (n%8) 16 + (kk%4) 4:
//       tile 0 = {Xhi(blocks 0-3), Xhi(0-3)}, tile 1 = {Xlo(0-3), 0}
// Outlier tile of a stage (shared, f16 128 rows x 64 columns K'):
//   (k/8) 2048 + (r/8) 128 + (r%8) 16 + (k%8) 2
__host__ __device__ constexpr std::uint32_t ex_bz_off(std::uint32_t N, bool lo) { return (lo ? 256u : 128u) * N; }
__host__ __device__ constexpr std::uint32_t ex_xbytes(std::uint32_t N, bool lo) {
    return (ex_bz_off(N, lo) + 64u * N + 127u) & ~127u;
}
constexpr std::uint32_t kExAOBytes = 16384;
constexpr std::uint32_t kExStaticMax = 6144;
constexpr std::uint32_t kExRecSlots = 4;  // record slots per cell row: two of lookahead, current, previous
constexpr int kExWork = 8;
constexpr int kExThreads = 32 * (kExWork + 1);
// stages in flight (TMEM code tiles) and x tile buffers, by MMA N
__host__ __device__ constexpr std::uint32_t ex_na(std::uint32_t N) { return N == 16 ? 4u : (N == 32 ? 3u : 2u); }
__host__ __device__ constexpr std::uint32_t ex_nx(std::uint32_t N) { return ex_na(N) + 3u; }

namespace tc {
// 16 TMEM lanes x C x 256 bits, registers 4j .. 4j+3 = (lane g, column 8j + 2t),
// (g, 8j + 2t + 1), (g + 8, 8j + 2t), (g + 8, 8j + 2t + 1): the m16n8 fragment layout
template <int C>
__device__ __forceinline__ void ld16(std::uint32_t taddr, std::uint32_t (&r)[4 * C]) {
    if constexpr (C == 2) {
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else if constexpr (C == 4) {
        asm volatile(
            "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else {
        static_assert(C == 8, "ld16: 2, 4 or 8 chunks");
        asm volatile(
            "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
    }
}
__device__ __forceinline__ void st16_x1(std::uint32_t taddr, std::uint32_t r0, std::uint32_t r1, std::uint32_t r2,
                                        std::uint32_t r3) {
    asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r0), "r"(r1), "r"(r2),
                 "r"(r3)
                 : "memory");
}
__device__ __forceinline__ void st16_x4(std::uint32_t taddr, const std::uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// issued by a whole warp (warp-uniform operands stay in uniform registers); one elected lane issues
template <int KIND>  // 0: f16, 1: tf32
__device__ __forceinline__ void mma_ts(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t b,
                                       std::uint32_t idesc, std::uint32_t accumulate) {
    if constexpr (KIND == 0)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate)
            : "memory");
}
__device__ __forceinline__ float tf32_rna(float v) {
    std::uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}
// block column K' (TMEM / x tile order) of a block's true column kk, and back
__host__ __device__ __forceinline__ constexpr std::uint32_t kprime(std::uint32_t kk) {
    return 4u * ((kk >> 1) & 3u) + 2u * (kk >> 3) + (kk & 1u);
}
__host__ __device__ __forceinline__ constexpr std::uint32_t ktrue(std::uint32_t kp) {
    return 8u * ((kp >> 1) & 1u) + 2u * (kp >> 2) + (kp & 1u);
}
}  // namespace tc

// x tiles of every stage.  Grid (N, S): CTA (n, s) finds column n's
// power-of-two scale e (the column max, recomputed by each of the S CTAs of
// the column: x is L2-resident) and writes the 16-column blocks s, s + S, ...
// Columns n >= B are zero.
static __global__ void __launch_bounds__(256) xprep_ex(const void* __restrict__ x, int x_f16, std::uint32_t n,
                                                       std::uint32_t B, std::uint32_t N, std::uint32_t Pn,
                                                       const std::uint32_t* __restrict__ order,
                                                       std::uint8_t* __restrict__ out, float* __restrict__ escale,
                                                       std::uint32_t xb, std::uint32_t lo, int bw) {
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
        const std::size_t esz = x_f16 ? 2 : 4;
        const bool vec = (reinterpret_cast<std::uintptr_t>(x) & 15u) == 0 && (n * esz) % 16u == 0;
        if (vec) {  // 16-B loads, four in flight per thread
            const uint4* xv = reinterpret_cast<const uint4*>(static_cast<const std::uint8_t*>(x) + col0 * esz);
            const std::uint32_t nv = static_cast<std::uint32_t>(n * esz / 16u);
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
        std::uint8_t* base = out + static_cast<std::size_t>(k >> 2) * xb;
        const std::uint32_t bl = k & 3u;
        const int m_ = static_cast<int>(k & 7u) % mpc;
        // pre-scaled by 2^-p_c (p_c by the true column's k half), in the block order K' of the code tile
        const float ps0 = __uint_as_float(static_cast<std::uint32_t>(127 - T::prescale_p(bw, 2 * m_)) << 23);
        const float ps1 = __uint_as_float(static_cast<std::uint32_t>(127 - T::prescale_p(bw, 2 * m_ + 1)) << 23);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            std::uint32_t w[4], wl[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k0 = static_cast<int>(tc::ktrue(8 * hf + 2 * q)), k1 = static_cast<int>(tc::ktrue(8 * hf + 2 * q + 1));
                const float a = v[k0] * (k0 >= 8 ? ps1 : ps0), b = v[k1] * (k1 >= 8 ? ps1 : ps0);
                w[q] = pack_h2_rn(a, b);
                const __half2 h = u32_as_h2(w[q]);
                wl[q] = pack_h2_rn(a - __low2float(h), b - __high2float(h));
            }
            const std::uint32_t o = (2u * bl + hf) * 16u * N + ncol;
            *reinterpret_cast<uint4*>(base + o) = make_uint4(w[0], w[1], w[2], w[3]);
            if (lo) *reinterpret_cast<uint4*>(base + 128u * N + o) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
        }
        // block sum, tf32 hi / lo (BZ)
        const float xh = tc::tf32_rna(X), xl = X - xh;
        std::uint8_t* bz = base + ex_bz_off(N, lo);
        auto at = [&](std::uint32_t t, std::uint32_t kk) {
            return reinterpret_cast<float*>(bz + t * 32u * N + (kk >> 2) * 16u * N + ncol + (kk & 3u) * 4u);
        };
        *at(0, bl) = xh;
        *at(0, 4 + bl) = xh;
        *at(1, bl) = xl;
        *at(1, 4 + bl) = 0.f;
    }
}

// outlier entry i of a cell: the record slot's copy, or (beyond the slot, rare) HBM through a
// volatile load the compiler cannot hoist out of the branch
__device__ __forceinline__ std::uint32_t ex_entry(const std::uint32_t* slot, std::uint32_t nfast,
                                                  const std::uint8_t* cells, std::uint32_t r0, std::uint32_t cell,
                                                  std::uint32_t i) {
    if (i < nfast) return slot[i];
    std::uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(cells + r0 + cell + 4ull * i));
    return v;
}

// an outlier entry (value16 | col << 16 | local row << 24) of cell row ci as
// quarter << 30 | byte offset in the stage's outlier tile << 16 | fp16(v 2^p_c)
template <int BW>
__device__ __forceinline__ std::uint32_t ex_outlier_item(std::uint32_t en, int ci) {
    const std::uint32_t col = (en >> 16) & 255u;
    const std::uint32_t row = 32u * static_cast<std::uint32_t>(ci) + (en >> 24);
    const std::uint32_t kk = (col & 48u) + tc::kprime(col & 15u);
    const int pc = T::column_prescale(BW, col >> 4, col & 15u);
    const float vv = h2f_bits(en & 0xffffu) * __uint_as_float(static_cast<std::uint32_t>(127 + pc) << 23);
    const std::uint32_t off = (kk >> 3) * 2048u + (row >> 3) * 128u + (row & 7u) * 16u + (kk & 7u) * 2u;
    return ((col >> 6) << 30) | (off << 16) | __half_as_ushort(__float2half_rn(vv));
}

#ifdef SPQR_TIMELINE
// tools-only (tools/ex_timeline.py): per warp ns spent in each wait class
#define EX_W(i, expr)                           \
    {                                           \
        const unsigned long long t0_ = gtime(); \
        expr;                                   \
        tw[i] += gtime() - t0_;                 \
    }
#else
#define EX_W(i, expr) expr;
#endif
template <int BW, int BS, int N>
__global__ void __launch_bounds__(kExThreads, 1) gemm_ex(const ExParams p) {
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BS);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BS);
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr std::uint32_t SMASK = (1u << BS) - 1u;
    constexpr float kMagic = 8388608.0f;
    constexpr std::uint32_t NA = ex_na(N), NX = ex_nx(N);
    constexpr int SBK = 128 / N >= 4 ? 4 : 128 / N;  // blocks per accumulator slot
    constexpr int SPS = 4 / SBK;                       // slots per stage
    constexpr std::uint32_t W = static_cast<std::uint32_t>(SBK * N);
    constexpr int C = N / 8;  // 256-bit chunks per accumulator row
    constexpr std::uint32_t NS = kExRecSlots;
    // TMEM: accumulator slots at 0, O (2 x N) after them, -s z tiles (8 columns) and code
    // tiles (32 columns) at the top
    constexpr std::uint32_t CODE_COL = 512u - 32u * NA;
    constexpr std::uint32_t AZ_COL = CODE_COL - 8u * NA;
    constexpr std::uint32_t R = (AZ_COL - 2u * N) / W > 4u ? 4u : (AZ_COL - 2u * N) / W;
    constexpr std::uint32_t O_COL = R * W;
    static_assert(R >= 2, "TMEM plan");
    constexpr int CTRL = kExWork;

    extern __shared__ __align__(128) std::uint8_t smem[];  // [NX][xb] x tiles, [NA][16 KB] outlier tiles, records
    __shared__ std::uint64_t rec_full[4][NS], rec_empty[4][NS], a_full[NA], a_free[NA], x_full[NX], x_free[NX],
        d_full[R], d_free[R], o_full[2], o_free[2];
    __shared__ std::uint32_t slot_r[4][NS][2];
    __shared__ std::uint32_t tmem_base;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef SPQR_TIMELINE
    unsigned long long tw[6] = {0, 0, 0, 0, 0, 0};
    const unsigned long long t_start = gtime();
#endif
    std::uint8_t* xbuf = smem;
    std::uint8_t* aobuf = smem + NX * p.xb;
    std::uint8_t* recs = aobuf + NA * kExAOBytes;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i)
            for (std::uint32_t k = 0; k < NS; ++k) {
                mbar_init(&rec_full[i][k], 1);
                mbar_init(&rec_empty[i][k], 2);  // the cell row's two workers
            }
        for (std::uint32_t b = 0; b < NA; ++b) {
            mbar_init(&a_full[b], kExWork);
            mbar_init(&a_free[b], 1);
        }
        for (std::uint32_t b = 0; b < NX; ++b) {
            mbar_init(&x_full[b], 1);
            mbar_init(&x_free[b], 1);  // the MMAs' commit
        }
        for (std::uint32_t r = 0; r < R; ++r) {
            mbar_init(&d_full[r], 1);
            mbar_init(&d_free[r], kExWork);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&o_full[b], 1);
            mbar_init(&o_free[b], kExWork);
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
    auto tile_end = [&](std::uint32_t s) {  // stage s is its tile's last in this range
        const std::uint32_t u = u0 + (s >> 2);
        return (s & 3u) == 3u && (u + 1 == u1 || u + 1 - tile_of(u) * p.Pn == p.Pn);
    };

    if (warp == CTRL) {
        // ------------------------------------------------------------ control --
        const std::uint32_t idesc_h = (1u << 4) | (static_cast<std::uint32_t>(N >> 3) << 17) | ((128u >> 4) << 24);
        const std::uint32_t idesc_t = idesc_h | (2u << 7) | (2u << 10);
        const std::uint32_t lo = p.lo;
        std::uint32_t dslot = 0, tile_i = 0;
        bool first = true;
#pragma unroll 1
        for (std::uint32_t s = 0; s < nst; ++s) {
            const std::uint32_t b = s % NA, bx = s % NX;
            EX_W(0, mbar_wait(&a_full[b], (s / NA) & 1u))
            EX_W(1, mbar_wait(&x_full[bx], (s / NX) & 1u))
            if (first && tile_i >= 2) EX_W(4, mbar_wait(&o_free[tile_i & 1u], ((tile_i >> 1) - 1u) & 1u))
            tc::fence_after();
            const std::uint32_t xs = smem_u32(xbuf + bx * p.xb);
            const std::uint32_t bxs = xs, bls = xs + 128u * N, bzs = xs + ex_bz_off(N, lo);
            const std::uint32_t at = tmem + CODE_COL + b * 32u;
#pragma unroll
            for (int sl = 0; sl < SPS; ++sl) {
                const std::uint32_t r = dslot % R;
                if (dslot >= R) {
                    EX_W(2, mbar_wait(&d_free[r], ((dslot / R) - 1u) & 1u))
                    tc::fence_after();
                }
#pragma unroll
                for (int j = 0; j < SBK; ++j) {
                    const std::uint32_t blk = static_cast<std::uint32_t>(sl * SBK + j);
                    const std::uint32_t d = tmem + r * W + static_cast<std::uint32_t>(j * N);
                    tc::mma_ts<0>(d, at + blk * 8u, tc::smem_desc(bxs + blk * 32u * N, 16u * N, 128u), idesc_h, 0u);
                    if (lo) tc::mma_ts<0>(d, at + blk * 8u, tc::smem_desc(bls + blk * 32u * N, 16u * N, 128u), idesc_h, 1u);
                }
                tc::commit_e(&d_full[r]);
                ++dslot;
            }
            // outliers and zero-point terms of the stage's 4 blocks into O
            const std::uint32_t o = tmem + O_COL + (tile_i & 1u) * N;
            const std::uint32_t ao = smem_u32(aobuf + b * kExAOBytes);
#pragma unroll
            for (std::uint32_t blk = 0; blk < 4; ++blk) {
                const std::uint64_t da = tc::smem_desc(ao + blk * 4096u, 2048u, 128u);
                tc::mma_f16_e(o, da, tc::smem_desc(bxs + blk * 32u * N, 16u * N, 128u), idesc_h,
                              (first && blk == 0) ? 0u : 1u);
                if (lo) tc::mma_f16_e(o, da, tc::smem_desc(bls + blk * 32u * N, 16u * N, 128u), idesc_h, 1u);
            }
            const std::uint32_t az = tmem + AZ_COL + b * 8u;
            tc::mma_ts<1>(o, az, tc::smem_desc(bzs, 16u * N, 128u), idesc_t, 1u);
            tc::mma_ts<1>(o, az, tc::smem_desc(bzs + 32u * N, 16u * N, 128u), idesc_t, 1u);
            first = false;
            tc::commit_e(&a_free[b]);   // code and -s z tiles of buffer b
            tc::commit_e(&x_free[bx]);  // the MMAs' share of the x tiles
            if (tile_end(s)) {
                tc::commit_e(&o_full[tile_i & 1u]);
                ++tile_i;
                first = true;
            }
        }
    } else {
        // ------------------------------------------------------------ workers --
        const int ci = warp & 3, uu = warp >> 2;
        const int g = lane >> 2, t = lane & 3;
        std::uint8_t* ring = recs + static_cast<std::uint32_t>(ci) * NS * p.slot_bytes;
        auto cell_of = [&](std::uint32_t u, std::uint32_t& q) {
            const std::uint32_t T_ = tile_of(u), P = u - T_ * p.Pn;
            const std::uint32_t Gq = 4u * T_ + static_cast<std::uint32_t>(ci);
            q = Gq * p.Pn + P;
            return Gq < p.Gn;
        };
        // records: cell u of this cell row is record k = u - u0 (a cell row stays valid up to the
        // layer's last tile), slot k % NS; two cells of lookahead
        std::uint32_t nr0 = 0, nr1 = 0;
        auto load_off = [&](std::uint32_t u) {
            std::uint32_t q;
            if (uu == 0 && lane == 0 && u < u1 && cell_of(u, q)) {
                nr0 = __ldg(p.cell_off + q);
                nr1 = __ldg(p.cell_off + q + 1);
            }
        };
        auto issue_rec = [&](std::uint32_t u) {
            std::uint32_t q;
            if (uu == 0 && lane == 0 && u < u1 && cell_of(u, q)) {
                const std::uint32_t k = u - u0, sl = k % NS;
                if (k >= NS) mbar_wait(&rec_empty[ci][sl], ((k / NS) - 1u) & 1u);
                slot_r[ci][sl][0] = nr0;
                slot_r[ci][sl][1] = nr1;
                const std::uint32_t nb = min(nr1 - nr0, p.rec_cap);
                mbar_expect_tx(&rec_full[ci][sl], nb);
                bulk_g2s(ring + sl * p.slot_bytes, p.cells + nr0, nb, &rec_full[ci][sl]);
            }
        };
        // x tiles of stage s (warp 0): buffer s % NX once the MMAs and every worker are done with stage s - NX
        auto issue_x = [&](std::uint32_t s) {
            if (warp == 0 && s < nst) {
                const std::uint32_t bx = s % NX;
                if (s >= NX) mbar_wait(&x_free[bx], ((s / NX) - 1u) & 1u);
                if (lane == 0) {
                    const std::uint32_t u = u0 + (s >> 2), P = u - tile_of(u) * p.Pn;
                    mbar_expect_tx(&x_full[bx], p.xb);
                    bulk_g2s(xbuf + bx * p.xb, p.xpanels + static_cast<std::size_t>(4u * P + (s & 3u)) * p.xb, p.xb,
                             &x_full[bx]);
                }
                __syncwarp();
            }
        };
        constexpr std::uint32_t XLA = NX - 2;  // x tiles issued this many stages ahead
        const std::uint32_t magic = 0x4B000000u;
        const std::uint32_t lanes16 = (32u * ci + 16u * uu) << 16;  // this worker's 16 TMEM lanes
        load_off(u0);
        issue_rec(u0);
        load_off(u0 + 1);
        issue_rec(u0 + 1);
        load_off(u0 + 2);
        if (warp == 0) {
            pdl_wait();  // xprep_ex has completed (the x tiles)
            for (std::uint32_t s = 0; s < XLA; ++s) issue_x(s);
        }
        pdl_wait();  // y, partial slots and counters are ours

        // this lane's statistics of the current cell (producer layout: rows g + 8 rho,
        // blocks 8h + 2t + {0, 1}): 2^24 s and -s z
        float2 sv[2][2], nz[2][2], sv_prev[2][2];
        std::uint32_t obeg = 0, oend = 0, onf = 0, oc0 = 0;  // this unit's outlier entries in the current cell
        std::uint32_t oit[4];  // ... precomputed (<= 128 of them): quarter << 30 | tile offset << 16 | fp16
        bool ofast = true;
        std::uint32_t cw[G::LANE_WORDS];
        float acc[N / 2];  // rows g, g + 8 x columns 2t + {0, 1} + 8j
#pragma unroll
        for (int i = 0; i < N / 2; ++i) acc[i] = 0.f;
        std::uint32_t dslot = 0, tile_i = 0;

        // fold stage s: block accumulators, outliers, tile end
        auto epilogue = [&](std::uint32_t s, const float2 (&svs)[2][2]) {
            const std::uint32_t k = s >> 2;
            const std::uint32_t u = u0 + k, T_ = tile_of(u), Q = s & 3u;
            // s of rows g, g + 8 for the stage's blocks 4Q + blk: from lane 4g + 2(Q&1) + (blk >> 1), half Q >> 1
            float s4[2][4];
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
                const int src = 4 * g + 2 * static_cast<int>(Q & 1u) + (blk >> 1);
#pragma unroll
                for (int rho = 0; rho < 2; ++rho) {
                    const float2 a = (Q >> 1) ? svs[1][rho] : svs[0][rho];
                    const float val = (blk & 1) ? a.y : a.x;
                    s4[rho][blk] = __shfl_sync(0xffffffffu, val, src);
                }
            }
#pragma unroll
            for (int sl = 0; sl < SPS; ++sl) {
                const std::uint32_t r = dslot % R;
                EX_W(1, mbar_wait(&d_full[r], (dslot / R) & 1u))
                tc::fence_after();
#pragma unroll
                for (int j = 0; j < SBK; ++j) {
                    const int blk = sl * SBK + j;
                    std::uint32_t d[4 * C];
                    tc::ld16<C>(tmem + lanes16 + r * W + static_cast<std::uint32_t>(j * N), d);
                    tc::wait_ld();
                    if (j == SBK - 1) {
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&d_free[r]);
                    }
                    const float2 sg = make_float2(s4[0][blk], s4[0][blk]), sh = make_float2(s4[1][blk], s4[1][blk]);
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        const float2 a0 = ffma2(sg, make_float2(__uint_as_float(d[4 * c]), __uint_as_float(d[4 * c + 1])),
                                                make_float2(acc[4 * c], acc[4 * c + 1]));
                        const float2 a1 = ffma2(sh, make_float2(__uint_as_float(d[4 * c + 2]), __uint_as_float(d[4 * c + 3])),
                                                make_float2(acc[4 * c + 2], acc[4 * c + 3]));
                        acc[4 * c] = a0.x;
                        acc[4 * c + 1] = a0.y;
                        acc[4 * c + 2] = a1.x;
                        acc[4 * c + 3] = a1.y;
                    }
                }
                ++dslot;
            }
            __syncwarp();
            if (tile_end(s)) {
                // y = (acc + O) 2^-e for this worker's 16 rows
                const std::uint32_t ob = tile_i & 1u;
                EX_W(2, mbar_wait(&o_full[ob], (tile_i >> 1) & 1u))
                tc::fence_after();
                std::uint32_t od[4 * C];
                tc::ld16<C>(tmem + lanes16 + O_COL + ob * N, od);
                tc::wait_ld();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&o_free[ob]);
#pragma unroll
                for (int i = 0; i < 4 * C; ++i) acc[i] += __uint_as_float(od[i]);
                const std::uint32_t rowl = 32u * ci + 16u * uu + g;  // + 8 rho
                const std::uint32_t ua = u0 > T_ * p.Pn ? u0 : T_ * p.Pn;
                const bool whole = ua == T_ * p.Pn && u + 1 == (T_ + 1) * p.Pn;
                auto col_of = [&](int i) { return static_cast<std::uint32_t>(8 * (i >> 2) + 2 * t + (i & 1)); };
                auto row_of = [&](int i) { return rowl + 8u * ((i >> 1) & 1); };
                if (whole) {
#pragma unroll
                    for (int i = 0; i < 4 * C; ++i) {
                        const std::uint32_t bcol = col_of(i), row = 128u * T_ + row_of(i);
                        if (bcol < p.B && row < p.m)
                            p.y[static_cast<std::size_t>(bcol) * p.m + row] = acc[i] * __ldg(p.escale + bcol);
                    }
                } else {
                    const uint2 gm = __ldg(reinterpret_cast<const uint2*>(p.gmap) + T_);
                    const std::uint32_t ord = __ldg(p.cmap + 2u * v + (T_ == tile_of(u0) ? 0u : 1u));
#pragma unroll
                    for (int i = 0; i < 4 * C; ++i)
                        __stcg(p.partial + (static_cast<std::size_t>(gm.x + ord) * N + col_of(i)) * 128u + row_of(i), acc[i]);
                    std::uint32_t prev = 0;
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;"
                                     : "=r"(prev)
                                     : "l"(p.counters + 16u * T_ + static_cast<std::uint32_t>(warp))
                                     : "memory");
                    prev = __shfl_sync(0xffffffffu, prev, 0);
                    __syncwarp();
                    if (prev == gm.y - 1u) {  // last contributor: add the partial tiles in range order
#pragma unroll 1
                        for (int i = 0; i < 4 * C; ++i) {
                            const std::uint32_t bcol = col_of(i), row = 128u * T_ + row_of(i);
                            float sum = 0.f;
                            for (std::uint32_t j = 0; j < gm.y; ++j)
                                sum += __ldcg(p.partial + (static_cast<std::size_t>(gm.x + j) * N + bcol) * 128u + row_of(i));
                            if (bcol < p.B && row < p.m) p.y[static_cast<std::size_t>(bcol) * p.m + row] = sum * __ldg(p.escale + bcol);
                        }
                        if (lane == 0) p.counters[16u * T_ + static_cast<std::uint32_t>(warp)] = 0;
                    }
                }
#pragma unroll
                for (int i = 0; i < N / 2; ++i) acc[i] = 0.f;
                ++tile_i;
            }
        };

#pragma unroll 1
        for (std::uint32_t u = u0; u < u1; ++u) {
            std::uint32_t q;
            const bool have = cell_of(u, q);
            if (have) {
                issue_rec(u + 2);
                load_off(u + 3);
            }
            const std::uint32_t k = u - u0, sl = k % NS;
            const std::uint8_t* unit = ring + sl * p.slot_bytes + uu * UNIT;
            const std::uint32_t* ees = reinterpret_cast<const std::uint32_t*>(ring + sl * p.slot_bytes + CELL);
            if (have) {
                EX_W(0, mbar_wait(&rec_full[ci][sl], (k / NS) & 1u))
                // this unit's run of the cell's (row, col)-sorted outlier list
                {
                    const std::uint32_t c0 = slot_r[ci][sl][0], c1 = slot_r[ci][sl][1];
                    const std::uint32_t cnt = (c1 - c0 - CELL) / 4u;
                    onf = (min(c1 - c0, p.rec_cap) - CELL) / 4u;
                    oc0 = c0;
                    // [obeg, oend): entries of local rows 16 uu .. 16 uu + 15, counted by ballots
                    std::uint32_t n16 = 0, nend = 0;
#pragma unroll 1
                    for (std::uint32_t i0 = 0; i0 < cnt; i0 += 32u) {
                        const std::uint32_t i = i0 + lane;
                        const std::uint32_t lr = i < cnt ? ex_entry(ees, onf, p.cells, oc0, CELL, i) >> 24 : 255u;
                        n16 += __popc(__ballot_sync(0xffffffffu, lr < 16u));
                        nend += __popc(__ballot_sync(0xffffffffu, lr < 16u * uu + 16u));
                    }
                    obeg = uu == 0 ? 0u : n16;
                    oend = nend;
                    // up to 128 entries: each lane precomputes its (quarter, tile offset, fp16 v 2^p_c)
                    ofast = oend - obeg <= 128u;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const std::uint32_t i = obeg + lane + 32u * j;
                        oit[j] = 0xFFFFFFFFu;
                        if (ofast && i < oend) {
                            const std::uint32_t en = ex_entry(ees, onf, p.cells, oc0, CELL, i);
                            oit[j] = ex_outlier_item<BW>(en, ci);
                        }
                    }
                }
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
                        sv[h][rho] = make_float2(s0 * 16777216.0f, s1 * 16777216.0f);
                        nz[h][rho] = make_float2(-__fmul_rn(s0, z0), -__fmul_rn(s1, z1));
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
#pragma unroll
            for (int Q = 0; Q < 4; ++Q) {
                const std::uint32_t s = 4u * k + Q;
                const std::uint32_t b = s % NA;
                issue_x(s + XLA);
                if (s >= NA) EX_W(3, mbar_wait(&a_free[b], ((s / NA) - 1u) & 1u))  // MMAs of stage s - NA done
                if (have) {
                    // codes of blocks 4Q .. 4Q+3 of the unit: binary16 subnormals q 2^(p-24), into TMEM
                    std::uint32_t ar[16];
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
                        ar[4 * jj] = a[0];
                        ar[4 * jj + 1] = a[2];
                        ar[4 * jj + 2] = a[1];
                        ar[4 * jj + 3] = a[3];
                    }
                    tc::st16_x4(tmem + lanes16 + CODE_COL + b * 32u, ar);
                    // -s z of blocks 4Q + 2(t & 1) + {0, 1}, rows g, g + 8: hi (t < 2) or lo (t >= 2),
                    // from lane 4g + 2(Q & 1) + (t & 1) of the producer layout
                    const int src = 4 * g + 2 * (Q & 1) + (t & 1);
                    std::uint32_t zr[4];
#pragma unroll
                    for (int rho = 0; rho < 2; ++rho) {
                        const float2 a = nz[Q >> 1][rho];
                        const float z0 = __shfl_sync(0xffffffffu, a.x, src), z1 = __shfl_sync(0xffffffffu, a.y, src);
                        // tf32 hi by truncation (lo = the exact rest; the tensor core truncates lo to tf32)
                        const float h0 = __uint_as_float(__float_as_uint(z0) & 0xFFFFE000u);
                        const float h1 = __uint_as_float(__float_as_uint(z1) & 0xFFFFE000u);
                        zr[2 * rho] = __float_as_uint(t < 2 ? h0 : z0 - h0);
                        zr[2 * rho + 1] = __float_as_uint(t < 2 ? h1 : z1 - h1);
                    }
                    tc::st16_x1(tmem + lanes16 + AZ_COL + b * 8u, zr[0], zr[1], zr[2], zr[3]);
                    // outlier tile of this unit's rows: zero, then the stage's entries (v 2^p_c, exact)
                    std::uint8_t* aot = aobuf + b * kExAOBytes;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const std::uint32_t c = static_cast<std::uint32_t>(lane + 32 * j), cm = c >> 3;
                        *reinterpret_cast<uint4*>(aot + (cm >> 1) * 2048u + (4u * ci + 2u * uu + (cm & 1u)) * 128u +
                                                  (c & 7u) * 16u) = make_uint4(0, 0, 0, 0);
                    }
                    __syncwarp();
                    if (ofast) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (oit[j] != 0xFFFFFFFFu && (oit[j] >> 30) == static_cast<std::uint32_t>(Q))
                                *reinterpret_cast<unsigned short*>(aot + ((oit[j] >> 16) & 0x3FFFu)) =
                                    static_cast<unsigned short>(oit[j] & 0xFFFFu);
                    } else {  // dense outliers: the entries straight from the list
#pragma unroll 1
                        for (std::uint32_t i = obeg + lane; i < oend; i += 32u) {
                            const std::uint32_t it = ex_outlier_item<BW>(ex_entry(ees, onf, p.cells, oc0, CELL, i), ci);
                            if ((it >> 30) == static_cast<std::uint32_t>(Q))
                                *reinterpret_cast<unsigned short*>(aot + ((it >> 16) & 0x3FFFu)) =
                                    static_cast<unsigned short>(it & 0xFFFFu);
                        }
                    }
                    tc::wait_st();
                }
                fence_proxy_async();  // the outlier tile (generic stores) -> tensor core reads
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[b]);
                // the previous stage's accumulators (its statistics: this cell's, or the last cell's at Q = 0)
                if (s > 0) {
                    if (Q == 0) epilogue(s - 1, sv_prev);
                    else epilogue(s - 1, sv);
                }
                if (Q == 3) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int rho = 0; rho < 2; ++rho) sv_prev[h][rho] = sv[h][rho];
                    if (have) {  // done with the cell's record
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&rec_empty[ci][sl]);
                    }
                }
            }
        }
        if (nst) epilogue(nst - 1, sv_prev);
    }
#ifdef SPQR_TIMELINE
    if (lane == 0 && blockIdx.x < 148) {
        unsigned long long* o = g_timeline + 8u * (blockIdx.x * 17u + warp);
        for (int i = 0; i < 6; ++i) o[i] = tw[i];
        o[6] = gtime() - t_start;
        o[7] = nst;
    }
#endif
    tc::fence_before();
    __syncthreads();
    if (warp == CTRL) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// gemm_ex.cu: the instantiations (bw, bs in {2, 3, 4}; N in {16, 32, 64}).
cudaError_t launch_gemm_ex(int bw, int bs, int n, const ExParams& p, std::uint32_t smem, std::uint32_t smem_limit,
                           cudaStream_t st);
