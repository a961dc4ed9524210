// kernels.cuh -- sm_100a kernels of the SpQR decode path.
//
//   gemv_cta ........... THE hot kernel (gemv_cta.cuh): x preparation + fused
//                        dequant-GEMV + CSR outlier merge (kernel.hpp:89-124)
//                        over the tiled HBM layout, one output write per row,
//                        deterministic.
//   xprep_tc + gemm_tc . batched path (gemm_tc.cuh): tcgen05 tensor cores.
//   xprep_ex + gemm_ex . batched path with exact codes (gemm_ex.cuh, gemm_ex.cu).
//   xprep_bm + gemm_bm . exact batched path, batch in the MMA's M (gemm_bm.cuh).
//   dequant_raw / outliers_raw ... bit-exact dequantize_full (kernel.hpp:17-25,
//                        solver.hpp:345-362) on the raw stream, any geometry.
//   xprep_raw / gemv_raw ......... generic matvec on the raw stream for layers
//                        outside the tiled geometry (any bits / group sizes).
//   dense_gemv_f16 ..... comparator: dense fp16 GEMV.
//
// Build: -gencode arch=compute_100a,code=sm_100a, no fast-math (IEEE fp32 with
// subnormals is part of the bit-exact contract).
#pragma once

#include <cuda_fp16.h>
#include <cstdint>
#include <type_traits>

#include "tiled.hpp"

namespace spqr_dev {

namespace T = spqr_tiled;

// ------------------------------------------------------------- PTX helpers --
__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// TMA bulk copy global -> shared, completion on an mbarrier (UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// D(16x8, fp32) += A(16x16, f16 row) * B(16x8, f16 col)
__device__ __forceinline__ void mma16816(float (&c)[4], const std::uint32_t (&a)[4], std::uint32_t b0,
                                         std::uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// four 8x8 b16 matrices from shared memory (rows addressed per lane)
__device__ __forceinline__ void ldsm_x4(std::uint32_t addr, std::uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ float u2f_small(std::uint32_t v) {  // exact for v < 2^23
    return __int_as_float(0x4B000000u | v) - 8388608.0f;
}

__device__ __forceinline__ __half2 u32_as_h2(std::uint32_t v) {
    __half2 h;
    memcpy(&h, &v, 4);
    return h;
}

__device__ __forceinline__ float h2f_bits(std::uint32_t h16) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(h16)));
}

// ============================================================ tiled path ====
template <int BW>
struct Geo {
    static constexpr int CW = T::words_per_container(BW);
    static constexpr int MPC = T::mmas_per_container(BW);
    static constexpr int NP = T::pairs_per_container(BW);
    static constexpr int CPU = T::containers_per_unit(BW);
    static constexpr int LANE_WORDS = 4 * BW;  // 16*BW bytes
};

// 16-bit window of a container's lo/hi streams starting at stream byte B.
template <int CW>
__device__ __forceinline__ std::uint32_t window(const std::uint32_t* w, int B) {
    if ((B & 1) == 0) return w[B >> 1];
    if ((B >> 1) + 1 < CW) return __byte_perm(w[B >> 1], w[(B >> 1) + 1], 0x6341);
    std::uint32_t r;  // w >> 8 on the FMA pipe (IMAD.HI)
    asm("mul.hi.u32 %0, %1, 16777216;" : "=r"(r) : "r"(w[B >> 1]));
    return r;
}

#include "helpers.cuh"
#include "gemv_cta.cuh"
#include "gemm_tc.cuh"
#include "gemm_ex.cuh"
#include "gemm_bm.cuh"
#include "dequant_cells.cuh"

// ============================================================== raw path ====
// Geometry of a raw .spqr stream resident in device memory (any config).
struct RawGeom {
    const std::uint8_t* s;         // whole stream
    const std::uint32_t* order;    // solve k -> source column (nullptr = identity)
    std::uint32_t rows, cols, b1, b2, nblocks, ngroups;
    int wb, sb, zb;
    std::uint64_t rec_off, col_block_bytes, csr_off, ent_off;

    __device__ __forceinline__ std::uint32_t block_width(std::uint32_t k) const {
        return k + 1 < nblocks ? b1 : cols - k * b1;
    }
    __device__ __forceinline__ std::uint32_t group_rows(std::uint32_t g) const {
        return g + 1 < ngroups ? b2 : rows - g * b2;
    }
    __device__ __forceinline__ static std::uint64_t packed(std::uint64_t count, int bits) {
        return (count * bits + 7) / 8;
    }
    __device__ __forceinline__ std::uint64_t side_bytes(std::uint32_t gr, int bits) const {
        return bits <= 8 ? 4 + packed(gr, bits) : 4ull * gr;
    }
    __device__ __forceinline__ std::uint64_t record_bytes(std::uint32_t gr, std::uint32_t bw) const {
        return side_bytes(gr, sb) + side_bytes(gr, zb) + packed(static_cast<std::uint64_t>(gr) * bw, wb);
    }
    __device__ __forceinline__ std::uint64_t record_offset(std::uint32_t k, std::uint32_t g) const {
        return rec_off + k * col_block_bytes + g * record_bytes(b2, block_width(k));
    }
    __device__ __forceinline__ std::uint32_t u16(std::uint64_t off) const {
        return static_cast<std::uint32_t>(s[off]) | (static_cast<std::uint32_t>(s[off + 1]) << 8);
    }
    __device__ __forceinline__ std::uint32_t u32(std::uint64_t off) const {
        return u16(off) | (u16(off + 2) << 16);
    }
    // element i of a packed field of `bits` (<= 8) starting at byte `off`
    __device__ __forceinline__ std::uint32_t bits_at(std::uint64_t off, std::uint64_t i, int bits) const {
        const std::uint64_t pos = i * bits;
        const std::uint32_t two = u16(off + (pos >> 3));  // the stream always has bytes after a field
        return (two >> (pos & 7)) & ((1u << bits) - 1u);
    }
    // first-level statistics of (block k, row r), bit-exact stat_dequant
    __device__ __forceinline__ void stats(std::uint32_t k, std::uint32_t r, float& sv, float& zv,
                                          std::uint64_t& wfield, std::uint32_t& rr, std::uint32_t& bw) const {
        const std::uint32_t g = r / b2;
        const std::uint32_t gr = group_rows(g);
        rr = r - g * b2;
        bw = block_width(k);
        std::uint64_t o = record_offset(k, g);
        const std::uint64_t sfield = o + (sb <= 8 ? 4 : 0) + (zb <= 8 ? 4 : 0);
        const std::uint64_t zfield = sfield + side_bytes(gr, sb) - (sb <= 8 ? 4 : 0);
        wfield = zfield + side_bytes(gr, zb) - (zb <= 8 ? 4 : 0);
        if (sb == 16) {
            sv = __uint_as_float(u32(sfield + 4ull * rr));
        } else {
            const float S = h2f_bits(u16(o)), Z = h2f_bits(u16(o + 2));
            sv = __fmul_rn(S, __fsub_rn(static_cast<float>(bits_at(sfield, rr, sb)), Z));
        }
        if (zb == 16) {
            zv = __uint_as_float(u32(zfield + 4ull * rr));
        } else {
            const std::uint64_t zh = o + (sb <= 8 ? 4 : 0);
            const float S = h2f_bits(u16(zh)), Z = h2f_bits(u16(zh + 2));
            zv = __fmul_rn(S, __fsub_rn(static_cast<float>(bits_at(zfield, rr, zb)), Z));
        }
    }
};

// W[r, order[c]] = s * (q - z), binary32 (dequant_value, quantizer.hpp:60-62)
static __global__ void dequant_raw(const RawGeom geo, float* __restrict__ w) {
    const std::uint64_t total = static_cast<std::uint64_t>(geo.rows) * geo.nblocks;
    for (std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        // consecutive threads take consecutive blocks of the same row
        const std::uint32_t r = static_cast<std::uint32_t>(idx / geo.nblocks);
        const std::uint32_t k = static_cast<std::uint32_t>(idx - static_cast<std::uint64_t>(r) * geo.nblocks);
        float sv, zv;
        std::uint64_t wf;
        std::uint32_t rr, bw;
        geo.stats(k, r, sv, zv, wf, rr, bw);
        for (std::uint32_t c = 0; c < bw; ++c) {
            const std::uint32_t q = geo.bits_at(wf, static_cast<std::uint64_t>(rr) * bw + c, geo.wb);
            const std::uint32_t col = k * geo.b1 + c;
            const std::uint32_t dst = geo.order ? __ldg(geo.order + col) : col;
            w[static_cast<std::uint64_t>(r) * geo.cols + dst] = __fmul_rn(sv, __fsub_rn(static_cast<float>(q), zv));
        }
    }
}

// outlier corrections: a separate binary32 add (solver.hpp:360)
static __global__ void outliers_raw(const RawGeom geo, float* __restrict__ w) {
    const std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= geo.rows) return;
    const std::uint32_t i0 = geo.u32(geo.csr_off + 4ull * r), i1 = geo.u32(geo.csr_off + 4ull * r + 4);
    for (std::uint32_t i = i0; i < i1; ++i) {
        const std::uint32_t col = geo.u16(geo.ent_off + 4ull * i);
        const float v = h2f_bits(geo.u16(geo.ent_off + 4ull * i + 2));
        const std::uint32_t dst = geo.order ? __ldg(geo.order + col) : col;
        float* pw = w + static_cast<std::uint64_t>(r) * geo.cols + dst;
        *pw = __fadd_rn(*pw, v);
    }
}

// xp[b][k] = x[b][order[k]] in fp32 (kernel.hpp:93-98)
static __global__ void xprep_raw(const void* __restrict__ x, int x_f16, std::uint32_t n, std::uint32_t batch,
                          const std::uint32_t* __restrict__ order, float* __restrict__ xp) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(n) * batch) return;
    const std::uint32_t b = static_cast<std::uint32_t>(idx / n), k = static_cast<std::uint32_t>(idx % n);
    const std::uint32_t src = order ? __ldg(order + k) : k;
    const std::uint64_t si = static_cast<std::uint64_t>(b) * n + src;
    xp[idx] = x_f16 ? __half2float(reinterpret_cast<const __half*>(x)[si]) : reinterpret_cast<const float*>(x)[si];
}

// generic matvec: one warp per row, lanes over column blocks, fp32 accumulate
static __global__ void gemv_raw(const RawGeom geo, const float* __restrict__ xp, float* __restrict__ y) {
    const std::uint32_t warps = blockDim.x >> 5;
    const std::uint32_t r = blockIdx.x * warps + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= geo.rows) return;
    float acc = 0.f;
    for (std::uint32_t k = lane; k < geo.nblocks; k += 32) {
        float sv, zv;
        std::uint64_t wf;
        std::uint32_t rr, bw;
        geo.stats(k, r, sv, zv, wf, rr, bw);
        float part = 0.f;
        for (std::uint32_t c = 0; c < bw; ++c) {
            const std::uint32_t q = geo.bits_at(wf, static_cast<std::uint64_t>(rr) * bw + c, geo.wb);
            part = fmaf(__fsub_rn(static_cast<float>(q), zv), xp[k * geo.b1 + c], part);
        }
        acc = fmaf(sv, part, acc);
    }
    const std::uint32_t i0 = geo.u32(geo.csr_off + 4ull * r), i1 = geo.u32(geo.csr_off + 4ull * r + 4);
    for (std::uint32_t i = i0 + lane; i < i1; i += 32)
        acc = fmaf(h2f_bits(geo.u16(geo.ent_off + 4ull * i + 2)), xp[geo.u16(geo.ent_off + 4ull * i)], acc);
#pragma unroll
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) y[r] = acc;
}

// ========================================================= dense baseline ==
// spqr_matvec_host: x from page-locked host memory (UVA-mapped) into the
// device, 16 B per thread -- a kernel node is cheaper than a copy-engine node
// for the 16-88 KB vectors of a decode step
static __global__ void __launch_bounds__(256) copy_in(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                      std::uint32_t n16) {
    pdl_launch();  // the decode kernel's prologue (record prefetch) overlaps the copy; it waits before reading x
    for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// spqr_matvec_host completion: the last node of the host-API graph bumps a
// device sequence number and posts it to a page-locked host word (after every
// y store of the preceding kernels, which completed first), so the caller
// spins on that word instead of paying a stream synchronisation.  Launched
// as a programmatic dependent: it is resident before the decode kernel ends
// and waits for its completion (and memory flush) in griddepcontrol.wait.
static __global__ void signal_host(std::uint32_t* __restrict__ seq, volatile std::uint32_t* __restrict__ flag) {
    pdl_wait();
    const std::uint32_t v = *seq + 1u;
    *seq = v;
    __threadfence_system();
    *flag = v;
}

// y = W16 * x16, fp32 accumulate; one warp per row, 128-bit loads.
static __global__ void dense_gemv_f16(const __half* __restrict__ w, const __half* __restrict__ x, float* __restrict__ y,
                               std::uint32_t rows, std::uint32_t cols) {
    const std::uint32_t warps = blockDim.x >> 5;
    const int lane = threadIdx.x & 31;
    for (std::uint32_t r = blockIdx.x * warps + (threadIdx.x >> 5); r < rows; r += gridDim.x * warps) {
        const uint4* wr = reinterpret_cast<const uint4*>(w + static_cast<std::uint64_t>(r) * cols);
        const uint4* xr = reinterpret_cast<const uint4*>(x);
        float acc = 0.f;
        const std::uint32_t n8 = (cols % 8 == 0) ? cols / 8 : 0;  // 128-bit rows need 16-B alignment
#pragma unroll 4
        for (std::uint32_t i = lane; i < n8; i += 32) {
            const uint4 a = __ldcs(wr + i);
            const uint4 b = __ldg(xr + i);
            const __half2* ah = reinterpret_cast<const __half2*>(&a);
            const __half2* bh = reinterpret_cast<const __half2*>(&b);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 fa = __half22float2(ah[j]), fb = __half22float2(bh[j]);
                acc = fmaf(fa.x, fb.x, acc);
                acc = fmaf(fa.y, fb.y, acc);
            }
        }
        for (std::uint32_t c = n8 * 8 + lane; c < cols; c += 32)
            acc = fmaf(__half2float(w[static_cast<std::uint64_t>(r) * cols + c]), __half2float(x[c]), acc);
#pragma unroll
        for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
        if (lane == 0) y[r] = acc;
    }
}

#include "transcode_dev.cuh"

}  // namespace spqr_dev
