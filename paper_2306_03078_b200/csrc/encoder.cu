// encoder.cu -- the SpQR encoder on the GPU: Hessian
// accumulation, damped inverse Cholesky, block-GPTQ with the leave-one-out
// outlier screen and the bilevel statistics fit, then encode.
//
// Reference semantics, step by step (all arithmetic in binary64 as the
// reference's Eigen::MatrixXd, fp16 / binary32 where it rounds):
//   HessianAccumulator::accumulate  hessian.hpp:59-69   H += p + p^T, p = X X^T
//   finalize / factor_regularized   hessian.hpp:103-143 dead-column rule, +lambda I,
//                                   LLT, solve(I), symmetrise, LLT again, C = L2^T
//   refactor_permuted / act_order   hessian.hpp:147-180, solver.hpp:381-404
//   spqr_quantize                   solver.hpp:417-533  per beta1 block:
//     detect_outliers_impl          solver.hpp:270-320  (thread per row)
//     fit_statistics_impl           solver.hpp:180-266  (first level per row,
//                                                        second level per beta2 group)
//     the column loop               solver.hpp:468-491  (thread per row: codes,
//                                                        outliers, in-block error feedback)
//     the cross-block update        solver.hpp:492-494  (one DGEMM: errs x C block)
//   relative_layer_error            solver.hpp:406-413  (two DGEMMs)
//   make_spqr_tensor + encode       format.hpp:69-89, :269-352 (host, byte-identical)
// Every per-row step is independent across rows, so rows map to threads; the
// rank-beta1 trailing update and the Hessian products go to cuBLAS DGEMM, the
// factorizations to cuSOLVER (both bound at run time with dlopen, like NCCL
// in sharded.cu: plain library GEMMs / factorizations, the loops are ours).
// Parity: the unmodified reference encoder (oracle/ref_encoder.cpp) produces
// the same stream bytes (tests/test_gpu_encoder.py).
#include <dlfcn.h>

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "internal.hpp"
#include "spqr/format.hpp"
#include "spqr_cuda.h"

namespace {

// ---- run-time bound cuBLAS / cuSOLVER --------------------------------------
struct LinAlg {
    cublasStatus_t (*create)(cublasHandle_t*) = nullptr;
    cublasStatus_t (*destroy)(cublasHandle_t) = nullptr;
    cublasStatus_t (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
    cublasStatus_t (*dgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const double*,
                            const double*, int, const double*, int, const double*, double*, int) = nullptr;
    cusolverStatus_t (*s_create)(cusolverDnHandle_t*) = nullptr;
    cusolverStatus_t (*s_destroy)(cusolverDnHandle_t) = nullptr;
    cusolverStatus_t (*s_set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
    cusolverStatus_t (*potrf_bs)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
    cusolverStatus_t (*potrf)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int, int*) = nullptr;
    cusolverStatus_t (*potrs)(cusolverDnHandle_t, cublasFillMode_t, int, int, const double*, int, double*, int,
                              int*) = nullptr;
};

const LinAlg& la() {
    static LinAlg a;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* hb = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        void* hs = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!hb || !hs) {
            err = std::string("encoder: cannot load cuBLAS / cuSOLVER: ") + dlerror();
            return;
        }
        auto sym = [&](void* h, auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && err.empty()) err = std::string("encoder: missing symbol ") + name;
        };
        sym(hb, a.create, "cublasCreate_v2");
        sym(hb, a.destroy, "cublasDestroy_v2");
        sym(hb, a.set_stream, "cublasSetStream_v2");
        sym(hb, a.dgemm, "cublasDgemm_v2");
        sym(hs, a.s_create, "cusolverDnCreate");
        sym(hs, a.s_destroy, "cusolverDnDestroy");
        sym(hs, a.s_set_stream, "cusolverDnSetStream");
        sym(hs, a.potrf_bs, "cusolverDnDpotrf_bufferSize");
        sym(hs, a.potrf, "cusolverDnDpotrf");
        sym(hs, a.potrs, "cusolverDnDpotrs");
    });
    if (!err.empty()) throw std::runtime_error(err);
    return a;
}

void cck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + what + ": " + cudaGetErrorString(e));
}
void bck(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string("cuBLAS: ") + what + " failed");
}
void sck(cusolverStatus_t s, const char* what) {
    if (s != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error(std::string("cuSOLVER: ") + what + " failed");
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(std::size_t count) : n(count) { cck(cudaMalloc(&p, std::max<std::size_t>(count, 1) * sizeof(T)), "cudaMalloc"); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        return *this;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct Handles {
    cublasHandle_t b = nullptr;
    cusolverDnHandle_t s = nullptr;
    Handles() {
        bck(la().create(&b), "create");
        sck(la().s_create(&s), "create");
    }
    ~Handles() {
        if (b) la().destroy(b);
        if (s) la().s_destroy(s);
    }
};

// ---- device helpers ---------------------------------------------------------
struct QFlags {
    bool full_range_sign, integer_zero;
};

// fit_group_minmax, quantizer.hpp:77-97
__device__ void fit_minmax(const double* v, std::uint32_t len, int bits, QFlags f, double& s, double& z) {
    // std::min / std::max semantics (keep the first operand unless the
    // second compares strictly smaller / larger: signed zeros as the host)
    auto smin = [](double a, double b) { return b < a ? b : a; };
    auto smax = [](double a, double b) { return a < b ? b : a; };
    double mn = v[0], mx = v[0];
    for (std::uint32_t i = 1; i < len; ++i) {
        mn = smin(mn, v[i]);
        mx = smax(mx, v[i]);
    }
    if (!f.full_range_sign) {
        mn = smin(mn, 0.0);
        mx = smax(mx, 0.0);
    }
    const double maxq = static_cast<double>((1u << bits) - 1u);
    if (mx == mn) {
        s = 1.0;
        z = -mn;
    } else {
        s = (mx - mn) / maxq;
        z = -mn / s;
    }
    if (f.integer_zero) z = smin(smax(floor(z + 0.5), 0.0), maxq);  // std::clamp
}
// quant_code, quantizer.hpp:50-56
__device__ __forceinline__ std::uint32_t qcode(double v, double s, double z, std::uint32_t maxq) {
    if (!(s > 0.0)) return 0;
    const double t = floor(v / s + z + 0.5);
    if (!(t > 0.0)) return 0;
    if (t >= static_cast<double>(maxq)) return maxq;
    return static_cast<std::uint32_t>(t);
}
// fp16_from_float (common.hpp:70-101): RNE, saturating at +-65504
__device__ std::uint16_t f2h_sat(float f) {
    const std::uint32_t x = __float_as_uint(f);
    const std::uint16_t sign = static_cast<std::uint16_t>((x >> 16) & 0x8000u);
    const std::uint32_t exp8 = (x >> 23) & 0xffu;
    std::uint32_t mant = x & 0x7fffffu;
    if (exp8 == 0xffu) return static_cast<std::uint16_t>(sign | 0x7c00u | (mant ? 0x200u : 0u));
    const int exp = static_cast<int>(exp8) - 127 + 15;
    if (exp >= 31) return static_cast<std::uint16_t>(sign | 0x7bffu);
    if (exp <= 0) {
        if (exp < -10) return sign;
        mant |= 0x800000u;
        const std::uint32_t shift = static_cast<std::uint32_t>(14 - exp);
        std::uint32_t half = mant >> shift;
        const std::uint32_t rem = mant & ((1u << shift) - 1u);
        const std::uint32_t halfway = 1u << (shift - 1u);
        if (rem > halfway || (rem == halfway && (half & 1u))) half++;
        return static_cast<std::uint16_t>(sign | half);
    }
    std::uint32_t half = (static_cast<std::uint32_t>(exp) << 10) | (mant >> 13);
    const std::uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) half++;
    if (half >= 0x7c00u) half = 0x7bffu;
    return static_cast<std::uint16_t>(sign | half);
}
__device__ __forceinline__ float h2f(std::uint16_t h) { return __half2float(__ushort_as_half(h)); }
// dequant_value / stat_dequant, quantizer.hpp:60-67 (binary32)
__device__ __forceinline__ float deq(float s, float z, std::uint32_t code) {
    return __fmul_rn(s, __fsub_rn(static_cast<float>(code), z));
}

constexpr int kMaxBeta1 = 256;

struct EncCfg {
    int wb, sb, zb;
    std::uint32_t b1, b2;
    QFlags flags;
    bool outliers;
    double tau;
};

// H += p + p^T (the exactly symmetric form of 2 X X^T), p = X X^T from DGEMM
__global__ void sym_add(double* H, const double* p, std::uint32_t n) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(n) * n) return;
    const std::uint32_t i = static_cast<std::uint32_t>(idx / n), j = static_cast<std::uint32_t>(idx % n);
    H[idx] += p[idx] + p[static_cast<std::uint64_t>(j) * n + i];
}
__global__ void f32_to_f64(const float* x, double* y, std::uint64_t count) {
    const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (i < count) y[i] = static_cast<double>(x[i]);
}
// A = regularized(Hp) (hessian.hpp:103-111) with Hp(i, j) = H(ord[i], ord[j])
__global__ void regularize(const double* H, const std::uint32_t* ord, double* A, std::uint32_t n, double lambda) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(n) * n) return;
    const std::uint32_t i = static_cast<std::uint32_t>(idx / n), j = static_cast<std::uint32_t>(idx % n);
    double v = H[static_cast<std::uint64_t>(ord[i]) * n + ord[j]];
    if (i == j) {
        if (v == 0.0) v = 1.0;  // dead-column rule
        v += lambda;
    }
    A[idx] = v;
}
// Minv = (Minv + Minv^T) / 2 (hessian.hpp:121), upper triangle from the lower
__global__ void symmetrize(double* M, std::uint32_t n) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(n) * n) return;
    const std::uint32_t i = static_cast<std::uint32_t>(idx / n), j = static_cast<std::uint32_t>(idx % n);
    if (i > j) return;
    const double a = M[idx], b = M[static_cast<std::uint64_t>(j) * n + i];
    const double v = (a + b) * 0.5;
    M[idx] = v;
    M[static_cast<std::uint64_t>(j) * n + i] = v;
}
// C (row-major, upper) = L2^T: the column-major lower factor read row-major;
// zero the other triangle
__global__ void keep_upper(double* C, std::uint32_t n) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(n) * n) return;
    const std::uint32_t i = static_cast<std::uint32_t>(idx / n), j = static_cast<std::uint32_t>(idx % n);
    if (j < i) C[idx] = 0.0;
}
__global__ void eye(double* I, std::uint32_t n) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(n) * n) return;
    I[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
}
// Wp(r, k) = W(r, ord[k]) in binary64 (solver.hpp:436-438)
__global__ void permute_w(const float* W, const std::uint32_t* ord, double* Wp, std::uint32_t m, std::uint32_t n) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(m) * n) return;
    const std::uint64_t r = idx / n, k = idx % n;
    Wp[idx] = static_cast<double>(W[r * n + ord[k]]);
}

// Per row: the leave-one-out outlier screen (detect_outliers_impl,
// solver.hpp:270-320) and the first-level (s, z) fit with outliers zeroed
// (fit_statistics_impl, solver.hpp:187-194).
__global__ void enc_screen_fit(const double* __restrict__ Wp, const double* __restrict__ C, std::uint32_t m,
                               std::uint32_t n, std::uint32_t i0, std::uint32_t bw, EncCfg cfg,
                               std::uint8_t* __restrict__ mask, double* __restrict__ s1, double* __restrict__ z1) {
    const std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    double row[kMaxBeta1], buf[kMaxBeta1], inv_d2[kMaxBeta1];
    for (std::uint32_t c = 0; c < bw; ++c) {
        row[c] = Wp[static_cast<std::uint64_t>(r) * n + i0 + c];
        const double d = C[static_cast<std::uint64_t>(i0 + c) * n + i0 + c];
        inv_d2[c] = 1.0 / (d * d);
    }
    std::uint8_t* mk = mask + static_cast<std::uint64_t>(r) * bw;
    const std::uint32_t maxq = (1u << cfg.wb) - 1u;
    for (std::uint32_t c = 0; c < bw; ++c) mk[c] = 0;
    if (cfg.outliers && !isinf(cfg.tau)) {
        double s, z;
        fit_minmax(row, bw, cfg.wb, cfg.flags, s, z);
        double e_base = 0.0;
        for (std::uint32_t c = 0; c < bw; ++c) {
            const double dq = s * (static_cast<double>(qcode(row[c], s, z, maxq)) - z);
            const double d = row[c] - dq;
            e_base += d * d * inv_d2[c];
        }
        for (std::uint32_t c = 0; c < bw; ++c) {
            double e_loo = 0.0;
            if (bw > 1) {
                std::uint32_t k = 0;
                for (std::uint32_t j = 0; j < bw; ++j)
                    if (j != c) buf[k++] = row[j];
                double s2, z2;
                fit_minmax(buf, bw - 1, cfg.wb, cfg.flags, s2, z2);
                k = 0;
                for (std::uint32_t j = 0; j < bw; ++j) {
                    if (j == c) continue;
                    const double v = buf[k++];
                    const double dq = s2 * (static_cast<double>(qcode(v, s2, z2, maxq)) - z2);
                    const double d = v - dq;
                    e_loo += d * d * inv_d2[j];
                }
            }
            if (e_base - e_loo > cfg.tau) mk[c] = 1;
        }
    }
    for (std::uint32_t c = 0; c < bw; ++c) buf[c] = mk[c] ? 0.0 : row[c];
    double s, z;
    fit_minmax(buf, bw, cfg.wb, cfg.flags, s, z);
    s1[r] = s;
    z1[r] = z;
}

// Per beta2 group: the second-level fits of the scales and zeros and the
// dequantized first-level statistics (fit_statistics_impl, solver.hpp:196-264).
// scal: [groups][4] u16 {scale_s, scale_z, zero_s, zero_z} (identity defaults).
__global__ void enc_fit2(const double* __restrict__ s1, const double* __restrict__ z1, std::uint32_t m, EncCfg cfg,
                         std::uint8_t* __restrict__ scode, std::uint8_t* __restrict__ zcode,
                         std::uint16_t* __restrict__ scal, float* __restrict__ sf, float* __restrict__ zf) {
    const std::uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    const std::uint32_t ng = (m + cfg.b2 - 1) / cfg.b2;
    if (g >= ng) return;
    const std::uint32_t r0 = g * cfg.b2, len = min(cfg.b2, m - r0);
    std::uint16_t* sc = scal + 4ull * g;
    sc[0] = 0x3c00;
    sc[1] = 0;
    sc[2] = 0x3c00;
    sc[3] = 0;
    const QFlags second{true, false};
    if (cfg.sb == 16) {
        for (std::uint32_t r = r0; r < r0 + len; ++r) sf[r] = static_cast<float>(s1[r]);
    } else {
        double ss, zs;
        fit_minmax(s1 + r0, len, cfg.sb, second, ss, zs);
        const std::uint16_t ss16 = f2h_sat(static_cast<float>(ss)), zs16 = f2h_sat(static_cast<float>(zs));
        sc[0] = ss16;
        sc[1] = zs16;
        const double sd = h2f(ss16), zd = h2f(zs16);
        const std::uint32_t maxq = (1u << cfg.sb) - 1u;
        for (std::uint32_t r = r0; r < r0 + len; ++r) {
            const std::uint32_t code = qcode(s1[r], sd, zd, maxq);
            scode[r] = static_cast<std::uint8_t>(code);
            sf[r] = deq(h2f(ss16), h2f(zs16), code);
        }
    }
    if (cfg.zb == 16) {
        for (std::uint32_t r = r0; r < r0 + len; ++r) zf[r] = static_cast<float>(z1[r]);
    } else if (cfg.flags.integer_zero) {
        for (std::uint32_t r = r0; r < r0 + len; ++r) {
            zcode[r] = static_cast<std::uint8_t>(z1[r]);
            zf[r] = static_cast<float>(zcode[r]);
        }
    } else {
        double sz, zz;
        fit_minmax(z1 + r0, len, cfg.zb, second, sz, zz);
        const std::uint16_t sz16 = f2h_sat(static_cast<float>(sz)), zz16 = f2h_sat(static_cast<float>(zz));
        sc[2] = sz16;
        sc[3] = zz16;
        const double sd = h2f(sz16), zd = h2f(zz16);
        const std::uint32_t maxq = (1u << cfg.zb) - 1u;
        for (std::uint32_t r = r0; r < r0 + len; ++r) {
            const std::uint32_t code = qcode(z1[r], sd, zd, maxq);
            zcode[r] = static_cast<std::uint8_t>(code);
            zf[r] = deq(h2f(sz16), h2f(zz16), code);
        }
    }
}

// Per row, the block's column loop (solver.hpp:468-491): code, binary32 base,
// error; an outlier keeps fp16(err), else errs = err / C(j, j) feeds the
// in-block update of the row's remaining block columns.
__global__ void enc_columns(double* __restrict__ Wp, const double* __restrict__ C, std::uint32_t m, std::uint32_t n,
                            std::uint32_t i0, std::uint32_t bw, int wb, const std::uint8_t* __restrict__ mask,
                            const float* __restrict__ sf, const float* __restrict__ zf,
                            std::uint8_t* __restrict__ codes, std::uint8_t* __restrict__ omask,
                            std::uint16_t* __restrict__ oval, double* __restrict__ errs) {
    const std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const std::uint32_t maxq = (1u << wb) - 1u;
    double* wr = Wp + static_cast<std::uint64_t>(r) * n;
    const float s = sf[r], z = zf[r];
    double* er = errs + static_cast<std::uint64_t>(r) * bw;
    for (std::uint32_t jl = 0; jl < bw; ++jl) {
        const std::uint32_t j = i0 + jl;
        const double cjj = C[static_cast<std::uint64_t>(j) * n + j];
        const double w = wr[j];
        const std::uint32_t code = qcode(w, s, z, maxq);
        codes[static_cast<std::uint64_t>(r) * n + j] = static_cast<std::uint8_t>(code);
        const float base = deq(s, z, code);
        const double err = w - static_cast<double>(base);
        double e = 0.0;
        if (mask[static_cast<std::uint64_t>(r) * bw + jl]) {
            omask[static_cast<std::uint64_t>(r) * n + j] = 1;
            oval[static_cast<std::uint64_t>(r) * n + j] = f2h_sat(static_cast<float>(err));
        } else {
            e = err / cjj;
        }
        er[jl] = e;
        for (std::uint32_t jj = jl + 1; jj < bw; ++jj) wr[i0 + jj] -= e * C[static_cast<std::uint64_t>(j) * n + i0 + jj];
    }
}

// delta(r, k) = reconstruct_solve_order(r, k) - W0p(r, k) (solver.hpp:509-514)
__global__ void recon_delta(const double* __restrict__ W0p, const std::uint8_t* __restrict__ codes,
                            const std::uint8_t* __restrict__ omask, const std::uint16_t* __restrict__ oval,
                            const float* __restrict__ sf_all, const float* __restrict__ zf_all, std::uint32_t m,
                            std::uint32_t n, std::uint32_t b1, double* __restrict__ delta) {
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(m) * n) return;
    const std::uint32_t r = static_cast<std::uint32_t>(idx / n), k = static_cast<std::uint32_t>(idx % n);
    const std::uint64_t sk = static_cast<std::uint64_t>(k / b1) * m + r;
    float v = deq(sf_all[sk], zf_all[sk], codes[idx]);
    if (omask[idx]) v = __fadd_rn(v, h2f(oval[idx]));
    delta[idx] = static_cast<double>(v) - W0p[idx];
}
__global__ void dot_sum(const double* a, const double* b, std::uint64_t count, double* out) {
    // one block: a fixed-order reduction (deterministic)
    __shared__ double part[256];
    double s = 0.0;
    for (std::uint64_t i = threadIdx.x; i < count; i += blockDim.x) s += a[i] * b[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (static_cast<int>(threadIdx.x) < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = part[0];
}

unsigned blocks_for(std::uint64_t count, unsigned t = 256) { return static_cast<unsigned>((count + t - 1) / t); }

struct NcclLikeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

}  // namespace

struct spqr_hessian {
    int device = 0;
    std::uint32_t n = 0;
    std::int64_t samples = 0;
    DevBuf<double> H;
};

namespace {
struct DevGuardE {
    int prev = -1;
    explicit DevGuardE(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DevGuardE() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// factor_regularized (hessian.hpp:113-133) of the permuted Hessian; C
// row-major upper (n x n), returns the device buffer
DevBuf<double> inverse_cholesky(const Handles& hd, const double* H, const std::uint32_t* d_ord, std::uint32_t n,
                                double lambda, cudaStream_t st) {
    const LinAlg& a = la();
    DevBuf<double> A(static_cast<std::size_t>(n) * n), I(static_cast<std::size_t>(n) * n);
    regularize<<<blocks_for(static_cast<std::uint64_t>(n) * n), 256, 0, st>>>(H, d_ord, A.p, n, lambda);
    int lwork = 0;
    sck(a.potrf_bs(hd.s, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), A.p, static_cast<int>(n), &lwork), "potrf_bufferSize");
    DevBuf<double> work(static_cast<std::size_t>(std::max(lwork, 1)));
    DevBuf<int> info(1);
    sck(a.potrf(hd.s, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), A.p, static_cast<int>(n), work.p, lwork, info.p), "potrf");
    int h_info = 0;
    cck(cudaMemcpyAsync(&h_info, info.p, 4, cudaMemcpyDeviceToHost, st), "D2H info");
    cck(cudaStreamSynchronize(st), "sync potrf");
    if (h_info != 0) spqr::fail(spqr::Errc::not_positive_definite, "regularized Hessian is not positive definite");
    eye<<<blocks_for(static_cast<std::uint64_t>(n) * n), 256, 0, st>>>(I.p, n);
    sck(a.potrs(hd.s, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), static_cast<int>(n), A.p, static_cast<int>(n), I.p,
                static_cast<int>(n), info.p),
        "potrs");
    symmetrize<<<blocks_for(static_cast<std::uint64_t>(n) * n), 256, 0, st>>>(I.p, n);
    sck(a.potrf(hd.s, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), I.p, static_cast<int>(n), work.p, lwork, info.p), "potrf 2");
    cck(cudaMemcpyAsync(&h_info, info.p, 4, cudaMemcpyDeviceToHost, st), "D2H info");
    cck(cudaStreamSynchronize(st), "sync potrf 2");
    if (h_info != 0) spqr::fail(spqr::Errc::not_positive_definite, "inverse Hessian lost positive definiteness");
    keep_upper<<<blocks_for(static_cast<std::uint64_t>(n) * n), 256, 0, st>>>(I.p, n);
    return I;
}
}  // namespace

extern "C" {

int spqr_hessian_create(uint32_t n, int device, spqr_hessian** out) {
    *out = nullptr;
    return spqr::detail::guard([&] {
        if (n == 0) spqr::fail(spqr::Errc::shape_mismatch, "dimension must be >= 1");
        DevGuardE dg(device);
        auto h = std::make_unique<spqr_hessian>();
        cck(cudaGetDevice(&h->device), "cudaGetDevice");
        h->n = n;
        h->H = DevBuf<double>(static_cast<std::size_t>(n) * n);
        cck(cudaMemset(h->H.p, 0, sizeof(double) * h->H.n), "memset H");
        *out = h.release();
    });
}

void spqr_hessian_destroy(spqr_hessian* h) { delete h; }

int spqr_hessian_accumulate(spqr_hessian* h, const float* x_dev, uint32_t samples, void* cuda_stream) {
    return spqr::detail::guard([&] {
        DevGuardE dg(h->device);
        if (samples == 0) return;
        auto st = static_cast<cudaStream_t>(cuda_stream);
        Handles hd;
        bck(la().set_stream(hd.b, st), "set stream");
        const std::uint64_t cnt = static_cast<std::uint64_t>(h->n) * samples;
        DevBuf<double> xd(cnt), p(static_cast<std::size_t>(h->n) * h->n);
        f32_to_f64<<<blocks_for(cnt), 256, 0, st>>>(x_dev, xd.p, cnt);
        // X row-major n x samples = column-major samples x n (XT); p = X X^T =
        // XT^T XT (symmetric, so its layout does not matter)
        const double one = 1.0, zero = 0.0;
        bck(la().dgemm(hd.b, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(h->n), static_cast<int>(h->n),
                       static_cast<int>(samples), &one, xd.p, static_cast<int>(samples), xd.p,
                       static_cast<int>(samples), &zero, p.p, static_cast<int>(h->n)),
            "dgemm X X^T");
        sym_add<<<blocks_for(static_cast<std::uint64_t>(h->n) * h->n), 256, 0, st>>>(h->H.p, p.p, h->n);
        cck(cudaGetLastError(), "launch sym_add");
        cck(cudaStreamSynchronize(st), "sync accumulate");
        h->samples += samples;
    });
}

int spqr_hessian_read(const spqr_hessian* h, double* out_host) {
    return spqr::detail::guard([&] {
        DevGuardE dg(h->device);
        cck(cudaMemcpy(out_host, h->H.p, sizeof(double) * h->H.n, cudaMemcpyDeviceToHost), "D2H H");
    });
}

int spqr_quantize_layer(const spqr_hessian* h, const float* w_dev, uint32_t m, const spqr_encoder_cfg* cfg_in,
                        uint8_t* out, size_t cap, size_t* len, double* report) {
    int rc = SPQR_OK;
    const int g = spqr::detail::guard([&] {
        DevGuardE dg(h->device);
        const spqr_encoder_cfg& cf = *cfg_in;
        const std::uint32_t n = h->n;
        // SolverConfig::validate (solver.hpp:46-66)
        if (cf.weight_bits < 1 || cf.weight_bits > 8) spqr::fail(spqr::Errc::config_invalid, "weight bits must be in [1, 8]");
        if ((cf.scale_bits < 1 || cf.scale_bits > 8) && cf.scale_bits != 16)
            spqr::fail(spqr::Errc::config_invalid, "scale bits must be in [1, 8] or 16");
        if ((cf.zero_bits < 1 || cf.zero_bits > 8) && cf.zero_bits != 16)
            spqr::fail(spqr::Errc::config_invalid, "zero bits must be in [1, 8] or 16");
        if (cf.beta1 < 1 || cf.beta2 < 1) spqr::fail(spqr::Errc::config_invalid, "group sizes must be >= 1");
        if (cf.beta1 > static_cast<std::uint32_t>(kMaxBeta1))
            spqr::fail(spqr::Errc::config_invalid, "GPU encoder: beta1 must be <= 256");
        if (std::isnan(cf.tau) || cf.tau < 0.0) spqr::fail(spqr::Errc::config_invalid, "tau must be >= 0");
        if (cf.lambda_rel < 0.0) spqr::fail(spqr::Errc::config_invalid, "lambda_rel must be >= 0");
        if (cf.integer_zero && cf.zero_bits != 16 && cf.zero_bits < cf.weight_bits)
            spqr::fail(spqr::Errc::config_invalid, "integer zero points need zero bits >= weight bits");
        if (h->samples < 1) spqr::fail(spqr::Errc::empty_input, "no calibration samples accumulated");
        if (m == 0) spqr::fail(spqr::Errc::shape_mismatch, "tensor dimensions must be >= 1");
        cudaStream_t st = nullptr;
        cck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{st};
        Handles hd;
        bck(la().set_stream(hd.b, st), "set stream");
        sck(la().s_set_stream(hd.s, st), "set stream");

        // lambda = lambda_rel * mean(diag(H)) (hessian.hpp:140-143)
        std::vector<double> Hh(static_cast<std::size_t>(n) * n);
        cck(cudaMemcpy(Hh.data(), h->H.p, sizeof(double) * Hh.size(), cudaMemcpyDeviceToHost), "D2H H");
        double dsum = 0.0;
        for (std::uint32_t j = 0; j < n; ++j) dsum += Hh[static_cast<std::size_t>(j) * n + j];
        const double lambda = cf.lambda_rel * (dsum / n);
        // permutation (make_permutation, solver.hpp:381-404)
        std::vector<std::uint32_t> ident(n), order(n);
        std::iota(ident.begin(), ident.end(), 0u);
        DevBuf<std::uint32_t> d_ident(n), d_ord(n);
        cck(cudaMemcpy(d_ident.p, ident.data(), 4ull * n, cudaMemcpyHostToDevice), "H2D ident");
        order = ident;
        if (cf.order == 1) {
            if (cf.act_order_key == 1) {  // ascending diagonal of the regularized inverse: ||C(:, j)||^2
                DevBuf<double> C0 = inverse_cholesky(hd, h->H.p, d_ident.p, n, lambda, st);
                std::vector<double> Ch(static_cast<std::size_t>(n) * n);
                cck(cudaMemcpy(Ch.data(), C0.p, sizeof(double) * Ch.size(), cudaMemcpyDeviceToHost), "D2H C");
                std::vector<double> d(n, 0.0);
                for (std::uint32_t j = 0; j < n; ++j)
                    for (std::uint32_t i = 0; i < n; ++i) d[j] += Ch[static_cast<std::size_t>(i) * n + j] * Ch[static_cast<std::size_t>(i) * n + j];
                std::stable_sort(order.begin(), order.end(), [&](std::uint32_t x, std::uint32_t y) { return d[x] < d[y]; });
            } else {
                std::stable_sort(order.begin(), order.end(), [&](std::uint32_t x, std::uint32_t y) {
                    return Hh[static_cast<std::size_t>(x) * n + x] > Hh[static_cast<std::size_t>(y) * n + y];
                });
            }
        } else if (cf.order == 2) {
            std::mt19937_64 rng(cf.seed);
            std::shuffle(order.begin(), order.end(), rng);
        } else if (cf.order != 0) {
            spqr::fail(spqr::Errc::config_invalid, "unknown column order");
        }
        const bool identity = std::equal(order.begin(), order.end(), ident.begin());
        cck(cudaMemcpy(d_ord.p, order.data(), 4ull * n, cudaMemcpyHostToDevice), "H2D order");
        DevBuf<double> C = inverse_cholesky(hd, h->H.p, d_ord.p, n, lambda, st);

        // working copy in solve order (binary64) and its pristine copy
        const std::uint64_t mn = static_cast<std::uint64_t>(m) * n;
        DevBuf<double> Wp(mn), W0p(mn);
        permute_w<<<blocks_for(mn), 256, 0, st>>>(w_dev, d_ord.p, Wp.p, m, n);
        cck(cudaMemcpyAsync(W0p.p, Wp.p, sizeof(double) * mn, cudaMemcpyDeviceToDevice, st), "copy W0p");
        DevBuf<std::uint8_t> codes(mn), omask(mn), mask(static_cast<std::size_t>(m) * cf.beta1);
        DevBuf<std::uint16_t> oval(mn);
        cck(cudaMemsetAsync(omask.p, 0, mn, st), "memset omask");
        const std::uint32_t nblk = (n + cf.beta1 - 1) / cf.beta1, ng = (m + cf.beta2 - 1) / cf.beta2;
        DevBuf<double> s1(m), z1(m), errs(static_cast<std::size_t>(m) * cf.beta1);
        DevBuf<std::uint8_t> scode(static_cast<std::size_t>(nblk) * m), zcode(static_cast<std::size_t>(nblk) * m);
        DevBuf<std::uint16_t> scal(static_cast<std::size_t>(nblk) * ng * 4);
        DevBuf<float> sf(static_cast<std::size_t>(nblk) * m), zf(static_cast<std::size_t>(nblk) * m);
        EncCfg ec{cf.weight_bits, cf.scale_bits, cf.zero_bits, cf.beta1, cf.beta2,
                  QFlags{cf.full_range_sign != 0, cf.integer_zero != 0}, cf.outliers_enabled != 0, cf.tau};
        const double minus_one = -1.0, one = 1.0;
        for (std::uint32_t k = 0; k < nblk; ++k) {
            const std::uint32_t i0 = k * cf.beta1, bw = std::min(cf.beta1, n - i0);
            enc_screen_fit<<<blocks_for(m, 128), 128, 0, st>>>(Wp.p, C.p, m, n, i0, bw, ec, mask.p, s1.p, z1.p);
            enc_fit2<<<blocks_for(ng, 128), 128, 0, st>>>(s1.p, z1.p, m, ec, scode.p + static_cast<std::size_t>(k) * m,
                                                          zcode.p + static_cast<std::size_t>(k) * m,
                                                          scal.p + static_cast<std::size_t>(k) * ng * 4,
                                                          sf.p + static_cast<std::size_t>(k) * m,
                                                          zf.p + static_cast<std::size_t>(k) * m);
            enc_columns<<<blocks_for(m, 128), 128, 0, st>>>(Wp.p, C.p, m, n, i0, bw, cf.weight_bits, mask.p,
                                                            sf.p + static_cast<std::size_t>(k) * m,
                                                            zf.p + static_cast<std::size_t>(k) * m, codes.p, omask.p,
                                                            oval.p, errs.p);
            cck(cudaGetLastError(), "launch encoder block kernels");
            if (i0 + bw < n) {
                // Wp(:, i0+bw:) -= errs (m x bw) * C(i0:i0+bw, i0+bw:)  (solver.hpp:492-494), in
                // column-major terms: WpT(i0+bw:, :) -= CT(i0+bw:, i0:i0+bw) * errsT
                const int M = static_cast<int>(n - i0 - bw), N = static_cast<int>(m), K = static_cast<int>(bw);
                bck(la().dgemm(hd.b, CUBLAS_OP_N, CUBLAS_OP_N, M, N, K, &minus_one,
                               C.p + static_cast<std::size_t>(i0) * n + i0 + bw, static_cast<int>(n), errs.p,
                               static_cast<int>(bw), &one, Wp.p + i0 + bw, static_cast<int>(n)),
                    "dgemm trailing update");
            }
        }
        // report: relative layer error against the (permuted) Hessian (solver.hpp:406-413, :509-517)
        double num = 0.0, den = 0.0;
        {
            DevBuf<double> delta(mn), T(mn), Hp(static_cast<std::size_t>(n) * n), acc(2);
            recon_delta<<<blocks_for(mn), 256, 0, st>>>(W0p.p, codes.p, omask.p, oval.p, sf.p, zf.p, m, n, cf.beta1,
                                                        delta.p);
            // Hp(i, j) = H(ord[i], ord[j]) without regularization: regularize with lambda 0 and the
            // dead-column rule off is not available, so gather directly
            std::vector<double> Hph(static_cast<std::size_t>(n) * n);
            for (std::uint32_t i = 0; i < n; ++i)
                for (std::uint32_t j = 0; j < n; ++j)
                    Hph[static_cast<std::size_t>(i) * n + j] = Hh[static_cast<std::size_t>(order[i]) * n + order[j]];
            cck(cudaMemcpyAsync(Hp.p, Hph.data(), sizeof(double) * Hph.size(), cudaMemcpyHostToDevice, st), "H2D Hp");
            const double zero = 0.0;
            // T = delta * Hp (row-major m x n): column-major T^T = Hp^T delta^T = Hp delta^T
            bck(la().dgemm(hd.b, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(m), static_cast<int>(n),
                           &one, Hp.p, static_cast<int>(n), delta.p, static_cast<int>(n), &zero, T.p, static_cast<int>(n)),
                "dgemm delta H");
            dot_sum<<<1, 256, 0, st>>>(T.p, delta.p, mn, acc.p);
            bck(la().dgemm(hd.b, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(m), static_cast<int>(n),
                           &one, Hp.p, static_cast<int>(n), W0p.p, static_cast<int>(n), &zero, T.p, static_cast<int>(n)),
                "dgemm W0 H");
            dot_sum<<<1, 256, 0, st>>>(T.p, W0p.p, mn, acc.p + 1);
            double hv[2];
            cck(cudaMemcpyAsync(hv, acc.p, 16, cudaMemcpyDeviceToHost, st), "D2H report");
            cck(cudaStreamSynchronize(st), "sync encoder");
            num = hv[0];
            den = hv[1];
        }
        // the tensor on the host (make_spqr_tensor, format.hpp:69-89) and encode
        spqr::SpqrTensor t;
        t.rows = m;
        t.cols = n;
        t.weight_bits = cf.weight_bits;
        t.scale_bits = cf.scale_bits;
        t.zero_bits = cf.zero_bits;
        t.beta1 = cf.beta1;
        t.beta2 = cf.beta2;
        t.act_order = cf.order == 1;
        t.integer_zero = cf.integer_zero != 0;
        t.full_range_sign = cf.full_range_sign != 0;
        t.outliers_enabled = cf.outliers_enabled != 0;
        t.tau = static_cast<float>(cf.tau);
        t.lambda_rel = static_cast<float>(cf.lambda_rel);
        t.permutation = identity ? spqr::Permutation::identity(n) : spqr::Permutation::from_order(order);
        t.codes.rows = m;
        t.codes.cols = n;
        t.codes.bits = cf.weight_bits;
        t.codes.codes.resize(mn);
        cck(cudaMemcpy(t.codes.codes.data(), codes.p, mn, cudaMemcpyDeviceToHost), "D2H codes");
        t.stats.rows = m;
        t.stats.cols = n;
        t.stats.beta1 = cf.beta1;
        t.stats.beta2 = cf.beta2;
        t.stats.scale_bits = cf.scale_bits;
        t.stats.zero_bits = cf.zero_bits;
        {
            std::vector<std::uint8_t> sc(static_cast<std::size_t>(nblk) * m), zc(static_cast<std::size_t>(nblk) * m);
            std::vector<std::uint16_t> scl(static_cast<std::size_t>(nblk) * ng * 4);
            std::vector<float> sfh(static_cast<std::size_t>(nblk) * m), zfh(static_cast<std::size_t>(nblk) * m);
            cck(cudaMemcpy(sc.data(), scode.p, sc.size(), cudaMemcpyDeviceToHost), "D2H scode");
            cck(cudaMemcpy(zc.data(), zcode.p, zc.size(), cudaMemcpyDeviceToHost), "D2H zcode");
            cck(cudaMemcpy(scl.data(), scal.p, 2 * scl.size(), cudaMemcpyDeviceToHost), "D2H scalars");
            cck(cudaMemcpy(sfh.data(), sf.p, 4 * sfh.size(), cudaMemcpyDeviceToHost), "D2H sf");
            cck(cudaMemcpy(zfh.data(), zf.p, 4 * zfh.size(), cudaMemcpyDeviceToHost), "D2H zf");
            const bool any_codes = cf.scale_bits != 16 || cf.zero_bits != 16;
            for (std::uint32_t k = 0; k < nblk; ++k) {
                spqr::BlockStats b;
                const std::size_t o = static_cast<std::size_t>(k) * m;
                if (cf.scale_bits == 16)
                    b.raw_scales.assign(sfh.begin() + o, sfh.begin() + o + m);
                else
                    b.scale_codes.assign(sc.begin() + o, sc.begin() + o + m);
                if (cf.zero_bits == 16)
                    b.raw_zeros.assign(zfh.begin() + o, zfh.begin() + o + m);
                else
                    b.zero_codes.assign(zc.begin() + o, zc.begin() + o + m);
                if (any_codes) {
                    b.groups.resize(ng);
                    for (std::uint32_t gi = 0; gi < ng; ++gi) {
                        const std::uint16_t* q = &scl[(static_cast<std::size_t>(k) * ng + gi) * 4];
                        b.groups[gi].scale_s = q[0];
                        b.groups[gi].scale_z = q[1];
                        b.groups[gi].zero_s = q[2];
                        b.groups[gi].zero_z = q[3];
                    }
                }
                t.stats.blocks.push_back(std::move(b));
            }
        }
        {
            std::vector<std::uint8_t> om(mn);
            std::vector<std::uint16_t> ov(mn);
            cck(cudaMemcpy(om.data(), omask.p, mn, cudaMemcpyDeviceToHost), "D2H omask");
            cck(cudaMemcpy(ov.data(), oval.p, 2 * mn, cudaMemcpyDeviceToHost), "D2H oval");
            t.outliers.rows = m;
            t.outliers.cols = n;
            for (std::uint32_t r = 0; r < m; ++r)
                for (std::uint32_t k = 0; k < n; ++k)
                    if (om[static_cast<std::size_t>(r) * n + k])
                        t.outliers.items.push_back({r, k, ov[static_cast<std::size_t>(r) * n + k]});
            t.outliers.validate();  // outlier_budget_exceeded above 5 % (solver.hpp:94-96)
        }
        const std::vector<std::uint8_t> bytes = spqr::encode(t);
        if (report) {
            report[0] = den <= 0.0 ? 0.0 : num / den;
            report[1] = t.outliers.rate();
            report[2] = spqr::measured_bits_per_param(t.layout());
        }
        *len = bytes.size();
        if (!out || cap < bytes.size()) {
            spqr::detail::set_last_error("buffer too small");
            rc = SPQR_E_BUFFER_TOO_SMALL;
            return;
        }
        std::memcpy(out, bytes.data(), bytes.size());
    });
    return g ? g : rc;
}

// tune_tau (solver.hpp:546-640): the smallest tau on the 0.05-step grid over
// [0.1, 1.0] whose outlier rate stays at or below the target, by the
// reference's binary search; report[3] = that tau, report[4] = target reached.
int spqr_quantize_layer_tuned(const spqr_hessian* h, const float* w_dev, uint32_t m, const spqr_encoder_cfg* cfg,
                              double target_rate, uint8_t* out, size_t cap, size_t* len, double* report) {
    return spqr::detail::guard([&] {
        if (!(target_rate > 0.0) || target_rate > 0.05)
            spqr::fail(spqr::Errc::config_invalid, "target outlier rate must be in (0, 0.05]");
        spqr_encoder_cfg c = *cfg;
        c.outliers_enabled = 1;
        constexpr double kTauMin = 0.1, kTauStep = 0.05;
        constexpr int kGridMax = 18;
        auto tau_at = [&](int k) { return kTauMin + kTauStep * k; };
        std::vector<std::uint8_t> best;
        double best_rep[3] = {0, 0, 0};
        int best_k = -1;
        auto probe = [&](int k) {  // true: feasible (rate <= target)
            c.tau = tau_at(k);
            std::vector<std::uint8_t> buf(cap ? cap : 1);
            std::size_t n = 0;
            double rep[3];
            const int st = spqr_quantize_layer(h, w_dev, m, &c, buf.data(), buf.size(), &n, rep);
            if (st == 1 + static_cast<int>(spqr::Errc::outlier_budget_exceeded)) return false;
            if (st) throw spqr::Error(static_cast<spqr::Errc>(st - 1), spqr_last_error());
            if (rep[1] <= target_rate) {
                buf.resize(n);
                best = std::move(buf);
                std::copy(rep, rep + 3, best_rep);
                best_k = k;
                return true;
            }
            return false;
        };
        int chosen = -1;
        bool reached = true;
        if (probe(0)) {
            chosen = 0;
        } else if (!probe(kGridMax)) {  // above target even at tau = 1.0: report, do not fail
            reached = false;
            c.tau = tau_at(kGridMax);
            std::vector<std::uint8_t> buf(cap ? cap : 1);
            std::size_t n = 0;
            const int st = spqr_quantize_layer(h, w_dev, m, &c, buf.data(), buf.size(), &n, best_rep);
            if (st) throw spqr::Error(static_cast<spqr::Errc>(st - 1), spqr_last_error());
            buf.resize(n);
            best = std::move(buf);
            chosen = kGridMax;
        } else {
            int lo = 0, hi = kGridMax;
            while (hi - lo > 1) {
                const int mid = (lo + hi) / 2;
                if (probe(mid))
                    hi = mid;
                else
                    lo = mid;
            }
            if (best_k != hi) probe(hi);
            chosen = hi;
        }
        if (report) {
            std::copy(best_rep, best_rep + 3, report);
            report[3] = tau_at(chosen);
            report[4] = reached ? 1.0 : 0.0;
        }
        *len = best.size();
        if (!out || cap < best.size()) spqr::fail(spqr::Errc::config_invalid, "output buffer too small");
        std::memcpy(out, best.data(), best.size());
    });
}

}  // extern "C"
