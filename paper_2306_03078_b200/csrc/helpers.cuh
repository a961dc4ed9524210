// helpers.cuh -- packed f32x2 math, FMA-pipe shifts and the statistics-field
// readers shared by the sm_100a kernels.  Included by kernels.cuh (inside
// namespace spqr_dev).

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

// A lane's statistics field (tiled.hpp) as its two code streams: st[0] =
// rows g (lo stream), st[1] = rows g + 8 (hi stream), pair j at bit BS*j.
template <int BS>
__device__ __forceinline__ void load_stat_streams(const std::uint8_t* stats, int lane, std::uint32_t (&st)[2]) {
    std::uint32_t w0, w1 = 0;
    if constexpr (BS == 3) {
        w0 = reinterpret_cast<const std::uint32_t*>(stats)[lane];
        w1 = __byte_perm(reinterpret_cast<const std::uint16_t*>(stats + 128)[lane], 0u, 0x4140);
    } else if constexpr (BS == 2) {
        w0 = reinterpret_cast<const std::uint32_t*>(stats)[lane];
    } else {
        const uint2 v = reinterpret_cast<const uint2*>(stats)[lane];
        w0 = v.x;
        w1 = v.y;
    }
    st[0] = __byte_perm(w0, w1, 0x5410);  // lo halves
    st[1] = __byte_perm(w0, w1, 0x7632);  // hi halves
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
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

