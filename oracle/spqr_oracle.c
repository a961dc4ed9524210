/*
 * spqr_oracle.c -- CPU restatement of the reference SpQR decode path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product (paper_2306_03078_b200/) never links or calls it.
 *
 * It restates, in plain C99, the algorithm of the header-only C++ reference
 * under /root/reference/proj/include/spqr/ (read-only, never copied):
 *
 *   fp16 conversions ........ common.hpp:70-126
 *   quant arithmetic ........ quantizer.hpp:45-67  (max_code, dequant_value, stat_dequant)
 *   stream size model ....... layout.hpp:12-77
 *   BilevelStats::scale_at .. solver.hpp:129-141
 *   Permutation ............. hessian.hpp:14-48
 *   encode / decode ......... format.hpp:98-500
 *   estimate_avg_bits ....... format.hpp:531-542
 *   reconstruct_solve_order . solver.hpp:345-362
 *   dequantize_full ......... kernel.hpp:17-25
 *   build_tile_plan ......... kernel.hpp:54-84
 *   matvec (tiled, fp64) .... kernel.hpp:89-124
 *   matvec_naive ............ kernel.hpp:131-142
 *   relative_l2 ............. kernel.hpp:154-163
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement against the
 * reference itself compiled from /root/reference (oracle/_ref/, built by
 * oracle/Makefile) and against the committed golden fixtures in tests/golden/.
 *
 * Error convention: functions return 0 on success, 1 + Errc (same enumerator
 * order as common.hpp:10-27) on failure.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Errc order, common.hpp:10-27 */
enum {
    E_MALFORMED_HEADER = 1, E_SHAPE_MISMATCH, E_NON_FINITE, E_IO, E_PARSE, E_MISSING_FILE,
    E_EMPTY_INPUT, E_NOT_PD, E_DIM_MISMATCH, E_CONFIG_INVALID, E_COL_OVERFLOW,
    E_MALFORMED_STREAM, E_VERSION, E_CORRUPT_CSR, E_ILL_COND, E_OUTLIER_BUDGET
};

#define RAW_STATS_BITS 16 /* quantizer.hpp:45 */
#define HEADER_BYTES 48   /* layout.hpp:12 */

/* ---------------------------------------------------------------- fp16 -- */
/* common.hpp:70-99: RNE narrowing, saturating to +-65504 instead of inf. */
uint16_t oracle_fp16_from_float(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
    uint32_t e8 = (x >> 23) & 0xffu, mant = x & 0x7fffffu;
    if (e8 == 0xffu) return (uint16_t)(sign | 0x7c00u | (mant ? 0x200u : 0u));
    int e = (int)e8 - 127 + 15;
    if (e >= 31) return (uint16_t)(sign | 0x7bffu);
    if (e <= 0) {
        if (e < -10) return sign;
        mant |= 0x800000u;
        uint32_t sh = (uint32_t)(14 - e);
        uint32_t h = mant >> sh, rem = mant & ((1u << sh) - 1u), half = 1u << (sh - 1u);
        if (rem > half || (rem == half && (h & 1u))) h++;
        return (uint16_t)(sign | h);
    }
    uint32_t h = ((uint32_t)e << 10) | (mant >> 13), rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
    if (h >= 0x7c00u) h = 0x7bffu;
    return (uint16_t)(sign | h);
}

/* common.hpp:101-126: exact widening (subnormals renormalised). */
float oracle_fp16_to_float(uint16_t h) {
    uint32_t sign = (uint32_t)(h & 0x8000u) << 16, e = (h >> 10) & 0x1fu, m = h & 0x3ffu, x;
    if (e == 0) {
        if (m == 0) {
            x = sign;
        } else {
            int s = 0;
            while (!(m & 0x400u)) { m <<= 1; s++; }
            m &= 0x3ffu;
            x = sign | ((uint32_t)(127 - 15 + 1 - s) << 23) | (m << 13);
        }
    } else if (e == 31) {
        x = sign | 0x7f800000u | (m << 13);
    } else {
        x = sign | ((e - 15 + 127) << 23) | (m << 13);
    }
    float f;
    memcpy(&f, &x, 4);
    return f;
}

/* quantizer.hpp:60-67 -- binary32 reconstruction shared by every pipeline. */
static float dequant_value(float s, float z, uint32_t code) { return s * ((float)code - z); }
static float stat_dequant(uint16_t s16, uint16_t z16, uint32_t code) {
    return dequant_value(oracle_fp16_to_float(s16), oracle_fp16_to_float(z16), code);
}

/* ---------------------------------------------------------- size model -- */
static size_t packed_bytes(size_t count, int bits) { return (count * (size_t)bits + 7) / 8; } /* layout.hpp:14-16 */

static size_t record_bytes(int sb, int zb, int wb, uint32_t gr, uint32_t bw) { /* layout.hpp:30-44 */
    size_t b = 0;
    b += sb <= 8 ? 4 + packed_bytes(gr, sb) : 4 * (size_t)gr;
    b += zb <= 8 ? 4 + packed_bytes(gr, zb) : 4 * (size_t)gr;
    b += packed_bytes((size_t)gr * bw, wb);
    return b;
}

size_t oracle_payload_bytes(uint32_t rows, uint32_t cols, int wb, int sb, int zb, uint32_t b1,
                            uint32_t b2, uint32_t nnz, int has_perm) { /* layout.hpp:47-64 */
    size_t bytes = has_perm ? 4 * (size_t)cols : 0;
    uint32_t nb = (cols + b1 - 1) / b1, ng = (rows + b2 - 1) / b2;
    for (uint32_t k = 0; k < nb; ++k) {
        uint32_t bw = b1 < cols - k * b1 ? b1 : cols - k * b1;
        for (uint32_t g = 0; g < ng; ++g) {
            uint32_t gr = b2 < rows - g * b2 ? b2 : rows - g * b2;
            bytes += record_bytes(sb, zb, wb, gr, bw);
        }
    }
    return bytes + 4 * ((size_t)rows + 1) + 4 * (size_t)nnz;
}

/* format.hpp:531-542 */
int oracle_estimate_avg_bits(int bw, int bs, int bz, uint32_t b1, uint32_t b2, double ro, double* out) {
    if (bw < 1 || bs < 1 || bz < 1 || b1 < 1 || b2 < 1 || ro < 0.0) return E_CONFIG_INVALID;
    out[1] = bw;
    out[2] = (double)(bs + bz) / b1;
    out[3] = 64.0 / ((double)b1 * b2);
    out[4] = 32.0 * ro;
    out[0] = out[1] + out[2] + out[3] + out[4];
    return 0;
}

/* -------------------------------------------------------------- tensor -- */
/* Mirror of SpqrTensor (format.hpp:32-67) with BilevelStats / OutlierSet /
 * Permutation (solver.hpp:66-142, hessian.hpp:14-48) flattened into arrays. */
typedef struct oracle_tensor {
    uint32_t rows, cols;
    int wb, sb, zb;
    uint32_t b1, b2;
    uint16_t flags;
    float tau, lambda_rel;
    int has_perm;
    uint32_t* order;     /* n: solve position -> source column */
    uint8_t* codes;      /* m*n row-major, solve order */
    uint8_t* scodes;     /* nblocks*m */
    uint8_t* zcodes;     /* nblocks*m */
    float* raw_s;        /* nblocks*m */
    float* raw_z;        /* nblocks*m */
    uint16_t* scal;      /* nblocks*ngroups*4: scale_s, scale_z, zero_s, zero_z */
    uint32_t nnz;
    uint32_t* orow;
    uint32_t* ocol;
    uint16_t* oval;
} oracle_tensor;

void oracle_free(oracle_tensor* t) {
    if (!t) return;
    free(t->order); free(t->codes); free(t->scodes); free(t->zcodes);
    free(t->raw_s); free(t->raw_z); free(t->scal); free(t->orow); free(t->ocol); free(t->oval);
    free(t);
}

static uint32_t nblocks(const oracle_tensor* t) { return (t->cols + t->b1 - 1) / t->b1; }
static uint32_t ngroups(const oracle_tensor* t) { return (t->rows + t->b2 - 1) / t->b2; }

/* BilevelStats::scale_at / zero_at, solver.hpp:129-141 */
static float scale_at(const oracle_tensor* t, uint32_t k, uint32_t r) {
    size_t i = (size_t)k * t->rows + r;
    if (t->sb == RAW_STATS_BITS) return t->raw_s[i];
    const uint16_t* g = t->scal + ((size_t)k * ngroups(t) + r / t->b2) * 4;
    return stat_dequant(g[0], g[1], t->scodes[i]);
}
static float zero_at(const oracle_tensor* t, uint32_t k, uint32_t r) {
    size_t i = (size_t)k * t->rows + r;
    if (t->zb == RAW_STATS_BITS) return t->raw_z[i];
    const uint16_t* g = t->scal + ((size_t)k * ngroups(t) + r / t->b2) * 4;
    return stat_dequant(g[2], g[3], t->zcodes[i]);
}

void oracle_info(const oracle_tensor* t, uint32_t* u32_out, int32_t* i32_out) {
    u32_out[0] = t->rows; u32_out[1] = t->cols; u32_out[2] = t->b1; u32_out[3] = t->b2;
    u32_out[4] = t->nnz; u32_out[5] = t->flags;
    i32_out[0] = t->wb; i32_out[1] = t->sb; i32_out[2] = t->zb; i32_out[3] = t->has_perm;
}

/* ---------------------------------------------------------------- decode -- */
typedef struct { const uint8_t* p; size_t n, pos; } rd_t;
static int rd_need(rd_t* r, size_t k) { return r->n - r->pos >= k; }
static uint32_t rd_u32(rd_t* r) {
    const uint8_t* q = r->p + r->pos; r->pos += 4;
    return (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16) | ((uint32_t)q[3] << 24);
}
static uint16_t rd_u16(rd_t* r) { const uint8_t* q = r->p + r->pos; r->pos += 2; return (uint16_t)(q[0] | (q[1] << 8)); }
/* ByteReader::packed, format.hpp:169-186: LSB-first, field padded to a byte. */
static void rd_packed(rd_t* r, uint8_t* dst, size_t count, int bits) {
    uint64_t acc = 0; int have = 0; size_t bp = r->pos; uint32_t mask = (1u << bits) - 1u;
    for (size_t i = 0; i < count; ++i) {
        while (have < bits) { acc |= (uint64_t)r->p[bp++] << have; have += 8; }
        dst[i] = (uint8_t)(acc & mask); acc >>= bits; have -= bits;
    }
    r->pos += packed_bytes(count, bits);
}

#define FAIL(code) do { rc = (code); goto fail; } while (0)

/* decode, format.hpp:354-500, with the same validation order and Errc codes. */
int oracle_decode(const uint8_t* bytes, size_t n, oracle_tensor** out) {
    int rc = 0;
    rd_t r = {bytes, n, 0};
    oracle_tensor* t = (oracle_tensor*)calloc(1, sizeof(oracle_tensor));
    uint32_t* rs = NULL;
    *out = NULL;
    if (!rd_need(&r, HEADER_BYTES)) FAIL(E_MALFORMED_STREAM);
    if (memcmp(bytes, "SPQR", 4) != 0) FAIL(E_MALFORMED_STREAM);
    r.pos = 4;
    if (rd_u16(&r) != 1) FAIL(E_VERSION);
    t->flags = rd_u16(&r);
    t->rows = rd_u32(&r); t->cols = rd_u32(&r);
    t->wb = bytes[16]; t->sb = bytes[17]; t->zb = bytes[18]; r.pos = 20;
    t->b1 = rd_u32(&r); t->b2 = rd_u32(&r);
    uint32_t nnz = rd_u32(&r);
    { uint32_t u = rd_u32(&r); memcpy(&t->tau, &u, 4); u = rd_u32(&r); memcpy(&t->lambda_rel, &u, 4); }
    r.pos = HEADER_BYTES;
    if (t->rows == 0 || t->cols == 0) FAIL(E_MALFORMED_STREAM);
    if (t->wb < 1 || t->wb > 8) FAIL(E_MALFORMED_STREAM);
#define STAT_OK(b) (((b) >= 1 && (b) <= 8) || (b) == RAW_STATS_BITS)
    if (!STAT_OK(t->sb) || !STAT_OK(t->zb)) FAIL(E_MALFORMED_STREAM);
    if (t->b1 < 1 || t->b2 < 1) FAIL(E_MALFORMED_STREAM);
    if (nnz > 0 && t->cols > 0xffffu) FAIL(E_MALFORMED_STREAM);
    t->has_perm = (t->flags & 1u) != 0;
    if (n != HEADER_BYTES + oracle_payload_bytes(t->rows, t->cols, t->wb, t->sb, t->zb, t->b1, t->b2,
                                                 nnz, t->has_perm))
        FAIL(E_MALFORMED_STREAM);

    const uint32_t m = t->rows, nc = t->cols, NB = nblocks(t), NG = ngroups(t);
    t->order = (uint32_t*)malloc(sizeof(uint32_t) * nc);
    if (t->has_perm) { /* Permutation::from_order, hessian.hpp:27-39 */
        uint8_t* seen = (uint8_t*)calloc(nc, 1);
        for (uint32_t k = 0; k < nc; ++k) {
            uint32_t s = rd_u32(&r);
            if (s >= nc || seen[s]) { free(seen); FAIL(E_MALFORMED_STREAM); }
            seen[s] = 1; t->order[k] = s;
        }
        free(seen);
        /* SpqrTensor::has_permutation() is !is_identity(): an identity order
         * stored with the flag re-encodes without it (format.hpp:52). */
        int ident = 1;
        for (uint32_t k = 0; k < nc; ++k) if (t->order[k] != k) { ident = 0; break; }
        if (ident) t->has_perm = 0;
    } else {
        for (uint32_t k = 0; k < nc; ++k) t->order[k] = k;
    }

    const int anyq = t->sb != RAW_STATS_BITS || t->zb != RAW_STATS_BITS;
    t->codes = (uint8_t*)calloc((size_t)m * nc, 1);
    if (t->sb != RAW_STATS_BITS) t->scodes = (uint8_t*)calloc((size_t)NB * m, 1);
    else t->raw_s = (float*)calloc((size_t)NB * m, 4);
    if (t->zb != RAW_STATS_BITS) t->zcodes = (uint8_t*)calloc((size_t)NB * m, 1);
    else t->raw_z = (float*)calloc((size_t)NB * m, 4);
    t->scal = (uint16_t*)malloc(sizeof(uint16_t) * 4 * (size_t)NB * NG);
    for (size_t i = 0; i < (size_t)NB * NG; ++i) { /* StatGroupScalars defaults, solver.hpp:102-107 */
        t->scal[4 * i + 0] = 0x3c00; t->scal[4 * i + 1] = 0; t->scal[4 * i + 2] = 0x3c00; t->scal[4 * i + 3] = 0;
    }
    (void)anyq;
    uint8_t* wbuf = (uint8_t*)malloc((size_t)t->b1 * t->b2 + 1);
    for (uint32_t k = 0; k < NB; ++k) { /* format.hpp:428-471 */
        uint32_t c0 = k * t->b1, bw = t->b1 < nc - c0 ? t->b1 : nc - c0;
        for (uint32_t g = 0; g < NG; ++g) {
            uint32_t r0 = g * t->b2, gr = t->b2 < m - r0 ? t->b2 : m - r0;
            uint16_t* gs = t->scal + ((size_t)k * NG + g) * 4;
            if (t->sb != RAW_STATS_BITS) {
                gs[0] = rd_u16(&r); gs[1] = rd_u16(&r);
                if (oracle_fp16_to_float(gs[0]) < 0.0f) { free(wbuf); FAIL(E_MALFORMED_STREAM); }
            }
            if (t->zb != RAW_STATS_BITS) { gs[2] = rd_u16(&r); gs[3] = rd_u16(&r); }
            if (t->sb != RAW_STATS_BITS) rd_packed(&r, t->scodes + (size_t)k * m + r0, gr, t->sb);
            else for (uint32_t i = 0; i < gr; ++i) { uint32_t u = rd_u32(&r); memcpy(&t->raw_s[(size_t)k * m + r0 + i], &u, 4); }
            if (t->zb != RAW_STATS_BITS) rd_packed(&r, t->zcodes + (size_t)k * m + r0, gr, t->zb);
            else for (uint32_t i = 0; i < gr; ++i) { uint32_t u = rd_u32(&r); memcpy(&t->raw_z[(size_t)k * m + r0 + i], &u, 4); }
            rd_packed(&r, wbuf, (size_t)gr * bw, t->wb);
            for (uint32_t rr = 0; rr < gr; ++rr)
                for (uint32_t c = 0; c < bw; ++c)
                    t->codes[(size_t)(r0 + rr) * nc + c0 + c] = wbuf[(size_t)rr * bw + c];
        }
    }
    free(wbuf);

    /* CSR, format.hpp:473-498 */
    rs = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)m + 1));
    for (uint32_t i = 0; i <= m; ++i) rs[i] = rd_u32(&r);
    if (rs[0] != 0) FAIL(E_CORRUPT_CSR);
    for (uint32_t i = 0; i < m; ++i) if (rs[i + 1] < rs[i]) FAIL(E_CORRUPT_CSR);
    if (rs[m] != nnz) FAIL(E_CORRUPT_CSR);
    t->nnz = nnz;
    t->orow = (uint32_t*)malloc(4 * ((size_t)nnz + 1));
    t->ocol = (uint32_t*)malloc(4 * ((size_t)nnz + 1));
    t->oval = (uint16_t*)malloc(2 * ((size_t)nnz + 1));
    {
        uint32_t row = 0;
        for (uint32_t i = 0; i < nnz; ++i) {
            while (row < m && rs[row + 1] <= i) ++row;
            t->orow[i] = row; t->ocol[i] = rd_u16(&r); t->oval[i] = rd_u16(&r);
            if (t->ocol[i] >= nc) FAIL(E_CORRUPT_CSR);
            if (i > 0 && t->orow[i - 1] == row && t->ocol[i - 1] >= t->ocol[i]) FAIL(E_CORRUPT_CSR);
        }
    }
    if (r.pos != n) FAIL(E_MALFORMED_STREAM);
    free(rs);
    *out = t;
    return 0;
fail:
    free(rs);
    oracle_free(t);
    return rc;
}

/* ---------------------------------------------------------------- encode -- */
typedef struct { uint8_t* p; size_t n, cap; int oom; } wr_t;
static void wr_byte(wr_t* w, uint8_t b) { if (w->n < w->cap) w->p[w->n] = b; else w->oom = 1; w->n++; }
static void wr_u16(wr_t* w, uint16_t v) { wr_byte(w, (uint8_t)v); wr_byte(w, (uint8_t)(v >> 8)); }
static void wr_u32(wr_t* w, uint32_t v) { for (int i = 0; i < 4; ++i) wr_byte(w, (uint8_t)(v >> (8 * i))); }
/* BitWriter + put_packed, format.hpp:98-124, 212-217 */
static void wr_packed(wr_t* w, const uint8_t* src, size_t count, int bits) {
    uint64_t acc = 0; int nb = 0;
    for (size_t i = 0; i < count; ++i) {
        acc |= (uint64_t)src[i] << nb; nb += bits;
        while (nb >= 8) { wr_byte(w, (uint8_t)acc); acc >>= 8; nb -= 8; }
    }
    if (nb > 0) wr_byte(w, (uint8_t)acc);
}

/* encode, format.hpp:269-352 (validation subset: format.hpp:219-265). */
int oracle_encode(const oracle_tensor* t, uint8_t* out, size_t cap, size_t* len) {
    const uint32_t m = t->rows, nc = t->cols, NB = nblocks(t), NG = ngroups(t);
    const uint32_t maxq = (1u << t->wb) - 1u;
    if (m == 0 || nc == 0) return E_SHAPE_MISMATCH;
    for (size_t i = 0; i < (size_t)m * nc; ++i) if (t->codes[i] > maxq) return E_SHAPE_MISMATCH;
    for (uint32_t i = 0; i + 1 < t->nnz; ++i) {
        int lt = t->orow[i] != t->orow[i + 1] ? t->orow[i] < t->orow[i + 1] : t->ocol[i] < t->ocol[i + 1];
        if (!lt) return E_CORRUPT_CSR;
    }
    for (uint32_t i = 0; i < t->nnz; ++i) if (t->orow[i] >= m || t->ocol[i] >= nc) return E_CORRUPT_CSR;
    if ((double)t->nnz / ((double)m * nc) > 0.05) return E_OUTLIER_BUDGET;
    if (t->nnz > 0 && nc > 0xffffu) return E_COL_OVERFLOW;

    wr_t w = {out, 0, cap, 0};
    uint16_t flags = t->flags & (uint16_t)~1u;
    if (t->has_perm) flags |= 1u;
    wr_byte(&w, 'S'); wr_byte(&w, 'P'); wr_byte(&w, 'Q'); wr_byte(&w, 'R');
    wr_u16(&w, 1); wr_u16(&w, flags); wr_u32(&w, m); wr_u32(&w, nc);
    wr_byte(&w, (uint8_t)t->wb); wr_byte(&w, (uint8_t)t->sb); wr_byte(&w, (uint8_t)t->zb); wr_byte(&w, 0);
    wr_u32(&w, t->b1); wr_u32(&w, t->b2); wr_u32(&w, t->nnz);
    { uint32_t u; memcpy(&u, &t->tau, 4); wr_u32(&w, u); memcpy(&u, &t->lambda_rel, 4); wr_u32(&w, u); }
    for (int i = 0; i < 8; ++i) wr_byte(&w, 0);
    if (t->has_perm) for (uint32_t k = 0; k < nc; ++k) wr_u32(&w, t->order[k]);
    uint8_t* wbuf = (uint8_t*)malloc((size_t)t->b1 * t->b2 + 1);
    for (uint32_t k = 0; k < NB; ++k) {
        uint32_t c0 = k * t->b1, bw = t->b1 < nc - c0 ? t->b1 : nc - c0;
        for (uint32_t g = 0; g < NG; ++g) {
            uint32_t r0 = g * t->b2, gr = t->b2 < m - r0 ? t->b2 : m - r0;
            const uint16_t* gs = t->scal + ((size_t)k * NG + g) * 4;
            if (t->sb != RAW_STATS_BITS) { wr_u16(&w, gs[0]); wr_u16(&w, gs[1]); }
            if (t->zb != RAW_STATS_BITS) { wr_u16(&w, gs[2]); wr_u16(&w, gs[3]); }
            if (t->sb != RAW_STATS_BITS) wr_packed(&w, t->scodes + (size_t)k * m + r0, gr, t->sb);
            else for (uint32_t i = 0; i < gr; ++i) { uint32_t u; memcpy(&u, &t->raw_s[(size_t)k * m + r0 + i], 4); wr_u32(&w, u); }
            if (t->zb != RAW_STATS_BITS) wr_packed(&w, t->zcodes + (size_t)k * m + r0, gr, t->zb);
            else for (uint32_t i = 0; i < gr; ++i) { uint32_t u; memcpy(&u, &t->raw_z[(size_t)k * m + r0 + i], 4); wr_u32(&w, u); }
            for (uint32_t rr = 0; rr < gr; ++rr)
                for (uint32_t c = 0; c < bw; ++c) wbuf[(size_t)rr * bw + c] = t->codes[(size_t)(r0 + rr) * nc + c0 + c];
            wr_packed(&w, wbuf, (size_t)gr * bw, t->wb);
        }
    }
    free(wbuf);
    /* CSR section, format.hpp:337-350 */
    uint32_t cursor = 0; size_t item = 0;
    wr_u32(&w, 0);
    for (uint32_t rr = 0; rr < m; ++rr) {
        while (item < t->nnz && t->orow[item] == rr) { ++item; ++cursor; }
        wr_u32(&w, cursor);
    }
    for (uint32_t i = 0; i < t->nnz; ++i) { wr_u16(&w, (uint16_t)t->ocol[i]); wr_u16(&w, t->oval[i]); }
    *len = w.n;
    return w.oom ? E_IO : 0;
}

/* Build a tensor from flat arrays (the layout documented on oracle_tensor);
 * used by tests to encode synthetic tensors.  Arrays are copied. */
int oracle_from_arrays(uint32_t rows, uint32_t cols, int wb, int sb, int zb, uint32_t b1, uint32_t b2,
                       uint16_t flags, float tau, float lambda_rel, const uint32_t* order,
                       const uint8_t* codes, const uint8_t* scodes, const uint8_t* zcodes,
                       const float* raw_s, const float* raw_z, const uint16_t* scal, uint32_t nnz,
                       const uint32_t* orow, const uint32_t* ocol, const uint16_t* oval,
                       oracle_tensor** out) {
    oracle_tensor* t = (oracle_tensor*)calloc(1, sizeof(oracle_tensor));
    t->rows = rows; t->cols = cols; t->wb = wb; t->sb = sb; t->zb = zb; t->b1 = b1; t->b2 = b2;
    t->flags = flags; t->tau = tau; t->lambda_rel = lambda_rel;
    const uint32_t NB = nblocks(t), NG = ngroups(t);
    t->order = (uint32_t*)malloc(4 * (size_t)cols);
    t->has_perm = 0;
    for (uint32_t k = 0; k < cols; ++k) {
        t->order[k] = order ? order[k] : k;
        if (t->order[k] != k) t->has_perm = 1;
    }
    t->codes = (uint8_t*)malloc((size_t)rows * cols);
    memcpy(t->codes, codes, (size_t)rows * cols);
    if (sb != RAW_STATS_BITS) { t->scodes = (uint8_t*)malloc((size_t)NB * rows); memcpy(t->scodes, scodes, (size_t)NB * rows); }
    else { t->raw_s = (float*)malloc(4 * (size_t)NB * rows); memcpy(t->raw_s, raw_s, 4 * (size_t)NB * rows); }
    if (zb != RAW_STATS_BITS) { t->zcodes = (uint8_t*)malloc((size_t)NB * rows); memcpy(t->zcodes, zcodes, (size_t)NB * rows); }
    else { t->raw_z = (float*)malloc(4 * (size_t)NB * rows); memcpy(t->raw_z, raw_z, 4 * (size_t)NB * rows); }
    t->scal = (uint16_t*)malloc(8 * (size_t)NB * NG);
    if (scal) memcpy(t->scal, scal, 8 * (size_t)NB * NG);
    else for (size_t i = 0; i < (size_t)NB * NG; ++i) { t->scal[4*i] = 0x3c00; t->scal[4*i+1] = 0; t->scal[4*i+2] = 0x3c00; t->scal[4*i+3] = 0; }
    t->nnz = nnz;
    t->orow = (uint32_t*)malloc(4 * ((size_t)nnz + 1));
    t->ocol = (uint32_t*)malloc(4 * ((size_t)nnz + 1));
    t->oval = (uint16_t*)malloc(2 * ((size_t)nnz + 1));
    if (nnz) { memcpy(t->orow, orow, 4 * (size_t)nnz); memcpy(t->ocol, ocol, 4 * (size_t)nnz); memcpy(t->oval, oval, 2 * (size_t)nnz); }
    *out = t;
    return 0;
}

/* ---------------------------------------------------------- dequantize -- */
/* reconstruct_solve_order (solver.hpp:345-362) + column un-permute
 * (kernel.hpp:17-25).  `out` is m*n row-major in ORIGINAL column order. */
int oracle_dequantize_full(const oracle_tensor* t, float* out) {
    const uint32_t m = t->rows, nc = t->cols, NB = nblocks(t);
    float* solve = t->has_perm ? (float*)malloc(4 * (size_t)m * nc) : out;
    for (uint32_t k = 0; k < NB; ++k) {
        uint32_t c0 = k * t->b1, bw = t->b1 < nc - c0 ? t->b1 : nc - c0;
        for (uint32_t r = 0; r < m; ++r) {
            float s = scale_at(t, k, r), z = zero_at(t, k, r);
            for (uint32_t c = c0; c < c0 + bw; ++c)
                solve[(size_t)r * nc + c] = dequant_value(s, z, t->codes[(size_t)r * nc + c]);
        }
    }
    for (uint32_t i = 0; i < t->nnz; ++i) /* separate binary32 add, solver.hpp:360 */
        solve[(size_t)t->orow[i] * nc + t->ocol[i]] += oracle_fp16_to_float(t->oval[i]);
    if (t->has_perm) {
        for (uint32_t r = 0; r < m; ++r)
            for (uint32_t k = 0; k < nc; ++k) out[(size_t)r * nc + t->order[k]] = solve[(size_t)r * nc + k];
        free(solve);
    }
    return 0;
}

/* -------------------------------------------------------------- matvec -- */
/* build_tile_plan (kernel.hpp:54-84) + matvec (kernel.hpp:89-124): tiles of
 * tile_rows x beta1, per-(tile,row) CSR slices, binary64 accumulation. */
int oracle_matvec(const oracle_tensor* t, const float* x, float* y, uint32_t tile_rows) {
    if (tile_rows == 0) return E_CONFIG_INVALID;
    const uint32_t m = t->rows, nc = t->cols, NB = nblocks(t);
    float* xp = (float*)malloc(4 * (size_t)nc);
    for (uint32_t k = 0; k < nc; ++k) xp[k] = x[t->order[k]];
    uint32_t* rs = (uint32_t*)calloc((size_t)m + 1, 4);
    for (uint32_t i = 0; i < t->nnz; ++i) rs[t->orow[i] + 1]++;
    for (uint32_t r = 0; r < m; ++r) rs[r + 1] += rs[r];
    double* acc_y = (double*)calloc(m, sizeof(double));
    for (uint32_t r0 = 0; r0 < m; r0 += tile_rows) {
        uint32_t r1 = r0 + tile_rows < m ? r0 + tile_rows : m;
        for (uint32_t k = 0; k < NB; ++k) {
            uint32_t c0 = k * t->b1, c1 = c0 + t->b1 < nc ? c0 + t->b1 : nc;
            for (uint32_t r = r0; r < r1; ++r) {
                float s = scale_at(t, k, r), z = zero_at(t, k, r);
                double acc = 0.0;
                const uint8_t* cr = t->codes + (size_t)r * nc;
                for (uint32_t c = c0; c < c1; ++c) acc += (double)dequant_value(s, z, cr[c]) * (double)xp[c];
                uint32_t beg = rs[r], end = rs[r + 1];
                while (beg < end && t->ocol[beg] < c0) ++beg;
                for (uint32_t i = beg; i < end && t->ocol[i] < c1; ++i)
                    acc += (double)oracle_fp16_to_float(t->oval[i]) * (double)xp[t->ocol[i]];
                acc_y[r] += acc;
            }
        }
    }
    for (uint32_t r = 0; r < m; ++r) y[r] = (float)acc_y[r];
    free(acc_y); free(rs); free(xp);
    return 0;
}

/* matvec_naive, kernel.hpp:131-142 */
int oracle_matvec_naive(const oracle_tensor* t, const float* x, float* y) {
    const uint32_t m = t->rows, nc = t->cols;
    float* w = (float*)malloc(4 * (size_t)m * nc);
    oracle_dequantize_full(t, w);
    for (uint32_t r = 0; r < m; ++r) {
        double acc = 0.0;
        for (uint32_t c = 0; c < nc; ++c) acc += (double)w[(size_t)r * nc + c] * (double)x[c];
        y[r] = (float)acc;
    }
    free(w);
    return 0;
}

/* relative_l2, kernel.hpp:154-163 */
double oracle_relative_l2(const float* a, const float* b, size_t n) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double d = (double)a[i] - b[i];
        num += d * d;
        den += (double)b[i] * b[i];
    }
    return den == 0.0 ? sqrt(num) : sqrt(num / den);
}
