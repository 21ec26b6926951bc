/*
 * paro_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the PAROAttention reference hot path, used ONLY by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker. Nothing in the product (paro_b200/, include/) links or calls this.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference's proj/ directory). Compile with -ffp-contract=off: the
 * reference's bit-exact contract forbids mul+add contraction
 * (proj/CMakeLists.txt:12-14).
 *
 * Parity of this restatement is pinned two ways (see tests/test_oracle.py):
 *   1. against the reference library itself built from its own sources into
 *      oracle/_ref/ (bit-exact: permutations, masks, quantizer codes/scales,
 *      and the fp-QK engine output with PARO_KERNELS=scalar), and
 *   2. against golden fixtures under tests/golden/ generated from that build.
 * The INT8-QK engine mode has no reference implementation;
 * it differs from the pinned fp-QK mode only in the logit line.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_CONFIG 2 /* ConfigError/ShapeError/InputError, error.hpp:21-30 */
#define ORACLE_FORMAT 3 /* FormatError/IoError, error.hpp:31-36 */

/* ------------------------------------------------------------------------- */
/* Token grid + permutation: tensor.cpp:70-93 (flat_index, grid_coords),     */
/* reorder.cpp:49-72 (make_perm).                                              */
/* ------------------------------------------------------------------------- */
int oracle_make_perm(int ndim, const char* labels, const uint32_t* extents, const char* order,
                     uint32_t* forward, uint32_t* inverse) {
    if ((int)strlen(order) != ndim)
        return ORACLE_CONFIG; /* reorder.cpp:50-51 */
    int src_axis[3];
    uint32_t pext[3];
    for (int a = 0; a < ndim; ++a) {
        int found = -1;
        for (int b = 0; b < ndim; ++b)
            if (labels[b] == order[a])
                found = b;
        if (found < 0)
            return ORACLE_CONFIG; /* axis_index throws InputError, tensor.cpp:56-61 */
        src_axis[a] = found;
        pext[a] = extents[found];
    }
    size_t n = 1;
    for (int a = 0; a < ndim; ++a)
        n *= extents[a];
    for (size_t old = 0; old < n; ++old) {
        uint32_t coords[3];
        size_t idx = old;
        for (int a = ndim; a-- > 0;) { /* grid_coords: tensor.cpp:84-93 */
            coords[a] = (uint32_t)(idx % extents[a]);
            idx /= extents[a];
        }
        size_t nw = 0;
        for (int a = 0; a < ndim; ++a) /* flat_index over the permuted grid */
            nw = nw * pext[a] + coords[src_axis[a]];
        forward[old] = (uint32_t)nw;
        inverse[nw] = (uint32_t)old;
    }
    return ORACLE_OK;
}

/* apply_perm_rows: out.row(i) = m.row(inverse[i]) (reorder.cpp:93-101). */
void oracle_apply_perm_rows(const float* m, size_t rows, size_t cols, const uint32_t* inverse, float* out) {
    for (size_t i = 0; i < rows; ++i)
        memcpy(out + i * cols, m + (size_t)inverse[i] * cols, cols * sizeof(float));
}

/* ------------------------------------------------------------------------- */
/* Scalar kernels: kernels_scalar.cpp:37-42 (max_abs), :44-53 (min_max),       */
/* :78-85 (quant_affine, round half away from zero).                           */
/* ------------------------------------------------------------------------- */
static float k_max_abs(const float* x, size_t n) {
    float m = 0.0f;
    for (size_t i = 0; i < n; ++i) {
        float a = fabsf(x[i]);
        m = m > a ? m : a; /* std::max(m, fabs(x)) keeps m on ties */
    }
    return m;
}

static void k_min_max(const float* x, size_t n, float* mn, float* mx) {
    float lo = x[0], hi = x[0];
    for (size_t i = 1; i < n; ++i) {
        lo = (x[i] < lo) ? x[i] : lo; /* std::min(lo, x) */
        hi = (hi < x[i]) ? x[i] : hi; /* std::max(hi, x) */
    }
    *mn = lo;
    *mx = hi;
}

static void k_quant_affine(const float* x, size_t n, float offset, float scale, int32_t qmin, int32_t qmax,
                           int32_t* codes) {
    for (size_t i = 0; i < n; ++i) {
        float q = (x[i] - offset) / scale;
        float fmx = (float)qmax, fmn = (float)qmin;
        q = (q > fmn) ? q : fmn; /* std::max(qmin, q) */
        q = (fmx < q) ? fmx : q; /* std::min(qmax, q) */
        codes[i] = (int32_t)roundf(q);
    }
}

/* round-half-away KAT helper (test_kernels.cpp:100-117) */
void oracle_quant_affine(const float* x, size_t n, float offset, float scale, int32_t qmin, int32_t qmax,
                         int32_t* codes) {
    k_quant_affine(x, n, offset, scale, qmin, qmax, codes);
}

/* ------------------------------------------------------------------------- */
/* quantize(m, {bits, mode, PerBlock, block}) -- quant.cpp:45-56 (group order)  */
/* and :60-104. mode 0 = Unsigned, 1 = Symmetric (quant.hpp:19-22).            */
/* scales/offsets are emitted in group order; offsets only for Unsigned.      */
/* Returns ORACLE_CONFIG for bad bits/block or negative unsigned input.       */
/* ------------------------------------------------------------------------- */
int oracle_quantize(const float* m, size_t rows, size_t cols, int bits, int mode, size_t block, int32_t* codes,
                    float* scales, float* offsets) {
    if ((bits != 4 && bits != 8) || block < 1)
        return ORACLE_CONFIG; /* quant.cpp:15-20 */
    const int32_t qmin = mode == 0 ? 0 : -((1 << (bits - 1)) - 1); /* quant.cpp:22-28 */
    const int32_t qmax = mode == 0 ? (1 << bits) - 1 : (1 << (bits - 1)) - 1;
    const float fq = (float)qmax;
    size_t gi = 0;
    for (size_t r0 = 0; r0 < rows; r0 += block) {
        const size_t r1 = r0 + block < rows ? r0 + block : rows;
        for (size_t c0 = 0; c0 < cols; c0 += block) {
            const size_t c1 = c0 + block < cols ? c0 + block : cols;
            float scale = 1.0f, offset = 0.0f;
            if (mode == 0) {
                float mn = m[r0 * cols + c0], mx = mn;
                for (size_t r = r0; r < r1; ++r) {
                    float rmn, rmx;
                    k_min_max(m + r * cols + c0, c1 - c0, &rmn, &rmx);
                    mn = rmn < mn ? rmn : mn;
                    mx = mx < rmx ? rmx : mx;
                }
                if (mn < 0.0f)
                    return ORACLE_CONFIG; /* InputError, quant.cpp:82-83 */
                scale = (mx - mn) / fq;
                offset = mn;
                if (scale == 0.0f)
                    scale = 1.0f;
            } else {
                float amax = 0.0f;
                for (size_t r = r0; r < r1; ++r) {
                    float a = k_max_abs(m + r * cols + c0, c1 - c0);
                    amax = amax < a ? a : amax;
                }
                scale = amax / fq;
                if (scale == 0.0f)
                    scale = 1.0f;
            }
            scales[gi] = scale;
            if (mode == 0 && offsets)
                offsets[gi] = offset;
            ++gi;
            for (size_t r = r0; r < r1; ++r)
                k_quant_affine(m + r * cols + c0, c1 - c0, offset, scale, qmin, qmax, codes + r * cols + c0);
        }
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------- */
/* V tile quantizer inside the engine: attention.cpp:104-126.                  */
/* One symmetric group per key tile over all d columns; colsum per column.     */
/* ------------------------------------------------------------------------- */
void oracle_quant_v(const float* v, size_t n, size_t d, size_t block, int bits, int32_t* codes, float* scales,
                    int64_t* colsum) {
    const size_t kb = (n + block - 1) / block;
    const float qmax = (float)((1 << (bits - 1)) - 1);
    for (size_t bj = 0; bj < kb; ++bj) {
        const size_t ks = bj * block, ke = ks + block < n ? ks + block : n;
        float amax = 0.0f;
        for (size_t r = ks; r < ke; ++r) {
            float a = k_max_abs(v + r * d, d);
            amax = amax < a ? a : amax;
        }
        const float s = amax == 0.0f ? 1.0f : amax / qmax;
        scales[bj] = s;
        for (size_t r = ks; r < ke; ++r)
            k_quant_affine(v + r * d, d, 0.0f, s, -(int32_t)qmax, (int32_t)qmax, codes + r * d);
        for (size_t c = 0; c < d; ++c) {
            int64_t acc = 0;
            for (size_t r = ks; r < ke; ++r)
                acc += codes[r * d + c];
            colsum[bj * d + c] = acc;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* stream_engine restatement: attention.cpp:84-254 (quantized variant, with    */
/* dense_prefix handling of :148-199).                                          */
/*   qk_mode 0: logits = scale * fp64 dot of fp32 rows (reference semantics,    */
/*              attention.cpp:162-168 / kernels_scalar.cpp:11-16);             */
/*   qk_mode 1: logits = scale * sum_g (sq[qb,g]*sk[bj,g]) * S_g with S_g the   */
/*              int32 dot of the per-64x64-group int8 codes produced by         */
/*              quantize({8, Symmetric, PerBlock, block}) (the restated INT8-QK */
/*              stage); the rest is unchanged.                  */
/*   pv_bits 0: unquantized masked streaming (masked_blocked_attention,         */
/*              attention.cpp:262-264); 4/8: quantized_blocked_attention.       */
/* mask: k x k bytes row-major (BlockMask::bits, mask.hpp:15-32) or NULL.       */
/* zeroed: n bytes, set to 1 for rows with no kept tile (attention.cpp:244-247).*/
/* ------------------------------------------------------------------------- */
static double dot_f(const float* a, const float* b, size_t n) {
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i)
        acc += (double)a[i] * (double)b[i];
    return acc;
}

/* Rows of q-blocks [qb_begin, qb_end) only (the engine is independent per
 * q-tile, attention.cpp:134); other output rows are left untouched. */
/* Optional P-code dump of the quantized tiles of one q-block (test hook): per
 * kept tile in the engine's order, the key block, the group's (lo, pscale) and
 * the codes [block][block] (rows x true key columns, row-major, rest 0). */
typedef struct {
    size_t qb, max_tiles, ntiles;
    uint8_t* codes;
    float* lo;
    float* pscale;
    int32_t* bj;
} pdump_t;

static int engine_impl(const float* q, const float* k, const float* v, size_t n, size_t d, float scale_in,
                       size_t dense_prefix, size_t block, const uint8_t* mask, int pv_bits, int qk_mode,
                       size_t qb_begin, size_t qb_end, float* out, uint8_t* zeroed, pdump_t* dump) {
    if (n == 0 || d == 0 || block < 1)
        return ORACLE_CONFIG;
    if (dense_prefix > n)
        return ORACLE_CONFIG;
    if (pv_bits != 0 && pv_bits != 4 && pv_bits != 8)
        return ORACLE_CONFIG;
    const size_t kblocks = (n + block - 1) / block;
    const double scale = scale_in != 0.0f ? (double)scale_in : 1.0 / sqrt((double)d); /* attention.cpp:26-28 */
    const size_t dp = dense_prefix;

    /* restated INT8-QK prologue */
    int32_t *qc = NULL, *kc = NULL;
    float *qs = NULL, *ks_ = NULL;
    const size_t dg = (d + block - 1) / block;
    if (qk_mode == 1) {
        qc = (int32_t*)malloc(n * d * sizeof(int32_t));
        kc = (int32_t*)malloc(n * d * sizeof(int32_t));
        qs = (float*)malloc(kblocks * dg * sizeof(float));
        ks_ = (float*)malloc(kblocks * dg * sizeof(float));
        oracle_quantize(q, n, d, 8, 1, block, qc, qs, NULL);
        oracle_quantize(k, n, d, 8, 1, block, kc, ks_, NULL);
    }

    int32_t* vcodes = NULL;
    float* vscale = NULL;
    int64_t* vcolsum = NULL;
    if (pv_bits) {
        vcodes = (int32_t*)malloc(n * d * sizeof(int32_t));
        vscale = (float*)malloc(kblocks * sizeof(float));
        vcolsum = (int64_t*)malloc(kblocks * d * sizeof(int64_t));
        oracle_quant_v(v, n, d, block, pv_bits, vcodes, vscale, vcolsum);
    }

    double* row_max = (double*)malloc(block * sizeof(double));
    double* row_sum = (double*)malloc(block * sizeof(double));
    double* acc = (double*)malloc(block * d * sizeof(double));
    double* s = (double*)malloc(block * block * sizeof(double));
    float* ptile = (float*)malloc(block * block * sizeof(float));
    int32_t* pcodes = (int32_t*)malloc(block * sizeof(int32_t));
    for (size_t qs0 = qb_begin * block; qs0 < n && qs0 < qb_end * block; qs0 += block) {
        const size_t qe = qs0 + block < n ? qs0 + block : n;
        const size_t qn = qe - qs0;
        const size_t qb = qs0 / block;
        for (size_t r = 0; r < qn; ++r) {
            row_max[r] = -INFINITY;
            row_sum[r] = 0.0;
        }
        memset(acc, 0, qn * d * sizeof(double));

        for (size_t bj = 0; bj < kblocks; ++bj) {
            const size_t ks0 = bj * block;
            const size_t ke = ks0 + block < n ? ks0 + block : n;
            const size_t kn = ke - ks0;
            const int tile_dense = ks0 < dp;
            const int tile_kept = tile_dense || mask == NULL || mask[qb * kblocks + bj];
            const int has_prefix_rows = qs0 < dp;
            if (!tile_kept && !has_prefix_rows)
                continue;
            int any_quant_rows = 0;
            for (size_t r = 0; r < qn; ++r) {
                const size_t i = qs0 + r;
                const int row_dense = i < dp;
                if (!tile_kept && !row_dense)
                    continue;
                double* srow = s + r * kn;
                double tmax = -INFINITY;
                for (size_t j = 0; j < kn; ++j) {
                    double logit;
                    if (qk_mode == 1) {
                        double acc_g = 0.0;
                        for (size_t g = 0; g < dg; ++g) {
                            const size_t c0 = g * block, c1 = c0 + block < d ? c0 + block : d;
                            int64_t sg = 0;
                            for (size_t c = c0; c < c1; ++c)
                                sg += (int64_t)qc[i * d + c] * kc[(ks0 + j) * d + c];
                            acc_g += ((double)qs[qb * dg + g] * (double)ks_[bj * dg + g]) * (double)sg;
                        }
                        logit = scale * acc_g;
                    } else {
                        logit = scale * dot_f(q + i * d, k + (ks0 + j) * d, d);
                    }
                    srow[j] = logit;
                    tmax = tmax < logit ? logit : tmax;
                }
                const double m_new = row_max[r] < tmax ? tmax : row_max[r];
                if (row_sum[r] > 0.0) {
                    const double gamma = exp(row_max[r] - m_new);
                    if (gamma != 1.0) {
                        row_sum[r] *= gamma;
                        for (size_t c = 0; c < d; ++c)
                            acc[r * d + c] *= gamma;
                    }
                }
                row_max[r] = m_new;
                float* prow = ptile + r * kn;
                double psum = 0.0;
                for (size_t j = 0; j < kn; ++j) {
                    const double p = exp(srow[j] - m_new);
                    psum += p;
                    srow[j] = p;
                    prow[j] = (float)p;
                }
                row_sum[r] += psum;
                const int quantize_row = pv_bits && !row_dense && !tile_dense;
                if (!quantize_row) {
                    for (size_t j = 0; j < kn; ++j)
                        for (size_t c = 0; c < d; ++c) /* axpy_scalar, kernels_scalar.cpp:18-21 */
                            acc[r * d + c] += srow[j] * (double)v[(ks0 + j) * d + c];
                } else {
                    any_quant_rows = 1;
                }
            }
            if (pv_bits && any_quant_rows) { /* attention.cpp:201-239 */
                float mn = 0.0f, mx = 0.0f;
                int first = 1;
                for (size_t r = 0; r < qn; ++r) {
                    const size_t i = qs0 + r;
                    if (i < dp || (!tile_kept && i >= dp))
                        continue;
                    float rmn, rmx;
                    k_min_max(ptile + r * kn, kn, &rmn, &rmx);
                    mn = first ? rmn : (rmn < mn ? rmn : mn);
                    mx = first ? rmx : (mx < rmx ? rmx : mx);
                    first = 0;
                }
                const float qmax = (float)((1u << pv_bits) - 1);
                float pscale = (mx - mn) / qmax;
                if (pscale == 0.0f)
                    pscale = 1.0f;
                const float poffset = mn;
                uint8_t* dcodes = NULL;
                if (dump && qb == dump->qb && dump->ntiles < dump->max_tiles) {
                    const size_t t = dump->ntiles++;
                    dump->lo[t] = poffset;
                    dump->pscale[t] = pscale;
                    dump->bj[t] = (int32_t)bj;
                    dcodes = dump->codes + t * block * block;
                    memset(dcodes, 0, block * block);
                }
                for (size_t r = 0; r < qn; ++r) {
                    const size_t i = qs0 + r;
                    if (i < dp || (!tile_kept && i >= dp))
                        continue;
                    k_quant_affine(ptile + r * kn, kn, poffset, pscale, 0, (int32_t)qmax, pcodes);
                    if (dcodes)
                        for (size_t j = 0; j < kn; ++j)
                            dcodes[r * block + j] = (uint8_t)pcodes[j];
                    const double ss = (double)pscale * (double)vscale[bj];
                    const double os = (double)poffset * (double)vscale[bj];
                    for (size_t c = 0; c < d; ++c) {
                        int64_t ip = 0;
                        for (size_t j = 0; j < kn; ++j)
                            ip += (int64_t)pcodes[j] * vcodes[(ks0 + j) * d + c];
                        acc[r * d + c] += ss * (double)ip + os * (double)vcolsum[bj * d + c];
                    }
                }
            }
        }
        for (size_t r = 0; r < qn; ++r) {
            float* o = out + (qs0 + r) * d;
            zeroed[qs0 + r] = 0;
            if (row_sum[r] == 0.0) {
                zeroed[qs0 + r] = 1;
                memset(o, 0, d * sizeof(float));
                continue;
            }
            for (size_t c = 0; c < d; ++c)
                o[c] = (float)(acc[r * d + c] / row_sum[r]);
        }
    }
    free(row_max);
    free(row_sum);
    free(acc);
    free(s);
    free(ptile);
    free(pcodes);
    free(qc);
    free(kc);
    free(qs);
    free(ks_);
    free(vcodes);
    free(vscale);
    free(vcolsum);
    return ORACLE_OK;
}

int oracle_stream_engine_range(const float* q, const float* k, const float* v, size_t n, size_t d, float scale_in,
                               size_t dense_prefix, size_t block, const uint8_t* mask, int pv_bits, int qk_mode,
                               size_t qb_begin, size_t qb_end, float* out, uint8_t* zeroed) {
    return engine_impl(q, k, v, n, d, scale_in, dense_prefix, block, mask, pv_bits, qk_mode, qb_begin, qb_end, out,
                       zeroed, NULL);
}

/* q-block qb's output rows plus its P-code dump (codes [max_tiles][block][block],
 * lo / pscale / bj [max_tiles]); returns the number of quantized tiles in *ntiles */
int oracle_stream_engine_pdump(const float* q, const float* k, const float* v, size_t n, size_t d, float scale_in,
                               size_t block, const uint8_t* mask, int pv_bits, size_t qb, size_t max_tiles,
                               uint8_t* codes, float* lo, float* pscale, int32_t* bj, size_t* ntiles, float* out,
                               uint8_t* zeroed) {
    pdump_t dmp = {qb, max_tiles, 0, codes, lo, pscale, bj};
    const int rc = engine_impl(q, k, v, n, d, scale_in, 0, block, mask, pv_bits, 1, qb, qb + 1, out, zeroed, &dmp);
    *ntiles = dmp.ntiles;
    return rc;
}

int oracle_stream_engine(const float* q, const float* k, const float* v, size_t n, size_t d, float scale_in,
                         size_t dense_prefix, size_t block, const uint8_t* mask, int pv_bits, int qk_mode, float* out,
                         uint8_t* zeroed) {
    return oracle_stream_engine_range(q, k, v, n, d, scale_in, dense_prefix, block, mask, pv_bits, qk_mode, 0,
                                      (n + block - 1) / block, out, zeroed);
}

/* ------------------------------------------------------------------------- */
/* One head through cmd_run's chain (proj/tools/main.cpp:276-305): permute Q/K/V */
/* by the plan (apply_perm_rows x3), run the engine on the permuted rows with   */
/* the mask, then undo the permutation of the output (plan.inverted()).         */
/* zeroed is reported in PERMUTED row order, as AttnResult::zeroed_rows is.     */
/* ------------------------------------------------------------------------- */
int oracle_paro_head(const float* q, const float* k, const float* v, size_t n, size_t d, float scale,
                     const uint32_t* forward, const uint32_t* inverse, const uint8_t* mask, int pv_bits, int qk_mode,
                     float* out, uint8_t* zeroed) {
    float* pq = (float*)malloc(n * d * sizeof(float));
    float* pk = (float*)malloc(n * d * sizeof(float));
    float* pv = (float*)malloc(n * d * sizeof(float));
    float* po = (float*)malloc(n * d * sizeof(float));
    oracle_apply_perm_rows(q, n, d, inverse, pq);
    oracle_apply_perm_rows(k, n, d, inverse, pk);
    oracle_apply_perm_rows(v, n, d, inverse, pv);
    int rc = oracle_stream_engine(pq, pk, pv, n, d, scale, 0, 64, mask, pv_bits, qk_mode, po, zeroed);
    if (rc == ORACLE_OK)
        oracle_apply_perm_rows(po, n, d, forward, out); /* inverted(): inverse <- forward */
    free(pq);
    free(pk);
    free(pv);
    free(po);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* PMSK blob (mask.cpp:197-244): 18-byte header, rows padded to bytes, LSB first */
/* ------------------------------------------------------------------------- */
static void put_u32(uint8_t* p, uint32_t v) {
    p[0] = (uint8_t)(v & 0xff);
    p[1] = (uint8_t)((v >> 8) & 0xff);
    p[2] = (uint8_t)((v >> 16) & 0xff);
    p[3] = (uint8_t)((v >> 24) & 0xff);
}
static uint32_t get_u32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

size_t oracle_pmsk_size(size_t k_rows, size_t k_cols) {
    return 18 + k_rows * ((k_cols + 7) / 8);
}

void oracle_serialize_mask(const uint8_t* bits, size_t k_rows, size_t k_cols, size_t block, uint8_t* out) {
    const size_t row_bytes = (k_cols + 7) / 8;
    memcpy(out, "PMSK", 4);
    out[4] = 1;
    out[5] = 0;
    put_u32(out + 6, (uint32_t)k_rows);
    put_u32(out + 10, (uint32_t)k_cols);
    put_u32(out + 14, (uint32_t)block);
    memset(out + 18, 0, k_rows * row_bytes);
    for (size_t i = 0; i < k_rows; ++i)
        for (size_t j = 0; j < k_cols; ++j)
            if (bits[i * k_cols + j])
                out[18 + i * row_bytes + j / 8] |= (uint8_t)(1u << (j % 8));
}

/* returns 0 or ORACLE_FORMAT; fills dims; bits (k_rows*k_cols) may be NULL */
int oracle_deserialize_mask(const uint8_t* data, size_t size, uint32_t* k_rows, uint32_t* k_cols, uint32_t* block,
                            uint8_t* bits, size_t* consumed) {
    if (size < 18 || memcmp(data, "PMSK", 4) != 0 || data[4] != 1)
        return ORACLE_FORMAT;
    const uint32_t kr = get_u32(data + 6), kc = get_u32(data + 10), b = get_u32(data + 14);
    if (kr == 0 || kc == 0 || b == 0)
        return ORACLE_FORMAT;
    const size_t row_bytes = (kc + 7) / 8;
    const size_t need = 18 + (size_t)kr * row_bytes;
    if (size < need)
        return ORACLE_FORMAT;
    *k_rows = kr;
    *k_cols = kc;
    *block = b;
    if (bits)
        for (size_t i = 0; i < kr; ++i)
            for (size_t j = 0; j < kc; ++j)
                bits[i * kc + j] = (data[18 + i * row_bytes + j / 8] >> (j % 8)) & 1u;
    if (consumed)
        *consumed = need;
    return ORACLE_OK;
}
