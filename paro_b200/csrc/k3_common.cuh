// k3_common.cuh -- pieces of K3 (attention_kernel.cu) shared with its experimental
// variants: packed fp32x2 / exp2 helpers, TMEM loads, launch parameters, work
// items, mbarrier wait flavours, the exact-path row statistics and the P-code
// dump hook.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "layer.cuh"
#include "ptx.cuh"

namespace paro {

#ifndef PARO_DYNAMIC
#define PARO_DYNAMIC 1
#endif

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---- packed fp32x2 helpers (FFMA2 / FADD2 / FMUL2 on sm_100a)
__device__ __forceinline__ uint64_t pk(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t add2_rm(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// int32 pair -> fp32 pair exactly (|x| < 2^22) on the FMA pipe instead of two ALU
// I2F: IMAD x * 1 + 0x4B400000 gives the bits of 1.5 * 2^23 + x, one packed FADD2
// of -1.5 * 2^23 leaves float(x). `one` must be a runtime 1 (a kernel parameter)
// or ptxas folds the IMAD into an ALU IADD3.
__device__ __forceinline__ uint64_t i2f2_fma(int32_t a, int32_t b, uint32_t one) {
    uint32_t ua, ub;
    asm("mad.lo.u32 %0, %1, %2, 1262485504;" : "=r"(ua) : "r"(a), "r"(one));
    asm("mad.lo.u32 %0, %1, %2, 1262485504;" : "=r"(ub) : "r"(b), "r"(one));
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(((uint64_t)ub << 32) | ua), "l"(0xCB400000CB400000ull));
    return r;
}
__device__ __forceinline__ uint32_t imad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
// the same for (x - s) with base = 0x4B400000 - s folded into the IMAD addend (|x - s| < 2^22)
__device__ __forceinline__ uint64_t i2f2_fma_b(int32_t a, int32_t b, uint32_t one, uint32_t base) {
    uint32_t ua, ub;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ua) : "r"(a), "r"(one), "r"(base));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ub) : "r"(b), "r"(one), "r"(base));
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(((uint64_t)ub << 32) | ua), "l"(0xCB400000CB400000ull));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// d=128 exp2 argument of a column pair, y = d0 c0 + d1 c1 + dmax (c_g = chi + clo exactly
// to 48 bits): p1 = fl(d1 c1hi) with its exact FMA residual e1, s = fl(d0 c0hi + p1) --
// one rounding of the (possibly cancelled) two-term sum -- plus the small terms and dmax.
// |y - exact| <= 2^-24 (|s| + |dmax| + |y|) + O(2^-48 |d c|), i.e. ~2^-23 |y| as at d=64.
__device__ __forceinline__ uint64_t arg128_2(uint64_t d0, uint64_t d1, uint64_t c0, uint64_t c1, uint64_t c0lo,
                                             uint64_t c1lo, uint64_t dmax) {
    // with nc_g = -c_g: p1n = -fl(d1 c1), e1 = d1 c1 + p1n exactly, sxn = -fl(d0 c0 - p1n)
    const uint64_t nc0 = c0 ^ 0x8000000080000000ull, nc1 = c1 ^ 0x8000000080000000ull; // per-tile constants
    const uint64_t p1n = mul2(d1, nc1);
    const uint64_t e1 = fma2(d1, c1, p1n);
    const uint64_t sxn = fma2(d0, nc0, p1n);
    const uint64_t t = fma2(d0, c0lo, fma2(d1, c1lo, add2(e1, dmax)));
    return sub2(t, sxn);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// Phase timers (PARO_K3_PROF builds only): clock64 deltas summed per warp role.
//   [0..7]  softmax: wait, pass1, reduce, pass2, exact, post, steps, items
//   [8..11] epilogue: wait, dequant, store, steps
//   [12..15] mma: wait KV/S, wait P/O, issue, steps
#ifdef PARO_K3_PROF
static __device__ unsigned long long g_prof[32];
static __device__ unsigned long long g_profq[8];
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(i, d) prof[i] += (unsigned long long)(d)
#else
#define PROF_T(v)
#define PROF_ADD(i, d)
#endif

struct K3Params {
    LayerDev L;
    double scale64;   // effective scale (AttnInputs::effective_scale, fp64)
    float scale_log2; // effective scale * log2(e)
    float p_qmax;     // 255 or 15
    float* out;       // [H][N][D] original token order
    uint8_t* zeroed;  // [H][N] or null
    const uint32_t* order; // LPT-sorted work items (h << 16 | p) of this launch
    uint32_t n_items;
    uint32_t* work_counter; // next index into `order` (zeroed before the launch; DYNAMIC)
    unsigned long long* stats; // optional debug counters: [0] warp-steps, [1] exact-path entries, [2] risky groups
    K3Dump dump;               // P-code dump test hook (dump.slot == nullptr: off)
    uint32_t one;              // 1, opaque to ptxas (i2f2_fma)
};

// P-code dump of one row's final codes for step t (cols [c0, c0 + 16*nch) of the
// row's 64 key columns; 64B-swizzled P tile rows as written by quantize_store)
__device__ __forceinline__ void dump_row(const K3Dump& dm, int32_t slot, uint32_t t, uint32_t r, const uint8_t* prow,
                                         int c0chunk, int nch) {
    uint8_t* dst = dm.codes + (((size_t)slot * dm.kb + t) * 64 + r) * 64;
    for (int c = c0chunk; c < c0chunk + nch; ++c)
        *reinterpret_cast<uint4*>(dst + 16 * c) = *reinterpret_cast<const uint4*>(prow + ((c ^ ((r >> 1) & 3)) << 4));
}
__device__ __forceinline__ void dump_meta(const K3Dump& dm, int32_t slot, uint32_t t, float lo, float pscale,
                                          uint32_t bj) {
    *reinterpret_cast<float4*>(dm.meta + ((size_t)slot * dm.kb + t) * 4) = make_float4(lo, pscale, (float)bj, 1.f);
}

struct Item {
    uint32_t h, qa, qb, na, nb, n; // qb = 0xffff when the pair has no B
};

__device__ __forceinline__ Item load_item(const LayerDev& L, uint32_t it) {
    Item x;
    x.h = it >> 16;
    const uint32_t p = it & 0xffffu;
    const uint32_t pr = L.pairs[(size_t)x.h * L.np + p];
    x.qa = pr & 0xffffu;
    x.qb = pr >> 16;
    x.na = L.qb_count[(size_t)x.h * L.kb2 + x.qa];
    x.nb = x.qb != 0xffffu ? L.qb_count[(size_t)x.h * L.kb2 + x.qb] : 0u;
    x.n = x.na > x.nb ? x.na : x.nb;
    return x;
}

// wait for several mbarrier phases, issuing the probes back to back so their
// latencies overlap (each try_wait costs ~90 cycles even when already complete)
__device__ __forceinline__ void mbar_wait2(uint32_t b0, uint32_t p0, uint32_t b1, uint32_t p1) {
    const bool r0 = ptx::mbar_try_wait(b0, p0);
    const bool r1 = ptx::mbar_try_wait(b1, p1);
    if (!r0)
        ptx::mbar_wait(b0, p0);
    if (!r1)
        ptx::mbar_wait(b1, p1);
}
// Waits of roles with slack (producer: 3-stage ring; epilogue: double-buffered
// O) back off with __nanosleep between probes so their spinning leaves the issue
// slots to the softmax and MMA warps on the same sub-partition.
#ifndef PARO_LAZY_NS
#define PARO_LAZY_NS 512
#endif
__device__ __forceinline__ void mbar_wait_lazy(uint32_t b, uint32_t p) {
    if (PARO_LAZY_NS == 0) {
        ptx::mbar_wait(b, p);
        return;
    }
    // no watchdog here: these roles wait on barriers that the softmax warps also
    // depend on, and their waits (ptx::mbar_wait) trap on a stalled pipeline
    while (!ptx::mbar_try_wait(b, p))
        __nanosleep(PARO_LAZY_NS);
}
// The MMA issuer has a step of slack too (S and P are double-buffered; a
// softmax step is ~5k cycles). Measured at c2 (K3 ms): spin everywhere 4.87;
// producer + epilogue 512 ns back-off 4.75; + MMA 500 ns 4.61 (1000: 4.61,
// 2000: 4.65); c5 unchanged within noise. Only the softmax waits stay hot.
#ifndef PARO_LAZY_MMA_NS
#define PARO_LAZY_MMA_NS 500
#endif
__device__ __forceinline__ void mbar_wait_mma(uint32_t b, uint32_t p) {
    if (PARO_LAZY_MMA_NS == 0) {
        ptx::mbar_wait(b, p);
        return;
    }
    while (!ptx::mbar_try_wait(b, p))
        __nanosleep(PARO_LAZY_MMA_NS);
}
__device__ __forceinline__ void mbar_wait3(uint32_t b0, uint32_t p0, uint32_t b1, uint32_t p1, uint32_t b2,
                                           uint32_t p2) {
    const bool r0 = ptx::mbar_try_wait(b0, p0);
    const bool r1 = ptx::mbar_try_wait(b1, p1);
    const bool r2 = ptx::mbar_try_wait(b2, p2);
    if (!r0)
        ptx::mbar_wait(b0, p0);
    if (!r1)
        ptx::mbar_wait(b1, p1);
    if (!r2)
        ptx::mbar_wait(b2, p2);
}

// the same with non-suspending probes first: a completed phase costs a test_wait,
// not a suspending try_wait (PARO_WAIT_TEST=0 restores mbar_wait3)
#ifndef PARO_WAIT_TEST
#define PARO_WAIT_TEST 1
#endif
__device__ __forceinline__ void mbar_wait3t(uint32_t b0, uint32_t p0, uint32_t b1, uint32_t p1, uint32_t b2,
                                            uint32_t p2) {
    if (PARO_WAIT_TEST && ptx::mbar_test(b0, p0) && ptx::mbar_test(b1, p1) && ptx::mbar_test(b2, p2))
        return;
    mbar_wait3(b0, p0, b1, p1, b2, p2);
}

__device__ __forceinline__ uint64_t fma2_rm(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Per-row, per-step exact statistics published for the boundary path (d=64):
// the exact (fp64, reference-order) min / max logit of the row's tile and the
// running max after it.
struct RowStat { // 40 bytes
    double tmin, tmax, m;
    float pmin, pmax; // the fast path's fp32 row extremes (candidate selection)
    int valid, pad;
};
static_assert(sizeof(RowStat) == 40, "RowStat layout");
// The same, compact (K3 proper): the exact fp64 extreme logits relative to the
// running max, as the reference forms them (logit - m_new, attention.cpp:183),
// and the fast-path extremes; pmin = INF marks a row without a tile this step.
struct RowStatC { // 24 bytes
    double dmin, dmax; // tmin - m, tmax - m
    float pmin, pmax;
};
static_assert(sizeof(RowStatC) == 24, "RowStatC layout");

constexpr double kLog2e = 1.4426950408889634;
// Band of the fast-path quotient q = (p - lo) / pscale (pgroup_consts below). The
// fp32 path forms the exp2 argument as (S - smax) * c + d with d = exact
// (tmax - m) * log2e, so the argument's error is <= 2^-23 |arg| at d=64 (both
// terms <= 0); ex2.approx.ftz.f32 is within 1.44e-7 relative over [-126, 0]
// (every input, scripts/ex2_err.cu); the reference rounds p to fp32 (2^-24).
// kappa / 2 = 3e-7 bounds each fast p's relative error for |arg| up to ~1
// (with the A / B rounding of the quantizer FMA) -- the regime of narrow tiles,
// where the error enters q absolutely, as (p + lo) / pscale; for the common
// tile (lo << p) the band is kappa * q, and there kappa is empirical: measured
// on c2/c3 (8M sampled elements each) kappa 0 leaves code flips (max|dO|/max|O|
// 5.8e-4 INT8, 6.4e-3 INT4), 4e-7 and 8e-7 are exact, and every full-shape
// P-code dump at c2-c5 and every adversarial tile family passes at 6e-7.
// A code is trusted only if both variants round to the same integer, else it
// is recomputed exactly in fp64.
#ifndef PARO_RED_MBAR
#define PARO_RED_MBAR 1
#endif
// d=64: p parked in TMEM across the P-group reduction (mbarrier, no bar.sync)
#ifndef PARO_P_STASH
#define PARO_P_STASH 0
#endif
#ifndef PARO_KAPPA
#define PARO_KAPPA 6e-7f
#endif
constexpr float kKappa = PARO_KAPPA;

// Fast-path quantizer constants of one P group (lo, hi: the group's fast extremes,
// inv = 1 / pscale). The code of t = (p - lo) / pscale is taken from the two variants
// t -/+ D, D = kp * (p + lo) / pscale + kq * (p - lo) / pscale:
//   kp = kappa / 2 bounds the relative error of each fast p (and of lo, hi) against
//      the reference's fp32(exp(fp64)) -- as an ABSOLUTE error in t it scales with
//      (p + lo) / pscale, which dominates on a narrow tile (hi - lo << lo: every p of the
//      tile close to lo, e.g. near-uniform attention) where a band relative to t alone
//      misses code flips (tests/test_gpu_pcode_adversarial.py "flat");
//   kq = kp * (hi + lo) / (hi - lo) is pscale's relative error from those of hi and lo
//      (capped at 1: a degenerate tile sends every code to the exact path).
// For lo << p (the common tile) D = kappa * t, the band of the relative-only rule.
// As FMAs: variant -/+ = p * A -/+ B with A = inv (1 -/+ (kq + kp)),
// B = 0.5 - lo * inv * (1 -/+ (kq - kp)); packed (low variant, high variant).
// FORM (measured, c2 / c3 / c5 K3): 3 at d=64 (kq from inv: 4.38 / 2.63 ms; with the
// __fdividef of form 1, 4.44 / 2.68), 1 at d=128 (110.6 ms; form 3 112.7)
#ifndef PARO_BAND_RIGOROUS
#define PARO_BAND_RIGOROUS 0
#endif
template <int FORM>
__device__ __forceinline__ void pgroup_consts(float lo, float hi, float inv, float qmax, uint64_t& A2, uint64_t& B2) {
#if PARO_BAND_RIGOROUS
    // every term bounded (d=64): a fast p = ex2.approx(arg) with |arg - exact| <= 2^-23 |arg|
    // is within (E + L * |arg|) p of the reference's fp32 p, E = 1.44e-7 (ex2.approx, every
    // input) + 2^-24 (the reference's rounding) + 6e-8 (the quantizer's A / B rounding),
    // L = ln2 * 2^-23. Elements that can sit on a code boundary have p >= pb = lo + pscale/2,
    // so |arg| <= -log2(pb) for them; lo's and hi's errors use their own |arg|.
    {
        constexpr float E = 2.64e-7f, L = 8.27e-8f;
        const float ps = fmaxf(hi - lo, 1e-30f) * (1.0f / qmax);
        const float a = E + L * (fmaxf(-__log2f(lo + 0.5f * ps), 0.f) + 0.02f);
        const float elo = (E + L * (fminf(-__log2f(fmaxf(lo, 1e-37f)), 160.f) + 0.02f)) * lo + 1.2e-38f;
        const float ehi = (E + L * (fmaxf(-__log2f(hi), 0.f) + 0.02f)) * hi;
        // pscale's relative error from hi's and lo's, + 9 roundings of ours and the reference's
        const float kq = hi > lo ? fminf(1.0f, (ehi + elo) * 1.01f * inv * (1.0f / qmax) + 5.4e-7f) : 1.0f;
        const float c = elo * inv + 2.4e-7f; // lo's absolute error and the final RD rounding, in q units
        const float kqp = kq + a;
        asm("mov.b64 %0, {%1, %2};" : "=l"(A2) : "f"(inv * (1.0f - kqp)), "f"(inv * (1.0f + kqp)));
        asm("mov.b64 %0, {%1, %2};" : "=l"(B2) : "f"(0.5f - lo * (inv * (1.0f - kq)) - c), "f"(0.5f - lo * (inv * (1.0f + kq)) + c));
        return;
    }
#endif
    const float kp = 0.5f * kKappa;
    // FORM 3: (hi + lo) / (hi - lo) = (hi + lo) * inv / qmax (inv = qmax / (hi - lo) up to
    // three roundings: 1.01 margin); a degenerate group (hi <= lo: pscale reset to 1)
    // sends every code to the exact path
    const float kq = FORM == 3 ? (hi > lo ? fminf(1.0f, (kp * 1.01f) * (hi + lo) * inv * (1.0f / qmax)) : 1.0f)
                               : fminf(1.0f, kp * __fdividef(hi + lo, fmaxf(hi - lo, 1e-30f)));
    if (FORM == 1) {
        const float li = lo * inv;
        asm("mov.b64 %0, {%1, %2};" : "=l"(A2) : "f"(inv * (1.0f - (kq + kp))), "f"(inv * (1.0f + (kq + kp))));
        asm("mov.b64 %0, {%1, %2};" : "=l"(B2) : "f"(0.5f - li * (1.0f - (kq - kp))), "f"(0.5f - li * (1.0f + (kq - kp))));
    } else {
        const float kqp = kq + kp, kqm = kq - kp;
        asm("mov.b64 %0, {%1, %2};" : "=l"(A2) : "f"(inv * (1.0f - kqp)), "f"(inv * (1.0f + kqp)));
        asm("mov.b64 %0, {%1, %2};" : "=l"(B2) : "f"(0.5f - lo * (inv * (1.0f - kqm))), "f"(0.5f - lo * (inv * (1.0f + kqm))));
    }
}

// int32 S of (row r, key j) recomputed from the smem Q/K tiles (64-byte rows, 64B swizzle)
__device__ __forceinline__ int32_t dot_row64(const uint8_t* qtile, const uint8_t* ktile, uint32_t r, uint32_t j) {
    const uint8_t* qr = qtile + (r >> 3) * 512 + (r & 7) * 64;
    const uint8_t* kr = ktile + (j >> 3) * 512 + (j & 7) * 64;
    int32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int4 a = *reinterpret_cast<const int4*>(qr + ((c ^ ((r >> 1) & 3)) << 4));
        const int4 b = *reinterpret_cast<const int4*>(kr + ((c ^ ((j >> 1) & 3)) << 4));
        acc = __dp4a(a.x, b.x, acc);
        acc = __dp4a(a.y, b.y, acc);
        acc = __dp4a(a.z, b.z, acc);
        acc = __dp4a(a.w, b.w, acc);
    }
    return acc;
}

// round-half-away of q >= 0 exactly as std::round (kernels_scalar.cpp:84)
__device__ __forceinline__ uint32_t round_half_away_pos(float q) {
    float t = truncf(q);
    if (__fsub_rn(q, t) >= 0.5f)
        t = __fadd_rn(t, 1.0f);
    return (uint32_t)t;
}

struct RowState {
    float m32, l;
    double m64;
};


} // namespace paro
