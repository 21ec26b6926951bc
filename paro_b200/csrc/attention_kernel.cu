// attention_kernel.cu -- K3: block-sparse INT8-QK / INT8|INT4-PV attention on
// sm_100a tensor cores (tcgen05.mma kind::i8, accumulators in TMEM), with the
// inverse PARO permutation fused into the output store.
//
// Semantics: the reference stream_engine (attention.cpp:84-254) with the
// restated INT8-QK prologue: per kept (q-block, k-block) tile
//   S_g  = int32 sum over column group g of q_code * k_code           (tcgen05)
//   s    = scale * sum_g sq[qb,g] * sk[bj,g] * S_g
//   m'   = max(m, max_j s); rescale l, acc by exp(m - m') when l > 0 (:169-179)
//   p    = exp(s - m');  l += sum p (unquantized, :181-189)
//   P    = one unsigned group over the tile's true rows x true columns:
//          lo/hi = min/max p, pscale = (hi-lo)/qmax (0 -> 1), codes
//          round-half-away((p - lo)/pscale) (:201-228)
//   ip   = int32 sum_j P_code * V_code                              (tcgen05)
//   acc += (pscale*vscale)*ip + (lo*vscale)*colsum                 (:229-238)
//   O    = acc / l, l == 0 -> zero row + flag (:242-251), stored at the
//          ORIGINAL token row (apply_perm_rows(out, plan.inverted()), main.cpp:304)
// Arithmetic is fp32 with ex2.approx (tolerance-gated);
// P codes follow the reference's fp32 quantizer exactly given p (round half
// away, fp32 (p - lo) then * 1/pscale).
//
// Work unit: two q-blocks A, B of one head (paired by K2 with similar kept
// counts), each running its OWN kept list through independent M = 64 MMAs:
// A's accumulators sit in TMEM lanes 0-15 of each 32-lane quadrant, B's in
// lanes 16-31 (the M=64 datapath layout at lane offset 0 / 16). Step t runs
// tile A.list[t] and tile B.list[t] side by side, so every softmax lane works
// on a kept tile (no union of mask rows) and the pair costs max(nA, nB) steps.
// Units are LPT-sorted by K2; each persistent CTA takes the next one from a
// global counter when its producer is ready (greedy LPT), and hands it to its
// other roles through a 2-slot mbarrier queue.
//
// Warp roles (320 threads; 2 CTAs/SM at d=64, 1 at d=128):
//   warp 0     TMA producer: Q tiles, per step the K/V tiles + meta of A and B
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5  softmax: TMEM S -> two passes (row extremes, then p / codes)
//              -> P codes (u8) into swizzled smem; per-tile column offsets
//   warps 6-9  epilogue: TMEM int32 PV -> dequant + rescale into fp32 registers,
//              final normalisation + inverse-permuted row store
// A thread of quadrant q (= warp % 4), lane i owns row 16q + (i & 15) of
// q-block (i < 16 ? A : B).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "k3_common.cuh"
#include "layer.cuh"
#include "ptx.cuh"

namespace paro {

// d=64 per-half (softmax) and per-chunk (epilogue) loops: unrolled (rolling them
// measured c2 4.39 -> 4.76 ms here; the decoupled kernel is the opposite case)
// PFULL: one arrival per compute THREAD (each releases its own smem writes -- the
// P codes, row meta and column offsets the MMA and the epilogue read) instead of
// __syncwarp + one lane
#ifndef PARO_PFULL_ALL
#define PARO_PFULL_ALL 1
#endif
#ifndef PARO_M128
#define PARO_M128 0
#endif
// exact path: the tile's exact P extremes from one fp64 exp each (monotone in the
// reduced argument) instead of exp over the candidate rows. 1: at d=128 only
// (measured c5 123.9 -> 120.4 ms; at d=64 the code change costs c2 3%), 2: both
// d=128 pass 1: re-test an unsure argmax / argmin gap with the row's own largest
// |S_g| before the fp64 rescan
#ifndef PARO_DQ_BATCH
#define PARO_DQ_BATCH 0  // 1: d=128 dequant issues every O chunk load before one wait (measured neutral)
#endif
#ifndef PARO_TIGHT_SLACK
#define PARO_TIGHT_SLACK 1
#endif
// the P-group extremes within a warp by redux.sync on the fp32 bit patterns. 1: at
// d=128 only (c5 111.8 -> 110.5 ms; at d=64 it costs c2 2%), 2: both
#ifndef PARO_REDUX
#define PARO_REDUX 1
#endif
#ifndef PARO_EXACT_MONO
#define PARO_EXACT_MONO 1
#endif
#ifndef PARO_I2F_FMA
// int32 -> fp32 conversions on the FMA pipe (IMAD + FADD2, k3_common.cuh i2f2_fma)
// instead of ALU I2F: bit 0 = the d=128 pass-1 scan, bit 1 = pass 2 at d=128,
// bit 2 = pass 2 at d=64, bit 3 = the d=64 epilogue's P.V dequant, bit 4 = the d=128
// dequant (|P.V| <= 64 * 255 * 127 < 2^22) (measured: bit 2 c2 K3 4.280 -> 4.213 ms; bits 0 / 1 cost
// d=128 3% / 5%, c5 109.8 -> 112.9 / 115.0 ms)
#define PARO_I2F_FMA 4
#endif
#ifndef PARO_PACK_IMAD
#define PARO_PACK_IMAD 0 // P-code word packing by IMAD (FMA pipe): bit 0 = the low variant, bit 1 = the stored high one
#endif
#ifndef PARO_ARG128_EXACT
// d=128 exactness against S-group cancellation (opt-in, DESIGN.md section 8 item 2):
// bit 1 = pass 2's exp2 argument (S0 - S0x) c0 + (S1 - S1x) c1 + dmax with c_g split in
// fp32 hi + lo parts and the two products summed with one rounding (arg128_2), so its
// error scales with the argument, not with the two terms; bit 0 = the row's fast min p
// from the exact fp64 (tmin - m). Both (3): the adversarial "cancel" family passes;
// c5 K3 +7% (bit 1) and +0.9% (bit 0). INT4 P passes the family without it (15 levels
// leave each code boundary far wider than the argument error), so by default (-1) only
// the d=128 INT8-P instantiation carries it
#define PARO_ARG128_EXACT -1 // -1: both bits for INT8 P at d=128 (c4 K3 +7%), off for INT4 P (c5)
#endif
#ifndef PARO_K3_W12
#define PARO_K3_W12 0
#endif
#ifndef PARO_K3_UNROLL
#define PARO_K3_UNROLL 4
#endif
constexpr int kK3Unroll = PARO_K3_UNROLL;

template <int D>
struct K3Cfg {
    static constexpr int G = D / 64;
    static constexpr int NS = 3;
    static constexpr int MINB = D == 64 ? 2 : 1; // CTAs per SM
    // SPLIT (d=128): 12 warps, warpgroup 0 = TMA producer, MMA issuer, 2 idle
    // (registers released with setmaxnreg), warpgroups 1-2 = 8 compute warps
    // (TMEM quadrant x key-column half), each doing softmax + dequant of its half.
    // !SPLIT (d=64): 10 warps, producer, MMA, 4 softmax, 4 epilogue (at d=64 the
    // split's two warps per quadrant contend for one SMSP in the synchronised
    // pass 2; measured 5.71 vs 4.86 ms at c2, while d=128 gains 188 -> 165 ms).
    static constexpr bool SPLIT = D == 128;
    // d=64 W12 (opt-in PARO_K3_W12): the same roles on 12 warps -- warpgroup 0 = producer,
    // MMA, 2 idle (setmaxnreg down), softmax on warps 4-7, epilogue on 8-11, so the
    // softmax and epilogue warpgroups get REG_COMPUTE registers instead of the 96 of
    // the 10-warp launch
    static constexpr bool W12 = D == 64 && PARO_K3_W12 && !PARO_M128;
    static constexpr int THREADS = (SPLIT || W12) ? 384 : 320;
    static constexpr uint32_t SM0 = W12 ? 4 : 2; // first softmax warp (d=64)
    static constexpr uint32_t NCW = SPLIT ? 8 : 4; // warps arriving on the S / P / O barriers
    static constexpr uint32_t REG_LAUNCH = (65536 / (THREADS * MINB)) / 8 * 8;
    static constexpr uint32_t REG_LOW = 32;
    static constexpr uint32_t REG_COMPUTE = ((REG_LAUNCH * THREADS - REG_LOW * 128) / 256) / 8 * 8;
    static constexpr uint32_t QT_BYTES = 64 * D; // one q-block tile
    static constexpr uint32_t KV_BYTES = 64 * D;
    static constexpr uint32_t META_BYTES = (4 + D) * 4; // multiple of 16
    static constexpr uint32_t STAGE_BYTES = (4 * KV_BYTES + 2 * META_BYTES + 1023) / 1024 * 1024;
    static constexpr uint32_t P_BYTES = 64 * 64; // one side's P tile
    static constexpr uint32_t S_COLS = G * 64;
    static constexpr uint32_t TM_S = 0;          // two S buffers
    static constexpr uint32_t TM_O = 2 * S_COLS; // two O buffers
    static constexpr uint32_t TMEM_COLS = (2 * S_COLS + 2 * D) <= 256 ? 256 : 512;
    // d=64 (M128, opt-in: measured c2 4.74 vs 4.28 ms, c3 2.71 vs 2.53): QK is one M = 128 MMA per side with a zero-padded Q operand --
    // [Q_A; 0] and [0; Q_B] accumulated into the same 64 TMEM columns -- so q-block A
    // lands in TMEM lanes 0-63 (quadrants 0-1) and B in lanes 64-127 (quadrants 2-3):
    // a tile's 64 rows span two softmax warps instead of four, and its P-group
    // hand-off is a 64-thread barrier of that pair. An item buffer holds Q_A, a zero
    // tile and Q_B contiguously (the 128-row operands overlap on the zero tile).
    static constexpr bool M128 = D == 64 && PARO_M128;
    // M128 layout of one item buffer, in 32-row (2 KB) slots: [A0 | 0 | A1 | 0 | B0 | 0 | B1]
    // (X0 / X1 = rows 0-31 / 32-63). Side A's operand [A0; 0; A1; 0] starts at slot 0 and
    // puts its rows in TMEM quadrants 0 and 2; side B's [0; B0; 0; B1] starts at slot 3,
    // quadrants 1 and 3 -- each q-block's pair of warps on sub-partitions {0, 2} or {1, 3}.
    static constexpr uint32_t HALF = QT_BYTES / 2;
    static constexpr uint32_t QBUF = M128 ? 7 * HALF : 2 * QT_BYTES; // one item's Q tiles
    static constexpr uint32_t QB_OFF = M128 ? 4 * HALF : QT_BYTES;   // side B's rows 0-31 in it
    static constexpr uint32_t QOP_B = M128 ? 3 * HALF : QT_BYTES;    // side B's MMA operand
    static constexpr uint32_t OFF_Q = 0; // [2 item buffers][A, B] q-block tiles
    static constexpr uint32_t OFF_STAGE = 2 * QBUF;
    // within a stage: K_A, K_B, V_A, V_B, meta_A, meta_B
    static constexpr uint32_t OFF_P = OFF_STAGE + NS * STAGE_BYTES; // [2 buf][2 side]
    static constexpr uint32_t OFF_ROWMETA = OFF_P + 4 * P_BYTES;     // [2 buf][2 side][64] float4
    static constexpr uint32_t OFF_U = OFF_ROWMETA + 2 * 2 * 64 * 16;  // [2 buf][2 side][D]
    static constexpr uint32_t OFF_RED = OFF_U + 2 * 2 * D * 4;        // [2 parity][4 quad][2 side] float2
    static constexpr uint32_t OFF_L = OFF_RED + 2 * 4 * 2 * 8;        // [2 item][2 half][2 side][64] partial row sums
    static constexpr uint32_t OFF_ROWSTAT = OFF_L + 2 * 2 * 2 * 64 * 4;       // [2 parity][2 side][64] RowStatC (24 B)
    static constexpr uint32_t OFF_XCH = OFF_ROWSTAT + 2 * 2 * 64 * 24; // SPLIT d=128: [2 half][2 side][64] float4
    static constexpr uint32_t OFF_XLIST = OFF_XCH + (SPLIT ? 2 * 2 * 64 * (16 + 16) : 0); // + int4 S pairs
    // exact path: per compute warp, its risky (owner lane, group) list (<= 32 x 16 entries)
    // INT4 V arrives nibble-packed (D/2 bytes per key row); d = 64 unpacks it in place
    // (the packed tile lands in the upper half of its V tile), d = 128 from this staging
    static constexpr uint32_t VPK_BYTES = 64 * D / 2;
    static constexpr uint32_t OFF_VPK = OFF_XLIST + NCW * 512 * 2; // d = 128: [NS][2 side] packed V tiles
    static constexpr uint32_t OFF_BAR = OFF_VPK + (SPLIT ? NS * 2 * VPK_BYTES : 0);
    static constexpr uint32_t NBAR = 2 + 3 * NS + 21; // == Bars<NS>::COUNT (static_assert below)
    // warps reading the item queue: MMA + 8 (softmax + epilogue | compute) + at d = 128
    // the two warpgroup-0 warps that unpack INT4 V (one side each)
    static constexpr uint32_t NCONS = SPLIT ? 11 : 9;
    static constexpr uint32_t NVFULL = SPLIT ? 2 : 1; // arrivals per VFULL phase
    static constexpr uint32_t OFF_TMEMPTR = OFF_BAR + NBAR * 8;
    static constexpr uint32_t SMEM_BYTES = OFF_TMEMPTR + 16;
    // swizzle: rows of D int8 -> 64B (D=64) or 128B (D=128) swizzle atoms of 8 rows
    static constexpr uint32_t LAYOUT = D == 64 ? ptx::kSwizzle64B : ptx::kSwizzle128B;
    static constexpr uint32_t ATOM = 8 * D; // bytes per 8-row swizzle atom
    static constexpr uint32_t IDESC_QK = ptx::idesc_i8(true, true, false, false, 64, 64);
    static constexpr uint32_t IDESC_QK128 = ptx::idesc_i8(true, true, false, false, 128, 64);
    static constexpr uint32_t IDESC_PV = ptx::idesc_i8(false, true, false, true, 64, D);
    static constexpr uint32_t LANE16 = 16u << 16; // TMEM address of lane 16 (side B)
};

enum : uint32_t { B_QFULL = 0, B_QEMPTY = 1 };
template <int NS>
struct Bars {
    static constexpr uint32_t KVFULL = 2, KVEMPTY = 2 + NS, SFULL = 2 + 2 * NS, SEMPTY = SFULL + 2,
                              PFULL = SEMPTY + 2, PEMPTY = PFULL + 2, OFULL = PEMPTY + 2, OEMPTY = OFULL + 2,
                              LFULL = OEMPTY + 2, LEMPTY = LFULL + 1, RED = LEMPTY + 1,
                              QFULL1 = RED + 1, QEMPTY1 = RED + 2, ITEMFULL = QEMPTY1 + 1, ITEMEMPTY = ITEMFULL + 2,
                              VFULL = ITEMEMPTY + 2, // packed INT4 V of a stage unpacked (producer)
                              COUNT = VFULL + NS;
};
static_assert(Bars<K3Cfg<64>::NS>::COUNT == K3Cfg<64>::NBAR && Bars<K3Cfg<128>::NS>::COUNT == K3Cfg<128>::NBAR,
              "mbarrier block must hold every barrier (the TMEM pointer slot follows it)");

// K-major operand rows of D bytes (Q, K): SBO = one 8-row atom.
template <int D>
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
    return ptx::smem_desc(saddr, 16, K3Cfg<D>::ATOM, K3Cfg<D>::LAYOUT);
}
// P: 64 rows x 64 u8 (K = keys), K-major, 64B swizzle.
__device__ __forceinline__ uint64_t desc_p(uint32_t saddr) { return ptx::smem_desc(saddr, 16, 512, ptx::kSwizzle64B); }
// V: [key][D] row-major = MN-major B operand (N = D contiguous); SBO = 8 keys.
template <int D>
__device__ __forceinline__ uint64_t desc_v(uint32_t saddr) {
    return ptx::smem_desc(saddr, K3Cfg<D>::ATOM * 8, K3Cfg<D>::ATOM, K3Cfg<D>::LAYOUT);
}

// QK issue for one q-block tile (M = 64): S_g in TMEM columns tm_s + 64*g at the
// tile's lane offset; two K=32 steps per 64-column group.
template <int D>
__device__ __forceinline__ void issue_qk(uint32_t tmem, uint32_t sq, uint32_t sk) {
    using C = K3Cfg<D>;
#pragma unroll
    for (int g = 0; g < C::G; ++g)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const uint32_t koff = g * 64 + kk * 32;
            ptx::mma_i8(tmem + g * 64, desc_kmajor<D>(sq + koff), desc_kmajor<D>(sk + koff), C::IDESC_QK, kk);
        }
}

// M128 (d=64): one side's QK as an M = 128 MMA whose A operand interleaves the
// q-block's two 32-row halves with zero slots (K3Cfg::QBUF); the first MMA of the
// step overwrites the buffer, the other accumulates its rows onto the first's zeros
__device__ __forceinline__ void issue_qk128(uint32_t tmem, uint32_t sa, uint32_t sk, bool first) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
        ptx::mma_i8(tmem, desc_kmajor<64>(sa + kk * 32), desc_kmajor<64>(sk + kk * 32), K3Cfg<64>::IDESC_QK128,
                    (first && kk == 0) ? 0u : 1u);
}

// ---------------------------------------------------------------------------
// Softmax, one step for this thread's row. Pass 1 reads S for the row extremes
// (exact in the integer domain at d=64); the tile group's lo/hi then come from
// two exp2 per row (p at the extreme columns, computed with the same formula
// the elements use, so they are the true min/max of the p values); pass 2
// re-reads S and produces p, the row sum and the P codes. Lanes whose q-block
// has no tile this step (`live` false) run the same instructions but change
// no state and contribute neutral extremes.
// ---------------------------------------------------------------------------

// d=128: the two int32 group sums S_0, S_1 of (row r, key j) from the smem Q/K
// tiles (128-byte rows, 128B swizzle: 16-B chunk c of row r at c ^ (r & 7))
__device__ __forceinline__ void dot_row128(const uint8_t* qtile, const uint8_t* ktile, uint32_t r, uint32_t j,
                                           int32_t& s0, int32_t& s1) {
    const uint8_t* qr = qtile + (r >> 3) * 1024 + (r & 7) * 128;
    const uint8_t* kr = ktile + (j >> 3) * 1024 + (j & 7) * 128;
    int32_t acc[2] = {0, 0};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int4 a = *reinterpret_cast<const int4*>(qr + ((c ^ (r & 7)) << 4));
        const int4 b = *reinterpret_cast<const int4*>(kr + ((c ^ (j & 7)) << 4));
        int32_t& t = acc[c >> 2];
        t = __dp4a(a.x, b.x, t);
        t = __dp4a(a.y, b.y, t);
        t = __dp4a(a.z, b.z, t);
        t = __dp4a(a.w, b.w, t);
    }
    s0 = acc[0];
    s1 = acc[1];
}

// both (S_0, S_1) pairs of columns ja and jb of row r in one pass (shared Q-row loads)
__device__ __forceinline__ void dot2_row128(const uint8_t* qtile, const uint8_t* ktile, uint32_t r, uint32_t ja,
                                            uint32_t jb, int32_t& a0, int32_t& a1, int32_t& b0, int32_t& b1) {
    const uint8_t* qr = qtile + (r >> 3) * 1024 + (r & 7) * 128;
    const uint8_t* ka = ktile + (ja >> 3) * 1024 + (ja & 7) * 128;
    const uint8_t* kb = ktile + (jb >> 3) * 1024 + (jb & 7) * 128;
    int32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int4 q = *reinterpret_cast<const int4*>(qr + ((c ^ (r & 7)) << 4));
        const int4 x = *reinterpret_cast<const int4*>(ka + ((c ^ (ja & 7)) << 4));
        const int4 y = *reinterpret_cast<const int4*>(kb + ((c ^ (jb & 7)) << 4));
        int32_t& t = acc[c >> 2];
        int32_t& u = acc[2 + (c >> 2)];
        t = __dp4a(q.x, x.x, t);
        u = __dp4a(q.x, y.x, u);
        t = __dp4a(q.y, x.y, t);
        u = __dp4a(q.y, y.y, u);
        t = __dp4a(q.z, x.z, t);
        u = __dp4a(q.z, y.z, u);
        t = __dp4a(q.w, x.w, t);
        u = __dp4a(q.w, y.w, u);
    }
    a0 = acc[0];
    a1 = acc[1];
    b0 = acc[2];
    b1 = acc[3];
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// d=128 logit in the reference's fp64 order (paro_oracle.c qk_mode 1, attention.cpp:166):
// scale * ((a0 * S_0) + (a1 * S_1)), a_g = sq_g * sk_g exact in fp64
__device__ __forceinline__ double logit128(double scale64, double a0, double a1, int32_t s0, int32_t s1) {
    return __dmul_rn(scale64, __dadd_rn(__dmul_rn(a0, (double)s0), __dmul_rn(a1, (double)s1)));
}

// x[j] for a per-lane index j < 32 without local memory: a 5-level select tree
__device__ __forceinline__ uint32_t sel32(const uint32_t (&x)[32], uint32_t j) {
    uint32_t a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
        a[i] = (j & 16u) ? x[i + 16] : x[i];
#pragma unroll
    for (int w = 8; w > 0; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i)
            a[i] = (j & (uint32_t)w) ? a[i + w] : a[i];
    return a[0];
}

// column-tagged fp32 logit: the low 6 mantissa bits carry the column, so a max /
// min over keys also names its column (perturbation < 64 ulp, covered by kGapSlack)
__device__ __forceinline__ float tagf(float y, uint32_t j) {
    return __uint_as_float((__float_as_uint(y) & ~63u) | j);
}
// |fp32 logit (log2 units) - exact| <= kErrS * (c0 + c1) * kSBound (+ tag slack): a
// top-2 / bottom-2 gap below that bound falls back to an exact rescan
constexpr float kSBound = 64.f * 127.f * 127.f; // |S_g| <= 64 * 127^2
constexpr float kErrS = 5e-7f, kGapSlack = 2e-5f;

// ---------------------------------------------------------------------------
// Softmax, one step for this thread's row (v3 order: pass 1 extremes -> group
// reduction -> pass 2 p / codes).
//   d=64 (G=1): the row extremes are integer maxima of S, so the reference's
//   exact fp64 logits of the extremes and the exact running max m64 are known
//   every step. d=128 (G=2): the logit is c0 * S_0 + c1 * S_1, so the extremes
//   come from a column-tagged fp32 scan (top-2 / bottom-2 per row), their fp64
//   logits from the selected columns' (S_0, S_1), and a near tie within the
//   fp32 error bound sends the row to an exact fp64 rescan of its candidates.
//   Both: P codes are made BIT-EXACT with the reference's fp32 quantizer of
//   the fp64 p: the fast path computes each code twice from (1 -/+ kappa)-
//   perturbed quotients (one packed FFMA2.RM per element); where the two
//   differ (~1e-4 of elements) the code is recomputed in fp64 from the exact
//   tile lo/hi (from every row's published extremes) and S re-derived with
//   dp4a from the Q/K tiles still in smem.
// Lanes whose q-block has no tile this step (`live` false) run the same
// instructions but change no state and contribute neutral extremes.
// ---------------------------------------------------------------------------
#ifdef PARO_K3_PROF
// [0..1][4]: the four softmax warps' barrier arrivals, [2..3][4]: their step starts (by step parity)
__device__ __forceinline__ long long (*prof_smem())[4] {
    __shared__ long long a[4][4];
    return a;
}
#endif
template <int D, bool SPLIT, bool P4 = false>
__device__ __forceinline__ void softmax_step(uint32_t s_addr, float sq, float sk0, float sk1, double scale64,
                                             float scale_log2, uint32_t ncol, bool live, bool valid_row,
                                             RowState& st, float p_qmax, float2* red_w, const float2* red_r,
                                             RowStatC* rs_w, const RowStatC* rs_r, uint32_t side,
                                             const uint8_t* qtile, const uint8_t* ktile, uint8_t* prow, uint32_t r,
                                             float sq1, float& gamma_out, float& lo_out, float& pscale_out,
                                             uint32_t half, float4* xch, uint16_t* xlist, uint32_t red_bar,
                                             uint32_t red_par, unsigned long long (&prof)[18], uint32_t one) {
    PROF_T(tp0);
    constexpr int G = D / 64;
    // M128 (d=64): all 32 lanes of this warp hold rows of ONE q-block (side), whose
    // other 32 rows sit in the partner warp of the same side
    constexpr bool M128 = !SPLIT && K3Cfg<D>::M128;
    const uint32_t lane = threadIdx.x & 31;
    // M128: this warp's side as a vote result, so the compiler sees it warp-uniform (a
    // branch on a threadIdx-derived value makes it wrap every later shuffle in
    // divergence handling: +13% code and instruction-fetch stalls)
    const uint32_t wside = M128 ? (__ballot_sync(0xffffffffu, side != 0) ? 1u : 0u) : side;
    const bool valid = live && valid_row;
    // -------- pass 1: row extremes (4 independent chains)
    float m32, pmax_r, pmin_r, c0, c1 = 0.f, dmax = 0.f;
    constexpr int kArg = G == 2 ? (PARO_ARG128_EXACT >= 0 ? PARO_ARG128_EXACT : (P4 ? 0 : 3)) : 0;
    float c0lo = 0.f, c1lo = 0.f; // d=128 (kArg): c_g - fp32(c_g)
    int32_t smax_i = 0, smax1_i = 0; // d=64: row max of S; d=128: (S_0, S_1) of the row's argmax column
    double a64 = 0.0, a64b = 0.0, m64 = st.m64;
    if (G == 1) {
        int32_t mx[4] = {INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN},
                mn[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
#pragma unroll kK3Unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t x[32];
            ptx::tmem_ld32(s_addr + h2 * 32, x);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) { // padded key columns repeat column 0 (K1): no masking
                mx[j & 3] = max(mx[j & 3], (int32_t)x[j]);
                mn[j & 3] = min(mn[j & 3], (int32_t)x[j]);
            }
        }
        const int32_t smax = max(max(mx[0], mx[1]), max(mx[2], mx[3]));
        const int32_t smin = min(min(mn[0], mn[1]), min(mn[2], mn[3]));
        // reference order: logit = scale * ((sq * sk) * S) in fp64 (paro_oracle.c, attention.cpp:166)
        a64 = __dmul_rn((double)sq, (double)sk0);
        const double tmax64 = __dmul_rn(scale64, __dmul_rn(a64, (double)smax));
        const double tmin64 = __dmul_rn(scale64, __dmul_rn(a64, (double)smin));
        if (live)
            m64 = fmax(st.m64, tmax64);
        c0 = (float)(__dmul_rn(__dmul_rn(scale64, a64), kLog2e));
        m32 = (float)(m64 * kLog2e);
        // exp2 argument of element j = (S_j - smax) * c0 + dmax: exact integer
        // difference, dmax = (tmax - m) * log2e from the fp64 logits
        dmax = (float)((tmax64 - m64) * kLog2e);
        smax_i = smax;
        pmax_r = ex2(dmax);
        pmin_r = ex2(fmaf(__int2float_rn(smin - smax), c0, dmax));
        if (!SPLIT || half == 0)
            *rs_w = RowStatC{tmin64 - m64, tmax64 - m64, valid ? pmin_r : INFINITY, valid ? pmax_r : 0.f};
    } else {
        // d=128: the argmax / argmin columns from column-tagged fp32 logits (two
        // chains of top-2 / bottom-2), their exact fp64 logits from dp4a over the
        // Q/K tiles, and an exact warp-uniform rescan of the near candidates when a
        // top-2 / bottom-2 gap is within the fp32 error bound (rare)
        a64 = __dmul_rn((double)sq, (double)sk0);
        a64b = __dmul_rn((double)sq1, (double)sk1);
        {
            const double c0d = __dmul_rn(__dmul_rn(scale64, a64), kLog2e), c1d = __dmul_rn(__dmul_rn(scale64, a64b), kLog2e);
            c0 = (float)c0d;
            c1 = (float)c1d;
            if (kArg & 2) {
                c0lo = (float)(c0d - (double)c0);
                c1lo = (float)(c1d - (double)c1);
            }
        }
        // 4 chains (pair k -> chain k & 3) for latency; top-2 / bottom-2 merges with
        // 3-input min / max: M2' = max(M2, min(M1, hi), lo), M1' = max(M1, hi)
        float M1[4], M2[4], N1[4], N2[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            M1[c] = M2[c] = -INFINITY;
            N1[c] = N2[c] = INFINITY;
        }
        // SPLIT: each warp of the quadrant pair scans its 32 key columns; the pair
        // then exchanges its top-2 / bottom-2 through smem (one 64-thread barrier)
        int32_t ls0x = 0, ls1x = 0, ls0n = 0, ls1n = 0; // SPLIT: (S_0, S_1) of this half's argmax / argmin
#pragma unroll
        for (int hh = 0; hh < (SPLIT ? 1 : 2); ++hh) {
            const int h2 = SPLIT ? (int)half : hh;
            uint32_t x0[32], x1[32];
            ptx::tmem_ld32(s_addr + h2 * 32, x0);
            ptx::tmem_ld32(s_addr + 64 + h2 * 32, x1);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint32_t ja = h2 * 32 + 2 * k, jb = ja + 1;
                // y = fma(S_1, c1, S_0 * c0) per column, two columns per packed FMUL2 / FFMA2
                const uint64_t f1 = (PARO_I2F_FMA & 1) ? i2f2_fma((int32_t)x1[2 * k], (int32_t)x1[2 * k + 1], one)
                                                       : pk(__int2float_rn((int32_t)x1[2 * k]), __int2float_rn((int32_t)x1[2 * k + 1]));
                const uint64_t f0 = (PARO_I2F_FMA & 1) ? i2f2_fma((int32_t)x0[2 * k], (int32_t)x0[2 * k + 1], one)
                                                       : pk(__int2float_rn((int32_t)x0[2 * k]), __int2float_rn((int32_t)x0[2 * k + 1]));
                const uint64_t y2 = fma2(f1, pk(c1, c1), mul2(f0, pk(c0, c0)));
                float ya, yb;
                upk(y2, ya, yb);
                const float ka = tagf(ya, ja), kb = tagf(yb, jb);
                const float hi = fmaxf(ka, kb), lo = fminf(ka, kb);
                const int c = k & 3;
                M2[c] = fmax3(M2[c], fminf(M1[c], hi), lo);
                M1[c] = fmaxf(M1[c], hi);
                N2[c] = fmin3(N2[c], fmaxf(N1[c], lo), hi);
                N1[c] = fminf(N1[c], lo);
            }
            if (SPLIT) { // the integer S of this half's argmax / argmin, still in registers
                const float lmx = fmaxf(fmaxf(M1[0], M1[1]), fmaxf(M1[2], M1[3]));
                const float lmn = fminf(fminf(N1[0], N1[1]), fminf(N1[2], N1[3]));
                const uint32_t jx = __float_as_uint(lmx) & 31u, jn = __float_as_uint(lmn) & 31u;
                ls0x = (int32_t)sel32(x0, jx);
                ls1x = (int32_t)sel32(x1, jx);
                ls0n = (int32_t)sel32(x0, jn);
                ls1n = (int32_t)sel32(x1, jn);
            }
        }
        // merge chains pairwise (same top-2 rule)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            M2[c] = fmax3(fmaxf(M2[c], M2[c + 2]), fminf(M1[c], M1[c + 2]), -INFINITY);
            M1[c] = fmaxf(M1[c], M1[c + 2]);
            N2[c] = fmin3(fminf(N2[c], N2[c + 2]), fmaxf(N1[c], N1[c + 2]), INFINITY);
            N1[c] = fminf(N1[c], N1[c + 2]);
        }
        float mA = fmaxf(M1[0], M1[1]), mB = fmax3(fminf(M1[0], M1[1]), M2[0], M2[1]);
        float nA = fminf(N1[0], N1[1]), nB = fmin3(fmaxf(N1[0], N1[1]), N2[0], N2[1]);
        PROF_T(tq0);
        int32_t s0x, s1x, s0n, s1n;
        if (SPLIT) { // one exchange: top-2 / bottom-2 and the S pairs of each half's extremes
            int4* xs = reinterpret_cast<int4*>(xch + 2 * 2 * 64);
            xch[(half * 2 + side) * 64 + r] = make_float4(mA, mB, nA, nB);
            xs[(half * 2 + side) * 64 + r] = make_int4(ls0x, ls1x, ls0n, ls1n);
            ptx::named_bar_sync(2 + r / 16, 64); // the quadrant's two warps
            const float4 o = xch[((half ^ 1) * 2 + side) * 64 + r];
            const int4 os = xs[((half ^ 1) * 2 + side) * 64 + r];
            // merge in half order so both warps get bit-identical results (tags
            // name distinct columns, so the extremes never tie across halves)
            const float4 a = half ? o : make_float4(mA, mB, nA, nB), b = half ? make_float4(mA, mB, nA, nB) : o;
            const int4 sa = half ? os : make_int4(ls0x, ls1x, ls0n, ls1n),
                       sb = half ? make_int4(ls0x, ls1x, ls0n, ls1n) : os;
            mA = fmaxf(a.x, b.x);
            mB = fmax3(fminf(a.x, b.x), a.y, b.y);
            nA = fminf(a.z, b.z);
            nB = fmin3(fmaxf(a.z, b.z), a.w, b.w);
            const bool xa = a.x >= b.x, na = a.z <= b.z;
            s0x = xa ? sa.x : sb.x;
            s1x = xa ? sa.y : sb.y;
            s0n = na ? sa.z : sb.z;
            s1n = na ? sa.w : sb.w;
        }
        PROF_T(tq1);
        const float slack = kErrS * (c0 + c1) * kSBound + kGapSlack * fmaxf(fabsf(mA), fabsf(nA));
        const bool unsure = !(mA - mB > slack) || !(nB - nA > slack);
        if (!SPLIT) {
            dot2_row128(qtile, ktile, r, __float_as_uint(mA) & 63u, __float_as_uint(nA) & 63u, s0x, s1x, s0n, s1n);
        }
        double tmax64 = logit128(scale64, a64, a64b, s0x, s1x);
        double tmin64 = logit128(scale64, a64, a64b, s0n, s1n);
#ifdef PARO_K3_PROF
        asm volatile("" ::"d"(tmax64 + tmin64));
#endif
        PROF_T(tq2);
        bool unsure_t = unsure;
        float slack_t = slack;
        if (PARO_TIGHT_SLACK && __any_sync(0xffffffffu, unsure && valid)) {
            // the bound above assumes |S_g| = 64 * 127^2; the row's own largest |S_g|
            // (both key halves) usually settles the gap test without the fp64 rescan
            int32_t M0 = 0, M1 = 0;
#pragma unroll 1
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t x0[32], x1[32];
                ptx::tmem_ld32(s_addr + h2 * 32, x0);
                ptx::tmem_ld32(s_addr + 64 + h2 * 32, x1);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    M0 = max(M0, abs((int32_t)x0[j]));
                    M1 = max(M1, abs((int32_t)x1[j]));
                }
            }
            slack_t = kErrS * (c0 * (float)M0 + c1 * (float)M1) + kGapSlack * fmaxf(fabsf(mA), fabsf(nA));
            unsure_t = unsure && (!(mA - mB > slack_t) || !(nB - nA > slack_t));
#ifdef PARO_K3_PROF
            if (lane == 0) {
                atomicAdd(&g_profq[0], 1ull);
                if (__any_sync(0xffffffffu, unsure_t && valid))
                    atomicAdd(&g_profq[1], 1ull);
            } else {
                (void)__any_sync(0xffffffffu, unsure_t && valid);
            }
#endif
        }
        if (__any_sync(0xffffffffu, unsure_t && valid)) {
            const float thr_hi = mA - slack_t, thr_lo = nA + slack_t;
#pragma unroll 1
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t x0[32], x1[32];
                ptx::tmem_ld32(s_addr + h2 * 32, x0);
                ptx::tmem_ld32(s_addr + 64 + h2 * 32, x1);
                ptx::tmem_ld_wait();
                // the half's candidate columns as a bitmask (branch-free), then each lane
                // walks its own few candidates in ascending order (the same order and
                // tie-breaking as a column loop, without 32 warp-divergent fp64 branches)
                uint32_t cm = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float y =
                        fmaf(__int2float_rn((int32_t)x1[j]), c1, __int2float_rn((int32_t)x0[j]) * c0);
                    const bool cand = unsure_t && (uint32_t)(h2 * 32 + j) < ncol && (y >= thr_hi || y <= thr_lo);
                    cm |= (cand ? 1u : 0u) << j;
                }
                while (cm) {
                    const uint32_t j = __ffs(cm) - 1;
                    cm &= cm - 1;
                    const int32_t a = (int32_t)sel32(x0, j), b = (int32_t)sel32(x1, j);
                    const double L = logit128(scale64, a64, a64b, a, b);
                    if (L > tmax64) {
                        tmax64 = L;
                        s0x = a;
                        s1x = b;
                    }
                    if (L < tmin64) {
                        tmin64 = L;
                        s0n = a;
                        s1n = b;
                    }
                }
            }
        }
        PROF_T(tq3);
        if (live)
            m64 = fmax(st.m64, tmax64);
        m32 = (float)(m64 * kLog2e);
        dmax = (float)((tmax64 - m64) * kLog2e);
        smax_i = s0x;
        smax1_i = s1x;
        // exp2 argument of element j = (S0_j - S0x) * c0 + (S1_j - S1x) * c1 + dmax
        pmax_r = ex2(dmax);
        pmin_r = (kArg & 1) ? ex2((float)((tmin64 - m64) * kLog2e)) // no S-group cancellation
                                   : ex2(fmaf(__int2float_rn(s1n - s1x), c1, fmaf(__int2float_rn(s0n - s0x), c0, dmax)));
        if (!SPLIT || half == 0)
            *rs_w = RowStatC{tmin64 - m64, tmax64 - m64, valid ? pmin_r : INFINITY, valid ? pmax_r : 0.f};
        PROF_T(tq4);
        PROF_ADD(8, tq0 - tp0);
        PROF_ADD(9, tq1 - tq0);
        PROF_ADD(10, tq2 - tq1);
        PROF_ADD(11, tq3 - tq2);
        PROF_ADD(12, tq4 - tq3);
        if (__any_sync(0xffffffffu, unsure && valid))
            PROF_ADD(13, 1);
    }
    // rescale when an earlier tile of the item was live (the reference's l > 0,
    // attention.cpp:170): both column halves agree on it
    const float gamma = st.m32 != -INFINITY ? ex2(st.m32 - m32) : 1.0f;
    PROF_T(tp1);
    PROF_ADD(1, tp1 - tp0);
    if (!valid) {
        pmin_r = INFINITY;
        pmax_r = 0.f;
    }
    // -------- P group extremes over the q-block's 64 rows: 16 lanes x 4 warps
    // (M128: 32 lanes x 2 warps)
    if (PARO_REDUX == 2 || (PARO_REDUX == 1 && (G == 2 || P4))) {
        // p >= 0 (INF marks an idle row), so the fp32 bit patterns order like the values:
        // one redux.sync per side and extreme instead of a 4-level shuffle chain
        const uint32_t bmin = __float_as_uint(pmin_r), bmax = __float_as_uint(pmax_r);
        if (M128) {
            pmin_r = __uint_as_float(__reduce_min_sync(0xffffffffu, bmin));
            pmax_r = __uint_as_float(__reduce_max_sync(0xffffffffu, bmax));
        } else {
            const bool sb = lane >= 16;
            const uint32_t mnA = __reduce_min_sync(0xffffffffu, sb ? 0xffffffffu : bmin);
            const uint32_t mnB = __reduce_min_sync(0xffffffffu, sb ? bmin : 0xffffffffu);
            const uint32_t mxA = __reduce_max_sync(0xffffffffu, sb ? 0u : bmax);
            const uint32_t mxB = __reduce_max_sync(0xffffffffu, sb ? bmax : 0u);
            pmin_r = __uint_as_float(sb ? mnB : mnA);
            pmax_r = __uint_as_float(sb ? mxB : mxA);
        }
    } else {
#pragma unroll
        for (int o = M128 ? 16 : 8; o > 0; o >>= 1) {
            pmin_r = fminf(pmin_r, __shfl_xor_sync(0xffffffffu, pmin_r, o));
            pmax_r = fmaxf(pmax_r, __shfl_xor_sync(0xffffffffu, pmax_r, o));
        }
    }
    if ((!SPLIT || half == 0) && (M128 ? lane == 0 : (lane & 15) == 0))
        *red_w = make_float2(pmin_r, pmax_r);
    // -------- pass 2: p, row sum, codes (two perturbed variants per element)
    const uint64_t c00 = pk(c0, c0), c11 = pk(c1, c1), nm = pk(dmax, dmax);
    const uint64_t c0lo2 = pk(c0lo, c0lo), c1lo2 = pk(c1lo, c1lo);
    uint64_t sum2 = pk(0.f, 0.f);
    const bool tail_any = __any_sync(0xffffffffu, ncol < 64u);
    auto compute_p = [&](int h2, float (&pv)[32], bool mask_tail) { // p of the row's 32 columns of half h2, + row sum
        if (G == 1) {
            uint32_t x[32];
            ptx::tmem_ld32(s_addr + h2 * 32, x);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint64_t y2 =
                    fma2((PARO_I2F_FMA & 4) ? i2f2_fma_b((int32_t)x[2 * k], (int32_t)x[2 * k + 1], one, 0x4B400000u - (uint32_t)smax_i)
                                            : pk(__int2float_rn((int32_t)x[2 * k] - smax_i), __int2float_rn((int32_t)x[2 * k + 1] - smax_i)),
                         c00, nm);
                float ya, yb;
                upk(y2, ya, yb);
                pv[2 * k] = ex2(ya);
                pv[2 * k + 1] = ex2(yb);
            }
        } else {
            uint32_t x0[32], x1[32];
            ptx::tmem_ld32(s_addr + h2 * 32, x0);
            ptx::tmem_ld32(s_addr + 64 + h2 * 32, x1);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint64_t d0 = (PARO_I2F_FMA & 2) ? i2f2_fma_b((int32_t)x0[2 * k], (int32_t)x0[2 * k + 1], one, 0x4B400000u - (uint32_t)smax_i)
                                                       : pk(__int2float_rn((int32_t)x0[2 * k] - smax_i),
                                                            __int2float_rn((int32_t)x0[2 * k + 1] - smax_i));
                const uint64_t d1 = (PARO_I2F_FMA & 2) ? i2f2_fma_b((int32_t)x1[2 * k], (int32_t)x1[2 * k + 1], one, 0x4B400000u - (uint32_t)smax1_i)
                                                       : pk(__int2float_rn((int32_t)x1[2 * k] - smax1_i),
                                                            __int2float_rn((int32_t)x1[2 * k + 1] - smax1_i));
                const uint64_t y2 = (kArg & 2) ? arg128_2(d0, d1, c00, c11, c0lo2, c1lo2, nm)
                                                      : fma2(d1, c11, fma2(d0, c00, nm));
                float ya, yb;
                upk(y2, ya, yb);
                pv[2 * k] = ex2(ya);
                pv[2 * k + 1] = ex2(yb);
            }
        }
        if (mask_tail && tail_any) { // tail tile: the padded key columns (copies of column 0) leave the row sum
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if ((uint32_t)(h2 * 32 + j) >= ncol)
                    pv[j] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            sum2 = add2(sum2, pk(pv[2 * k], pv[2 * k + 1]));
    };
    // SPLIT (d=128): publish this warp's extremes and keep going -- the p values
    // of the warp's column half need only the row's own max, so they overlap the
    // wait for the other compute warps (an mbarrier, so arriving never blocks;
    // c5 132.7 -> 129.0 ms). At d=64 holding 32 p values across the wait spills
    // (96 registers) and measured slower, so it keeps bar.sync.
    // (Measured at d=64 with 12 warps and setmaxnreg giving the softmax 120 registers
    // for the row's 64 p values: 5.32 vs 4.52 ms at c2, branch k3-multislot-experiment.)
    constexpr bool kOverlap = SPLIT && PARO_RED_MBAR;
    // d=64 (PARO_P_STASH): the same overlap without holding p in registers -- the
    // row's 64 p values are computed before the wait and parked in TMEM over the
    // row's S columns (S is dead once p exists; the exact path re-derives S from
    // the smem Q/K tiles), then read back for the codes once lo/hi are known. The
    // compute warps no longer meet at a barrier every step, so a warp that took
    // the exact path delays the others only when it falls a whole pass behind.
    constexpr bool kStash = !SPLIT && PARO_P_STASH;
    float pv0[32];
#ifdef PARO_K3_PROF
    long long tbar = 0;
#endif
    if constexpr (kOverlap) {
        __syncwarp();
        if (PARO_PFULL_ALL || lane == 0) // every lane releases its own row stats / extremes
            ptx::mbar_arrive(red_bar);
        compute_p((int)half, pv0, true);
        ptx::mbar_wait(red_bar, red_par);
    } else if constexpr (kStash) {
        __syncwarp();
        if (PARO_PFULL_ALL || lane == 0) // every lane releases its own row stats / extremes
            ptx::mbar_arrive(red_bar);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            float pv[32];
            compute_p(h2, pv, true);
            ptx::tmem_st32(s_addr + h2 * 32, reinterpret_cast<const uint32_t(&)[32]>(pv));
        }
        ptx::mbar_wait(red_bar, red_par);
    } else {
        PROF_T(tb0);
#ifdef PARO_K3_PROF
        long long(*prof_arrive)[4] = prof_smem();
        if (G == 1 && lane == 0)
            prof_arrive[red_par][(threadIdx.x >> 5) & 3] = tb0;
#endif
        if (M128) { // the side's two softmax warps
            if (wside)
                ptx::named_bar_sync_c<2>(64);
            else
                ptx::named_bar_sync_c<1>(64);
        }
        else
            ptx::named_bar_sync(1, SPLIT ? 256 : 128); // the compute (softmax) warps
        PROF_T(tb1);
#ifdef PARO_K3_PROF
        tbar = tb1;
        if (G == 1) {
            PROF_ADD(11, tb0 - tp1);
            PROF_ADD(12, tb1 - tb0);
            if (((threadIdx.x >> 5) & 3) == 0) { // spread of the four arrivals, once per CTA step
                long long a0 = prof_arrive[red_par][0], mn = a0, mx = a0;
                for (int w = 1; w < 4; ++w) {
                    mn = min(mn, prof_arrive[red_par][w]);
                    mx = max(mx, prof_arrive[red_par][w]);
                }
                PROF_ADD(14, mx - mn);
                PROF_ADD(15, 1);
                a0 = prof_arrive[2 + red_par][0], mn = a0, mx = a0;
                for (int w = 1; w < 4; ++w) {
                    mn = min(mn, prof_arrive[2 + red_par][w]);
                    mx = max(mx, prof_arrive[2 + red_par][w]);
                }
                (void)(mx - mn); // (the step-start spread: see k3_experiments.md)
            }
        }
#endif
    }
    float lo = red_r[0].x, hi = red_r[0].y;
#pragma unroll
    for (int q = 1; q < (M128 ? 2 : 4); ++q) {
        lo = fminf(lo, red_r[2 * q].x);
        hi = fmaxf(hi, red_r[2 * q].y);
    }
    float pscale = __fdiv_rn(hi - lo, p_qmax);
    if (pscale == 0.f)
        pscale = 1.f;
    const float inv = __frcp_rn(pscale);
    PROF_T(tp2);
    PROF_ADD(2, tp2 - tp1);
#ifdef PARO_K3_PROF
    if (G == 1 && !kOverlap && !kStash)
        PROF_ADD(13, tp2 - tbar);
#endif
    uint64_t A2, B2;
    pgroup_consts<G == 1 ? 3 : 1>(lo, hi, inv, p_qmax, A2, B2);
    const uint64_t magic2 = pk(8388608.0f, 8388608.0f);
    uint32_t risk = 0; // bit g: 4-element group g has a code that needs the exact path
    const uint32_t m8 = one << 8, m16 = one << 16, m24 = one << 24; // runtime 256^e: IMAD, not SHF / LEA
    auto quantize_store = [&](int h2, const float (&pv)[32]) {
        uint32_t whi[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            uint32_t hi4 = 0, lo4 = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 4 * w + e;
                // variants (q(1-kappa), q(1+kappa)) of element k; floor(. + 0.5) via round-down adds
                const uint64_t u2 = add2_rm(fma2_rm(pk(pv[k], pv[k]), A2, B2), magic2);
                float ul, uh;
                upk(u2, ul, uh);
                // PARO_PACK_IMAD: the word as sum_e 256^e * bits(u_e) - 0x4B000000 mod 2^32 (bits(u_e) =
                // 0x4B000000 + code_e; every higher multiple of 0x4B000000 vanishes mod 2^32) on the FMA pipe
                if (e == 0) {
                    hi4 = (PARO_PACK_IMAD & 2) ? imad_u32(__float_as_uint(uh), one, 0xB5000000u) : __float_as_uint(uh);
                    lo4 = (PARO_PACK_IMAD & 1) ? imad_u32(__float_as_uint(ul), one, 0xB5000000u) : __float_as_uint(ul);
                } else { // insert byte 0 of the code word at byte e
                    const uint32_t sel = e == 1 ? 0x3240u : (e == 2 ? 0x3410u : 0x4210u);
                    const uint32_t m = e == 1 ? m8 : (e == 2 ? m16 : m24);
                    hi4 = (PARO_PACK_IMAD & 2) ? imad_u32(__float_as_uint(uh), m, hi4) : __byte_perm(hi4, __float_as_uint(uh), sel);
                    lo4 = (PARO_PACK_IMAD & 1) ? imad_u32(__float_as_uint(ul), m, lo4) : __byte_perm(lo4, __float_as_uint(ul), sel);
                }
            }
            whi[w] = hi4;
            if (hi4 != lo4)
                risk |= 1u << (h2 * 8 + w);
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int chunk = h2 * 2 + c;
            *reinterpret_cast<uint4*>(prow + ((chunk ^ ((r >> 1) & 3)) << 4)) =
                make_uint4(whi[4 * c], whi[4 * c + 1], whi[4 * c + 2], whi[4 * c + 3]);
        }
    };
    if constexpr (kOverlap) {
        quantize_store((int)half, pv0);
    } else if constexpr (kStash) {
        ptx::tmem_st_wait();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t x[32];
            ptx::tmem_ld32(s_addr + h2 * 32, x);
            ptx::tmem_ld_wait();
            quantize_store(h2, reinterpret_cast<const float(&)[32]>(x));
        }
    } else {
#pragma unroll kK3Unroll
        for (int hh = 0; hh < (SPLIT ? 1 : 2); ++hh) { // the warp's key-column half (SPLIT) or both
            const int h2 = SPLIT ? (int)half : hh;
            float pv[32];
            // the tail mask is applied below, not here: a warp-uniform branch between
            // the exponentials and the quantizer keeps ptxas from overlapping them
            compute_p(h2, pv, SPLIT);
            quantize_store(h2, pv);
        }
        if (!SPLIT && tail_any) { // rare (the last key block): the row sum again without the padded columns
            sum2 = pk(0.f, 0.f);
#pragma unroll 1
            for (int h2 = 0; h2 < 2; ++h2) {
                float pv[32];
                compute_p(h2, pv, true);
            }
        }
    }
    if (!valid)
        risk = 0;
    PROF_T(tp3);
    PROF_ADD(3, tp3 - tp2);
    // -------- exact boundary path: rare, warp-uniform entry
#ifdef PARO_EXP_NOEXACT
    risk = 0;
#endif
    if (__any_sync(0xffffffffu, risk != 0)) {
        // exact tile lo/hi of both q-blocks from every row's published extremes
        // (only rows whose fast-path extreme is within 1e-5 of the fast tile
        // extreme can hold the exact one: fp64 exp runs for those few rows, and
        // only for the q-blocks that have a risky code in this warp)
        const uint32_t rmask = __ballot_sync(0xffffffffu, risk != 0);
        float lo_e[2] = {INFINITY, INFINITY}, hi_e[2] = {0.f, 0.f};
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
            if (M128 ? sd != (int)wside : !((sd ? rmask >> 16 : rmask & 0xffffu)))
                continue;
            const float2* rd = M128 ? red_r : red_r - (int)side + sd; // the side's quadrant extremes
            float lo_a = rd[0].x, hi_a = rd[0].y;
#pragma unroll
            for (int q = 1; q < (M128 ? 2 : 4); ++q) {
                lo_a = fminf(lo_a, rd[2 * q].x);
                hi_a = fmaxf(hi_a, rd[2 * q].y);
            }
            float mn = INFINITY, mx = 0.f;
            if (PARO_EXACT_MONO == 2 || (PARO_EXACT_MONO == 1 && (G == 2 || P4))) {
                // exp and the fp32 rounding are monotone, so the tile's exact extremes are
                // float(exp()) of the smallest / largest (logit - m) over its valid rows:
                // reduce the fp64 arguments over the 64 rows, then one exp each
                double dmn = INFINITY, dmx = -INFINITY;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const RowStatC q = rs_r[sd * 64 + lane + 32 * k];
                    if (q.pmin == INFINITY) // no tile in this row this step
                        continue;
                    dmn = fmin(dmn, q.dmin);
                    dmx = fmax(dmx, q.dmax);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
                    dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
                }
                mn = dmn == INFINITY ? INFINITY : (float)exp(dmn);
                mx = dmx == -INFINITY ? 0.f : (dmx == 0.0 ? 1.0f : (float)exp(dmx));
            } else {
                double args[4];
                uint32_t kinds = 0, cnt = 0; // bit i: arg i is a max candidate
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const RowStatC q = rs_r[sd * 64 + lane + 32 * k];
                    if (q.pmin == INFINITY) // no tile in this row this step
                        continue;
                    if (q.pmin <= lo_a * 1.00001f)
                        args[cnt++] = q.dmin;
                    if (q.pmax >= hi_a * 0.99999f) {
                        if (q.dmax == 0.0)
                            mx = 1.0f; // exp(0)
                        else {
                            kinds |= 1u << cnt;
                            args[cnt++] = q.dmax;
                        }
                    }
                }
                for (uint32_t it = 0; __any_sync(0xffffffffu, it < cnt); ++it) {
                    if (it < cnt) {
                        const float e = (float)exp(args[it]);
                        if ((kinds >> it) & 1u)
                            mx = fmaxf(mx, e);
                        else
                            mn = fminf(mn, e);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
            }
            lo_e[sd] = mn;
            hi_e[sd] = mx;
        }
        PROF_T(tx1);
        PROF_ADD(8, tx1 - tp3);
        // exact tile pscale of both sides (warp-uniform) and each side's fast-variant
        // coefficients (uniform within a side: taken from lanes 0 and 16)
        float ps_e[2];
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
            ps_e[sd] = __fdiv_rn(hi_e[sd] - lo_e[sd], p_qmax);
            if (ps_e[sd] == 0.f)
                ps_e[sd] = 1.f;
        }
        const uint64_t A2s[2] = {M128 ? A2 : __shfl_sync(0xffffffffu, A2, 0), M128 ? A2 : __shfl_sync(0xffffffffu, A2, 16)};
        const uint64_t B2s[2] = {M128 ? B2 : __shfl_sync(0xffffffffu, B2, 0), M128 ? B2 : __shfl_sync(0xffffffffu, B2, 16)};
        // the warp's risky 4-element groups, listed (owner lane, group) and spread
        // over all 32 lanes one element each, instead of serially in their owner lanes
        const uint32_t ng = __popc(risk);
        uint32_t incl = ng;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o)
                incl += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        {
            uint32_t pos = incl - ng, rr = risk;
            while (rr) {
                const uint32_t g = __ffs(rr) - 1;
                rr &= rr - 1;
                xlist[pos++] = (uint16_t)((lane << 4) | g);
            }
        }
        __syncwarp();
        const int32_t rowoff = (int32_t)((r >> 3) * 512 + (r & 7) * 64);
        for (uint32_t base = 0; base < 4 * total; base += 32) {
            const uint32_t item = base + lane;
            const bool act = item < 4 * total;
            const uint32_t ent = act ? xlist[item >> 2] : (lane << 4);
            const uint32_t o = ent >> 4, j = ((ent & 15u) << 2) + (item & 3u);
            // the owner row's parameters
            const uint32_t r_o = __shfl_sync(0xffffffffu, r, (int)o);
            const int32_t smax_o = __shfl_sync(0xffffffffu, smax_i, (int)o);
            const int32_t smax1_o = __shfl_sync(0xffffffffu, smax1_i, (int)o);
            const float c0_o = __shfl_sync(0xffffffffu, c0, (int)o);
            const float c1_o = __shfl_sync(0xffffffffu, c1, (int)o);
            const float c0lo_o = (kArg & 2) ? __shfl_sync(0xffffffffu, c0lo, (int)o) : 0.f;
            const float c1lo_o = (kArg & 2) ? __shfl_sync(0xffffffffu, c1lo, (int)o) : 0.f;
            const float dmax_o = __shfl_sync(0xffffffffu, dmax, (int)o);
            const double a64_o = __shfl_sync(0xffffffffu, a64, (int)o);
            const double a64b_o = __shfl_sync(0xffffffffu, a64b, (int)o);
            const double m64_o = __shfl_sync(0xffffffffu, m64, (int)o);
            const uint32_t ncol_o = __shfl_sync(0xffffffffu, ncol, (int)o);
            if (!act || j >= ncol_o)
                continue;
            const uint32_t so = M128 ? wside : o >> 4;
            const int32_t dside = (int32_t)so - (int32_t)side;
            const uint8_t* qt = qtile + dside * (int32_t)(64 * D);
            const uint8_t* kt = ktile + dside * (int32_t)(64 * D);
            int32_t Sj, S1j = 0;
            if (G == 1)
                Sj = dot_row64(qt + (M128 ? (r_o >> 5) * K3Cfg<64>::HALF : 0u), kt, r_o, j); // M128: rows 32-63 one slot on
            else
                dot_row128(qt, kt, r_o, j, Sj, S1j);
            { // re-run the two fast variants of this element; only a split pair needs fp64
                float pf;
                if (!(kArg & 2)) {
                    pf = G == 1 ? ex2(fmaf(__int2float_rn(Sj - smax_o), c0_o, dmax_o))
                                : ex2(fmaf(__int2float_rn(S1j - smax1_o), c1_o, fmaf(__int2float_rn(Sj - smax_o), c0_o, dmax_o)));
                } else { // the same arithmetic as pass 2 (arg128_2), one lane of the pair
                    const float d0f = __int2float_rn(Sj - smax_o), d1f = __int2float_rn(S1j - smax1_o);
                    float ya, yb;
                    upk(arg128_2(pk(d0f, d0f), pk(d1f, d1f), pk(c0_o, c0_o), pk(c1_o, c1_o), pk(c0lo_o, c0lo_o),
                                 pk(c1lo_o, c1lo_o), pk(dmax_o, dmax_o)), ya, yb);
                    pf = ex2(ya);
                }
                float ul, uh;
                upk(add2_rm(fma2_rm(pk(pf, pf), A2s[so], B2s[so]), magic2), ul, uh);
                if (__float_as_uint(ul) == __float_as_uint(uh))
                    continue;
            }
            const double logit = G == 1 ? __dmul_rn(scale64, __dmul_rn(a64_o, (double)Sj))
                                        : logit128(scale64, a64_o, a64b_o, Sj, S1j);
            const float p = (float)exp(logit - m64_o);
            float q = __fdiv_rn(__fsub_rn(p, lo_e[so]), ps_e[so]);
            q = fminf(p_qmax, fmaxf(0.f, q));
            uint8_t* prow_o = prow + dside * (int32_t)(64 * 64) - rowoff +
                              (int32_t)((r_o >> 3) * 512 + (r_o & 7) * 64);
            const int chunk = j >> 4;
            prow_o[((chunk ^ ((r_o >> 1) & 3)) << 4) + (j & 15)] = (uint8_t)round_half_away_pos(q);
        }
        __syncwarp();
        PROF_T(tx2);
        PROF_ADD(9, tx2 - tx1);
        PROF_ADD(10, 1);
    }
    PROF_T(tp4);
    PROF_ADD(4, tp4 - tp3);
    float sa, sb;
    upk(sum2, sa, sb);
    if (live) {
        st.l = st.l * gamma + (sa + sb);
        st.m32 = m32;
        st.m64 = m64;
    }
    gamma_out = gamma;
    lo_out = lo;
    pscale_out = pscale;
}

// INT4 V: one 64-key tile from its nibble-packed form (row r: D/2 bytes, byte b =
// columns 2b (low nibble) and 2b+1, two's complement) into the i8 tile of the P.V
// MMA's B operand (rows of D bytes, 64B / 128B swizzle), by the 32 lanes of a warp.
// d = 64 unpacks in place (the packed tile sits in the upper half of the output
// tile: every lane reads its two rows before any lane writes).
// nibble n -> byte sext(n) in every byte lane without cross-byte carries:
// ((n ^ 8) + 0x78) ^ 0x80 = (n ^ 8) - 8 (the sum stays within 0x78..0x87)
__device__ __forceinline__ uint32_t sext_nibbles(uint32_t n4) {
    return ((n4 ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
}
__device__ __forceinline__ void nib8(uint32_t w, uint32_t& o0, uint32_t& o1) {
    const uint32_t lo = sext_nibbles(w & 0x0F0F0F0Fu), hi = sext_nibbles((w >> 4) & 0x0F0F0F0Fu);
    o0 = __byte_perm(lo, hi, 0x5140); // columns 0..3 of the word's 8
    o1 = __byte_perm(lo, hi, 0x7362); // columns 4..7
}
template <int D>
__device__ __forceinline__ void unpack_v_tile(const uint8_t* pk, uint8_t* vt, uint32_t lane) {
    if (D == 64) {
        uint4 w[4]; // rows 2 lane, 2 lane + 1: 32 packed bytes each
#pragma unroll
        for (int i = 0; i < 4; ++i)
            w[i] = *reinterpret_cast<const uint4*>(pk + lane * 64 + i * 16);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t r = 2 * lane + k;
            uint8_t* row = vt + (r >> 3) * 512 + (r & 7) * 64;
#pragma unroll
            for (int c = 0; c < 4; ++c) { // 16-column chunk c <- packed words 2c, 2c+1 of the row
                const uint4& src = w[2 * k + (c >> 1)];
                const uint32_t wa = (c & 1) ? src.z : src.x, wb = (c & 1) ? src.w : src.y;
                uint4 o;
                nib8(wa, o.x, o.y);
                nib8(wb, o.z, o.w);
                *reinterpret_cast<uint4*>(row + ((c ^ ((r >> 1) & 3)) << 4)) = o;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 2; ++k) { // rows lane, lane + 32: 64 packed bytes each
            const uint32_t r = lane + 32 * k;
            uint8_t* row = vt + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 src = *reinterpret_cast<const uint4*>(pk + r * 64 + q * 16);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int c = 2 * q + h;
                    uint4 o;
                    nib8(h ? src.z : src.x, o.x, o.y);
                    nib8(h ? src.w : src.y, o.z, o.w);
                    *reinterpret_cast<uint4*>(row + ((c ^ (r & 7)) << 4)) = o;
                }
            }
        }
    }
}

// DUMP: the P-code dump test hook is compiled in (a separate instantiation, so the
// product kernel carries no extra registers for it)
#ifndef PARO_DIAG_NOI2F
#define PARO_DIAG_NOI2F 0 // diagnostic builds only: epilogue reads int32 P.V as fp32 bits (wrong results)
#endif
#ifndef PARO_DIAG_NOUNPACK
#define PARO_DIAG_NOUNPACK 0 // diagnostic builds only: skip the INT4 unpack (wrong results)
#endif
// PACKED: INT4 V arrives nibble-packed and is unpacked in shared memory (a separate
// instantiation: the INT8 kernels carry none of that code)
template <int D, bool DUMP, bool PACKED, bool P4 = false>
__global__ void __launch_bounds__(K3Cfg<D>::THREADS, K3Cfg<D>::MINB)
    k3_attention(const __grid_constant__ K3Params P, const __grid_constant__ CUtensorMap tm_q,
                 const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                 const __grid_constant__ CUtensorMap tm_vp, const __grid_constant__ CUtensorMap tm_q32) {
    using C = K3Cfg<D>;
    using BR = Bars<C::NS>;
    constexpr int G = C::G;
#ifdef PARO_K3_PROF
    const unsigned long long cta_t0 = ptx::globaltimer();
#endif
    constexpr int NS = C::NS;
    // dynamic smem is 1024-B aligned (SWIZZLE_128B atoms); declared __shared__ so
    // the compiler emits LDS/STS rather than generic loads
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bar0 = sbase + C::OFF_BAR;
    auto bar = [&](uint32_t i) { return bar0 + 8 * i; };
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const LayerDev& L = P.L;

    if (threadIdx.x == 0) {
        // Q tiles are double-buffered by item parity; a buffer is free once the
        // item's last QK retired AND the softmax warps finished the item (the
        // exact boundary path re-reads Q from smem)
        ptx::mbar_init(bar(B_QFULL), 1);
        ptx::mbar_init(bar(B_QEMPTY), 1 + C::NCW);
        ptx::mbar_init(bar(BR::QFULL1), 1);
        ptx::mbar_init(bar(BR::QEMPTY1), 1 + C::NCW);
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(bar(BR::KVFULL + s), 1);
            ptx::mbar_init(bar(BR::KVEMPTY + s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(bar(BR::SFULL + b), 1);
            ptx::mbar_init(bar(BR::SEMPTY + b), C::NCW);
            ptx::mbar_init(bar(BR::PFULL + b), C::NCW * (PARO_PFULL_ALL ? 32 : 1));
            ptx::mbar_init(bar(BR::PEMPTY + b), 1 + C::NCW);
            ptx::mbar_init(bar(BR::OFULL + b), 1);
            ptx::mbar_init(bar(BR::OEMPTY + b), C::NCW);
        }
        // P-group extremes and row stats published (one arrival per compute thread)
        ptx::mbar_init(bar(BR::RED), C::NCW * (PARO_PFULL_ALL ? 32 : 1));
        for (int i = 0; i < 2; ++i) { // item queue: producer -> the other roles
            ptx::mbar_init(bar(BR::ITEMFULL + i), 1);
            ptx::mbar_init(bar(BR::ITEMEMPTY + i), C::NCONS);
        }
        for (int s = 0; s < NS; ++s)
            ptx::mbar_init(bar(BR::VFULL + s), C::NVFULL);
        // !SPLIT: softmax -> epilogue row sums (one arrival per thread, as PFULL)
        ptx::mbar_init(bar(BR::LFULL), 4 * (PARO_PFULL_ALL ? 32 : 1));
        ptx::mbar_init(bar(BR::LEMPTY), 4 * (PARO_PFULL_ALL ? 32 : 1));
        ptx::fence_barrier_init();
    }
    if (warp == 1)
        ptx::tmem_alloc<C::TMEM_COLS>(sbase + C::OFF_TMEMPTR);
    if (C::M128) { // the zero slots (1, 3, 5) of both item buffers (read by the tensor core only)
        constexpr uint32_t W = C::HALF / 16;
        for (uint32_t i = threadIdx.x; i < 2 * 3 * W; i += C::THREADS) {
            const uint32_t buf = i / (3 * W), slot = 1 + 2 * ((i / W) % 3), off = (i % W) * 16;
            *reinterpret_cast<uint4*>(smem + C::OFF_Q + buf * C::QBUF + slot * C::HALF + off) = make_uint4(0, 0, 0, 0);
        }
        ptx::fence_proxy_async_smem();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::OFF_TMEMPTR);

    const uint32_t G_cta = gridDim.x;
    const uint32_t rounds = (P.n_items + G_cta - 1) / G_cta;
    // static snake dealing of the LPT-sorted work list (PARO_DYNAMIC=0 builds)
    auto item_at = [&](uint32_t r) -> int {
        const uint32_t idx = r * G_cta + ((r & 1) ? (G_cta - 1 - blockIdx.x) : blockIdx.x);
        return idx < P.n_items ? (int)P.order[idx] : -1;
    };
    // DYNAMIC: the producer takes the next LPT item from a global counter (a CTA
    // that finishes early takes more: greedy LPT instead of a static deal -- the
    // tail matters at a few items per CTA) and hands it to the other roles
    // through a 2-slot queue; -1 ends the CTA's work
    volatile int* ring = reinterpret_cast<volatile int*>(smem + C::OFF_TMEMPTR + 8);
    auto next_item = [&](uint32_t k, bool lazy) -> int { // consumers: the CTA's k-th item
        if (!PARO_DYNAMIC)
            return k < rounds ? item_at(k) : -1;
        const uint32_t slot = k & 1;
        if (lazy)
            mbar_wait_lazy(bar(BR::ITEMFULL + slot), (k >> 1) & 1);
        else
            ptx::mbar_wait(bar(BR::ITEMFULL + slot), (k >> 1) & 1);
        return ring[slot];
    };
    auto release_item = [&](uint32_t k) { // one arrival per consumer warp (caller: one lane)
        if (PARO_DYNAMIC)
            ptx::mbar_arrive(bar(BR::ITEMEMPTY + (k & 1)));
    };
    auto stage = [&](uint32_t s) { return sbase + C::OFF_STAGE + s * C::STAGE_BYTES; };
    auto qfull = [&](uint32_t i) { return bar((i & 1) ? BR::QFULL1 : (uint32_t)B_QFULL); };
    auto qempty = [&](uint32_t i) { return bar((i & 1) ? BR::QEMPTY1 : (uint32_t)B_QEMPTY); };
    auto qbuf = [&](uint32_t i) { return sbase + C::OFF_Q + (i & 1) * C::QBUF; };

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        // Lane 0 issues the TMA; with INT4 V (P.v_packed) the whole warp also unpacks
        // each stage's nibble-packed V tiles into the i8 swizzled layout the P.V MMA
        // reads (Blackwell has no INT4 MMA), one step behind the loads, and releases
        // them with VFULL -- QK waits only for K.
        if (C::SPLIT || C::W12)
            ptx::setmaxnreg_dec<C::REG_LOW>();
        constexpr bool packed = PACKED;
        if (lane == 0) {
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(packed ? &tm_vp : &tm_v);
        }
        uint32_t T = 0, I = 0;
        uint32_t pend = 0; // bit 0: a step's packed V waits for its unpack; bits 1-2: sides A / B
        auto unpack_pending = [&]() {
            if (!(pend & 1u))
                return;
            const uint32_t U = T - 1, s = U % NS;
            ptx::mbar_wait(bar(BR::KVFULL + s), (U / NS) & 1);
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                if (!((pend >> (1 + side)) & 1u) || PARO_DIAG_NOUNPACK)
                    continue;
                uint8_t* vt = smem + C::OFF_STAGE + s * C::STAGE_BYTES + (2 + side) * C::KV_BYTES;
                const uint8_t* pk8 = C::SPLIT ? smem + C::OFF_VPK + (s * 2 + side) * C::VPK_BYTES : vt + C::KV_BYTES / 2;
                unpack_v_tile<D>(pk8, vt, lane);
            }
            ptx::fence_proxy_async_smem(); // the unpacked codes -> the tensor core's view
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(BR::VFULL + s));
            pend = 0;
        };
        // only d = 64 with INT4 V needs the whole warp in the loop (it unpacks); else lane 0 alone
        const bool all_lanes = packed && !C::SPLIT;
        const uint32_t wmask = all_lanes ? 0xffffffffu : 1u;
        for (uint32_t r = 0; all_lanes || lane == 0; ++r) {
            int it = 0;
            if (PARO_DYNAMIC) {
                if (lane == 0) {
                    const uint32_t idx = atomicAdd(P.work_counter, 1u);
                    it = idx < P.n_items ? (int)P.order[idx] : -1;
                }
                it = __shfl_sync(wmask, it, 0);
                const uint32_t slot = r & 1;
                mbar_wait_lazy(bar(BR::ITEMEMPTY + slot), ((r >> 1) & 1) ^ 1);
                if (lane == 0) {
                    ring[slot] = it;
                    ptx::mbar_arrive(bar(BR::ITEMFULL + slot));
                }
                __syncwarp(wmask);
                if (it < 0)
                    break;
            } else {
                if (r >= rounds)
                    break;
                it = item_at(r);
                if (it < 0)
                    continue;
            }
            const Item x = load_item(L, (uint32_t)it);
            const uint16_t* la = L.items + ((size_t)x.h * L.kb + x.qa) * L.kb;
            const uint16_t* lb = L.items + ((size_t)x.h * L.kb + (x.qb != 0xffffu ? x.qb : 0)) * L.kb;
            const int32_t row0 = (int32_t)(x.h * L.kb2 * 64);
            ptx::mbar_wait(qempty(I), ((I >> 1) & 1) ^ 1);
            if (lane == 0) {
                ptx::mbar_arrive_expect_tx(qfull(I), (x.qb != 0xffffu ? 2 : 1) * C::QT_BYTES);
                if (C::M128) { // 32-row halves into slots 0, 2 (A) and 4, 6 (B)
                    ptx::tma_load_2d(qbuf(I), &tm_q32, 0, row0 + (int32_t)x.qa * 64, qfull(I));
                    ptx::tma_load_2d(qbuf(I) + 2 * C::HALF, &tm_q32, 0, row0 + (int32_t)x.qa * 64 + 32, qfull(I));
                    if (x.qb != 0xffffu) {
                        ptx::tma_load_2d(qbuf(I) + 4 * C::HALF, &tm_q32, 0, row0 + (int32_t)x.qb * 64, qfull(I));
                        ptx::tma_load_2d(qbuf(I) + 6 * C::HALF, &tm_q32, 0, row0 + (int32_t)x.qb * 64 + 32,
                                         qfull(I));
                    }
                } else {
                    ptx::tma_load_2d(qbuf(I), &tm_q, 0, row0 + (int32_t)x.qa * 64, qfull(I));
                    if (x.qb != 0xffffu)
                        ptx::tma_load_2d(qbuf(I) + C::QB_OFF, &tm_q, 0, row0 + (int32_t)x.qb * 64, qfull(I));
                }
            }
            for (uint32_t t = 0; t < x.n; ++t) {
                const uint32_t s = T % NS;
                mbar_wait_lazy(bar(BR::KVEMPTY + s), ((T / NS) & 1) ^ 1);
                const bool ha = t < x.na, hb = t < x.nb;
                if (lane == 0) {
                    const uint32_t vbytes = packed ? C::VPK_BYTES : C::KV_BYTES;
                    ptx::mbar_arrive_expect_tx(bar(BR::KVFULL + s), (ha + hb) * (C::KV_BYTES + vbytes + C::META_BYTES));
                    const uint32_t st = stage(s);
#pragma unroll
                    for (int side = 0; side < 2; ++side) {
                        if (side ? hb : ha) {
                            const uint32_t bj = side ? lb[t] : la[t];
                            ptx::tma_load_2d(st + side * C::KV_BYTES, &tm_k, 0, row0 + (int32_t)bj * 64,
                                             bar(BR::KVFULL + s));
                            if (packed)
                                ptx::tma_load_2d(C::SPLIT ? sbase + C::OFF_VPK + (s * 2 + side) * C::VPK_BYTES
                                                          : st + (2 + side) * C::KV_BYTES + C::KV_BYTES / 2,
                                                 &tm_vp, 0, row0 + (int32_t)bj * 64, bar(BR::KVFULL + s));
                            else
                                ptx::tma_load_2d(st + (2 + side) * C::KV_BYTES, &tm_v, 0, row0 + (int32_t)bj * 64,
                                                 bar(BR::KVFULL + s));
                            ptx::bulk_load(st + 4 * C::KV_BYTES + side * C::META_BYTES,
                                           L.meta + ((size_t)x.h * L.kb2 + bj) * meta_stride(D), C::META_BYTES,
                                           bar(BR::KVFULL + s));
                        }
                    }
                }
                if (packed && !C::SPLIT) { // unpack the previous step while this one's loads are in flight
                    if (all_lanes)
            unpack_pending();
                    pend = 1u | (ha ? 2u : 0u) | (hb ? 4u : 0u);
                }
                ++T;
            }
            ++I;
        }
        unpack_pending();
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (C::SPLIT || C::W12)
            ptx::setmaxnreg_dec<C::REG_LOW>();
        if (lane == 0) {
            uint32_t T = 0, I = 0;
            unsigned long long prof[4] = {0, 0, 0, 0};
            auto issue_pv = [&](uint32_t U, bool ha, bool hb) {
                const uint32_t s = U % NS, b = U & 1, ph = (U >> 1) & 1;
                PROF_T(tm0);
                mbar_wait_mma(bar(BR::PFULL + b), ph);
                mbar_wait_mma(bar(BR::OEMPTY + b), ph ^ 1);
                if (PACKED) // the unpacked V is usually ready: wait without a sleep back-off
                    ptx::mbar_wait(bar(BR::VFULL + s), (U / NS) & 1);
                ptx::tc_fence_after();
                PROF_T(tm1);
                PROF_ADD(1, tm1 - tm0);
#pragma unroll
                for (int side = 0; side < 2; ++side) {
                    if (side ? hb : ha) {
                        const uint32_t sp = sbase + C::OFF_P + (b * 2 + side) * C::P_BYTES;
                        const uint32_t sv = stage(s) + (2 + side) * C::KV_BYTES;
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk)
                            ptx::mma_i8(tmem + (side ? C::LANE16 : 0u) + C::TM_O + b * D, desc_p(sp + kk * 32),
                                        desc_v<D>(sv + kk * 32 * D), C::IDESC_PV, kk);
                    }
                }
                ptx::mma_commit(bar(BR::OFULL + b));
                ptx::mma_commit(bar(BR::KVEMPTY + s));
                ptx::mma_commit(bar(BR::PEMPTY + b));
            };
            for (uint32_t r = 0;; ++r) {
                if (!PARO_DYNAMIC && r >= rounds)
                    break;
                const int it = next_item(r, true);
                release_item(r);
                if (it < 0) {
                    if (PARO_DYNAMIC)
                        break;
                    continue;
                }
                const Item x = load_item(L, (uint32_t)it);
                ptx::mbar_wait(qfull(I), (I >> 1) & 1);
                ptx::tc_fence_after();
                for (uint32_t t = 0; t < x.n; ++t, ++T) {
                    const uint32_t s = T % NS, b = T & 1;
                    PROF_T(tm2);
                    mbar_wait_mma(bar(BR::KVFULL + s), (T / NS) & 1);
                    mbar_wait_mma(bar(BR::SEMPTY + b), ((T >> 1) & 1) ^ 1);
                    ptx::tc_fence_after();
                    PROF_T(tm3);
                    PROF_ADD(0, tm3 - tm2);
                    PROF_ADD(3, 1);
                    if (C::M128) {
                        if (t < x.na)
                            issue_qk128(tmem + C::TM_S + b * C::S_COLS, qbuf(I), stage(s), true);
                        if (t < x.nb)
                            issue_qk128(tmem + C::TM_S + b * C::S_COLS, qbuf(I) + C::QOP_B, stage(s) + C::KV_BYTES,
                                        t >= x.na);
                    } else {
                        if (t < x.na)
                            issue_qk<D>(tmem + C::TM_S + b * C::S_COLS, qbuf(I), stage(s));
                        if (t < x.nb)
                            issue_qk<D>(tmem + C::LANE16 + C::TM_S + b * C::S_COLS, qbuf(I) + C::QT_BYTES,
                                        stage(s) + C::KV_BYTES);
                    }
                    ptx::mma_commit(bar(BR::SFULL + b));
                    if (t + 1 == x.n)
                        ptx::mma_commit(qempty(I));
                    if (t > 0)
                        issue_pv(T - 1, t - 1 < x.na, t - 1 < x.nb);
                }
                if (x.n > 0)
                    issue_pv(T - 1, x.n - 1 < x.na, x.n - 1 < x.nb);
                else
                    ptx::mma_commit(qempty(I));
                ++I;
            }
#ifdef PARO_K3_PROF
            for (int i = 0; i < 4; ++i)
                atomicAdd(&g_prof[12 + i], prof[i]);
#endif
        }
    } else if (!C::SPLIT && (!C::W12 || warp >= 4)) {
        if (C::W12)
            ptx::setmaxnreg_inc<C::REG_COMPUTE>();
        if (warp < C::SM0 + 4) {
        // ------------------------------------------------------------ softmax
        const uint32_t quad = warp & 3;
        // M128: quadrants 0 / 2 hold q-block A's rows 0-31 / 32-63, quadrants 1 / 3 B's
        const uint32_t side = C::M128 ? quad & 1 : lane >> 4;
        const uint32_t r = C::M128 ? (quad >> 1) * 32 + lane : quad * 16 + (lane & 15); // row within its q-block
        const uint32_t lane_base = (quad * 32) << 16;
        float2* red = reinterpret_cast<float2*>(smem + C::OFF_RED);
        float4* rowmeta = reinterpret_cast<float4*>(smem + C::OFF_ROWMETA);
        float* usm = reinterpret_cast<float*>(smem + C::OFF_U);
        float* lsm = reinterpret_cast<float*>(smem + C::OFF_L);
        const uint32_t tail = L.N & 63;
        uint32_t T = 0, I = 0;
        unsigned long long prof[18] = {};
        for (uint32_t rr = 0;; ++rr) {
            if (!PARO_DYNAMIC && rr >= rounds)
                break;
            PROF_T(ti2);
            const int it = next_item(rr, false);
            PROF_T(ti3);
            PROF_ADD(16, ti3 - ti2);
            __syncwarp();
            if (lane == 0)
                release_item(rr);
            if (it < 0) {
                if (PARO_DYNAMIC)
                    break;
                continue;
            }
            const Item x = load_item(L, (uint32_t)it);
            const bool has_qb = side ? x.qb != 0xffffu : true;
            const uint32_t qb = side ? (has_qb ? x.qb : 0u) : x.qa;
            const uint32_t nmine = side ? x.nb : x.na;
            const uint16_t* list = L.items + ((size_t)x.h * L.kb + qb) * L.kb;
            const bool valid_row = has_qb && qb * 64 + r < L.N && qb * 64 + r >= L.dp; // dense rows: K4
            const float sq0 = L.qsc[((size_t)x.h * L.kb2 + qb) * G];
            const float sq1 = G == 2 ? L.qsc[((size_t)x.h * L.kb2 + qb) * G + G - 1] : 0.f;
            RowState st{-INFINITY, 0.f, -INFINITY};
            if (L.dp && valid_row) { // continue from K4's dense-prefix state
                const size_t srow = (size_t)x.h * L.kb2 * 64 + qb * 64 + r;
                st.m64 = L.init_m[srow];
                st.m32 = (float)(st.m64 * kLog2e);
                st.l = L.init_l[srow];
            }
            RowStatC* rowstat = reinterpret_cast<RowStatC*>(smem + C::OFF_ROWSTAT);
            const int32_t dslot = DUMP && has_qb ? P.dump.slot[(size_t)x.h * L.kb2 + qb] : -1;
            for (uint32_t t = 0; t < x.n; ++t, ++T) {
                const uint32_t s = T % NS, b = T & 1, ph = (T >> 1) & 1;
                const bool live = t < nmine;
                const uint32_t bj = live ? list[t] : 0u;
                PROF_T(tw0);
                mbar_wait3t(bar(BR::SFULL + b), ph, bar(BR::PEMPTY + b), ph ^ 1, bar(BR::KVFULL + s), (T / NS) & 1);
                ptx::tc_fence_after();
                PROF_T(tw1);
                PROF_ADD(0, tw1 - tw0);
#ifdef PARO_K3_PROF
                if (lane == 0)
                    prof_smem()[2 + (T & 1)][quad] = tw1;
#endif
                const float* meta =
                    reinterpret_cast<const float*>(smem + C::OFF_STAGE + s * C::STAGE_BYTES + 4 * C::KV_BYTES +
                                                   side * C::META_BYTES);
                uint8_t* prow = smem + C::OFF_P + (b * 2 + side) * C::P_BYTES + (r >> 3) * 512 + (r & 7) * 64;
                const uint32_t s_addr = tmem + lane_base + C::TM_S + b * C::S_COLS;
                // M128: one extreme pair per quadrant, a side's two quadrants at red_r[0], red_r[2]
                float2* red_w = C::M128 ? red + (T & 1) * 8 + side * 4 + (quad >> 1) * 2
                                        : red + ((T & 1) * 4 + quad) * 2 + side;
                const float2* red_r = red + (T & 1) * 8 + (C::M128 ? side * 4 : side);
                const bool tail_tile = tail != 0 && live && bj == L.kb - 1;
                RowStatC* rs_w = rowstat + ((T & 1) * 2 + side) * 64 + r;
                const RowStatC* rs_r = rowstat + (T & 1) * 128;
                const uint8_t* qtile = smem + C::OFF_Q + (I & 1) * C::QBUF + side * C::QB_OFF;
                const uint8_t* ktile = smem + C::OFF_STAGE + s * C::STAGE_BYTES + side * C::KV_BYTES;
                float gamma, lo, pscale;
                softmax_step<D, false, P4>(s_addr, sq0, meta[0], meta[1], P.scale64, P.scale_log2, tail_tile ? tail : 64u, live,
                                valid_row, st, P.p_qmax, red_w, red_r, rs_w, rs_r, side, qtile, ktile, prow, r, sq1,
                                gamma, lo, pscale, 0u, nullptr,
                                reinterpret_cast<uint16_t*>(smem + C::OFF_XLIST) + quad * 512, bar(BR::RED),
                                T & 1, prof, P.one);
                if (DUMP && dslot >= 0 && live) {
                    dump_row(P.dump, dslot, t, r, prow, 0, 4);
                    if (r == 0)
                        dump_meta(P.dump, dslot, t, lo, pscale, bj);
                }
                PROF_T(tw2);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    ptx::mbar_arrive(bar(BR::SEMPTY + b));
                const float vsc = meta[2];
                rowmeta[(b * 2 + side) * 64 + r] =
                    make_float4(live ? gamma : 1.f, live ? pscale * vsc : 0.f, 0.f, live ? 1.f : 0.f);
                // per-column offset term of this tile: (lo * vscale) * colsum[c]; exactly 0
                // when idle (an idle side's meta slot is not loaded: stale smem, maybe NaN)
                const float os = lo * vsc;
                float* u = usm + (b * 2 + side) * D;
#pragma unroll
                for (int c = 0; c < D / 64; ++c)
                    u[r + 64 * c] = live ? os * meta[4 + r + 64 * c] : 0.f;
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (PARO_PFULL_ALL || lane == 0) // every lane releases its own P codes / row meta / offsets
                    ptx::mbar_arrive(bar(BR::PFULL + b));
                PROF_T(tw3);
                PROF_ADD(5, tw3 - tw2);
                PROF_ADD(6, 1);
            }
            PROF_ADD(7, 1);
            PROF_T(ti0);
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(qempty(I)); // this warp no longer reads the item's Q tiles
            ptx::mbar_wait(bar(BR::LEMPTY), (I & 1) ^ 1);
            PROF_T(ti1);
            PROF_ADD(17, ti1 - ti0);
            lsm[side * 64 + r] = st.l;
            __syncwarp();
            if (PARO_PFULL_ALL || lane == 0)
                ptx::mbar_arrive(bar(BR::LFULL));
            ++I;
        }
#ifdef PARO_K3_PROF
        if (lane == 0) {
            for (int i = 0; i < 8; ++i)
                atomicAdd(&g_prof[i], prof[i]);
            for (int i = 8; i < 18; ++i)
                if (i < 11 || i > 13 || G == 1)
                    atomicAdd(&g_prof[8 + i], prof[i]);
        }
#endif
        } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t quad = warp & 3;
        const uint32_t side = lane >> 4;
        const uint32_t r = quad * 16 + (lane & 15);
        const uint32_t lane_base = (quad * 32) << 16;
        const float4* rowmeta = reinterpret_cast<const float4*>(smem + C::OFF_ROWMETA);
        const float* usm = reinterpret_cast<const float*>(smem + C::OFF_U);
        const float* lsm = reinterpret_cast<const float*>(smem + C::OFF_L);
        uint32_t T = 0, I = 0;
        unsigned long long prof[4] = {0, 0, 0, 0};
        for (uint32_t rr = 0;; ++rr) {
            if (!PARO_DYNAMIC && rr >= rounds)
                break;
            const int it = next_item(rr, true);
            __syncwarp();
            if (lane == 0)
                release_item(rr);
            if (it < 0) {
                if (PARO_DYNAMIC)
                    break;
                continue;
            }
            const Item x = load_item(L, (uint32_t)it);
            const bool has_qb = side ? x.qb != 0xffffu : true;
            const uint32_t qb = side ? (has_qb ? x.qb : 0u) : x.qa;
            const bool valid_row = has_qb && qb * 64 + r < L.N && qb * 64 + r >= L.dp; // dense rows: K4
            uint64_t acc[D / 2];
#pragma unroll
            for (int c = 0; c < D / 2; ++c)
                acc[c] = 0ull;
            if (L.dp && valid_row) {
                const float2* a0 = reinterpret_cast<const float2*>(
                    L.init_acc + ((size_t)x.h * L.kb2 * 64 + qb * 64 + r) * D);
#pragma unroll
                for (int c = 0; c < D / 2; ++c)
                    acc[c] = pk(a0[c].x, a0[c].y);
            }
            for (uint32_t t = 0; t < x.n; ++t, ++T) {
                const uint32_t b = T & 1, ph = (T >> 1) & 1;
                PROF_T(te0);
                mbar_wait_lazy(bar(BR::OFULL + b), ph);
                mbar_wait_lazy(bar(BR::PFULL + b), ph);
                ptx::tc_fence_after();
                PROF_T(te1);
                PROF_ADD(0, te1 - te0);
                // idle rows carry gamma 1, ss 0 and u 0: acc*1 + 0*ip + 0 == acc exactly
                const float4 rm = rowmeta[(b * 2 + side) * 64 + r];
                const uint64_t g2 = pk(rm.x, rm.x), ss2 = pk(rm.y, rm.y);
                const float4* u4 = reinterpret_cast<const float4*>(usm + (b * 2 + side) * D);
#pragma unroll
                for (int ch = 0; ch < D / 16; ++ch) {
                    uint32_t raw[16];
                    tmem_ld16(tmem + lane_base + C::TM_O + b * D + ch * 16, raw);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 uu = u4[ch * 4 + q4];
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int j = q4 * 4 + hh * 2;
                            const uint64_t x2 =
                                PARO_DIAG_NOI2F ? pk(__int_as_float(raw[j]), __int_as_float(raw[j + 1])) : (PARO_I2F_FMA & 8) ? i2f2_fma((int32_t)raw[j], (int32_t)raw[j + 1], P.one) : pk(__int2float_rn((int32_t)raw[j]), __int2float_rn((int32_t)raw[j + 1]));
                            const uint64_t t2 = fma2(ss2, x2, hh ? pk(uu.z, uu.w) : pk(uu.x, uu.y));
                            acc[(ch * 16 + j) / 2] = fma2(acc[(ch * 16 + j) / 2], g2, t2);
                        }
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(bar(BR::OEMPTY + b));
                    ptx::mbar_arrive(bar(BR::PEMPTY + b));
                }
                PROF_T(te2);
                PROF_ADD(1, te2 - te1);
                PROF_ADD(3, 1);
            }
            PROF_T(te3);
            ptx::mbar_wait(bar(BR::LFULL), I & 1);
            const float l = lsm[side * 64 + r];
            __syncwarp();
            if (PARO_PFULL_ALL || lane == 0)
                ptx::mbar_arrive(bar(BR::LEMPTY));
            ++I;
            if (valid_row) {
                const uint32_t orig = perm_src(L.perm[x.h], qb * 64 + r);
                float4* dst = reinterpret_cast<float4*>(P.out + ((size_t)x.h * L.N + orig) * D);
                if (l == 0.f) {
#pragma unroll
                    for (int c = 0; c < D / 4; ++c)
                        dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
                    const float il = 1.0f / l;
#pragma unroll
                    for (int c = 0; c < D / 4; ++c) {
                        float a0, a1, a2, a3;
                        upk(acc[2 * c], a0, a1);
                        upk(acc[2 * c + 1], a2, a3);
                        dst[c] = make_float4(a0 * il, a1 * il, a2 * il, a3 * il);
                    }
                }
                if (P.zeroed)
                    P.zeroed[(size_t)x.h * L.N + orig] = l == 0.f ? 1 : 0;
            }
            PROF_T(te4);
            PROF_ADD(2, te4 - te3);
        }
#ifdef PARO_K3_PROF
        if (lane == 0)
            for (int i = 0; i < 4; ++i)
                atomicAdd(&g_prof[8 + i], prof[i]);
#endif
        }
    } else if (C::W12) {
        ptx::setmaxnreg_dec<C::REG_LOW>(); // warps 2-3 of the d=64 W12 layout: idle
    } else if (warp >= 4) {
        // ------------------------------------------------------------ compute warps
        // warp 4 + 4*half + quad: TMEM lane quadrant `quad` (rows 16q..16q+15 of
        // q-blocks A and B), key columns / O columns of half `half`. Pass 1 runs on
        // the whole row in both warps of a quadrant (identical results); pass 2, the
        // P codes, the exact path and the dequant cover the warp's half only.
        ptx::setmaxnreg_inc<C::REG_COMPUTE>();
        const uint32_t quad = warp & 3;
        const uint32_t half = (uint32_t)(warp - 4) >> 2;
        const uint32_t side = lane >> 4;
        const uint32_t r = quad * 16 + (lane & 15); // row within its q-block
        const uint32_t lane_base = (quad * 32) << 16;
        float2* red = reinterpret_cast<float2*>(smem + C::OFF_RED);
        float4* rowmeta = reinterpret_cast<float4*>(smem + C::OFF_ROWMETA);
        float* usm = reinterpret_cast<float*>(smem + C::OFF_U);
        float* lsm = reinterpret_cast<float*>(smem + C::OFF_L); // [2 item parity][2 half][2 side][64]
        RowStatC* rowstat = reinterpret_cast<RowStatC*>(smem + C::OFF_ROWSTAT);
        const uint32_t tail = L.N & 63;
        constexpr int DH = D / 2; // O columns per warp
        uint32_t T = 0, I = 0;
        unsigned long long prof[18] = {};
        for (uint32_t rr = 0;; ++rr) {
            if (!PARO_DYNAMIC && rr >= rounds)
                break;
            const int it = next_item(rr, false);
            __syncwarp();
            if (lane == 0)
                release_item(rr);
            if (it < 0) {
                if (PARO_DYNAMIC)
                    break;
                continue;
            }
            const Item x = load_item(L, (uint32_t)it);
            const bool has_qb = side ? x.qb != 0xffffu : true;
            const uint32_t qb = side ? (has_qb ? x.qb : 0u) : x.qa;
            const uint32_t nmine = side ? x.nb : x.na;
            const uint16_t* list = L.items + ((size_t)x.h * L.kb + qb) * L.kb;
            const bool valid_row = has_qb && qb * 64 + r < L.N && qb * 64 + r >= L.dp; // dense rows: K4
            const float sq0 = L.qsc[((size_t)x.h * L.kb2 + qb) * G];
            const float sq1 = G == 2 ? L.qsc[((size_t)x.h * L.kb2 + qb) * G + G - 1] : 0.f;
            RowState st{-INFINITY, 0.f, -INFINITY};
            if (L.dp && valid_row) { // continue from K4's dense-prefix state (l: half 0 carries it)
                const size_t srow = (size_t)x.h * L.kb2 * 64 + qb * 64 + r;
                st.m64 = L.init_m[srow];
                st.m32 = (float)(st.m64 * kLog2e);
                st.l = half == 0 ? L.init_l[srow] : 0.f;
            }
            uint64_t acc[DH / 2];
#pragma unroll
            for (int c = 0; c < DH / 2; ++c)
                acc[c] = 0ull;
            if (L.dp && valid_row) {
                const float2* a0 = reinterpret_cast<const float2*>(
                    L.init_acc + ((size_t)x.h * L.kb2 * 64 + qb * 64 + r) * D + half * DH);
#pragma unroll
                for (int c = 0; c < DH / 2; ++c)
                    acc[c] = pk(a0[c].x, a0[c].y);
            }
            const int32_t dslot = DUMP && has_qb ? P.dump.slot[(size_t)x.h * L.kb2 + qb] : -1;
            // acc = gamma * acc + (pscale * vscale) * ip + u_c over this warp's O columns,
            // for step U (its P side was published before this warp's own PFULL arrive)
            auto dequant = [&](uint32_t U) {
                const uint32_t b = U & 1, ph = (U >> 1) & 1;
                PROF_T(te0);
                // PFULL(U) (already complete: every compute warp arrived) orders the
                // half-0 warp's rowmeta / column-offset writes before these reads
                // directly, not only through the MMA's commit of O
                mbar_wait2(bar(BR::OFULL + b), ph, bar(BR::PFULL + b), ph);
                ptx::tc_fence_after();
                PROF_T(te1);
                PROF_ADD(5, te1 - te0);
                // idle rows carry gamma 1, ss 0 and u 0: acc*1 + 0*ip + 0 == acc exactly
                const float4 rm = rowmeta[(b * 2 + side) * 64 + r];
                const uint64_t g2 = pk(rm.x, rm.x), ss2 = pk(rm.y, rm.y);
                const float4* u4 = reinterpret_cast<const float4*>(usm + (b * 2 + side) * D + half * DH);
#if PARO_DQ_BATCH
                // every chunk's TMEM load issued before the single wait: one round trip
                uint32_t rawv[DH / 16][16];
#pragma unroll
                for (int ch = 0; ch < DH / 16; ++ch)
                    tmem_ld16(tmem + lane_base + C::TM_O + b * D + half * DH + ch * 16, rawv[ch]);
                ptx::tmem_ld_wait();
#endif
#pragma unroll
                for (int ch = 0; ch < DH / 16; ++ch) {
#if PARO_DQ_BATCH
                    const uint32_t (&raw)[16] = rawv[ch];
#else
                    uint32_t raw[16];
                    tmem_ld16(tmem + lane_base + C::TM_O + b * D + half * DH + ch * 16, raw);
                    ptx::tmem_ld_wait();
#endif
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 uu = u4[ch * 4 + q4];
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int j = q4 * 4 + hh * 2;
                            const uint64_t x2 =
                                PARO_DIAG_NOI2F ? pk(__int_as_float(raw[j]), __int_as_float(raw[j + 1])) : (PARO_I2F_FMA & 16) ? i2f2_fma((int32_t)raw[j], (int32_t)raw[j + 1], P.one) : pk(__int2float_rn((int32_t)raw[j]), __int2float_rn((int32_t)raw[j + 1]));
                            const uint64_t t2 = fma2(ss2, x2, hh ? pk(uu.z, uu.w) : pk(uu.x, uu.y));
                            acc[(ch * 16 + j) / 2] = fma2(acc[(ch * 16 + j) / 2], g2, t2);
                        }
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(bar(BR::OEMPTY + b));
                    ptx::mbar_arrive(bar(BR::PEMPTY + b));
                }
                PROF_T(te2);
                PROF_ADD(6, te2 - te1);
            };
            for (uint32_t t = 0; t < x.n; ++t, ++T) {
                const uint32_t s = T % NS, b = T & 1, ph = (T >> 1) & 1;
                const bool live = t < nmine;
                const uint32_t bj = live ? list[t] : 0u;
                PROF_T(tw0);
                mbar_wait3t(bar(BR::SFULL + b), ph, bar(BR::PEMPTY + b), ph ^ 1, bar(BR::KVFULL + s), (T / NS) & 1);
                ptx::tc_fence_after();
                PROF_T(tw1);
                PROF_ADD(0, tw1 - tw0);
                const float* meta =
                    reinterpret_cast<const float*>(smem + C::OFF_STAGE + s * C::STAGE_BYTES + 4 * C::KV_BYTES +
                                                   side * C::META_BYTES);
                uint8_t* prow = smem + C::OFF_P + (b * 2 + side) * C::P_BYTES + (r >> 3) * 512 + (r & 7) * 64;
                const uint32_t s_addr = tmem + lane_base + C::TM_S + b * C::S_COLS;
                float2* red_w = red + ((T & 1) * 4 + quad) * 2 + side;
                const float2* red_r = red + (T & 1) * 8 + side;
                const bool tail_tile = tail != 0 && live && bj == L.kb - 1;
                RowStatC* rs_w = rowstat + ((T & 1) * 2 + side) * 64 + r;
                const RowStatC* rs_r = rowstat + (T & 1) * 128;
                const uint8_t* qtile = smem + C::OFF_Q + (I & 1) * C::QBUF + side * C::QB_OFF;
                const uint8_t* ktile = smem + C::OFF_STAGE + s * C::STAGE_BYTES + side * C::KV_BYTES;
                float gamma, lo, pscale;
                softmax_step<D, true, P4>(s_addr, sq0, meta[0], meta[1], P.scale64, P.scale_log2,
                                      tail_tile ? tail : 64u, live, valid_row, st, P.p_qmax, red_w, red_r, rs_w, rs_r,
                                      side, qtile, ktile, prow, r, sq1, gamma, lo, pscale, half,
                                      reinterpret_cast<float4*>(smem + C::OFF_XCH),
                                      reinterpret_cast<uint16_t*>(smem + C::OFF_XLIST) + (warp - 4) * 512,
                                      bar(BR::RED), T & 1, prof, P.one);
                if (DUMP && dslot >= 0 && live) {
                    dump_row(P.dump, dslot, t, r, prow, (int)half * 2, 2);
                    if (r == 0 && half == 0)
                        dump_meta(P.dump, dslot, t, lo, pscale, bj);
                }
                PROF_T(tw2);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    ptx::mbar_arrive(bar(BR::SEMPTY + b));
                if (half == 0) {
                    const float vsc = meta[2];
                    rowmeta[(b * 2 + side) * 64 + r] =
                        make_float4(live ? gamma : 1.f, live ? pscale * vsc : 0.f, 0.f, live ? 1.f : 0.f);
                    // per-column offset term of this tile: (lo * vscale) * colsum[c]; exactly 0
                    // when idle (an idle side's meta slot is not loaded: stale smem, maybe NaN)
                    const float os = lo * vsc;
                    float* u = usm + (b * 2 + side) * D;
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        u[r + 64 * c] = live ? os * meta[4 + r + 64 * c] : 0.f;
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (PARO_PFULL_ALL || lane == 0) // every lane releases its own P codes / row meta / offsets
                    ptx::mbar_arrive(bar(BR::PFULL + b));
                PROF_T(tw3);
                PROF_ADD(4, tw3 - tw2);
                if (t > 0) // its PV was issued a whole step earlier
                    dequant(T - 1);
                PROF_ADD(7, 1);
            }
            if (x.n > 0)
                dequant(T - 1);
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(qempty(I)); // this warp no longer reads the item's Q tiles
            // row sum = the two halves' partial sums (same order in both warps)
            float* lw = lsm + (I & 1) * 256;
            lw[(half * 2 + side) * 64 + r] = st.l;
            ptx::named_bar_sync(2 + quad, 64);
            const float l = lw[side * 64 + r] + lw[(2 + side) * 64 + r];
            ++I;
            if (valid_row) {
                const uint32_t orig = perm_src(L.perm[x.h], qb * 64 + r);
                float4* dst = reinterpret_cast<float4*>(P.out + ((size_t)x.h * L.N + orig) * D + half * DH);
                if (l == 0.f) {
#pragma unroll
                    for (int c = 0; c < DH / 4; ++c)
                        dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
                    const float il = 1.0f / l;
#pragma unroll
                    for (int c = 0; c < DH / 4; ++c) {
                        float a0, a1, a2, a3;
                        upk(acc[2 * c], a0, a1);
                        upk(acc[2 * c + 1], a2, a3);
                        dst[c] = make_float4(a0 * il, a1 * il, a2 * il, a3 * il);
                    }
                }
                if (P.zeroed && half == 0)
                    P.zeroed[(size_t)x.h * L.N + orig] = l == 0.f ? 1 : 0;
            }
        }
#ifdef PARO_K3_PROF
        if (lane == 0) {
            for (int i = 0; i < 8; ++i)
                atomicAdd(&g_prof[i], prof[i]);
            for (int i = 8; i < 18; ++i)
                atomicAdd(&g_prof[8 + i], prof[i]);
        }
#endif
    } else {
        // warps 2-3 (d = 128): with INT4 V, warp 2 unpacks side A's and warp 3 side B's
        // nibble-packed V tile of every step from the staging buffer (their SMSPs,
        // not the producer's, carry the work); both arrive on VFULL every step
        ptx::setmaxnreg_dec<C::REG_LOW>();
        const uint32_t side = (uint32_t)warp - 2;
        uint32_t T = 0;
        for (uint32_t rr = 0;; ++rr) {
            if (!PARO_DYNAMIC && rr >= rounds)
                break;
            const int it = next_item(rr, true);
            __syncwarp();
            if (lane == 0)
                release_item(rr);
            if (it < 0) {
                if (PARO_DYNAMIC)
                    break;
                continue;
            }
            const Item x = load_item(L, (uint32_t)it);
            if (!PACKED) {
                T += x.n;
                continue;
            }
            const uint32_t nmine = side ? x.nb : x.na;
            for (uint32_t t = 0; t < x.n; ++t, ++T) {
                const uint32_t s = T % NS;
                // every step waits for its stage, even with no tile on this side: a warp
                // must not arrive on VFULL(s) for step T + NS while step T's phase is open
                ptx::mbar_wait(bar(BR::KVFULL + s), (T / NS) & 1);
                if (t < nmine && !PARO_DIAG_NOUNPACK) {
                    unpack_v_tile<D>(smem + C::OFF_VPK + (s * 2 + side) * C::VPK_BYTES,
                                     smem + C::OFF_STAGE + s * C::STAGE_BYTES + (2 + side) * C::KV_BYTES, lane);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                }
                if (lane == 0)
                    ptx::mbar_arrive(bar(BR::VFULL + s));
            }
        }
    }

#ifdef PARO_K3_PROF
    if (threadIdx.x == 0) { // CTA lifetime (globaltimer ns): sum, and the latest end
        atomicAdd(&g_profq[6], (unsigned long long)(ptx::globaltimer() - cta_t0));
        atomicMax(&g_profq[7], (unsigned long long)ptx::globaltimer());
        atomicMin(&g_profq[5], (unsigned long long)cta_t0);
    }
#endif
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1)
        ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// Debug / parity: int32 S_g tiles for a list of (h, qb, bj) through the same
// TMA maps, smem swizzle, descriptors and M=64 tcgen05 issue as K3; even q-blocks
// go to TMEM lane offset 0 (side A), odd ones to lane offset 16 (side B), so
// both placements are checked. One CTA (4 warps) per tile; writes
// S[tile][g][row][col].
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128, 1)
    k3_debug_qk(const __grid_constant__ LayerDev L, const __grid_constant__ CUtensorMap tm_q,
                const __grid_constant__ CUtensorMap tm_q32, const __grid_constant__ CUtensorMap tm_k,
                const uint32_t* __restrict__ tiles, int32_t* S) {
    using C = K3Cfg<D>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = ptx::smem_u32(smem);
    // M128: 2 KB slots [0 | Q0 | 0 | Q1 | 0 | K] -- side A's operand [Q0; 0; Q1; 0] at slot 1,
    // side B's [0; Q0; 0; Q1] at slot 0 (after an A-side MMA, as K3 accumulates B onto A);
    // otherwise [Q | K]
    const uint32_t sq = sbase + (C::M128 ? C::HALF : 0u), sk = sbase + (C::M128 ? 5 * C::HALF : C::QT_BYTES);
    const uint32_t bar_ld = sk + C::KV_BYTES, bar_mma = bar_ld + 8, tptr = bar_ld + 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t h = tiles[3 * blockIdx.x], qb = tiles[3 * blockIdx.x + 1], bj = tiles[3 * blockIdx.x + 2];
    const uint32_t side = qb & 1;
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar_ld, 1);
        ptx::mbar_init(bar_mma, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0)
        ptx::tmem_alloc<128>(tptr);
    if (C::M128) { // zero slots 0, 2, 4
        for (uint32_t i = threadIdx.x; i < 3 * C::HALF / 16; i += 128) {
            const uint32_t slot = 2 * (i / (C::HALF / 16)), off = (i % (C::HALF / 16)) * 16;
            *reinterpret_cast<uint4*>(smem + slot * C::HALF + off) = make_uint4(0, 0, 0, 0);
        }
        ptx::fence_proxy_async_smem();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (tptr - sbase));
    if (threadIdx.x == 0) {
        const int32_t row0 = (int32_t)(h * L.kb2 * 64);
        ptx::mbar_arrive_expect_tx(bar_ld, C::QT_BYTES + C::KV_BYTES);
        if (C::M128) {
            ptx::tma_load_2d(sq, &tm_q32, 0, row0 + (int32_t)qb * 64, bar_ld);
            ptx::tma_load_2d(sq + 2 * C::HALF, &tm_q32, 0, row0 + (int32_t)qb * 64 + 32, bar_ld);
        } else {
            ptx::tma_load_2d(sq, &tm_q, 0, row0 + (int32_t)qb * 64, bar_ld);
        }
        ptx::tma_load_2d(sk, &tm_k, 0, row0 + (int32_t)bj * 64, bar_ld);
        ptx::mbar_wait(bar_ld, 0);
        ptx::tc_fence_after();
        if (C::M128) {
            issue_qk128(tmem, sq, sk, true);
            if (side)
                issue_qk128(tmem, sq - C::HALF, sk, false);
        } else {
            issue_qk<D>(tmem + (side ? C::LANE16 : 0u), sq, sk);
        }
        ptx::mma_commit(bar_mma);
    }
    ptx::mbar_wait(bar_mma, 0);
    ptx::tc_fence_after();
    const uint32_t row = C::M128 ? (warp >> 1) * 32 + lane : warp * 16 + (lane & 15);
    const uint32_t my_side = C::M128 ? (uint32_t)warp & 1 : (uint32_t)lane >> 4;
    for (int g = 0; g < C::G; ++g)
        for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t raw[32];
            ptx::tmem_ld32(tmem + ((warp * 32) << 16) + g * 64 + h2 * 32, raw);
            ptx::tmem_ld_wait();
            if (my_side == side) {
                int32_t* dst = S + (((size_t)blockIdx.x * C::G + g) * 64 + row) * 64 + h2 * 32;
                for (int j = 0; j < 32; ++j)
                    dst[j] = (int32_t)raw[j];
            }
        }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0)
        ptx::tmem_dealloc<128>(tmem);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static void init_watchdog() {
    static bool done = false;
    if (done)
        return;
    done = true;
    if (const char* e = getenv("PARO_WATCHDOG_S")) {
        const unsigned long long ns = (unsigned long long)(atof(e) * 1e9);
        cudaMemcpyToSymbol(ptx::g_watchdog_ns, &ns, sizeof(ns));
    }
}

template <int D>
static cudaError_t launch_k3_t(const K3Params& p, const CUtensorMap& tq, const CUtensorMap& tk,
                               const CUtensorMap& tv, const CUtensorMap& tvp, const CUtensorMap& tq32, int grid,
                               cudaStream_t st) {
    init_watchdog();
    const uint32_t smem = K3Cfg<D>::SMEM_BYTES;
    // d=64 with INT4 P codes: its own instantiation with the monotone exact extremes and
    // redux.sync group extremes (c3 K3 2.63 -> 2.55 ms; at INT8 P they cost c2 2-3%)
    auto kern = p.L.v_packed ? (p.dump.slot ? k3_attention<D, true, true> : k3_attention<D, false, true>)
                             : (p.dump.slot ? k3_attention<D, true, false> : k3_attention<D, false, false>);
    // INT4 P: its own instantiations -- at d=64 with the monotone exact extremes
    // and redux group extremes, at d=128 without the S-group-cancellation arithmetic
    if (p.p_qmax == 15.0f)
        kern = p.L.v_packed ? (p.dump.slot ? k3_attention<D, true, true, true> : k3_attention<D, false, true, true>)
                            : (p.dump.slot ? k3_attention<D, true, false, true> : k3_attention<D, false, false, true>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    // two CTAs per SM at d=64 need the largest shared-memory carveout (-1: driver default)
#ifndef PARO_K3_CARVEOUT
#define PARO_K3_CARVEOUT 100
#endif
    if (PARO_K3_CARVEOUT >= 0) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, PARO_K3_CARVEOUT);
        if (e != cudaSuccess)
            return e;
    }
    kern<<<grid, K3Cfg<D>::THREADS, smem, st>>>(p, tq, tk, tv, tvp, tq32);
    return cudaGetLastError();
}

cudaError_t launch_k3_64(const K3Params& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         int num_sms, cudaStream_t st);
cudaError_t launch_k3_dec(const K3Params& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          int num_sms, cudaStream_t st);

cudaError_t launch_k3(const LayerDev& L, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const CUtensorMap& tvp, const CUtensorMap& tq32, double scale, int pv_bits, float* out, uint8_t* zeroed, int num_sms, cudaStream_t st,
                      uint32_t head_begin, uint32_t head_count, bool chunked, const K3Dump* dump) {
    if (head_count == 0)
        return cudaSuccess;
    K3Params p;
    p.L = L;
    p.one = 1;
    p.scale64 = scale;
    p.scale_log2 = (float)(scale * kLog2e);
    p.p_qmax = pv_bits == 4 ? 15.0f : 255.0f;
    p.out = out;
    p.zeroed = zeroed;
    p.order = (chunked ? L.order_chunk : L.order) + (size_t)head_begin * L.np;
    p.n_items = head_count * L.np;
    p.stats = nullptr;
    p.dump = dump ? *dump : K3Dump{nullptr, nullptr, nullptr, 0};
    p.work_counter = L.work_counter;
    if (PARO_DYNAMIC) {
        const cudaError_t e = cudaMemsetAsync(L.work_counter, 0, sizeof(uint32_t), st);
        if (e != cudaSuccess)
            return e;
    }
#ifdef PARO_K3_STATS
    static unsigned long long* dstats = nullptr;
    if (!dstats) {
        cudaMalloc(&dstats, 32);
        cudaMemset(dstats, 0, 32);
    }
    p.stats = dstats;
    if (getenv("PARO_K3_STATS_PRINT")) {
        unsigned long long h[3];
        cudaDeviceSynchronize();
        cudaMemcpy(h, dstats, 24, cudaMemcpyDeviceToHost);
        fprintf(stderr, "[k3 stats] warp-steps %llu exact-path %llu risky-groups %llu\n", h[0], h[1], h[2]);
    }
#endif
#ifdef PARO_K3_PROF
    static unsigned long long gridDim_last = 1;
    if (getenv("PARO_K3_PROF_PRINT")) {
        unsigned long long h[32];
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(h, g_prof, sizeof(h));
        const double n = (double)(h[7] ? h[7] : 1);
        fprintf(stderr,
                "[k3 prof] compute warp/step: wait %.0f pass1 %.0f reduce %.0f pass2 %.0f exact+publish %.0f "
                "dequant-wait %.0f dequant %.0f (warp-steps %llu)\n",
                h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[4] / n, h[5] / n, h[6] / n, h[7]);
        fprintf(stderr, "[k3 prof] mma/step: wait KV+S %.0f wait P+O %.0f (steps %llu)\n", (double)h[12] / h[15],
                (double)h[13] / h[15], h[15]);
        fprintf(stderr, "[k3 prof] exact path: entries %llu, candidates %.0f, elements %.0f cycles/entry\n", h[18],
                (double)h[16] / (h[18] ? h[18] : 1), (double)h[17] / (h[18] ? h[18] : 1));
        fprintf(stderr, "[k3 prof] d=128 pass1: scan %.0f exchange %.0f dp4a %.0f rescan %.0f tail %.0f (rescans %.4f)\n",
                h[16] / n, h[17] / n, h[18] / n, h[19] / n, h[20] / n, h[21] / n);
        {
            unsigned long long q[8];
            cudaMemcpyFromSymbol(q, g_profq, sizeof(q));
            const double ns = (double)(h[23] ? h[23] : 1);
            fprintf(stderr, "[k3 prof] d=128 unsure warp-steps: loose %llu, after the tight re-test %llu\n", q[0], q[1]);
            fprintf(stderr, "[k3 prof] CTA lifetime: mean %.1f us, kernel span %.1f us (first start to last end)\n",
                    q[6] / 1e3 / (double)gridDim_last, (q[7] - q[5]) / 1e3);
            memset(q, 0, sizeof(q));
            q[5] = ~0ull;
            cudaMemcpyToSymbol(g_profq, q, sizeof(q));
        }
        fprintf(stderr, "[k3 prof] d=64 softmax per warp-step: item-queue wait %.0f, item-end LEMPTY wait %.0f\n", h[24] / n, h[25] / n);
        fprintf(stderr, "[k3 prof] d=64 reduce: to-barrier %.0f barrier %.0f after %.0f; arrival spread %.0f per CTA step\n",
                h[19] / n, h[20] / n, h[21] / n, (double)h[22] / (h[23] ? h[23] : 1));
        memset(h, 0, sizeof(h));
        cudaMemcpyToSymbol(g_prof, h, sizeof(h));
    }
#endif
    // d = 64 multi-slot kernel (attention64_kernel.cu), opt-in while it is measured (PARO_K3_SLOTS=1)
    static const bool slots64 = getenv("PARO_K3_SLOTS") && atoi(getenv("PARO_K3_SLOTS")) != 0;
    if (L.D == 64 && slots64 && !L.v_packed)
        return launch_k3_64(p, tq, tk, tv, num_sms, st);
    // d = 64 decoupled softmax / quantizer layout (attention_dec_kernel.cu); packed INT4 V stays here
    static const bool dec64 = getenv("PARO_K3_DEC") && atoi(getenv("PARO_K3_DEC")) != 0;
    if (L.D == 64 && dec64 && !L.v_packed && PARO_DYNAMIC)
        return launch_k3_dec(p, tq, tk, tv, num_sms, st);
    const uint32_t slots = (uint32_t)num_sms * (L.D == 64 ? K3Cfg<64>::MINB : K3Cfg<128>::MINB);
    const int grid = (int)(p.n_items < slots ? p.n_items : slots);
#ifdef PARO_K3_PROF
    gridDim_last = (unsigned long long)grid;
#endif
    return L.D == 64 ? launch_k3_t<64>(p, tq, tk, tv, tvp, tq32, grid, st)
                     : launch_k3_t<128>(p, tq, tk, tv, tvp, tq32, grid, st);
}

cudaError_t launch_debug_qk(const LayerDev& L, const CUtensorMap& tq, const CUtensorMap& tq32, const CUtensorMap& tk,
                            uint32_t n_tiles,
                            const uint32_t* tiles, int32_t* S, cudaStream_t st) {
    if (n_tiles == 0)
        return cudaSuccess;
    if (L.D == 64) {
        const uint32_t smem = (K3Cfg<64>::M128 ? 5 * K3Cfg<64>::HALF : K3Cfg<64>::QT_BYTES) + K3Cfg<64>::KV_BYTES + 64;
        cudaFuncSetAttribute(k3_debug_qk<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k3_debug_qk<64><<<n_tiles, 128, smem, st>>>(L, tq, tq32, tk, tiles, S);
    } else {
        const uint32_t smem = K3Cfg<128>::QT_BYTES + K3Cfg<128>::KV_BYTES + 64;
        cudaFuncSetAttribute(k3_debug_qk<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k3_debug_qk<128><<<n_tiles, 128, smem, st>>>(L, tq, tq32, tk, tiles, S);
    }
    return cudaGetLastError();
}

} // namespace paro
