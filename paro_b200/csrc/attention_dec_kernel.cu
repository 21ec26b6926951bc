// attention_dec_kernel.cu -- K3 at d = 64 (c1/c2/c3), decoupled layout: the
// softmax warps never wait for each other.
//
// Semantics are those of attention_kernel.cu (the reference stream_engine,
// attention.cpp:84-254, with the restated INT8-QK prologue): per kept (q-block,
// k-block) tile S = Q.K^T (int32, tcgen05 kind::i8, TMEM), exact fp64 row
// extremes and running max, p = exp2 of exact integer differences, one unsigned
// P group per tile (:201-228) with bit-exact codes (two perturbed variants + the
// fp64 boundary path), P.V (u8 x s8 -> s32, tcgen05) dequantised into fp32
// accumulators (:229-238), O = acc / l stored at the ORIGINAL token row.
//
// Why a second layout. In attention_kernel.cu the four softmax warps of a CTA
// meet at a named barrier every step (the P group spans the tile's 64 rows, which
// the M = 64 TMEM layout spreads over all four lane quadrants, i.e. four warps on
// four SM sub-partitions). Measured with phase timers at c2: the four warps START
// a step ~1,100 cycles apart (contention noise from the co-resident CTA and the
// epilogue warps on each sub-partition), so every step pays the slowest of four.
// Here the only per-tile cross-warp dependency moves off the softmax warps:
//
//   softmax warps (warpgroup 1, one per quadrant): pass 1 (integer row extremes
//     -> exact fp64 logits / running max, published with the row's fast p
//     extremes), pass 2 (p = exp2 of exact integer differences, row sum) and
//     tcgen05.st of the row's 64 p values back over its S columns -- then the
//     next step. No barrier among the four.
//   quantizer warps (warpgroup 2, one per quadrant), one step behind: wait until
//     all four softmax warps published step t, reduce the tile's P-group lo/hi,
//     read p from TMEM, write the P codes (exact boundary path included), the
//     per-column offsets, arrive for the P.V MMA, then dequantise step t-1's
//     int32 P.V into the row's fp32 accumulators.
//
// TMEM: a ring of four 64-column buffers per CTA. Step t's buffer holds S (MMA),
// then p (softmax), then the int32 P.V (MMA, issued once the quantizers read p),
// and is released after the quantizers' dequant -- so QK runs up to four steps
// ahead of the dequant and the softmax warps rarely wait for S. Work items are
// pairs of q-blocks (A: TMEM lanes 0-15 of each quadrant, B: lanes 16-31) taken
// dynamically in K2's L2-grouped LPT order, as in attention_kernel.cu.
//
// Warps (384 threads, 2 CTAs/SM): 0 TMA producer, 1 TMEM allocator + MMA issuer
// (polls both the QK and the P.V streams), 2-3 idle (their registers go to the
// quantizers via setmaxnreg), 4-7 softmax, 8-11 quantizer + dequant.
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

// The four roles' hot loops share each sub-partition's instruction cache: the
// per-half / per-chunk loops stay rolled (ncu: no_instruction stalls otherwise)
#ifndef PARO_DEC_UNROLL
#define PARO_DEC_UNROLL 1
#endif
constexpr int kDecUnroll = PARO_DEC_UNROLL;

struct KDec {
    static constexpr int D = 64;
    static constexpr int NS = 3;  // K/V stages
    static constexpr int NB = 3;  // TMEM buffers (S -> p -> P.V), 64 columns each; columns 192-255: the accumulators
    static constexpr uint32_t TM_ACC = 192;
    static constexpr int THREADS = 512;
    static constexpr int MINB = 2;
    static constexpr uint32_t REG_LAUNCH = (65536 / (THREADS * MINB)) / 8 * 8; // 64
    static constexpr uint32_t REG_CTRL = 24;
#ifndef PARO_DEC_MMA_NS
#define PARO_DEC_MMA_NS 64
#endif
#ifndef PARO_DEC_RS3
#define PARO_DEC_RS3 1
#endif
#ifndef PARO_DEC_REG_SOFT
#define PARO_DEC_REG_SOFT 96
#endif
#ifndef PARO_DEC_REG_QUANT
#define PARO_DEC_REG_QUANT 80
#endif
    // warpgroup 0's release goes to the others: 128 x (24 + 96 + 80 + 56) = 512 x 64
    static constexpr uint32_t REG_SOFT = PARO_DEC_REG_SOFT;
    static constexpr uint32_t REG_QUANT = PARO_DEC_REG_QUANT;
    static constexpr uint32_t REG_EPI = 4 * REG_LAUNCH - REG_CTRL - REG_SOFT - REG_QUANT;
    static constexpr uint32_t QT_BYTES = 64 * 64, KV_BYTES = 64 * 64;
    static constexpr uint32_t META_BYTES = (4 + 64) * 4;
    static constexpr uint32_t STAGE_BYTES = (4 * KV_BYTES + 2 * META_BYTES + 1023) / 1024 * 1024;
    static constexpr uint32_t P_BYTES = 64 * 64;
    static constexpr uint32_t OFF_Q = 0;                                   // [2 item][A, B]
    static constexpr uint32_t OFF_STAGE = 4 * QT_BYTES;                    // K_A, K_B, V_A, V_B, meta_A, meta_B
    static constexpr uint32_t OFF_P = OFF_STAGE + NS * STAGE_BYTES;        // [2 parity][2 side] P codes
    static constexpr uint32_t OFF_U = OFF_P + 4 * P_BYTES;                 // [NB][2 side][64] column offsets
    static constexpr uint32_t OFF_RM = OFF_U + NB * 2 * 64 * 4;            // [NB][2 side][64] float4 row meta
    // row statistics / P extremes ring: RS deep. RS = NB needs no quantizer -> softmax hand-back (the
    // S buffer ring already keeps the softmax within NB steps of the epilogue); RS = 2 uses QDONE
    static constexpr int RS = PARO_DEC_RS3 ? NB : 2;
    static constexpr uint32_t OFF_RED = OFF_RM + NB * 2 * 64 * 16;         // [RS][4 quad][2 side] float2
    static constexpr uint32_t OFF_ROWSTAT = OFF_RED + RS * 4 * 2 * 8;      // [RS][2 side][64] RowStatD
    static constexpr uint32_t OFF_XLIST = OFF_ROWSTAT + RS * 2 * 64 * 48;  // [4 quantizer warps][512] u16
    static constexpr uint32_t OFF_BAR = OFF_XLIST + 4 * 512 * 2;
    static constexpr uint32_t NBAR = 34;
    static constexpr uint32_t OFF_TMEMPTR = OFF_BAR + NBAR * 8;
    static constexpr uint32_t SMEM = OFF_TMEMPTR + 16;
    static constexpr uint32_t IDESC_QK = ptx::idesc_i8(true, true, false, false, 64, 64);
    static constexpr uint32_t IDESC_PV = ptx::idesc_i8(false, true, false, true, 64, 64);
    static constexpr uint32_t LANE16 = 16u << 16;
};
static_assert(KDec::SMEM * 2 <= 227 * 1024, "two CTAs per SM");
static_assert(KDec::REG_EPI >= 56, "epilogue registers");

// barrier indices
enum : uint32_t {
    DB_QFULL = 0,     // [2] Q tiles of an item (by item parity)
    DB_QEMPTY = 2,    // [2] MMA commit after the item's last QK + 4 quantizer warps (exact path reads Q)
    DB_KVFULL = 4,    // [NS]
    DB_KVEMPTY = 7,   // [NS] MMA commit after the step's P.V
    DB_SFULL = 10,    // [NB] QK of the step landed in its buffer
    DB_RED = 13,      // [RS] 4 softmax warps: row stats, P extremes and p of the step published
    DB_QDONE = 16,    // [2] (RS = 2 only) 4 quantizer warps: done with the step's row stats / extremes
    DB_PFULL = 18,    // [4] 4 quantizer warps: P codes, column offsets and row meta of the step written.
                      //     Four deep: the epilogue tests it after the quantizers may have run two steps
                      //     further (a two-deep ring would have wrapped its phase parity)
    DB_PEMPTY = 22,   // [2] MMA commit after the step's P.V (P tile free)
    DB_OFULL = 24,    // [NB] P.V of the step landed in its buffer
    DB_BEMPTY = 27,   // [NB] 4 epilogue warps: the step's P.V read (buffer free for QK of step + NB)
    DB_ITEMFULL = 30, // [2]
    DB_ITEMEMPTY = 32 // [2]
};
static_assert(DB_ITEMEMPTY + 2 <= KDec::NBAR, "barrier block");

// per row and step, written by the softmax warp, read by the quantizers
struct RowStatD { // 48 bytes
    double tmin, tmax, m; // exact fp64 extreme logits of the row's tile and the running max after it
    float pmin, pmax;     // fast-path p at the extremes (INF / 0 when the row is not valid this step)
    float gamma, l;       // rescale factor of the step and the row sum after it
    int32_t smax;         // integer row max of S (the fast path's exact-difference origin)
    uint32_t valid;
};
static_assert(sizeof(RowStatD) == 48, "RowStatD layout");

__device__ __forceinline__ uint64_t ddesc_k(uint32_t saddr) { return ptx::smem_desc(saddr, 16, 512, ptx::kSwizzle64B); }
__device__ __forceinline__ uint64_t ddesc_v(uint32_t saddr) {
    return ptx::smem_desc(saddr, 512 * 8, 512, ptx::kSwizzle64B);
}

// a wait that is usually already satisfied: one non-blocking probe first (a
// suspending try_wait costs ~90 cycles even on a completed phase)
__device__ __forceinline__ void dwait(uint32_t b, uint32_t p) {
    if (!ptx::mbar_test(b, p))
        ptx::mbar_wait(b, p);
}

template <bool DUMP>
__global__ void __launch_bounds__(KDec::THREADS, KDec::MINB)
    k3_attention_dec(const __grid_constant__ K3Params P, const __grid_constant__ CUtensorMap tm_q,
                     const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v) {
    using C = KDec;
    constexpr int NS = C::NS, NB = C::NB;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bar0 = sbase + C::OFF_BAR;
    auto bar = [&](uint32_t i) { return bar0 + 8 * i; };
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const LayerDev& L = P.L;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar(DB_QFULL + i), 1);
            ptx::mbar_init(bar(DB_QEMPTY + i), 1 + 4);
            ptx::mbar_init(bar(DB_QDONE + i), 4);
            ptx::mbar_init(bar(DB_PEMPTY + i), 1);
            ptx::mbar_init(bar(DB_ITEMFULL + i), 1);
            ptx::mbar_init(bar(DB_ITEMEMPTY + i), 1 + 4 + 4 + 4); // MMA, softmax, quantizer, epilogue warps
        }
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(bar(DB_KVFULL + s), 1);
            ptx::mbar_init(bar(DB_KVEMPTY + s), 1);
        }
        for (int i = 0; i < 4; ++i)
            ptx::mbar_init(bar(DB_PFULL + i), 4);
        for (int i = 0; i < C::RS; ++i)
            ptx::mbar_init(bar(DB_RED + i), 4);
        for (int b = 0; b < NB; ++b) {
            ptx::mbar_init(bar(DB_SFULL + b), 1);
            ptx::mbar_init(bar(DB_OFULL + b), 1);
            ptx::mbar_init(bar(DB_BEMPTY + b), 4);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1)
        ptx::tmem_alloc<256>(sbase + C::OFF_TMEMPTR); // NB x 64 ring + 64 accumulator columns
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::OFF_TMEMPTR);

    volatile int* ring = reinterpret_cast<volatile int*>(smem + C::OFF_TMEMPTR + 8);
    auto next_item = [&](uint32_t k) -> int { // consumers (blocking): the CTA's k-th item, -1 = done
        ptx::mbar_wait(bar(DB_ITEMFULL + (k & 1)), (k >> 1) & 1);
        return ring[k & 1];
    };
    auto stage = [&](uint32_t s) { return sbase + C::OFF_STAGE + s * C::STAGE_BYTES; };
    auto qbuf = [&](uint32_t i) { return sbase + C::OFF_Q + (i & 1) * 2 * C::QT_BYTES; };
    RowStatD* rowstat = reinterpret_cast<RowStatD*>(smem + C::OFF_ROWSTAT);
    float2* red = reinterpret_cast<float2*>(smem + C::OFF_RED);
    float* usm = reinterpret_cast<float*>(smem + C::OFF_U);

    if (warp < 4) {
        ptx::setmaxnreg_dec<C::REG_CTRL>();
        if (warp == 0 && lane == 0) {
            // -------------------------------------------------------- producer
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
            uint32_t T = 0, I = 0;
            for (uint32_t r = 0;; ++r) {
                const uint32_t idx = atomicAdd(P.work_counter, 1u);
                const int it = idx < P.n_items ? (int)P.order[idx] : -1;
                mbar_wait_lazy(bar(DB_ITEMEMPTY + (r & 1)), ((r >> 1) & 1) ^ 1);
                ring[r & 1] = it;
                ptx::mbar_arrive(bar(DB_ITEMFULL + (r & 1)));
                if (it < 0)
                    break;
                const Item x = load_item(L, (uint32_t)it);
                const uint16_t* la = L.items + ((size_t)x.h * L.kb + x.qa) * L.kb;
                const uint16_t* lb = L.items + ((size_t)x.h * L.kb + (x.qb != 0xffffu ? x.qb : 0)) * L.kb;
                const int32_t row0 = (int32_t)(x.h * L.kb2 * 64);
                mbar_wait_lazy(bar(DB_QEMPTY + (I & 1)), ((I >> 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(bar(DB_QFULL + (I & 1)), (x.qb != 0xffffu ? 2 : 1) * C::QT_BYTES);
                ptx::tma_load_2d(qbuf(I), &tm_q, 0, row0 + (int32_t)x.qa * 64, bar(DB_QFULL + (I & 1)));
                if (x.qb != 0xffffu)
                    ptx::tma_load_2d(qbuf(I) + C::QT_BYTES, &tm_q, 0, row0 + (int32_t)x.qb * 64,
                                     bar(DB_QFULL + (I & 1)));
                for (uint32_t t = 0; t < x.n; ++t, ++T) {
                    const uint32_t s = T % NS;
                    mbar_wait_lazy(bar(DB_KVEMPTY + s), ((T / NS) & 1) ^ 1);
                    const bool ha = t < x.na, hb = t < x.nb;
                    ptx::mbar_arrive_expect_tx(bar(DB_KVFULL + s), (ha + hb) * (2 * C::KV_BYTES + C::META_BYTES));
#pragma unroll
                    for (int side = 0; side < 2; ++side) {
                        if (side ? hb : ha) {
                            const uint32_t bj = side ? lb[t] : la[t];
                            ptx::tma_load_2d(stage(s) + side * C::KV_BYTES, &tm_k, 0, row0 + (int32_t)bj * 64,
                                             bar(DB_KVFULL + s));
                            ptx::tma_load_2d(stage(s) + (2 + side) * C::KV_BYTES, &tm_v, 0, row0 + (int32_t)bj * 64,
                                             bar(DB_KVFULL + s));
                            ptx::bulk_load(stage(s) + 4 * C::KV_BYTES + side * C::META_BYTES,
                                           L.meta + ((size_t)x.h * L.kb2 + bj) * meta_stride(64), C::META_BYTES,
                                           bar(DB_KVFULL + s));
                        }
                    }
                }
                ++I;
            }
        } else if (warp == 1 && lane == 0) {
            // ----------------------------------------------------- MMA issuer
            // Two in-order streams polled without blocking: QK of step Tq (needs its
            // K/V stage, its TMEM buffer back from the dequant of step Tq - 4 and, at an
            // item's first step, the item's Q tiles) and P.V of step Tp < Tq (needs the
            // quantizers' P codes). Blocking on one would stall the other.
            uint32_t Tq = 0, Tp = 0, rq = 0, Iq = 0, tq = 0, pvf = 0;
            bool have = false, done = false;
            Item xq{};
            unsigned long long prof[4] = {0, 0, 0, 0};
            for (;;) {
                bool prog = false;
                if (!have && !done && ptx::mbar_test(bar(DB_ITEMFULL + (rq & 1)), (rq >> 1) & 1)) {
                    const int it = ring[rq & 1];
                    ptx::mbar_arrive(bar(DB_ITEMEMPTY + (rq & 1)));
                    ++rq;
                    if (it < 0) {
                        done = true;
                    } else {
                        xq = load_item(L, (uint32_t)it);
                        tq = 0;
                        have = true;
                    }
                    prog = true;
                }
                if (have && xq.n == 0) { // nothing to issue: the item's Q buffer is free once the quantizers are
                    ptx::mma_commit(bar(DB_QEMPTY + (Iq & 1)));
                    ++Iq;
                    have = false;
                    prog = true;
                } else if (have && ptx::mbar_test(bar(DB_BEMPTY + Tq % NB), ((Tq / NB) & 1) ^ 1) &&
                           ptx::mbar_test(bar(DB_KVFULL + Tq % NS), (Tq / NS) & 1) &&
                           (tq > 0 || ptx::mbar_test(bar(DB_QFULL + (Iq & 1)), (Iq >> 1) & 1))) {
                    ptx::tc_fence_after();
                    const uint32_t s = Tq % NS, tb = tmem + (Tq % NB) * 64;
                    const bool ha = tq < xq.na, hb = tq < xq.nb;
#pragma unroll
                    for (int side = 0; side < 2; ++side) {
                        if (side ? hb : ha) {
                            const uint32_t sq = qbuf(Iq) + side * C::QT_BYTES, sk = stage(s) + side * C::KV_BYTES;
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                ptx::mma_i8(tb + (side ? C::LANE16 : 0u), ddesc_k(sq + kk * 32), ddesc_k(sk + kk * 32),
                                            C::IDESC_QK, kk);
                        }
                    }
                    ptx::mma_commit(bar(DB_SFULL + Tq % NB));
                    const uint32_t sh = 2 * (Tq % NB);
                    pvf = (pvf & ~(3u << sh)) | ((ha ? 1u : 0u) << sh) | ((hb ? 2u : 0u) << sh);
                    ++Tq;
                    if (++tq == xq.n) {
                        ptx::mma_commit(bar(DB_QEMPTY + (Iq & 1)));
                        ++Iq;
                        have = false;
                    }
                    prog = true;
                }
                if (Tp < Tq && ptx::mbar_test(bar(DB_PFULL + (Tp & 3)), (Tp >> 2) & 1)) {
                    ptx::tc_fence_after();
                    const uint32_t s = Tp % NS, b = Tp & 1, tb = tmem + (Tp % NB) * 64;
                    const uint32_t f = pvf >> (2 * (Tp % NB));
#pragma unroll
                    for (int side = 0; side < 2; ++side) {
                        if ((f >> side) & 1u) {
                            const uint32_t sp = sbase + C::OFF_P + (b * 2 + side) * C::P_BYTES;
                            const uint32_t sv = stage(s) + (2 + side) * C::KV_BYTES;
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                ptx::mma_i8(tb + (side ? C::LANE16 : 0u), ddesc_k(sp + kk * 32),
                                            ddesc_v(sv + kk * 32 * 64), C::IDESC_PV, kk);
                        }
                    }
                    ptx::mma_commit(bar(DB_OFULL + Tp % NB));
                    ptx::mma_commit(bar(DB_KVEMPTY + s));
                    ptx::mma_commit(bar(DB_PEMPTY + b));
                    ++Tp;
                    prog = true;
                }
                if (done && !have && Tp == Tq)
                    break;
                if (!prog)
                    __nanosleep(PARO_DEC_MMA_NS);
            }
            (void)prof;
        }
    } else if (warp < 8) {
        // ------------------------------------------------------------ softmax
        if (C::REG_SOFT > C::REG_LAUNCH)
            ptx::setmaxnreg_inc<(C::REG_SOFT > C::REG_LAUNCH ? C::REG_SOFT : C::REG_LAUNCH)>();
        const uint32_t quad = warp & 3;
        const uint32_t side = lane >> 4;
        const uint32_t r = quad * 16 + (lane & 15); // row within its q-block
        const uint32_t lane_base = (quad * 32) << 16;
        const uint32_t tail = L.N & 63;
        uint32_t T = 0;
        unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t rr = 0;; ++rr) {
            const int it = next_item(rr);
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(DB_ITEMEMPTY + (rr & 1)));
            if (it < 0)
                break;
            const Item x = load_item(L, (uint32_t)it);
            const bool has_qb = side ? x.qb != 0xffffu : true;
            const uint32_t qb = side ? (has_qb ? x.qb : 0u) : x.qa;
            const uint32_t nmine = side ? x.nb : x.na;
            const uint16_t* list = L.items + ((size_t)x.h * L.kb + qb) * L.kb;
            const bool valid_row = has_qb && qb * 64 + r < L.N && qb * 64 + r >= L.dp; // dense rows: K4
            const float sq = L.qsc[(size_t)x.h * L.kb2 + qb];
            RowState st{-INFINITY, 0.f, -INFINITY};
            if (L.dp && valid_row) { // continue from K4's dense-prefix state
                const size_t srow = (size_t)x.h * L.kb2 * 64 + qb * 64 + r;
                st.m64 = L.init_m[srow];
                st.m32 = (float)(st.m64 * kLog2e);
                st.l = L.init_l[srow];
            }
            for (uint32_t t = 0; t < x.n; ++t, ++T) {
                const uint32_t s = T % NS, b = T % NB, par = T & 1;
                const uint32_t rsl = T % C::RS, rsp = (T / C::RS) & 1; // row-stat ring slot, phase parity
                const bool live = t < nmine;
                const bool valid = live && valid_row;
                const uint32_t bj = live ? list[t] : 0u;
                PROF_T(tw0);
                // S of the step; the step's K/V stage (meta); the quantizers are done with step T - 2's stats
#ifdef PARO_K3_PROF
                if (C::RS == 2)
                    ptx::mbar_wait(bar(DB_QDONE + par), ((T >> 1) & 1) ^ 1);
                PROF_T(twa);
                ptx::mbar_wait(bar(DB_SFULL + b), (T / NB) & 1);
                PROF_T(twb);
                PROF_ADD(3, twa - tw0);
                PROF_ADD(4, twb - twa);
#endif
                if (C::RS == 2)
                    dwait(bar(DB_QDONE + par), ((T >> 1) & 1) ^ 1);
                dwait(bar(DB_SFULL + b), (T / NB) & 1);
                dwait(bar(DB_KVFULL + s), (T / NS) & 1);
                ptx::tc_fence_after();
                PROF_T(tw1);
                const float* meta = reinterpret_cast<const float*>(smem + C::OFF_STAGE + s * C::STAGE_BYTES +
                                                                   4 * C::KV_BYTES + side * C::META_BYTES);
                const float sk0 = meta[0];
                const uint32_t s_addr = tmem + lane_base + b * 64;
                const uint32_t ncol = (tail != 0 && live && bj == L.kb - 1) ? tail : 64u;
                // -------- pass 1: integer row extremes (4 independent chains)
                int32_t mx[4] = {INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN},
                        mn[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
#pragma unroll kDecUnroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    uint32_t xs[32];
                    ptx::tmem_ld32(s_addr + h2 * 32, xs);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) { // padded key columns repeat column 0 (K1): no masking
                        mx[j & 3] = max(mx[j & 3], (int32_t)xs[j]);
                        mn[j & 3] = min(mn[j & 3], (int32_t)xs[j]);
                    }
                }
                const int32_t smax = max(max(mx[0], mx[1]), max(mx[2], mx[3]));
                const int32_t smin = min(min(mn[0], mn[1]), min(mn[2], mn[3]));
                // reference order: logit = scale * ((sq * sk) * S) in fp64 (paro_oracle.c, attention.cpp:166)
                const double a64 = __dmul_rn((double)sq, (double)sk0);
                const double tmax64 = __dmul_rn(P.scale64, __dmul_rn(a64, (double)smax));
                const double tmin64 = __dmul_rn(P.scale64, __dmul_rn(a64, (double)smin));
                const double m64 = live ? fmax(st.m64, tmax64) : st.m64;
                const float c0 = (float)(__dmul_rn(__dmul_rn(P.scale64, a64), kLog2e));
                const float m32 = (float)(m64 * kLog2e);
                // exp2 argument of element j = (S_j - smax) * c0 + dmax: exact integer
                // difference, dmax = (tmax - m) * log2e from the fp64 logits
                const float dmax = (float)((tmax64 - m64) * kLog2e);
                float pmax_r = ex2(dmax);
                float pmin_r = ex2(fmaf(__int2float_rn(smin - smax), c0, dmax));
                // rescale when an earlier tile of the item was live (the reference's l > 0, attention.cpp:170)
                const float gamma = st.m32 != -INFINITY ? ex2(st.m32 - m32) : 1.0f;
                if (!valid) {
                    pmin_r = INFINITY;
                    pmax_r = 0.f;
                }
                // the q-block's P-group extremes over this warp's 16 rows
                float gmin = pmin_r, gmax = pmax_r;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) {
                    gmin = fminf(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
                    gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
                }
                if ((lane & 15) == 0)
                    red[(rsl * 4 + quad) * 2 + side] = make_float2(gmin, gmax);
                PROF_T(tw2);
                // -------- pass 2: p, row sum; p parked in TMEM over the row's S
                const uint64_t c00 = pk(c0, c0), nm = pk(dmax, dmax);
                uint64_t sum2 = pk(0.f, 0.f);
#pragma unroll kDecUnroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    uint32_t xs[32];
                    ptx::tmem_ld32(s_addr + h2 * 32, xs);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const uint64_t y2 = fma2(pk(__int2float_rn((int32_t)xs[2 * k] - smax),
                                                    __int2float_rn((int32_t)xs[2 * k + 1] - smax)),
                                                 c00, nm);
                        float ya, yb;
                        upk(y2, ya, yb);
                        const float pa = ex2(ya), pb = ex2(yb);
                        sum2 = add2(sum2, pk(pa, pb));
                        xs[2 * k] = __float_as_uint(pa);
                        xs[2 * k + 1] = __float_as_uint(pb);
                    }
                    ptx::tmem_st32(s_addr + h2 * 32, xs);
                }
                ptx::tmem_st_wait();
                if (__any_sync(0xffffffffu, ncol < 64u)) {
                    // rare (the last key block): the row sum again without the padded
                    // columns (copies of column 0), in the same order
                    sum2 = pk(0.f, 0.f);
#pragma unroll 1
                    for (int h2 = 0; h2 < 2; ++h2) {
                        uint32_t xs[32];
                        ptx::tmem_ld32(s_addr + h2 * 32, xs);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const float pa = (uint32_t)(h2 * 32 + 2 * k) < ncol ? __uint_as_float(xs[2 * k]) : 0.f;
                            const float pb =
                                (uint32_t)(h2 * 32 + 2 * k + 1) < ncol ? __uint_as_float(xs[2 * k + 1]) : 0.f;
                            sum2 = add2(sum2, pk(pa, pb));
                        }
                    }
                }
                float sa, sb;
                upk(sum2, sa, sb);
                if (live) {
                    st.l = st.l * gamma + (sa + sb);
                    st.m32 = m32;
                    st.m64 = m64;
                }
                rowstat[(rsl * 2 + side) * 64 + r] =
                    RowStatD{tmin64, tmax64, m64,   valid ? pmin_r : INFINITY, valid ? pmax_r : 0.f,
                             live ? gamma : 1.f, st.l, smax, valid ? 1u : 0u};
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    ptx::mbar_arrive(bar(DB_RED + rsl));
                PROF_T(tw3);
                PROF_ADD(0, tw1 - tw0);
                PROF_ADD(1, tw2 - tw1);
                PROF_ADD(2, tw3 - tw2);
                PROF_ADD(7, 1);
            }
        }
#ifdef PARO_K3_PROF
        if (lane == 0)
            for (int i = 0; i < 8; ++i)
                atomicAdd(&g_prof[i], prof[i]);
#endif
    } else if (warp < 12) {
        // -------------------------------------------------------- quantizer
        ptx::setmaxnreg_inc<C::REG_QUANT>();
        const uint32_t quad = warp & 3;
        const uint32_t side = lane >> 4;
        const uint32_t r = quad * 16 + (lane & 15);
        const uint32_t lane_base = (quad * 32) << 16;
        const uint32_t tail = L.N & 63;
        uint16_t* xlist = reinterpret_cast<uint16_t*>(smem + C::OFF_XLIST) + quad * 512;
        float4* rmeta = reinterpret_cast<float4*>(smem + C::OFF_RM);
        uint32_t T = 0, I = 0;
        unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t rr = 0;; ++rr) {
            const int it = next_item(rr);
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(DB_ITEMEMPTY + (rr & 1)));
            if (it < 0)
                break;
            const Item x = load_item(L, (uint32_t)it);
            const bool has_qb = side ? x.qb != 0xffffu : true;
            const uint32_t qb = side ? (has_qb ? x.qb : 0u) : x.qa;
            const uint32_t nmine = side ? x.nb : x.na;
            const uint16_t* list = L.items + ((size_t)x.h * L.kb + qb) * L.kb;
            const bool valid_row = has_qb && qb * 64 + r < L.N && qb * 64 + r >= L.dp;
            const float sq = L.qsc[(size_t)x.h * L.kb2 + qb];
            const int32_t dslot = DUMP && has_qb ? P.dump.slot[(size_t)x.h * L.kb2 + qb] : -1;
            for (uint32_t t = 0; t < x.n; ++t, ++T) {
                const uint32_t s = T % NS, b = T % NB, par = T & 1;
                const uint32_t rsl = T % C::RS, rsp = (T / C::RS) & 1; // row-stat ring slot, phase parity
                const bool live = t < nmine;
                const bool valid = live && valid_row;
                const uint32_t bj = live ? list[t] : 0u;
                PROF_T(tq0);
#ifdef PARO_K3_PROF
                ptx::mbar_wait(bar(DB_RED + rsl), rsp);
                PROF_T(tqa);
                PROF_ADD(3, tqa - tq0);
#endif
                // the step's p and row stats; its P tile free (P.V of step T - 2); its stage (meta, K tiles)
                dwait(bar(DB_RED + rsl), rsp);
                dwait(bar(DB_PEMPTY + par), ((T >> 1) & 1) ^ 1);
                dwait(bar(DB_KVFULL + s), (T / NS) & 1);
                ptx::tc_fence_after();
                PROF_T(tq1);
                const float* meta = reinterpret_cast<const float*>(smem + C::OFF_STAGE + s * C::STAGE_BYTES +
                                                                   4 * C::KV_BYTES + side * C::META_BYTES);
                const float2* red_r = red + rsl * 8 + side; // [quad q] at red_r[2 q]
                const RowStatD* rs_r = rowstat + rsl * 128;
                const RowStatD me = rs_r[side * 64 + r];
                uint8_t* prow = smem + C::OFF_P + (par * 2 + side) * C::P_BYTES + (r >> 3) * 512 + (r & 7) * 64;
                float lo = red_r[0].x, hi = red_r[0].y;
#pragma unroll
                for (int q = 1; q < 4; ++q) {
                    lo = fminf(lo, red_r[2 * q].x);
                    hi = fmaxf(hi, red_r[2 * q].y);
                }
                float pscale = __fdiv_rn(hi - lo, P.p_qmax);
                if (pscale == 0.f)
                    pscale = 1.f;
                const float inv = __frcp_rn(pscale);
                uint64_t A2, B2;
                pgroup_consts<3>(lo, hi, inv, P.p_qmax, A2, B2);
                const uint64_t magic2 = pk(8388608.0f, 8388608.0f);
                uint32_t risk = 0; // bit g: 4-element group g has a code that needs the exact path
#pragma unroll kDecUnroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    uint32_t xs[32];
                    ptx::tmem_ld32(tmem + lane_base + b * 64 + h2 * 32, xs);
                    ptx::tmem_ld_wait();
                    uint32_t whi[8];
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        uint32_t hi4 = 0, lo4 = 0;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float p = __uint_as_float(xs[4 * w + e]);
                            // variants (q(1-kappa), q(1+kappa)); floor(. + 0.5) via round-down adds
                            const uint64_t u2 = add2_rm(fma2_rm(pk(p, p), A2, B2), magic2);
                            float ul, uh;
                            upk(u2, ul, uh);
                            if (e == 0) {
                                hi4 = __float_as_uint(uh);
                                lo4 = __float_as_uint(ul);
                            } else { // insert byte 0 of the code word at byte e
                                const uint32_t sel = e == 1 ? 0x3240u : (e == 2 ? 0x3410u : 0x4210u);
                                hi4 = __byte_perm(hi4, __float_as_uint(uh), sel);
                                lo4 = __byte_perm(lo4, __float_as_uint(ul), sel);
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
                }
                if (!valid)
                    risk = 0;
                PROF_T(tq2);
#ifdef PARO_EXP_NOEXACT
                risk = 0;
#endif
                // -------- exact boundary path: rare, warp-uniform entry
                if (__any_sync(0xffffffffu, risk != 0)) {
                    const uint32_t ncol = (tail != 0 && live && bj == L.kb - 1) ? tail : 64u;
                    // this row's fast-path parameters, as the softmax warp formed them
                    const double a64 = __dmul_rn((double)sq, (double)meta[0]);
                    const float c0 = (float)(__dmul_rn(__dmul_rn(P.scale64, a64), kLog2e));
                    const float dmax = (float)((me.tmax - me.m) * kLog2e);
                    const int32_t smax_i = me.smax;
                    const double m64 = me.m;
                    // exact tile lo/hi of both q-blocks from every row's published extremes
                    // (only rows whose fast extreme is within 1e-5 of the fast tile extreme
                    // can hold the exact one; fp64 exp for those few rows only)
                    const uint32_t rmask = __ballot_sync(0xffffffffu, risk != 0);
                    float lo_e[2] = {INFINITY, INFINITY}, hi_e[2] = {0.f, 0.f};
#pragma unroll
                    for (int sd = 0; sd < 2; ++sd) {
                        if (!((sd ? rmask >> 16 : rmask & 0xffffu)))
                            continue;
                        const float2* rd = red + rsl * 8 + sd;
                        float lo_a = rd[0].x, hi_a = rd[0].y;
#pragma unroll
                        for (int q = 1; q < 4; ++q) {
                            lo_a = fminf(lo_a, rd[2 * q].x);
                            hi_a = fmaxf(hi_a, rd[2 * q].y);
                        }
                        float mnv = INFINITY, mxv = 0.f;
                        double args[4];
                        uint32_t kinds = 0, cnt = 0; // bit i: arg i is a max candidate
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            const RowStatD q = rs_r[sd * 64 + lane + 32 * k];
                            if (!q.valid)
                                continue;
                            if (q.pmin <= lo_a * 1.00001f)
                                args[cnt++] = q.tmin - q.m;
                            if (q.pmax >= hi_a * 0.99999f) {
                                if (q.tmax == q.m)
                                    mxv = 1.0f; // exp(0)
                                else {
                                    kinds |= 1u << cnt;
                                    args[cnt++] = q.tmax - q.m;
                                }
                            }
                        }
                        for (uint32_t i2 = 0; __any_sync(0xffffffffu, i2 < cnt); ++i2) {
                            if (i2 < cnt) {
                                const float e = (float)exp(args[i2]);
                                if ((kinds >> i2) & 1u)
                                    mxv = fmaxf(mxv, e);
                                else
                                    mnv = fminf(mnv, e);
                            }
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            mnv = fminf(mnv, __shfl_xor_sync(0xffffffffu, mnv, o));
                            mxv = fmaxf(mxv, __shfl_xor_sync(0xffffffffu, mxv, o));
                        }
                        lo_e[sd] = mnv;
                        hi_e[sd] = mxv;
                    }
                    float ps_e[2];
#pragma unroll
                    for (int sd = 0; sd < 2; ++sd) {
                        ps_e[sd] = __fdiv_rn(hi_e[sd] - lo_e[sd], P.p_qmax);
                        if (ps_e[sd] == 0.f)
                            ps_e[sd] = 1.f;
                    }
                    // each side's fast-variant coefficients (uniform within a side: lanes 0 and 16)
                    const uint64_t A2s[2] = {__shfl_sync(0xffffffffu, A2, 0), __shfl_sync(0xffffffffu, A2, 16)};
                    const uint64_t B2s[2] = {__shfl_sync(0xffffffffu, B2, 0), __shfl_sync(0xffffffffu, B2, 16)};
                    // the warp's risky 4-element groups, listed (owner lane, group) and spread
                    // over all 32 lanes one element each
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
                        uint32_t pos = incl - ng, rr2 = risk;
                        while (rr2) {
                            const uint32_t g = __ffs(rr2) - 1;
                            rr2 &= rr2 - 1;
                            xlist[pos++] = (uint16_t)((lane << 4) | g);
                        }
                    }
                    __syncwarp();
                    const uint8_t* qtile = smem + C::OFF_Q + ((I & 1) * 2 + side) * C::QT_BYTES;
                    const uint8_t* ktile = smem + C::OFF_STAGE + s * C::STAGE_BYTES + side * C::KV_BYTES;
                    const int32_t rowoff = (int32_t)((r >> 3) * 512 + (r & 7) * 64);
                    for (uint32_t base = 0; base < 4 * total; base += 32) {
                        const uint32_t item = base + lane;
                        const bool act = item < 4 * total;
                        const uint32_t ent = act ? xlist[item >> 2] : (lane << 4);
                        const uint32_t o = ent >> 4, j = ((ent & 15u) << 2) + (item & 3u);
                        const uint32_t r_o = __shfl_sync(0xffffffffu, r, (int)o);
                        const int32_t smax_o = __shfl_sync(0xffffffffu, smax_i, (int)o);
                        const float c0_o = __shfl_sync(0xffffffffu, c0, (int)o);
                        const float dmax_o = __shfl_sync(0xffffffffu, dmax, (int)o);
                        const double a64_o = __shfl_sync(0xffffffffu, a64, (int)o);
                        const double m64_o = __shfl_sync(0xffffffffu, m64, (int)o);
                        const uint32_t ncol_o = __shfl_sync(0xffffffffu, ncol, (int)o);
                        if (!act || j >= ncol_o)
                            continue;
                        const uint32_t so = o >> 4;
                        const int32_t dside = (int32_t)so - (int32_t)side;
                        const uint8_t* qt = qtile + dside * (int32_t)C::QT_BYTES;
                        const uint8_t* kt = ktile + dside * (int32_t)C::KV_BYTES;
                        const int32_t Sj = dot_row64(qt, kt, r_o, j);
                        { // re-run the two fast variants of this element; only a split pair needs fp64
                            const float pf = ex2(fmaf(__int2float_rn(Sj - smax_o), c0_o, dmax_o));
                            float ul, uh;
                            upk(add2_rm(fma2_rm(pk(pf, pf), A2s[so], B2s[so]), magic2), ul, uh);
                            if (__float_as_uint(ul) == __float_as_uint(uh))
                                continue;
                        }
                        const double logit = __dmul_rn(P.scale64, __dmul_rn(a64_o, (double)Sj));
                        const float p = (float)exp(logit - m64_o);
                        float q = __fdiv_rn(__fsub_rn(p, lo_e[so]), ps_e[so]);
                        q = fminf(P.p_qmax, fmaxf(0.f, q));
                        uint8_t* prow_o = prow + dside * (int32_t)C::P_BYTES - rowoff +
                                          (int32_t)((r_o >> 3) * 512 + (r_o & 7) * 64);
                        const int chunk = j >> 4;
                        prow_o[((chunk ^ ((r_o >> 1) & 3)) << 4) + (j & 15)] = (uint8_t)round_half_away_pos(q);
                    }
                    __syncwarp();
                    PROF_ADD(6, 1);
                }
                PROF_T(tq3);
                if (DUMP && dslot >= 0 && live) {
                    dump_row(P.dump, dslot, t, r, prow, 0, 4);
                    if (r == 0)
                        dump_meta(P.dump, dslot, t, lo, pscale, bj);
                }
                // per-column offset term of this tile: (lo * vscale) * colsum[c]; exactly 0
                // when idle (an idle side's meta slot is not loaded: stale smem, maybe NaN)
                const float vsc = meta[2];
                usm[(b * 2 + side) * 64 + r] = live ? (lo * vsc) * meta[4 + r] : 0.f;
                // the epilogue's row meta of the step: gamma, (pscale * vscale), the row sum after it
                rmeta[(b * 2 + side) * 64 + r] = make_float4(live ? me.gamma : 1.f, live ? pscale * vsc : 0.f, me.l, 0.f);
                ptx::fence_proxy_async_smem(); // P codes -> the tensor core's view
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(bar(DB_PFULL + (T & 3)));
                    if (C::RS == 2)
                        ptx::mbar_arrive(bar(DB_QDONE + par));
                }
                PROF_ADD(0, tq1 - tq0);
                PROF_ADD(1, tq2 - tq1);
                PROF_ADD(2, tq3 - tq2);
                PROF_ADD(7, 1);
            }
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(DB_QEMPTY + (I & 1))); // no more exact-path reads of the item's Q tiles
            ++I;
        }
#ifdef PARO_K3_PROF
        if (lane == 0)
            for (int i = 0; i < 8; ++i)
                atomicAdd(&g_prof[8 + i], prof[i]);
#endif
    } else {
        // --------------------------------------------------------- epilogue
        // acc (fp32, TMEM columns 192-255, the row's lane) = gamma acc + (pscale vscale) ip + u_c
        // per step, then O = acc / l at the ORIGINAL token row
        ptx::setmaxnreg_dec<C::REG_EPI>();
        const uint32_t quad = warp & 3;
        const uint32_t side = lane >> 4;
        const uint32_t r = quad * 16 + (lane & 15);
        const uint32_t lane_base = (quad * 32) << 16;
        const uint32_t tacc = tmem + lane_base + C::TM_ACC;
        const float4* rmeta = reinterpret_cast<const float4*>(smem + C::OFF_RM);
        uint32_t T = 0;
        unsigned long long prof[4] = {0, 0, 0, 0};
        for (uint32_t rr = 0;; ++rr) {
            const int it = next_item(rr);
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(DB_ITEMEMPTY + (rr & 1)));
            if (it < 0)
                break;
            const Item x = load_item(L, (uint32_t)it);
            const bool has_qb = side ? x.qb != 0xffffu : true;
            const uint32_t qb = side ? (has_qb ? x.qb : 0u) : x.qa;
            const bool valid_row = has_qb && qb * 64 + r < L.N && qb * 64 + r >= L.dp;
            float l_fin = 0.f;
            { // the row's starting accumulators: 0, or K4's dense-prefix state
                const size_t srow = (size_t)x.h * L.kb2 * 64 + qb * 64 + r;
                const bool init = L.dp && valid_row;
                if (init)
                    l_fin = L.init_l[srow];
#pragma unroll kDecUnroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t a[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        a[j] = init ? __float_as_uint(L.init_acc[srow * 64 + ch * 16 + j]) : 0u;
                    tmem_st16(tacc + ch * 16, a);
                }
            }
            for (uint32_t t = 0; t < x.n; ++t, ++T) {
                const uint32_t b = T % NB;
                PROF_T(te0);
                // PFULL orders the quantizers' column offsets and row meta before these reads
                dwait(bar(DB_OFULL + b), (T / NB) & 1);
                dwait(bar(DB_PFULL + (T & 3)), (T >> 2) & 1);
                ptx::tc_fence_after();
                PROF_T(te1);
                const float4 rm = rmeta[(b * 2 + side) * 64 + r];
                l_fin = rm.z;
                const uint64_t g2 = pk(rm.x, rm.x), ss2 = pk(rm.y, rm.y);
                const float4* u4 = reinterpret_cast<const float4*>(usm + (b * 2 + side) * 64);
                ptx::tmem_st_wait(); // the previous step's accumulator stores
#pragma unroll kDecUnroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t raw[16], a[16];
                    tmem_ld16(tmem + lane_base + b * 64 + ch * 16, raw);
                    tmem_ld16(tacc + ch * 16, a);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 uu = u4[ch * 4 + q4];
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int j = q4 * 4 + hh * 2;
                            const uint64_t x2 =
                                pk(__int2float_rn((int32_t)raw[j]), __int2float_rn((int32_t)raw[j + 1]));
                            const uint64_t t2 = fma2(ss2, x2, hh ? pk(uu.z, uu.w) : pk(uu.x, uu.y));
                            const uint64_t a2 = fma2(pk(__uint_as_float(a[j]), __uint_as_float(a[j + 1])), g2, t2);
                            float y0, y1;
                            upk(a2, y0, y1);
                            a[j] = __float_as_uint(y0);
                            a[j + 1] = __float_as_uint(y1);
                        }
                    }
                    tmem_st16(tacc + ch * 16, a);
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    ptx::mbar_arrive(bar(DB_BEMPTY + b));
                PROF_T(te2);
                PROF_ADD(0, te1 - te0);
                PROF_ADD(1, te2 - te1);
                PROF_ADD(3, 1);
            }
            ptx::tmem_st_wait();
            // (tcgen05.ld is warp-collective: every lane loads, valid rows store)
            const float l = l_fin;
            const uint32_t orig = valid_row ? perm_src(L.perm[x.h], qb * 64 + r) : 0u;
            float4* dst = reinterpret_cast<float4*>(P.out + ((size_t)x.h * L.N + orig) * 64);
            const float il = l == 0.f ? 0.f : 1.0f / l;
#pragma unroll kDecUnroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t a[16];
                tmem_ld16(tacc + ch * 16, a);
                ptx::tmem_ld_wait();
                if (valid_row) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        dst[ch * 4 + c] = make_float4(__uint_as_float(a[4 * c]) * il, __uint_as_float(a[4 * c + 1]) * il,
                                                      __uint_as_float(a[4 * c + 2]) * il, __uint_as_float(a[4 * c + 3]) * il);
                }
            }
            if (valid_row && P.zeroed)
                P.zeroed[(size_t)x.h * L.N + orig] = l == 0.f ? 1 : 0;
        }
#ifdef PARO_K3_PROF
        if (lane == 0)
            for (int i = 0; i < 4; ++i)
                atomicAdd(&g_prof[16 + i], prof[i]);
#endif
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1)
        ptx::tmem_dealloc<256>(tmem);
}

cudaError_t launch_k3_dec(const K3Params& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          int num_sms, cudaStream_t st) {
    static bool wd_done = false; // this translation unit's copy of the watchdog switch
    if (!wd_done) {
        wd_done = true;
        if (const char* e = getenv("PARO_WATCHDOG_S")) {
            const unsigned long long ns = (unsigned long long)(atof(e) * 1e9);
            cudaMemcpyToSymbol(ptx::g_watchdog_ns, &ns, sizeof(ns));
        }
    }
#ifdef PARO_K3_PROF
    if (getenv("PARO_K3_PROF_PRINT")) {
        unsigned long long h[32];
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(h, g_prof, sizeof(h));
        const double n = (double)(h[7] ? h[7] : 1), m = (double)(h[15] ? h[15] : 1);
        const double e = (double)(h[19] ? h[19] : 1);
        fprintf(stderr,
                "[k3dec prof] softmax warp/step: wait %.0f (QDONE %.0f then S %.0f) pass1 %.0f pass2+publish %.0f | "
                "quantizer: wait %.0f (RED %.0f) quantize %.0f exact %.0f (exact entries %.4f) | epilogue: wait %.0f "
                "dequant %.0f\n",
                h[0] / n, h[3] / n, h[4] / n, h[1] / n, h[2] / n, h[8] / m, h[11] / m, h[9] / m, h[10] / m, h[14] / m,
                h[16] / e, h[17] / e);
        memset(h, 0, sizeof(h));
        cudaMemcpyToSymbol(g_prof, h, sizeof(h));
    }
#endif
    auto kern = p.dump.slot ? k3_attention_dec<true> : k3_attention_dec<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KDec::SMEM);
    if (e != cudaSuccess)
        return e;
    const uint32_t slots = (uint32_t)num_sms * KDec::MINB;
    const uint32_t grid = p.n_items < slots ? p.n_items : slots;
    kern<<<grid, KDec::THREADS, KDec::SMEM, st>>>(p, tq, tk, tv);
    return cudaGetLastError();
}

} // namespace paro
