// attention64_kernel.cu -- K3 at d = 64 (c1/c2/c3): block-sparse INT8-QK /
// INT8|INT4-PV attention on tcgen05, multi-slot layout.
//
// Semantics are those of attention_kernel.cu (the reference stream_engine,
// attention.cpp:84-254, with the restated INT8-QK prologue): per kept (q-block,
// k-block) tile S = Q.K^T (int32, tcgen05 kind::i8, TMEM), exact fp64 row
// extremes and running max, p = exp2 of exact integer differences, one unsigned
// P group per tile with bit-exact codes (two perturbed variants + the fp64
// boundary path), P.V (u8 x s8 -> s32, tcgen05) dequantised into fp32
// accumulators, O = acc / l stored at the ORIGINAL token row.
//
// Layout (one persistent CTA per SM, 640 threads): THREE independent slots, each
// running its own stream of work items (a pair of q-blocks A, B of one head with
// independent kept lists, as in K2) through its own TMEM (S and O, 64 columns
// each: A in lanes 0-15 of every 32-lane quadrant, B in lanes 16-31), its own
// K/V stage ring and P tile in shared memory, and its own compute warpgroup:
//   warps 0-2     single-thread tcgen05.mma issuer of slot 0-2 (warp 3 idle)
//   warps 4-6     TMA producer of slot 0-2 (items from the global LPT counter)
//   warps 8-19    compute: warpgroup 2+s serves slot s; warp (quadrant q) owns
//                 rows 16q..16q+15 of A and of B (lane = TMEM lane). Each warp
//                 runs softmax AND dequant for its rows, software-pipelined:
//                   pass 1 (t)  -> publish the row's P extremes (mbarrier)
//                   dequant (t-1): acc = gamma acc + (ps vs) ip + (lo vs) colsum
//                   pass 2 (t)  once the q-block's extremes are in -> P codes
//                 so the group-reduction wait overlaps the previous step's dequant.
// Per SMSP three compute warps (one per slot) interleave; TMEM holds 3 x 128
// columns. Every wait is a hardware-suspending mbarrier try_wait (no spinning
// probes). setmaxnreg: the control warpgroups drop to 24 registers, the compute
// warps rise to 144.
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

#ifndef PARO_K64_SLOTS
#define PARO_K64_SLOTS 2
#endif
#ifndef PARO_K64_STAGES
#define PARO_K64_STAGES 3
#endif
#ifndef PARO_K64_DS
#define PARO_K64_DS (PARO_K64_SLOTS <= 2) // double-buffered S (QK of step t+2 issued once pass 2 of t is done)
#endif
struct K64 {
    static constexpr int NSLOT = PARO_K64_SLOTS;
    static constexpr int NS = PARO_K64_STAGES;         // K/V stages per slot
    static constexpr int THREADS = 128 * (2 + NSLOT); // 2 control warpgroups + one compute warpgroup per slot
    // the launch allocates ALLOC registers per thread; the two control warpgroups
    // release 256 x (ALLOC - 24) of them and the compute warps take the rest
    static constexpr uint32_t ALLOC = (65536 / THREADS) / 8 * 8;
    static constexpr uint32_t REG_LOW = 24;
    static constexpr uint32_t REG_COMPUTE_RAW = ALLOC + 256 * (ALLOC - REG_LOW) / (128 * NSLOT);
    static constexpr uint32_t REG_COMPUTE = (REG_COMPUTE_RAW > 240 ? 240 : REG_COMPUTE_RAW) / 8 * 8;
    static_assert(256 * (ALLOC - REG_LOW) >= 128 * NSLOT * (REG_COMPUTE - ALLOC), "setmaxnreg pool");
    static constexpr uint32_t TILE = 64 * 64;                                      // one 64x64 int8 / u8 tile
    static constexpr uint32_t META = (4 + 64) * 4;                                 // {ksc, -, vsc, 0, colsum[64]}
    static constexpr uint32_t STAGE = (4 * TILE + 2 * META + 1023) / 1024 * 1024; // K_A K_B V_A V_B meta_A meta_B
    // per-slot shared memory
    static constexpr uint32_t S_Q = 0;                       // Q_A, Q_B
    static constexpr uint32_t S_ST = 2 * TILE;               // NS stages
    static constexpr uint32_t S_P = S_ST + NS * STAGE;       // P_A, P_B (64B-swizzled u8 rows)
    static constexpr uint32_t S_U = S_P + 2 * TILE;          // [2 parity][2 side][64] per-column offset terms
    static constexpr uint32_t S_RED = S_U + 2 * 2 * 64 * 4;  // [2 parity][4 quad][2 side] float2 (P extremes)
    static constexpr uint32_t S_RS = S_RED + 2 * 4 * 2 * 8;  // [2 parity][2 side][64] RowStat
    static constexpr uint32_t S_XL = S_RS + 2 * 2 * 64 * 40; // [4 warps][512] u16 exact-path lists
    static constexpr uint32_t SLOT = (S_XL + 4 * 512 * 2 + 1023) / 1024 * 1024;
    enum : uint32_t {
        B_QFULL = 0,
        B_QEMPTY,
        B_KVFULL,
        B_KVEMPTY = B_KVFULL + NS,
        B_SFULL = B_KVEMPTY + NS, // [2] with DS
        B_PFULL = B_SFULL + 2,
        B_OFULL,
        B_RED,
        B_ITEMFULL,
        B_ITEMEMPTY = B_ITEMFULL + 2,
        NB = B_ITEMEMPTY + 2
    };
    static constexpr uint32_t OFF_BAR = NSLOT * SLOT;
    static constexpr uint32_t OFF_RING = OFF_BAR + NSLOT * NB * 8; // [NSLOT][2] int
    static constexpr uint32_t OFF_TMEMPTR = OFF_RING + NSLOT * 2 * 4;
    static constexpr uint32_t SMEM = OFF_TMEMPTR + 16;
    static constexpr uint32_t IDESC_QK = ptx::idesc_i8(true, true, false, false, 64, 64);
    static constexpr uint32_t IDESC_PV = ptx::idesc_i8(false, true, false, true, 64, 64);
    static constexpr uint32_t LANE16 = 16u << 16; // TMEM address of lane 16 (side B)
};
static_assert(K64::SMEM <= 227 * 1024, "K3 d=64 shared memory");
constexpr bool kDS = PARO_K64_DS;
constexpr uint32_t kSlotCols = kDS ? 192 : 128; // S (x2 with DS) + O, 64 columns each
constexpr uint32_t kOcol = kDS ? 128 : 64;
static_assert(K64::NSLOT * kSlotCols <= 512, "TMEM columns per slot");

// UMMA operand descriptors (64-byte rows, 64B swizzle, 8-row atoms of 512 B)
__device__ __forceinline__ uint64_t d64_k(uint32_t a) { return ptx::smem_desc(a, 16, 512, ptx::kSwizzle64B); }
__device__ __forceinline__ uint64_t d64_v(uint32_t a) { return ptx::smem_desc(a, 4096, 512, ptx::kSwizzle64B); }

__device__ __forceinline__ void qk64(uint32_t d, uint32_t sq, uint32_t sk) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
        ptx::mma_i8(d, d64_k(sq + kk * 32), d64_k(sk + kk * 32), K64::IDESC_QK, kk);
}
__device__ __forceinline__ void pv64(uint32_t d, uint32_t sp, uint32_t sv) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
        ptx::mma_i8(d, d64_k(sp + kk * 32), d64_v(sv + kk * 32 * 64), K64::IDESC_PV, kk);
}

// ---------------------------------------------------------------------------
// Softmax of one step for this thread's row, split at the q-block's P-group
// reduction so the caller can put the previous step's dequant in between.
// ---------------------------------------------------------------------------
struct Pass1 {
    double a64, m64;       // sq*sk (exact in fp64); running max after this tile
    float c0, dmax, m32;   // exp2 argument of column j: (S_j - smax) * c0 + dmax
    float gamma;           // exp(m_old - m_new) (1 when no earlier tile)
    int32_t smax;
};

// pass 1: the row's integer S extremes, the exact fp64 logits of the extremes
// (logit = scale * ((sq * sk) * S), monotone in S at d = 64), the running max and
// the p extremes (same formula as the elements, so they are the true min / max of
// the row's p values); publishes (pmin, pmax) of the q-block's 16 rows of this
// quadrant and the row's RowStat for the exact path
__device__ __forceinline__ Pass1 softmax_pass1(uint32_t s_addr, float sq, float sk, double scale64, bool live,
                                               bool valid, const RowState& st, RowStat* rs_w, float2* red_w,
                                               uint32_t lane) {
    Pass1 o;
    int32_t mx[4] = {INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN}, mn[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
    {
        uint32_t x[32], y[32];
        ptx::tmem_ld32(s_addr, x);
        ptx::tmem_ld32(s_addr + 32, y);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) { // padded key columns repeat column 0 (K1): no masking
            mx[j & 3] = max(mx[j & 3], max((int32_t)x[j], (int32_t)y[j]));
            mn[j & 3] = min(mn[j & 3], min((int32_t)x[j], (int32_t)y[j]));
        }
    }
    const int32_t smax = max(max(mx[0], mx[1]), max(mx[2], mx[3]));
    const int32_t smin = min(min(mn[0], mn[1]), min(mn[2], mn[3]));
    o.a64 = __dmul_rn((double)sq, (double)sk);
    const double tmax64 = __dmul_rn(scale64, __dmul_rn(o.a64, (double)smax));
    const double tmin64 = __dmul_rn(scale64, __dmul_rn(o.a64, (double)smin));
    o.m64 = live ? fmax(st.m64, tmax64) : st.m64;
    o.c0 = (float)(__dmul_rn(__dmul_rn(scale64, o.a64), kLog2e));
    o.m32 = (float)(o.m64 * kLog2e);
    o.dmax = (float)((tmax64 - o.m64) * kLog2e);
    o.smax = smax;
    float pmax_r = ex2(o.dmax);
    float pmin_r = ex2(fmaf(__int2float_rn(smin - smax), o.c0, o.dmax));
    *rs_w = RowStat{tmin64, tmax64, o.m64, valid ? pmin_r : INFINITY, valid ? pmax_r : 0.f, valid ? 1 : 0, 0};
    o.gamma = st.m32 != -INFINITY ? ex2(st.m32 - o.m32) : 1.0f;
    if (!valid) {
        pmin_r = INFINITY;
        pmax_r = 0.f;
    }
#pragma unroll
    for (int k = 8; k > 0; k >>= 1) {
        pmin_r = fminf(pmin_r, __shfl_xor_sync(0xffffffffu, pmin_r, k));
        pmax_r = fmaxf(pmax_r, __shfl_xor_sync(0xffffffffu, pmax_r, k));
    }
    if ((lane & 15) == 0)
        *red_w = make_float2(pmin_r, pmax_r);
    return o;
}

// pass 2 (after the q-block's extremes are published): p, row sum and the P
// codes of the row (two (1 -/+ kappa)-perturbed variants per element; a warp
// whose variants disagree anywhere takes the fp64 boundary path for those
// elements, see attention_kernel.cu softmax_step). Returns lo / pscale of the
// tile group; updates the row state.
__device__ __forceinline__ void softmax_pass2(const Pass1& a, uint32_t s_addr, double scale64, uint32_t ncol,
                                              bool live, bool valid, RowState& st, float p_qmax, const float2* red_r,
                                              const RowStat* rs_r, uint32_t side, const uint8_t* qtile,
                                              const uint8_t* ktile, uint8_t* prow, uint32_t r, uint16_t* xlist,
                                              float& lo_out, float& pscale_out) {
    const uint32_t lane = threadIdx.x & 31;
    float lo = red_r[0].x, hi = red_r[0].y;
#pragma unroll
    for (int q = 1; q < 4; ++q) {
        lo = fminf(lo, red_r[2 * q].x);
        hi = fmaxf(hi, red_r[2 * q].y);
    }
    float pscale = __fdiv_rn(hi - lo, p_qmax);
    if (pscale == 0.f)
        pscale = 1.f;
    const float inv = __frcp_rn(pscale);
    const uint64_t c00 = pk(a.c0, a.c0), nm = pk(a.dmax, a.dmax);
    uint64_t A2, B2;
    pgroup_consts<3>(lo, hi, inv, p_qmax, A2, B2);
    const uint64_t magic2 = pk(8388608.0f, 8388608.0f);
    const bool tail_any = __any_sync(0xffffffffu, ncol < 64u);
    uint64_t sum2 = pk(0.f, 0.f);
    uint32_t risk = 0; // bit g: 4-element group g has a code that needs the exact path
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t x[32];
        ptx::tmem_ld32(s_addr + h2 * 32, x);
        ptx::tmem_ld_wait();
        float pv[32];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint64_t y2 = fma2(pk(__int2float_rn((int32_t)x[2 * k] - a.smax),
                                        __int2float_rn((int32_t)x[2 * k + 1] - a.smax)),
                                     c00, nm);
            float ya, yb;
            upk(y2, ya, yb);
            pv[2 * k] = ex2(ya);
            pv[2 * k + 1] = ex2(yb);
        }
        if (tail_any) { // tail tile: the padded key columns (copies of column 0) leave the row sum
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if ((uint32_t)(h2 * 32 + j) >= ncol)
                    pv[j] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            sum2 = add2(sum2, pk(pv[2 * k], pv[2 * k + 1]));
        uint32_t whi[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            uint32_t hi4 = 0, lo4 = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 4 * w + e;
                // variants (q(1-kappa), q(1+kappa)); floor(. + 0.5) via round-down adds
                const uint64_t u2 = add2_rm(fma2_rm(pk(pv[k], pv[k]), A2, B2), magic2);
                float ul, uh;
                upk(u2, ul, uh);
                if (e == 0) {
                    hi4 = __float_as_uint(uh);
                    lo4 = __float_as_uint(ul);
                } else {
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
    // -------- exact boundary path: rare, warp-uniform entry
    if (__any_sync(0xffffffffu, risk != 0)) {
        // exact tile lo / hi of the q-blocks with a risky code in this warp, from every
        // row's published fp64 extremes (fp64 exp only for rows whose fast-path extreme
        // is within 1e-5 of the fast tile extreme)
        const uint32_t rmask = __ballot_sync(0xffffffffu, risk != 0);
        float lo_e[2] = {INFINITY, INFINITY}, hi_e[2] = {0.f, 0.f};
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
            if (!((sd ? rmask >> 16 : rmask & 0xffffu)))
                continue;
            float lo_a = red_r[-(int)side + sd].x, hi_a = red_r[-(int)side + sd].y;
#pragma unroll
            for (int q = 1; q < 4; ++q) {
                lo_a = fminf(lo_a, red_r[-(int)side + sd + 2 * q].x);
                hi_a = fmaxf(hi_a, red_r[-(int)side + sd + 2 * q].y);
            }
            float mn = INFINITY, mx = 0.f;
            double args[4];
            uint32_t kinds = 0, cnt = 0; // bit i: arg i is a max candidate
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const RowStat q = rs_r[sd * 64 + lane + 32 * k];
                if (!q.valid)
                    continue;
                if (q.pmin <= lo_a * 1.00001f)
                    args[cnt++] = q.tmin - q.m;
                if (q.pmax >= hi_a * 0.99999f) {
                    if (q.tmax == q.m)
                        mx = 1.0f; // exp(0)
                    else {
                        kinds |= 1u << cnt;
                        args[cnt++] = q.tmax - q.m;
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
            for (int k = 16; k > 0; k >>= 1) {
                mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, k));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, k));
            }
            lo_e[sd] = mn;
            hi_e[sd] = mx;
        }
        float ps_e[2];
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
            ps_e[sd] = __fdiv_rn(hi_e[sd] - lo_e[sd], p_qmax);
            if (ps_e[sd] == 0.f)
                ps_e[sd] = 1.f;
        }
        const uint64_t A2s[2] = {__shfl_sync(0xffffffffu, A2, 0), __shfl_sync(0xffffffffu, A2, 16)};
        const uint64_t B2s[2] = {__shfl_sync(0xffffffffu, B2, 0), __shfl_sync(0xffffffffu, B2, 16)};
        // the warp's risky 4-element groups, listed (owner lane, group), spread over all lanes
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
            const uint32_t r_o = __shfl_sync(0xffffffffu, r, (int)o);
            const int32_t smax_o = __shfl_sync(0xffffffffu, a.smax, (int)o);
            const float c0_o = __shfl_sync(0xffffffffu, a.c0, (int)o);
            const float dmax_o = __shfl_sync(0xffffffffu, a.dmax, (int)o);
            const double a64_o = __shfl_sync(0xffffffffu, a.a64, (int)o);
            const double m64_o = __shfl_sync(0xffffffffu, a.m64, (int)o);
            const uint32_t ncol_o = __shfl_sync(0xffffffffu, ncol, (int)o);
            if (!act || j >= ncol_o)
                continue;
            const uint32_t so = o >> 4;
            const int32_t dside = (int32_t)so - (int32_t)side;
            const int32_t Sj = dot_row64(qtile + dside * (int32_t)K64::TILE, ktile + dside * (int32_t)K64::TILE,
                                         r_o, j);
            { // re-run the two fast variants of this element; only a split pair needs fp64
                const float pf = ex2(fmaf(__int2float_rn(Sj - smax_o), c0_o, dmax_o));
                float ul, uh;
                upk(add2_rm(fma2_rm(pk(pf, pf), A2s[so], B2s[so]), magic2), ul, uh);
                if (__float_as_uint(ul) == __float_as_uint(uh))
                    continue;
            }
            const double logit = __dmul_rn(scale64, __dmul_rn(a64_o, (double)Sj));
            const float p = (float)exp(logit - m64_o);
            float q = __fdiv_rn(__fsub_rn(p, lo_e[so]), ps_e[so]);
            q = fminf(p_qmax, fmaxf(0.f, q));
            uint8_t* prow_o = prow + dside * (int32_t)K64::TILE - rowoff + (int32_t)((r_o >> 3) * 512 + (r_o & 7) * 64);
            const int chunk = j >> 4;
            prow_o[((chunk ^ ((r_o >> 1) & 3)) << 4) + (j & 15)] = (uint8_t)round_half_away_pos(q);
        }
        __syncwarp();
    }
    float sa, sb;
    upk(sum2, sa, sb);
    if (live) {
        st.l = st.l * a.gamma + (sa + sb);
        st.m32 = a.m32;
        st.m64 = a.m64;
    }
    lo_out = lo;
    pscale_out = pscale;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <bool DUMP> // the P-code dump test hook compiled in (separate instantiation)
__global__ void __launch_bounds__(K64::THREADS, 1)
    k3_attention64(const __grid_constant__ K3Params P, const __grid_constant__ CUtensorMap tm_q,
                   const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v) {
    using C = K64;
    constexpr int NS = C::NS;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = ptx::smem_u32(smem);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const LayerDev& L = P.L;
    auto bar = [&](uint32_t s, uint32_t i) { return sbase + C::OFF_BAR + (s * C::NB + i) * 8; };
    auto slot_base = [&](uint32_t s) { return s * C::SLOT; }; // byte offset of slot s in smem
    volatile int* ring = reinterpret_cast<volatile int*>(smem + C::OFF_RING);

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < C::NSLOT; ++s) {
            ptx::mbar_init(bar(s, C::B_QFULL), 1);
            ptx::mbar_init(bar(s, C::B_QEMPTY), 1 + 4); // last QK retired + the 4 compute warps done with Q
            for (int i = 0; i < NS; ++i) {
                ptx::mbar_init(bar(s, C::B_KVFULL + i), 1);
                ptx::mbar_init(bar(s, C::B_KVEMPTY + i), 1);
            }
            ptx::mbar_init(bar(s, C::B_SFULL), 1);
            ptx::mbar_init(bar(s, C::B_SFULL + 1), 1);
            ptx::mbar_init(bar(s, C::B_PFULL), 4);
            ptx::mbar_init(bar(s, C::B_OFULL), 1);
            ptx::mbar_init(bar(s, C::B_RED), 4);
            for (int i = 0; i < 2; ++i) {
                ptx::mbar_init(bar(s, C::B_ITEMFULL + i), 1);
                ptx::mbar_init(bar(s, C::B_ITEMEMPTY + i), 1 + 4); // the MMA issuer + 4 compute warps
            }
        }
        ptx::fence_barrier_init();
    }
    if (warp == 0)
        ptx::tmem_alloc<512>(sbase + C::OFF_TMEMPTR);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::OFF_TMEMPTR);

    if (warp < 8) {
        ptx::setmaxnreg_dec<C::REG_LOW>();
        if (warp < C::NSLOT && lane == 0) {
            // ------------------------------------------------------------ MMA issuer of slot `warp`
            const uint32_t s = (uint32_t)warp;
            const uint32_t so = slot_base(s);
            const uint32_t ts = tmem + s * kSlotCols; // S at +0 (+64: the second S with DS), O at +kOcol
            uint32_t I = 0, T = 0;
            for (uint32_t r = 0;; ++r) {
                const uint32_t k = r & 1;
                ptx::mbar_wait(bar(s, C::B_ITEMFULL + k), (r >> 1) & 1);
                const int it = ring[s * 2 + k];
                ptx::mbar_arrive(bar(s, C::B_ITEMEMPTY + k));
                if (it < 0)
                    break;
                const Item x = load_item(L, (uint32_t)it);
                ptx::mbar_wait(bar(s, C::B_QFULL), I & 1);
                ptx::tc_fence_after();
                if (x.n == 0) // no kept tile in either q-block: zero rows only
                    ptx::mma_commit(bar(s, C::B_QEMPTY));
                const uint32_t sq = sbase + so + C::S_Q, sp = sbase + so + C::S_P;
                auto qk = [&](uint32_t t) { // QK of item step t (global step T + t)
                    const uint32_t U = T + t, st = U % NS;
                    const uint32_t sk = sbase + so + C::S_ST + st * C::STAGE;
                    const uint32_t sb = kDS ? (U & 1) : 0u;
                    ptx::mbar_wait(bar(s, C::B_KVFULL + st), (U / NS) & 1);
                    ptx::tc_fence_after();
                    if (t < x.na)
                        qk64(ts + sb * 64, sq, sk);
                    if (t < x.nb)
                        qk64(ts + sb * 64 + C::LANE16, sq + C::TILE, sk + C::TILE);
                    ptx::mma_commit(bar(s, C::B_SFULL + sb));
                    if (t + 1 == x.n)
                        ptx::mma_commit(bar(s, C::B_QEMPTY)); // this item's QKs are issued
                };
                const uint32_t ahead = kDS ? 2u : 1u;
                for (uint32_t t = 0; t < ahead && t < x.n; ++t)
                    qk(t);
                for (uint32_t t = 0; t < x.n; ++t) {
                    const uint32_t U = T + t, st = U % NS;
                    const uint32_t sk = sbase + so + C::S_ST + st * C::STAGE;
                    ptx::mbar_wait(bar(s, C::B_PFULL), U & 1);
                    ptx::tc_fence_after();
                    if (t < x.na)
                        pv64(ts + kOcol, sp, sk + 2 * C::TILE);
                    if (t < x.nb)
                        pv64(ts + C::LANE16 + kOcol, sp + C::TILE, sk + 3 * C::TILE);
                    ptx::mma_commit(bar(s, C::B_OFULL));
                    ptx::mma_commit(bar(s, C::B_KVEMPTY + st));
                    if (t + ahead < x.n) // S buffer of step t is free again (pass 2 of t is done)
                        qk(t + ahead);
                }
                T += x.n;
                ++I;
            }
        } else if (warp >= 4 && warp < 4 + C::NSLOT && lane == 0) {
            // ------------------------------------------------------------ producer of slot warp-4
            const uint32_t s = (uint32_t)warp - 4;
            const uint32_t so = slot_base(s);
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
            uint32_t T = 0, I = 0;
            for (uint32_t r = 0;; ++r) {
                const uint32_t idx = atomicAdd(P.work_counter, 1u);
                const int it = idx < P.n_items ? (int)P.order[idx] : -1;
                const uint32_t k = r & 1;
                ptx::mbar_wait(bar(s, C::B_ITEMEMPTY + k), ((r >> 1) & 1) ^ 1);
                ring[s * 2 + k] = it;
                ptx::mbar_arrive(bar(s, C::B_ITEMFULL + k));
                if (it < 0)
                    break;
                const Item x = load_item(L, (uint32_t)it);
                const uint16_t* la = L.items + ((size_t)x.h * L.kb + x.qa) * L.kb;
                const uint16_t* lb = L.items + ((size_t)x.h * L.kb + (x.qb != 0xffffu ? x.qb : 0)) * L.kb;
                const int32_t row0 = (int32_t)(x.h * L.kb2 * 64);
                auto load_kv = [&](uint32_t t) {
                    const uint32_t st = T % NS;
                    ptx::mbar_wait(bar(s, C::B_KVEMPTY + st), ((T / NS) & 1) ^ 1);
                    const bool ha = t < x.na, hb = t < x.nb;
                    const uint32_t fb = bar(s, C::B_KVFULL + st);
                    ptx::mbar_arrive_expect_tx(fb, (ha + hb) * (2 * C::TILE + C::META));
                    const uint32_t sst = sbase + so + C::S_ST + st * C::STAGE;
#pragma unroll
                    for (int side = 0; side < 2; ++side) {
                        if (side ? hb : ha) {
                            const uint32_t bj = side ? lb[t] : la[t];
                            ptx::tma_load_2d(sst + side * C::TILE, &tm_k, 0, row0 + (int32_t)bj * 64, fb);
                            ptx::tma_load_2d(sst + (2 + side) * C::TILE, &tm_v, 0, row0 + (int32_t)bj * 64, fb);
                            ptx::bulk_load(sst + 4 * C::TILE + side * C::META,
                                           L.meta + ((size_t)x.h * L.kb2 + bj) * meta_stride(64), C::META, fb);
                        }
                    }
                    ++T;
                };
                // the first K/V stage goes ahead of Q: the Q buffer frees only when the
                // previous item's last QK retired and its compute warps are done with Q
                if (x.n > 0)
                    load_kv(0);
                ptx::mbar_wait(bar(s, C::B_QEMPTY), (I & 1) ^ 1);
                const uint32_t qf = bar(s, C::B_QFULL);
                ptx::mbar_arrive_expect_tx(qf, (x.qb != 0xffffu ? 2 : 1) * C::TILE);
                ptx::tma_load_2d(sbase + so + C::S_Q, &tm_q, 0, row0 + (int32_t)x.qa * 64, qf);
                if (x.qb != 0xffffu)
                    ptx::tma_load_2d(sbase + so + C::S_Q + C::TILE, &tm_q, 0, row0 + (int32_t)x.qb * 64, qf);
                for (uint32_t t = 1; t < x.n; ++t)
                    load_kv(t);
                ++I;
            }
        }
    } else {
        // ------------------------------------------------------------ compute warps
        ptx::setmaxnreg_inc<C::REG_COMPUTE>();
        const uint32_t s = (uint32_t)(warp - 8) >> 2;
        const uint32_t quad = warp & 3;
        const uint32_t side = lane >> 4;
        const uint32_t r = quad * 16 + (lane & 15); // row within its q-block (and column index for u)
        uint8_t* sm = smem + slot_base(s);
        const uint32_t s_addr = tmem + ((quad * 32) << 16) + s * kSlotCols; // S (buffer 0); O at +kOcol
        const uint32_t tail = L.N & 63;
        float* usm = reinterpret_cast<float*>(sm + C::S_U);
        float2* red = reinterpret_cast<float2*>(sm + C::S_RED);
        RowStat* rowstat = reinterpret_cast<RowStat*>(sm + C::S_RS);
        uint16_t* xlist = reinterpret_cast<uint16_t*>(sm + C::S_XL) + quad * 512;
        const uint8_t* qtile = sm + C::S_Q + side * C::TILE;
        uint8_t* prow = sm + C::S_P + side * C::TILE + (r >> 3) * 512 + (r & 7) * 64;
        uint32_t T = 0, I = 0;
        unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t rr = 0;; ++rr) {
            const uint32_t kq = rr & 1;
            PROF_T(ti0);
            ptx::mbar_wait(bar(s, C::B_ITEMFULL + kq), (rr >> 1) & 1);
            PROF_T(ti1);
            PROF_ADD(7, ti1 - ti0);
            const int it = ring[s * 2 + kq];
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(s, C::B_ITEMEMPTY + kq));
            if (it < 0)
                break;
            const Item x = load_item(L, (uint32_t)it);
            const bool has_qb = side ? x.qb != 0xffffu : true;
            const uint32_t qb = side ? (has_qb ? x.qb : 0u) : x.qa;
            const uint32_t nmine = side ? x.nb : x.na;
            const uint16_t* list = L.items + ((size_t)x.h * L.kb + qb) * L.kb;
            const bool valid_row = has_qb && qb * 64 + r < L.N && qb * 64 + r >= L.dp; // dense rows: K4
            const float sq0 = L.qsc[((size_t)x.h * L.kb2 + qb)];
            const int32_t dslot = DUMP && has_qb ? P.dump.slot[(size_t)x.h * L.kb2 + qb] : -1;
            RowState st{-INFINITY, 0.f, -INFINITY};
            uint64_t acc[32];
#pragma unroll
            for (int c = 0; c < 32; ++c)
                acc[c] = 0ull;
            if (L.dp && valid_row) { // continue from K4's dense-prefix state
                const size_t srow = (size_t)x.h * L.kb2 * 64 + qb * 64 + r;
                st.m64 = L.init_m[srow];
                st.m32 = (float)(st.m64 * kLog2e);
                st.l = L.init_l[srow];
                const float2* a0 = reinterpret_cast<const float2*>(L.init_acc + srow * 64);
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    acc[c] = pk(a0[c].x, a0[c].y);
            }
            float g_prev = 1.f, ss_prev = 0.f; // dequant parameters of the previous step
            for (uint32_t t = 0; t <= x.n; ++t) {
                const uint32_t Tc = T + t;
                const uint32_t par = Tc & 1, stg = Tc % NS;
                const bool live = t < nmine;
                const bool valid = live && valid_row;
                const uint32_t bj = live ? list[t] : 0u;
                const float* meta = reinterpret_cast<const float*>(sm + C::S_ST + stg * C::STAGE + 4 * C::TILE +
                                                                  side * C::META);
                Pass1 a{};
                PROF_T(tp0);
                if (t < x.n) {
                    const uint32_t sb = kDS ? par : 0u;
                    mbar_wait2(bar(s, C::B_SFULL + sb), kDS ? (Tc >> 1) & 1 : par, bar(s, C::B_KVFULL + stg),
                               (Tc / NS) & 1);
                    ptx::tc_fence_after();
                    PROF_T(tp1);
                    PROF_ADD(0, tp1 - tp0);
                    a = softmax_pass1(s_addr + (kDS ? par * 64 : 0u), sq0, meta[0], P.scale64, live, valid, st,
                                      rowstat + (par * 2 + side) * 64 + r, red + (par * 4 + quad) * 2 + side, lane);
                    __syncwarp();
                    if (lane == 0)
                        ptx::mbar_arrive(bar(s, C::B_RED));
                }
                PROF_T(tp2);
                PROF_ADD(1, tp2 - tp0);
                if (t > 0) { // dequant of step t-1 (its P.V was issued after every warp's pass 2)
                    const uint32_t pp = (Tc - 1) & 1;
                    mbar_wait2(bar(s, C::B_OFULL), pp, bar(s, C::B_PFULL), pp);
                    ptx::tc_fence_after();
                    PROF_T(tp3);
                    PROF_ADD(2, tp3 - tp2);
                    const uint64_t g2 = pk(g_prev, g_prev), ss2 = pk(ss_prev, ss_prev);
                    const float4* u4 = reinterpret_cast<const float4*>(usm + (pp * 2 + side) * 64);
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t raw[16];
                        tmem_ld16(s_addr + kOcol + ch * 16, raw);
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
                                acc[(ch * 16 + j) / 2] = fma2(acc[(ch * 16 + j) / 2], g2, t2);
                            }
                        }
                    }
                }
                PROF_T(tp4);
                PROF_ADD(3, tp4 - tp2);
                if (t < x.n) {
                    ptx::mbar_wait(bar(s, C::B_RED), par);
                    PROF_T(tp5);
                    PROF_ADD(4, tp5 - tp4);
                    float lo, pscale;
                    const bool tail_tile = tail != 0 && live && bj == L.kb - 1;
                    softmax_pass2(a, s_addr + (kDS ? par * 64 : 0u), P.scale64, tail_tile ? tail : 64u, live, valid, st, P.p_qmax,
                                  red + par * 8 + side, rowstat + par * 128, side, qtile,
                                  sm + C::S_ST + stg * C::STAGE + side * C::TILE, prow, r, xlist, lo, pscale);
                    if (DUMP && dslot >= 0 && live) {
                        dump_row(P.dump, dslot, t, r, prow, 0, 4);
                        if (r == 0)
                            dump_meta(P.dump, dslot, t, lo, pscale, bj);
                    }
                    const float vsc = meta[2];
                    // per-column offset of this tile, (lo * vscale) * colsum[c] for c = r; exactly
                    // 0 when idle (an idle side's meta slot is not loaded: stale smem, maybe NaN)
                    usm[(par * 2 + side) * 64 + r] = live ? (lo * vsc) * meta[4 + r] : 0.f;
                    g_prev = live ? a.gamma : 1.f;
                    ss_prev = live ? pscale * vsc : 0.f;
                    ptx::fence_proxy_async_smem(); // P codes -> the tensor core's view
                    ptx::tc_fence_before();        // S and O reads of this warp are complete
                    __syncwarp();
                    if (lane == 0)
                        ptx::mbar_arrive(bar(s, C::B_PFULL));
                    PROF_T(tp6);
                    PROF_ADD(5, tp6 - tp5);
                    PROF_ADD(6, 1);
                }
            }
            T += x.n;
            ++I;
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(s, C::B_QEMPTY)); // this warp no longer reads the item's Q tiles
            if (valid_row) {
                const float l = st.l;
                const uint32_t orig = perm_src(L.perm[x.h], qb * 64 + r);
                float4* dst = reinterpret_cast<float4*>(P.out + ((size_t)x.h * L.N + orig) * 64);
                if (l == 0.f) {
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
                    const float il = 1.0f / l;
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        float a0, a1, a2, a3;
                        upk(acc[2 * c], a0, a1);
                        upk(acc[2 * c + 1], a2, a3);
                        dst[c] = make_float4(a0 * il, a1 * il, a2 * il, a3 * il);
                    }
                }
                if (P.zeroed)
                    P.zeroed[(size_t)x.h * L.N + orig] = l == 0.f ? 1 : 0;
            }
        }
#ifdef PARO_K3_PROF
        if (lane == 0)
            for (int i = 0; i < 8; ++i)
                atomicAdd(&g_prof[i], prof[i]);
#endif
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0)
        ptx::tmem_dealloc<512>(tmem);
}

cudaError_t launch_k3_64(const K3Params& p, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
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
        unsigned long long h[24];
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(h, g_prof, sizeof(h));
        const double n = (double)(h[6] ? h[6] : 1);
        fprintf(stderr,
                "[k3v2 prof] compute warp/step: wait S %.0f pass1 %.0f | wait O %.0f dequant %.0f | wait RED %.0f pass2+publish "
                "%.0f (warp-steps %llu, item wait total %.3g)\n",
                h[0] / n, (h[1] - h[0]) / n, h[2] / n, (h[3] - h[2]) / n, h[4] / n, h[5] / n, h[6], (double)h[7]);
        memset(h, 0, sizeof(h));
        cudaMemcpyToSymbol(g_prof, h, sizeof(h));
    }
#endif
    auto kern = p.dump.slot ? k3_attention64<true> : k3_attention64<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K64::SMEM);
    if (e != cudaSuccess)
        return e;
    const uint32_t grid = p.n_items < (uint32_t)num_sms ? p.n_items : (uint32_t)num_sms;
    kern<<<grid, K64::THREADS, K64::SMEM, st>>>(p, tq, tk, tv);
    return cudaGetLastError();
}

} // namespace paro
