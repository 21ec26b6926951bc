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
// Work unit: one (head, q-block pair) -- rows 0..63 = q-block 2p, 64..127 =
// 2p+1 -- so each MMA is M = 128 over the union of the pair's kept key blocks;
// a q-block's warps skip tiles its own mask row drops (no softmax work, the
// garbage half of the MMA output is never read). Units are LPT-sorted by K2
// and dealt to persistent CTAs in snake order.
//
// Warp roles (320 threads; 2 CTAs/SM at d=64, 1 at d=128):
//   warp 0     TMA producer: Q pair tile, K/V tiles + per-block meta (NS-stage ring)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5  softmax: TMEM S -> two passes (row extremes, then p / codes)
//              -> P codes (u8) into swizzled smem; per-tile column offsets
//   warps 6-9  epilogue: TMEM int32 PV -> dequant + rescale into fp32 registers,
//              final normalisation + inverse-permuted row store
// Warp w owns TMEM lanes 32*(w%4)..+31 (hardware lane-quadrant rule), i.e.
// rows of one q-block: quadrants 0,1 -> q-block A, 2,3 -> q-block B.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "layer.cuh"
#include "ptx.cuh"

namespace paro {

template <int D>
struct K3Cfg {
    static constexpr int G = D / 64;
    static constexpr int NS = 4;
    static constexpr int MINB = D == 64 ? 2 : 1; // CTAs per SM
    static constexpr uint32_t Q_BYTES = 128 * D;
    static constexpr uint32_t KV_BYTES = 64 * D;
    static constexpr uint32_t META_BYTES = (4 + D) * 4; // multiple of 16
    static constexpr uint32_t P_BYTES = 128 * 64;
    static constexpr uint32_t S_COLS = G * 64;
    static constexpr uint32_t TM_S = 0;          // two S buffers
    static constexpr uint32_t TM_O = 2 * S_COLS; // two O buffers
    static constexpr uint32_t TMEM_COLS = (2 * S_COLS + 2 * D) <= 256 ? 256 : 512;
    static constexpr uint32_t OFF_Q = 0;
    static constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
    static constexpr uint32_t OFF_V = OFF_K + NS * KV_BYTES;
    static constexpr uint32_t OFF_P = OFF_V + NS * KV_BYTES;
    static constexpr uint32_t OFF_META = OFF_P + 2 * P_BYTES;
    static constexpr uint32_t OFF_ROWMETA = OFF_META + NS * META_BYTES;
    static constexpr uint32_t OFF_U = OFF_ROWMETA + 2 * 128 * 16; // [2 buf][2 q-block][D] column offsets
    static constexpr uint32_t OFF_RED = OFF_U + 2 * 2 * D * 4;
    static constexpr uint32_t OFF_L = OFF_RED + 2 * 2 * 2 * 8;
    static constexpr uint32_t OFF_BAR = OFF_L + 128 * 4;
    static constexpr uint32_t NBAR = 2 + 2 * NS + 12;
    static constexpr uint32_t OFF_TMEMPTR = OFF_BAR + NBAR * 8;
    static constexpr uint32_t SMEM_BYTES = OFF_TMEMPTR + 16;
    // swizzle: rows of D int8 -> 64B (D=64) or 128B (D=128) swizzle atoms of 8 rows
    static constexpr uint32_t LAYOUT = D == 64 ? ptx::kSwizzle64B : ptx::kSwizzle128B;
    static constexpr uint32_t ATOM = 8 * D; // bytes per 8-row swizzle atom
    static constexpr uint32_t IDESC_QK = ptx::idesc_i8(true, true, false, false, 128, 64);
    static constexpr uint32_t IDESC_PV = ptx::idesc_i8(false, true, false, true, 128, D);
};

enum : uint32_t { B_QFULL = 0, B_QEMPTY = 1 };
template <int NS>
struct Bars {
    static constexpr uint32_t KVFULL = 2, KVEMPTY = 2 + NS, SFULL = 2 + 2 * NS, SEMPTY = SFULL + 2,
                              PFULL = SEMPTY + 2, PEMPTY = PFULL + 2, OFULL = PEMPTY + 2, OEMPTY = OFULL + 2,
                              LFULL = OEMPTY + 2, LEMPTY = LFULL + 1;
};

// K-major operand rows of D bytes (Q, K): SBO = one 8-row atom.
template <int D>
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
    return ptx::smem_desc(saddr, 16, K3Cfg<D>::ATOM, K3Cfg<D>::LAYOUT);
}
// P: 128 rows x 64 u8 (K = keys), K-major, 64B swizzle.
__device__ __forceinline__ uint64_t desc_p(uint32_t saddr) { return ptx::smem_desc(saddr, 16, 512, ptx::kSwizzle64B); }
// V: [key][D] row-major = MN-major B operand (N = D contiguous); SBO = 8 keys.
template <int D>
__device__ __forceinline__ uint64_t desc_v(uint32_t saddr) {
    return ptx::smem_desc(saddr, K3Cfg<D>::ATOM * 8, K3Cfg<D>::ATOM, K3Cfg<D>::LAYOUT);
}

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
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// QK issue for one tile: S_g (g < G) in TMEM columns tm_s + 64*g, two K=32 steps per group
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

struct K3Params {
    LayerDev L;
    float scale_log2; // effective scale * log2(e)
    float p_qmax;     // 255 or 15
    float* out;       // [H][N][D] original token order
    uint8_t* zeroed;  // [H][N] or null
    uint32_t n_items;
};

// ---------------------------------------------------------------------------
// Softmax, one kept tile for this thread's row. Pass 1 reads S for the row
// extremes (exact in the integer domain at d=64); the q-block's tile group
// lo/hi then come from two exp2 per row (p at the extreme columns, computed
// with the same formula the elements use, so they are the true min/max of the
// p values); pass 2 re-reads S and produces p, the row sum and the P codes.
// ---------------------------------------------------------------------------
struct RowState {
    float m, l;
};

template <int D, bool TAIL>
__device__ __forceinline__ void softmax_tile(uint32_t s_addr, const float* meta, float cq0, float cq1, uint32_t ncol,
                                             bool valid_row, RowState& st, float p_qmax, float2* red_slot,
                                             const float2* red_pair, uint32_t bar_id, uint8_t* prow, uint32_t row,
                                             float& gamma_out, float& lo_out, float& pscale_out) {
    constexpr int G = D / 64;
    const float c0 = cq0 * meta[0];
    const float c1 = G == 2 ? cq1 * meta[1] : 0.f;
    // -------- pass 1: row extremes
    float m_new, pmax_r, pmin_r;
    if (G == 1) {
        int32_t smax = INT32_MIN, smin = INT32_MAX;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t r[32];
            ptx::tmem_ld32(s_addr + h2 * 32, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (!TAIL || (uint32_t)(h2 * 32 + j) < ncol) {
                    smax = max(smax, (int32_t)r[j]);
                    smin = min(smin, (int32_t)r[j]);
                }
            }
        }
        const float tm = __int2float_rn(smax) * c0;
        m_new = fmaxf(st.m, tm);
        pmax_r = ex2(fmaf(__int2float_rn(smax), c0, -m_new));
        pmin_r = ex2(fmaf(__int2float_rn(smin), c0, -m_new));
    } else {
        float ymax = -INFINITY, ymin = INFINITY;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t r0[32], r1[32];
            ptx::tmem_ld32(s_addr + h2 * 32, r0);
            ptx::tmem_ld32(s_addr + 64 + h2 * 32, r1);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float y = fmaf(__int2float_rn((int32_t)r1[j]), c1, __int2float_rn((int32_t)r0[j]) * c0);
                if (!TAIL || (uint32_t)(h2 * 32 + j) < ncol) {
                    ymax = fmaxf(ymax, y);
                    ymin = fminf(ymin, y);
                }
            }
        }
        m_new = fmaxf(st.m, ymax);
        pmax_r = ex2(ymax - m_new);
        pmin_r = ex2(ymin - m_new);
    }
    const float gamma = st.l > 0.f ? ex2(st.m - m_new) : 1.0f;
    if (!valid_row) {
        pmin_r = INFINITY;
        pmax_r = 0.f;
    }
    // -------- P group extremes over the q-block's 64 rows (p >= 0: compare as uint)
    const uint32_t umin = __reduce_min_sync(0xffffffffu, __float_as_uint(pmin_r));
    const uint32_t umax = __reduce_max_sync(0xffffffffu, __float_as_uint(pmax_r));
    if ((row & 31) == 0)
        *red_slot = make_float2(__uint_as_float(umin), __uint_as_float(umax));
    ptx::named_bar_sync(bar_id, 64);
    const float2 ra = red_pair[0], rb = red_pair[1];
    const float lo = fminf(ra.x, rb.x), hi = fmaxf(ra.y, rb.y);
    float pscale = __fdiv_rn(hi - lo, p_qmax);
    if (pscale == 0.f)
        pscale = 1.f;
    const float inv = __frcp_rn(pscale);
    // -------- pass 2: p, row sum, codes
    const uint64_t c00 = pk(c0, c0), nm = pk(-m_new, -m_new), nlo = pk(-lo, -lo), inv2 = pk(inv, inv);
    const uint64_t half2 = pk(0.5f, 0.5f), magic2 = pk(8388608.0f, 8388608.0f);
    uint64_t sum2 = pk(0.f, 0.f);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        float pv[32];
        if (G == 1) {
            uint32_t r[32];
            ptx::tmem_ld32(s_addr + h2 * 32, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint64_t y2 =
                    fma2(pk(__int2float_rn((int32_t)r[2 * k]), __int2float_rn((int32_t)r[2 * k + 1])), c00, nm);
                float ya, yb;
                upk(y2, ya, yb);
                pv[2 * k] = ex2(ya);
                pv[2 * k + 1] = ex2(yb);
            }
        } else {
            uint32_t r0[32], r1[32];
            ptx::tmem_ld32(s_addr + h2 * 32, r0);
            ptx::tmem_ld32(s_addr + 64 + h2 * 32, r1);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float y = fmaf(__int2float_rn((int32_t)r1[j]), c1, __int2float_rn((int32_t)r0[j]) * c0);
                pv[j] = ex2(y - m_new);
            }
        }
        if (TAIL) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if ((uint32_t)(h2 * 32 + j) >= ncol)
                    pv[j] = 0.f;
        }
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint64_t p2 = pk(pv[2 * k], pv[2 * k + 1]);
            sum2 = add2(sum2, p2);
            // q = (p - lo) * (1/pscale); code = floor(q + 0.5) via two round-down adds
            const uint64_t u2 = add2_rm(add2_rm(mul2(add2(p2, nlo), inv2), half2), magic2);
            float ua, ub;
            upk(u2, ua, ub);
            const uint32_t pair = __byte_perm(__float_as_uint(ua), __float_as_uint(ub), 0x0040);
            if (k & 1)
                w[k >> 1] = __byte_perm(w[k >> 1], pair, 0x5410);
            else
                w[k >> 1] = pair;
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int chunk = h2 * 2 + c;
            *reinterpret_cast<uint4*>(prow + ((chunk ^ ((row >> 1) & 3)) << 4)) =
                make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
        }
    }
    float sa, sb;
    upk(sum2, sa, sb);
    st.l = st.l * gamma + (sa + sb);
    st.m = m_new;
    gamma_out = gamma;
    lo_out = lo;
    pscale_out = pscale;
}

template <int D>
__global__ void __launch_bounds__(320, K3Cfg<D>::MINB)
    k3_attention(const __grid_constant__ K3Params P, const __grid_constant__ CUtensorMap tm_q,
                 const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v) {
    using C = K3Cfg<D>;
    using BR = Bars<C::NS>;
    constexpr int G = C::G;
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
        ptx::mbar_init(bar(B_QFULL), 1);
        ptx::mbar_init(bar(B_QEMPTY), 1);
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(bar(BR::KVFULL + s), 1);
            ptx::mbar_init(bar(BR::KVEMPTY + s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(bar(BR::SFULL + b), 1);
            ptx::mbar_init(bar(BR::SEMPTY + b), 4);
            ptx::mbar_init(bar(BR::PFULL + b), 4);
            ptx::mbar_init(bar(BR::PEMPTY + b), 1 + 4);
            ptx::mbar_init(bar(BR::OFULL + b), 1);
            ptx::mbar_init(bar(BR::OEMPTY + b), 4);
        }
        ptx::mbar_init(bar(BR::LFULL), 4);
        ptx::mbar_init(bar(BR::LEMPTY), 4);
        ptx::fence_barrier_init();
    }
    if (warp == 1)
        ptx::tmem_alloc<C::TMEM_COLS>(sbase + C::OFF_TMEMPTR);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::OFF_TMEMPTR);

    const uint32_t G_cta = gridDim.x;
    const uint32_t rounds = (P.n_items + G_cta - 1) / G_cta;
    // snake dealing of the LPT-sorted work list
    auto item_at = [&](uint32_t r) -> int {
        const uint32_t idx = r * G_cta + ((r & 1) ? (G_cta - 1 - blockIdx.x) : blockIdx.x);
        return idx < P.n_items ? (int)L.order[idx] : -1;
    };

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
            uint32_t T = 0, I = 0;
            for (uint32_t r = 0; r < rounds; ++r) {
                const int it = item_at(r);
                if (it < 0)
                    continue;
                const uint32_t h = (uint32_t)it >> 16, p = (uint32_t)it & 0xffffu;
                const uint32_t n = L.pair_count[h * L.np + p];
                const uint16_t* list = L.items + ((size_t)h * L.np + p) * L.kb;
                const int32_t row0 = (int32_t)(h * L.kb2 * 64);
                ptx::mbar_wait(bar(B_QEMPTY), (I & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(bar(B_QFULL), C::Q_BYTES);
                ptx::tma_load_2d(sbase + C::OFF_Q, &tm_q, 0, row0 + (int32_t)p * 128, bar(B_QFULL));
                for (uint32_t t = 0; t < n; ++t, ++T) {
                    const uint32_t s = T % NS;
                    ptx::mbar_wait(bar(BR::KVEMPTY + s), ((T / NS) & 1) ^ 1);
                    const uint32_t bj = list[t] & 0x3fffu;
                    ptx::mbar_arrive_expect_tx(bar(BR::KVFULL + s), 2 * C::KV_BYTES + C::META_BYTES);
                    ptx::tma_load_2d(sbase + C::OFF_K + s * C::KV_BYTES, &tm_k, 0, row0 + (int32_t)bj * 64,
                                     bar(BR::KVFULL + s));
                    ptx::tma_load_2d(sbase + C::OFF_V + s * C::KV_BYTES, &tm_v, 0, row0 + (int32_t)bj * 64,
                                     bar(BR::KVFULL + s));
                    ptx::bulk_load(sbase + C::OFF_META + s * C::META_BYTES,
                                   L.meta + ((size_t)h * L.kb2 + bj) * meta_stride(D), C::META_BYTES,
                                   bar(BR::KVFULL + s));
                }
                ++I;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t T = 0, I = 0;
            auto issue_pv = [&](uint32_t U) {
                const uint32_t s = U % NS, b = U & 1, ph = (U >> 1) & 1;
                ptx::mbar_wait(bar(BR::PFULL + b), ph);
                ptx::mbar_wait(bar(BR::OEMPTY + b), ph ^ 1);
                ptx::tc_fence_after();
                const uint32_t sp = sbase + C::OFF_P + b * C::P_BYTES;
                const uint32_t sv = sbase + C::OFF_V + s * C::KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    ptx::mma_i8(tmem + C::TM_O + b * D, desc_p(sp + kk * 32), desc_v<D>(sv + kk * 32 * D),
                                C::IDESC_PV, kk);
                ptx::mma_commit(bar(BR::OFULL + b));
                ptx::mma_commit(bar(BR::KVEMPTY + s));
                ptx::mma_commit(bar(BR::PEMPTY + b));
            };
            for (uint32_t r = 0; r < rounds; ++r) {
                const int it = item_at(r);
                if (it < 0)
                    continue;
                const uint32_t h = (uint32_t)it >> 16, p = (uint32_t)it & 0xffffu;
                const uint32_t n = L.pair_count[h * L.np + p];
                ptx::mbar_wait(bar(B_QFULL), I & 1);
                ptx::tc_fence_after();
                for (uint32_t t = 0; t < n; ++t, ++T) {
                    const uint32_t s = T % NS, b = T & 1;
                    ptx::mbar_wait(bar(BR::KVFULL + s), (T / NS) & 1);
                    ptx::mbar_wait(bar(BR::SEMPTY + b), ((T >> 1) & 1) ^ 1);
                    ptx::tc_fence_after();
                    issue_qk<D>(tmem + C::TM_S + b * C::S_COLS, sbase + C::OFF_Q,
                                sbase + C::OFF_K + s * C::KV_BYTES);
                    ptx::mma_commit(bar(BR::SFULL + b));
                    if (t + 1 == n)
                        ptx::mma_commit(bar(B_QEMPTY));
                    if (t > 0)
                        issue_pv(T - 1);
                }
                if (n > 0)
                    issue_pv(T - 1);
                else
                    ptx::mma_commit(bar(B_QEMPTY));
                ++I;
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------------------ softmax
        const uint32_t quad = warp & 3;
        const uint32_t row = quad * 32 + lane;
        const uint32_t qsel = quad >> 1, wip = quad & 1;
        const uint32_t lane_base = (quad * 32) << 16;
        const uint32_t rl = row & 63;
        float2* red = reinterpret_cast<float2*>(smem + C::OFF_RED);
        float4* rowmeta = reinterpret_cast<float4*>(smem + C::OFF_ROWMETA);
        float* usm = reinterpret_cast<float*>(smem + C::OFF_U);
        float* lsm = reinterpret_cast<float*>(smem + C::OFF_L);
        const uint32_t tail = L.N & 63;
        uint32_t T = 0, I = 0;
        for (uint32_t r = 0; r < rounds; ++r) {
            const int it = item_at(r);
            if (it < 0)
                continue;
            const uint32_t h = (uint32_t)it >> 16, p = (uint32_t)it & 0xffffu;
            const uint32_t n = L.pair_count[h * L.np + p];
            const uint16_t* list = L.items + ((size_t)h * L.np + p) * L.kb;
            const uint32_t qb = 2 * p + qsel;
            const bool valid_row = qb < L.kb && qb * 64 + rl < L.N;
            const float cq0 = P.scale_log2 * L.qsc[((size_t)h * L.kb2 + qb) * G];
            const float cq1 = G == 2 ? P.scale_log2 * L.qsc[((size_t)h * L.kb2 + qb) * G + G - 1] : 0.f;
            RowState st{-INFINITY, 0.f};
            for (uint32_t t = 0; t < n; ++t, ++T) {
                const uint32_t s = T % NS, b = T & 1, ph = (T >> 1) & 1;
                const uint32_t e = list[t];
                const uint32_t bj = e & 0x3fffu;
                const bool keep = (e >> (14 + qsel)) & 1u;
                ptx::mbar_wait(bar(BR::SFULL + b), ph);
                ptx::mbar_wait(bar(BR::PEMPTY + b), ph ^ 1);
                if (keep) {
                    ptx::mbar_wait(bar(BR::KVFULL + s), (T / NS) & 1);
                    ptx::tc_fence_after();
                    const float* meta = reinterpret_cast<const float*>(smem + C::OFF_META + s * C::META_BYTES);
                    uint8_t* prow = smem + C::OFF_P + b * C::P_BYTES + (row >> 3) * 512 + (row & 7) * 64;
                    const uint32_t s_addr = tmem + lane_base + C::TM_S + b * C::S_COLS;
                    float2* slot = red + (T & 1) * 4 + qsel * 2 + wip;
                    const float2* pair = red + (T & 1) * 4 + qsel * 2;
                    float gamma, lo, pscale;
                    if (tail != 0 && bj == L.kb - 1)
                        softmax_tile<D, true>(s_addr, meta, cq0, cq1, tail, valid_row, st, P.p_qmax, slot, pair,
                                              1 + qsel, prow, row, gamma, lo, pscale);
                    else
                        softmax_tile<D, false>(s_addr, meta, cq0, cq1, 64, valid_row, st, P.p_qmax, slot, pair,
                                               1 + qsel, prow, row, gamma, lo, pscale);
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                        ptx::mbar_arrive(bar(BR::SEMPTY + b));
                    const float vsc = meta[2];
                    rowmeta[b * 128 + row] = make_float4(gamma, pscale * vsc, 0.f, 1.f);
                    // per-column offset term of this tile: (lo * vscale) * colsum[c]
                    const float os = lo * vsc;
                    float* u = usm + (b * 2 + qsel) * D;
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        u[rl + 64 * c] = os * meta[4 + rl + 64 * c];
                } else {
                    __syncwarp();
                    if (lane == 0)
                        ptx::mbar_arrive(bar(BR::SEMPTY + b));
                    rowmeta[b * 128 + row] = make_float4(1.f, 0.f, 0.f, 0.f);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0)
                    ptx::mbar_arrive(bar(BR::PFULL + b));
            }
            ptx::mbar_wait(bar(BR::LEMPTY), (I & 1) ^ 1);
            lsm[row] = st.l;
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(BR::LFULL));
            ++I;
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t quad = warp & 3;
        const uint32_t row = quad * 32 + lane;
        const uint32_t qsel = quad >> 1;
        const uint32_t lane_base = (quad * 32) << 16;
        const uint32_t rl = row & 63;
        const float4* rowmeta = reinterpret_cast<const float4*>(smem + C::OFF_ROWMETA);
        const float* usm = reinterpret_cast<const float*>(smem + C::OFF_U);
        const float* lsm = reinterpret_cast<const float*>(smem + C::OFF_L);
        uint32_t T = 0, I = 0;
        for (uint32_t r = 0; r < rounds; ++r) {
            const int it = item_at(r);
            if (it < 0)
                continue;
            const uint32_t h = (uint32_t)it >> 16, p = (uint32_t)it & 0xffffu;
            const uint32_t n = L.pair_count[h * L.np + p];
            const uint32_t qb = 2 * p + qsel;
            const bool valid_row = qb < L.kb && qb * 64 + rl < L.N;
            uint64_t acc[D / 2];
#pragma unroll
            for (int c = 0; c < D / 2; ++c)
                acc[c] = 0ull;
            for (uint32_t t = 0; t < n; ++t, ++T) {
                const uint32_t b = T & 1, ph = (T >> 1) & 1;
                ptx::mbar_wait(bar(BR::OFULL + b), ph);
                ptx::mbar_wait(bar(BR::PFULL + b), ph);
                ptx::tc_fence_after();
                const float4 rm = rowmeta[b * 128 + row];
                if (rm.w != 0.f) {
                    const uint64_t g2 = pk(rm.x, rm.x), ss2 = pk(rm.y, rm.y);
                    const float4* u4 = reinterpret_cast<const float4*>(usm + (b * 2 + qsel) * D);
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
                                    pk(__int2float_rn((int32_t)raw[j]), __int2float_rn((int32_t)raw[j + 1]));
                                const uint64_t t2 = fma2(ss2, x2, hh ? pk(uu.z, uu.w) : pk(uu.x, uu.y));
                                acc[(ch * 16 + j) / 2] = fma2(acc[(ch * 16 + j) / 2], g2, t2);
                            }
                        }
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(bar(BR::OEMPTY + b));
                    ptx::mbar_arrive(bar(BR::PEMPTY + b));
                }
            }
            ptx::mbar_wait(bar(BR::LFULL), I & 1);
            const float l = lsm[row];
            __syncwarp();
            if (lane == 0)
                ptx::mbar_arrive(bar(BR::LEMPTY));
            ++I;
            if (valid_row) {
                const uint32_t orig = perm_src(L.perm[h], qb * 64 + rl);
                float4* dst = reinterpret_cast<float4*>(P.out + ((size_t)h * L.N + orig) * D);
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
                    P.zeroed[(size_t)h * L.N + orig] = l == 0.f ? 1 : 0;
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1)
        ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// Debug / parity: int32 S_g tiles for a list of (h, qb, bj) through the same
// TMA maps, smem swizzle, descriptors and tcgen05 issue as K3. One CTA (4
// warps) per tile; writes S[tile][g][row][col] for the 64 rows of qb.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128, 1)
    k3_debug_qk(const __grid_constant__ LayerDev L, const __grid_constant__ CUtensorMap tm_q,
                const __grid_constant__ CUtensorMap tm_k, const uint32_t* __restrict__ tiles, int32_t* S) {
    using C = K3Cfg<D>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t sq = sbase, sk = sbase + C::Q_BYTES;
    const uint32_t bar_ld = sk + C::KV_BYTES, bar_mma = bar_ld + 8, tptr = bar_ld + 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t h = tiles[3 * blockIdx.x], qb = tiles[3 * blockIdx.x + 1], bj = tiles[3 * blockIdx.x + 2];
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar_ld, 1);
        ptx::mbar_init(bar_mma, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0)
        ptx::tmem_alloc<128>(tptr);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (tptr - sbase));
    if (threadIdx.x == 0) {
        const int32_t row0 = (int32_t)(h * L.kb2 * 64);
        ptx::mbar_arrive_expect_tx(bar_ld, C::Q_BYTES + C::KV_BYTES);
        ptx::tma_load_2d(sq, &tm_q, 0, row0 + (int32_t)(qb / 2) * 128, bar_ld);
        ptx::tma_load_2d(sk, &tm_k, 0, row0 + (int32_t)bj * 64, bar_ld);
        ptx::mbar_wait(bar_ld, 0);
        ptx::tc_fence_after();
        issue_qk<D>(tmem, sq, sk);
        ptx::mma_commit(bar_mma);
    }
    ptx::mbar_wait(bar_mma, 0);
    ptx::tc_fence_after();
    const uint32_t row = warp * 32 + lane;
    for (int g = 0; g < C::G; ++g)
        for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t raw[32];
            ptx::tmem_ld32(tmem + ((warp * 32) << 16) + g * 64 + h2 * 32, raw);
            ptx::tmem_ld_wait();
            if ((row >> 6) == (qb & 1)) {
                int32_t* dst = S + (((size_t)blockIdx.x * C::G + g) * 64 + (row & 63)) * 64 + h2 * 32;
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
template <int D>
static cudaError_t launch_k3_t(const K3Params& p, const CUtensorMap& tq, const CUtensorMap& tk,
                               const CUtensorMap& tv, int grid, cudaStream_t st) {
    const uint32_t smem = K3Cfg<D>::SMEM_BYTES;
    cudaError_t e = cudaFuncSetAttribute(k3_attention<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    k3_attention<D><<<grid, 320, smem, st>>>(p, tq, tk, tv);
    return cudaGetLastError();
}

cudaError_t launch_k3(const LayerDev& L, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      float scale_log2, int pv_bits, float* out, uint8_t* zeroed, int num_sms, cudaStream_t st) {
    K3Params p;
    p.L = L;
    p.scale_log2 = scale_log2;
    p.p_qmax = pv_bits == 4 ? 15.0f : 255.0f;
    p.out = out;
    p.zeroed = zeroed;
    p.n_items = L.H * L.np;
    const uint32_t slots = (uint32_t)num_sms * (L.D == 64 ? K3Cfg<64>::MINB : K3Cfg<128>::MINB);
    const int grid = (int)(p.n_items < slots ? p.n_items : slots);
    return L.D == 64 ? launch_k3_t<64>(p, tq, tk, tv, grid, st) : launch_k3_t<128>(p, tq, tk, tv, grid, st);
}

cudaError_t launch_debug_qk(const LayerDev& L, const CUtensorMap& tq, const CUtensorMap& tk, uint32_t n_tiles,
                            const uint32_t* tiles, int32_t* S, cudaStream_t st) {
    if (n_tiles == 0)
        return cudaSuccess;
    if (L.D == 64) {
        const uint32_t smem = K3Cfg<64>::Q_BYTES + K3Cfg<64>::KV_BYTES + 64;
        cudaFuncSetAttribute(k3_debug_qk<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k3_debug_qk<64><<<n_tiles, 128, smem, st>>>(L, tq, tk, tiles, S);
    } else {
        const uint32_t smem = K3Cfg<128>::Q_BYTES + K3Cfg<128>::KV_BYTES + 64;
        cudaFuncSetAttribute(k3_debug_qk<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k3_debug_qk<128><<<n_tiles, 128, smem, st>>>(L, tq, tk, tiles, S);
    }
    return cudaGetLastError();
}

} // namespace paro
