// prep_kernels.cu -- K1 (PARO reorder gather + per-block quantization), K2
// (block mask -> per q-block-pair kept lists + LPT work order) and the small
// standalone stages (device permutation tables, apply_perm_rows, quantize).
//
// K1 is HBM-bound: per head it reads 3*N*D*4 bytes of fp32 Q/K/V once and
// writes 3*N*D bytes of int8 codes plus per-block scales/colsums. One CTA
// owns one 64-token block (permuted order) of one head for all three tensors;
// each thread issues all its 16-byte gather loads up front (MLP) before the
// block reductions. The quantizer arithmetic is IEEE-exact (this TU is built
// with -fmad=false, explicit __fdiv_rn) so codes/scales are bit-identical to
// quantize() / the engine's V tile quantizer.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "layer.cuh"

namespace paro {

// ---------------------------------------------------------------------------
// quant_affine(x, 0, scale, -qmax, qmax) of kernels_scalar.cpp:78-85:
// (x - 0)/scale in IEEE fp32, clamp to [-qmax, qmax] BEFORE rounding, round
// half away from zero (std::round). x - 0.0f == x for every finite x.
//
// The quotient is the correctly rounded x/scale without a per-element MUFU:
// with rs = RN(1/scale) (one __frcp_rn per group), q0 = RN(x*rs) is within
// 1 ulp and one FMA residual step gives RN(x/scale) (Markstein's theorem;
// no overflow/underflow for the bounded quotients here -- a tiny x only
// changes the sign of a zero code). Round-half-away of |q| uses two
// round-down adds: floor(RD(|q| + 0.5)) == floor(|q| + 0.5), and
// RD(t + 2^23) leaves floor(t) in the mantissa. No XU-pipe instruction.
__device__ __forceinline__ int quant_sym(float x, float scale, float rs, float qmax) {
    if (scale < 0x1p-100f) // tiny scale: see quant_sym4
        return (int)roundf(fminf(qmax, fmaxf(-qmax, __fdiv_rn(x, scale))));
    const float q0 = __fmul_rn(x, rs);
    const float e = __fmaf_rn(-q0, scale, x);
    float q = __fmaf_rn(e, rs, q0);
    q = fminf(qmax, fmaxf(-qmax, q));
    const float t = __fadd_rd(fabsf(q), 0.5f);
    const int m = (int)(__float_as_uint(__fadd_rd(t, 8388608.0f)) & 0x7fffffu);
    return q < 0.0f ? -m : m;
}

// Four codes of one float4 for K1. The clamp is provably a no-op there: the
// group scale is RN(amax/qmax) >= (amax/qmax)(1 - 2^-24) and |x| <= amax, so
// |x/scale| <= qmax(1 + 2^-23) and RN of it rounds (half away) to at most qmax
// -- the same code the reference's clamp-then-round gives. The quotients are
// formed two at a time with packed IEEE f32x2 ops (same per-lane rounding as
// quant_sym's __fmul_rn / __fmaf_rn).
__device__ __forceinline__ uint64_t f2pk(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2upk(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t quot2(uint64_t x2, uint64_t scale2, uint64_t rs2, uint64_t neg_scale2) {
    uint64_t q0, e, q;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(q0) : "l"(x2), "l"(rs2));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(e) : "l"(q0), "l"(neg_scale2), "l"(x2));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(q) : "l"(e), "l"(rs2), "l"(q0));
    (void)scale2;
    return q;
}
__device__ __forceinline__ int round_half_away(float q) {
    const float t = __fadd_rd(fabsf(q), 0.5f);
    const int m = (int)(__float_as_uint(__fadd_rd(t, 8388608.0f)) & 0x7fffffu);
    return q < 0.0f ? -m : m;
}
__device__ __forceinline__ int quant_ieee(float x, float scale, float qmax) {
    return round_half_away(fminf(qmax, fmaxf(-qmax, __fdiv_rn(x, scale))));
}
__device__ __forceinline__ void quant_sym4(float4 v, float scale, float rs, float qmax, int& c0, int& c1, int& c2,
                                           int& c3) {
    if (scale < 0x1p-100f) {
        // tiny group scale: for x near a rounding boundary (|x| ~ (k + 1/2) scale) the
        // residual x - q0*scale falls below 2^-126 (or RN(1/scale) overflows), so the
        // residual step no longer gives RN(x/scale); such groups take the IEEE
        // quotient and the clamp as written (group-uniform branch; found by the
        // every-amax-bit-pattern proof in tests/test_gpu_fullshape_int.py)
        c0 = quant_ieee(v.x, scale, qmax);
        c1 = quant_ieee(v.y, scale, qmax);
        c2 = quant_ieee(v.z, scale, qmax);
        c3 = quant_ieee(v.w, scale, qmax);
        return;
    }
    const uint64_t s2 = f2pk(scale, scale), r2 = f2pk(rs, rs), ns2 = f2pk(-scale, -scale);
    float a, b, c, d;
    f2upk(quot2(f2pk(v.x, v.y), s2, r2, ns2), a, b);
    f2upk(quot2(f2pk(v.z, v.w), s2, r2, ns2), c, d);
    c0 = round_half_away(a);
    c1 = round_half_away(b);
    c2 = round_half_away(c);
    c3 = round_half_away(d);
}

__device__ __forceinline__ float4 ld_stream(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ float amax4(float4 v) {
    return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
    return (uint32_t)(a & 0xff) | ((uint32_t)(b & 0xff) << 8) | ((uint32_t)(c & 0xff) << 16) |
           ((uint32_t)(d & 0xff) << 24);
}

// ---------------------------------------------------------------------------
// K1. grid (kb2, H), 256 threads. D/4 threads cover one row (float4 each);
// a pass covers 256/(D/4) rows, PASSES passes cover the 64-row block.
//   Q, K: quantize(.., {8, Symmetric, PerBlock, 64}) (quant.cpp:60-104): one
//         group per 64x64 tile, scale = amax/127 (0 -> 1).
//   V   : engine V-tile quantizer (attention.cpp:104-126): one group per key
//         block over all D columns, scale = amax==0 ? 1 : amax/qmax, colsum.
// Rows i >= N (block padding): Q and V read as zero and write zero codes (an
// all-zero row never changes amax or colsum, so groups keep the reference's
// true-extent semantics). K padding rows are copies of the block's first row:
// in K3 a padded key column then repeats key column 0's logit, so row and tile
// extremes are those of the true columns without per-element masking, and the
// zero V rows keep it out of P.V (K3 only corrects the row sum on tail tiles).
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256, D == 64 ? 4 : 2) k1_reorder_quantize(LayerDev L, const float* __restrict__ q,
                                                           const float* __restrict__ k, const float* __restrict__ v,
                                                           int v_bits, uint32_t head_begin) {
    constexpr int F4 = D / 4;        // float4 per row
    constexpr int RPP = 256 / F4;    // rows per pass
    constexpr int PASSES = 64 / RPP; // 4 (D=64) or 8 (D=128)
    constexpr int G = D / 64;
    const uint32_t b = blockIdx.x, h = head_begin + blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c4 = tid % F4;
    const int r0 = tid / F4;
    const int grp = (c4 * 4) / 64;

    __shared__ float s_amax[3][8][2];
    __shared__ int s_colsum[8][D];
    __shared__ uint32_t s_src[64]; // original token of each row of the block (one div/mod per row, not per thread)

    const size_t head_in = (size_t)h * L.N * D;
    if (tid < 64) {
        const PermDesc pd = L.perm[h];
        const uint32_t i = b * 64 + tid;
        // rows past N: K takes the block's first row (padding duplicates), Q/V are zero
        s_src[tid] = i < L.N ? perm_src(pd, i) : (b * 64 < L.N ? perm_src(pd, b * 64) : 0xffffffffu);
    }
    __syncthreads();
    float4 xq[PASSES], xk[PASSES], xv[PASSES];
#pragma unroll
    for (int j = 0; j < PASSES; ++j) {
        const uint32_t rr = r0 + RPP * j, i = b * 64 + rr, src = s_src[rr];
        const size_t off = head_in + (size_t)src * D + c4 * 4;
        if (i < L.N) {
            xq[j] = ld_stream(q + off);
            xk[j] = ld_stream(k + off);
            xv[j] = ld_stream(v + off);
        } else {
            xq[j] = xv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            xk[j] = src != 0xffffffffu ? ld_stream(k + off)
                                       : make_float4(0.f, 0.f, 0.f, 0.f); // the even-count filler block stays zero
        }
    }
    if (L.rope_cos) {
        // out[2i] = x[2i] cos[2i] - x[2i+1] sin[2i], out[2i+1] = x[2i+1] cos[2i+1] + x[2i] sin[2i+1],
        // each product and sum rounded on its own (this TU is built with -fmad=false), i.e. the
        // eager `x * cos + rotate_half(x) * sin` of the DiT's apply_rotary_emb in fp32
        auto rot = [](float4 x, float4 c, float4 s) {
            return make_float4(__fsub_rn(__fmul_rn(x.x, c.x), __fmul_rn(x.y, s.x)),
                               __fadd_rn(__fmul_rn(x.y, c.y), __fmul_rn(x.x, s.y)),
                               __fsub_rn(__fmul_rn(x.z, c.z), __fmul_rn(x.w, s.z)),
                               __fadd_rn(__fmul_rn(x.w, c.w), __fmul_rn(x.z, s.w)));
        };
#pragma unroll
        for (int j = 0; j < PASSES; ++j) {
            const uint32_t rr = r0 + RPP * j, i = b * 64 + rr, src = s_src[rr];
            if (src == 0xffffffffu || src < L.dp) // filler rows; text tokens carry no rotary embedding
                continue;
            const size_t t = (size_t)(src - L.dp) * D + c4 * 4;
            const float4 c = __ldg(reinterpret_cast<const float4*>(L.rope_cos + t));
            const float4 s = __ldg(reinterpret_cast<const float4*>(L.rope_sin + t));
            xk[j] = rot(xk[j], c, s); // K padding rows repeat the block's first (rotated) row
            if (i < L.N)
                xq[j] = rot(xq[j], c, s);
        }
    }

    // per-thread amax: Q/K per column group, V over everything
    float aq = 0.f, ak = 0.f, av = 0.f;
#pragma unroll
    for (int j = 0; j < PASSES; ++j) {
        aq = fmaxf(aq, amax4(xq[j]));
        ak = fmaxf(ak, amax4(xk[j]));
        av = fmaxf(av, amax4(xv[j]));
    }
    // warp reduce. D=64: the whole warp is one group. D=128: lanes 0-15 are
    // group 0, 16-31 group 1 (one row per warp) -> reduce within 16 lanes.
#pragma unroll
    for (int o = (G == 2 ? 8 : 16); o > 0; o >>= 1) {
        aq = fmaxf(aq, __shfl_xor_sync(0xffffffffu, aq, o));
        ak = fmaxf(ak, __shfl_xor_sync(0xffffffffu, ak, o));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        av = fmaxf(av, __shfl_xor_sync(0xffffffffu, av, o));
    if (lane == 0 || (G == 2 && lane == 16)) {
        const int g = (G == 2 && lane == 16) ? 1 : 0;
        s_amax[0][warp][g] = aq;
        s_amax[1][warp][g] = ak;
        if (g == 0)
            s_amax[2][warp][0] = av;
    }
    __syncthreads();
    float gq = 0.f, gk = 0.f, gv = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        gq = fmaxf(gq, s_amax[0][w][grp]);
        gk = fmaxf(gk, s_amax[1][w][grp]);
        gv = fmaxf(gv, s_amax[2][w][0]);
    }
    float sq = __fdiv_rn(gq, 127.0f);
    if (sq == 0.0f)
        sq = 1.0f;
    float sk = __fdiv_rn(gk, 127.0f);
    if (sk == 0.0f)
        sk = 1.0f;
    const float vq = v_bits == 4 ? 7.0f : 127.0f;
    const float sv = gv == 0.0f ? 1.0f : __fdiv_rn(gv, vq);
    const float rq = __frcp_rn(sq), rk = __frcp_rn(sk), rv = __frcp_rn(sv);

    const size_t head_codes = (size_t)h * L.kb2 * 64 * D;
    int cs0 = 0, cs1 = 0, cs2 = 0, cs3 = 0;
#pragma unroll
    for (int j = 0; j < PASSES; ++j) {
        const size_t off = head_codes + (size_t)(b * 64 + r0 + RPP * j) * D + c4 * 4;
        const float4 a = xq[j], c = xk[j], e = xv[j];
        int a0, a1, a2, a3, k0, k1, k2, k3, v0, v1, v2, v3;
        quant_sym4(a, sq, rq, 127.0f, a0, a1, a2, a3);
        quant_sym4(c, sk, rk, 127.0f, k0, k1, k2, k3);
        quant_sym4(e, sv, rv, vq, v0, v1, v2, v3);
        *reinterpret_cast<uint32_t*>(L.q + off) = pack4(a0, a1, a2, a3);
        *reinterpret_cast<uint32_t*>(L.k + off) = pack4(k0, k1, k2, k3);
        if (L.v_packed) // INT4, two codes per byte, low nibble first (PARQ payload, quant.cpp:237-243)
            *reinterpret_cast<uint16_t*>(L.v + off / 2) =
                (uint16_t)((v0 & 15) | ((v1 & 15) << 4) | ((v2 & 15) << 8) | ((v3 & 15) << 12));
        else
            *reinterpret_cast<uint32_t*>(L.v + off) = pack4(v0, v1, v2, v3);
        cs0 += v0;
        cs1 += v1;
        cs2 += v2;
        cs3 += v3;
    }
    if (G == 1) { // lanes l and l^16 hold the same columns
        cs0 += __shfl_xor_sync(0xffffffffu, cs0, 16);
        cs1 += __shfl_xor_sync(0xffffffffu, cs1, 16);
        cs2 += __shfl_xor_sync(0xffffffffu, cs2, 16);
        cs3 += __shfl_xor_sync(0xffffffffu, cs3, 16);
    }
    if (G == 2 || lane < 16) {
        s_colsum[warp][c4 * 4 + 0] = cs0;
        s_colsum[warp][c4 * 4 + 1] = cs1;
        s_colsum[warp][c4 * 4 + 2] = cs2;
        s_colsum[warp][c4 * 4 + 3] = cs3;
    }
    __syncthreads();
    float* meta = L.meta + ((size_t)h * L.kb2 + b) * meta_stride(D);
    if (tid < D) {
        int s = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w)
            s += s_colsum[w][tid];
        meta[4 + tid] = (float)s;
    }
    if (tid == 0) {
        meta[0] = sk;
        meta[2] = sv;
        meta[3] = 0.f;
        L.qsc[((size_t)h * L.kb2 + b) * G + 0] = sq;
    }
    if (tid == F4 - 1) { // a thread of the last column group
        if (G == 2) {
            meta[1] = sk;
            L.qsc[((size_t)h * L.kb2 + b) * G + 1] = sq;
        } else {
            meta[1] = 0.f;
        }
    }
}

// ---------------------------------------------------------------------------
// K1, one tensor per CTA: grid (kb2, H, 3), blockIdx.z = 0 Q, 1 K, 2 V -- the
// same per-element arithmetic, reductions and outputs as k1_reorder_quantize,
// with a third of its registers, so 4 CTAs fit an SM at d=128 and a small layer
// (c4: 1536 blocks) is not cut into 5.2 waves of 2 CTAs per SM
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256, 4) k1_reorder_quantize_split(LayerDev L, const float* __restrict__ q,
                                                                 const float* __restrict__ k,
                                                                 const float* __restrict__ v, int v_bits,
                                                                 uint32_t head_begin) {
    constexpr int F4 = D / 4;
    constexpr int RPP = 256 / F4;
    constexpr int PASSES = 64 / RPP;
    constexpr int G = D / 64;
    const uint32_t b = blockIdx.x, h = head_begin + blockIdx.y, which = blockIdx.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c4 = tid % F4;
    const int r0 = tid / F4;
    const int grp = (c4 * 4) / 64;

    __shared__ float s_amax[8][2];
    __shared__ int s_colsum[8][D];
    __shared__ uint32_t s_src[64];

    const size_t head_in = (size_t)h * L.N * D;
    if (tid < 64) {
        const PermDesc pd = L.perm[h];
        const uint32_t i = b * 64 + tid;
        s_src[tid] = i < L.N ? perm_src(pd, i) : (b * 64 < L.N ? perm_src(pd, b * 64) : 0xffffffffu);
    }
    __syncthreads();
    const float* __restrict__ in = which == 0 ? q : (which == 1 ? k : v);
    float4 x[PASSES];
#pragma unroll
    for (int j = 0; j < PASSES; ++j) {
        const uint32_t rr = r0 + RPP * j, i = b * 64 + rr, src = s_src[rr];
        const size_t off = head_in + (size_t)src * D + c4 * 4;
        if (i < L.N)
            x[j] = ld_stream(in + off);
        else // K padding rows repeat the block's first row; Q / V padding rows are zero
            x[j] = which == 1 && src != 0xffffffffu ? ld_stream(in + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (L.rope_cos && which < 2) {
        auto rot = [](float4 x, float4 c, float4 s) {
            return make_float4(__fsub_rn(__fmul_rn(x.x, c.x), __fmul_rn(x.y, s.x)),
                               __fadd_rn(__fmul_rn(x.y, c.y), __fmul_rn(x.x, s.y)),
                               __fsub_rn(__fmul_rn(x.z, c.z), __fmul_rn(x.w, s.z)),
                               __fadd_rn(__fmul_rn(x.w, c.w), __fmul_rn(x.z, s.w)));
        };
#pragma unroll
        for (int j = 0; j < PASSES; ++j) {
            const uint32_t rr = r0 + RPP * j, i = b * 64 + rr, src = s_src[rr];
            if (src == 0xffffffffu || src < L.dp)
                continue;
            const size_t t = (size_t)(src - L.dp) * D + c4 * 4;
            const float4 c = __ldg(reinterpret_cast<const float4*>(L.rope_cos + t));
            const float4 sn = __ldg(reinterpret_cast<const float4*>(L.rope_sin + t));
            if (which == 1 || i < L.N)
                x[j] = rot(x[j], c, sn);
        }
    }
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < PASSES; ++j)
        a = fmaxf(a, amax4(x[j]));
    if (which < 2) { // Q / K: per 64-column group (d=128: lanes 0-15 group 0, 16-31 group 1)
#pragma unroll
        for (int o = (G == 2 ? 8 : 16); o > 0; o >>= 1)
            a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    }
    if (lane == 0 || (G == 2 && lane == 16))
        s_amax[warp][(G == 2 && lane == 16) ? 1 : 0] = a;
    __syncthreads();
    const int gsel = which < 2 ? grp : 0;
    float gm = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w)
        gm = fmaxf(gm, s_amax[w][gsel]);
    const float qmax = which < 2 ? 127.0f : (v_bits == 4 ? 7.0f : 127.0f);
    float sc;
    if (which < 2) {
        sc = __fdiv_rn(gm, 127.0f);
        if (sc == 0.0f)
            sc = 1.0f;
    } else {
        sc = gm == 0.0f ? 1.0f : __fdiv_rn(gm, qmax);
    }
    const float rs = __frcp_rn(sc);

    const size_t head_codes = (size_t)h * L.kb2 * 64 * D;
    int cs0 = 0, cs1 = 0, cs2 = 0, cs3 = 0;
#pragma unroll
    for (int j = 0; j < PASSES; ++j) {
        const size_t off = head_codes + (size_t)(b * 64 + r0 + RPP * j) * D + c4 * 4;
        int e0, e1, e2, e3;
        quant_sym4(x[j], sc, rs, qmax, e0, e1, e2, e3);
        if (which == 0) {
            *reinterpret_cast<uint32_t*>(L.q + off) = pack4(e0, e1, e2, e3);
        } else if (which == 1) {
            *reinterpret_cast<uint32_t*>(L.k + off) = pack4(e0, e1, e2, e3);
        } else {
            if (L.v_packed)
                *reinterpret_cast<uint16_t*>(L.v + off / 2) =
                    (uint16_t)((e0 & 15) | ((e1 & 15) << 4) | ((e2 & 15) << 8) | ((e3 & 15) << 12));
            else
                *reinterpret_cast<uint32_t*>(L.v + off) = pack4(e0, e1, e2, e3);
            cs0 += e0;
            cs1 += e1;
            cs2 += e2;
            cs3 += e3;
        }
    }
    float* meta = L.meta + ((size_t)h * L.kb2 + b) * meta_stride(D);
    if (which == 2) {
        if (G == 1) {
            cs0 += __shfl_xor_sync(0xffffffffu, cs0, 16);
            cs1 += __shfl_xor_sync(0xffffffffu, cs1, 16);
            cs2 += __shfl_xor_sync(0xffffffffu, cs2, 16);
            cs3 += __shfl_xor_sync(0xffffffffu, cs3, 16);
        }
        if (G == 2 || lane < 16) {
            s_colsum[warp][c4 * 4 + 0] = cs0;
            s_colsum[warp][c4 * 4 + 1] = cs1;
            s_colsum[warp][c4 * 4 + 2] = cs2;
            s_colsum[warp][c4 * 4 + 3] = cs3;
        }
        __syncthreads();
        if (tid < D) {
            int sum = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w)
                sum += s_colsum[w][tid];
            meta[4 + tid] = (float)sum;
        }
        if (tid == 0) {
            meta[2] = sc;
            meta[3] = 0.f;
        }
    } else if (which == 1) {
        if (tid == 0)
            meta[0] = sc;
        if (tid == F4 - 1)
            meta[1] = G == 2 ? sc : 0.f;
    } else {
        if (tid == 0)
            L.qsc[((size_t)h * L.kb2 + b) * G + 0] = sc;
        if (G == 2 && tid == F4 - 1)
            L.qsc[((size_t)h * L.kb2 + b) * G + 1] = sc;
    }
}

// ---------------------------------------------------------------------------
// Standalone quantize(m, {bits, Symmetric, PerBlock, 64}) for cols in {64,128}
// (same arithmetic as K1's Q/K path, identity row order).
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_quantize_sym(const float* __restrict__ in, uint32_t rows, int bits,
                                                      int8_t* __restrict__ codes, float* __restrict__ scales) {
    constexpr int F4 = D / 4, RPP = 256 / F4, PASSES = 64 / RPP, G = D / 64;
    const uint32_t b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c4 = tid % F4, r0 = tid / F4, grp = (c4 * 4) / 64;
    __shared__ float s_amax[8][2];
    float4 x[PASSES];
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < PASSES; ++j) {
        const uint32_t i = b * 64 + r0 + RPP * j;
        x[j] = i < rows ? ld_stream(in + (size_t)i * D + c4 * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        a = fmaxf(a, amax4(x[j]));
    }
#pragma unroll
    for (int o = (G == 2 ? 8 : 16); o > 0; o >>= 1)
        a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0 || (G == 2 && lane == 16))
        s_amax[warp][(G == 2 && lane == 16) ? 1 : 0] = a;
    __syncthreads();
    float g = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w)
        g = fmaxf(g, s_amax[w][grp]);
    const float qmax = bits == 4 ? 7.0f : 127.0f;
    float s = __fdiv_rn(g, qmax);
    if (s == 0.0f)
        s = 1.0f;
    const float rs = __frcp_rn(s);
#pragma unroll
    for (int j = 0; j < PASSES; ++j) {
        const uint32_t i = b * 64 + r0 + RPP * j;
        if (i < rows)
            *reinterpret_cast<uint32_t*>(codes + (size_t)i * D + c4 * 4) =
                pack4(quant_sym(x[j].x, s, rs, qmax), quant_sym(x[j].y, s, rs, qmax), quant_sym(x[j].z, s, rs, qmax),
                      quant_sym(x[j].w, s, rs, qmax));
    }
    if (tid == 0)
        scales[(size_t)b * G] = s;
    if (G == 2 && tid == F4 - 1)
        scales[(size_t)b * G + 1] = s;
}

// apply_perm_rows: out.row(i) = in.row(inverse[i]) (reorder.cpp:93-101)
__global__ void k_apply_perm_rows(const float* __restrict__ in, uint32_t rows, uint32_t cols,
                                  const uint32_t* __restrict__ inverse, float* __restrict__ out) {
    const uint32_t i = blockIdx.x;
    if (i >= rows)
        return;
    const float* src = in + (size_t)inverse[i] * cols;
    float* dst = out + (size_t)i * cols;
    for (uint32_t c = threadIdx.x; c < cols; c += blockDim.x)
        dst[c] = src[c];
}

// device permutation tables from the per-head descriptors (bit-exact with make_perm)
__global__ void k_perm_tables(const PermDesc* __restrict__ perm, uint32_t H, uint32_t N, uint32_t* __restrict__ fwd,
                              uint32_t* __restrict__ inv) {
    const uint32_t h = blockIdx.y;
    const PermDesc pd = perm[h];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const uint32_t old = perm_src(pd, i);
        inv[(size_t)h * N + i] = old;
        fwd[(size_t)h * N + old] = i;
    }
}

// ---------------------------------------------------------------------------
// K2a. One CTA (128 threads) per (head, q-block): compacts the mask row
// (BlockMask::bits, one byte per block, mask.hpp:15-32) into the ascending list
// of kept key blocks and its count (a q-block with 0 kept blocks is zeroed and
// flagged, attention.cpp:242-247). bits == nullptr means all blocks kept.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k2_qblock_lists(LayerDev L, const uint8_t* __restrict__ bits) {
    const uint32_t qb = blockIdx.x, h = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ uint32_t s_warp[4];
    __shared__ uint32_t s_base;
    if (tid == 0)
        s_base = 0;
    __syncthreads();
    const uint8_t* row = bits ? bits + ((size_t)h * L.kb + qb) * L.kb : nullptr;
    uint16_t* out = L.items + ((size_t)h * L.kb + qb) * L.kb;
    for (uint32_t c0 = 0; c0 < L.kb; c0 += 128) {
        const uint32_t j = c0 + tid;
        // dense key tiles (K4) and q-blocks made only of dense rows never reach K3
        const bool keep = j < L.kb && j >= L.nd && (qb + 1) * 64 > L.dp && (row ? row[j] != 0 : true);
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0)
            s_warp[warp] = __popc(m);
        __syncthreads();
        uint32_t off = s_base;
        for (int w = 0; w < warp; ++w)
            off += s_warp[w];
        if (keep)
            out[off + __popc(m & ((1u << lane) - 1u))] = (uint16_t)j;
        __syncthreads();
        if (tid == 0)
            s_base += s_warp[0] + s_warp[1] + s_warp[2] + s_warp[3];
        __syncthreads();
    }
    if (tid == 0)
        L.qb_count[(size_t)h * L.kb2 + qb] = s_base;
}

// K2b. One CTA per head: stable counting sort of the head's q-blocks by kept
// count (descending); neighbours become a K3 work pair, so the two
// independent pipelines of a pair run nearly the same number of steps.
__global__ void __launch_bounds__(256) k2_pair_qblocks(LayerDev L) {
    extern __shared__ uint32_t s_buf[]; // hist[kb + 1] then sorted[kb]
    uint32_t* hist = s_buf;
    uint32_t* sorted = s_buf + L.kb + 1;
    const uint32_t h = blockIdx.x;
    const uint32_t* cnt = L.qb_count + (size_t)h * L.kb2;
    for (uint32_t i = threadIdx.x; i <= L.kb; i += blockDim.x)
        hist[i] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < L.kb; i += blockDim.x)
        atomicAdd(&hist[cnt[i]], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int key = (int)L.kb; key >= 0; --key) {
            const uint32_t c = hist[key];
            hist[key] = run;
            run += c;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) { // stable placement, one warp walking q-blocks in order
        const uint32_t lane = threadIdx.x;
        for (uint32_t base = 0; base < L.kb; base += 32) {
            const uint32_t i = base + lane;
            const bool valid = i < L.kb;
            const uint32_t key = valid ? cnt[i] : 0xffffffffu;
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const uint32_t pos = valid ? hist[key] + __popc(peers & ((1u << lane) - 1u)) : 0;
            __syncwarp();
            if (valid && lane == (uint32_t)(__ffs(peers) - 1))
                hist[key] += __popc(peers);
            __syncwarp();
            if (valid)
                sorted[pos] = i;
        }
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < L.np; p += blockDim.x) {
        const uint32_t a = sorted[2 * p];
        const uint32_t b = 2 * p + 1 < L.kb ? sorted[2 * p + 1] : 0xffffu;
        L.pairs[(size_t)h * L.np + p] = a | (b << 16);
        L.pair_count[(size_t)h * L.np + p] = cnt[a]; // sorted descending: A has the larger count
    }
}

// K2c. Counting sort of work items by step count, longest first (LPT order
// for K3's greedy dynamic distribution): block-wide scan of the descending histogram,
// then atomic placement (the order of equal-count items is unspecified -- each
// item's result is independent of when it runs, so outputs are unaffected; a
// single-warp stable placement cost 48 us at c2). Block 0 sorts all H*np items
// into L.order; block c >= 1 sorts the items of chunk c-1's heads into
// the same span of L.order_chunk (the chunked host-buffer pipeline runs K3
// once per chunk).
// Block 0's whole-layer order is LPT inside consecutive groups of L.l2_group heads
// (all heads when 0): the persistent K3 CTAs then work on about one group at a
// time, whose K/V codes the host sized to half of L2, so the K/V tiles re-read by
// every q-block pair of a head stay L2-resident instead of streaming from HBM.
__device__ void k2_lpt_range(const LayerDev& L, uint32_t h0, uint32_t h1, uint32_t* out, uint32_t* s_hist);

__global__ void __launch_bounds__(1024) k2_work_order(LayerDev L) {
    extern __shared__ uint32_t s_hist[]; // kb + 1 buckets
    if (blockIdx.x > 0) {
        k2_lpt_range(L, L.chunk_start[blockIdx.x - 1], L.chunk_start[blockIdx.x], L.order_chunk, s_hist);
        return;
    }
    const uint32_t g = L.l2_group ? L.l2_group : L.H;
    for (uint32_t h0 = 0; h0 < L.H; h0 += g) {
        k2_lpt_range(L, h0, h0 + g < L.H ? h0 + g : L.H, L.order, s_hist);
        __syncthreads();
    }
}

__device__ void k2_lpt_range(const LayerDev& L, uint32_t h0, uint32_t h1, uint32_t* out, uint32_t* s_hist) {
    const uint32_t first = h0 * L.np, total = (h1 - h0) * L.np;
    const uint32_t* key_of = L.pair_count + first;
    out += first;
    for (uint32_t i = threadIdx.x; i <= L.kb; i += blockDim.x)
        s_hist[i] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x)
        atomicAdd(&s_hist[key_of[i]], 1u);
    __syncthreads();
    // exclusive offsets in descending key order: block-wide scan over the
    // reversed histogram, 1024 buckets per pass
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0)
        s_carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint32_t base = 0; base <= L.kb; base += blockDim.x) {
        const uint32_t j = base + threadIdx.x;            // position in descending order
        const int key = (int)L.kb - (int)j;               // bucket
        const uint32_t c = j <= L.kb ? s_hist[key] : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o)
                incl += v;
        }
        if (lane == 31)
            s_warp[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = lane < blockDim.x / 32 ? s_warp[lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= (uint32_t)o)
                    w += v;
            }
            s_warp[lane] = w; // inclusive warp totals
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        const uint32_t excl = carry + (wid ? s_warp[wid - 1] : 0u) + incl - c;
        __syncthreads(); // every thread has read s_carry / s_warp
        if (j <= L.kb)
            s_hist[key] = excl;
        if (threadIdx.x == blockDim.x - 1)
            s_carry = carry + s_warp[blockDim.x / 32 - 1];
        __syncthreads();
    }
    // placement: the items of a key in any order (each item's result is
    // independent of when it runs; only the LPT key order matters)
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
        const uint32_t pos = atomicAdd(&s_hist[key_of[i]], 1u);
        out[pos] = ((h0 + i / L.np) << 16) | (i % L.np);
    }
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
// d=128 layers below ~16 waves of the fused kernel (2 CTAs per SM) take the split
// kernel: c4 (1536 blocks) K1 45.5 -> 41.8 us; at c5 (47k blocks) the fused kernel
// wins, 0.960 vs 1.005 ms, as it does at d=64 (c2 0.134 vs 0.173 ms)
constexpr size_t kK1SplitBelow = 296 * 16;
cudaError_t launch_k1(const LayerDev& L, const float* q, const float* k, const float* v, int v_bits,
                      uint32_t head_begin, uint32_t head_count, cudaStream_t st) {
    if (head_count == 0)
        return cudaSuccess;
    // one CTA per tensor where the fused kernel's CTAs (2 per SM at d=128, 4 at d=64)
    // would leave a ragged last wave; PARO_K1_SPLIT=0 / 1 forces either
    static const int force = [] {
        const char* e = getenv("PARO_K1_SPLIT");
        return e ? atoi(e) : -1;
    }();
    const bool split = force >= 0 ? force != 0 : L.D == 128 && (size_t)L.kb2 * head_count < kK1SplitBelow;
    if (split) {
        dim3 grid(L.kb2, head_count, 3);
        if (L.D == 64)
            k1_reorder_quantize_split<64><<<grid, 256, 0, st>>>(L, q, k, v, v_bits, head_begin);
        else
            k1_reorder_quantize_split<128><<<grid, 256, 0, st>>>(L, q, k, v, v_bits, head_begin);
        return cudaGetLastError();
    }
    dim3 grid(L.kb2, head_count);
    if (L.D == 64)
        k1_reorder_quantize<64><<<grid, 256, 0, st>>>(L, q, k, v, v_bits, head_begin);
    else
        k1_reorder_quantize<128><<<grid, 256, 0, st>>>(L, q, k, v, v_bits, head_begin);
    return cudaGetLastError();
}

cudaError_t launch_quantize_sym(const float* in, uint32_t rows, uint32_t cols, int bits, int8_t* codes,
                                float* scales, cudaStream_t st) {
    const uint32_t nb = (rows + 63) / 64;
    if (cols == 64)
        k_quantize_sym<64><<<nb, 256, 0, st>>>(in, rows, bits, codes, scales);
    else
        k_quantize_sym<128><<<nb, 256, 0, st>>>(in, rows, bits, codes, scales);
    return cudaGetLastError();
}

cudaError_t launch_apply_perm_rows(const float* in, uint32_t rows, uint32_t cols, const uint32_t* inverse, float* out,
                                   cudaStream_t st) {
    k_apply_perm_rows<<<rows, 128, 0, st>>>(in, rows, cols, inverse, out);
    return cudaGetLastError();
}

cudaError_t launch_perm_tables(const PermDesc* perm, uint32_t H, uint32_t N, uint32_t* fwd, uint32_t* inv,
                               cudaStream_t st) {
    dim3 grid((N + 255) / 256, H);
    k_perm_tables<<<grid, 256, 0, st>>>(perm, H, N, fwd, inv);
    return cudaGetLastError();
}

cudaError_t launch_k2_order(const LayerDev& L, cudaStream_t st);

cudaError_t launch_k2(const LayerDev& L, const uint8_t* bits, cudaStream_t st) {
    dim3 grid(L.kb, L.H);
    k2_qblock_lists<<<grid, 128, 0, st>>>(L, bits);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return e;
    // dynamic smem above the 48 KB default once kb > ~6143 (N > ~393K tokens)
    const int smem_pair = (int)((2 * L.kb + 1) * sizeof(uint32_t));
    if (smem_pair > 48 * 1024 &&
        (e = cudaFuncSetAttribute(k2_pair_qblocks, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pair)) !=
            cudaSuccess)
        return e;
    k2_pair_qblocks<<<L.H, 256, smem_pair, st>>>(L);
    e = cudaGetLastError();
    if (e != cudaSuccess)
        return e;
    return launch_k2_order(L, st);
}

cudaError_t launch_k2_order(const LayerDev& L, cudaStream_t st) {
    const int smem = (int)((L.kb + 1) * sizeof(uint32_t));
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(k2_work_order, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess)
            return e;
    }
    k2_work_order<<<1 + L.nchunks, 1024, smem, st>>>(L);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Test hook (paro_debug_k1_quant_proof): K1's quantizer -- the reciprocal +
// one-FMA-residual quotient and the dropped clamp of quant_sym4, and the
// standalone quantize's quant_sym -- against the
// reference arithmetic (kernels_scalar.cpp:78-85: IEEE x/scale, clamp to
// [-qmax, qmax], round half away) for every amax bit pattern in [lo, lo + count):
// scale = amax/qmax (0 -> 1) exactly as K1 forms it, x = +amax, -amax and nx
// pseudo-random x with |x| <= amax (uniform over the bit patterns <= amax, random
// sign), for qmax 127 (Q/K, V INT8) and 7 (V INT4). Counts mismatches; records
// the first one (amax bits, x bits, qmax, K1 code, reference code).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ int ref_code(float x, float scale, float qmax) {
    float q = __fdiv_rn(x, scale);
    q = fminf(qmax, fmaxf(-qmax, q));
    return (int)roundf(q);
}
__global__ void __launch_bounds__(256) k1_quant_proof(uint32_t lo, uint32_t count, uint32_t nx, uint32_t seed,
                                                      unsigned long long* bad, uint32_t* first) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint32_t ab = lo + i;
        const float amax = __uint_as_float(ab);
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const float qmax = v ? 7.0f : 127.0f;
            float scale = __fdiv_rn(amax, qmax);
            if (scale == 0.0f)
                scale = 1.0f;
            const float rs = __frcp_rn(scale);
            for (uint32_t j = 0; j < nx + 2; j += 4) {
                float xs[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t jj = j + e;
                    if (jj == 0)
                        xs[e] = amax;
                    else if (jj == 1)
                        xs[e] = -amax;
                    else {
                        const uint32_t h = mix32(ab * 0x9e3779b9u ^ mix32(jj * 0x85ebca6bu + seed + (uint32_t)v));
                        const uint32_t xb = (uint32_t)(((unsigned long long)mix32(h) * ((unsigned long long)ab + 1)) >> 32);
                        xs[e] = __uint_as_float(xb | (h & 0x80000000u));
                    }
                }
                int c[4];
                quant_sym4(make_float4(xs[0], xs[1], xs[2], xs[3]), scale, rs, qmax, c[0], c[1], c[2], c[3]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (j + e >= nx + 2)
                        continue;
                    const int r = ref_code(xs[e], scale, qmax);
                    const int cs = quant_sym(xs[e], scale, rs, qmax); // the standalone quantize's element path
                    if (c[e] != r || cs != r) {
                        if (atomicAdd(bad, 1ull) == 0ull) {
                            first[0] = ab;
                            first[1] = __float_as_uint(xs[e]);
                            first[2] = (uint32_t)qmax;
                            first[3] = (uint32_t)(c[e] != r ? c[e] : cs);
                            first[4] = (uint32_t)r;
                        }
                    }
                }
            }
        }
    }
}

cudaError_t launch_k1_quant_proof(uint32_t lo, uint32_t count, uint32_t nx, uint32_t seed, unsigned long long* bad,
                                  uint32_t* first, int num_sms, cudaStream_t st) {
    if (count == 0)
        return cudaSuccess;
    const uint32_t blocks = (count + 255) / 256;
    const uint32_t cap = (uint32_t)num_sms * 8;
    k1_quant_proof<<<blocks < cap ? blocks : cap, 256, 0, st>>>(lo, count, nx, seed, bad, first);
    return cudaGetLastError();
}

} // namespace paro
