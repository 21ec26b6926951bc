// dense_kernel.cu -- K4: the dense text-token prefix of a PARO layer
// (AttnInputs::dense_prefix), in the reference's
// stream_engine semantics (attention.cpp:134-199, 242-251):
//   * rows i < dp ("dense rows") attend to EVERY key tile, mask or not, and
//     are never quantized: p = exp(s - m) times the fp32 V rows;
//   * every other row first sees the dense key tiles (bj < nd = ceil(dp/64),
//     kept regardless of the mask) the same unquantized way; K3 then continues
//     its running (m, l, acc) over the row's kept non-dense tiles, quantized.
// Logits are the restated INT8-QK stage of K3 (scale * sum_g (sq*sk) * S_g in
// fp64, reference order), so the running max m handed to K3 is exact and its
// exact P-code path stays bit-exact. p, l and acc use fp32 (tolerance-level:
// these tiles carry no codes).
//
// Work units (one CTA of 4 warps each, warp w = rows 16w..16w+15 of a q-block):
//   * the nd q-blocks holding dense rows, split into CB key chunks of CH tiles
//     (the dense rows span all kb tiles: without the split the prefix CTAs are
//     the long pole of the layer); each unit writes a partial (m, l, acc) per
//     row, and k4_combine merges the CB partials;
//   * every other q-block, one unit over its nd dense tiles, writing K3's
//     initial state directly.
// Per tile (cp.async, prefetched one tile ahead: K codes + the split V^T tile):
//   S = Q.K^T with mma.sync m16n8k32 s8 (exact int32 per 64-column group);
//   the row max is found on fp32 approximations, and the candidates within the
//   fp32 error bound are re-evaluated in fp64 in the reference's order, so m is
//   exact; p = exp2(c . (S - S_argmax) + (m_tile - m) log2e) from integer
//   differences; P.V with mma.sync m16n8k16 bf16 in a 3-term split
//   (x = hi + lo, 16 significant bits; hi.hi + hi.lo + lo.hi). V is split once
//   per layer by K4a into transposed bf16 hi / lo tiles in HBM (permuted order),
//   which each CTA stages with cp.async and reads with ldmatrix.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "layer.cuh"
#include "ptx.cuh"

namespace paro {

constexpr double kLog2eD = 1.4426950408889634;

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void mma_s8(int32_t (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// x = hi + lo with hi, lo bf16 (16 significant bits together); packs two
// values (element k in the low half, k+1 in the high half)
__device__ __forceinline__ void bf16_split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    uint32_t h, l;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
    const float h0 = __uint_as_float(h << 16), h1 = __uint_as_float(h & 0xffff0000u);
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(x1 - h1), "f"(x0 - h0));
    hi = h;
    lo = l;
}

template <int D>
struct K4Cfg {
    static constexpr int KS = D + 16;   // K code row stride, bytes (conflict-free B fragments)
    static constexpr int TS = 64 + 8;   // transposed bf16 V row stride, elements (conflict-free ldmatrix)
    static constexpr int K_BYTES = 64 * KS;
    static constexpr int T_BYTES = D * TS * 2;
    static constexpr int STAGE = K_BYTES + 2 * T_BYTES; // K codes, V^T hi, V^T lo of one tile
    static constexpr int SMEM = 2 * STAGE;               // double-buffered
};

// K4a: the permuted V of the layer's heads as transposed bf16 hi / lo tiles
// ([H][kb2][D][64] each, key pairs packed low-first) -- split once per layer
// instead of once per (q-block, tile) in every K4 CTA.
template <int D>
__global__ void __launch_bounds__(256) k4_vsplit(LayerDev L, const float* __restrict__ v, uint32_t head_begin) {
    // HBM-bound: one permutation lookup per row (not per element), 16-byte streaming
    // row loads, 16-byte stores of four packed key pairs
    __shared__ float tile[64][D + 1];
    __shared__ uint32_t src[64];
    const uint32_t bj = blockIdx.x, h = head_begin + blockIdx.y, tid = threadIdx.x;
    if (tid < 64) {
        const uint32_t kj = bj * 64 + tid;
        src[tid] = kj < L.N ? perm_src(L.perm[h], kj) : 0xffffffffu;
    }
    __syncthreads();
    constexpr uint32_t C4 = D / 4; // float4 per row
#pragma unroll
    for (uint32_t e = tid; e < 64 * C4; e += 256) {
        const uint32_t j = e / C4, c4 = e % C4, sj = src[j];
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (sj != 0xffffffffu)
            x = __ldcs(reinterpret_cast<const float4*>(v + ((size_t)h * L.N + sj) * D) + c4);
        tile[j][4 * c4] = x.x;
        tile[j][4 * c4 + 1] = x.y;
        tile[j][4 * c4 + 2] = x.z;
        tile[j][4 * c4 + 3] = x.w;
    }
    __syncthreads();
    uint4* hi = reinterpret_cast<uint4*>(L.vsplit_hi) + ((size_t)h * L.kb2 + bj) * D * 8;
    uint4* lo = reinterpret_cast<uint4*>(L.vsplit_lo) + ((size_t)h * L.kb2 + bj) * D * 8;
#pragma unroll
    for (uint32_t e = tid; e < D * 8; e += 256) { // row c of V^T, key pairs 4q..4q+3
        const uint32_t c = e / 8, q = e % 8;
        uint32_t wh[4], wl[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            bf16_split2(tile[8 * q + 2 * k][c], tile[8 * q + 2 * k + 1][c], wh[k], wl[k]);
        hi[e] = make_uint4(wh[0], wh[1], wh[2], wh[3]);
        lo[e] = make_uint4(wl[0], wl[1], wl[2], wl[3]);
    }
}

// exact logit of one (row, key): scale * sum_g (sq_g*sk_g) * S_g in fp64, reference order
template <int G>
__device__ __forceinline__ double k4_exact(double scale64, const double (&a)[G], const int32_t (&sv)[G]) {
    double accg = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g)
        accg = __dadd_rn(accg, __dmul_rn(a[g], (double)sv[g]));
    return __dmul_rn(scale64, accg);
}

template <int D>
__global__ void __launch_bounds__(128) k4_dense(LayerDev L, double scale64,
                                                float* __restrict__ out, uint8_t* __restrict__ zeroed,
                                                uint32_t head_begin) {
    using C = K4Cfg<D>;
    constexpr int G = D / 64;
    constexpr int KSTEPS = D / 32; // k32 steps of Q.K^T (2 per 64-column group)
    constexpr int NT = D / 8;      // n8 tiles of the output columns
    extern __shared__ __align__(16) uint8_t k4_smem[];
    const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(k4_smem);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const uint32_t h = head_begin + blockIdx.y, u = blockIdx.x;
    const uint32_t ndense_units = L.nd * L.k4_cb;
    uint32_t qb, t0, t1, chunk = 0;
    if (u < ndense_units) { // q-block with dense rows, key chunk `chunk`
        qb = u / L.k4_cb;
        chunk = u % L.k4_cb;
        t0 = chunk * L.k4_ch;
        t1 = min(L.kb, t0 + L.k4_ch);
    } else { // q-block without dense rows: its dense tiles only
        qb = L.nd + (u - ndense_units);
        t0 = 0;
        t1 = L.nd;
    }
    const size_t row0 = (size_t)h * L.kb2 * 64;
    const uint32_t rows[2] = {qb * 64 + warp * 16 + gq, qb * 64 + warp * 16 + gq + 8};

    uint32_t qa[KSTEPS][4]; // Q codes, A fragments (row gq / gq+8, k = 4tq.. / 16+4tq..)
    {
        const uint8_t* qr0 = reinterpret_cast<const uint8_t*>(L.q) + (row0 + rows[0]) * D;
        const uint8_t* qr1 = reinterpret_cast<const uint8_t*>(L.q) + (row0 + rows[1]) * D;
#pragma unroll
        for (int s = 0; s < KSTEPS; ++s) {
            qa[s][0] = *reinterpret_cast<const uint32_t*>(qr0 + 32 * s + 4 * tq);
            qa[s][1] = *reinterpret_cast<const uint32_t*>(qr1 + 32 * s + 4 * tq);
            qa[s][2] = *reinterpret_cast<const uint32_t*>(qr0 + 32 * s + 16 + 4 * tq);
            qa[s][3] = *reinterpret_cast<const uint32_t*>(qr1 + 32 * s + 16 + 4 * tq);
        }
    }
    float sq[G];
#pragma unroll
    for (int g = 0; g < G; ++g)
        sq[g] = L.qsc[((size_t)h * L.kb2 + qb) * G + g];

    double m64[2] = {-INFINITY, -INFINITY};
    float lp[2] = {0.f, 0.f}; // this lane's share of l per row
    float acc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n)
        acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;

    // tile bj -> stage bj & 1: K codes and the pre-split V^T hi / lo rows (K4a), async
    auto issue = [&](uint32_t bj) {
        const uint32_t st = smem_base + (bj & 1) * C::STAGE;
        const uint8_t* ksrc = reinterpret_cast<const uint8_t*>(L.k) + (row0 + (size_t)bj * 64) * D;
#pragma unroll
        for (int e = tid; e < 64 * D / 16; e += 128) {
            const int j = e / (D / 16), w = e % (D / 16);
            cp_async16(st + j * C::KS + w * 16, ksrc + (size_t)j * D + w * 16, 16);
        }
        const size_t toff = ((size_t)h * L.kb2 + bj) * D * 64; // bf16 elements
        const uint8_t* vh = reinterpret_cast<const uint8_t*>(L.vsplit_hi) + toff * 2;
        const uint8_t* vl = reinterpret_cast<const uint8_t*>(L.vsplit_lo) + toff * 2;
#pragma unroll 4
        for (int e = tid; e < D * 8; e += 128) { // D rows of 64 bf16 = 8 x 16 B
            const int c = e / 8, w = e % 8;
            cp_async16(st + C::K_BYTES + c * C::TS * 2 + w * 16, vh + (size_t)c * 128 + w * 16, 16);
            cp_async16(st + C::K_BYTES + C::T_BYTES + c * C::TS * 2 + w * 16, vl + (size_t)c * 128 + w * 16, 16);
        }
        cp_async_commit();
    };

    issue(t0);
    for (uint32_t bj = t0; bj < t1; ++bj) {
        cp_async_wait_all();
        __syncthreads(); // tile bj landed; every warp is done with tile bj-1 (its stage is reissued next)
        if (bj + 1 < t1)
            issue(bj + 1);
        bool act[2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
            act[x] = rows[x] < L.N && (rows[x] < L.dp || bj < L.nd);
        if (!__any_sync(0xffffffffu, act[0] || act[1]))
            continue;
        const uint8_t* sk = k4_smem + (bj & 1) * C::STAGE;
        const uint32_t kn = min(64u, L.N - bj * 64);
        // ---- S = Q.K^T (exact int32 per group)
        int32_t S[G][8][4];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int n = 0; n < 8; ++n)
                S[g][n][0] = S[g][n][1] = S[g][n][2] = S[g][n][3] = 0;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            const uint8_t* kr = sk + (n * 8 + gq) * C::KS + 4 * tq;
#pragma unroll
            for (int s = 0; s < KSTEPS; ++s) {
                const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + 32 * s);
                const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + 32 * s + 16);
                mma_s8(S[s / 2][n], qa[s], b0, b1);
            }
        }
        // ---- exact row max of the tile: fp32 screen, fp64 on the candidates
        double a[G];
        float af[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            a[g] = __dmul_rn((double)sq[g], (double)L.meta[((size_t)h * L.kb2 + bj) * meta_stride(D) + g]);
            af[g] = (float)a[g];
        }
        double best[2] = {-INFINITY, -INFINITY};
        int32_t bs[2][G];
        if constexpr (G == 1) {
            // one group: the logit is a non-negative multiple of S, so the
            // integer argmax is the exact argmax (ties share the logit)
            int32_t im[2] = {INT32_MIN, INT32_MIN};
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (n * 8 + 2 * tq + (e & 1) < kn)
                        im[e >> 1] = max(im[e >> 1], S[0][n][e]);
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                im[x] = max(im[x], __shfl_xor_sync(0xffffffffu, im[x], 1));
                im[x] = max(im[x], __shfl_xor_sync(0xffffffffu, im[x], 2));
                bs[x][0] = im[x];
                const int32_t sv[1] = {im[x]};
                best[x] = k4_exact<G>(scale64, a, sv);
            }
        } else {
        float mx[2] = {-INFINITY, -INFINITY}, mag[2] = {0.f, 0.f};
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t key = n * 8 + 2 * tq + (e & 1);
                float x = 0.f, mg = 0.f;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float tv = af[g] * (float)S[g][n][e];
                    x += tv;
                    mg += fabsf(tv);
                }
                if (key < kn) {
                    mx[e >> 1] = fmaxf(mx[e >> 1], x);
                    mag[e >> 1] = fmaxf(mag[e >> 1], mg);
                }
            }
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                mx[x] = fmaxf(mx[x], __shfl_xor_sync(0xffffffffu, mx[x], o));
                mag[x] = fmaxf(mag[x], __shfl_xor_sync(0xffffffffu, mag[x], o));
            }
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int g = 0; g < G; ++g)
                bs[x][g] = 0;
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int x = e >> 1;
                const uint32_t key = n * 8 + 2 * tq + (e & 1);
                float xv = 0.f;
#pragma unroll
                for (int g = 0; g < G; ++g)
                    xv += af[g] * (float)S[g][n][e];
                // fp32 error <= ~3 ulp of the magnitude per element: 1e-6 * mag covers two
                if (key < kn && xv >= mx[x] - 1e-6f * mag[x]) {
                    int32_t sv[G];
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        sv[g] = S[g][n][e];
                    const double lg = k4_exact<G>(scale64, a, sv);
                    if (lg > best[x]) {
                        best[x] = lg;
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            bs[x][g] = sv[g];
                    }
                }
            }
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best[x], o);
                int32_t os[G];
#pragma unroll
                for (int g = 0; g < G; ++g)
                    os[g] = __shfl_xor_sync(0xffffffffu, bs[x][g], o);
                if (ob > best[x]) {
                    best[x] = ob;
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        bs[x][g] = os[g];
                }
            }
        }
        // ---- running max, rescale, p
        float base[2], cg[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
            cg[g] = (float)(scale64 * a[g] * kLog2eD);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            if (!act[x]) {
                base[x] = -INFINITY;
                continue;
            }
            const double mn = fmax(m64[x], best[x]);
            if (mn != m64[x]) { // (attention.cpp:170-178); m = -inf -> gamma 0 on zero state
                const float gam = ex2f((float)((m64[x] - mn) * kLog2eD));
                lp[x] *= gam;
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    acc[n][2 * x] *= gam;
                    acc[n][2 * x + 1] *= gam;
                }
                m64[x] = mn;
            }
            base[x] = (float)((best[x] - mn) * kLog2eD);
        }
        float P[8][4];
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int x = e >> 1;
                const uint32_t key = n * 8 + 2 * tq + (e & 1);
                float arg = base[x];
#pragma unroll
                for (int g = 0; g < G; ++g)
                    arg = fmaf(cg[g], (float)(S[g][n][e] - bs[x][g]), arg);
                const float p = key < kn ? ex2f(arg) : 0.f; // base -inf (inactive row) -> 0
                P[n][e] = p;
                lp[x] += p;
            }
        // ---- acc += P.V: bf16 m16n8k16, 3-term split (hi.hi + hi.lo + lo.hi)
        const uint32_t thi = smem_base + (bj & 1) * C::STAGE + C::K_BYTES, tlo = thi + C::T_BYTES;
        const uint32_t lrow = (lane & 7) + ((lane >> 4) << 3); // ldmatrix row: n within a pair of n-tiles
        const uint32_t lk = ((lane >> 3) & 1) * 8;              // k half of the 16-key chunk
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            uint32_t ah[4], al[4];
            bf16_split2(P[2 * ks][0], P[2 * ks][1], ah[0], al[0]);         // row gq,   keys 16ks+2tq..
            bf16_split2(P[2 * ks][2], P[2 * ks][3], ah[1], al[1]);         // row gq+8
            bf16_split2(P[2 * ks + 1][0], P[2 * ks + 1][1], ah[2], al[2]); // row gq,   keys 16ks+8+2tq..
            bf16_split2(P[2 * ks + 1][2], P[2 * ks + 1][3], ah[3], al[3]); // row gq+8
#pragma unroll
            for (int n = 0; n < NT; n += 2) {
                const uint32_t off = ((n * 8 + lrow) * C::TS + ks * 16 + lk) * 2;
                uint32_t bh[4], bl[4];
                ldsm_x4(thi + off, bh[0], bh[1], bh[2], bh[3]);
                ldsm_x4(tlo + off, bl[0], bl[1], bl[2], bl[3]);
                mma_bf16(acc[n], al, bh[0], bh[1]);
                mma_bf16(acc[n], ah, bl[0], bl[1]);
                mma_bf16(acc[n], ah, bh[0], bh[1]);
                mma_bf16(acc[n + 1], al, bh[2], bh[3]);
                mma_bf16(acc[n + 1], ah, bl[2], bl[3]);
                mma_bf16(acc[n + 1], ah, bh[2], bh[3]);
            }
        }
    }

    // ---- per-row results: l = quad sum; lane holds columns n*8 + 2tq, +1
#pragma unroll
    for (int x = 0; x < 2; ++x) {
        lp[x] += __shfl_xor_sync(0xffffffffu, lp[x], 1);
        lp[x] += __shfl_xor_sync(0xffffffffu, lp[x], 2);
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
        const uint32_t i = rows[x];
        if (i >= L.N)
            continue;
        float* dst;
        if (u < ndense_units) { // partial of (row, chunk)
            const size_t p = ((size_t)h * L.nd * 64 + i) * L.k4_cb + chunk;
            if (tq == 0) {
                L.part_m[p] = m64[x];
                L.part_l[p] = lp[x];
            }
            dst = L.part_acc + p * D;
        } else { // K3's initial state (no dense rows in this q-block)
            const size_t sr = row0 + i;
            if (tq == 0) {
                L.init_m[sr] = m64[x];
                L.init_l[sr] = lp[x];
            }
            dst = L.init_acc + sr * D;
        }
#pragma unroll
        for (int n = 0; n < NT; ++n)
            *reinterpret_cast<float2*>(dst + n * 8 + 2 * tq) = make_float2(acc[n][2 * x], acc[n][2 * x + 1]);
    }
}

// ---------------------------------------------------------------------------
// K4 on the 5th-generation tensor cores (default; PARO_K4_LEGACY=1 keeps the
// mma.sync kernel above). Same work units, semantics and outputs; per key tile:
//   S = Q.K^T       tcgen05.mma kind::i8, M = 64 (TMEM lanes 0-15 of each
//                   quadrant), N = 64 per column group, exact int32
//   row max / p     one thread per row (lanes 0-15 of warp w own rows 16w..):
//                   exact fp64 max as in k4_dense, p = exp2 of integer
//                   differences, split into bf16 hi + lo and written as the
//                   K-major SW128 A operand
//   O_tile = P.V    tcgen05.mma kind::f16 (bf16 x bf16 -> fp32), 3-term split
//                   Phi.Vhi + Phi.Vlo + Plo.Vhi accumulated in TMEM
//   acc = gamma acc + O_tile in registers
// K, V^T hi / lo tiles arrive by TMA, double-buffered one tile ahead.
// ---------------------------------------------------------------------------
template <int D>
struct K4T {
    static constexpr int G = D / 64;
    static constexpr uint32_t QT = 64 * D;             // Q / K code tile
    static constexpr uint32_t VT = D * 128;            // V^T bf16 tile (D rows of 64 keys)
    static constexpr uint32_t PT = 64 * 128;           // P bf16 tile (64 rows of 64 keys)
    static constexpr uint32_t STAGE = QT + 2 * VT;     // K, Vhi, Vlo (all 1024-aligned)
    static constexpr uint32_t OFF_Q = 0, OFF_ST = QT, OFF_P = OFF_ST + 2 * STAGE, OFF_BAR = OFF_P + 2 * PT;
    static constexpr uint32_t SMEM = OFF_BAR + 64;
    static constexpr uint32_t TMEM_COLS = G * 64 + D <= 128 ? 128 : 256; // S groups, then O
    static constexpr uint32_t LAYOUT = D == 64 ? ptx::kSwizzle64B : ptx::kSwizzle128B;
    static constexpr uint32_t IDESC_QK = ptx::idesc_i8(true, true, false, false, 64, 64);
    static constexpr uint32_t IDESC_PV = ptx::idesc_bf16(64, D);
};

// 16 TMEM lanes x 256 bits, 8 repetitions: the mma.sync accumulator fragment
// layout -- thread t gets rows t/4 and t/4 + 8 of its quadrant's 16 lanes,
// columns 8k + 2(t%4) + {0,1} for k = 0..7 (registers 4k..4k+3 = (r, c), (r, c+1),
// (r+8, c), (r+8, c+1)); M = 64 keeps a q-block's rows in lanes 0-15 of each quadrant
__device__ __forceinline__ void k4_ld_frag(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

template <int D>
__global__ void __launch_bounds__(128) k4_dense_tc(const __grid_constant__ LayerDev L, double scale64,
                                                   const __grid_constant__ CUtensorMap tm_q,
                                                   const __grid_constant__ CUtensorMap tm_k,
                                                   const __grid_constant__ CUtensorMap tm_vh,
                                                   const __grid_constant__ CUtensorMap tm_vl, uint32_t head_begin) {
    using C = K4T<D>;
    constexpr int G = C::G;
    constexpr int NT = D / 8; // 8-column blocks of the output
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = ptx::smem_u32(smem);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const uint32_t h = head_begin + blockIdx.y, u = blockIdx.x;
    const uint32_t ndense_units = L.nd * L.k4_cb;
    uint32_t qb, t0, t1, chunk = 0;
    if (u < ndense_units) { // q-block with dense rows, key chunk `chunk`
        qb = u / L.k4_cb;
        chunk = u % L.k4_cb;
        t0 = chunk * L.k4_ch;
        t1 = min(L.kb, t0 + L.k4_ch);
    } else { // q-block without dense rows: its dense tiles only
        qb = L.nd + (u - ndense_units);
        t0 = 0;
        t1 = L.nd;
    }
    const int32_t row0 = (int32_t)(h * L.kb2 * 64);
    const uint32_t rl[2] = {warp * 16 + gq, warp * 16 + gq + 8}; // rows within the q-block
    const uint32_t rows[2] = {qb * 64 + rl[0], qb * 64 + rl[1]};
    const uint32_t b_full = sb + C::OFF_BAR, b_q = b_full + 16, b_s = b_full + 24, b_o = b_full + 32;
    if (tid == 0) {
        ptx::mbar_init(b_full, 1);
        ptx::mbar_init(b_full + 8, 1);
        ptx::mbar_init(b_q, 1);
        ptx::mbar_init(b_s, 1);
        ptx::mbar_init(b_o, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0)
        ptx::tmem_alloc<C::TMEM_COLS>(sb + C::OFF_BAR + 48);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::OFF_BAR + 48);
    auto load_tile = [&](uint32_t bj, uint32_t st) {
        const uint32_t dst = sb + C::OFF_ST + st * C::STAGE, bar = b_full + 8 * st;
        ptx::mbar_arrive_expect_tx(bar, C::QT + 2 * C::VT);
        ptx::tma_load_2d(dst, &tm_k, 0, row0 + (int32_t)bj * 64, bar);
        const int32_t vrow = (int32_t)((h * L.kb2 + bj) * D);
        ptx::tma_load_2d(dst + C::QT, &tm_vh, 0, vrow, bar);
        ptx::tma_load_2d(dst + C::QT + C::VT, &tm_vl, 0, vrow, bar);
    };
    if (tid == 0) {
        ptx::mbar_arrive_expect_tx(b_q, C::QT);
        ptx::tma_load_2d(sb + C::OFF_Q, &tm_q, 0, row0 + (int32_t)qb * 64, b_q);
        if (t0 < t1)
            load_tile(t0, 0);
    }
    float sq[G];
#pragma unroll
    for (int g = 0; g < G; ++g)
        sq[g] = L.qsc[((size_t)h * L.kb2 + qb) * G + g];
    double m64[2] = {-INFINITY, -INFINITY};
    float lp[2] = {0.f, 0.f}; // this lane's share of l per row
    float acc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n)
        acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    const uint32_t tl = tmem + ((warp * 32) << 16); // this warp's TMEM lane quadrant (rows in lanes 0-15)
    ptx::mbar_wait(b_q, 0);
    for (uint32_t bj = t0; bj < t1; ++bj) {
        const uint32_t it = bj - t0, st = it & 1;
        if (tid == 0 && bj + 1 < t1)
            load_tile(bj + 1, st ^ 1); // that stage's previous tile finished (the loop ends in __syncthreads)
        ptx::mbar_wait(b_full + 8 * st, (it >> 1) & 1);
        const uint32_t kst = sb + C::OFF_ST + st * C::STAGE;
        if (tid == 0) { // S = Q.K^T, exact int32 per 64-column group
            ptx::tc_fence_after();
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const uint32_t off = g * 64 + kk * 32;
                    ptx::mma_i8(tmem + g * 64, ptx::smem_desc(sb + C::OFF_Q + off, 16, 8 * D, C::LAYOUT),
                                ptx::smem_desc(kst + off, 16, 8 * D, C::LAYOUT), C::IDESC_QK, kk);
                }
            ptx::mma_commit(b_s);
        }
        bool act[2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
            act[x] = rows[x] < L.N && (rows[x] < L.dp || bj < L.nd);
        const uint32_t kn = min(64u, L.N - bj * 64);
        double a[G];
        float af[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            a[g] = __dmul_rn((double)sq[g], (double)L.meta[((size_t)h * L.kb2 + bj) * meta_stride(D) + g]);
            af[g] = (float)a[g];
        }
        ptx::mbar_wait(b_s, it & 1);
        ptx::tc_fence_after();
        int32_t S[G][8][4];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            uint32_t f[32];
            k4_ld_frag(tl + g * 64, f);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    S[g][n][e] = (int32_t)f[4 * n + e];
        }
        // ---- exact row max of the tile (k4_dense): fp32 screen, fp64 on the candidates
        double best[2] = {-INFINITY, -INFINITY};
        int32_t bs[2][G];
        if constexpr (G == 1) {
            int32_t im[2] = {INT32_MIN, INT32_MIN};
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (n * 8 + 2 * tq + (e & 1) < kn)
                        im[e >> 1] = max(im[e >> 1], S[0][n][e]);
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                im[x] = max(im[x], __shfl_xor_sync(0xffffffffu, im[x], 1));
                im[x] = max(im[x], __shfl_xor_sync(0xffffffffu, im[x], 2));
                bs[x][0] = im[x];
                const int32_t sv[1] = {im[x]};
                best[x] = k4_exact<G>(scale64, a, sv);
            }
        } else {
            float mx[2] = {-INFINITY, -INFINITY}, mag[2] = {0.f, 0.f};
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t key = n * 8 + 2 * tq + (e & 1);
                    float xv = 0.f, mg = 0.f;
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float tv = af[g] * (float)S[g][n][e];
                        xv += tv;
                        mg += fabsf(tv);
                    }
                    if (key < kn) {
                        mx[e >> 1] = fmaxf(mx[e >> 1], xv);
                        mag[e >> 1] = fmaxf(mag[e >> 1], mg);
                    }
                }
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int o = 1; o <= 2; o <<= 1) {
                    mx[x] = fmaxf(mx[x], __shfl_xor_sync(0xffffffffu, mx[x], o));
                    mag[x] = fmaxf(mag[x], __shfl_xor_sync(0xffffffffu, mag[x], o));
                }
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int g = 0; g < G; ++g)
                    bs[x][g] = 0;
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int x = e >> 1;
                    const uint32_t key = n * 8 + 2 * tq + (e & 1);
                    float xv = 0.f;
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        xv += af[g] * (float)S[g][n][e];
                    if (key < kn && xv >= mx[x] - 1e-6f * mag[x]) {
                        int32_t sv[G];
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            sv[g] = S[g][n][e];
                        const double lg = k4_exact<G>(scale64, a, sv);
                        if (lg > best[x]) {
                            best[x] = lg;
#pragma unroll
                            for (int g = 0; g < G; ++g)
                                bs[x][g] = sv[g];
                        }
                    }
                }
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int o = 1; o <= 2; o <<= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, best[x], o);
                    int32_t os[G];
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        os[g] = __shfl_xor_sync(0xffffffffu, bs[x][g], o);
                    if (ob > best[x]) {
                        best[x] = ob;
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            bs[x][g] = os[g];
                    }
                }
        }
        // ---- running max, p -> bf16 hi / lo P rows (K-major, 128B swizzle: 16-B chunk n of row r at n ^ (r & 7))
        float base[2], gam[2] = {1.f, 1.f}, cg[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
            cg[g] = (float)(scale64 * a[g] * kLog2eD);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            if (!act[x]) {
                base[x] = -INFINITY;
                continue;
            }
            const double mn = fmax(m64[x], best[x]);
            if (mn != m64[x]) { // (attention.cpp:170-178); m = -inf -> gamma 0 on zero state
                gam[x] = ex2f((float)((m64[x] - mn) * kLog2eD));
                lp[x] *= gam[x];
                m64[x] = mn;
            }
            base[x] = (float)((best[x] - mn) * kLog2eD);
        }
        uint8_t* prow[2] = {smem + C::OFF_P + (rl[0] >> 3) * 1024 + (rl[0] & 7) * 128,
                            smem + C::OFF_P + (rl[1] >> 3) * 1024 + (rl[1] & 7) * 128};
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            float P[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int x = e >> 1;
                const uint32_t key = n * 8 + 2 * tq + (e & 1);
                float arg = base[x];
#pragma unroll
                for (int g = 0; g < G; ++g)
                    arg = fmaf(cg[g], (float)(S[g][n][e] - bs[x][g]), arg);
                P[e] = key < kn ? ex2f(arg) : 0.f; // base -inf (inactive row) -> 0
                lp[x] += P[e];
            }
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                uint32_t wh, wl;
                bf16_split2(P[2 * x], P[2 * x + 1], wh, wl);
                const uint32_t off = ((n ^ (rl[x] & 7)) << 4) + tq * 4;
                *reinterpret_cast<uint32_t*>(prow[x] + off) = wh;
                *reinterpret_cast<uint32_t*>(prow[x] + C::PT + off) = wl;
            }
        }
        ptx::fence_proxy_async_smem(); // P rows -> the tensor core's view
        ptx::tc_fence_before();        // S reads done before the next QK overwrites S
        __syncthreads();
        if (tid == 0) { // O_tile = Phi.Vhi + Phi.Vlo + Plo.Vhi (fp32 in TMEM)
            ptx::tc_fence_after();
            const uint32_t pa[3] = {sb + C::OFF_P, sb + C::OFF_P, sb + C::OFF_P + C::PT};
            const uint32_t vb[3] = {kst + C::QT, kst + C::QT + C::VT, kst + C::QT};
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    ptx::mma_f16(tmem + G * 64, ptx::smem_desc(pa[t] + ks * 32, 16, 1024, ptx::kSwizzle128B),
                                 ptx::smem_desc(vb[t] + ks * 32, 16, 1024, ptx::kSwizzle128B), C::IDESC_PV,
                                 (t | ks) != 0);
            ptx::mma_commit(b_o);
        }
        ptx::mbar_wait(b_o, it & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c64 = 0; c64 < D / 64; ++c64) {
            uint32_t f[32];
            k4_ld_frag(tl + G * 64 + c64 * 64, f);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    acc[c64 * 8 + n][e] = fmaf(acc[c64 * 8 + n][e], gam[e >> 1], __uint_as_float(f[4 * n + e]));
        }
        ptx::tc_fence_before();
        __syncthreads(); // P, S, O and this tile's stage are free again
    }
    // ---- per-row results (as k4_dense): l = quad sum; lane holds columns n*8 + 2tq, +1
#pragma unroll
    for (int x = 0; x < 2; ++x) {
        lp[x] += __shfl_xor_sync(0xffffffffu, lp[x], 1);
        lp[x] += __shfl_xor_sync(0xffffffffu, lp[x], 2);
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
        const uint32_t i = rows[x];
        if (i >= L.N)
            continue;
        float* dst;
        if (u < ndense_units) { // partial of (row, chunk)
            const size_t pp = ((size_t)h * L.nd * 64 + i) * L.k4_cb + chunk;
            if (tq == 0) {
                L.part_m[pp] = m64[x];
                L.part_l[pp] = lp[x];
            }
            dst = L.part_acc + pp * D;
        } else { // K3's initial state (no dense rows in this q-block)
            const size_t sr = (size_t)row0 + i;
            if (tq == 0) {
                L.init_m[sr] = m64[x];
                L.init_l[sr] = lp[x];
            }
            dst = L.init_acc + sr * D;
        }
#pragma unroll
        for (int n = 0; n < NT; ++n)
            *reinterpret_cast<float2*>(dst + n * 8 + 2 * tq) = make_float2(acc[n][2 * x], acc[n][2 * x + 1]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0)
        ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// final dense row (original token order, attention.cpp:242-251) or K3's initial state
template <int D>
__device__ __forceinline__ void k4_finish(const LayerDev& L, uint32_t h, uint32_t i, double m64, float l,
                                          const float (&acc)[D / 2], float* __restrict__ out,
                                          uint8_t* __restrict__ zeroed) {
    constexpr int DH = D / 2;
    const uint32_t hf = threadIdx.x >> 6;
    if (i >= L.N)
        return;
    if (i < L.dp) {
        const uint32_t orig = perm_src(L.perm[h], i);
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)h * L.N + orig) * D + hf * DH);
        const float il = l == 0.f ? 0.f : 1.0f / l;
#pragma unroll
        for (int c = 0; c < DH / 4; ++c)
            dst[c] = make_float4(acc[4 * c] * il, acc[4 * c + 1] * il, acc[4 * c + 2] * il, acc[4 * c + 3] * il);
        if (zeroed && hf == 0)
            zeroed[(size_t)h * L.N + orig] = l == 0.f ? 1 : 0;
    } else {
        const size_t s = (size_t)h * L.kb2 * 64 + i;
        if (hf == 0) {
            L.init_m[s] = m64;
            L.init_l[s] = l;
        }
        float4* dst = reinterpret_cast<float4*>(L.init_acc + s * D + hf * DH);
#pragma unroll
        for (int c = 0; c < DH / 4; ++c)
            dst[c] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
    }
}

// merge the CB key-chunk partials of the rows of the nd dense q-blocks
template <int D>
__global__ void __launch_bounds__(128) k4_combine(LayerDev L, float* __restrict__ out, uint8_t* __restrict__ zeroed,
                                                  uint32_t head_begin) {
    constexpr int DH = D / 2;
    const uint32_t h = head_begin + blockIdx.y, qb = blockIdx.x;
    const uint32_t r = threadIdx.x & 63, hf = threadIdx.x >> 6;
    const uint32_t i = qb * 64 + r;
    if (i >= L.N)
        return;
    const size_t p0 = ((size_t)h * L.nd * 64 + qb * 64 + r) * L.k4_cb;
    double m64 = -INFINITY;
    for (uint32_t c = 0; c < L.k4_cb; ++c)
        m64 = fmax(m64, L.part_m[p0 + c]);
    float l = 0.f;
    float acc[DH];
#pragma unroll
    for (int e = 0; e < DH; ++e)
        acc[e] = 0.f;
    for (uint32_t c = 0; c < L.k4_cb; ++c) {
        const float lc = L.part_l[p0 + c];
        if (lc == 0.f)
            continue;
        const float gam = ex2f((float)((L.part_m[p0 + c] - m64) * kLog2eD));
        l = fmaf(lc, gam, l);
        const float4* src = reinterpret_cast<const float4*>(L.part_acc + (p0 + c) * D + hf * DH);
#pragma unroll
        for (int e = 0; e < DH / 4; ++e) {
            const float4 a = src[e];
            acc[4 * e] = fmaf(a.x, gam, acc[4 * e]);
            acc[4 * e + 1] = fmaf(a.y, gam, acc[4 * e + 1]);
            acc[4 * e + 2] = fmaf(a.z, gam, acc[4 * e + 2]);
            acc[4 * e + 3] = fmaf(a.w, gam, acc[4 * e + 3]);
        }
    }
    k4_finish<D>(L, h, i, m64, l, acc, out, zeroed);
}

// key chunks for the dense q-blocks: about 4096 dense units over all heads,
// at least 8 tiles per chunk
void k4_chunking(uint32_t kb, uint32_t nd, uint32_t heads, uint32_t& cb, uint32_t& ch) {
    const uint64_t work = (uint64_t)kb * nd * heads;
    ch = (uint32_t)((work + 4095) / 4096);
    if (ch < 8)
        ch = 8;
    if (ch > kb)
        ch = kb;
    cb = (kb + ch - 1) / ch;
}

// K4a: the dense-prefix path's bf16 hi/lo V^T tiles, split from the fp32 V at
// reorder_quantize time (so attention never reads the caller's fp32 V)
cudaError_t launch_k4a(const LayerDev& L, const float* v, uint32_t head_begin, uint32_t head_count, cudaStream_t st) {
    if (L.dp == 0 || head_count == 0)
        return cudaSuccess;
    const dim3 vgrid(L.kb, head_count);
    if (L.D == 64)
        k4_vsplit<64><<<vgrid, 256, 0, st>>>(L, v, head_begin);
    else
        k4_vsplit<128><<<vgrid, 256, 0, st>>>(L, v, head_begin);
    return cudaGetLastError();
}

cudaError_t launch_k4(const LayerDev& L, double scale, float* out, uint8_t* zeroed, uint32_t head_begin,
                      uint32_t head_count, cudaStream_t st, const CUtensorMap* tq, const CUtensorMap* tk,
                      const CUtensorMap* tvh, const CUtensorMap* tvl) {
    if (L.dp == 0 || head_count == 0)
        return cudaSuccess;
    const dim3 grid(L.nd * L.k4_cb + (L.kb - L.nd), head_count);
    const dim3 cgrid(L.nd, head_count);
    static const bool legacy = getenv("PARO_K4_LEGACY") && atoi(getenv("PARO_K4_LEGACY")) != 0;
    if (!legacy && tvh) { // tcgen05 K4 (the combine kernel is shared)
        cudaError_t e;
        if (L.D == 64) {
            if ((e = cudaFuncSetAttribute(k4_dense_tc<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)K4T<64>::SMEM)) != cudaSuccess)
                return e;
            k4_dense_tc<64><<<grid, 128, K4T<64>::SMEM, st>>>(L, scale, *tq, *tk, *tvh, *tvl, head_begin);
            k4_combine<64><<<cgrid, 128, 0, st>>>(L, out, zeroed, head_begin);
        } else {
            if ((e = cudaFuncSetAttribute(k4_dense_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)K4T<128>::SMEM)) != cudaSuccess)
                return e;
            k4_dense_tc<128><<<grid, 128, K4T<128>::SMEM, st>>>(L, scale, *tq, *tk, *tvh, *tvl, head_begin);
            k4_combine<128><<<cgrid, 128, 0, st>>>(L, out, zeroed, head_begin);
        }
        return cudaGetLastError();
    }
    if (L.D == 64) {
        constexpr size_t smem = K4Cfg<64>::SMEM;
        cudaFuncSetAttribute(k4_dense<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k4_dense<64><<<grid, 128, smem, st>>>(L, scale, out, zeroed, head_begin);
        k4_combine<64><<<cgrid, 128, 0, st>>>(L, out, zeroed, head_begin);
    } else {
        constexpr size_t smem = K4Cfg<128>::SMEM;
        cudaFuncSetAttribute(k4_dense<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k4_dense<128><<<grid, 128, smem, st>>>(L, scale, out, zeroed, head_begin);
        k4_combine<128><<<cgrid, 128, 0, st>>>(L, out, zeroed, head_begin);
    }
    return cudaGetLastError();
}

} // namespace paro
