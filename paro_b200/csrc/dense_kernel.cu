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
// these tiles carry no codes). One CTA per (q-block, head), one thread per row;
// the K-code tile and the permuted fp32 V tile are staged in shared memory.
#include <cuda_runtime.h>

#include <cstdint>

#include "layer.cuh"

namespace paro {

constexpr double kLog2eD = 1.4426950408889634;

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int D>
__global__ void __launch_bounds__(64) k4_dense_prefix(LayerDev L, const float* __restrict__ v, double scale64,
                                                      float* __restrict__ out, uint8_t* __restrict__ zeroed,
                                                      uint32_t head_begin) {
    constexpr int G = D / 64;
    constexpr int W = D / 4; // int32 words of one code row
    const uint32_t qb = blockIdx.x, h = head_begin + blockIdx.y;
    const uint32_t r = threadIdx.x;
    const uint32_t i = qb * 64 + r; // permuted row
    const uint32_t q0 = qb * 64;
    const uint32_t ntiles = q0 < L.dp ? L.kb : L.nd; // tiles the CTA has to stage
    __shared__ __align__(16) int32_t ks[64][W];
    __shared__ __align__(16) float vs[64][D];
    __shared__ float ksc[G];
    const bool row_valid = i < L.N;
    const bool row_dense = i < L.dp;
    const uint32_t my_tiles = row_dense ? L.kb : L.nd;
    const PermDesc pd = L.perm[h];
    const size_t row0 = (size_t)h * L.kb2 * 64;
    int32_t qv[W];
    {
        const int4* src = reinterpret_cast<const int4*>(L.q + (row0 + i) * D);
#pragma unroll
        for (int w = 0; w < W / 4; ++w) {
            const int4 t = src[w];
            qv[4 * w] = t.x;
            qv[4 * w + 1] = t.y;
            qv[4 * w + 2] = t.z;
            qv[4 * w + 3] = t.w;
        }
    }
    float sq[G];
#pragma unroll
    for (int g = 0; g < G; ++g)
        sq[g] = L.qsc[((size_t)h * L.kb2 + qb) * G + g];
    double m64 = -INFINITY;
    float l = 0.f;
    float acc[D];
#pragma unroll
    for (int c = 0; c < D; ++c)
        acc[c] = 0.f;
    for (uint32_t bj = 0; bj < ntiles; ++bj) {
        __syncthreads(); // previous tile consumed
        { // stage the K codes (row j = thread) and the permuted fp32 V rows of tile bj
            const uint32_t j = threadIdx.x, kj = bj * 64 + j;
            const int4* ksrc = reinterpret_cast<const int4*>(L.k + (row0 + kj) * D);
#pragma unroll
            for (int w = 0; w < W / 4; ++w)
                reinterpret_cast<int4*>(ks[j])[w] = ksrc[w];
            if (kj < L.N) {
                const float4* vsrc = reinterpret_cast<const float4*>(v + ((size_t)h * L.N + perm_src(pd, kj)) * D);
#pragma unroll
                for (int w = 0; w < D / 4; ++w)
                    reinterpret_cast<float4*>(vs[j])[w] = vsrc[w];
            } else {
#pragma unroll
                for (int w = 0; w < D / 4; ++w)
                    reinterpret_cast<float4*>(vs[j])[w] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (threadIdx.x < G)
                ksc[threadIdx.x] = L.meta[((size_t)h * L.kb2 + bj) * meta_stride(D) + threadIdx.x];
        }
        __syncthreads();
        if (!row_valid || bj >= my_tiles)
            continue;
        const uint32_t kn = min(64u, L.N - bj * 64);
        double a[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
            a[g] = __dmul_rn((double)sq[g], (double)ksc[g]);
        auto logit = [&](uint32_t j) -> double { // attention.cpp:162-168 with the INT8-QK dot
            double accg = 0.0;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                int32_t s = 0;
#pragma unroll
                for (int w = 0; w < 16; ++w)
                    s = __dp4a(qv[g * 16 + w], ks[j][g * 16 + w], s);
                accg = __dadd_rn(accg, __dmul_rn(a[g], (double)s));
            }
            return __dmul_rn(scale64, accg);
        };
        double tmax = -INFINITY;
        for (uint32_t j = 0; j < kn; ++j)
            tmax = fmax(tmax, logit(j));
        const double m_new = fmax(m64, tmax);
        if (l > 0.f && m_new != m64) { // rescale (attention.cpp:170-178)
            const float gam = ex2f((float)((m64 - m_new) * kLog2eD));
            l *= gam;
#pragma unroll
            for (int c = 0; c < D; ++c)
                acc[c] *= gam;
        }
        m64 = m_new;
        for (uint32_t j = 0; j < kn; ++j) { // p = exp(s - m), l += p, acc += p * v (:181-199)
            const float p = ex2f((float)((logit(j) - m_new) * kLog2eD));
            l += p;
#pragma unroll
            for (int c = 0; c < D; ++c)
                acc[c] = fmaf(p, vs[j][c], acc[c]);
        }
    }
    if (!row_valid)
        return;
    if (row_dense) { // final row, stored at its original token (attention.cpp:242-251)
        const uint32_t orig = perm_src(pd, i);
        float* dst = out + ((size_t)h * L.N + orig) * D;
        if (l == 0.f) {
#pragma unroll
            for (int c = 0; c < D; ++c)
                dst[c] = 0.f;
        } else {
            const float il = 1.0f / l;
#pragma unroll
            for (int c = 0; c < D; ++c)
                dst[c] = acc[c] * il;
        }
        if (zeroed)
            zeroed[(size_t)h * L.N + orig] = l == 0.f ? 1 : 0;
    } else { // hand the running state to K3
        const size_t s = row0 + i;
        L.init_m[s] = m64;
        L.init_l[s] = l;
#pragma unroll
        for (int c = 0; c < D; ++c)
            L.init_acc[s * D + c] = acc[c];
    }
}

cudaError_t launch_k4(const LayerDev& L, const float* v, double scale, float* out, uint8_t* zeroed,
                      uint32_t head_begin, uint32_t head_count, cudaStream_t st) {
    if (L.dp == 0 || head_count == 0)
        return cudaSuccess;
    const dim3 grid(L.kb, head_count);
    if (L.D == 64)
        k4_dense_prefix<64><<<grid, 64, 0, st>>>(L, v, scale, out, zeroed, head_begin);
    else
        k4_dense_prefix<128><<<grid, 64, 0, st>>>(L, v, scale, out, zeroed, head_begin);
    return cudaGetLastError();
}

} // namespace paro
