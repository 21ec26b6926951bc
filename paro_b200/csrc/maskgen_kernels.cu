// maskgen_kernels.cu -- K5: the producer of K3's block mask on the GPU
// (SURVEY.md 8(f) rank 2): the permuted block sums of a calibration attention
// map (apply_perm_map + block_sums, reorder.cpp:103-114 + metrics.cpp:41-58,
// fused: the N x N map is read once, the permuted map never exists) and the
// keep-order mask selection of gen_mask / build_schedule (mask.cpp:56-172).
//
// Bit-exactness: block sums follow the reference's scalar order exactly
// (per permuted row, per permuted column block: a sequential fp64 sum of |a|
// over the block's columns in permuted order, kernels_scalar.cpp:30-35; rows
// accumulated in order into a zero-initialised fp64 grid). gen_mask's
// selection is order-exact (strict total order: larger sum, then smaller
// (row, col)), including guard blocks and the degenerate-row repair.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "ptx.cuh"

namespace paro {

// ---------------------------------------------------------------------------
// K5a: permuted block sums. One warp per (permuted row block bi, permuted
// column block bj): lane l sums |a| over the block's columns in permuted order
// for its rows (l, l+32, ...; a sequential fp64 sum per row, as sum_abs_scalar),
// then lane 0 adds the row sums in row order (block_sums' accumulation). The
// column gathers hit L2: a row block's rows (block x N x 4 B) are read by all
// k column-block warps of that row block, which the grid schedules together.
// ---------------------------------------------------------------------------
constexpr int K5_WARPS = 8;
constexpr int K5_MAXBLOCK = 256;

template <bool STATS>
__global__ void __launch_bounds__(K5_WARPS * 32) k5_perm_block_sums(const float* __restrict__ map, size_t ld,
                                                                    uint32_t n, const uint32_t* __restrict__ inv,
                                                                    uint32_t block, uint32_t k, float eps,
                                                                    double* __restrict__ sums, float* __restrict__ maxs,
                                                                    uint32_t* __restrict__ counts) {
    __shared__ double racc[K5_WARPS][K5_MAXBLOCK];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bi = blockIdx.x, bj = blockIdx.y * K5_WARPS + warp;
    if (bj >= k)
        return;
    const uint32_t r0 = bi * block, r1 = min(n, r0 + block);
    const uint32_t c0 = bj * block, c1 = min(n, c0 + block);
    float mx = 0.f;
    uint32_t cnt = 0;
    for (uint32_t rp = r0 + lane; rp < r1; rp += 32) {
        const uint32_t i = inv ? __ldg(inv + rp) : rp;
        const float* row = map + (size_t)i * ld;
        double acc = 0.0; // sum_abs_scalar order over the permuted columns
        uint32_t cp = c0;
        for (; cp + 8 <= c1; cp += 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = __ldg(row + (inv ? __ldg(inv + cp + u) : cp + u));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                acc = __dadd_rn(acc, fabs((double)v[u]));
                if (STATS) {
                    mx = fmaxf(mx, fabsf(v[u]));
                    cnt += fabsf(v[u]) < eps ? 1u : 0u;
                }
            }
        }
        for (; cp < c1; ++cp) {
            const float v = __ldg(row + (inv ? __ldg(inv + cp) : cp));
            acc = __dadd_rn(acc, fabs((double)v));
            if (STATS) {
                mx = fmaxf(mx, fabsf(v));
                cnt += fabsf(v) < eps ? 1u : 0u;
            }
        }
        racc[warp][rp - r0] = acc;
    }
    if (STATS) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
    }
    __syncwarp();
    if (lane == 0) {
        double tot = 0.0; // rows accumulated in order into the zero-initialised grid
        for (uint32_t r = 0; r < r1 - r0; ++r)
            tot = __dadd_rn(tot, racc[warp][r]);
        sums[(size_t)bi * k + bj] = tot;
        if (STATS) {
            maxs[(size_t)bi * k + bj] = mx;
            counts[(size_t)bi * k + bj] = cnt;
        }
    }
}

// ---------------------------------------------------------------------------
// K5a (staged, the default when 3 x N x 4 B fits shared memory: N <= 18.9K):
// one CTA per permuted row block walks its rows in order; the permutation's
// inverse table and a double-buffered copy of the current / next original row
// live in shared memory (the next row is prefetched into registers while the
// current one is reduced), and thread t owns column blocks t, t + 512, ...:
// a sequential fp64 sum of |a| over the block's columns in permuted order
// (sum_abs_scalar), added in row order to its running block totals.
// ---------------------------------------------------------------------------
constexpr int K5S_THREADS = 512;
constexpr int K5S_MAXB = 4; // column blocks per thread (k <= 2048)
constexpr int K5S_PF = 40;  // prefetched row words per thread (n <= 20480)

template <bool STATS>
__global__ void __launch_bounds__(K5S_THREADS) k5_perm_block_sums_staged(const float* __restrict__ map, size_t ld,
                                                                        uint32_t n, const uint32_t* __restrict__ inv,
                                                                        uint32_t block, uint32_t k, float eps,
                                                                        double* __restrict__ sums,
                                                                        float* __restrict__ maxs,
                                                                        uint32_t* __restrict__ counts) {
    extern __shared__ __align__(16) uint32_t sm[];
    // inverse table transposed, sinvT[u * k + bj] = inv[bj * block + u]: the
    // threads of a warp (consecutive bj) read consecutive words (no bank conflicts)
    const uint32_t kb = k * block;
    uint32_t* sinvT = sm;                               // [block][k]
    float* srow0 = reinterpret_cast<float*>(sm + kb);   // [n]
    float* srow1 = srow0 + n;                           // [n]
    const uint32_t bi = blockIdx.x;
    const uint32_t r0 = bi * block, r1 = min(n, r0 + block);
    for (uint32_t c = threadIdx.x; c < kb; c += K5S_THREADS) {
        const uint32_t u = c / k, bj = c - u * k, cp = bj * block + u;
        sinvT[c] = cp < n ? (inv ? __ldg(inv + cp) : cp) : 0u;
    }
    double tot[K5S_MAXB];
    float tmx[K5S_MAXB];
    uint32_t tcnt[K5S_MAXB];
#pragma unroll
    for (int q = 0; q < K5S_MAXB; ++q) {
        tot[q] = 0.0;
        tmx[q] = 0.f;
        tcnt[q] = 0;
    }
    float pf[K5S_PF];
    auto fetch = [&](uint32_t rp) { // original row of permuted row rp -> registers
        const float* row = map + (size_t)(inv ? __ldg(inv + rp) : rp) * ld;
#pragma unroll
        for (int u = 0; u < K5S_PF; ++u) {
            const uint32_t c = threadIdx.x + (uint32_t)u * K5S_THREADS;
            pf[u] = c < n ? __ldcs(row + c) : 0.f;
        }
    };
    auto stash = [&](float* dst) {
#pragma unroll
        for (int u = 0; u < K5S_PF; ++u) {
            const uint32_t c = threadIdx.x + (uint32_t)u * K5S_THREADS;
            if (c < n)
                dst[c] = pf[u];
        }
    };
    fetch(r0);
    stash(srow0);
    __syncthreads();
    for (uint32_t rp = r0; rp < r1; ++rp) {
        const float* cur = ((rp - r0) & 1) ? srow1 : srow0;
        float* nxt = ((rp - r0) & 1) ? srow0 : srow1;
        if (rp + 1 < r1)
            fetch(rp + 1); // in flight while this row is reduced
#pragma unroll
        for (int q = 0; q < K5S_MAXB; ++q) {
            const uint32_t bj = threadIdx.x + (uint32_t)q * K5S_THREADS;
            if (bj < k) {
                const uint32_t c0 = bj * block, c1 = min(n, c0 + block);
                double acc = 0.0;
                uint32_t cp = c0;
                for (; cp + 8 <= c1; cp += 8) {
                    float v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        v[u] = cur[sinvT[(cp - c0 + u) * k + bj]];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        acc = __dadd_rn(acc, fabs((double)v[u]));
                        if (STATS) { // max_abs / count_abs_lt (order-free)
                            tmx[q] = fmaxf(tmx[q], fabsf(v[u]));
                            tcnt[q] += fabsf(v[u]) < eps ? 1u : 0u;
                        }
                    }
                }
                for (; cp < c1; ++cp) {
                    const float v = cur[sinvT[(cp - c0) * k + bj]];
                    acc = __dadd_rn(acc, fabs((double)v));
                    if (STATS) {
                        tmx[q] = fmaxf(tmx[q], fabsf(v));
                        tcnt[q] += fabsf(v) < eps ? 1u : 0u;
                    }
                }
                tot[q] = __dadd_rn(tot[q], acc);
            }
        }
        if (rp + 1 < r1)
            stash(nxt); // nxt was last read two rows ago (barrier below separates)
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < K5S_MAXB; ++q) {
        const uint32_t bj = threadIdx.x + (uint32_t)q * K5S_THREADS;
        if (bj < k) {
            sums[(size_t)bi * k + bj] = tot[q];
            if (STATS) {
                maxs[(size_t)bi * k + bj] = tmx[q];
                counts[(size_t)bi * k + bj] = tcnt[q];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K5a, TMA variant (block <= 64, n <= K5T_MAXN): same sums / stats and the same
// fp64 order as the staged kernel, restructured so HBM streams while the sums
// run: each original row arrives in shared memory by ONE 1-D bulk copy (three
// row buffers, two rows in flight ahead of the one being reduced), and each
// thread keeps its column block's source columns in registers (16-bit pairs)
// instead of re-reading an inverse table per element. Measured at c2 (one
// 1.23 GB map): 0.24 ms for the reordering candidates; the identity order is
// 1.23 ms -- its 32 lanes (consecutive column blocks, 64 floats apart) read one
// shared-memory bank per step. Splitting the row into padded 256-B bulk copies
// removes that conflict but costs more than it saves (1.30 ms for every order:
// small bulk copies are issue-bound), so the single copy stays.
// ---------------------------------------------------------------------------
constexpr int K5T_NBUF = 3;
constexpr uint32_t K5T_MAXN = 18900; // 3 row buffers of (n + 8) floats within 227 KB

template <bool STATS>
__global__ void __launch_bounds__(512) k5_perm_block_sums_tma(const float* __restrict__ map, size_t ld, uint32_t n,
                                                            const uint32_t* __restrict__ inv, uint32_t block,
                                                            uint32_t k, float eps, double* __restrict__ sums,
                                                            float* __restrict__ maxs,
                                                            uint32_t* __restrict__ counts) {
    extern __shared__ __align__(16) uint8_t k5t_smem[];
    const uint32_t rb = ((n + 8) * 4 + 15) & ~15u; // bytes per row buffer
    float* bufs = reinterpret_cast<float*>(k5t_smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(k5t_smem + K5T_NBUF * rb);
    uint32_t* shift = reinterpret_cast<uint32_t*>(bars + K5T_NBUF);
    const uint32_t sbase = ptx::smem_u32(k5t_smem), bar0 = ptx::smem_u32(bars);
    const uint32_t bi = blockIdx.x, tid = threadIdx.x;
    const uint32_t r0 = bi * block, r1 = min(n, r0 + block), rows = r1 - r0;
    // this thread's column block: its permuted columns' original columns, 2 per word
    const uint32_t bj = tid, c0 = bj * block;
    const uint32_t len = bj < k ? min(n, c0 + block) - c0 : 0u;
    uint32_t idx[32];
#pragma unroll
    for (int w = 0; w < 32; ++w) {
        const uint32_t u = 2 * w;
        const uint32_t a = u < len ? (inv ? __ldg(inv + c0 + u) : c0 + u) : 0u;
        const uint32_t b = u + 1 < len ? (inv ? __ldg(inv + c0 + u + 1) : c0 + u + 1) : 0u;
        idx[w] = a | b << 16;
    }
    // row r0 + j -> buffer j % NBUF (thread 0): the 16-B aligned body by one bulk
    // copy from the row's aligned floor, the <= 3 trailing floats by plain loads
    auto issue = [&](uint32_t j) {
        const uint32_t orig = inv ? __ldg(inv + r0 + j) : r0 + j;
        const float* src = map + (size_t)orig * ld;
        const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
        const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(src) - a) / 4;
        const uint32_t full = (sh + n) * 4, body = full & ~15u;
        const uint32_t b = j % K5T_NBUF;
        float* dst = bufs + (size_t)b * (rb / 4);
        for (uint32_t c = body / 4; c < full / 4; ++c)
            dst[c] = reinterpret_cast<const float*>(a)[c];
        shift[b] = sh;
        ptx::mbar_arrive_expect_tx(bar0 + 8 * b, body);
        if (body)
            ptx::bulk_load(sbase + b * rb, reinterpret_cast<const void*>(a), body, bar0 + 8 * b);
    };
    if (tid == 0) {
        for (int b = 0; b < K5T_NBUF; ++b)
            ptx::mbar_init(bar0 + 8 * b, 1);
        ptx::fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0)
        for (uint32_t j = 0; j < min(rows, (uint32_t)K5T_NBUF); ++j)
            issue(j);
    double tot = 0.0;
    float tmx = 0.f;
    uint32_t tcnt = 0;
    for (uint32_t j = 0; j < rows; ++j) {
        const uint32_t b = j % K5T_NBUF;
        ptx::mbar_wait(bar0 + 8 * b, (j / K5T_NBUF) & 1);
        const float* cur = bufs + (size_t)b * (rb / 4) + shift[b];
        if (len && !inv && len == 64) {
            // identity order: the block's 64 columns are contiguous -> 16-B loads
            // (4 values per shared-memory wavefront where scalar gathers get 1;
            // the warp's blocks are 256 B apart, one bank group)
            const uint32_t sh = shift[b];
            const float4* base = reinterpret_cast<const float4*>(bufs + (size_t)b * (rb / 4)) + ((c0 + sh) >> 2);
            double acc = 0.0;
            auto add = [&](float v) {
                acc = __dadd_rn(acc, fabs((double)v));
                if (STATS) {
                    tmx = fmaxf(tmx, fabsf(v));
                    tcnt += fabsf(v) < eps ? 1u : 0u;
                }
            };
            auto run = [&](auto off_c) { // columns c0 .. c0+63 start at word `off` of base[0]
                constexpr int OFF = decltype(off_c)::value;
#pragma unroll
                for (int q = 0; q < 4; ++q) { // 16 columns per quarter
                    float f[20];
#pragma unroll
                    for (int t = 0; t < 5; ++t) {
                        if (t == 4 && OFF == 0)
                            break;
                        const float4 x = base[q * 4 + t];
                        f[4 * t] = x.x;
                        f[4 * t + 1] = x.y;
                        f[4 * t + 2] = x.z;
                        f[4 * t + 3] = x.w;
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        add(f[OFF + i]);
                }
            };
            switch ((c0 + sh) & 3u) {
            case 0: run(std::integral_constant<int, 0>{}); break;
            case 1: run(std::integral_constant<int, 1>{}); break;
            case 2: run(std::integral_constant<int, 2>{}); break;
            default: run(std::integral_constant<int, 3>{}); break;
            }
            tot = __dadd_rn(tot, acc);
        } else if (len) {
            double acc = 0.0; // the reference's per-row order (staged kernel), then tot += acc
#pragma unroll
            for (int w = 0; w < 32; ++w) {
                if (2u * w < len) {
                    const float v0 = cur[idx[w] & 0xffffu];
                    acc = __dadd_rn(acc, fabs((double)v0));
                    if (STATS) {
                        tmx = fmaxf(tmx, fabsf(v0));
                        tcnt += fabsf(v0) < eps ? 1u : 0u;
                    }
                }
                if (2u * w + 1 < len) {
                    const float v1 = cur[idx[w] >> 16];
                    acc = __dadd_rn(acc, fabs((double)v1));
                    if (STATS) {
                        tmx = fmaxf(tmx, fabsf(v1));
                        tcnt += fabsf(v1) < eps ? 1u : 0u;
                    }
                }
            }
            tot = __dadd_rn(tot, acc);
        }
        __syncthreads(); // buffer b free
        if (tid == 0 && j + K5T_NBUF < rows)
            issue(j + K5T_NBUF);
    }
    if (len) {
        sums[(size_t)bi * k + bj] = tot;
        if (STATS) {
            maxs[(size_t)bi * k + bj] = tmx;
            counts[(size_t)bi * k + bj] = tcnt;
        }
    }
}

// ---------------------------------------------------------------------------
// K5b: gen_mask for `count` independent (kr x kc) sum grids, one CTA each.
// Keep order: rank key = ~ord(sum) (ord: order-preserving map of fp64 to u64,
// so a smaller key is a larger sum), ties by row-major index (row, col). The
// K = target - guard_count most preferred non-guard blocks are found by an
// exact 64-bit radix select (8 passes of 8 bits) plus an index-ordered prefix
// count among the boundary ties; guard blocks are set; then the reference's
// degenerate-row repair runs with CTA-wide argmax / arg-least-preferred scans.
// ---------------------------------------------------------------------------
constexpr int K5G_THREADS = 1024;

__device__ __forceinline__ uint64_t rank_key(double s) {
    s = __dadd_rn(s, 0.0); // -0.0 == +0.0 in the reference's comparisons
    uint64_t u = (uint64_t)__double_as_longlong(s);
    u = (u >> 63) ? ~u : (u | 0x8000000000000000ull); // ascending with s
    return ~u;                                           // ascending with preference
}

__device__ __forceinline__ uint64_t block_reduce_min_u64(uint64_t v, uint64_t* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0)
        sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (K5G_THREADS / 32) ? sh[threadIdx.x] : ~0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
            v = w < v ? w : v;
        }
        if (threadIdx.x == 0)
            sh[0] = v;
    }
    __syncthreads();
    return sh[0];
}

__global__ void __launch_bounds__(K5G_THREADS) k5_gen_mask(const double* __restrict__ sums_all, uint32_t kr,
                                                           uint32_t kc, uint32_t guard, uint64_t K,
                                                           uint8_t* __restrict__ bits_all, uint32_t* __restrict__ row_kept_all,
                                                           uint32_t* __restrict__ repaired_out, int* __restrict__ status) {
    const size_t total = (size_t)kr * kc;
    const double* sums = sums_all + (size_t)blockIdx.x * total;
    uint8_t* bits = bits_all + (size_t)blockIdx.x * total;
    uint32_t* row_kept = row_kept_all + (size_t)blockIdx.x * kr;
    __shared__ uint32_t hist[256];
    __shared__ uint64_t sh64[32];
    __shared__ uint64_t s_prefix, s_rank;
    __shared__ uint32_t s_scan[K5G_THREADS];
    auto guarded = [&](size_t idx) { return (idx / kc) < guard || (idx % kc) < guard; };

    // ---- exact radix select of the K-th (1-based) smallest rank key among candidates
    uint64_t prefix = 0, mask_hi = 0, rank = K; // rank: 1-based position still to find
    for (int pass = 0; pass < 8 && K > 0; ++pass) {
        const int shift = 56 - 8 * pass;
        for (int b = threadIdx.x; b < 256; b += K5G_THREADS)
            hist[b] = 0;
        __syncthreads();
        for (size_t idx = threadIdx.x; idx < total; idx += K5G_THREADS) {
            if (guarded(idx))
                continue;
            const uint64_t key = rank_key(sums[idx]);
            if ((key & mask_hi) == prefix)
                atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t cum = 0;
            uint32_t b = 0;
            for (; b < 256; ++b) {
                if (cum + hist[b] >= rank)
                    break;
                cum += hist[b];
            }
            s_prefix = prefix | ((uint64_t)b << shift);
            s_rank = rank - cum;
        }
        __syncthreads();
        prefix = s_prefix;
        rank = s_rank;
        mask_hi |= 0xffull << shift;
    }
    const uint64_t tkey = prefix; // the K-th key; `rank` of its ties (in index order) are kept
    // ---- mark: guard blocks, keys below tkey, and the first `rank` ties in index order
    const size_t per = (total + K5G_THREADS - 1) / K5G_THREADS; // contiguous index range per thread
    const size_t lo = (size_t)threadIdx.x * per, hi = min(total, lo + per);
    uint32_t ties = 0;
    if (K > 0)
        for (size_t idx = lo; idx < hi; ++idx)
            if (!guarded(idx) && rank_key(sums[idx]) == tkey)
                ++ties;
    s_scan[threadIdx.x] = ties;
    __syncthreads();
    for (int o = 1; o < K5G_THREADS; o <<= 1) { // inclusive scan
        const uint32_t v = threadIdx.x >= (unsigned)o ? s_scan[threadIdx.x - o] : 0u;
        __syncthreads();
        s_scan[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t tie_rank = s_scan[threadIdx.x] - ties; // ties before this thread's range
    for (size_t idx = lo; idx < hi; ++idx) {
        uint8_t keep = 0;
        if (guarded(idx))
            keep = 1;
        else if (K > 0) {
            const uint64_t key = rank_key(sums[idx]);
            if (key < tkey)
                keep = 1;
            else if (key == tkey)
                keep = (uint64_t)(tie_rank++) < rank ? 1 : 0;
        }
        bits[idx] = keep;
    }
    __syncthreads();
    // ---- row counts
    for (uint32_t i = threadIdx.x; i < kr; i += K5G_THREADS) {
        uint32_t c = 0;
        for (uint32_t j = 0; j < kc; ++j)
            c += bits[(size_t)i * kc + j];
        row_kept[i] = c;
    }
    __syncthreads();
    // ---- degenerate-row repair (mask.cpp:95-128), rows in order; rare
    uint32_t repaired = 0;
    for (uint32_t i = 0; i < kr; ++i) {
        if (row_kept[i] > 0) // uniform: written before the last barrier
            continue;
        // best = first argmax of sums over row i (strict '>' scan, mask.cpp:100-103):
        // the smallest rank key, then the smallest j
        // full-precision argmax: reduce (key) then the smallest j with that key
        uint64_t kmin = ~0ull;
        for (uint32_t j = threadIdx.x; j < kc; j += K5G_THREADS) {
            const uint64_t key = rank_key(sums[(size_t)i * kc + j]);
            kmin = key < kmin ? key : kmin;
        }
        kmin = block_reduce_min_u64(kmin, sh64);
        uint64_t jmin = ~0ull;
        for (uint32_t j = threadIdx.x; j < kc; j += K5G_THREADS)
            if (rank_key(sums[(size_t)i * kc + j]) == kmin)
                jmin = (uint64_t)j < jmin ? (uint64_t)j : jmin;
        jmin = block_reduce_min_u64(jmin, sh64);
        if (threadIdx.x == 0) {
            bits[(size_t)i * kc + jmin] = 1;
            row_kept[i] += 1;
        }
        ++repaired;
        __syncthreads();
        // drop the least-preferred kept non-guard block whose row keeps >= 2
        // (largest (rank key, index) -> reduce the complement)
        uint64_t wkey = ~0ull;
        for (size_t idx = threadIdx.x; idx < total; idx += K5G_THREADS) {
            if (guarded(idx) || !bits[idx] || row_kept[idx / kc] < 2)
                continue;
            const uint64_t c = ~rank_key(sums[idx]);
            wkey = c < wkey ? c : wkey;
        }
        wkey = block_reduce_min_u64(wkey, sh64);
        if (wkey == ~0ull) {
            if (threadIdx.x == 0)
                *status = 1; // cannot repair (ConfigError on the host)
            return;
        }
        uint64_t widx = ~0ull;
        for (size_t idx = threadIdx.x; idx < total; idx += K5G_THREADS) {
            if (guarded(idx) || !bits[idx] || row_kept[idx / kc] < 2)
                continue;
            if (~rank_key(sums[idx]) == wkey)
                widx = ~(uint64_t)idx < widx ? ~(uint64_t)idx : widx; // largest index among equal keys
        }
        widx = ~block_reduce_min_u64(widx, sh64);
        if (threadIdx.x == 0) {
            bits[widx] = 0;
            row_kept[widx / kc] -= 1;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        repaired_out[blockIdx.x] = repaired;
}

// K5c: schedule mean of the late timesteps: mean[i] = (sum_t sums[t][i]) / late,
// t = half..T-1 added in order (mask.cpp:160-166).
__global__ void k5_late_mean(const double* __restrict__ sums, uint32_t T, size_t total, double* __restrict__ mean) {
    const uint32_t half = T / 2;
    const double late = (double)(T - half);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        for (uint32_t t = half; t < T; ++t)
            v = __dadd_rn(v, sums[(size_t)t * total + i]);
        mean[i] = __ddiv_rn(v, late);
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
// block statistics of the permuted (sub)map: map points at its (0, 0) element,
// rows are `ld` floats apart; maxs / counts (both or neither) add max|a| and
// count(|a| < eps) per block (m_quant / m_sparse inputs)
cudaError_t launch_perm_block_stats(const float* map, size_t ld, uint32_t n, const uint32_t* inv, uint32_t block,
                                    float eps, double* sums, float* maxs, uint32_t* counts, cudaStream_t st) {
    const uint32_t k = (n + block - 1) / block;
    if (block > (uint32_t)K5_MAXBLOCK || k > 65535u * K5_WARPS)
        return cudaErrorInvalidValue;
    const bool stats = maxs != nullptr;
    if (block <= 64 && n <= K5T_MAXN && k <= 512 && n < 65536) {
        const uint32_t rb = ((n + 8) * 4 + 15) & ~15u;
        const size_t tsmem = (size_t)K5T_NBUF * rb + K5T_NBUF * 8 + K5T_NBUF * 4;
        auto kern = stats ? k5_perm_block_sums_tma<true> : k5_perm_block_sums_tma<false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
        if (e != cudaSuccess)
            return e;
        const uint32_t threads = (k + 31) / 32 * 32;
        kern<<<k, threads, tsmem, st>>>(map, ld, n, inv, block, k, eps, sums, maxs, counts);
        return cudaGetLastError();
    }
    const size_t smem = ((size_t)2 * n + (size_t)k * block) * 4;
    if (smem <= 227 * 1024 && n <= (uint32_t)K5S_PF * K5S_THREADS && k <= (uint32_t)K5S_MAXB * K5S_THREADS) {
        auto kern = stats ? k5_perm_block_sums_staged<true> : k5_perm_block_sums_staged<false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return e;
        kern<<<k, K5S_THREADS, smem, st>>>(map, ld, n, inv, block, k, eps, sums, maxs, counts);
        return cudaGetLastError();
    }
    const dim3 grid(k, (k + K5_WARPS - 1) / K5_WARPS); // wide maps: warp per block, gathers from L2
    if (stats)
        k5_perm_block_sums<true><<<grid, K5_WARPS * 32, 0, st>>>(map, ld, n, inv, block, k, eps, sums, maxs, counts);
    else
        k5_perm_block_sums<false><<<grid, K5_WARPS * 32, 0, st>>>(map, ld, n, inv, block, k, eps, sums, maxs,
                                                                  counts);
    return cudaGetLastError();
}

cudaError_t launch_perm_block_sums(const float* map, uint32_t n, const uint32_t* inv, uint32_t block, double* sums,
                                   cudaStream_t st) {
    return launch_perm_block_stats(map, n, n, inv, block, 1.f, sums, nullptr, nullptr, st);
}

cudaError_t launch_gen_mask(const double* sums, uint32_t count, uint32_t kr, uint32_t kc, uint32_t guard, uint64_t K,
                            uint8_t* bits, uint32_t* row_kept_scratch, uint32_t* repaired, int* status,
                            cudaStream_t st) {
    k5_gen_mask<<<count, K5G_THREADS, 0, st>>>(sums, kr, kc, guard, K, bits, row_kept_scratch, repaired, status);
    return cudaGetLastError();
}

// Per-block terms of m_sparse / m_quant (metrics.cpp:60-83, 114-133) from K5a's
// statistics: term[b] = max == 0 ? 1 : max / (sum / cnt) (the reference's fp64
// ops, IEEE-rounded like the host) and the count of blocks whose near-zero
// share reaches sigma (an exact integer sum). The host adds the terms in
// block order, so the score stays bit-identical.
__global__ void k5_block_terms(const double* __restrict__ sums, const float* __restrict__ maxs,
                               const uint32_t* __restrict__ counts, uint32_t k, uint32_t n, uint32_t block, float sigma,
                               double* __restrict__ terms, uint32_t* __restrict__ sparse) {
    uint32_t local = 0;
    const size_t kk = (size_t)k * k;
    for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < kk; b += (size_t)gridDim.x * blockDim.x) {
        const uint32_t bi = (uint32_t)(b / k), bj = (uint32_t)(b % k);
        const uint32_t r0 = bi * block, c0 = bj * block;
        const uint32_t rn = min(n, r0 + block) - r0, cn = min(n, c0 + block) - c0;
        const double cnt = (double)((size_t)rn * cn);
        if (__ddiv_rn((double)counts[b], cnt) >= (double)sigma)
            ++local;
        const double mx = (double)maxs[b];
        terms[b] = mx == 0.0 ? 1.0 : __ddiv_rn(mx, __ddiv_rn(sums[b], cnt));
    }
    for (int o = 16; o > 0; o >>= 1)
        local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local)
        atomicAdd(sparse, local);
}

cudaError_t launch_block_terms(const double* sums, const float* maxs, const uint32_t* counts, uint32_t k, uint32_t n,
                               uint32_t block, float sigma, double* terms, uint32_t* sparse, cudaStream_t st) {
    const size_t kk = (size_t)k * k;
    const int grid = (int)((kk + 255) / 256 < 2048 ? (kk + 255) / 256 : 2048);
    k5_block_terms<<<grid > 0 ? grid : 1, 256, 0, st>>>(sums, maxs, counts, k, n, block, sigma, terms, sparse);
    return cudaGetLastError();
}

cudaError_t launch_late_mean(const double* sums, uint32_t T, size_t total, double* mean, cudaStream_t st) {
    const int grid = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    k5_late_mean<<<grid > 0 ? grid : 1, 256, 0, st>>>(sums, T, total, mean);
    return cudaGetLastError();
}

} // namespace paro
