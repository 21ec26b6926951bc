// layer.cuh -- HBM layout shared by the host orchestration and the kernels.
//
// All per-layer device state for H heads of N tokens, head dim D in {64,128},
// block 64, kb = ceil(N/64) key/query blocks, kb2 = kb rounded up to even.
// K3 runs two q-blocks of a head per work item (A in TMEM lanes 0-15 of each
// lane quadrant, B in lanes 16-31, independent M = 64 tcgen05 MMAs), so K2
// pairs q-blocks of a head with similar kept counts.
//
//   codes  q/k/v  int8 [H][kb2*64][D]  PERMUTED token order, zero-padded rows
//   qsc          fp32 [H][kb2][G]     Q scale per (block, 64-column group), G = D/64
//   meta         fp32 [H][kb2][4 + D] per key block: {ksc[0], ksc[1], vsc, 0, colsum[D]}
//                                      (colsum = sum of V codes per column, exact in fp32)
//   perm         PermDesc [H]          permuted index -> original token (div/mod form)
//   items        u16  [H][kb][kb]       per q-block: kept key blocks, ascending
//   qb_count     u32  [H][kb2]         kept key blocks per q block (0 => zeroed rows)
//   pairs        u32  [H][np]          q-block pair p: A | B << 16 (B = 0xffff: none);
//                                      q-blocks sorted by kept count, neighbours paired
//   pair_count   u32  [H][np]          max(count A, count B) = K3 steps of the pair
//   order        u32  [H*np]           work items (h << 16 | p), longest first (LPT)
#pragma once
#include <cstdint>

namespace paro {

constexpr int kBlock = 64;
constexpr uint32_t kMaxChunks = 64;

// Permuted index i -> original token: decompose i row-major over the permuted
// extents (pext), then recombine with the original strides of those axes.
// Equals PermPlan::inverse[i] of make_perm (reorder.cpp:49-72). 2-D grids use
// pext[0] = 1, ostride[0] = 0. `prefix` leading (text) tokens stay in place and
// the grid tokens follow them (PermPlan::with_prefix, reorder.cpp:30-47).
struct PermDesc {
    uint32_t pext[3];
    uint32_t ostride[3];
    uint32_t prefix;
};

// Branch-free on purpose: with a branch per row, K1 no longer issues all its
// gathered row loads back to back (d=128 K1 0.96 -> 1.66 ms measured).
__host__ __device__ inline uint32_t perm_src(const PermDesc& pd, uint32_t i) {
    const uint32_t j = i - pd.prefix; // wraps for prefix rows; that result is discarded
    const uint32_t c2 = j % pd.pext[2];
    const uint32_t t = j / pd.pext[2];
    const uint32_t c1 = t % pd.pext[1];
    const uint32_t c0 = t / pd.pext[1];
    const uint32_t g = pd.prefix + c0 * pd.ostride[0] + c1 * pd.ostride[1] + c2 * pd.ostride[2];
    return i < pd.prefix ? i : g;
}

struct LayerDev {
    uint32_t H, N, D, G, kb, kb2, np;
    PermDesc* perm;
    int8_t *q, *k, *v;      // v: int8 rows of D, or (v_packed) D/2 bytes of INT4 pairs, low nibble first
    uint32_t v_packed;      // the last reorder_quantize wrote 4-bit V codes packed
    float* qsc;
    float* meta;
    uint16_t* items;
    uint32_t* pairs;
    uint32_t* pair_count;
    uint32_t* qb_count;
    uint32_t* order;       // [H*np] global LPT order (h << 16 | p)
    uint32_t* order_chunk; // [H*np] per-chunk LPT order, chunk c = heads [chunk_start[c], chunk_start[c+1])
    uint32_t nchunks;      // host-buffer pipeline chunks (<= kMaxChunks)
    uint32_t chunk_start[65];
    uint32_t* work_counter;
    uint32_t l2_group;     // heads per L2 group of the whole-layer LPT order (0: one group)
    // dense text-token prefix (AttnInputs::dense_prefix): dp rows / tokens, nd =
    // ceil(dp/64) dense key tiles; K4 hands K3 each non-dense row's running
    // state after the dense tiles: m (fp64), l, acc [H][kb2*64][(D)]
    uint32_t dp, nd;
    double* init_m;
    float* init_l;
    float* init_acc;
    // K4 splits the keys of the nd dense q-blocks into k4_cb chunks of k4_ch
    // tiles; per (row, chunk) partial (m, l, acc): [H][nd*64][k4_cb](·D)
    uint32_t k4_cb, k4_ch;
    double* part_m;
    float* part_l;
    float* part_acc;
    // K4a: permuted V as transposed bf16 hi / lo tiles [H][kb2][D][64] (bf16 bits)
    uint16_t* vsplit_hi;
    uint16_t* vsplit_lo;
    // rotary embedding fused into K1 (the producer's last elementwise op, SURVEY
    // 8(f) rank 4): [N - dp][D] fp32 cos / sin per ORIGINAL grid token, applied
    // to Q and K pairs (2i, 2i+1) before quantisation; nullptr = off
    const float* rope_cos;
    const float* rope_sin;
};

__host__ __device__ inline uint32_t meta_stride(uint32_t D) { return 4 + D; }

// Test hook (paro_layer_debug_pdump): K3 copies the final P codes of every
// quantized tile of the selected (head, q-block)s -- after the exact boundary
// path -- with the tile group's (lo, pscale) and key block. slot == nullptr: off.
struct K3Dump {
    const int32_t* slot; // [H][kb2]: dump slot of (h, qb) or -1
    uint8_t* codes;      // [nslot][kb][64][64] (row-major, key columns)
    float* meta;         // [nslot][kb][4]: lo, pscale, key block, 1
    uint32_t kb;
};

} // namespace paro
