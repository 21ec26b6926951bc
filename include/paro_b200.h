/*
 * paro_b200.h -- C ABI of the B200-native PAROAttention hot path.
 *
 * This is the drop-in boundary for the reference's C++ library API on the hot
 * path (reference proj/include/paro/ headers). Plain pointers
 * and sizes only; no exceptions cross it. Every call returns a status:
 *
 *   PARO_OK (0) or an error class whose tens digit is the reference exit code
 *   (proj/include/paro/error.hpp:11-40): 2x = ConfigError/ShapeError/InputError,
 *   3x = FormatError/IoError, 4x = InvariantError, 5x = CUDA runtime failure
 *   (no reference counterpart). paro_last_error() returns the thread-local
 *   message of the last failing call on the calling thread.
 *
 * Supported hot-path configuration (anything else is rejected with
 * PARO_E_CONFIG, never served by a CPU fallback): block = 64, d in {64, 128},
 * P/V bits in {4, 8}, 2-D (H,W) or 3-D (F,H,W) token grids, any dense_prefix
 * (paro_layer_create_prefix).
 *
 * Threading: one paro_ctx per GPU, used from one host thread; layers belong to
 * the context they were created on. Device pointers are caller-owned unless a
 * function says otherwise; all device work is enqueued on the given stream.
 */
#ifndef PARO_B200_H
#define PARO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARO_OK 0
#define PARO_E_CONFIG 20    /* ConfigError    (error.hpp:21-23) */
#define PARO_E_SHAPE 21     /* ShapeError     (error.hpp:24-26) */
#define PARO_E_INPUT 22     /* InputError     (error.hpp:27-29) */
#define PARO_E_FORMAT 30    /* FormatError    (error.hpp:30-32) */
#define PARO_E_IO 31        /* IoError        (error.hpp:33-35) */
#define PARO_E_INVARIANT 40 /* InvariantError (error.hpp:36-38) */
#define PARO_E_CUDA 50      /* CUDA runtime error (new) */

#define PARO_BLOCK 64

typedef void* paro_stream_t; /* a cudaStream_t; NULL = legacy default stream */
typedef struct paro_ctx paro_ctx;
typedef struct paro_layer paro_layer;

const char* paro_last_error(void);
const char* paro_version(void);

/* ---------------------------------------------------------------------------
 * Host-side integer stages (no GPU needed).
 * ------------------------------------------------------------------------- */

/* parse_grid("F:13,H:30,W:45") -- replaces paro::parse_grid + TokenGrid
 * validation (tensor.cpp:26-47, 95-114). labels/extents hold >= 3 slots. */
int paro_parse_grid(const char* text, int* ndim, char* labels, uint32_t* extents);

/* make_perm(grid, order) -- replaces paro::make_perm (reorder.hpp:32,
 * reorder.cpp:49-72). forward[old] = new, inverse[new] = old, N entries each. */
int paro_make_perm(int ndim, const char* labels, const uint32_t* extents, const char* order, uint32_t* forward,
                   uint32_t* inverse);

/* enumerate_perms(grid) orders -- replaces paro::enumerate_perms
 * (reorder.cpp:74-91): identity first, then lexicographic. `orders` receives
 * count*ndim chars (no terminators); count = ndim! (<= 6). */
int paro_enumerate_orders(int ndim, const char* labels, char* orders, int* count);

/* load_plan_file (reorder.cpp:193-216) on an in-memory plan text ("head_id,order"
 * lines; `name` prefixes FormatError messages like the file path does). Query
 * with heads/orders NULL: *count entries, *orders_size bytes for the orders
 * (each NUL-terminated, in file order). */
int paro_parse_plan(const char* text, size_t len, const char* name, uint32_t* count, uint32_t* heads, char* orders,
                    size_t* orders_size);
/* plan_for_head (tools/main.cpp:118-126) for n heads: text NULL -> identity
 * order; else the first entry naming each head (InputError "<name>: no plan
 * entry for head h" when none), validated as make_perm does. orders_out: n*ndim
 * chars, ready for paro_layer_create. */
int paro_plan_for_heads(const char* text, size_t len, const char* name, const char* grid_text, uint32_t n,
                        const uint32_t* head_ids, char* orders_out);

/* PMSK blob decode -- replaces paro::deserialize_mask (mask.hpp:74,
 * mask.cpp:217-244). bits (k_rows*k_cols bytes, row-major) may be NULL to
 * query the header; consumed may be NULL. */
int paro_deserialize_mask(const uint8_t* data, size_t size, uint32_t* k_rows, uint32_t* k_cols, uint32_t* block,
                          uint8_t* bits, size_t* consumed);

/* PMSK blob encode -- replaces paro::serialize_mask (mask.cpp:197-215).
 * out may be NULL to query *size. */
int paro_serialize_mask(const uint8_t* bits, uint32_t k_rows, uint32_t k_cols, uint32_t block, uint8_t* out,
                        size_t* size);

/* PSCH schedule lookup -- replaces load_schedule(path).at(t)
 * (mask.cpp:132-140, 267-305) on an in-memory PSCH image. bits may be NULL. */
int paro_schedule_at(const uint8_t* data, size_t size, uint32_t t, uint32_t* k_rows, uint32_t* k_cols,
                     uint32_t* block, uint8_t* bits);

/* ---- PAT1 / PARQ interchange (golden and fixture exchange).
 * In-memory, byte-exact with save_tensor / load_tensor (tensor_io.cpp:45-120) and
 * save_quant_tensor / load_quant_tensor (quant.cpp:219-326); FormatError (PARO_E_FORMAT)
 * messages carry the byte offset like the reference's. Encoders: out NULL -> *size = bytes
 * needed; otherwise *size is the capacity on entry and the byte count on return. */
int paro_tensor_encode(const uint32_t* shape, uint32_t ndim, const float* values, uint8_t* out, size_t* size);
/* shape: room for 255 extents; values NULL -> header check only */
int paro_tensor_decode(const uint8_t* data, size_t size, uint32_t* ndim, uint32_t* shape, float* values);
typedef struct {
    unsigned bits;
    int mode;     /* 0 unsigned, 1 symmetric (quant.hpp:15-18) */
    int grouping; /* 0 per block, 1 per row (quant.hpp:20-23) */
    uint32_t block, rows, cols, groups;
} paro_quant_header;
/* offsets read only in unsigned mode */
int paro_quant_encode(unsigned bits, int mode, int grouping, uint32_t block, uint32_t rows, uint32_t cols,
                      const int32_t* codes, const float* scales, const float* offsets, uint8_t* out, size_t* size);
/* codes / scales / offsets NULL -> header only */
int paro_quant_decode(const uint8_t* data, size_t size, paro_quant_header* header, int32_t* codes, float* scales,
                      float* offsets);

/* ---------------------------------------------------------------------------
 * Mask producer on the GPU. Device pointers; the
 * calls validate like the reference and return its error classes.
 * ------------------------------------------------------------------------- */

/* block_sums(AttnMap(apply_perm_map(map, plan), block)) fused -- replaces
 * reorder.cpp:103-114 + metrics.cpp:41-58 (cmd_maskgen, main.cpp:236-238):
 * map fp32 [n][n] (device), inverse = plan.inverse (device, NULL = identity),
 * sums fp64 [k][k] (device), k = ceil(n/block), block <= 256. The N x N map is read
 * once; sums are bit-identical to the reference's scalar kernels. */
int paro_perm_block_sums_device(paro_ctx* ctx, paro_stream_t stream, const float* map, uint32_t n,
                                const uint32_t* inverse, uint32_t block, double* sums);

/* gen_mask(sums, density, block, guard) for `count` grids -- replaces
 * mask.cpp:56-130 (incl. guard blocks and the degenerate-row repair):
 * sums fp64 [count][k_rows][k_cols] (device), bits [count][k_rows][k_cols]
 * (device, one byte per block), repaired_rows (host, count entries, may be
 * NULL). Synchronises `stream`. Bit-identical to the reference. */
int paro_gen_mask_device(paro_ctx* ctx, paro_stream_t stream, const double* sums, uint32_t count, uint32_t k_rows,
                         uint32_t k_cols, double density, uint32_t block, uint32_t guard, uint8_t* bits,
                         uint32_t* repaired_rows);

/* build_schedule(calib sums, density, T, block, guard) -- replaces
 * mask.cpp:142-172: sums fp64 [T][k_rows][k_cols] (device); masks receives
 * the T/2 distinct early masks then the shared late mask,
 * [(T/2)+1][k_rows][k_cols] bytes (device); repaired_rows (host) = total.
 * Serialize with paro_serialize_mask for a PSCH image. */
int paro_build_schedule_device(paro_ctx* ctx, paro_stream_t stream, const double* sums, uint32_t timesteps,
                               uint32_t k_rows, uint32_t k_cols, double density, uint32_t block, uint32_t guard,
                               uint8_t* masks, uint32_t* repaired_rows);

/* select_permutation(calib, grid, cfg, dense_prefix) -- replaces
 * reorder.cpp:130-181 with metrics.cpp:60-133 (m_sparse, m_quant) over every
 * candidate order (enumerate_perms): maps fp32 [count][n+p][n+p] (device,
 * p = dense_prefix, the prefix rows / columns are stripped), grid text as in
 * parse_grid, cfg = {block <= 256, eps, sigma, alpha}. Each permuted map's
 * block statistics (sum|a| in the reference's fp64 order, max|a|, #|a| < eps)
 * come from one fused pass over the map; the final reductions run on the host
 * in the reference's order, so scores are bit-identical. Outputs (host):
 * orders (nperm*ndim chars), scores [nperm][5] = {sparse_mean, quant_mean,
 * sparse_share, quant_share, combined}, nperm, chosen (first argmin). */
int paro_select_permutation_device(paro_ctx* ctx, paro_stream_t stream, const float* maps, uint32_t count,
                                   const char* grid_text, uint32_t block, float eps, float sigma, float alpha,
                                   uint32_t dense_prefix, char* orders, double* scores, int* nperm, int* chosen);

/* Synthetic N(0,1) fp32 inputs: MT19937-64, u = (x>>11)*2^-53, Box-Muller on
 * (1-u1, u2), the generator documented in synth.cpp:20-22,173-182. */
int paro_synth_randn(uint64_t seed, size_t count, float* out);

/* ---------------------------------------------------------------------------
 * Device context.
 * ------------------------------------------------------------------------- */
int paro_ctx_create(int device, paro_ctx** out);
int paro_ctx_destroy(paro_ctx* ctx);
int paro_ctx_num_sms(const paro_ctx* ctx, int* out);
/* visible CUDA devices (one paro_ctx per device, each driven from its own host
 * thread: the multi-GPU head shard) */
int paro_device_count(int* out);

/* pinned host buffers for the e2e path (cudaHostAlloc / cudaFreeHost) */
int paro_host_alloc(size_t bytes, void** out);
int paro_host_free(void* p);
/* device buffers (cudaMalloc / cudaFree) for C callers without another allocator */
int paro_device_alloc(size_t bytes, void** out);
int paro_device_free(void* p);
int paro_memcpy(void* dst, const void* src, size_t bytes, paro_stream_t stream); /* cudaMemcpyDefault, async */
int paro_stream_sync(paro_stream_t stream);

/* ---------------------------------------------------------------------------
 * Standalone device stages (bit-exact with the reference functions they name).
 * ------------------------------------------------------------------------- */

/* apply_perm_rows on the GPU -- replaces paro::apply_perm_rows
 * (reorder.cpp:93-101): out.row(i) = in.row(inverse[i]); fp32 [rows, cols]. */
int paro_apply_perm_rows_device(paro_ctx* ctx, paro_stream_t stream, const float* in, uint32_t rows, uint32_t cols,
                                const uint32_t* inverse, float* out);

/* quantize(m, {bits, Symmetric, PerBlock, 64}) on the GPU -- replaces
 * paro::quantize (quant.cpp:60-104) for the hot path's Q/K configuration.
 * codes: int8 [rows, cols] row-major; scales: ceil(rows/64)*ceil(cols/64) fp32
 * in the reference's group order (quant.cpp:45-56). cols must be <= 128. */
int paro_quantize_sym_device(paro_ctx* ctx, paro_stream_t stream, const float* in, uint32_t rows, uint32_t cols,
                             int bits, int8_t* codes, float* scales);

/* ---------------------------------------------------------------------------
 * Layer: the per-head chain of cmd_run (proj/tools/main.cpp:276-305) for H
 * heads at once -- per-head PARO permutation, block-mask application,
 * Q/K INT8 + P/V INT8|INT4 quantized block-sparse attention, inverse
 * permutation of the output. Q/K/V/O are fp32 [H, N, d] in ORIGINAL token
 * order; N must equal the grid's token count.
 * ------------------------------------------------------------------------- */

/* orders: H*ndim chars (head h's axis order at orders[h*ndim]), or NULL for
 * the identity plan of every head (plan_for_head without a plan file,
 * main.cpp:118-120). */
int paro_layer_create(paro_ctx* ctx, uint32_t heads, uint32_t head_dim, const char* grid_text, const char* orders,
                      paro_layer** out);

/* paro_layer_create with a dense text-token prefix (AttnInputs::dense_prefix,
 * attention.cpp:134-199; PermPlan::with_prefix, reorder.cpp:30-47): the layer
 * has N = grid tokens + dense_prefix rows, the first dense_prefix tokens keep
 * their position under every head's order, attend densely and unquantized to
 * all keys, and every key tile touching the prefix stays dense and unquantized
 * for all rows (K4); the rest follows the quantized path (K3). Masks cover
 * ceil(N/64)^2 blocks (gen_mask's guard blocks are the dense tiles). */
int paro_layer_create_prefix(paro_ctx* ctx, uint32_t heads, uint32_t head_dim, const char* grid_text,
                             const char* orders, uint32_t dense_prefix, paro_layer** out);
int paro_layer_destroy(paro_layer* layer);

/* Masks: H*k*k bytes (BlockMask::bits per head, mask.hpp:15-32), k = ceil(N/64);
 * NULL = every block kept (quantized_blocked_attention(in, nullptr, ...)).
 * Runs K2 (mask -> per q-block-pair kept lists + LPT work order) on `stream`.
 * The _device variant reads device bytes. */
int paro_layer_set_masks(paro_layer* layer, paro_stream_t stream, const uint8_t* host_bits);
int paro_layer_set_masks_device(paro_layer* layer, paro_stream_t stream, const uint8_t* device_bits);
/* The same from one serialized PMSK blob per head (deserialize_mask, mask.cpp:217-244): block 64,
 * a ceil(N/64)^2 grid; errors name the head. */
/* Per-timestep mask schedule (MaskSchedule, mask.hpp; load_schedule / at(t),
 * mask.cpp:132-140, 267-305): one PSCH image per head, all covering the same T
 * timesteps. The T/2 distinct masks and the shared late mask of every head are
 * uploaded once. resident_lists = 0: K2 builds every entry's kept lists now, and
 * paro_layer_select_timestep is a pointer switch (no K2 in the step);
 * resident_lists = 2: two list buffers -- select_timestep(t) makes t's lists
 * current and builds t+1's on a side stream while step t runs (the paper's
 * double-buffered prefetch). A later set_masks* ends the
 * schedule. select_timestep: at(t) semantics and errors (t >= T: InputError). */
int paro_layer_set_schedule(paro_layer* layer, paro_stream_t stream, const uint8_t* const* psch, const size_t* sizes,
                            uint32_t resident_lists);
int paro_layer_select_timestep(paro_layer* layer, paro_stream_t stream, uint32_t t);
/* timesteps T, entries T/2 + 1, the entry whose lists are current (-1: none) */
int paro_layer_schedule_info(const paro_layer* layer, uint32_t* timesteps, uint32_t* entries, int* current_entry);

int paro_layer_set_masks_pmsk(paro_layer* layer, paro_stream_t stream, const uint8_t* const* blobs,
                              const size_t* sizes);

/* Rotary embedding fused into K1 (the permutation and quantisation
 * folded into the producer's last elementwise op). cos / sin: [N - dense_prefix][d] fp32 per
 * ORIGINAL grid token (the DiT's real-valued freqs, e.g. diffusers' freqs_cos / freqs_sin),
 * host or device memory, copied into the layer on `stream`. Q and K rows of grid tokens become
 *   x'[2i] = x[2i] cos[2i] - x[2i+1] sin[2i],  x'[2i+1] = x[2i+1] cos[2i+1] + x[2i] sin[2i+1]
 * (each product and sum rounded separately, fp32) before the reference quantizer; the text
 * prefix and V are untouched. Both NULL turns it off. Pinned or device tables must stay valid
 * until `stream` has passed the copy (pageable ones are staged before the call returns). The same numbers as rotating the fp32
 * inputs first and calling the layer without it (tests/test_gpu_parity.py). */
int paro_layer_set_rope(paro_layer* layer, paro_stream_t stream, const float* cos, const float* sin);

/* K1: permuted gather + per-block quantization into layer-owned buffers (with a
 * dense prefix also K4a: the bf16 hi/lo V^T tiles of the dense path). Device
 * buffers (Q/K/V here, out in attention / forward) must be 16-byte aligned
 * (PARO_E_CONFIG otherwise): rows are read and written as 16-byte vectors. Q/K/V are
 * read only by the kernels queued here: once they have run on `stream` the caller
 * may free or reuse them -- attention works from the layer-owned buffers alone. */
int paro_layer_reorder_quantize(paro_layer* layer, paro_stream_t stream, const float* q, const float* k,
                                const float* v, int v_bits);

/* K3: block-sparse quantized attention from the layer-owned codes; writes
 * out [H,N,d] in original token order and zeroed [H,N] bytes (1 = row had no
 * kept block, indexed by ORIGINAL token; may be NULL). scale 0 -> 1/sqrt(d)
 * (AttnInputs::effective_scale, attention.cpp:26-28). pv_bits must equal the
 * v_bits of the preceding reorder_quantize. */
int paro_layer_attention(paro_layer* layer, paro_stream_t stream, float scale, int pv_bits, float* out,
                         uint8_t* zeroed);

/* K1 + K3 on device buffers. */
int paro_layer_forward(paro_layer* layer, paro_stream_t stream, const float* q, const float* k, const float* v,
                       float scale, int pv_bits, float* out, uint8_t* zeroed);

/* End to end from HOST buffers (pinned for full speed): H2D of Q/K/V, K1, K3,
 * D2H of O (and zeroed if non-NULL), synchronised before returning. Heads are
 * processed in chunks (default: at least 8, at most ~96 MB of Q/K/V each, the last
 * one tapered into halving pieces so little work follows the final upload) whose
 * uploads, kernels and downloads are pipelined on three streams. */
int paro_layer_forward_host(paro_layer* layer, paro_stream_t stream, const float* q, const float* k, const float* v,
                            float scale, int pv_bits, float* out, uint8_t* zeroed);

/* INT4 V storage: packed = 1 stores 4-bit V codes two per
 * byte in HBM (low nibble first, two's complement -- the PARQ payload layout) and K3
 * unpacks each tile to i8 in shared memory for the kind::i8 P.V MMA (Blackwell has
 * no INT4 MMA); 0 (default; PARO_V_PACKED=1 flips it) keeps one code per byte, which
 * K3 feeds to the MMA directly. Measured (round 2): packing halves V's footprint
 * (c5: 387 -> 194 MB) and costs K3 14-19% (the unpack competes with the softmax
 * for issue slots; K3 is not HBM-bound). Applies from the next reorder_quantize. */
int paro_layer_set_v_packing(paro_layer* layer, int packed);

/* Number of head chunks forward_host pipelines (clamped to [1, heads]).
 * Re-sorts the per-chunk work lists on `stream` if masks are already set. */
int paro_layer_set_pipeline_chunks(paro_layer* layer, paro_stream_t stream, uint32_t chunks);

/* ---- introspection for parity tests ---- */
/* Device buffers owned by the layer (kb = ceil(N/64), kb2 = kb rounded up to
 * even, rows per head = kb2*64; all codes in PERMUTED token order, zero-padded). */
typedef struct {
    uint32_t heads, tokens, head_dim, kblocks, kblocks_padded; /* kblocks_padded = kb2 */
    uint32_t groups;   /* head_dim/64 column groups of Q/K */
    int8_t* q_codes;   /* [H, kb2*64, d] int8 */
    int8_t* k_codes;   /* [H, kb2*64, d] int8 */
    int8_t* v_codes;   /* [H, kb2*64, d] int8 codes; with v_packed: [H, kb2*64, d/2] bytes, two
                          two's-complement INT4 codes per byte, low nibble = even column
                          (the PARQ payload layout, quant.cpp:237-243) */
    float* q_scales;   /* [H, kb2, groups] */
    float* tile_meta;  /* [H, kb2, 4+d]: k_scale[g0], k_scale[g1] (0 if d=64), v_scale, 0,
                          v_colsum[d] (exact integers in fp32) */
    uint32_t* inverse; /* [H, N] device perm tables (filled at create) */
    uint32_t* forward; /* [H, N] */
    uint32_t v_bits;   /* V code width of the last reorder_quantize (0: none yet) */
    uint32_t v_packed; /* 1: v_codes hold nibble-packed INT4 (paro_layer_set_v_packing) */
} paro_layer_buffers;
int paro_layer_get_buffers(const paro_layer* layer, paro_layer_buffers* out);

/* One head's permuted codes of the last reorder_quantize as a PARQ blob (which: 0 Q, 1 K,
 * 2 V), byte-identical to save_quant_tensor(quantize(apply_perm_rows(X, plan), {bits,
 * Symmetric, PerBlock, 64})) (quant.cpp:60-104, 219-251): Q/K 8 bits, V the layer's V bits
 * (d = 64 only: V groups span all d columns, PerBlock expresses that only at d = 64). */
int paro_layer_export_parq(paro_layer* layer, paro_stream_t stream, uint32_t head, int which, uint8_t* out,
                           size_t* size);

/* K2 output: per head, per q-block kept-count (kept[H*k]), total kept tiles */
int paro_layer_mask_stats(paro_layer* layer, uint32_t* kept_per_qblock, uint64_t* total_kept);

/* Debug: int32 QK^T accumulators of (head, q-block, k-block) tiles through the
 * same tcgen05 path K3 uses. tiles: n_tiles*3 uint32 (device); S: n_tiles *
 * groups * 64 * 64 int32 (device), [tile][group][row][col]. */
int paro_layer_debug_qk(paro_layer* layer, paro_stream_t stream, uint32_t n_tiles, const uint32_t* tiles, int32_t* S);

/* Launch accounting: number of kernels the last forward launched, and the
 * last K3 kernel's grid size. */
/* Test hook: K1's quantizer arithmetic (reciprocal + FMA-residual quotient, no
 * clamp) vs the reference quant_affine (IEEE x/scale, clamp, round half away) for
 * every amax bit pattern in [bits_begin, bits_begin + bits_count) (finite), x =
 * +-amax and nx pseudo-random |x| <= amax, qmax 127 and 7. *mismatches = count;
 * first[5] = (amax bits, x bits, qmax, K1 code, reference code) of the first. */
int paro_debug_k1_quant_proof(paro_ctx* ctx, uint32_t bits_begin, uint64_t bits_count, uint32_t nx, uint32_t seed,
                              uint64_t* mismatches, uint32_t* first);

/* Test hook: runs K3 (as paro_layer_attention, output discarded) and returns the
 * FINAL P codes of every quantized tile of the n_targets (head, q-block) pairs
 * (targets: 2*n u32), in each q-block's kept order: codes [n][kb][64][64] (rows x
 * key columns; a tail tile's padded columns are 0 in the reference), meta
 * [n][kb][4] = (lo, pscale, key block, 1) per tile (attention.cpp:201-228);
 * unused tile slots are zero. Host pointers; synchronises. */
int paro_layer_debug_pdump(paro_layer* layer, paro_stream_t stream, float scale, int pv_bits, uint32_t n_targets,
                           const uint32_t* targets, uint8_t* codes, float* meta);

int paro_layer_last_launches(const paro_layer* layer, int* kernels);

#ifdef __cplusplus
}
#endif
#endif /* PARO_B200_H */
