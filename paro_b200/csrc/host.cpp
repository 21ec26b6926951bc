// host.cpp -- C-ABI implementation of include/paro_b200.h.
//
// Host-side integer stages restate the reference's TokenGrid / make_perm /
// PMSK / PSCH / gen_mask contracts (cited per function); the device stages
// launch the sm_100a kernels in prep_kernels.cu and attention_kernel.cu.
// There is no CPU fallback for any device stage: without a usable sm_100
// device every device call fails with PARO_E_CUDA.
#include "../../include/paro_b200.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "layer.cuh"

namespace paro {
cudaError_t launch_k1(const LayerDev& L, const float* q, const float* k, const float* v, int v_bits,
                      uint32_t head_begin, uint32_t head_count, cudaStream_t st);
cudaError_t launch_quantize_sym(const float* in, uint32_t rows, uint32_t cols, int bits, int8_t* codes,
                                float* scales, cudaStream_t st);
cudaError_t launch_apply_perm_rows(const float* in, uint32_t rows, uint32_t cols, const uint32_t* inverse, float* out,
                                   cudaStream_t st);
cudaError_t launch_perm_tables(const PermDesc* perm, uint32_t H, uint32_t N, uint32_t* fwd, uint32_t* inv,
                               cudaStream_t st);
cudaError_t launch_k2(const LayerDev& L, const uint8_t* bits, cudaStream_t st);
cudaError_t launch_perm_block_sums(const float* map, uint32_t n, const uint32_t* inv, uint32_t block, double* sums,
                                   cudaStream_t st);
cudaError_t launch_gen_mask(const double* sums, uint32_t count, uint32_t kr, uint32_t kc, uint32_t guard, uint64_t K,
                            uint8_t* bits, uint32_t* row_kept_scratch, uint32_t* repaired, int* status,
                            cudaStream_t st);
cudaError_t launch_late_mean(const double* sums, uint32_t T, size_t total, double* mean, cudaStream_t st);
cudaError_t launch_block_terms(const double* sums, const float* maxs, const uint32_t* counts, uint32_t k, uint32_t n,
                               uint32_t block, float sigma, double* terms, uint32_t* sparse, cudaStream_t st);
void k4_chunking(uint32_t kb, uint32_t nd, uint32_t heads, uint32_t& cb, uint32_t& ch);
cudaError_t launch_k4a(const LayerDev& L, const float* v, uint32_t head_begin, uint32_t head_count, cudaStream_t st);
cudaError_t launch_k4(const LayerDev& L, double scale, float* out, uint8_t* zeroed,
                      uint32_t head_begin, uint32_t head_count, cudaStream_t st, const CUtensorMap* tq,
                      const CUtensorMap* tk, const CUtensorMap* tvh, const CUtensorMap* tvl);
cudaError_t launch_perm_block_stats(const float* map, size_t ld, uint32_t n, const uint32_t* inv, uint32_t block,
                                    float eps, double* sums, float* maxs, uint32_t* counts, cudaStream_t st);
cudaError_t launch_k2_order(const LayerDev& L, cudaStream_t st);
cudaError_t launch_k3(const LayerDev& L, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const CUtensorMap& tvp, const CUtensorMap& tq32, double scale, int pv_bits, float* out, uint8_t* zeroed, int num_sms, cudaStream_t st,
                      uint32_t head_begin, uint32_t head_count, bool chunked, const K3Dump* dump = nullptr);
cudaError_t launch_k1_quant_proof(uint32_t lo, uint32_t count, uint32_t nx, uint32_t seed, unsigned long long* bad,
                                  uint32_t* first, int num_sms, cudaStream_t st);
cudaError_t launch_debug_qk(const LayerDev& L, const CUtensorMap& tq, const CUtensorMap& tq32, const CUtensorMap& tk,
                            uint32_t n_tiles, const uint32_t* tiles, int32_t* S, cudaStream_t st);
} // namespace paro

using paro::LayerDev;
using paro::PermDesc;

namespace {

thread_local std::string g_last_error;

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(PARO_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return PARO_OK;
    } catch (const Fail& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return PARO_E_INVARIANT;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return PARO_E_INVARIANT;
    }
}

// ---------------------------------------------------------------- grid
struct Grid {
    int ndim = 0;
    char labels[3] = {0, 0, 0};
    uint32_t ext[3] = {0, 0, 0};
    size_t tokens() const {
        size_t n = 1;
        for (int a = 0; a < ndim; ++a)
            n *= ext[a];
        return n;
    }
    int axis_index(char c) const {
        for (int a = 0; a < ndim; ++a)
            if (labels[a] == c)
                return a;
        fail(PARO_E_INPUT, std::string("grid has no axis labeled '") + c + "'"); // tensor.cpp:56-61
    }
};

// TokenGrid constructor rules (tensor.cpp:26-47)
void validate_grid(const Grid& g) {
    if (g.ndim != 2 && g.ndim != 3)
        fail(PARO_E_CONFIG, "token grid must have 2 or 3 axes, got " + std::to_string(g.ndim));
    unsigned seen = 0;
    for (int a = 0; a < g.ndim; ++a) {
        unsigned bit;
        switch (g.labels[a]) {
        case 'F': bit = 1; break;
        case 'H': bit = 2; break;
        case 'W': bit = 4; break;
        default: fail(PARO_E_CONFIG, std::string("unknown grid axis label '") + g.labels[a] + "'");
        }
        if (seen & bit)
            fail(PARO_E_CONFIG, std::string("duplicate grid axis label '") + g.labels[a] + "'");
        seen |= bit;
        if (g.ext[a] == 0)
            fail(PARO_E_CONFIG, std::string("grid axis '") + g.labels[a] + "' has zero extent");
    }
    if (g.ndim == 2 && (seen & 1))
        fail(PARO_E_CONFIG, "2D grids use labels H and W only");
}

// parse_grid (tensor.cpp:95-114)
Grid parse_grid_text(const char* text) {
    if (!text)
        fail(PARO_E_CONFIG, "null grid text");
    Grid g;
    std::string s(text);
    size_t pos = 0;
    std::vector<std::string> parts;
    while (true) {
        size_t c = s.find(',', pos);
        parts.push_back(s.substr(pos, c == std::string::npos ? std::string::npos : c - pos));
        if (c == std::string::npos)
            break;
        pos = c + 1;
    }
    if (s.empty())
        parts.clear();
    if (parts.size() > 3)
        fail(PARO_E_CONFIG, "token grid must have 2 or 3 axes, got " + std::to_string(parts.size()));
    for (const auto& part : parts) {
        const size_t colon = part.find(':');
        if (colon != 1 || part.size() < 3)
            fail(PARO_E_CONFIG, "bad grid axis '" + part + "', expected LABEL:EXTENT (e.g. F:13)");
        unsigned long v = 0;
        try {
            size_t used = 0;
            v = std::stoul(part.substr(2), &used);
            (void)used;
        } catch (const std::exception&) {
            fail(PARO_E_CONFIG, "bad grid extent in '" + part + "'");
        }
        g.labels[g.ndim] = part[0];
        g.ext[g.ndim] = static_cast<uint32_t>(v);
        ++g.ndim;
    }
    validate_grid(g);
    return g;
}

Grid grid_from(int ndim, const char* labels, const uint32_t* extents) {
    if (ndim < 0 || ndim > 3)
        fail(PARO_E_CONFIG, "token grid must have 2 or 3 axes, got " + std::to_string(ndim));
    Grid g;
    g.ndim = ndim;
    for (int a = 0; a < ndim; ++a) {
        g.labels[a] = labels[a];
        g.ext[a] = extents[a];
    }
    validate_grid(g);
    return g;
}

// Per-head permutation descriptor for `order` (make_perm, reorder.cpp:49-72):
// new index = row-major index of the old coordinates re-listed in `order`.
PermDesc perm_desc(const Grid& g, const std::string& order) {
    if ((int)order.size() != g.ndim)
        fail(PARO_E_CONFIG, "permutation order '" + order + "' does not cover the grid axes");
    uint32_t stride[3];
    uint32_t s = 1;
    for (int a = g.ndim; a-- > 0;) {
        stride[a] = s;
        s *= g.ext[a];
    }
    PermDesc pd{{1, 1, 1}, {0, 0, 0}, 0};
    const int off = 3 - g.ndim;
    for (int a = 0; a < g.ndim; ++a) {
        const int src = g.axis_index(order[a]);
        pd.pext[off + a] = g.ext[src];
        pd.ostride[off + a] = stride[src];
    }
    // a repeated label would make this a non-bijection; make_perm builds a
    // TokenGrid from the re-listed axes, which rejects duplicates (tensor.cpp:39-40)
    unsigned seen = 0;
    for (int a = 0; a < g.ndim; ++a) {
        const unsigned bit = 1u << g.axis_index(order[a]);
        if (seen & bit)
            fail(PARO_E_CONFIG, std::string("duplicate grid axis label '") + order[a] + "'");
        seen |= bit;
    }
    return pd;
}

// ---------------------------------------------------------------- PMSK helpers (mask.cpp:179-244)
uint32_t get_u32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
void put_u32(uint8_t* p, uint32_t v) {
    p[0] = (uint8_t)(v & 0xff);
    p[1] = (uint8_t)((v >> 8) & 0xff);
    p[2] = (uint8_t)((v >> 16) & 0xff);
    p[3] = (uint8_t)((v >> 24) & 0xff);
}

size_t decode_pmsk(const uint8_t* data, size_t size, uint32_t* kr, uint32_t* kc, uint32_t* block, uint8_t* bits) {
    if (size < 18)
        fail(PARO_E_FORMAT, "mask blob truncated: need 18 header bytes, have " + std::to_string(size));
    if (std::memcmp(data, "PMSK", 4) != 0)
        fail(PARO_E_FORMAT, "bad mask magic, expected \"PMSK\" (at byte offset 0)");
    if (data[4] != 1)
        fail(PARO_E_FORMAT, "unsupported mask version " + std::to_string(data[4]) + " (at byte offset 4)");
    const uint32_t r = get_u32(data + 6), c = get_u32(data + 10), b = get_u32(data + 14);
    if (r == 0 || c == 0 || b == 0)
        fail(PARO_E_FORMAT, "mask dimensions must be nonzero");
    const size_t row_bytes = (c + 7) / 8;
    const size_t need = 18 + (size_t)r * row_bytes;
    if (size < need)
        fail(PARO_E_FORMAT, "mask blob truncated: need " + std::to_string(need) + " bytes, have " + std::to_string(size));
    if (kr)
        *kr = r;
    if (kc)
        *kc = c;
    if (block)
        *block = b;
    if (bits)
        for (size_t i = 0; i < r; ++i) {
            const uint8_t* row = data + 18 + i * row_bytes;
            for (size_t j = 0; j < c; ++j)
                bits[i * c + j] = (row[j / 8] >> (j % 8)) & 1u;
        }
    return need;
}

} // namespace

// ============================================================================
// device context / layer objects
// ============================================================================
struct paro_ctx {
    int device = 0;
    int num_sms = 0;
    size_t l2_bytes = 0;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    char* pinned = nullptr; // host staging of select_permutation, grown on demand
    size_t pinned_bytes = 0;
    ~paro_ctx() {
        if (pinned)
            cudaFreeHost(pinned);
    }
    char* pinned_scratch(size_t bytes) {
        if (bytes > pinned_bytes) {
            if (pinned)
                cudaFreeHost(pinned);
            pinned = nullptr;
            pinned_bytes = 0;
            cuda_check(cudaMallocHost(reinterpret_cast<void**>(&pinned), bytes), "pinned staging");
            pinned_bytes = bytes;
        }
        return pinned;
    }
};

struct paro_layer {
    paro_ctx* ctx = nullptr;
    Grid grid;
    LayerDev L{};
    std::vector<PermDesc> perm_host;
    uint32_t* fwd = nullptr; // [H][N]
    uint32_t* inv = nullptr; // [H][N]
    uint8_t* mask_dev = nullptr;
    bool masks_set = false;
    int last_v_bits = 0;
    int last_launches = 0;
    CUtensorMap tm_q, tm_k, tm_v, tm_vp; // tm_vp: nibble-packed INT4 V (D/2 bytes per row)
    CUtensorMap tm_q32;                  // Q codes in 32-row boxes (K3's M = 128 layout, PARO_M128)
    CUtensorMap tm_vh, tm_vl;            // dense prefix: K4a's bf16 V^T hi / lo tiles (K4 on tcgen05)
    // e2e staging
    float* rope = nullptr; // [2][N - dp][D]: cos, sin (paro_layer_set_rope)
    float *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr;
    uint8_t* dzero = nullptr;
    cudaStream_t s_in = nullptr, s_out = nullptr; // H2D / D2H copy streams
    std::vector<cudaEvent_t> ev;                  // [0] start, then per chunk: in, computed, out
    // per-timestep mask schedule (paro_layer_set_schedule)
    struct Lists { // K2 outputs of one schedule entry, all heads
        uint16_t* items = nullptr;
        uint32_t *pairs = nullptr, *pair_count = nullptr, *qb_count = nullptr, *order = nullptr, *order_chunk = nullptr;
        int entry = -1;
        cudaEvent_t ready = nullptr;
    };
    bool v_pack = false; // INT4 V nibble-packed in HBM (paro_layer_set_v_packing)
    uint32_t sched_T = 0, sched_entries = 0, sched_resident = 0;
    uint8_t* sched_masks = nullptr; // [entries][H][kb][kb] (block bytes, uploaded once)
    std::vector<Lists> sched_lists; // entries (resident) or 2 (double-buffered prefetch)
    int sched_cur = -1;             // index into sched_lists of the current timestep's lists
    cudaStream_t s_k2 = nullptr;    // prefetch stream
    cudaEvent_t ev_prefetch = nullptr;
    Lists base;                     // the layer's own K2 buffers (set_masks)
};

namespace {

// Host-buffer pipeline depth (paro_layer_set_pipeline_chunks overrides): at
// least 8 chunks, and no chunk uploading more than ~96 MB of Q/K/V, so the
// un-overlapped first upload and last download stay short when the layer is
// compute-bound (c5: 40 chunks, e2e 152 -> 141 ms) while PCIe-bound layers keep
// chunks big enough to amortise launches (c2 8, c4 8; measured sweeps).
constexpr uint32_t kMinChunks = 8;
constexpr size_t kChunkBytes = 96u << 20;
uint32_t default_heads_per_chunk(uint32_t heads, size_t tokens, uint32_t d) {
    const size_t per_head = tokens * d * 4 * 3;
    const uint32_t by_count = (heads + kMinChunks - 1) / kMinChunks;
    const uint32_t by_bytes = (uint32_t)std::max<size_t>(1, kChunkBytes / per_head);
    return std::max(1u, std::min(by_count, by_bytes));
}

// Chunk table of the host-buffer pipeline: chunks of hpc heads, the last one
// tapered into halving pieces (hpc/2, hpc/4, ..., 1) when `taper`: what runs
// after the final upload (its kernels and download) shrinks to about one head's
// worth (c2: the last chunk's 0.67 ms kernels + 0.5 ms download were the tail).
void set_chunks(paro::LayerDev& L, uint32_t hpc, bool taper) {
    std::vector<uint32_t> sizes;
    uint32_t left = L.H;
    while (left > 0) {
        const uint32_t n = std::min(hpc, left);
        sizes.push_back(n);
        left -= n;
    }
    if (taper && sizes.back() > 1) {
        uint32_t last = sizes.back();
        sizes.pop_back();
        while (last > 1) {
            const uint32_t piece = (last + 1) / 2;
            sizes.push_back(piece);
            last -= piece;
        }
        sizes.push_back(last);
    }
    while (sizes.size() > paro::kMaxChunks) { // merge the leading chunks pairwise
        std::vector<uint32_t> merged;
        for (size_t i = 0; i < sizes.size(); i += 2)
            merged.push_back(sizes[i] + (i + 1 < sizes.size() ? sizes[i + 1] : 0));
        sizes = merged;
    }
    L.nchunks = (uint32_t)sizes.size();
    L.chunk_start[0] = 0;
    for (uint32_t c = 0; c < L.nchunks; ++c)
        L.chunk_start[c + 1] = L.chunk_start[c] + sizes[c];
}

void set_device(const paro_ctx* ctx) { cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice"); }

template <typename T>
T* dalloc(size_t count) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    return static_cast<T*>(p);
}

// K4a's V^T tiles: [H*kb2*D rows][64 bf16], 128B swizzle, one tile = D rows (the
// K-major B operand of K4's bf16 P.V MMA)
void encode_vt_map(paro_ctx* ctx, CUtensorMap* m, uint16_t* base, uint32_t D, uint64_t rows) {
    cuuint64_t dims[2] = {64, rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, D};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = ctx->encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(PARO_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// nibble-packed INT4 V: rows of D/2 bytes, no swizzle (K3 unpacks into the swizzled tile)
void encode_packed_map(paro_ctx* ctx, CUtensorMap* m, int8_t* base, uint32_t D, uint64_t rows, uint32_t box_rows) {
    cuuint64_t dims[2] = {D / 2, rows};
    cuuint64_t strides[1] = {D / 2};
    cuuint32_t box[2] = {D / 2, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = ctx->encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(PARO_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

void encode_codes_map(paro_ctx* ctx, CUtensorMap* m, int8_t* base, uint32_t D, uint64_t rows, uint32_t box_rows) {
    cuuint64_t dims[2] = {D, rows};
    cuuint64_t strides[1] = {D};
    cuuint32_t box[2] = {D, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = ctx->encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE,
                             D == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(PARO_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// ---------------------------------------------------------------- mask schedules
static void use_lists(paro_layer* l, const paro_layer::Lists& x) {
    l->L.items = x.items;
    l->L.pairs = x.pairs;
    l->L.pair_count = x.pair_count;
    l->L.qb_count = x.qb_count;
    l->L.order = x.order;
    l->L.order_chunk = x.order_chunk;
}
static paro_layer::Lists current_lists(const paro_layer* l) {
    paro_layer::Lists x;
    x.items = l->L.items;
    x.pairs = l->L.pairs;
    x.pair_count = l->L.pair_count;
    x.qb_count = l->L.qb_count;
    x.order = l->L.order;
    x.order_chunk = l->L.order_chunk;
    return x;
}
static paro_layer::Lists alloc_lists(const LayerDev& L) {
    paro_layer::Lists x;
    x.items = dalloc<uint16_t>((size_t)L.H * L.kb * L.kb);
    x.pairs = dalloc<uint32_t>((size_t)L.H * L.np);
    x.pair_count = dalloc<uint32_t>((size_t)L.H * L.np);
    x.qb_count = dalloc<uint32_t>((size_t)L.H * L.kb2);
    x.order = dalloc<uint32_t>((size_t)L.H * L.np);
    x.order_chunk = dalloc<uint32_t>((size_t)L.H * L.np);
    cuda_check(cudaMemset(x.qb_count, 0, (size_t)L.H * L.kb2 * 4), "cudaMemset");
    cuda_check(cudaEventCreateWithFlags(&x.ready, cudaEventDisableTiming), "event create");
    return x;
}
void clear_schedule(paro_layer* l) {
    if (!l->sched_T)
        return;
    for (auto& x : l->sched_lists) {
        cudaFree(x.items);
        cudaFree(x.pairs);
        cudaFree(x.pair_count);
        cudaFree(x.qb_count);
        cudaFree(x.order);
        cudaFree(x.order_chunk);
        cudaEventDestroy(x.ready);
    }
    l->sched_lists.clear();
    cudaFree(l->sched_masks);
    l->sched_masks = nullptr;
    if (l->s_k2)
        cudaStreamDestroy(l->s_k2);
    if (l->ev_prefetch)
        cudaEventDestroy(l->ev_prefetch);
    l->s_k2 = nullptr;
    l->ev_prefetch = nullptr;
    l->sched_T = l->sched_entries = 0;
    l->sched_cur = -1;
    use_lists(l, l->base);
    l->masks_set = false;
}
// K2 of schedule entry e into list buffer x, on stream st
static void build_entry(paro_layer* l, paro_layer::Lists& x, uint32_t e, cudaStream_t st) {
    LayerDev tmp = l->L;
    tmp.items = x.items;
    tmp.pairs = x.pairs;
    tmp.pair_count = x.pair_count;
    tmp.qb_count = x.qb_count;
    tmp.order = x.order;
    tmp.order_chunk = x.order_chunk;
    const size_t per = (size_t)l->L.H * l->L.kb * l->L.kb;
    cuda_check(paro::launch_k2(tmp, l->sched_masks + (size_t)e * per, st), "k2 launch (schedule)");
    cuda_check(cudaEventRecord(x.ready, st), "event record");
    x.entry = (int)e;
}

void free_layer(paro_layer* l) {
    clear_schedule(l); // restores the layer's own K2 buffers into l->L
    cudaFree(l->L.perm);
    cudaFree(l->L.q);
    cudaFree(l->L.k);
    cudaFree(l->L.v);
    cudaFree(l->L.qsc);
    cudaFree(l->L.meta);
    cudaFree(l->L.items);
    cudaFree(l->L.pairs);
    cudaFree(l->L.pair_count);
    cudaFree(l->L.qb_count);
    cudaFree(l->L.order);
    cudaFree(l->L.work_counter);
    cudaFree(l->fwd);
    cudaFree(l->inv);
    cudaFree(l->mask_dev);
    cudaFree(l->rope);
    cudaFree(l->dq);
    cudaFree(l->dk);
    cudaFree(l->dv);
    cudaFree(l->dout);
    cudaFree(l->dzero);
    cudaFree(l->L.order_chunk);
    cudaFree(l->L.init_m);
    cudaFree(l->L.init_l);
    cudaFree(l->L.init_acc);
    cudaFree(l->L.part_m);
    cudaFree(l->L.part_l);
    cudaFree(l->L.part_acc);
    cudaFree(l->L.vsplit_hi);
    cudaFree(l->L.vsplit_lo);
    for (cudaEvent_t e : l->ev)
        cudaEventDestroy(e);
    if (l->s_in)
        cudaStreamDestroy(l->s_in);
    if (l->s_out)
        cudaStreamDestroy(l->s_out);
}

void check_bits(int bits) {
    if (bits != 4 && bits != 8)
        fail(PARO_E_CONFIG, "quantization bitwidth must be 4 or 8, got " + std::to_string(bits)); // quant.cpp:15-17
}

// K1 / K4a read Q/K/V rows and K3 writes O rows with 16-byte vector accesses
void check_aligned16(const void* p, const char* what) {
    if (reinterpret_cast<uintptr_t>(p) & 15u)
        fail(PARO_E_CONFIG, std::string(what) + " must be 16-byte aligned (vectorised row access)");
}

void check_layer(const paro_layer* l) {
    if (!l)
        fail(PARO_E_CONFIG, "null layer");
}

void run_attention(paro_layer* l, cudaStream_t st, float scale, int pv_bits, float* out, uint8_t* zeroed,
                   uint32_t head_begin = 0, uint32_t head_count = ~0u, bool chunked = false,
                   const paro::K3Dump* dump = nullptr) {
    check_bits(pv_bits);
    if (!l->masks_set)
        fail(PARO_E_CONFIG, "paro_layer_set_masks must be called before attention");
    if (pv_bits != l->last_v_bits)
        fail(PARO_E_CONFIG, "pv_bits " + std::to_string(pv_bits) + " does not match the V codes (" +
                                std::to_string(l->last_v_bits) + " bits); rerun reorder_quantize");
    if (!out)
        fail(PARO_E_CONFIG, "null output");
    // AttnInputs::effective_scale (attention.cpp:26-28), in fp64 exactly as the reference
    const double eff = scale != 0.0f ? (double)scale : 1.0 / std::sqrt((double)l->L.D);
    if (head_count == ~0u)
        head_count = l->L.H;
    if (l->L.dp) { // dense text-token prefix: dense rows done, the others' state for K3
        cuda_check(paro::launch_k4(l->L, eff, out, zeroed, head_begin, head_count, st, &l->tm_q, &l->tm_k, &l->tm_vh,
                                   &l->tm_vl),
                   "k4 launch");
    }
    cuda_check(paro::launch_k3(l->L, l->tm_q, l->tm_k, l->tm_v, l->tm_vp, l->tm_q32, eff, pv_bits, out, zeroed, l->ctx->num_sms, st,
                               head_begin, head_count, chunked, dump),
               "k3_attention launch");
}

} // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* paro_last_error(void) { return g_last_error.c_str(); }
const char* paro_version(void) { return "paro_b200 0.1 (sm_100a)"; }

int paro_parse_grid(const char* text, int* ndim, char* labels, uint32_t* extents) {
    return guarded([&] {
        Grid g = parse_grid_text(text);
        *ndim = g.ndim;
        for (int a = 0; a < g.ndim; ++a) {
            labels[a] = g.labels[a];
            extents[a] = g.ext[a];
        }
    });
}

int paro_make_perm(int ndim, const char* labels, const uint32_t* extents, const char* order, uint32_t* forward,
                   uint32_t* inverse) {
    return guarded([&] {
        Grid g = grid_from(ndim, labels, extents);
        PermDesc pd = perm_desc(g, order ? std::string(order) : std::string());
        const size_t n = g.tokens();
        for (size_t i = 0; i < n; ++i) {
            const uint32_t old = paro::perm_src(pd, (uint32_t)i);
            inverse[i] = old;
            forward[old] = (uint32_t)i;
        }
    });
}

// ---------------------------------------------------------------- per-head plan text
// load_plan_file (reorder.cpp:193-216) on an in-memory image: one "head_id,order"
// per line, empty lines skipped; the head id parses like std::stoul (leading
// blanks, sign, trailing text allowed; no digits or out of range -> "bad head id");
// the order is the text after the first comma (validated when a plan is made).
namespace {
struct PlanEntry {
    uint32_t head;
    std::string order;
};
std::vector<PlanEntry> parse_plan(const char* text, size_t len, const std::string& name) {
    std::vector<PlanEntry> out;
    size_t pos = 0, lineno = 0;
    while (pos < len) {
        size_t end = pos;
        while (end < len && text[end] != '\n')
            ++end;
        const std::string line(text + pos, end - pos);
        pos = end + 1;
        ++lineno;
        if (line.empty())
            continue;
        const size_t comma = line.find(',');
        if (comma == std::string::npos)
            fail(PARO_E_FORMAT, name + ":" + std::to_string(lineno) + ": expected head_id,order");
        const std::string id = line.substr(0, comma);
        errno = 0;
        char* stop = nullptr;
        const unsigned long v = std::strtoul(id.c_str(), &stop, 10);
        if (stop == id.c_str() || errno == ERANGE)
            fail(PARO_E_FORMAT, name + ":" + std::to_string(lineno) + ": bad head id");
        out.push_back({static_cast<uint32_t>(v), line.substr(comma + 1)});
    }
    return out;
}
} // namespace

int paro_parse_plan(const char* text, size_t len, const char* name, uint32_t* count, uint32_t* heads, char* orders,
                    size_t* orders_size) {
    return guarded([&] {
        const auto e = parse_plan(text ? text : "", text ? len : 0, name ? name : "plan");
        size_t need = 0;
        for (const auto& x : e)
            need += x.order.size() + 1;
        *count = (uint32_t)e.size();
        if (orders_size) {
            if (orders && *orders_size < need)
                fail(PARO_E_CONFIG, "plan orders buffer too small");
            *orders_size = need;
        }
        if (heads)
            for (size_t i = 0; i < e.size(); ++i)
                heads[i] = e[i].head;
        if (orders) {
            size_t o = 0;
            for (const auto& x : e) {
                std::memcpy(orders + o, x.order.c_str(), x.order.size() + 1);
                o += x.order.size() + 1;
            }
        }
    });
}

int paro_plan_for_heads(const char* text, size_t len, const char* name, const char* grid_text, uint32_t n,
                        const uint32_t* head_ids, char* orders_out) {
    return guarded([&] {
        // plan_for_head (tools/main.cpp:118-126): no plan -> identity (the grid's own
        // label order); otherwise the first entry naming the head, else InputError
        Grid g = parse_grid_text(grid_text);
        const std::string ident(g.labels, g.labels + g.ndim);
        std::vector<PlanEntry> e;
        const std::string nm = name ? name : "plan";
        if (text)
            e = parse_plan(text, len, nm);
        for (uint32_t i = 0; i < n; ++i) {
            std::string order = ident;
            if (text) {
                const PlanEntry* hit = nullptr;
                for (const auto& x : e)
                    if (x.head == head_ids[i]) {
                        hit = &x;
                        break;
                    }
                if (!hit)
                    fail(PARO_E_INPUT, nm + ": no plan entry for head " + std::to_string(head_ids[i]));
                order = hit->order;
            }
            perm_desc(g, order); // make_perm's validation of the order (ConfigError / InputError)
            std::memcpy(orders_out + (size_t)i * ident.size(), order.data(), ident.size());
        }
    });
}

int paro_enumerate_orders(int ndim, const char* labels, char* orders, int* count) {
    return guarded([&] {
        if (ndim != 2 && ndim != 3)
            fail(PARO_E_CONFIG, "token grid must have 2 or 3 axes, got " + std::to_string(ndim));
        // reorder.cpp:74-91: identity first, then the remaining orders in lexicographic order
        std::string ident(labels, labels + ndim);
        std::string perm = ident;
        std::sort(perm.begin(), perm.end());
        std::vector<std::string> out{ident};
        do {
            if (perm != ident)
                out.push_back(perm);
        } while (std::next_permutation(perm.begin(), perm.end()));
        *count = (int)out.size();
        for (size_t i = 0; i < out.size(); ++i)
            std::memcpy(orders + i * ndim, out[i].data(), ndim);
    });
}

int paro_deserialize_mask(const uint8_t* data, size_t size, uint32_t* k_rows, uint32_t* k_cols, uint32_t* block,
                          uint8_t* bits, size_t* consumed) {
    return guarded([&] {
        const size_t used = decode_pmsk(data, size, k_rows, k_cols, block, bits);
        if (consumed)
            *consumed = used;
    });
}

int paro_serialize_mask(const uint8_t* bits, uint32_t k_rows, uint32_t k_cols, uint32_t block, uint8_t* out,
                        size_t* size) {
    return guarded([&] {
        const size_t row_bytes = (k_cols + 7) / 8;
        const size_t total = 18 + (size_t)k_rows * row_bytes;
        *size = total;
        if (!out)
            return;
        std::memcpy(out, "PMSK", 4);
        out[4] = 1;
        out[5] = 0;
        put_u32(out + 6, k_rows);
        put_u32(out + 10, k_cols);
        put_u32(out + 14, block);
        std::memset(out + 18, 0, total - 18);
        for (size_t i = 0; i < k_rows; ++i)
            for (size_t j = 0; j < k_cols; ++j)
                if (bits[i * k_cols + j])
                    out[18 + i * row_bytes + j / 8] |= (uint8_t)(1u << (j % 8)); // LSB first
    });
}

// PSCH (mask.cpp:246-305): magic, u32 timesteps, u32 distinct (= T/2), (u32 t,
// PMSK) x distinct, shared PMSK. Validates like load_schedule and returns the
// T/2 + 1 PMSK blobs in at() order: distinct[i] by POSITION (at(t) ignores the
// stored timestep field, mask.cpp:132-140), then the shared late mask.
static uint32_t parse_psch(const uint8_t* data, size_t size, std::vector<std::pair<const uint8_t*, size_t>>& ent) {
    if (size < 12)
        fail(PARO_E_FORMAT, "truncated schedule header (at byte offset " + std::to_string(size) + ")");
    if (std::memcmp(data, "PSCH", 4) != 0)
        fail(PARO_E_FORMAT, "bad magic, expected \"PSCH\" (at byte offset 0)");
    const uint32_t T = get_u32(data + 4), nd = get_u32(data + 8);
    if (nd != T / 2)
        fail(PARO_E_FORMAT, "schedule declares " + std::to_string(nd) + " distinct masks, expected " +
                                std::to_string(T / 2));
    ent.clear();
    size_t off = 12;
    for (uint32_t i = 0; i < nd; ++i) {
        if (size < off + 4)
            fail(PARO_E_FORMAT, "truncated distinct entry (schedule parse position " + std::to_string(off) + ")");
        off += 4;
        const size_t used = decode_pmsk(data + off, size - off, nullptr, nullptr, nullptr, nullptr);
        ent.emplace_back(data + off, used);
        off += used;
    }
    const size_t used = decode_pmsk(data + off, size - off, nullptr, nullptr, nullptr, nullptr);
    ent.emplace_back(data + off, used);
    off += used;
    if (off != size)
        fail(PARO_E_FORMAT, std::to_string(size - off) + " trailing bytes (at byte offset " + std::to_string(off) + ")");
    return T;
}

// MaskSchedule::at(t) as an entry index into parse_psch's list (mask.cpp:132-140)
static uint32_t schedule_entry(uint32_t T, uint32_t t) {
    if (t >= T)
        fail(PARO_E_INPUT, "timestep " + std::to_string(t) + " out of range, schedule covers " + std::to_string(T));
    return t < T / 2 ? t : T / 2;
}

int paro_schedule_at(const uint8_t* data, size_t size, uint32_t t, uint32_t* k_rows, uint32_t* k_cols,
                     uint32_t* block, uint8_t* bits) {
    return guarded([&] {
        std::vector<std::pair<const uint8_t*, size_t>> ent;
        const uint32_t T = parse_psch(data, size, ent);
        const auto& e = ent[schedule_entry(T, t)];
        decode_pmsk(e.first, e.second, k_rows, k_cols, block, bits);
    });
}

// ---------------------------------------------------------------- PAT1 / PARQ interchange
// Byte-exact restatements of save_tensor / load_tensor (tensor_io.cpp:45-120,
// layout tensor_io.hpp:13-26) and save_quant_tensor / load_quant_tensor
// (quant.cpp:219-326, layout quant.hpp:68-72), in memory; FormatError messages
// name the byte offset of the first violation like the reference's.
namespace {
void put_u32(std::vector<uint8_t>& o, uint32_t v) {
    for (int i = 0; i < 4; ++i)
        o.push_back((uint8_t)(v >> (8 * i)));
}
void put_f32(std::vector<uint8_t>& o, float f) {
    uint32_t b;
    std::memcpy(&b, &f, 4);
    put_u32(o, b);
}
float get_f32(const uint8_t* p) {
    const uint32_t b = get_u32(p);
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}
void emit(const std::vector<uint8_t>& bytes, uint8_t* out, size_t* size) {
    if (out) {
        if (*size < bytes.size())
            fail(PARO_E_SHAPE, "output buffer holds " + std::to_string(*size) + " bytes, need " +
                                   std::to_string(bytes.size()));
        std::memcpy(out, bytes.data(), bytes.size());
    }
    *size = bytes.size();
}
[[noreturn]] void format_at(size_t off, const std::string& why) {
    fail(PARO_E_FORMAT, why + " (at byte offset " + std::to_string(off) + ")");
}
size_t quant_groups(int grouping, uint32_t block, uint32_t rows, uint32_t cols) {
    if (grouping == 1)
        return rows;
    return (size_t)((rows + block - 1) / block) * ((cols + block - 1) / block);
}
void quant_validate(unsigned bits, uint32_t block) { // QuantConfig::validate (quant.cpp:15-19)
    if (bits != 4 && bits != 8)
        fail(PARO_E_CONFIG, "quantization bitwidth must be 4 or 8, got " + std::to_string(bits));
    if (block < 1)
        fail(PARO_E_CONFIG, "quantization block must be >= 1");
}
std::vector<uint8_t> parq_bytes(unsigned bits, int mode, int grouping, uint32_t block, uint32_t rows, uint32_t cols,
                                const int32_t* codes, const float* scales, size_t ngroups, const float* offsets) {
    std::vector<uint8_t> o;
    const size_t count = (size_t)rows * cols;
    o.reserve(24 + 8 * ngroups + count);
    o.insert(o.end(), {'P', 'A', 'R', 'Q', 1, (uint8_t)bits, (uint8_t)mode, (uint8_t)grouping});
    put_u32(o, block);
    put_u32(o, rows);
    put_u32(o, cols);
    put_u32(o, (uint32_t)ngroups);
    for (size_t g = 0; g < ngroups; ++g)
        put_f32(o, scales[g]);
    if (mode == 0 && offsets)
        for (size_t g = 0; g < ngroups; ++g)
            put_f32(o, offsets[g]);
    if (bits == 8) {
        for (size_t i = 0; i < count; ++i)
            o.push_back((uint8_t)(codes[i] & 0xff));
    } else { // two per byte, low nibble first (quant.cpp:237-243)
        for (size_t i = 0; i < count; i += 2) {
            const unsigned lo = (unsigned)codes[i] & 0xfu, hi = i + 1 < count ? (unsigned)codes[i + 1] & 0xfu : 0u;
            o.push_back((uint8_t)(lo | hi << 4));
        }
    }
    return o;
}
} // namespace

int paro_tensor_encode(const uint32_t* shape, uint32_t ndim, const float* values, uint8_t* out, size_t* size) {
    return guarded([&] {
        if (ndim == 0 || ndim > 255)
            fail(PARO_E_CONFIG, "tensor ndim must be in [1,255]");
        size_t count = 1;
        for (uint32_t a = 0; a < ndim; ++a)
            count *= shape[a];
        std::vector<uint8_t> o{'P', 'A', 'R', 'O', 1, 0, (uint8_t)ndim, 0};
        for (uint32_t a = 0; a < ndim; ++a)
            put_u32(o, shape[a]);
        const size_t h = o.size();
        o.resize(h + count * 4);
        if (count)
            std::memcpy(o.data() + h, values, count * 4); // little-endian binary32
        emit(o, out, size);
    });
}

int paro_tensor_decode(const uint8_t* p, size_t size, uint32_t* ndim_out, uint32_t* shape, float* values) {
    return guarded([&] {
        if (size < 8)
            format_at(size, "truncated header, need 8 bytes");
        if (std::memcmp(p, "PARO", 4) != 0)
            format_at(0, "bad magic, expected \"PARO\"");
        if (p[4] != 1)
            format_at(4, "unsupported version " + std::to_string(p[4]));
        if (p[5] != 0)
            format_at(5, "unsupported dtype " + std::to_string(p[5]));
        const size_t ndim = p[6];
        if (ndim == 0)
            format_at(6, "ndim must be >= 1");
        if (p[7] != 0)
            format_at(7, "reserved byte must be 0");
        const size_t header = 8 + 4 * ndim;
        if (size < header)
            format_at(size, "truncated extents, need " + std::to_string(header) + " header bytes");
        size_t count = 1;
        for (size_t a = 0; a < ndim; ++a) {
            const uint32_t e = get_u32(p + 8 + 4 * a);
            if (e == 0)
                format_at(8 + 4 * a, "zero extent");
            if (shape)
                shape[a] = e;
            count *= e;
        }
        const size_t payload = count * 4;
        if (size != header + payload)
            format_at(size, "payload length mismatch, expected " + std::to_string(payload) + " bytes, found " +
                                std::to_string(size - header));
        *ndim_out = (uint32_t)ndim;
        if (values)
            std::memcpy(values, p + header, payload);
    });
}

int paro_quant_encode(unsigned bits, int mode, int grouping, uint32_t block, uint32_t rows, uint32_t cols,
                      const int32_t* codes, const float* scales, const float* offsets, uint8_t* out, size_t* size) {
    return guarded([&] {
        quant_validate(bits, block);
        if (mode != 0 && mode != 1)
            fail(PARO_E_CONFIG, "quantization mode must be 0 (unsigned) or 1 (symmetric)");
        if (grouping != 0 && grouping != 1)
            fail(PARO_E_CONFIG, "quantization grouping must be 0 (per block) or 1 (per row)");
        const size_t ng = quant_groups(grouping, block, rows, cols);
        emit(parq_bytes(bits, mode, grouping, block, rows, cols, codes, scales, ng, mode == 0 ? offsets : nullptr), out,
             size);
    });
}

int paro_quant_decode(const uint8_t* p, size_t size, paro_quant_header* hdr, int32_t* codes, float* scales,
                      float* offsets) {
    return guarded([&] {
        if (size < 24)
            format_at(size, "truncated header");
        if (std::memcmp(p, "PARQ", 4) != 0)
            format_at(0, "bad magic, expected \"PARQ\"");
        if (p[4] != 1)
            format_at(4, "unsupported version " + std::to_string(p[4]));
        const unsigned bits = p[5];
        if (p[6] > 1)
            format_at(6, "bad mode byte");
        if (p[7] > 1)
            format_at(7, "bad grouping byte");
        const uint32_t block = get_u32(p + 8);
        quant_validate(bits, block);
        const uint32_t rows = get_u32(p + 12), cols = get_u32(p + 16), ng = get_u32(p + 20);
        const int mode = p[6], grouping = p[7];
        if (ng != quant_groups(grouping, block, rows, cols))
            format_at(20, "group count " + std::to_string(ng) + " does not match shape");
        size_t off = 24;
        auto need = [&](size_t n, const char* what) {
            if (size < off + n)
                format_at(off, std::string("truncated ") + what);
        };
        need(4ull * ng, "scales");
        if (scales)
            for (uint32_t g = 0; g < ng; ++g)
                scales[g] = get_f32(p + off + 4ull * g);
        off += 4ull * ng;
        if (mode == 0) {
            need(4ull * ng, "offsets");
            if (offsets)
                for (uint32_t g = 0; g < ng; ++g)
                    offsets[g] = get_f32(p + off + 4ull * g);
            off += 4ull * ng;
        }
        const size_t count = (size_t)rows * cols;
        const size_t packed = bits == 8 ? count : (count + 1) / 2;
        need(packed, "codes");
        if (codes) {
            for (size_t i = 0; i < count; ++i) {
                int32_t v;
                if (bits == 8) {
                    v = p[off + i];
                    if (mode == 1 && v >= 128)
                        v -= 256;
                } else {
                    const unsigned byte = p[off + i / 2];
                    v = (int32_t)((i % 2 == 0) ? (byte & 0xfu) : (byte >> 4));
                    if (mode == 1 && v >= 8)
                        v -= 16;
                }
                codes[i] = v;
            }
        }
        off += packed;
        if (off != size)
            format_at(off, std::to_string(size - off) + " trailing bytes");
        hdr->bits = bits;
        hdr->mode = mode;
        hdr->grouping = grouping;
        hdr->block = block;
        hdr->rows = rows;
        hdr->cols = cols;
        hdr->groups = ng;
    });
}

// gen_mask's configuration checks (mask.cpp:57-76); returns the number of
// non-guard blocks to keep (target - guard_count)
static uint64_t gen_mask_keep_count(uint32_t kr, uint32_t kc, double density, uint32_t guard) {
    if (!(density > 0.0 && density <= 1.0))
        fail(PARO_E_CONFIG, "density must be in (0,1], got " + std::to_string(density));
    const size_t total = (size_t)kr * kc;
    const size_t target = (size_t)std::ceil(density * (double)total);
    size_t guard_count = 0;
    if (guard > 0) {
        const size_t gr = std::min<size_t>(guard, kr), gc = std::min<size_t>(guard, kc);
        guard_count = total - (kr - gr) * (kc - gc);
    }
    if (guard_count > target)
        fail(PARO_E_CONFIG, "density " + std::to_string(density) + " keeps " + std::to_string(target) +
                                " blocks but the dense prefix alone occupies " + std::to_string(guard_count));
    if (guard == 0 && target < kr)
        fail(PARO_E_CONFIG, "density " + std::to_string(density) + " keeps " + std::to_string(target) +
                                " blocks, fewer than the " + std::to_string(kr) + " rows that each need one");
    return (uint64_t)(target - guard_count);
}

int paro_perm_block_sums_device(paro_ctx* ctx, paro_stream_t stream, const float* map, uint32_t n,
                                const uint32_t* inverse, uint32_t block, double* sums) {
    return guarded([&] {
        if (block < 1)
            fail(PARO_E_CONFIG, "block must be >= 1");
        if (n == 0)
            fail(PARO_E_SHAPE, "empty attention map");
        if (block > 256)
            fail(PARO_E_CONFIG, "device block_sums supports block <= 256");
        set_device(ctx);
        cuda_check(paro::launch_perm_block_sums(map, n, inverse, block, sums, (cudaStream_t)stream),
                   "perm_block_sums");
    });
}

// gen_mask for `count` grids on the device (synchronises `stream` to return
// the repaired-row counts and the repair failure status)
static void gen_mask_device_impl(const double* sums, uint32_t count, uint32_t kr, uint32_t kc, double density,
                                 uint32_t guard, uint8_t* bits, uint32_t* repaired_rows, cudaStream_t st) {
    const uint64_t K = gen_mask_keep_count(kr, kc, density, guard);
    uint32_t* scratch = nullptr; // row_kept [count][kr] + repaired [count] + status
    const size_t words = (size_t)count * kr + count + 1;
    cuda_check(cudaMalloc(&scratch, words * 4), "gen_mask scratch");
    struct Free {
        uint32_t* p;
        ~Free() { cudaFree(p); }
    } guard_free{scratch};
    cuda_check(cudaMemsetAsync(scratch, 0, words * 4, st), "gen_mask scratch");
    uint32_t* rep_dev = scratch + (size_t)count * kr;
    int* status_dev = reinterpret_cast<int*>(rep_dev + count);
    cuda_check(paro::launch_gen_mask(sums, count, kr, kc, guard, K, bits, scratch, rep_dev, status_dev, st),
               "gen_mask");
    std::vector<uint32_t> host(count + 1);
    cuda_check(cudaMemcpyAsync(host.data(), rep_dev, (count + 1) * 4, cudaMemcpyDeviceToHost, st), "gen_mask");
    cuda_check(cudaStreamSynchronize(st), "gen_mask");
    if (host[count] != 0)
        fail(PARO_E_CONFIG, "cannot repair an empty mask row at density " + std::to_string(density));
    if (repaired_rows)
        std::memcpy(repaired_rows, host.data(), count * 4);
}

int paro_gen_mask_device(paro_ctx* ctx, paro_stream_t stream, const double* sums, uint32_t count, uint32_t k_rows,
                         uint32_t k_cols, double density, uint32_t block, uint32_t guard, uint8_t* bits,
                         uint32_t* repaired_rows) {
    return guarded([&] {
        (void)block; // recorded in the BlockMask only (mask.cpp:86)
        if (count == 0 || k_rows == 0 || k_cols == 0)
            fail(PARO_E_SHAPE, "empty block-sum grid");
        set_device(ctx);
        gen_mask_device_impl(sums, count, k_rows, k_cols, density, guard, bits, repaired_rows, (cudaStream_t)stream);
    });
}

int paro_build_schedule_device(paro_ctx* ctx, paro_stream_t stream, const double* sums, uint32_t timesteps,
                               uint32_t k_rows, uint32_t k_cols, double density, uint32_t block, uint32_t guard,
                               uint8_t* masks, uint32_t* repaired_rows) {
    return guarded([&] {
        (void)block;
        if (timesteps < 1)
            fail(PARO_E_CONFIG, "schedule needs at least one timestep");
        if (k_rows == 0 || k_cols == 0)
            fail(PARO_E_SHAPE, "empty block-sum grid");
        set_device(ctx);
        const cudaStream_t st = (cudaStream_t)stream;
        const uint32_t half = timesteps / 2;
        const size_t total = (size_t)k_rows * k_cols;
        uint32_t rep_total = 0;
        std::vector<uint32_t> rep(half > 0 ? half : 1);
        if (half > 0) { // distinct early masks, one per timestep (mask.cpp:155-159)
            gen_mask_device_impl(sums, half, k_rows, k_cols, density, guard, masks, rep.data(), st);
            for (uint32_t t = 0; t < half; ++t)
                rep_total += rep[t];
        }
        double* mean = nullptr; // shared late mask from the mean of the late sums (:160-169)
        cuda_check(cudaMalloc(&mean, total * sizeof(double)), "schedule mean");
        struct Free {
            double* p;
            ~Free() { cudaFree(p); }
        } guard_free{mean};
        cuda_check(paro::launch_late_mean(sums, timesteps, total, mean, st), "schedule mean");
        uint32_t r = 0;
        gen_mask_device_impl(mean, 1, k_rows, k_cols, density, guard, masks + (size_t)half * total, &r, st);
        rep_total += r;
        if (repaired_rows)
            *repaired_rows = rep_total;
    });
}

int paro_select_permutation_device(paro_ctx* ctx, paro_stream_t stream, const float* maps, uint32_t count,
                                   const char* grid_text, uint32_t block, float eps, float sigma, float alpha,
                                   uint32_t dense_prefix, char* orders, double* scores, int* nperm, int* chosen) {
    return guarded([&] {
        // MetricConfig::validate (metrics.cpp:13-22)
        if (block < 1)
            fail(PARO_E_CONFIG, "block must be >= 1");
        if (!(eps > 0.0f))
            fail(PARO_E_CONFIG, "eps must be > 0");
        if (!(sigma > 0.0f && sigma <= 1.0f))
            fail(PARO_E_CONFIG, "sigma must be in (0,1]");
        if (!(alpha >= 0.0f && alpha <= 1.0f))
            fail(PARO_E_CONFIG, "alpha must be in [0,1]");
        if (count == 0)
            fail(PARO_E_INPUT, "select_permutation: empty calibration set");
        if (block > 256)
            fail(PARO_E_CONFIG, "device select_permutation supports block <= 256");
        Grid g = parse_grid_text(grid_text);
        const size_t n = g.tokens(), nf = n + dense_prefix;
        const uint32_t k = (uint32_t)((n + block - 1) / block);
        set_device(ctx);
        const cudaStream_t st = (cudaStream_t)stream;
        // candidate orders (enumerate_perms, reorder.cpp:74-91)
        std::string ident(g.labels, g.labels + g.ndim);
        std::string perm = ident;
        std::sort(perm.begin(), perm.end());
        std::vector<std::string> ords{ident};
        do {
            if (perm != ident)
                ords.push_back(perm);
        } while (std::next_permutation(perm.begin(), perm.end()));
        const size_t P = ords.size(), kk = (size_t)k * k;
        // every (order, map) pass is queued on the stream with one sync at the
        // end: K5a statistics -> per-block terms + sparse count on the device,
        // terms staged through pinned memory, summed on the host in block order
        const size_t slots = P * count;
        auto up8 = [](size_t x) { return (x + 7) & ~size_t(7); };
        const size_t off_inv = 0, off_sum = up8(P * n * 4), off_max = off_sum + kk * 8, off_cnt = off_max + up8(kk * 4),
                     off_terms = off_cnt + up8(kk * 4), off_sparse = off_terms + slots * kk * 8;
        const size_t dbytes = off_sparse + slots * 4;
        const size_t hbytes = P * n * 4 + slots * kk * 8 + slots * 4;
        char* scratch = nullptr;
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&scratch), dbytes, st), "select_permutation scratch");
        struct Free {
            char* d;
            cudaStream_t st;
            ~Free() { cudaFreeAsync(d, st); }
        } guard_free{scratch, st};
        char* host = ctx->pinned_scratch(hbytes);
        uint32_t* hinv = reinterpret_cast<uint32_t*>(host);
        double* hterms = reinterpret_cast<double*>(host + P * n * 4);
        uint32_t* hsparse = reinterpret_cast<uint32_t*>(host + P * n * 4 + slots * kk * 8);
        for (size_t p = 0; p < P; ++p) {
            const PermDesc pd = perm_desc(g, ords[p]);
            for (size_t i = 0; i < n; ++i)
                hinv[p * n + i] = paro::perm_src(pd, (uint32_t)i);
        }
        uint32_t* dinv = reinterpret_cast<uint32_t*>(scratch + off_inv);
        double* dsum = reinterpret_cast<double*>(scratch + off_sum);
        float* dmax = reinterpret_cast<float*>(scratch + off_max);
        uint32_t* dcnt = reinterpret_cast<uint32_t*>(scratch + off_cnt);
        double* dterms = reinterpret_cast<double*>(scratch + off_terms);
        uint32_t* dsparse = reinterpret_cast<uint32_t*>(scratch + off_sparse);
        cuda_check(cudaMemcpyAsync(dinv, hinv, P * n * 4, cudaMemcpyHostToDevice, st), "select_permutation");
        cuda_check(cudaMemsetAsync(dsparse, 0, slots * 4, st), "select_permutation");
        for (size_t p = 0; p < P; ++p)
            for (uint32_t c = 0; c < count; ++c) {
                const size_t sl = p * count + c;
                // strip_prefix (reorder.cpp:119-127): the image-token submap
                const float* sub = maps + (size_t)c * nf * nf + (size_t)dense_prefix * nf + dense_prefix;
                // the identity order needs no table (and K5a reads its contiguous blocks vectorised)
                const uint32_t* pinv = ords[p] == ident ? nullptr : dinv + p * n;
                cuda_check(paro::launch_perm_block_stats(sub, nf, (uint32_t)n, pinv, block, eps, dsum, dmax, dcnt, st),
                           "select_permutation");
                cuda_check(paro::launch_block_terms(dsum, dmax, dcnt, k, (uint32_t)n, block, sigma, dterms + sl * kk,
                                                    dsparse + sl, st),
                           "select_permutation");
            }
        cuda_check(cudaMemcpyAsync(hterms, dterms, slots * kk * 8, cudaMemcpyDeviceToHost, st), "select_permutation");
        cuda_check(cudaMemcpyAsync(hsparse, dsparse, slots * 4, cudaMemcpyDeviceToHost, st), "select_permutation");
        cuda_check(cudaStreamSynchronize(st), "select_permutation");
        std::vector<double> sparse_mean(P), quant_mean(P), nonsparse(P), quant(P);
        for (size_t p = 0; p < P; ++p) {
            double s_acc = 0.0, q_acc = 0.0;
            for (uint32_t c = 0; c < count; ++c) {
                const size_t sl = p * count + c;
                const double* t = hterms + sl * kk;
                double total = 0.0; // block order (bi, bj), as metrics.cpp
                for (size_t b = 0; b < kk; ++b)
                    total += t[b];
                s_acc += (double)hsparse[sl] / (double)kk;
                q_acc += total / (double)kk;
            }
            const double cnt = (double)count;
            sparse_mean[p] = s_acc / cnt;
            quant_mean[p] = q_acc / cnt;
            nonsparse[p] = 1.0 - sparse_mean[p];
            quant[p] = quant_mean[p];
        }
        // shares, combined score, first argmin (reorder.cpp:160-179)
        double s_total = 0.0, q_total = 0.0;
        for (size_t p = 0; p < P; ++p) {
            s_total += nonsparse[p];
            q_total += quant[p];
        }
        const double equal_share = 1.0 / (double)P;
        size_t best = 0;
        std::vector<double> comb(P);
        for (size_t p = 0; p < P; ++p) {
            const double ss = s_total > 0.0 ? nonsparse[p] / s_total : equal_share;
            const double qs = q_total > 0.0 ? quant[p] / q_total : equal_share;
            comb[p] = (double)alpha * ss + (1.0 - (double)alpha) * qs;
            if (comb[p] < comb[best])
                best = p;
            if (scores) {
                double* o = scores + p * 5;
                o[0] = sparse_mean[p];
                o[1] = quant_mean[p];
                o[2] = ss;
                o[3] = qs;
                o[4] = comb[p];
            }
            if (orders)
                std::memcpy(orders + p * g.ndim, ords[p].data(), g.ndim);
        }
        if (nperm)
            *nperm = (int)P;
        if (chosen)
            *chosen = (int)best;
    });
}

int paro_synth_randn(uint64_t seed, size_t count, float* out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        auto unit = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
        for (size_t i = 0; i < count; ++i) {
            const double u1 = 1.0 - unit();
            const double u2 = unit();
            out[i] = static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2));
        }
    });
}

int paro_ctx_create(int device, paro_ctx** out) {
    return guarded([&] {
        int n = 0;
        cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n)
            fail(PARO_E_CONFIG, "device " + std::to_string(device) + " out of range (" + std::to_string(n) + " visible)");
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10)
            fail(PARO_E_CUDA, std::string("device ") + prop.name + " is sm_" + std::to_string(prop.major) +
                                  std::to_string(prop.minor) + "; these kernels are built for sm_100a only");
        auto* c = new paro_ctx;
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        c->l2_bytes = (size_t)prop.l2CacheSize;
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || !fn) {
            delete c;
            fail(PARO_E_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
        }
        c->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        *out = c;
    });
}

int paro_ctx_destroy(paro_ctx* ctx) {
    return guarded([&] { delete ctx; });
}

int paro_ctx_num_sms(const paro_ctx* ctx, int* out) {
    return guarded([&] { *out = ctx->num_sms; });
}

int paro_device_count(int* out) {
    return guarded([&] {
        int n = 0;
        cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        *out = n;
    });
}

int paro_host_alloc(size_t bytes, void** out) {
    return guarded([&] { cuda_check(cudaHostAlloc(out, bytes, cudaHostAllocDefault), "cudaHostAlloc"); });
}
int paro_host_free(void* p) {
    return guarded([&] { cuda_check(cudaFreeHost(p), "cudaFreeHost"); });
}
int paro_device_alloc(size_t bytes, void** out) {
    return guarded([&] { cuda_check(cudaMalloc(out, bytes), "cudaMalloc"); });
}
int paro_device_free(void* p) {
    return guarded([&] { cuda_check(cudaFree(p), "cudaFree"); });
}
int paro_memcpy(void* dst, const void* src, size_t bytes, paro_stream_t stream) {
    return guarded([&] {
        cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream), "cudaMemcpyAsync");
    });
}
int paro_stream_sync(paro_stream_t stream) {
    return guarded([&] { cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "cudaStreamSynchronize"); });
}

int paro_apply_perm_rows_device(paro_ctx* ctx, paro_stream_t stream, const float* in, uint32_t rows, uint32_t cols,
                                const uint32_t* inverse, float* out) {
    return guarded([&] {
        set_device(ctx);
        if (rows == 0)
            return;
        cuda_check(paro::launch_apply_perm_rows(in, rows, cols, inverse, out, (cudaStream_t)stream), "apply_perm_rows");
    });
}

int paro_quantize_sym_device(paro_ctx* ctx, paro_stream_t stream, const float* in, uint32_t rows, uint32_t cols,
                             int bits, int8_t* codes, float* scales) {
    return guarded([&] {
        check_bits(bits);
        if (cols != 64 && cols != 128)
            fail(PARO_E_CONFIG, "device quantize supports 64 or 128 columns, got " + std::to_string(cols));
        check_aligned16(in, "input");
        check_aligned16(codes, "codes"); // 4-byte code stores: 16 is the documented contract
        set_device(ctx);
        if (rows == 0)
            return;
        cuda_check(paro::launch_quantize_sym(in, rows, cols, bits, codes, scales, (cudaStream_t)stream), "quantize");
    });
}

int paro_layer_create(paro_ctx* ctx, uint32_t heads, uint32_t head_dim, const char* grid_text, const char* orders,
                      paro_layer** out) {
    return paro_layer_create_prefix(ctx, heads, head_dim, grid_text, orders, 0, out);
}

int paro_layer_create_prefix(paro_ctx* ctx, uint32_t heads, uint32_t head_dim, const char* grid_text,
                             const char* orders, uint32_t dense_prefix, paro_layer** out) {
    return guarded([&] {
        if (!ctx)
            fail(PARO_E_CONFIG, "null context");
        if (head_dim != 64 && head_dim != 128)
            fail(PARO_E_CONFIG, "head dim must be 64 or 128 on the B200 path, got " + std::to_string(head_dim));
        if (heads == 0 || heads > 65535)
            fail(PARO_E_CONFIG, "heads must be in [1, 65535]");
        Grid g = parse_grid_text(grid_text);
        const size_t N = g.tokens() + dense_prefix; // text tokens first (PermPlan::with_prefix)
        if (N == 0 || N > (size_t)16383 * 64)
            fail(PARO_E_CONFIG, "token count " + std::to_string(N) + " out of range");
        set_device(ctx);
        auto* l = new paro_layer;
        l->ctx = ctx;
        l->grid = g;
        try {
            for (uint32_t h = 0; h < heads; ++h) {
                std::string ord = orders ? std::string(orders + (size_t)h * g.ndim, g.ndim)
                                         : std::string(g.labels, g.labels + g.ndim);
                l->perm_host.push_back(perm_desc(g, ord));
                l->perm_host.back().prefix = dense_prefix;
            }
            LayerDev& L = l->L;
            L.H = heads;
            L.N = (uint32_t)N;
            L.D = head_dim;
            L.G = head_dim / 64;
            L.kb = (L.N + 63) / 64;
            L.kb2 = (L.kb + 1) & ~1u;
            L.np = L.kb2 / 2;
            L.dp = dense_prefix;
            L.nd = (dense_prefix + 63) / 64;
            const size_t rows = (size_t)heads * L.kb2 * 64;
            if (dense_prefix) {
                L.init_m = dalloc<double>(rows);
                L.init_l = dalloc<float>(rows);
                L.init_acc = dalloc<float>(rows * head_dim);
                paro::k4_chunking(L.kb, L.nd, heads, L.k4_cb, L.k4_ch);
                const size_t parts = (size_t)heads * L.nd * 64 * L.k4_cb;
                L.part_m = dalloc<double>(parts);
                L.part_l = dalloc<float>(parts);
                L.part_acc = dalloc<float>(parts * head_dim);
                L.vsplit_hi = dalloc<uint16_t>(rows * head_dim);
                L.vsplit_lo = dalloc<uint16_t>(rows * head_dim);
                encode_vt_map(ctx, &l->tm_vh, L.vsplit_hi, head_dim, rows / 64 * head_dim);
                encode_vt_map(ctx, &l->tm_vl, L.vsplit_lo, head_dim, rows / 64 * head_dim);
            }
            L.perm = dalloc<PermDesc>(heads);
            L.q = dalloc<int8_t>(rows * head_dim);
            L.k = dalloc<int8_t>(rows * head_dim);
            L.v = dalloc<int8_t>(rows * head_dim);
            L.qsc = dalloc<float>((size_t)heads * L.kb2 * L.G);
            L.meta = dalloc<float>((size_t)heads * L.kb2 * paro::meta_stride(head_dim));
            L.items = dalloc<uint16_t>((size_t)heads * L.kb * L.kb);
            L.pairs = dalloc<uint32_t>((size_t)heads * L.np);
            L.pair_count = dalloc<uint32_t>((size_t)heads * L.np);
            L.qb_count = dalloc<uint32_t>((size_t)heads * L.kb2);
            L.order = dalloc<uint32_t>((size_t)heads * L.np);
            L.order_chunk = dalloc<uint32_t>((size_t)heads * L.np);
            set_chunks(L, default_heads_per_chunk(heads, N, head_dim), true);
            // L2 groups of the whole-layer work order: as many heads as keep their
            // K + V codes within half of L2 (c2: 27 of 48 heads, c5: 3 of 40);
            // PARO_L2_GROUP_HEADS overrides (0 = one global LPT order)
            {
                const size_t kv = (size_t)L.kb2 * 64 * head_dim * 2;
                size_t g = std::max<size_t>(1, (ctx->l2_bytes / 2) / std::max<size_t>(kv, 1));
                if (const char* e = getenv("PARO_L2_GROUP_HEADS"))
                    g = (size_t)atoi(e);
                L.l2_group = (uint32_t)std::min<size_t>(g, heads);
            }
            L.work_counter = dalloc<uint32_t>(1);
            l->v_pack = getenv("PARO_V_PACKED") && atoi(getenv("PARO_V_PACKED")) != 0;
            l->fwd = dalloc<uint32_t>((size_t)heads * N);
            l->inv = dalloc<uint32_t>((size_t)heads * N);
            cuda_check(cudaMemset(L.q, 0, rows * head_dim), "cudaMemset");
            cuda_check(cudaMemset(L.k, 0, rows * head_dim), "cudaMemset");
            cuda_check(cudaMemset(L.v, 0, rows * head_dim), "cudaMemset");
            cuda_check(cudaMemset(L.qb_count, 0, (size_t)heads * L.kb2 * 4), "cudaMemset");
            cuda_check(cudaMemcpy(L.perm, l->perm_host.data(), heads * sizeof(PermDesc), cudaMemcpyHostToDevice),
                       "cudaMemcpy perm");
            cuda_check(paro::launch_perm_tables(L.perm, heads, L.N, l->fwd, l->inv, 0), "perm tables");
            encode_codes_map(ctx, &l->tm_q, L.q, head_dim, rows, 64);
            encode_codes_map(ctx, &l->tm_q32, L.q, head_dim, rows, 32);
            encode_codes_map(ctx, &l->tm_k, L.k, head_dim, rows, 64);
            encode_codes_map(ctx, &l->tm_v, L.v, head_dim, rows, 64);
            encode_packed_map(ctx, &l->tm_vp, L.v, head_dim, rows, 64);
            cuda_check(cudaDeviceSynchronize(), "layer init");
        } catch (...) {
            free_layer(l);
            delete l;
            throw;
        }
        *out = l;
    });
}

int paro_layer_destroy(paro_layer* layer) {
    return guarded([&] {
        if (!layer)
            return;
        set_device(layer->ctx);
        free_layer(layer);
        delete layer;
    });
}

static void set_masks_impl(paro_layer* l, cudaStream_t st, const uint8_t* bits, bool host) {
    check_layer(l);
    set_device(l->ctx);
    clear_schedule(l); // a plain mask set ends any schedule
    const uint8_t* dbits = nullptr;
    const size_t bytes = (size_t)l->L.H * l->L.kb * l->L.kb;
    if (bits) {
        if (host) {
            if (!l->mask_dev)
                l->mask_dev = dalloc<uint8_t>(bytes);
            cuda_check(cudaMemcpyAsync(l->mask_dev, bits, bytes, cudaMemcpyHostToDevice, st), "mask upload");
            dbits = l->mask_dev;
        } else {
            dbits = bits;
        }
    }
    cuda_check(paro::launch_k2(l->L, dbits, st), "k2 launch");
    l->masks_set = true;
}

int paro_layer_set_masks(paro_layer* layer, paro_stream_t stream, const uint8_t* host_bits) {
    return guarded([&] { set_masks_impl(layer, (cudaStream_t)stream, host_bits, true); });
}

int paro_layer_set_masks_pmsk(paro_layer* layer, paro_stream_t stream, const uint8_t* const* blobs,
                              const size_t* sizes) {
    return guarded([&] {
        check_layer(layer);
        const LayerDev& L = layer->L;
        if (!blobs || !sizes)
            fail(PARO_E_CONFIG, "null PMSK blob list");
        const size_t kk = (size_t)L.kb * L.kb;
        std::vector<uint8_t> bits((size_t)L.H * kk);
        for (uint32_t h = 0; h < L.H; ++h) {
            uint32_t kr = 0, kc = 0, block = 0;
            decode_pmsk(blobs[h], sizes[h], &kr, &kc, &block, nullptr); // header + size checks
            if (block != 64)
                fail(PARO_E_CONFIG, "head " + std::to_string(h) + ": mask block " + std::to_string(block) +
                                        ", the B200 path runs block 64");
            if (kr != L.kb || kc != L.kb)
                fail(PARO_E_SHAPE, "head " + std::to_string(h) + ": mask grid " + std::to_string(kr) + "x" +
                                       std::to_string(kc) + " does not cover " + std::to_string(L.kb) + "x" +
                                       std::to_string(L.kb) + " blocks");
            decode_pmsk(blobs[h], sizes[h], &kr, &kc, &block, bits.data() + (size_t)h * kk);
        }
        set_masks_impl(layer, (cudaStream_t)stream, bits.data(), true);
    });
}

int paro_layer_set_rope(paro_layer* layer, paro_stream_t stream, const float* cos, const float* sin) {
    return guarded([&] {
        check_layer(layer);
        LayerDev& L = layer->L;
        if (!cos != !sin)
            fail(PARO_E_CONFIG, "rope: cos and sin must both be given or both be null");
        if (!cos) {
            L.rope_cos = L.rope_sin = nullptr;
            return;
        }
        const size_t elems = (size_t)(L.N - L.dp) * L.D;
        if (!layer->rope)
            layer->rope = dalloc<float>(2 * elems);
        const cudaStream_t st = (cudaStream_t)stream;
        // host (pageable or pinned) or device tables: the copy kind is inferred (UVA)
        cuda_check(cudaMemcpyAsync(layer->rope, cos, elems * 4, cudaMemcpyDefault, st), "rope cos copy");
        cuda_check(cudaMemcpyAsync(layer->rope + elems, sin, elems * 4, cudaMemcpyDefault, st), "rope sin copy");
        L.rope_cos = layer->rope;
        L.rope_sin = layer->rope + elems;
    });
}

int paro_layer_set_masks_device(paro_layer* layer, paro_stream_t stream, const uint8_t* device_bits) {
    return guarded([&] { set_masks_impl(layer, (cudaStream_t)stream, device_bits, false); });
}

int paro_layer_set_schedule(paro_layer* layer, paro_stream_t stream, const uint8_t* const* psch, const size_t* sizes,
                            uint32_t resident_lists) {
    return guarded([&] {
        check_layer(layer);
        set_device(layer->ctx);
        const LayerDev& L = layer->L;
        if (!psch || !sizes)
            fail(PARO_E_CONFIG, "null PSCH blob list");
        if (resident_lists != 0 && resident_lists != 2)
            fail(PARO_E_CONFIG, "resident_lists must be 0 (every entry) or 2 (double-buffered prefetch)");
        const size_t kk = (size_t)L.kb * L.kb;
        uint32_t T = 0;
        std::vector<uint8_t> bits; // [entries][H][kb][kb]
        std::vector<std::pair<const uint8_t*, size_t>> ent;
        for (uint32_t h = 0; h < L.H; ++h) {
            const uint32_t Th = parse_psch(psch[h], sizes[h], ent);
            if (h == 0) {
                if (Th == 0)
                    fail(PARO_E_CONFIG, "schedule covers no timestep");
                T = Th;
                bits.assign((size_t)(T / 2 + 1) * L.H * kk, 0);
            } else if (Th != T) {
                fail(PARO_E_SHAPE, "head " + std::to_string(h) + ": schedule covers " + std::to_string(Th) +
                                       " timesteps, head 0 covers " + std::to_string(T));
            }
            for (size_t e = 0; e < ent.size(); ++e) {
                uint32_t kr = 0, kc = 0, block = 0;
                decode_pmsk(ent[e].first, ent[e].second, &kr, &kc, &block, nullptr);
                if (block != 64)
                    fail(PARO_E_CONFIG, "head " + std::to_string(h) + ": mask block " + std::to_string(block) +
                                            ", the B200 path runs block 64");
                if (kr != L.kb || kc != L.kb)
                    fail(PARO_E_SHAPE, "head " + std::to_string(h) + ": mask grid " + std::to_string(kr) + "x" +
                                           std::to_string(kc) + " does not cover " + std::to_string(L.kb) + "x" +
                                           std::to_string(L.kb) + " blocks");
                decode_pmsk(ent[e].first, ent[e].second, &kr, &kc, &block, bits.data() + (e * L.H + h) * kk);
            }
        }
        clear_schedule(layer);
        layer->base = current_lists(layer);
        cudaStream_t st = (cudaStream_t)stream;
        const uint32_t E = T / 2 + 1;
        layer->sched_masks = dalloc<uint8_t>(bits.size());
        cuda_check(cudaMemcpyAsync(layer->sched_masks, bits.data(), bits.size(), cudaMemcpyHostToDevice, st),
                   "schedule upload");
        cuda_check(cudaStreamSynchronize(st), "schedule upload"); // `bits` is a local host buffer
        layer->sched_T = T;
        layer->sched_entries = E;
        layer->sched_resident = resident_lists;
        if (resident_lists == 0) { // every entry's kept lists built once
            for (uint32_t e = 0; e < E; ++e) {
                layer->sched_lists.push_back(alloc_lists(L));
                build_entry(layer, layer->sched_lists.back(), e, st);
            }
        } else {
            for (int i = 0; i < 2; ++i)
                layer->sched_lists.push_back(alloc_lists(L));
            cuda_check(cudaStreamCreateWithFlags(&layer->s_k2, cudaStreamNonBlocking), "stream create");
            cuda_check(cudaEventCreateWithFlags(&layer->ev_prefetch, cudaEventDisableTiming), "event create");
        }
        layer->sched_cur = -1;
        layer->masks_set = false; // until a timestep is selected
    });
}

int paro_layer_select_timestep(paro_layer* layer, paro_stream_t stream, uint32_t t) {
    return guarded([&] {
        check_layer(layer);
        if (!layer->sched_T)
            fail(PARO_E_CONFIG, "paro_layer_set_schedule must be called before selecting a timestep");
        set_device(layer->ctx);
        cudaStream_t st = (cudaStream_t)stream;
        const uint32_t e = schedule_entry(layer->sched_T, t);
        auto& lists = layer->sched_lists;
        int cur = -1;
        if (layer->sched_resident == 0) {
            cur = (int)e;
        } else {
            for (int i = 0; i < 2; ++i)
                if (lists[i].entry == (int)e)
                    cur = i;
            if (cur >= 0) { // prefetched (or current): order this stream after its K2
                cuda_check(cudaStreamWaitEvent(st, lists[cur].ready, 0), "stream wait");
            } else { // not prefetched (first call, or a jump): build it now on the caller's stream
                cur = layer->sched_cur == 0 ? 1 : 0;
                build_entry(layer, lists[cur], e, st);
            }
            // prefetch t+1's lists into the other buffer on the side stream, after the
            // work already queued here (the previous step still reads that buffer)
            if (t + 1 < layer->sched_T) {
                const uint32_t e1 = schedule_entry(layer->sched_T, t + 1);
                auto& other = lists[1 - cur];
                if (e1 != e && other.entry != (int)e1) {
                    cuda_check(cudaEventRecord(layer->ev_prefetch, st), "event record");
                    cuda_check(cudaStreamWaitEvent(layer->s_k2, layer->ev_prefetch, 0), "stream wait");
                    build_entry(layer, other, e1, layer->s_k2);
                }
            }
        }
        layer->sched_cur = cur;
        use_lists(layer, lists[cur]);
        layer->masks_set = true;
    });
}

int paro_layer_schedule_info(const paro_layer* layer, uint32_t* timesteps, uint32_t* entries, int* current_entry) {
    return guarded([&] {
        check_layer(layer);
        if (timesteps)
            *timesteps = layer->sched_T;
        if (entries)
            *entries = layer->sched_entries;
        if (current_entry)
            *current_entry = layer->sched_cur >= 0 ? layer->sched_lists[layer->sched_cur].entry : -1;
    });
}

int paro_layer_reorder_quantize(paro_layer* layer, paro_stream_t stream, const float* q, const float* k,
                                const float* v, int v_bits) {
    return guarded([&] {
        check_layer(layer);
        check_bits(v_bits);
        if (!q || !k || !v)
            fail(PARO_E_CONFIG, "null Q/K/V");
        check_aligned16(q, "Q");
        check_aligned16(k, "K");
        check_aligned16(v, "V");
        set_device(layer->ctx);
        layer->L.v_packed = v_bits == 4 && layer->v_pack;
        cuda_check(paro::launch_k1(layer->L, q, k, v, v_bits, 0, layer->L.H, (cudaStream_t)stream), "k1 launch");
        cuda_check(paro::launch_k4a(layer->L, v, 0, layer->L.H, (cudaStream_t)stream), "k4a launch");
        layer->last_v_bits = v_bits;
    });
}

int paro_layer_attention(paro_layer* layer, paro_stream_t stream, float scale, int pv_bits, float* out,
                         uint8_t* zeroed) {
    return guarded([&] {
        check_layer(layer);
        check_aligned16(out, "out");
        set_device(layer->ctx);
        run_attention(layer, (cudaStream_t)stream, scale, pv_bits, out, zeroed);
    });
}

int paro_layer_forward(paro_layer* layer, paro_stream_t stream, const float* q, const float* k, const float* v,
                       float scale, int pv_bits, float* out, uint8_t* zeroed) {
    return guarded([&] {
        check_layer(layer);
        check_bits(pv_bits);
        if (!layer->masks_set)
            fail(PARO_E_CONFIG, "paro_layer_set_masks must be called before forward");
        if (!q || !k || !v)
            fail(PARO_E_CONFIG, "null Q/K/V");
        check_aligned16(q, "Q");
        check_aligned16(k, "K");
        check_aligned16(v, "V");
        check_aligned16(out, "out");
        set_device(layer->ctx);
        cudaStream_t st = (cudaStream_t)stream;
        layer->L.v_packed = pv_bits == 4 && layer->v_pack;
        cuda_check(paro::launch_k1(layer->L, q, k, v, pv_bits, 0, layer->L.H, st), "k1 launch");
        cuda_check(paro::launch_k4a(layer->L, v, 0, layer->L.H, st), "k4a launch");
        layer->last_v_bits = pv_bits;
        run_attention(layer, st, scale, pv_bits, out, zeroed);
        layer->last_launches = 2;
    });
}

int paro_layer_set_v_packing(paro_layer* layer, int packed) {
    return guarded([&] {
        check_layer(layer);
        layer->v_pack = packed != 0;
    });
}

int paro_layer_set_pipeline_chunks(paro_layer* layer, paro_stream_t stream, uint32_t chunks) {
    return guarded([&] {
        check_layer(layer);
        if (chunks == 0)
            fail(PARO_E_CONFIG, "pipeline chunk count must be >= 1");
        set_device(layer->ctx);
        LayerDev& L = layer->L;
        const uint32_t c = std::min(std::min(chunks, L.H), paro::kMaxChunks);
        set_chunks(L, (L.H + c - 1) / c, false);
        if (layer->sched_T) { // re-sort every built schedule entry's per-chunk lists
            for (auto& x : layer->sched_lists) {
                if (x.entry < 0)
                    continue;
                LayerDev tmp = L;
                tmp.pairs = x.pairs;
                tmp.pair_count = x.pair_count;
                tmp.qb_count = x.qb_count;
                tmp.order = x.order;
                tmp.order_chunk = x.order_chunk;
                cuda_check(cudaStreamWaitEvent((cudaStream_t)stream, x.ready, 0), "stream wait");
                cuda_check(paro::launch_k2_order(tmp, (cudaStream_t)stream), "k2 order launch");
                cuda_check(cudaEventRecord(x.ready, (cudaStream_t)stream), "event record");
            }
        } else if (layer->masks_set) { // re-sort the per-chunk work lists for the new split
            cuda_check(paro::launch_k2_order(L, (cudaStream_t)stream), "k2 order launch");
        }
    });
}

// Host-buffer forward. Heads are split into the chunks of L.chunk_start; chunk c's Q/K/V
// upload (stream s_in), K1 + K3 (caller's stream) and output download
// (stream s_out) are event-chained so PCIe traffic in both directions
// overlaps the kernels of the neighbouring chunks. Returns when `out` (and
// `zeroed`) hold the result.
int paro_layer_forward_host(paro_layer* layer, paro_stream_t stream, const float* q, const float* k, const float* v,
                            float scale, int pv_bits, float* out, uint8_t* zeroed) {
    return guarded([&] {
        check_layer(layer);
        check_bits(pv_bits);
        if (!layer->masks_set)
            fail(PARO_E_CONFIG, "paro_layer_set_masks must be called before forward");
        if (!q || !k || !v || !out)
            fail(PARO_E_CONFIG, "null Q/K/V/out");
        set_device(layer->ctx);
        cudaStream_t st = (cudaStream_t)stream;
        const LayerDev& L = layer->L;
        const size_t head_elems = (size_t)L.N * L.D;
        const size_t elems = (size_t)L.H * head_elems;
        if (!layer->dq) {
            layer->dq = dalloc<float>(elems);
            layer->dk = dalloc<float>(elems);
            layer->dv = dalloc<float>(elems);
            layer->dout = dalloc<float>(elems);
            layer->dzero = dalloc<uint8_t>((size_t)L.H * L.N);
            cuda_check(cudaStreamCreateWithFlags(&layer->s_in, cudaStreamNonBlocking), "stream create");
            cuda_check(cudaStreamCreateWithFlags(&layer->s_out, cudaStreamNonBlocking), "stream create");
        }
        const uint32_t nchunks = L.nchunks;
        while (layer->ev.size() < 1 + 3 * (size_t)nchunks) {
            cudaEvent_t e;
            cuda_check(cudaEventCreateWithFlags(&e, getenv("PARO_E2E_TRACE") ? cudaEventDefault
                                                                             : cudaEventDisableTiming),
                       "event create");
            layer->ev.push_back(e);
        }
        cudaEvent_t* ev = layer->ev.data();
        // stream order: the uploads (s_in) and downloads (s_out) start after the work
        // already queued on the caller's stream -- it may still be writing the pinned
        // host inputs (an async D2H into q/k/v) or reading the staging buffers; K1/K3
        // of each chunk run on that stream
        cuda_check(cudaEventRecord(ev[0], st), "event record");
        cuda_check(cudaStreamWaitEvent(layer->s_in, ev[0], 0), "stream wait");
        cuda_check(cudaStreamWaitEvent(layer->s_out, ev[0], 0), "stream wait");
        layer->last_v_bits = pv_bits;
        layer->L.v_packed = pv_bits == 4 && layer->v_pack;
        for (uint32_t c = 0; c < nchunks; ++c) {
            const uint32_t h0 = L.chunk_start[c], hn = L.chunk_start[c + 1] - h0;
            const size_t off = (size_t)h0 * head_elems, bytes = (size_t)hn * head_elems * 4;
            cudaEvent_t e_in = ev[1 + 3 * c], e_k = ev[2 + 3 * c], e_out = ev[3 + 3 * c];
            cuda_check(cudaMemcpyAsync(layer->dq + off, q + off, bytes, cudaMemcpyHostToDevice, layer->s_in), "H2D q");
            cuda_check(cudaMemcpyAsync(layer->dk + off, k + off, bytes, cudaMemcpyHostToDevice, layer->s_in), "H2D k");
            cuda_check(cudaMemcpyAsync(layer->dv + off, v + off, bytes, cudaMemcpyHostToDevice, layer->s_in), "H2D v");
            cuda_check(cudaEventRecord(e_in, layer->s_in), "event record");
            cuda_check(cudaStreamWaitEvent(st, e_in, 0), "stream wait");
            cuda_check(paro::launch_k1(L, layer->dq, layer->dk, layer->dv, pv_bits, h0, hn, st), "k1 launch");
            cuda_check(paro::launch_k4a(L, layer->dv, h0, hn, st), "k4a launch");
            run_attention(layer, st, scale, pv_bits, layer->dout, zeroed ? layer->dzero : nullptr, h0, hn, true);
            cuda_check(cudaEventRecord(e_k, st), "event record");
            cuda_check(cudaStreamWaitEvent(layer->s_out, e_k, 0), "stream wait");
            cuda_check(cudaMemcpyAsync(out + off, layer->dout + off, bytes, cudaMemcpyDeviceToHost, layer->s_out),
                       "D2H out");
            if (zeroed)
                cuda_check(cudaMemcpyAsync(zeroed + (size_t)h0 * L.N, layer->dzero + (size_t)h0 * L.N,
                                           (size_t)hn * L.N, cudaMemcpyDeviceToHost, layer->s_out),
                           "D2H zeroed");
            cuda_check(cudaEventRecord(e_out, layer->s_out), "event record");
        }
        cuda_check(cudaStreamWaitEvent(st, ev[3 * nchunks], 0), "stream wait");
        cuda_check(cudaStreamSynchronize(st), "forward_host sync");
        if (getenv("PARO_E2E_TRACE")) { // per chunk: upload done / kernels done / download done (ms from start)
            cudaEvent_t* e = layer->ev.data();
            for (uint32_t c = 0; c < nchunks; ++c) {
                float a = 0, b = 0, d = 0;
                cudaEventElapsedTime(&a, e[0], e[1 + 3 * c]);
                cudaEventElapsedTime(&b, e[0], e[2 + 3 * c]);
                cudaEventElapsedTime(&d, e[0], e[3 + 3 * c]);
                fprintf(stderr, "[e2e] chunk %u: in %.3f  kern %.3f  out %.3f\n", c, a, b, d);
            }
        }
        layer->last_launches = 2 * (int)nchunks;
    });
}

int paro_layer_get_buffers(const paro_layer* layer, paro_layer_buffers* out) {
    return guarded([&] {
        check_layer(layer);
        const LayerDev& L = layer->L;
        out->heads = L.H;
        out->tokens = L.N;
        out->head_dim = L.D;
        out->kblocks = L.kb;
        out->kblocks_padded = L.kb2;
        out->groups = L.G;
        out->q_codes = L.q;
        out->k_codes = L.k;
        out->v_codes = L.v;
        out->q_scales = L.qsc;
        out->tile_meta = L.meta;
        out->inverse = layer->inv;
        out->forward = layer->fwd;
        out->v_bits = (uint32_t)layer->last_v_bits;
        out->v_packed = L.v_packed;
    });
}

int paro_layer_export_parq(paro_layer* layer, paro_stream_t stream, uint32_t head, int which, uint8_t* out,
                           size_t* size) {
    return guarded([&] {
        check_layer(layer);
        const LayerDev& L = layer->L;
        if (head >= L.H)
            fail(PARO_E_SHAPE, "head " + std::to_string(head) + " out of range (" + std::to_string(L.H) + " heads)");
        if (which < 0 || which > 2)
            fail(PARO_E_CONFIG, "which must be 0 (Q), 1 (K) or 2 (V)");
        if (layer->last_v_bits == 0)
            fail(PARO_E_CONFIG, "reorder_quantize must run before export");
        if (which == 2 && L.D != 64)
            fail(PARO_E_CONFIG, "V codes are grouped per key tile over all d columns; PARQ's per-block grouping "
                                "expresses that only at d = 64");
        set_device(layer->ctx);
        const cudaStream_t st = (cudaStream_t)stream;
        const size_t rows = L.N, d = L.D;
        std::vector<int8_t> c8(rows * d);
        const bool nib = which == 2 && L.v_packed;
        const int8_t* src = (which == 0 ? L.q : which == 1 ? L.k : L.v) + (size_t)head * L.kb2 * 64 * (nib ? d / 2 : d);
        cuda_check(cudaMemcpyAsync(c8.data(), src, nib ? rows * d / 2 : rows * d, cudaMemcpyDeviceToHost, st),
                   "export codes");
        std::vector<float> meta((size_t)L.kb * paro::meta_stride(L.D)), qs((size_t)L.kb * L.G);
        cuda_check(cudaMemcpyAsync(meta.data(), L.meta + (size_t)head * L.kb2 * paro::meta_stride(L.D),
                                   meta.size() * 4, cudaMemcpyDeviceToHost, st),
                   "export scales");
        cuda_check(cudaMemcpyAsync(qs.data(), L.qsc + (size_t)head * L.kb2 * L.G, qs.size() * 4,
                                   cudaMemcpyDeviceToHost, st),
                   "export scales");
        cuda_check(cudaStreamSynchronize(st), "export");
        if (nib) // two's-complement nibbles, low first (the K1 layout) -> one code per element
            for (size_t i = rows * d; i-- > 0;) {
                const uint8_t byte = (uint8_t)c8[i / 2];
                const int v = (i & 1) ? (byte >> 4) : (byte & 15);
                c8[i] = (int8_t)(v > 7 ? v - 16 : v);
            }
        std::vector<int32_t> codes(c8.begin(), c8.end());
        // group order: row blocks x column blocks, row-major (quant.cpp:45-56)
        std::vector<float> scales;
        for (uint32_t b = 0; b < L.kb; ++b) {
            if (which == 2)
                scales.push_back(meta[(size_t)b * paro::meta_stride(L.D) + 2]);
            else
                for (uint32_t g = 0; g < L.G; ++g)
                    scales.push_back(which == 0 ? qs[(size_t)b * L.G + g] : meta[(size_t)b * paro::meta_stride(L.D) + g]);
        }
        const unsigned bits = which == 2 ? (unsigned)layer->last_v_bits : 8u;
        emit(parq_bytes(bits, 1, 0, 64, (uint32_t)rows, (uint32_t)d, codes.data(), scales.data(), scales.size(),
                        nullptr),
             out, size);
    });
}

int paro_layer_mask_stats(paro_layer* layer, uint32_t* kept_per_qblock, uint64_t* total_kept) {
    return guarded([&] {
        check_layer(layer);
        if (!layer->masks_set)
            fail(PARO_E_CONFIG, "masks not set");
        set_device(layer->ctx);
        const LayerDev& L = layer->L;
        std::vector<uint32_t> buf((size_t)L.H * L.kb2);
        cuda_check(cudaMemcpy(buf.data(), L.qb_count, buf.size() * 4, cudaMemcpyDeviceToHost), "D2H qb_count");
        uint64_t tot = 0;
        for (uint32_t h = 0; h < L.H; ++h)
            for (uint32_t b = 0; b < L.kb; ++b) {
                const uint32_t c = buf[(size_t)h * L.kb2 + b];
                tot += c;
                if (kept_per_qblock)
                    kept_per_qblock[(size_t)h * L.kb + b] = c;
            }
        if (total_kept)
            *total_kept = tot;
    });
}

int paro_layer_debug_qk(paro_layer* layer, paro_stream_t stream, uint32_t n_tiles, const uint32_t* tiles, int32_t* S) {
    return guarded([&] {
        check_layer(layer);
        set_device(layer->ctx);
        cuda_check(paro::launch_debug_qk(layer->L, layer->tm_q, layer->tm_q32, layer->tm_k, n_tiles, tiles, S,
                                         (cudaStream_t)stream),
                   "debug_qk launch");
    });
}

int paro_debug_k1_quant_proof(paro_ctx* ctx, uint32_t bits_begin, uint64_t bits_count, uint32_t nx, uint32_t seed,
                              uint64_t* mismatches, uint32_t* first) {
    return guarded([&] {
        if (!ctx || !mismatches)
            fail(PARO_E_CONFIG, "null argument");
        if ((uint64_t)bits_begin + bits_count > 0x7f800000ull)
            fail(PARO_E_CONFIG, "amax bit patterns must be finite (< 0x7f800000)");
        set_device(ctx);
        unsigned long long* dbad = dalloc<unsigned long long>(1);
        uint32_t* dfirst = dalloc<uint32_t>(5);
        struct Free {
            void* p[2];
            ~Free() {
                for (void* x : p)
                    cudaFree(x);
            }
        } guard{{dbad, dfirst}};
        cuda_check(cudaMemset(dbad, 0, 8), "memset");
        cuda_check(cudaMemset(dfirst, 0, 20), "memset");
        for (uint64_t off = 0; off < bits_count; off += 1ull << 30) {
            const uint32_t n = (uint32_t)std::min<uint64_t>(1ull << 30, bits_count - off);
            cuda_check(paro::launch_k1_quant_proof(bits_begin + (uint32_t)off, n, nx, seed, dbad, dfirst, ctx->num_sms,
                                                   nullptr),
                       "k1 quant proof");
        }
        cuda_check(cudaDeviceSynchronize(), "k1 quant proof sync");
        unsigned long long h = 0;
        cuda_check(cudaMemcpy(&h, dbad, 8, cudaMemcpyDeviceToHost), "D2H");
        *mismatches = h;
        if (first)
            cuda_check(cudaMemcpy(first, dfirst, 20, cudaMemcpyDeviceToHost), "D2H");
    });
}

int paro_layer_debug_pdump(paro_layer* layer, paro_stream_t stream, float scale, int pv_bits, uint32_t n_targets,
                           const uint32_t* targets, uint8_t* codes, float* meta) {
    return guarded([&] {
        check_layer(layer);
        set_device(layer->ctx);
        const LayerDev& L = layer->L;
        if (n_targets == 0)
            return;
        if (!targets || !codes || !meta)
            fail(PARO_E_CONFIG, "null pdump argument");
        std::vector<int32_t> slot((size_t)L.H * L.kb2, -1);
        for (uint32_t i = 0; i < n_targets; ++i) {
            const uint32_t h = targets[2 * i], qb = targets[2 * i + 1];
            if (h >= L.H || qb >= L.kb)
                fail(PARO_E_INPUT, "pdump target (" + std::to_string(h) + ", " + std::to_string(qb) + ") out of range");
            if (slot[(size_t)h * L.kb2 + qb] >= 0)
                fail(PARO_E_INPUT, "pdump target listed twice");
            slot[(size_t)h * L.kb2 + qb] = (int32_t)i;
        }
        cudaStream_t st = (cudaStream_t)stream;
        const size_t ncodes = (size_t)n_targets * L.kb * 64 * 64, nmeta = (size_t)n_targets * L.kb * 4;
        int32_t* dslot = dalloc<int32_t>(slot.size());
        uint8_t* dcodes = dalloc<uint8_t>(ncodes);
        float* dmeta = dalloc<float>(nmeta);
        float* dout = dalloc<float>((size_t)L.H * L.N * L.D);
        struct Free {
            void* p[4];
            ~Free() {
                for (void* x : p)
                    cudaFree(x);
            }
        } guard{{dslot, dcodes, dmeta, dout}};
        cuda_check(cudaMemcpyAsync(dslot, slot.data(), slot.size() * 4, cudaMemcpyHostToDevice, st), "pdump H2D");
        cuda_check(cudaMemsetAsync(dcodes, 0, ncodes, st), "pdump memset");
        cuda_check(cudaMemsetAsync(dmeta, 0, nmeta * 4, st), "pdump memset");
        const paro::K3Dump dm{dslot, dcodes, dmeta, L.kb};
        run_attention(layer, st, scale, pv_bits, dout, nullptr, 0, ~0u, false, &dm);
        cuda_check(cudaMemcpyAsync(codes, dcodes, ncodes, cudaMemcpyDeviceToHost, st), "pdump D2H");
        cuda_check(cudaMemcpyAsync(meta, dmeta, nmeta * 4, cudaMemcpyDeviceToHost, st), "pdump D2H");
        cuda_check(cudaStreamSynchronize(st), "pdump sync");
    });
}

int paro_layer_last_launches(const paro_layer* layer, int* kernels) {
    return guarded([&] { *kernels = layer->last_launches; });
}

} // extern "C"
