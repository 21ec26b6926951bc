// paro_b200.hpp -- header-only C++ adapter: the reference's hot-path entry
// points (proj/include/paro/{reorder,quant,mask,attention}.hpp) served by the
// B200 library through its C ABI (include/paro_b200.h).
//
// Include it AFTER the reference headers; it speaks the reference's own types
// (paro::Matrix, paro::PermPlan, paro::BlockMask, paro::QuantConfig,
// paro::AttnInputs/AttnResult) and throws the reference's exception classes
// (paro::ConfigError / ShapeError / InputError / FormatError / IoError /
// InvariantError, error.hpp:11-40), so a caller switches by namespace:
//
//     #include "paro/attention.hpp"
//     #include "paro_b200.hpp"
//     ...
//     paro::AttnResult r = paro_b200::quantized_blocked_attention(pin, &mask, qcfg);
//
// CUDA runtime failures (no reference counterpart) throw paro_b200::CudaError,
// an InvariantError (exit code 4). There is no CPU fallback.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "paro_b200.h"

namespace paro_b200 {

struct CudaError : paro::InvariantError {
    explicit CudaError(const std::string& w) : paro::InvariantError(w) {}
};

// status -> the reference exception class (tens digit = exit code)
inline void check(int status) {
    if (status == PARO_OK)
        return;
    const std::string msg = paro_last_error();
    switch (status) {
    case PARO_E_CONFIG: throw paro::ConfigError(msg);
    case PARO_E_SHAPE: throw paro::ShapeError(msg);
    case PARO_E_INPUT: throw paro::InputError(msg);
    case PARO_E_FORMAT: throw paro::FormatError(msg);
    case PARO_E_IO: throw paro::IoError(msg);
    case PARO_E_INVARIANT: throw paro::InvariantError(msg);
    default: throw CudaError(msg);
    }
}

// One context per device, created lazily (the reference API has no handles).
inline paro_ctx* context(int device = 0) {
    struct Holder {
        paro_ctx* ctx = nullptr;
        ~Holder() {
            if (ctx)
                paro_ctx_destroy(ctx);
        }
    };
    static thread_local Holder h;
    if (!h.ctx)
        check(paro_ctx_create(device, &h.ctx));
    return h.ctx;
}

// make_perm (reorder.hpp:32, reorder.cpp:49-72)
inline paro::PermPlan make_perm(const paro::TokenGrid& grid, const std::string& order) {
    char labels[3];
    uint32_t ext[3];
    for (size_t a = 0; a < grid.ndim() && a < 3; ++a) {
        labels[a] = grid.axes[a].label;
        ext[a] = grid.axes[a].extent;
    }
    paro::PermPlan p;
    p.order = order;
    p.forward.resize(grid.token_count());
    p.inverse.resize(grid.token_count());
    check(paro_make_perm((int)grid.ndim(), labels, ext, order.c_str(), p.forward.data(), p.inverse.data()));
    return p;
}

// deserialize_mask (mask.hpp:74, mask.cpp:217-244)
inline paro::BlockMask deserialize_mask(const uint8_t* data, size_t size, size_t* consumed = nullptr) {
    uint32_t kr = 0, kc = 0, b = 0;
    check(paro_deserialize_mask(data, size, &kr, &kc, &b, nullptr, nullptr));
    paro::BlockMask m(kr, kc, b, false);
    check(paro_deserialize_mask(data, size, &kr, &kc, &b, m.bits.data(), consumed));
    return m;
}

namespace detail {
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { check(paro_device_alloc(bytes ? bytes : 1, &p)); }
    ~DevBuf() { paro_device_free(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};
} // namespace detail

// apply_perm_rows (reorder.hpp:39) on the GPU
inline paro::Matrix apply_perm_rows(const paro::Matrix& m, const paro::PermPlan& plan) {
    if (m.rows != plan.forward.size())
        throw paro::ShapeError("apply_perm_rows: matrix has " + std::to_string(m.rows) + " rows, plan covers " +
                               std::to_string(plan.forward.size()));
    paro_ctx* ctx = context();
    detail::DevBuf din(m.data.size() * 4), dout(m.data.size() * 4), dinv(plan.inverse.size() * 4);
    check(paro_memcpy(din.p, m.data.data(), m.data.size() * 4, nullptr));
    check(paro_memcpy(dinv.p, plan.inverse.data(), plan.inverse.size() * 4, nullptr));
    check(paro_apply_perm_rows_device(ctx, nullptr, static_cast<const float*>(din.p), (uint32_t)m.rows,
                                      (uint32_t)m.cols, static_cast<const uint32_t*>(dinv.p),
                                      static_cast<float*>(dout.p)));
    paro::Matrix out(m.rows, m.cols);
    check(paro_memcpy(out.data.data(), dout.p, out.data.size() * 4, nullptr));
    check(paro_stream_sync(nullptr));
    return out;
}

// quantize (quant.hpp:49) for the hot path's Q/K configuration
// {4|8 bits, Symmetric, PerBlock, block 64}, cols 64 or 128.
inline paro::QuantBlockTensor quantize(const paro::Matrix& m, const paro::QuantConfig& cfg) {
    cfg.validate();
    if (cfg.mode != paro::QuantMode::Symmetric || cfg.grouping != paro::QuantGrouping::PerBlock || cfg.block != 64)
        throw paro::ConfigError("the B200 quantizer serves {Symmetric, PerBlock, 64} (the Q/K configuration)");
    paro_ctx* ctx = context();
    const size_t groups = ((m.rows + 63) / 64) * ((m.cols + 63) / 64);
    detail::DevBuf din(m.data.size() * 4), dcodes(m.data.size()), dscales(groups * 4);
    check(paro_memcpy(din.p, m.data.data(), m.data.size() * 4, nullptr));
    check(paro_quantize_sym_device(ctx, nullptr, static_cast<const float*>(din.p), (uint32_t)m.rows,
                                   (uint32_t)m.cols, (int)cfg.bits, static_cast<int8_t*>(dcodes.p),
                                   static_cast<float*>(dscales.p)));
    std::vector<int8_t> codes(m.data.size());
    paro::QuantBlockTensor q;
    q.rows = m.rows;
    q.cols = m.cols;
    q.config = cfg;
    q.scales.resize(groups);
    check(paro_memcpy(codes.data(), dcodes.p, codes.size(), nullptr));
    check(paro_memcpy(q.scales.data(), dscales.p, groups * 4, nullptr));
    check(paro_stream_sync(nullptr));
    q.codes.assign(codes.begin(), codes.end());
    return q;
}

// quantized_blocked_attention (attention.hpp:52) with the INT8-QK stage, one
// head on the GPU. The tile edge is mask->block, else qcfg.block
// (attention.cpp:266-269); the B200 path serves block 64 and any dense_prefix
// below the token count (identity grid after the prefix, K4 + K3).
inline paro::AttnResult quantized_blocked_attention(const paro::AttnInputs& in, const paro::BlockMask* mask,
                                                    const paro::QuantConfig& qcfg) {
    in.validate();
    qcfg.validate();
    const size_t block = mask ? mask->block : qcfg.block;
    if (block != 64)
        throw paro::ConfigError("the B200 path runs block 64, got " + std::to_string(block));
    const size_t n = in.tokens(), d = in.head_dim(), kb = (n + 63) / 64, dp = in.dense_prefix;
    if (n > 0 && dp >= n)
        throw paro::ConfigError("dense_prefix covering every token is not served by the B200 path");
    if (mask && (mask->k_rows != kb || mask->k_cols != kb))
        throw paro::ShapeError("mask grid " + std::to_string(mask->k_rows) + "x" + std::to_string(mask->k_cols) +
                               " does not cover " + std::to_string(kb) + "x" + std::to_string(kb) + " blocks");
    paro_ctx* ctx = context();
    const std::string grid = "H:1,W:" + std::to_string(n - dp); // identity token order after the prefix
    paro_layer* layer = nullptr;
    check(paro_layer_create_prefix(ctx, 1, (uint32_t)d, grid.c_str(), nullptr, (uint32_t)dp, &layer));
    std::unique_ptr<paro_layer, int (*)(paro_layer*)> guard(layer, paro_layer_destroy);
    check(paro_layer_set_masks(layer, nullptr, mask ? mask->bits.data() : nullptr));
    paro::AttnResult res;
    res.output = paro::Matrix(n, d);
    std::vector<uint8_t> zeroed(n);
    check(paro_layer_forward_host(layer, nullptr, in.q.data.data(), in.k.data.data(), in.v.data.data(), in.scale,
                                  (int)qcfg.bits, res.output.data.data(), zeroed.data()));
    for (size_t i = 0; i < n; ++i)
        if (zeroed[i])
            res.zeroed_rows.push_back((uint32_t)i);
    return res;
}

} // namespace paro_b200
