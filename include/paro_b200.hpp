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

#include <algorithm>
#include <cstdint>
#include <fstream>
#include <iterator>
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

// load_plan_file (reorder.hpp:74, reorder.cpp:193-216)
inline std::vector<std::pair<std::uint32_t, std::string>> load_plan_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f)
        throw paro::IoError("cannot open '" + path + "' for reading");
    const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    uint32_t n = 0;
    size_t bytes = 0;
    check(paro_parse_plan(text.data(), text.size(), path.c_str(), &n, nullptr, nullptr, &bytes));
    std::vector<uint32_t> heads(n ? n : 1);
    std::vector<char> orders(bytes ? bytes : 1);
    check(paro_parse_plan(text.data(), text.size(), path.c_str(), &n, heads.data(), orders.data(), &bytes));
    std::vector<std::pair<std::uint32_t, std::string>> out;
    for (size_t i = 0, o = 0; i < n; ++i) {
        out.emplace_back(heads[i], std::string(orders.data() + o));
        o += out.back().second.size() + 1;
    }
    return out;
}

// plan_for_head (tools/main.cpp:118-126): identity without a plan file, the head's
// entry otherwise (InputError when the plan does not name the head)
inline paro::PermPlan plan_for_head(const std::string& plan_path, const paro::TokenGrid& grid, std::uint32_t head) {
    std::string text;
    if (!plan_path.empty()) {
        std::ifstream f(plan_path, std::ios::binary);
        if (!f)
            throw paro::IoError("cannot open '" + plan_path + "' for reading");
        text.assign((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    }
    std::string gt;
    for (const auto& a : grid.axes)
        gt += (gt.empty() ? "" : ",") + std::string(1, a.label) + ":" + std::to_string(a.extent);
    std::string order(grid.ndim(), '\0');
    check(paro_plan_for_heads(plan_path.empty() ? nullptr : text.data(), text.size(), plan_path.c_str(), gt.c_str(), 1,
                              &head, order.data()));
    return paro_b200::make_perm(grid, order);
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

// cmd_run's per-head chain (tools/main.cpp:276-305) for a whole layer of H
// heads in one call: per-head orders (PermPlan::with_prefix when dense_prefix >
// 0), per-head masks, Q/K/V per head in original token order, outputs and
// zeroed rows per head -- the reference's types in and out, the B200 layer
// (K1, K2, K3 and, with a prefix, K4) underneath.
class Layer {
public:
    Layer(const paro::TokenGrid& grid, size_t heads, size_t head_dim, const std::vector<std::string>& orders,
          size_t dense_prefix = 0)
        : heads_(heads), head_dim_(head_dim), tokens_(grid.token_count() + dense_prefix), prefix_(dense_prefix) {
        if (orders.size() != heads)
            throw paro::ShapeError(std::to_string(orders.size()) + " orders for " + std::to_string(heads) +
                                   " heads");
        std::string labels, ords;
        for (const auto& a : grid.axes)
            labels += a.label;
        std::string text;
        for (const auto& a : grid.axes)
            text += (text.empty() ? "" : ",") + std::string(1, a.label) + ":" + std::to_string(a.extent);
        for (const auto& o : orders) {
            if (o.size() != labels.size())
                throw paro::ConfigError("order '" + o + "' does not name the grid's " + std::to_string(labels.size()) +
                                        " axes");
            ords += o;
        }
        check(paro_layer_create_prefix(context(), (uint32_t)heads, (uint32_t)head_dim, text.c_str(), ords.c_str(),
                                       (uint32_t)dense_prefix, &layer_));
    }
    Layer(const Layer&) = delete;
    Layer& operator=(const Layer&) = delete;
    ~Layer() {
        if (layer_)
            paro_layer_destroy(layer_);
    }
    // one k x k mask per head (block 64), the grid over the permuted tokens
    void set_masks(const std::vector<paro::BlockMask>& masks) {
        if (masks.size() != heads_)
            throw paro::ShapeError(std::to_string(masks.size()) + " masks for " + std::to_string(heads_) + " heads");
        const size_t kb = (tokens_ + 63) / 64;
        std::vector<uint8_t> bits;
        bits.reserve(heads_ * kb * kb);
        for (const auto& m : masks) {
            if (m.block != 64)
                throw paro::ConfigError("the B200 path runs block 64, got " + std::to_string(m.block));
            if (m.k_rows != kb || m.k_cols != kb)
                throw paro::ShapeError("mask grid " + std::to_string(m.k_rows) + "x" + std::to_string(m.k_cols) +
                                       " does not cover " + std::to_string(kb) + "x" + std::to_string(kb) + " blocks");
            bits.insert(bits.end(), m.bits.begin(), m.bits.end());
        }
        check(paro_layer_set_masks(layer_, nullptr, bits.data()));
    }
    // rotary embedding fused into the reorder+quantize pass (paro_layer_set_rope): cos / sin are
    // [grid tokens x d] per original grid token (the text prefix is not rotated); empty = off
    void set_rope(const paro::Matrix& cos, const paro::Matrix& sin) {
        if (cos.data.empty() && sin.data.empty()) {
            check(paro_layer_set_rope(layer_, nullptr, nullptr, nullptr));
            return;
        }
        const size_t rows = tokens_ - prefix_;
        if (cos.rows != rows || cos.cols != head_dim_ || !cos.same_shape(sin))
            throw paro::ShapeError("rope tables must be " + std::to_string(rows) + "x" + std::to_string(head_dim_));
        check(paro_layer_set_rope(layer_, nullptr, cos.data.data(), sin.data.data()));
        check(paro_stream_sync(nullptr));
    }
    // all heads' attention (scale 0 -> 1/sqrt(d)); pv_bits 8 or 4
    std::vector<paro::AttnResult> forward(const std::vector<paro::Matrix>& q, const std::vector<paro::Matrix>& k,
                                          const std::vector<paro::Matrix>& v, float scale, unsigned pv_bits) {
        const size_t per = tokens_ * head_dim_;
        if (q.size() != heads_ || k.size() != heads_ || v.size() != heads_)
            throw paro::ShapeError("Q/K/V need one matrix per head");
        std::vector<float> hq(heads_ * per), hk(heads_ * per), hv(heads_ * per), ho(heads_ * per);
        std::vector<uint8_t> hz(heads_ * tokens_);
        for (size_t h = 0; h < heads_; ++h) {
            for (const paro::Matrix* m : {&q[h], &k[h], &v[h]})
                if (m->rows != tokens_ || m->cols != head_dim_)
                    throw paro::ShapeError("head " + std::to_string(h) + ": expected " + std::to_string(tokens_) +
                                           "x" + std::to_string(head_dim_) + ", got " + std::to_string(m->rows) +
                                           "x" + std::to_string(m->cols));
            std::copy(q[h].data.begin(), q[h].data.end(), hq.begin() + h * per);
            std::copy(k[h].data.begin(), k[h].data.end(), hk.begin() + h * per);
            std::copy(v[h].data.begin(), v[h].data.end(), hv.begin() + h * per);
        }
        check(paro_layer_forward_host(layer_, nullptr, hq.data(), hk.data(), hv.data(), scale, (int)pv_bits,
                                      ho.data(), hz.data()));
        std::vector<paro::AttnResult> res(heads_);
        for (size_t h = 0; h < heads_; ++h) {
            res[h].output = paro::Matrix(tokens_, head_dim_);
            std::copy(ho.begin() + h * per, ho.begin() + (h + 1) * per, res[h].output.data.begin());
            for (size_t i = 0; i < tokens_; ++i)
                if (hz[h * tokens_ + i])
                    res[h].zeroed_rows.push_back((uint32_t)i);
        }
        return res;
    }
    size_t tokens() const { return tokens_; }

private:
    size_t heads_, head_dim_, tokens_, prefix_;
    paro_layer* layer_ = nullptr;
};

} // namespace paro_b200
