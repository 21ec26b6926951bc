// ref_shim.cpp -- ORACLE (test infrastructure only).
//
// extern "C" wrappers over the UNMODIFIED reference library (paro_core),
// compiled from the reference's own sources where they lie under
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libparo_ref.so.
// Used by tests/ to pin the C restatement (oracle/paro_oracle.c) and to
// generate tests/golden/ fixtures, and by bench.py's reference arm /
// cpu_baseline leg to time the reference's own CPU path. Nothing in the
// product links this.
//
// Error convention: paro::Error's exit code (proj/include/paro/error.hpp:14-40)
// is returned; 0 = ok; the message is available from ref_last_error().

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "oracles.hpp" // reference tests/oracles.hpp (random_matrix, test_value)
#include "paro/attention.hpp"
#include "paro/error.hpp"
#include "paro/kernels.hpp"
#include "paro/mask.hpp"
#include "paro/metrics.hpp"
#include "paro/quant.hpp"
#include "paro/reorder.hpp"
#include "paro/synth.hpp"
#include "paro/tensor.hpp"
#include "paro/tensor_io.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const paro::Error& e) {
        g_err = e.what();
        return e.exit_code();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

paro::TokenGrid grid_from(int ndim, const char* labels, const uint32_t* extents) {
    std::vector<paro::GridAxis> axes;
    for (int a = 0; a < ndim; ++a)
        axes.push_back({labels[a], extents[a]});
    return paro::TokenGrid(axes);
}

paro::Matrix mat(const float* p, size_t r, size_t c) { return paro::Matrix(r, c, std::vector<float>(p, p + r * c)); }

void export_result(const paro::AttnResult& res, float* out, uint32_t* zeroed, size_t* nzeroed) {
    std::memcpy(out, res.output.data.data(), res.output.data.size() * sizeof(float));
    if (nzeroed)
        *nzeroed = res.zeroed_rows.size();
    if (zeroed)
        std::copy(res.zeroed_rows.begin(), res.zeroed_rows.end(), zeroed);
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// PARO_KERNELS equivalent (kernels.cpp:41-63); call before spawning threads.
int ref_select_kernels(const char* impl) {
    return guarded([&] { paro::kernels::select(paro::kernels::parse_impl(impl)); });
}

const char* ref_active_kernels() { return paro::kernels::active().name; }

int ref_parse_grid(const char* text, int* ndim, char* labels, uint32_t* extents) {
    return guarded([&] {
        paro::TokenGrid g = paro::parse_grid(text);
        *ndim = (int)g.ndim();
        for (size_t a = 0; a < g.ndim(); ++a) {
            labels[a] = g.axes[a].label;
            extents[a] = g.axes[a].extent;
        }
    });
}

int ref_make_perm(int ndim, const char* labels, const uint32_t* extents, const char* order, uint32_t* forward,
                  uint32_t* inverse) {
    return guarded([&] {
        paro::PermPlan p = paro::make_perm(grid_from(ndim, labels, extents), order);
        std::copy(p.forward.begin(), p.forward.end(), forward);
        std::copy(p.inverse.begin(), p.inverse.end(), inverse);
    });
}

// orders: ndim! strings of ndim chars, concatenated (identity first, reorder.cpp:74-91)
int ref_enumerate_perms(int ndim, const char* labels, const uint32_t* extents, char* orders, int* count) {
    return guarded([&] {
        auto plans = paro::enumerate_perms(grid_from(ndim, labels, extents));
        *count = (int)plans.size();
        for (size_t i = 0; i < plans.size(); ++i)
            std::memcpy(orders + i * ndim, plans[i].order.data(), ndim);
    });
}

int ref_apply_perm_rows(const float* m, size_t rows, size_t cols, const uint32_t* forward, const uint32_t* inverse,
                        size_t plan_n, float* out) {
    return guarded([&] {
        paro::PermPlan p;
        p.forward.assign(forward, forward + plan_n);
        p.inverse.assign(inverse, inverse + plan_n);
        paro::Matrix r = paro::apply_perm_rows(mat(m, rows, cols), p);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    });
}

int ref_quantize(const float* m, size_t rows, size_t cols, unsigned bits, int mode, int grouping, size_t block,
                 int32_t* codes, float* scales, float* offsets, size_t* ngroups) {
    return guarded([&] {
        paro::QuantConfig cfg{bits, static_cast<paro::QuantMode>(mode), static_cast<paro::QuantGrouping>(grouping),
                              block};
        paro::QuantBlockTensor q = paro::quantize(mat(m, rows, cols), cfg);
        std::copy(q.codes.begin(), q.codes.end(), codes);
        std::copy(q.scales.begin(), q.scales.end(), scales);
        if (offsets)
            std::copy(q.offsets.begin(), q.offsets.end(), offsets);
        *ngroups = q.scales.size();
    });
}

// PAT1 / PARQ files through the reference's own writers / readers (tensor_io.cpp, quant.cpp:219-326)
int ref_save_tensor(const uint32_t* shape, size_t ndim, const float* values, const char* path) {
    return guarded([&] {
        paro::TensorData t;
        t.shape.assign(shape, shape + ndim);
        t.values.assign(values, values + t.element_count());
        paro::save_tensor(t, path);
    });
}

int ref_load_tensor(const char* path, uint32_t* ndim, uint32_t* shape, float* values) {
    return guarded([&] {
        paro::TensorData t = paro::load_tensor(path);
        *ndim = (uint32_t)t.shape.size();
        std::copy(t.shape.begin(), t.shape.end(), shape);
        if (values)
            std::copy(t.values.begin(), t.values.end(), values);
    });
}

int ref_save_quant_codes(unsigned bits, int mode, int grouping, size_t block, size_t rows, size_t cols,
                         const int32_t* codes, const float* scales, const float* offsets, const char* path) {
    return guarded([&] {
        paro::QuantBlockTensor q;
        q.rows = rows;
        q.cols = cols;
        q.config = paro::QuantConfig{bits, static_cast<paro::QuantMode>(mode), static_cast<paro::QuantGrouping>(grouping),
                                     block};
        q.codes.assign(codes, codes + rows * cols);
        q.scales.assign(scales, scales + q.group_count());
        if (mode == 0)
            q.offsets.assign(offsets, offsets + q.group_count());
        paro::save_quant_tensor(q, path);
    });
}

int ref_load_quant_tensor(const char* path, unsigned* bits, int* mode, size_t* rows, size_t* cols, int32_t* codes,
                          float* scales, size_t* ngroups) {
    return guarded([&] {
        paro::QuantBlockTensor q = paro::load_quant_tensor(path);
        *bits = q.config.bits;
        *mode = (int)q.config.mode;
        *rows = q.rows;
        *cols = q.cols;
        *ngroups = q.scales.size();
        if (codes)
            std::copy(q.codes.begin(), q.codes.end(), codes);
        if (scales)
            std::copy(q.scales.begin(), q.scales.end(), scales);
    });
}

int ref_save_quant_tensor(const float* m, size_t rows, size_t cols, unsigned bits, int mode, size_t block,
                          const char* path) {
    return guarded([&] {
        paro::QuantConfig cfg{bits, static_cast<paro::QuantMode>(mode), paro::QuantGrouping::PerBlock, block};
        paro::save_quant_tensor(paro::quantize(mat(m, rows, cols), cfg), path);
    });
}

static int run_engine(int which, const float* q, const float* k, const float* v, size_t n, size_t d, float scale,
                      size_t dense_prefix, const uint8_t* mask_bits, size_t mask_k, size_t block, unsigned bits,
                      float* out, uint32_t* zeroed, size_t* nzeroed) {
    return guarded([&] {
        paro::AttnInputs in{mat(q, n, d), mat(k, n, d), mat(v, n, d), scale, dense_prefix};
        paro::BlockMask m;
        if (mask_bits) {
            m = paro::BlockMask(mask_k, mask_k, block, false);
            std::memcpy(m.bits.data(), mask_bits, mask_k * mask_k);
        }
        paro::AttnResult r;
        if (which == 0)
            r = paro::blocked_attention_stream(in, block);
        else if (which == 1)
            r = paro::masked_blocked_attention(in, m);
        else {
            paro::QuantConfig qcfg{bits, paro::QuantMode::Unsigned, paro::QuantGrouping::PerBlock, block};
            r = paro::quantized_blocked_attention(in, mask_bits ? &m : nullptr, qcfg);
        }
        export_result(r, out, zeroed, nzeroed);
    });
}

int ref_blocked_attention_stream(const float* q, const float* k, const float* v, size_t n, size_t d, float scale,
                                 size_t dense_prefix, size_t block, float* out, uint32_t* zeroed, size_t* nzeroed) {
    return run_engine(0, q, k, v, n, d, scale, dense_prefix, nullptr, 0, block, 8, out, zeroed, nzeroed);
}

int ref_masked_blocked_attention(const float* q, const float* k, const float* v, size_t n, size_t d, float scale,
                                 size_t dense_prefix, const uint8_t* mask_bits, size_t mask_k, size_t block,
                                 float* out, uint32_t* zeroed, size_t* nzeroed) {
    return run_engine(1, q, k, v, n, d, scale, dense_prefix, mask_bits, mask_k, block, 8, out, zeroed, nzeroed);
}

int ref_quantized_blocked_attention(const float* q, const float* k, const float* v, size_t n, size_t d, float scale,
                                    size_t dense_prefix, const uint8_t* mask_bits, size_t mask_k, size_t block,
                                    unsigned bits, float* out, uint32_t* zeroed, size_t* nzeroed) {
    return run_engine(2, q, k, v, n, d, scale, dense_prefix, mask_bits, mask_k, block, bits, out, zeroed, nzeroed);
}

int ref_gen_mask(const double* sums, size_t kr, size_t kc, double density, size_t block, size_t guard,
                 uint8_t* bits, size_t* repaired) {
    return guarded([&] {
        paro::BlockGrid g(kr, kc);
        std::copy(sums, sums + kr * kc, g.v.begin());
        paro::MaskGenResult r = paro::gen_mask(g, density, block, guard);
        std::copy(r.mask.bits.begin(), r.mask.bits.end(), bits);
        *repaired = r.repaired_rows;
    });
}

int ref_serialize_mask(const uint8_t* bits, size_t kr, size_t kc, size_t block, uint8_t* out, size_t* size) {
    return guarded([&] {
        paro::BlockMask m(kr, kc, block, false);
        std::memcpy(m.bits.data(), bits, kr * kc);
        auto blob = paro::serialize_mask(m);
        if (out)
            std::copy(blob.begin(), blob.end(), out);
        *size = blob.size();
    });
}

int ref_deserialize_mask(const uint8_t* data, size_t size, uint32_t* kr, uint32_t* kc, uint32_t* block,
                         uint8_t* bits, size_t* consumed) {
    return guarded([&] {
        paro::BlockMask m = paro::deserialize_mask(data, size, consumed);
        *kr = (uint32_t)m.k_rows;
        *kc = (uint32_t)m.k_cols;
        *block = (uint32_t)m.block;
        if (bits)
            std::copy(m.bits.begin(), m.bits.end(), bits);
    });
}

// build_schedule + save_schedule (mask.cpp:142-172, :246-265); sums: T grids of kr*kc
int ref_build_and_save_schedule(const double* sums, size_t T, size_t kr, size_t kc, double density, size_t block,
                                const char* path) {
    return guarded([&] {
        std::vector<paro::BlockGrid> calib;
        for (size_t t = 0; t < T; ++t) {
            paro::BlockGrid g(kr, kc);
            std::copy(sums + t * kr * kc, sums + (t + 1) * kr * kc, g.v.begin());
            calib.push_back(g);
        }
        paro::save_schedule(paro::build_schedule(calib, density, (uint32_t)T, block), path);
    });
}

// load_schedule(path).at(t) (mask.cpp:132-140, :267-305)
int ref_schedule_at(const char* path, uint32_t t, uint8_t* bits, uint32_t* kr) {
    return guarded([&] {
        paro::MaskSchedule s = paro::load_schedule(path);
        const paro::BlockMask& m = s.at(t);
        *kr = (uint32_t)m.k_rows;
        if (bits)
            std::copy(m.bits.begin(), m.bits.end(), bits);
    });
}

// tests/oracles.hpp random_matrix / test_value fixtures
void ref_random_matrix(size_t rows, size_t cols, uint64_t seed, float lo, float hi, float* out) {
    paro::Matrix m = oracle::random_matrix(rows, cols, seed, lo, hi);
    std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
}

void ref_test_values(uint64_t state, size_t count, float* out) {
    for (size_t i = 0; i < count; ++i)
        out[i] = oracle::test_value(state);
}

// load_plan_file (reorder.cpp:193-216) -> count entries; heads[] and orders
// (count * 8 chars, NUL-padded) may be NULL to query the count
int ref_load_plan_file(const char* path, uint32_t* count, uint32_t* heads, char* orders) {
    return guarded([&] {
        auto e = paro::load_plan_file(path);
        *count = (uint32_t)e.size();
        for (size_t i = 0; i < e.size(); ++i) {
            if (heads)
                heads[i] = e[i].first;
            if (orders) {
                std::memset(orders + 8 * i, 0, 8);
                std::memcpy(orders + 8 * i, e[i].second.data(), std::min<size_t>(7, e[i].second.size()));
            }
        }
    });
}

// plan_for_head of tools/main.cpp:118-126 (the CLI helper is not in the library;
// its five lines are restated here over the library's load_plan_file / make_perm)
int ref_plan_for_head(const char* path, const char* grid_text, uint32_t head, uint32_t* inverse) {
    return guarded([&] {
        const paro::TokenGrid grid = paro::parse_grid(grid_text);
        paro::PermPlan plan;
        const std::string p = path ? path : "";
        if (p.empty()) {
            plan = paro::make_perm(grid, grid.label_string());
        } else {
            bool found = false;
            for (const auto& [h, order] : paro::load_plan_file(p))
                if (h == head) {
                    plan = paro::make_perm(grid, order);
                    found = true;
                    break;
                }
            if (!found)
                throw paro::InputError(p + ": no plan entry for head " + std::to_string(head));
        }
        std::memcpy(inverse, plan.inverse.data(), plan.inverse.size() * 4);
    });
}

// N(0,1) stream of the reference's synthetic generator: std::mt19937_64 seeded
// with `seed`, the documented uniform (rng() >> 11) * 2^-53 (synth.cpp:20-22) and
// Box-Muller on (1 - u1, u2), one value per pair (synth.cpp:173-182; that
// function's unit_uniform is file-local, so its two lines are restated here).
// `count` values per stream, `nstreams` streams with seeds seed0 + stride * s,
// generated on `threads` host threads -- bench.py's reference arm builds its
// inputs with this, never with the product library.
void ref_synth_randn_streams(uint64_t seed0, uint64_t stride, size_t nstreams, size_t count, int threads,
                             float* out) {
    std::atomic<size_t> next{0};
    auto worker = [&] {
        for (;;) {
            const size_t s = next.fetch_add(1);
            if (s >= nstreams)
                break;
            std::mt19937_64 rng(seed0 + stride * s);
            auto unit = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
            float* o = out + s * count;
            for (size_t i = 0; i < count; ++i) {
                const double u1 = 1.0 - unit();
                const double u2 = unit();
                o[i] = static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2));
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t)
        pool.emplace_back(worker);
    for (auto& th : pool)
        th.join();
}

// synth.cpp:136-184 gen_attention_inputs (spec: grid text, weights per axis)
int ref_gen_attention_inputs(const char* grid_text, const float* weights, float bandwidth, float noise, uint64_t seed,
                             size_t head_dim, float* q, float* k, float* v) {
    return guarded([&] {
        paro::AggregationSpec spec;
        spec.grid = paro::parse_grid(grid_text);
        spec.axis_weights.assign(weights, weights + spec.grid.ndim());
        spec.bandwidth = bandwidth;
        spec.noise = noise;
        spec.seed = seed;
        paro::AttnInputs in = paro::gen_attention_inputs(spec, head_dim);
        std::memcpy(q, in.q.data.data(), in.q.data.size() * sizeof(float));
        std::memcpy(k, in.k.data.data(), in.k.data.size() * sizeof(float));
        std::memcpy(v, in.v.data.data(), in.v.data.size() * sizeof(float));
    });
}

// ---------------------------------------------------------------------------
// CPU baseline: the reference's own hot chain, one head per call exactly as
// cmd_run does it (proj/tools/main.cpp:292-305: permuted_inputs ->
// quantized_blocked_attention -> apply_perm_rows(out, plan.inverted())),
// without the metrics tail (main.cpp:308-317). Heads are spread over
// `threads` std::threads, round-robin; kernels::active() is resolved before
// the threads start (select() is not thread-safe).
// Inputs: q/k/v [H_run, N, d] host fp32 (original token order), masks
// [H_run, k, k] bytes (or null = dense), orders: H_run strings of ndim chars.
// Output: out [H_run, N, d]. Returns wall seconds of the timed region.
// ---------------------------------------------------------------------------
int ref_run_heads(const char* grid_text, size_t H_run, size_t d, const float* q, const float* k, const float* v,
                  const char* orders, const uint8_t* masks, unsigned bits, float scale, int threads, float* out,
                  double* seconds) {
    return guarded([&] {
        paro::TokenGrid grid = paro::parse_grid(grid_text);
        const size_t n = grid.token_count();
        const size_t kb = (n + 63) / 64;
        (void)paro::kernels::active();
        std::vector<paro::PermPlan> plans;
        for (size_t h = 0; h < H_run; ++h)
            plans.push_back(paro::make_perm(grid, std::string(orders + h * grid.ndim(), grid.ndim())));
        std::atomic<size_t> next{0};
        std::atomic<int> failed{0};
        auto worker = [&] {
            for (;;) {
                const size_t h = next.fetch_add(1);
                if (h >= H_run)
                    break;
                try {
                    paro::AttnInputs in{mat(q + h * n * d, n, d), mat(k + h * n * d, n, d), mat(v + h * n * d, n, d),
                                        scale, 0};
                    paro::AttnInputs pin{paro::apply_perm_rows(in.q, plans[h]), paro::apply_perm_rows(in.k, plans[h]),
                                         paro::apply_perm_rows(in.v, plans[h]), scale, 0};
                    paro::BlockMask m;
                    if (masks) {
                        m = paro::BlockMask(kb, kb, 64, false);
                        std::memcpy(m.bits.data(), masks + h * kb * kb, kb * kb);
                    }
                    paro::QuantConfig qcfg{bits, paro::QuantMode::Unsigned, paro::QuantGrouping::PerBlock, 64};
                    paro::AttnResult r = paro::quantized_blocked_attention(pin, masks ? &m : nullptr, qcfg);
                    paro::Matrix o = paro::apply_perm_rows(r.output, plans[h].inverted());
                    std::memcpy(out + h * n * d, o.data.data(), n * d * sizeof(float));
                } catch (...) {
                    failed = 1;
                }
            }
        };
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < std::max(1, threads); ++t)
            pool.emplace_back(worker);
        for (auto& th : pool)
            th.join();
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (failed)
            throw paro::InvariantError("a reference head failed");
    });
}

// block_sums(AttnMap(apply_perm_map(m, plan), block, relaxed)) -- cmd_maskgen's
// sums (main.cpp:236-238); identity when forward is NULL
int ref_perm_block_sums(const float* m, size_t n, const uint32_t* forward, const uint32_t* inverse, size_t block,
                        double* out) {
    return guarded([&] {
        paro::Matrix mat(n, n);
        std::memcpy(mat.data.data(), m, n * n * sizeof(float));
        paro::Matrix pm = mat;
        if (forward) {
            paro::PermPlan plan;
            plan.forward.assign(forward, forward + n);
            plan.inverse.assign(inverse, inverse + n);
            pm = paro::apply_perm_map(mat, plan);
        }
        paro::BlockGrid g = paro::block_sums(paro::AttnMap(std::move(pm), block, /*relaxed=*/true));
        std::memcpy(out, g.v.data(), g.v.size() * sizeof(double));
    });
}

// select_permutation(calib, grid, cfg, dense_prefix) (reorder.cpp:130-181):
// maps [count][n][n], scores [nperm][5], orders nperm*ndim chars
int ref_select_permutation(const float* maps, size_t count, size_t n, const char* grid_text, size_t block, float eps,
                           float sigma, float alpha, size_t dense_prefix, char* orders, double* scores, int* nperm,
                           int* chosen) {
    return guarded([&] {
        std::vector<paro::Matrix> calib;
        for (size_t c = 0; c < count; ++c) {
            paro::Matrix m(n, n);
            std::memcpy(m.data.data(), maps + c * n * n, n * n * sizeof(float));
            calib.push_back(std::move(m));
        }
        paro::MetricConfig cfg;
        cfg.block = block;
        cfg.eps = eps;
        cfg.sigma = sigma;
        cfg.alpha = alpha;
        const paro::TokenGrid grid = paro::parse_grid(grid_text);
        paro::SelectionResult r = paro::select_permutation(calib, grid, cfg, dense_prefix);
        *nperm = (int)r.scores.size();
        *chosen = (int)r.chosen;
        for (size_t p = 0; p < r.scores.size(); ++p) {
            const paro::PermScore& sc = r.scores[p];
            std::memcpy(orders + p * sc.order.size(), sc.order.data(), sc.order.size());
            double* o = scores + p * 5;
            o[0] = sc.sparse_mean;
            o[1] = sc.quant_mean;
            o[2] = sc.sparse_share;
            o[3] = sc.quant_share;
            o[4] = sc.combined;
        }
    });
}

} // extern "C"
