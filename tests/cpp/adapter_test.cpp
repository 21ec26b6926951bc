// adapter_test.cpp -- the reference's own C++ API vs include/paro_b200.hpp.
//
// Built by __graft_entry__.build() against the reference headers and the
// reference library compiled from its sources (oracle/_ref/libparo_ref.so --
// test infrastructure), plus the C oracle for the INT8-QK engine. Reads like
// the reference's doctest cases: same calls, same exception classes.
//
//   adapter_test host   host-side stages (no GPU)
//   adapter_test gpu    device stages on cuda:0
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "paro/attention.hpp"
#include "paro/error.hpp"
#include "paro/mask.hpp"
#include "paro/quant.hpp"
#include "paro/reorder.hpp"
#include "paro/tensor.hpp"
#include "paro_b200.hpp"

extern "C" int oracle_stream_engine(const float* q, const float* k, const float* v, size_t n, size_t d,
                                    float scale, size_t dense_prefix, size_t block, const uint8_t* mask,
                                    int pv_bits, int qk_mode, float* out, uint8_t* zeroed);

static int failures = 0;
#define CHECK(cond)                                                                                          \
    do {                                                                                                     \
        if (!(cond)) {                                                                                       \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                   \
            ++failures;                                                                                      \
        }                                                                                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, Type)                                                                          \
    do {                                                                                                     \
        bool ok = false;                                                                                     \
        try {                                                                                                \
            (void)(expr);                                                                                    \
        } catch (const Type&) {                                                                              \
            ok = true;                                                                                       \
        } catch (...) {                                                                                      \
        }                                                                                                    \
        if (!ok) {                                                                                           \
            std::fprintf(stderr, "CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr);          \
            ++failures;                                                                                      \
        }                                                                                                    \
    } while (0)

static paro::Matrix randn(size_t r, size_t c, unsigned seed, float s = 1.0f) {
    std::mt19937 g(seed);
    std::normal_distribution<float> nd(0.f, s);
    paro::Matrix m(r, c);
    for (float& x : m.data)
        x = nd(g);
    return m;
}

static void host_tests() {
    // make_perm: every order of several grids, bit-exact (reorder.cpp:49-72)
    for (const char* text : {"F:2,H:8,W:8", "F:13,H:30,W:45", "H:64,W:64", "W:7,H:3", "H:5,F:3,W:2"}) {
        paro::TokenGrid g = paro::parse_grid(text);
        for (const paro::PermPlan& ref : paro::enumerate_perms(g)) {
            paro::PermPlan got = paro_b200::make_perm(g, ref.order);
            CHECK(got.forward == ref.forward);
            CHECK(got.inverse == ref.inverse);
        }
    }
    paro::TokenGrid cube({{'F', 4}, {'H', 4}, {'W', 4}});
    CHECK_THROWS_AS(paro_b200::make_perm(cube, "FH"), paro::ConfigError);
    CHECK_THROWS_AS(paro_b200::make_perm(cube, "FHX"), paro::InputError);
    // per-head plan files: the reference's writer, our reader and plan_for_head (a3)
    {
        const std::string path = "/tmp/paro_adapter_test.plan";
        paro::save_plan_file({{0, "WHF"}, {2, "HFW"}, {2, "FHW"}}, path);
        CHECK(paro_b200::load_plan_file(path) == paro::load_plan_file(path));
        CHECK(paro_b200::plan_for_head(path, cube, 2).inverse == paro::make_perm(cube, "HFW").inverse);
        CHECK(paro_b200::plan_for_head("", cube, 9).inverse == paro::make_perm(cube, "FHW").inverse);
        CHECK_THROWS_AS(paro_b200::plan_for_head(path, cube, 1), paro::InputError);
        CHECK_THROWS_AS(paro_b200::load_plan_file("/nonexistent/x.plan"), paro::IoError);
        std::remove(path.c_str());
    }
    // PMSK decode (mask.cpp:217-244)
    std::mt19937 g(3);
    for (auto [kr, kc] : {std::pair<size_t, size_t>{33, 17}, {275, 275}, {1, 1}}) {
        paro::BlockMask m(kr, kc, 64, false);
        for (auto& b : m.bits)
            b = (g() % 3) == 0;
        std::vector<uint8_t> blob = paro::serialize_mask(m);
        size_t used = 0;
        paro::BlockMask back = paro_b200::deserialize_mask(blob.data(), blob.size(), &used);
        CHECK(used == blob.size());
        CHECK(back.bits == m.bits && back.k_rows == kr && back.k_cols == kc && back.block == 64);
        CHECK_THROWS_AS(paro_b200::deserialize_mask(blob.data(), blob.size() - 1), paro::FormatError);
    }
}

static void gpu_tests() {
    // apply_perm_rows on the GPU == reference (reorder.cpp:93-101)
    paro::TokenGrid grid = paro::parse_grid("F:13,H:30,W:45");
    paro::PermPlan plan = paro::make_perm(grid, "WHF");
    paro::Matrix m = randn(grid.token_count(), 64, 1);
    CHECK(paro_b200::apply_perm_rows(m, plan).data == paro::apply_perm_rows(m, plan).data);
    // quantize == reference for the Q/K configuration (quant.cpp:60-104)
    for (unsigned bits : {4u, 8u})
        for (size_t cols : {64u, 128u}) {
            paro::Matrix x = randn(1000, cols, 7 + bits, 3.0f);
            paro::QuantConfig cfg{bits, paro::QuantMode::Symmetric, paro::QuantGrouping::PerBlock, 64};
            paro::QuantBlockTensor r = paro::quantize(x, cfg), b = paro_b200::quantize(x, cfg);
            CHECK(r.codes == b.codes);
            CHECK(r.scales == b.scales);
        }
    // quantized_blocked_attention vs the restated INT8-QK engine (bit-exact P codes at d=64)
    const size_t n = 500, d = 64, kb = (n + 63) / 64;
    paro::AttnInputs in{randn(n, d, 11), randn(n, d, 12), randn(n, d, 13), 0.0f, 0};
    paro::BlockMask mask(kb, kb, 64, false);
    for (size_t i = 0; i < kb; ++i)
        for (size_t j = 0; j < kb; ++j)
            mask.set(i, j, i == j || ((i * 7 + j * 3) % 5) < 2);
    for (unsigned bits : {8u, 4u}) {
        paro::QuantConfig qcfg{bits, paro::QuantMode::Unsigned, paro::QuantGrouping::PerBlock, 64};
        paro::AttnResult res = paro_b200::quantized_blocked_attention(in, &mask, qcfg);
        std::vector<float> ref(n * d);
        std::vector<uint8_t> z(n);
        oracle_stream_engine(in.q.data.data(), in.k.data.data(), in.v.data.data(), n, d, 0.0f, 0, 64,
                             mask.bits.data(), (int)bits, 1, ref.data(), z.data());
        double md = 0, mo = 0;
        for (size_t i = 0; i < n * d; ++i) {
            md = std::max(md, (double)std::fabs(res.output.data[i] - ref[i]));
            mo = std::max(mo, (double)std::fabs(ref[i]));
        }
        std::printf("quantized_blocked_attention bits=%u: max|dO|/max|O| = %.3e\n", bits, md / mo);
        CHECK(md / mo <= 1e-5);
        CHECK(res.zeroed_rows.empty());
    }
    // dense text-token prefix (AttnInputs::dense_prefix): K4 + K3 through the adapter
    for (size_t dp : {size_t(1), size_t(90), size_t(200)}) {
        paro::AttnInputs inp{in.q, in.k, in.v, 0.0f, dp};
        paro::QuantConfig qcfg{8, paro::QuantMode::Unsigned, paro::QuantGrouping::PerBlock, 64};
        paro::AttnResult res = paro_b200::quantized_blocked_attention(inp, &mask, qcfg);
        std::vector<float> ref(n * d);
        std::vector<uint8_t> z(n);
        oracle_stream_engine(in.q.data.data(), in.k.data.data(), in.v.data.data(), n, d, 0.0f, dp, 64,
                             mask.bits.data(), 8, 1, ref.data(), z.data());
        double md = 0, mo = 0;
        for (size_t i = 0; i < n * d; ++i) {
            md = std::max(md, (double)std::fabs(res.output.data[i] - ref[i]));
            mo = std::max(mo, (double)std::fabs(ref[i]));
        }
        std::printf("quantized_blocked_attention dense_prefix=%zu: max|dO|/max|O| = %.3e\n", dp, md / mo);
        CHECK(md / mo <= 1e-4); // dense tiles: bf16 3-term split P.V (tests/test_gpu_parity.py PREFIX_TOL)
    }
    paro::AttnInputs all_dense{in.q, in.k, in.v, 0.0f, n};
    CHECK_THROWS_AS(paro_b200::quantized_blocked_attention(all_dense, &mask, paro::QuantConfig{}), paro::ConfigError);
    // a whole layer (cmd_run's per-head chain for H heads): per-head orders, masks,
    // optional text prefix (PermPlan::with_prefix) vs the reference's permutation +
    // the restated engine + the reference's inverse permutation, head by head
    for (size_t dp : {size_t(0), size_t(20)}) {
        paro::TokenGrid g = paro::parse_grid("F:3,H:7,W:11");
        const std::vector<std::string> orders{"WHF", "HFW"};
        const size_t H = 2, d2 = 64, N = g.token_count() + dp, kb2 = (N + 63) / 64;
        paro_b200::Layer layer(g, H, d2, orders, dp);
        CHECK(layer.tokens() == N);
        std::vector<paro::BlockMask> masks;
        std::vector<paro::Matrix> q, k, v;
        for (size_t h = 0; h < H; ++h) {
            paro::BlockMask mk(kb2, kb2, 64, false);
            for (size_t i = 0; i < kb2; ++i)
                for (size_t j = 0; j < kb2; ++j)
                    mk.set(i, j, i == j || ((i * 5 + j * 3 + h) % 4) < 2);
            masks.push_back(mk);
            q.push_back(randn(N, d2, 40 + h));
            k.push_back(randn(N, d2, 50 + h));
            v.push_back(randn(N, d2, 60 + h));
        }
        layer.set_masks(masks);
        const std::vector<paro::AttnResult> out = layer.forward(q, k, v, 0.0f, 8);
        for (size_t h = 0; h < H; ++h) {
            paro::PermPlan plan = paro::make_perm(g, orders[h]);
            if (dp)
                plan = plan.with_prefix(dp);
            const paro::Matrix qp = paro::apply_perm_rows(q[h], plan), kp = paro::apply_perm_rows(k[h], plan),
                               vp = paro::apply_perm_rows(v[h], plan);
            paro::Matrix refp(N, d2);
            std::vector<uint8_t> z(N);
            oracle_stream_engine(qp.data.data(), kp.data.data(), vp.data.data(), N, d2, 0.0f, dp, 64,
                                 masks[h].bits.data(), 8, 1, refp.data.data(), z.data());
            const paro::Matrix ref = paro::apply_perm_rows(refp, plan.inverted());
            double md = 0, mo = 0;
            for (size_t i = 0; i < N * d2; ++i) {
                md = std::max(md, (double)std::fabs(out[h].output.data[i] - ref.data[i]));
                mo = std::max(mo, (double)std::fabs(ref.data[i]));
            }
            std::printf("Layer head %zu dense_prefix=%zu: max|dO|/max|O| = %.3e\n", h, dp, md / mo);
            CHECK(md / mo <= (dp ? 1e-4 : 1e-5));
            CHECK(out[h].zeroed_rows.empty());
        }
        CHECK_THROWS_AS(layer.set_masks({masks[0]}), paro::ShapeError);
        // rotary embedding fused into the reorder+quantize pass == rotating the fp32 rows first
        paro::Matrix rc(N - dp, d2), rs(N - dp, d2);
        for (size_t t = 0; t < N - dp; ++t)
            for (size_t c = 0; c < d2; ++c) {
                const double ang = (double)t * std::pow(10000.0, -(double)(c / 2) / (double)(d2 / 2));
                rc.data[t * d2 + c] = (float)std::cos(ang);
                rs.data[t * d2 + c] = (float)std::sin(ang);
            }
        std::vector<paro::Matrix> qr = q, kr = k;
        for (size_t h = 0; h < H; ++h)
            for (size_t t = dp; t < N; ++t)
                for (size_t c = 0; c < d2; c += 2) {
                    const size_t e = t * d2 + c, r = (t - dp) * d2 + c;
                    for (paro::Matrix* m : {&qr[h], &kr[h]}) {
                        const paro::Matrix& src = m == &qr[h] ? q[h] : k[h];
                        const float a = src.data[e], b = src.data[e + 1];
                        const float p0 = a * rc.data[r], p1 = b * rs.data[r];
                        const float p2 = b * rc.data[r + 1], p3 = a * rs.data[r + 1];
                        m->data[e] = p0 - p1;
                        m->data[e + 1] = p2 + p3;
                    }
                }
        const std::vector<paro::AttnResult> plain = layer.forward(qr, kr, v, 0.0f, 8);
        layer.set_rope(rc, rs);
        const std::vector<paro::AttnResult> fused = layer.forward(q, k, v, 0.0f, 8);
        for (size_t h = 0; h < H; ++h)
            CHECK(fused[h].output.data == plain[h].output.data);
        std::printf("Layer dense_prefix=%zu: fused rotary embedding bit-identical to the fp32 pre-rotation\n", dp);
        CHECK_THROWS_AS(layer.set_rope(paro::Matrix(N + 1, d2), paro::Matrix(N + 1, d2)), paro::ShapeError);
        layer.set_rope(paro::Matrix(), paro::Matrix());
        CHECK(layer.forward(qr, kr, v, 0.0f, 8)[0].output.data == plain[0].output.data);
    }
    paro::QuantConfig bad{16, paro::QuantMode::Unsigned, paro::QuantGrouping::PerBlock, 64};
    CHECK_THROWS_AS(paro_b200::quantized_blocked_attention(in, &mask, bad), paro::ConfigError);
    paro::AttnInputs short_v{in.q, in.k, randn(n - 1, d, 3), 0.0f, 0};
    CHECK_THROWS_AS(paro_b200::quantized_blocked_attention(short_v, &mask, paro::QuantConfig{}), paro::ShapeError);
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "host";
    try {
        if (mode == "host")
            host_tests();
        else
            gpu_tests();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "uncaught: %s\n", e.what());
        return 100;
    }
    std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
    return failures;
}
