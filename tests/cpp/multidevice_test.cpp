// multidevice_test.cpp -- the head-sharded multi-GPU path from C++ host threads,
// through the C ABI only (include/paro_b200.h).
//
// The reference runs one head per call (tools/main.cpp:276-300) and scales with a
// per-head worker pool; here W host threads each own one paro_ctx on
// device (w % devices) and one layer of a contiguous head shard [w*H/W, (w+1)*H/W)
// (no data crosses GPUs), run paro_layer_forward_host on their
// slice of the host buffers concurrently, and the reassembled layer must equal a
// single-context run of all heads bit for bit. W = max(2, devices): on a one-GPU
// box two contexts share the device, which still exercises concurrent contexts.
//   multidevice_test [grid] [heads] [d] [pv_bits]     exit code = failed checks
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "paro_b200.h"

static int failures = 0;
#define CHECK(cond)                                                                                          \
    do {                                                                                                     \
        if (!(cond)) {                                                                                       \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                   \
            ++failures;                                                                                      \
        }                                                                                                    \
    } while (0)
#define OK(call)                                                                                             \
    do {                                                                                                     \
        const int rc_ = (call);                                                                              \
        if (rc_) {                                                                                           \
            std::fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, paro_last_error());                    \
            std::exit(100);                                                                                  \
        }                                                                                                    \
    } while (0)

struct Shard {
    int device;
    uint32_t h0, hn;
};

// one layer of heads [h0, h0 + hn) on its own context: forward from host buffers
static void run_shard(const Shard& s, const char* grid, uint32_t d, int pv_bits, size_t N, const std::vector<std::string>& orders,
                      const std::vector<float>& q, const std::vector<float>& k, const std::vector<float>& v,
                      const std::vector<uint8_t>& masks, size_t kb, std::vector<float>& out, std::vector<uint8_t>& zeroed) {
    paro_ctx* ctx = nullptr;
    OK(paro_ctx_create(s.device, &ctx));
    std::string ords;
    for (uint32_t h = s.h0; h < s.h0 + s.hn; ++h)
        ords += orders[h];
    paro_layer* layer = nullptr;
    OK(paro_layer_create(ctx, s.hn, d, grid, ords.c_str(), &layer));
    OK(paro_layer_set_masks(layer, nullptr, masks.data() + (size_t)s.h0 * kb * kb));
    const size_t off = (size_t)s.h0 * N * d;
    OK(paro_layer_forward_host(layer, nullptr, q.data() + off, k.data() + off, v.data() + off, 0.0f, pv_bits,
                               out.data() + off, zeroed.data() + (size_t)s.h0 * N));
    OK(paro_layer_destroy(layer));
    OK(paro_ctx_destroy(ctx));
}

int main(int argc, char** argv) {
    const char* grid = argc > 1 ? argv[1] : "F:13,H:30,W:45";
    const uint32_t H = argc > 2 ? (uint32_t)atoi(argv[2]) : 8;
    const uint32_t d = argc > 3 ? (uint32_t)atoi(argv[3]) : 64;
    const int pv_bits = argc > 4 ? atoi(argv[4]) : 8;
    int ndim = 0;
    char labels[4] = {0};
    uint32_t ext[3] = {0, 0, 0};
    OK(paro_parse_grid(grid, &ndim, labels, ext));
    size_t N = 1;
    for (int a = 0; a < ndim; ++a)
        N *= ext[a];
    const size_t kb = (N + 63) / 64;
    char obuf[64];
    int norders = 0;
    OK(paro_enumerate_orders(ndim, labels, obuf, &norders));
    std::vector<std::string> orders;
    for (uint32_t h = 0; h < H; ++h)
        orders.emplace_back(obuf + (h % norders) * ndim, ndim);

    // inputs: the bench's seeded N(0,1) streams; masks ~30% random + the diagonal
    std::vector<float> q((size_t)H * N * d), k(q.size()), v(q.size());
    for (uint32_t h = 0; h < H; ++h) {
        OK(paro_synth_randn(1000 + 3 * h, N * d, q.data() + (size_t)h * N * d));
        OK(paro_synth_randn(1001 + 3 * h, N * d, k.data() + (size_t)h * N * d));
        OK(paro_synth_randn(1002 + 3 * h, N * d, v.data() + (size_t)h * N * d));
    }
    std::vector<uint8_t> masks((size_t)H * kb * kb);
    uint64_t x = 0x9e3779b97f4a7c15ull;
    for (size_t i = 0; i < masks.size(); ++i) {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        const size_t r = (i / kb) % kb, c = i % kb;
        masks[i] = (r == c || (x % 1000) < 300) ? 1 : 0;
    }

    int ndev = 0;
    OK(paro_device_count(&ndev));
    const uint32_t W = ndev >= 2 ? (uint32_t)ndev : 2u;
    if (H % W) {
        std::fprintf(stderr, "%u heads do not split over %u workers\n", H, W);
        return 100;
    }
    // single context, all heads
    std::vector<float> ref(q.size());
    std::vector<uint8_t> ref_z((size_t)H * N);
    run_shard({0, 0, H}, grid, d, pv_bits, N, orders, q, k, v, masks, kb, ref, ref_z);
    // W host threads, one context + head shard each
    std::vector<float> out(q.size(), -1.0f);
    std::vector<uint8_t> z((size_t)H * N, 7);
    std::vector<std::thread> pool;
    for (uint32_t w = 0; w < W; ++w)
        pool.emplace_back([&, w] {
            run_shard({(int)(w % (uint32_t)ndev), w * (H / W), H / W}, grid, d, pv_bits, N, orders, q, k, v, masks, kb,
                      out, z);
        });
    for (auto& t : pool)
        t.join();
    CHECK(std::memcmp(out.data(), ref.data(), out.size() * sizeof(float)) == 0);
    CHECK(std::memcmp(z.data(), ref_z.data(), z.size()) == 0);
    std::printf("multidevice_test: %s H=%u d=%u pv=%d, %u workers on %d device(s): %s\n", grid, H, d, pv_bits, W, ndev,
                failures ? "MISMATCH" : "bit-identical to one context");
    return failures;
}
