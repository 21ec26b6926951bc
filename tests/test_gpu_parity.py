"""GPU parity: every stage of the B200 path against the CPU oracle on the same inputs.

Bar (BASELINE north_star): bit-exact for permutation indices, kept lists, quantized
integer tensors (+ scales) and int32 QK^T accumulators; max|dO|/max|O| <= 1e-3 for
the attention output against the restated INT8-QK engine (oracle/paro_oracle.c).
"""
import numpy as np
import pytest

from conftest import randn, rel_err

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-3  # max|dO| / max|O| (north_star)
# d=64 P codes are bit-exact with the reference quantizer (boundary path), so the
# only differences left are fp32 accumulation order: any single code flip would
# exceed this bound.
EXACT_TOL = 1e-5


def tol(d):
    # d=128 P codes are bit-exact too (exact row extremes via the tagged
    # argmax + fp64 rescan); OUT_TOL stays the north_star bar
    return EXACT_TOL

# (grid, heads, d, orders) -- c1 from BASELINE.configs[0] plus ragged / 2-D / d=128 shapes
CASES = [
    ("F:2,H:8,W:8", 2, 64, ["HWF", "WFH"]),
    ("F:3,H:7,W:11", 3, 64, ["FHW", "WHF", "HFW"]),  # N=231: ragged tail (39 rows), odd kb=4? -> kb=4
    ("H:20,W:33", 2, 128, ["HW", "WH"]),  # N=660: kb=11 (odd: unpaired last q-block), tail 20
    ("F:5,H:9,W:14", 2, 128, ["WFH", "FWH"]),  # N=630
]


def permuted(x, inv):
    return np.ascontiguousarray(x[inv])


def make_inputs(H, N, d, seed):
    return randn(seed, (H, N, d)), randn(seed + 1, (H, N, d)), randn(seed + 2, (H, N, d))


def random_masks(H, kb, density, seed, empty_row=None):
    rng = np.random.default_rng(seed)
    m = (rng.random((H, kb, kb)) < density).astype(np.uint8)
    for h in range(H):
        np.fill_diagonal(m[h], 1)
    if empty_row is not None:
        m[:, empty_row, :] = 0
    return m


@pytest.mark.parametrize("grid,H,d,orders", CASES)
def test_perm_tables_bit_exact(paro, ctx, oracle, grid, H, d, orders):
    g = paro.parse_grid(grid)
    layer = paro.Layer(ctx, H, d, g, orders)
    b = layer.buffers()
    for h in range(H):
        fwd, inv = oracle.make_perm(g.labels, g.extents, orders[h])
        assert np.array_equal(b["inverse"][h], inv)
        assert np.array_equal(b["forward"][h], fwd)
    layer.close()


@pytest.mark.parametrize("grid,H,d,orders", CASES)
@pytest.mark.parametrize("v_bits", [8, 4])
def test_reorder_quantize_bit_exact(paro, ctx, oracle, grid, H, d, orders, v_bits):
    g = paro.parse_grid(grid)
    N = g.token_count()
    q, k, v = make_inputs(H, N, d, 11)
    layer = paro.Layer(ctx, H, d, g, orders)
    dq, dk, dv = (paro.DeviceBuffer.from_array(x) for x in (q, k, v))
    layer.reorder_quantize(dq.ptr, dk.ptr, dv.ptr, v_bits)
    paro.stream_sync()
    b = layer.buffers()
    kb = (N + 63) // 64
    G = d // 64
    for h in range(H):
        _, inv = oracle.make_perm(g.labels, g.extents, orders[h])
        for name, x, sc in (("q", q, b["q_scales"][h]), ("k", k, b["meta"][h][:, :G])):
            codes, scales, _ = oracle.quantize(permuted(x[h], inv), 8, 1, 64)
            assert np.array_equal(b[name][h][:N].astype(np.int32), codes), name
            if name == "q":
                assert np.all(b[name][h][N:] == 0)
            else:  # K padding rows repeat the last block's first row (K3 tail handling)
                assert np.all(b[name][h][N:kb * 64] == b[name][h][(kb - 1) * 64])
                assert np.all(b[name][h][kb * 64:] == 0)
            assert np.array_equal(sc[:kb].reshape(-1).view(np.uint32), scales.view(np.uint32)), name
        vc, vs, vcs = oracle.quant_v(permuted(v[h], inv), v_bits)
        assert np.array_equal(b["v"][h][:N].astype(np.int32), vc)
        assert np.array_equal(b["meta"][h][:kb, 2].view(np.uint32), vs.view(np.uint32))
        assert np.array_equal(b["meta"][h][:kb, 4:].astype(np.int64), vcs)
    layer.close()


@pytest.mark.parametrize("grid,H,d,orders", CASES)
def test_mask_lists(paro, ctx, grid, H, d, orders):
    g = paro.parse_grid(grid)
    kb = (g.token_count() + 63) // 64
    masks = random_masks(H, kb, 0.3, 5, empty_row=kb - 1)
    layer = paro.Layer(ctx, H, d, g, orders)
    layer.set_masks(masks)
    kept, total = layer.mask_stats()
    assert np.array_equal(kept, masks.sum(axis=2).astype(np.uint32))
    assert total == int(masks.sum())
    layer.close()


@pytest.mark.parametrize("grid,H,d,orders", CASES)
def test_qk_int32_accumulators_bit_exact(paro, ctx, grid, H, d, orders):
    g = paro.parse_grid(grid)
    N = g.token_count()
    kb = (N + 63) // 64
    q, k, v = make_inputs(H, N, d, 23)
    layer = paro.Layer(ctx, H, d, g, orders)
    dq, dk, dv = (paro.DeviceBuffer.from_array(x) for x in (q, k, v))
    layer.reorder_quantize(dq.ptr, dk.ptr, dv.ptr, 8)
    paro.stream_sync()
    b = layer.buffers()
    rng = np.random.default_rng(3)
    tiles = np.array([[h, qb, bj] for h in range(H) for qb in range(kb) for bj in range(kb)], np.uint32)
    if len(tiles) > 200:
        tiles = tiles[rng.choice(len(tiles), 200, replace=False)]
    S = layer.debug_qk(tiles)
    G = d // 64
    for t, (h, qb, bj) in enumerate(tiles):
        Q = b["q"][h][qb * 64:(qb + 1) * 64].astype(np.int64)
        K = b["k"][h][bj * 64:(bj + 1) * 64].astype(np.int64)
        for gi in range(G):
            ref = Q[:, gi * 64:(gi + 1) * 64] @ K[:, gi * 64:(gi + 1) * 64].T
            assert np.array_equal(S[t, gi].astype(np.int64), ref), (h, qb, bj, gi)
    layer.close()


def run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, masks, pv_bits, seed, scale=0.0):
    g = paro.parse_grid(grid)
    N = g.token_count()
    q, k, v = make_inputs(H, N, d, seed)
    layer = paro.Layer(ctx, H, d, g, orders)
    layer.set_masks(masks)
    out, zeroed = layer.forward_host(q, k, v, scale, pv_bits)
    layer.close()
    worst = 0.0
    for h in range(H):
        fwd, inv = oracle.make_perm(g.labels, g.extents, orders[h])
        ref, zref_perm = oracle.paro_head(q[h], k[h], v[h], fwd, inv, None if masks is None else masks[h], pv_bits,
                                          qk_mode=1, scale=scale)
        zref = np.zeros(N, bool)
        zref[inv[zref_perm]] = True  # permuted index -> original token
        assert np.array_equal(zeroed[h].astype(bool), zref)
        assert np.all(out[h][zref] == 0)
        worst = max(worst, rel_err(out[h], ref))
    print(f"[attn] {grid} H={H} d={d} pv={pv_bits} masks={'none' if masks is None else 'yes'}: max|dO|/max|O| = {worst:.3e}")
    return worst


@pytest.mark.parametrize("grid,H,d,orders", CASES)
@pytest.mark.parametrize("pv_bits", [8, 4])
def test_attention_matches_oracle(paro, ctx, oracle, grid, H, d, orders, pv_bits):
    kb = (paro.parse_grid(grid).token_count() + 63) // 64
    masks = random_masks(H, kb, 0.4, 7)
    err = run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, masks, pv_bits, 31)
    assert err <= tol(d), err


@pytest.mark.parametrize("d", [64, 128])
def test_attention_dense_and_zeroed_rows(paro, ctx, oracle, d):
    grid, H, orders = "F:4,H:10,W:12", 2, ["HWF", "FWH"]  # N=480, kb=8
    assert run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, None, 8, 41) <= tol(d)
    masks = random_masks(H, 8, 0.3, 9, empty_row=3)
    assert run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, masks, 8, 43) <= tol(d)


def test_single_head_api_matches_oracle(paro, ctx, oracle):
    n, d = 300, 64
    q, k, v = randn(1, (n, d)), randn(2, (n, d)), randn(3, (n, d))
    kb = (n + 63) // 64
    mask = paro.BlockMask(kb, kb, 64, random_masks(1, kb, 0.5, 4)[0])
    res = ctx.quantized_blocked_attention(paro.AttnInputs(q, k, v), mask, paro.QuantConfig(8))
    ref, z = oracle.stream_engine(q, k, v, mask.bits, 8, qk_mode=1)
    assert rel_err(res.output, ref) <= EXACT_TOL
    assert res.zeroed_rows == list(np.nonzero(z)[0])


def test_device_and_host_paths_identical(paro, ctx):
    grid, H, d = "F:3,H:8,W:8", 2, 64
    N = 192
    q, k, v = make_inputs(H, N, d, 50)
    masks = random_masks(H, 3, 0.5, 1)
    layer = paro.Layer(ctx, H, d, grid, ["WHF", "HFW"])
    layer.set_masks(masks)
    out_h, z_h = layer.forward_host(q, k, v, 0.0, 8)
    dq, dk, dv = (paro.DeviceBuffer.from_array(x) for x in (q, k, v))
    dout = paro.DeviceBuffer(q.nbytes)
    dz = paro.DeviceBuffer(H * N)
    layer.forward(dq.ptr, dk.ptr, dv.ptr, 0.0, 8, dout.ptr, dz.ptr)
    paro.stream_sync()
    assert np.array_equal(dout.download(q.shape, np.float32), out_h)
    assert np.array_equal(dz.download((H, N), np.uint8), z_h)
    # deterministic across runs
    out_h2, _ = layer.forward_host(q, k, v, 0.0, 8)
    assert np.array_equal(out_h, out_h2)
    layer.close()


@pytest.mark.parametrize("chunks", [1, 2, 3, 5])
def test_pipelined_host_forward_matches_device_forward(paro, ctx, chunks):
    """forward_host's chunked upload/compute/download pipeline (per-chunk LPT
    work lists, K1 head ranges) reproduces the one-shot device forward bit for
    bit, for chunk counts that do and do not divide the head count."""
    grid, H, d = "F:3,H:7,W:11", 5, 64
    N = 231
    q, k, v = make_inputs(H, N, d, 70)
    masks = random_masks(H, 4, 0.4, 3, empty_row=1)
    layer = paro.Layer(ctx, H, d, grid, ["WHF", "HFW", "FHW", "FWH", "HWF"])
    layer.set_masks(masks)
    dq, dk, dv = (paro.DeviceBuffer.from_array(x) for x in (q, k, v))
    dout = paro.DeviceBuffer(q.nbytes)
    dz = paro.DeviceBuffer(H * N)
    layer.forward(dq.ptr, dk.ptr, dv.ptr, 0.0, 8, dout.ptr, dz.ptr)
    paro.stream_sync()
    ref, zref = dout.download(q.shape, np.float32), dz.download((H, N), np.uint8)
    layer.set_pipeline_chunks(chunks)
    out_h, z_h = layer.forward_host(q, k, v, 0.0, 8)
    assert np.all(np.isfinite(ref))
    assert np.array_equal(out_h, ref)
    assert np.array_equal(z_h, zref)
    layer.close()


def test_device_apply_perm_rows_and_quantize(paro, ctx, oracle):
    g = paro.parse_grid("F:13,H:30,W:45")
    plan = paro.make_perm(g, "WHF")
    m = randn(8, (g.token_count(), 64))
    got = ctx.apply_perm_rows(m, plan)
    assert np.array_equal(got, m[plan.inverse])
    for cols in (64, 128):
        for bits in (4, 8):
            x = randn(9 + cols + bits, (1000, cols)) * 3
            qt = ctx.quantize(x, paro.QuantConfig(bits, paro.SYMMETRIC, paro.PER_BLOCK, 64))
            codes, scales, _ = oracle.quantize(x, bits, 1, 64)
            assert np.array_equal(qt.codes, codes)
            assert np.array_equal(qt.scales.view(np.uint32), scales.view(np.uint32))


def test_gpu_errors(paro, ctx):
    with pytest.raises(paro.ConfigError):
        paro.Layer(ctx, 2, 96, "H:8,W:8")
    layer = paro.Layer(ctx, 1, 64, "H:8,W:8")
    layer.set_masks(None)
    q = randn(0, (1, 64, 64))
    with pytest.raises(paro.ConfigError):
        layer.forward_host(q, q, q, 0.0, 6)
    with pytest.raises(paro.ShapeError):
        layer.forward_host(q[:, :32], q[:, :32], q[:, :32], 0.0, 8)
    layer.close()
    with pytest.raises(paro.ConfigError):
        ctx.quantized_blocked_attention(paro.AttnInputs(q[0], q[0], q[0]), None, paro.QuantConfig(16))


def test_misaligned_device_buffers_rejected(paro, ctx):
    # K1 / K4a read rows and K3 writes rows with 16-byte vector accesses: a device
    # pointer that is not 16-byte aligned is a ConfigError, not a fault
    H, d, grid = 1, 64, "H:8,W:8"
    q = randn(3, (H, 64, d))
    layer = paro.Layer(ctx, H, d, grid)
    layer.set_masks(None)
    buf = paro.DeviceBuffer(q.nbytes + 64)
    out = paro.DeviceBuffer(q.nbytes + 64)
    for off in (4, 8):
        with pytest.raises(paro.ConfigError):
            layer.reorder_quantize(buf.ptr + off, buf.ptr, buf.ptr, 8)
        with pytest.raises(paro.ConfigError):
            layer.forward(buf.ptr, buf.ptr, buf.ptr + off, 0.0, 8, out.ptr, None)
        with pytest.raises(paro.ConfigError):
            layer.forward(buf.ptr, buf.ptr, buf.ptr, 0.0, 8, out.ptr + off, None)
    layer.forward(buf.ptr + 16, buf.ptr + 16, buf.ptr + 16, 0.0, 8, out.ptr + 16, None)  # 16-byte offsets are fine
    paro.stream_sync()
    layer.close()


# dense-prefix tiles are unquantized: K4 runs P.V on the tensor cores as a
# 3-term bf16 split (16 significant bits per operand, fp32 accumulation);
# observed <= 7e-6, bound set 10x under the north_star 1e-3.
PREFIX_TOL = 1e-4


def prefix_inverse(oracle, g, order, dp):
    """PermPlan::with_prefix (reorder.cpp:30-47): text tokens [0, dp) stay in
    place, the grid's permutation follows offset by dp. Returns inverse."""
    _, inv = oracle.make_perm(g.labels, g.extents, order)
    return np.concatenate([np.arange(dp, dtype=np.int64), dp + inv.astype(np.int64)])


def run_prefix_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, dp, masks, pv_bits, seed):
    g = paro.parse_grid(grid)
    N = g.token_count() + dp
    q, k, v = make_inputs(H, N, d, seed)
    layer = paro.Layer(ctx, H, d, g, orders, dense_prefix=dp)
    assert layer.N == N
    layer.set_masks(masks)
    out, zeroed = layer.forward_host(q, k, v, 0.0, pv_bits)
    layer.close()
    worst = 0.0
    for h in range(H):
        inv = prefix_inverse(oracle, g, orders[h], dp)
        ref_p, z_p = oracle.stream_engine(q[h][inv], k[h][inv], v[h][inv], None if masks is None else masks[h],
                                          pv_bits, qk_mode=1, dense_prefix=dp)
        ref = np.empty_like(ref_p)
        ref[inv] = ref_p
        zref = np.zeros(N, bool)
        zref[inv[z_p]] = True
        assert np.array_equal(zeroed[h].astype(bool), zref), h
        assert np.all(out[h][zref] == 0)
        worst = max(worst, rel_err(out[h], ref))
    print(f"[prefix] {grid}+{dp} H={H} d={d} pv={pv_bits}: max|dO|/max|O| = {worst:.3e}")
    return worst


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("dp", [1, 40, 64, 100, 130])
@pytest.mark.parametrize("pv_bits", [8, 4])
def test_dense_prefix_layer_matches_oracle(paro, ctx, oracle, d, dp, pv_bits):
    """AttnInputs::dense_prefix (attention.cpp:148-199): prefix rows dense over
    every key tile, dense key tiles kept and unquantized for every row (K4),
    the rest quantized from K4's running state (K3)."""
    grid, H, orders = "F:3,H:7,W:11", 2, ["WHF", "HFW"]
    kb = (231 + dp + 63) // 64
    masks = random_masks(H, kb, 0.35, 11 + dp, empty_row=kb - 1)
    assert run_prefix_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, dp, masks, pv_bits, 60 + dp) <= PREFIX_TOL


@pytest.mark.parametrize("d", [64, 128])
def test_dense_prefix_without_masks_and_all_empty(paro, ctx, oracle, d):
    grid, H, orders = "H:9,W:20", 2, ["HW", "WH"]  # 180 grid tokens
    dp = 77
    kb = (180 + dp + 63) // 64
    assert run_prefix_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, dp, None, 8, 90) <= PREFIX_TOL
    # every mask row empty: non-prefix rows see only the dense tiles
    masks = np.zeros((H, kb, kb), np.uint8)
    assert run_prefix_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, dp, masks, 8, 91) <= PREFIX_TOL


@pytest.mark.parametrize("dp", [1, 63, 200])
def test_single_head_api_dense_prefix(paro, ctx, oracle, dp):
    n, d = 300, 64
    q, k, v = randn(5, (n, d)), randn(6, (n, d)), randn(7, (n, d))
    kb = (n + 63) // 64
    mask = paro.BlockMask(kb, kb, 64, random_masks(1, kb, 0.5, dp)[0])
    res = ctx.quantized_blocked_attention(paro.AttnInputs(q, k, v, dense_prefix=dp), mask, paro.QuantConfig(8))
    ref, z = oracle.stream_engine(q, k, v, mask.bits, 8, qk_mode=1, dense_prefix=dp)
    assert rel_err(res.output, ref) <= PREFIX_TOL
    assert res.zeroed_rows == list(np.nonzero(z)[0])
    with pytest.raises(paro.ConfigError):
        ctx.quantized_blocked_attention(paro.AttnInputs(q, k, v, dense_prefix=n), mask, paro.QuantConfig(8))


@pytest.mark.parametrize("grid,d", [("H:3,W:5", 64), ("H:8,W:8", 64), ("H:5,W:13", 128), ("H:1,W:65", 64),
                                    ("F:1,H:9,W:14", 128), ("F:2,H:1,W:1", 64)])
@pytest.mark.parametrize("pv_bits", [8, 4])
def test_tiny_and_edge_shapes(paro, ctx, oracle, grid, d, pv_bits):
    """N < 64 (one partial block: K padding only), N = 64 (one full block, the
    unpaired q-block), N = 65 (a one-row tail block), one-token extents, N = 2."""
    g = paro.parse_grid(grid)
    N = g.token_count()
    kb = (N + 63) // 64
    orders = paro.enumerate_orders(g)[:2]
    H = len(orders)
    masks = np.ones((H, kb, kb), np.uint8)
    assert run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, masks, pv_bits, 101 + N) <= tol(d)
    assert run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, None, pv_bits, 102 + N) <= tol(d)


@pytest.mark.parametrize("d,scale", [(64, 0.5), (64, 0.01), (128, 0.3), (128, 2.0)])
def test_explicit_scale(paro, ctx, oracle, d, scale):
    """AttnInputs::scale != 0 (attention.cpp:26-28): sharp (2.0) and flat (0.01)
    softmax regimes exercise the exact row extremes and the P-group range."""
    grid, H, orders = "F:3,H:7,W:11", 2, ["WHF", "HFW"]
    masks = random_masks(H, 4, 0.5, 17)
    for pv in (8, 4):
        assert run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, orders, masks, pv, 200 + d, scale=scale) <= tol(d)


def test_set_masks_from_pmsk_blobs(paro, ctx):
    """paro_layer_set_masks_pmsk == set_masks on the deserialized bits (bit-identical
    output), and the reference's error classes for a bad blob / grid / block."""
    grid, H, d = "F:3,H:7,W:11", 2, 64
    N, kb = 231, 4
    q, k, v = make_inputs(H, N, d, 80)
    masks = random_masks(H, kb, 0.5, 5)
    blobs = [paro.serialize_mask(paro.BlockMask(kb, kb, 64, masks[h])) for h in range(H)]
    layer = paro.Layer(ctx, H, d, grid, ["WHF", "HFW"])
    layer.set_masks(masks)
    ref, zref = layer.forward_host(q, k, v, 0.0, 8)
    layer.set_masks_pmsk(blobs)
    out, z = layer.forward_host(q, k, v, 0.0, 8)
    assert np.array_equal(out, ref) and np.array_equal(z, zref)
    with pytest.raises(paro.FormatError):
        layer.set_masks_pmsk([blobs[0][:-1], blobs[1]])
    with pytest.raises(paro.ShapeError):
        layer.set_masks_pmsk([paro.serialize_mask(paro.BlockMask(3, 3, 64, np.ones((3, 3), np.uint8)))] * H)
    with pytest.raises(paro.ConfigError):
        layer.set_masks_pmsk([paro.serialize_mask(paro.BlockMask(kb, kb, 32, masks[0]))] * H)
    layer.close()


# ---- rotary embedding fused into K1 (paro_layer_set_rope)
def rope_tables(n, d, seed, interleaved=True):
    """3-axis-style rotary tables [n, d]: diffusers' real form (cos/sin repeated per pair) when
    `interleaved`, else independent values per element (exercises the general formula)."""
    rng = np.random.default_rng(seed)
    if interleaved:
        pos = np.arange(n, dtype=np.float64)[:, None]
        freqs = 1.0 / (10000.0 ** (np.arange(d // 2, dtype=np.float64) / (d // 2)))
        ang = np.repeat(pos * freqs[None, :] * (1.0 + rng.random((1, d // 2))), 2, axis=1)
    else:
        ang = rng.random((n, d)) * 6.3
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def np_rope(x, cos, sin, dp):
    """x' = x*cos + rotate_half(x)*sin on the grid tokens, fp32, every op rounded (numpy)."""
    y = x.copy()
    g = x[:, dp:]
    a, b = g[..., 0::2], g[..., 1::2]
    y[:, dp:, 0::2] = a * cos[None, :, 0::2] - b * sin[None, :, 0::2]
    y[:, dp:, 1::2] = b * cos[None, :, 1::2] + a * sin[None, :, 1::2]
    return y


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("dp", [0, 40])
@pytest.mark.parametrize("interleaved", [True, False])
def test_rope_fused_equals_rotate_then_layer(paro, ctx, oracle, d, dp, interleaved):
    grid, H, orders = ("F:3,H:7,W:11", 2, ["WHF", "FWH"])
    g = paro.parse_grid(grid)
    N = g.token_count() + dp
    q, k, v = make_inputs(H, N, d, 77)
    cos, sin = rope_tables(N - dp, d, 5, interleaved)
    masks = random_masks(H, (N + 63) // 64, 0.6, 9)
    a = paro.Layer(ctx, H, d, g, orders, dense_prefix=dp)
    a.set_masks(masks)
    a.set_rope(cos, sin)
    out_a, z_a = a.forward_host(q, k, v, 0.0, 8)
    b = paro.Layer(ctx, H, d, g, orders, dense_prefix=dp)
    b.set_masks(masks)
    qr, kr = np_rope(q, cos, sin, dp), np_rope(k, cos, sin, dp)
    out_b, z_b = b.forward_host(qr, kr, v, 0.0, 8)
    # bit-identical: the fused rotation rounds exactly like the fp32 pre-pass
    assert np.array_equal(out_a, out_b) and np.array_equal(z_a, z_b)
    # turning it off restores the plain layer
    a.set_rope(None, None)
    out_c, _ = a.forward_host(qr, kr, v, 0.0, 8)
    assert np.array_equal(out_c, out_b)
    a.close()
    b.close()
    if dp == 0:
        worst = 0.0
        for h in range(H):
            fwd, inv = oracle.make_perm(g.labels, g.extents, orders[h])
            ref, _ = oracle.paro_head(qr[h], kr[h], v[h], fwd, inv, masks[h], 8, qk_mode=1)
            worst = max(worst, rel_err(out_a[h], ref))
        assert worst <= EXACT_TOL, worst


def test_rope_errors(paro, ctx):
    g = paro.parse_grid("H:8,W:8")
    layer = paro.Layer(ctx, 1, 64, g, ["HW"], dense_prefix=3)
    cos, sin = rope_tables(67, 64, 1)
    with pytest.raises(paro.ShapeError):
        layer.set_rope(cos, sin)  # the tables cover the 64 grid tokens, not the 3 text tokens
    cos, sin = rope_tables(64, 64, 1)
    with pytest.raises(paro.ConfigError):
        layer.set_rope(cos, None)
    with pytest.raises(paro.ConfigError):  # the C ABI itself rejects half a table
        paro._check(paro._lib.paro_layer_set_rope(paro.P(layer.ptr), None, paro.P(paro._ptr(cos)), None))
    layer.close()
