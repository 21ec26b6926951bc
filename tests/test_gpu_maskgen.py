"""K5 (the block-mask producer on the GPU) against the
reference library itself (oracle/_ref): fused apply_perm_map + block_sums of a
calibration attention map (bit-exact vs the reference's scalar kernels),
gen_mask (keep-order selection, ties, guard blocks, degenerate-row repair) and
build_schedule (distinct early masks + the shared mean-of-late mask)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def attn_map(rng, n):
    a = rng.random((n, n), dtype=np.float32) ** 4
    return (a / a.sum(axis=1, keepdims=True)).astype(np.float32)


@pytest.mark.parametrize("grid,order", [("F:3,H:7,W:11", "WHF"), ("H:20,W:33", "WH"), ("F:2,H:8,W:8", "HWF"),
                                        ("F:4,H:10,W:12", None)])
def test_perm_block_sums_bit_exact(paro, ctx, reference, grid, order):
    reference.select_kernels("scalar")
    g = paro.parse_grid(grid)
    n = g.token_count()
    m = attn_map(np.random.default_rng(n), n)
    plan = paro.make_perm(g, order) if order else None
    for block in (64, 16, 100):
        got = ctx.block_sums(m, block, plan)
        ref = reference.perm_block_sums(m, block, None if plan is None else plan.forward,
                                        None if plan is None else plan.inverse)
        assert got.view(np.uint64).tolist() == ref.view(np.uint64).tolist(), (grid, order, block)


def _sums(rng, k, ties):
    s = rng.random((k, k)) + 2.0 * np.eye(k)
    if ties:  # coarse values -> many equal sums (the (row, col) tie-break decides)
        s = np.round(s * 8) / 8
    return s


@pytest.mark.parametrize("k,density,guard,ties", [(11, 0.3, 0, False), (64, 0.3, 0, True), (275, 0.2, 0, False),
                                                  (40, 0.5, 3, True), (9, 1.0, 0, False), (33, 0.04, 0, True)])
def test_gen_mask_matches_reference(paro, ctx, reference, k, density, guard, ties):
    rng = np.random.default_rng(k * 7 + guard)
    stack = np.stack([_sums(rng, k, ties) for _ in range(3)])
    masks, reps = ctx.gen_mask(stack, density, 64, guard)
    for i in range(3):
        rc, bits, rep = reference.gen_mask(stack[i], density, 64, guard)
        assert rc == 0
        assert np.array_equal(masks[i].bits, bits), (k, density, guard, i)
        assert reps[i] == rep


def test_gen_mask_matches_golden(paro, ctx, kat):
    """The committed reference fixture (tests/golden/make_golden.py: gen_mask(U, 0.4, 16))."""
    m, rep = ctx.gen_mask(kat["gen_mask_sums"], 0.4, 16)
    assert np.array_equal(m.bits, kat["gen_mask_bits"])


@pytest.mark.parametrize("kb,density,seed", [(275, 0.3, 1), (275, 0.2, 2), (64, 0.3, 3), (2, 0.3, 4), (40, 0.05, 5)])
def test_gen_mask_ties_vs_reference(paro, ctx, reference, kb, density, seed):
    rng = np.random.default_rng(seed)
    sums = rng.random((kb, kb))
    sums[rng.random((kb, kb)) < 0.2] = 0.5  # ties exercise the (row, col) tie-break
    if seed != 5:
        sums += 2.0 * np.eye(kb)
    m, rep = ctx.gen_mask(sums, density, 64)
    rc, bits, rep2 = reference.gen_mask(sums, density, 64)
    assert rc == 0 and np.array_equal(m.bits, bits) and rep == rep2
    assert m.popcount() == int(np.ceil(density * kb * kb))


def test_gen_mask_repairs_empty_rows(paro, ctx, reference):
    k = 24
    s = np.full((k, k), 1.0)
    s[5, :] = 1e-9  # row 5 would keep nothing at this density
    s[17, :] = 1e-12
    s += np.random.default_rng(1).random((k, k)) * 1e-3
    m, rep = ctx.gen_mask(s, 0.1, 64)
    rc, bits, rep_ref = reference.gen_mask(s, 0.1, 64)
    assert rc == 0 and rep_ref >= 2
    assert np.array_equal(m.bits, bits) and rep == rep_ref


def test_gen_mask_errors(paro, ctx):
    s = np.random.default_rng(0).random((8, 8))
    with pytest.raises(paro.ConfigError):
        ctx.gen_mask(s, 0.0, 64)
    with pytest.raises(paro.ConfigError):
        ctx.gen_mask(s, 0.05, 64)  # fewer kept blocks than rows
    with pytest.raises(paro.ConfigError):
        ctx.gen_mask(s, 0.3, 64, guard_blocks=4)  # the guard alone exceeds the budget


@pytest.mark.parametrize("T", [1, 4, 5])
def test_build_schedule_matches_reference(paro, ctx, reference, tmp_path, T):
    k = 30
    rng = np.random.default_rng(T)
    sums = np.stack([_sums(rng, k, t % 2 == 0) for t in range(T)])
    masks, rep = ctx.build_schedule(sums, 0.25, 64)
    path = str(tmp_path / "s.psch")
    reference.build_and_save_schedule(sums, 0.25, 64, path)
    for t in range(T):
        rc, bits = reference.schedule_at(path, t)
        assert rc == 0
        want = masks[t] if t < T // 2 else masks[T // 2]
        assert np.array_equal(want.bits, bits), (T, t)


def _structured_maps(rng, grid_paro, count, prefix):
    """Maps with an axis-local structure so the orders score differently."""
    n = grid_paro.token_count()
    nf = n + prefix
    ext = grid_paro.extents
    coords = np.stack(np.unravel_index(np.arange(n), ext), axis=1).astype(np.float64)
    out = np.empty((count, nf, nf), np.float32)
    for c in range(count):
        w = rng.random(len(ext)) * 2.0
        d = np.zeros((n, n))
        for a in range(len(ext)):
            d += w[a] * np.abs(coords[:, None, a] - coords[None, :, a])
        core = np.exp(-d) * (0.5 + rng.random((n, n)))
        full = rng.random((nf, nf)) * 0.01
        full[prefix:, prefix:] = core
        full /= full.sum(axis=1, keepdims=True)
        out[c] = full
    return out


@pytest.mark.parametrize("grid,count,prefix,block", [("F:3,H:7,W:11", 2, 0, 64), ("F:3,H:7,W:11", 1, 5, 16),
                                                     ("H:20,W:33", 2, 0, 64), ("F:4,H:6,W:5", 3, 3, 8)])
def test_select_permutation_matches_reference(paro, ctx, reference, grid, count, prefix, block):
    reference.select_kernels("scalar")
    g = paro.parse_grid(grid)
    maps = _structured_maps(np.random.default_rng(count + prefix), g, count, prefix)
    for eps, sigma, alpha in ((1e-3, 0.9, 0.5), (2e-3, 0.5, 0.8)):
        o1, s1, c1 = ctx.select_permutation(maps, g, block, eps, sigma, alpha, prefix)
        o2, s2, c2 = reference.select_permutation(maps, grid, block, eps, sigma, alpha, prefix)
        assert o1 == o2
        assert s1.view(np.uint64).tolist() == s2.view(np.uint64).tolist(), (grid, eps, sigma, alpha)
        assert c1 == c2


def test_select_permutation_errors(paro, ctx):
    g = paro.parse_grid("H:8,W:8")
    m = np.ones((1, 64, 64), np.float32) / 64
    with pytest.raises(paro.ConfigError):
        ctx.select_permutation(m, g, 64, eps=0.0)
    with pytest.raises(paro.ConfigError):
        ctx.select_permutation(m, g, 64, sigma=1.5)
    with pytest.raises(paro.ConfigError):
        ctx.select_permutation(m, g, 64, alpha=-0.1)
