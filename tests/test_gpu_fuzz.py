"""Seeded random layers on the GPU vs the oracle: grids (2-D / 3-D, ragged), head
counts, per-head orders, densities (incl. empty rows / fully dense), INT8 / INT4
P.V, d = 64 / 128, explicit scales and input magnitudes. Every case must be
bit-exact in its P codes (max|dO|/max|O| <= 1e-5) with identical zeroed rows."""
import numpy as np
import pytest

from test_gpu_parity import EXACT_TOL, random_masks, run_layer_vs_oracle

pytestmark = pytest.mark.gpu


def case(seed):
    rng = np.random.default_rng(seed)
    if rng.random() < 0.5:
        grid = f"H:{rng.integers(1, 40)},W:{rng.integers(1, 60)}"
    else:
        grid = f"F:{rng.integers(1, 6)},H:{rng.integers(1, 12)},W:{rng.integers(1, 16)}"
    d = int(rng.choice([64, 128]))
    pv = int(rng.choice([8, 4]))
    density = float(rng.choice([0.0, 0.15, 0.4, 1.0]))
    scale = float(rng.choice([0.0, 0.05, 0.5]))
    return grid, d, pv, density, scale


@pytest.mark.parametrize("seed", list(range(64)))
def test_random_layer_matches_oracle(paro, ctx, oracle, seed):
    grid, d, pv, density, scale = case(1000 + seed)
    g = paro.parse_grid(grid)
    N = g.token_count()
    kb = (N + 63) // 64
    orders = paro.enumerate_orders(g)
    rng = np.random.default_rng(seed)
    H = int(rng.integers(1, 4))
    ords = [orders[int(rng.integers(0, len(orders)))] for _ in range(H)]
    masks = random_masks(H, kb, density, seed, empty_row=(kb - 1 if density == 0.15 else None))
    err = run_layer_vs_oracle(paro, ctx, oracle, grid, H, d, ords, masks, pv, 500 + seed, scale=scale)
    assert err <= EXACT_TOL, (grid, d, pv, density, scale, err)


@pytest.mark.parametrize("seed", list(range(16)))
def test_random_dense_prefix_layer_matches_oracle(paro, ctx, oracle, seed):
    """Random text-prefix lengths (K4a / K4 / combine + K3 from K4's state)."""
    from test_gpu_parity import PREFIX_TOL, run_prefix_layer_vs_oracle

    grid, d, pv, density, _ = case(2000 + seed)
    g = paro.parse_grid(grid)
    rng = np.random.default_rng(seed + 77)
    dp = int(rng.integers(1, 300))
    N = g.token_count() + dp
    kb = (N + 63) // 64
    orders = paro.enumerate_orders(g)
    H = int(rng.integers(1, 3))
    ords = [orders[int(rng.integers(0, len(orders)))] for _ in range(H)]
    masks = random_masks(H, kb, max(density, 0.1), seed + 5)
    err = run_prefix_layer_vs_oracle(paro, ctx, oracle, grid, H, d, ords, dp, masks, pv, 700 + seed)
    assert err <= PREFIX_TOL, (grid, dp, d, pv, err)
