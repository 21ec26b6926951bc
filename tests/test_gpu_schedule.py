"""Per-timestep mask schedules on the device (second half).

The reference consumes one PSCH schedule per head through load_schedule(path)
and MaskSchedule::at(t) (mask.cpp:132-140, 267-305): T/2 distinct early masks by
position and one shared mask for every later step. paro_layer_set_schedule
uploads every head's T/2 + 1 masks once; select_timestep(t) then makes at(t)
current either by a pointer switch (all entries' kept lists resident) or from a
double-buffered pair whose t+1 half K2 fills on a side stream while step t runs
(PAPER.md:576, 661-666). For every t (and for out-of-order jumps) the kept lists
must be those of the reference's at(t), and the layer output bit-identical to
set_masks(at(t)).
"""
import os

import numpy as np
import pytest

from conftest import randn

GRID, H, D = "F:3,H:7,W:11", 3, 64  # N = 231: ragged tail, kb = 4


def _reference_schedules(reference, tmp_path, T, density, kb, seed):
    """One PSCH file per head from the reference's build_schedule + save_schedule."""
    rng = np.random.default_rng(seed)
    blobs, paths = [], []
    for h in range(H):
        sums = rng.random((T, kb, kb)) + 2.0 * np.eye(kb)[None]
        path = str(tmp_path / f"sched_{seed}_{h}.psch")
        reference.build_and_save_schedule(sums, density, 64, path)
        with open(path, "rb") as f:
            blobs.append(f.read())
        paths.append(path)
    return blobs, paths


def test_serialize_schedule_matches_reference_writer(paro, reference, tmp_path):
    blobs, paths = _reference_schedules(reference, tmp_path, 5, 0.4, 4, 1)
    for blob, path in zip(blobs, paths):
        T = int.from_bytes(blob[4:8], "little")
        masks = [paro.schedule_at(blob, t) for t in range(T // 2)] + [paro.schedule_at(blob, T - 1)]
        assert paro.serialize_schedule(T, masks) == blob


@pytest.mark.gpu
@pytest.mark.parametrize("resident", [0, 2])
@pytest.mark.parametrize("T", [1, 5, 6])
def test_select_timestep_matches_at_t(paro, ctx, reference, tmp_path, resident, T):
    g = paro.parse_grid(GRID)
    N = g.token_count()
    kb = (N + 63) // 64
    orders = ["FHW", "WHF", "HFW"]
    blobs, paths = _reference_schedules(reference, tmp_path, T, 0.4, kb, T)
    q, k, v = randn(5, (H, N, D)), randn(6, (H, N, D)), randn(7, (H, N, D))
    sched = paro.Layer(ctx, H, D, g, orders)
    sched.set_schedule(blobs, resident)
    assert sched.schedule_info()[:2] == (T, T // 2 + 1)
    plain = paro.Layer(ctx, H, D, g, orders)
    order = list(range(T)) + list(reversed(range(T))) + [T - 1, 0]  # forward, backward and jumps
    for t in order:
        sched.select_timestep(t)
        at_t = np.stack([reference.schedule_at(p, t)[1] for p in paths])
        kept, total = sched.mask_stats()
        assert np.array_equal(kept, at_t.sum(axis=2).astype(np.uint32)), t
        assert total == int(at_t.sum())
        out_s, z_s = sched.forward_host(q, k, v, 0.0, 8)
        plain.set_masks(at_t)
        out_p, z_p = plain.forward_host(q, k, v, 0.0, 8)
        assert np.array_equal(out_s.view(np.uint32), out_p.view(np.uint32)), t
        assert np.array_equal(z_s, z_p)
    sched.close()
    plain.close()


@pytest.mark.gpu
def test_schedule_errors(paro, ctx, reference, tmp_path):
    g = paro.parse_grid(GRID)
    kb = (g.token_count() + 63) // 64
    layer = paro.Layer(ctx, H, D, g, ["FHW", "WHF", "HFW"])
    with pytest.raises(paro.ConfigError):
        layer.select_timestep(0)  # no schedule
    blobs, _ = _reference_schedules(reference, tmp_path, 4, 0.4, kb, 3)
    layer.set_schedule(blobs)
    with pytest.raises(paro.InputError):
        layer.select_timestep(4)  # at(t >= T) throws InputError (mask.cpp:133-135)
    other, _ = _reference_schedules(reference, tmp_path, 6, 0.4, kb, 4)
    with pytest.raises(paro.ShapeError):
        layer.set_schedule(blobs[:2] + other[2:])  # heads disagree on T
    with pytest.raises(paro.FormatError):
        layer.set_schedule([blobs[0][:-1]] + blobs[1:])  # truncated image
    # a plain set_masks ends the schedule
    layer.set_masks(np.ones((H, kb, kb), np.uint8))
    assert layer.schedule_info()[0] == 0
    layer.close()
