"""N>1 path on CPU: world_size-2 gloo processes each own a head shard
(paro_b200.sharding), compute it (with the CPU oracle -- there is no GPU here),
and reassemble the layer with the same all-gather bench/tests use over NCCL.
The gathered layer must equal the single-process layer bit for bit, and the
max-over-ranks timing reduction must return the slowest rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


GRID, H, D = "F:2,H:8,W:8", 4, 64


def _layer_inputs():
    rng = np.random.default_rng(5)
    q, k, v = (rng.standard_normal((H, 128, D)).astype(np.float32) for _ in range(3))
    masks = np.ones((H, 2, 2), np.uint8)
    masks[:, 0, 1] = 0
    return q, k, v, masks


def _head_outputs(heads):
    import paro_b200 as paro
    from oracle.pyoracle import Oracle

    orc = Oracle()
    g = paro.parse_grid(GRID)
    orders = paro.enumerate_orders(g)
    q, k, v, masks = _layer_inputs()
    outs = []
    for h in heads:
        plan = paro.make_perm(g, orders[h % len(orders)])
        o, _ = orc.paro_head(q[h], k[h], v[h], plan.forward, plan.inverse, masks[h], 8, qk_mode=1)
        outs.append(o)
    return np.stack(outs)


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    from paro_b200.sharding import gather_layer, max_over_ranks, shard_heads

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_heads(H, world, rank)
    local = torch.from_numpy(_head_outputs(mine))
    full = gather_layer(local)
    slowest = max_over_ranks(1.0 + rank)
    if rank == 0:
        np.save(result_path, full.numpy())
        np.save(result_path + ".t.npy", np.array([slowest]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_heads_partition():
    from paro_b200.sharding import shard_heads

    for heads, world in [(48, 1), (48, 2), (48, 8), (40, 8), (24, 4)]:
        parts = [shard_heads(heads, world, r) for r in range(world)]
        assert sum(parts, []) == list(range(heads))
    with pytest.raises(ValueError):
        shard_heads(48, 5, 0)


def test_gloo_world2_gather_equals_single_process(tmp_path):
    world = 2
    out = str(tmp_path / "layer.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    gathered = np.load(out)
    single = _head_outputs(list(range(H)))
    assert np.array_equal(gathered.view(np.uint32), single.view(np.uint32))
    assert float(np.load(out + ".t.npy")[0]) == 2.0
