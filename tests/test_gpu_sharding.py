"""The head-sharded multi-GPU path with the GPU layer itself.

* world-size 2, each rank a process with its own paro.Context on device
  (rank % visible devices) running its contiguous head shard through K1/K2/K3,
  the shards reassembled with sharding.gather_layer: over gloo (ranks may share
  the one GPU of a single-GPU box) and over NCCL (needs >= 2 GPUs, else skipped).
  The gathered layer equals the single-process layer bit for bit.
* `python bench.py --gpus 2` (no torchrun) spawns its two ranks itself and
  reports n_gpus 2 (gloo here so it also runs on a one-GPU box).
* the C++ host-thread path: one paro_ctx per device from std::threads
  (tests/cpp/multidevice_test.cpp), bit-identical to one context.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("F:13,H:30,W:45", 4, 64, 0.3, 8), ("H:64,W:64", 4, 128, 0.3, 4)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _layer(heads, grid, d, density, bits, device=0):
    import bench
    import paro_b200 as paro

    g = paro.parse_grid(grid)
    N = g.token_count()
    ctx = paro.Context(device)
    orders, q, k, v, masks = bench.workload_ours(paro, ctx, heads, grid, N, d, density, "random")
    layer = paro.Layer(ctx, len(heads), d, g, orders)
    layer.set_masks(masks)
    out, zeroed = layer.forward_host(q, k, v, 0.0, bits)
    layer.close()
    ctx.close()
    return out, zeroed


def _worker(rank, world, port, backend, case, result_path):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paro_b200.sharding import gather_layer, shard_heads

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    grid, H, d, density, bits = case
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    out, zeroed = _layer(shard_heads(H, world, rank), grid, d, density, bits, dev)
    local = torch.from_numpy(out)
    if backend == "nccl":
        local = local.cuda()
    full = gather_layer(local).cpu().numpy()
    if rank == 0:
        np.save(result_path, full)
    dist.barrier()
    dist.destroy_process_group()


def _run_world2(backend, case, tmp_path):
    out = str(tmp_path / f"layer_{backend}.npy")
    mp.spawn(_worker, args=(2, _free_port(), backend, case, out), nprocs=2, join=True)
    gathered = np.load(out)
    grid, H, d, density, bits = case
    single, _ = _layer(list(range(H)), grid, d, density, bits)
    assert gathered.shape == single.shape
    assert np.array_equal(gathered.view(np.uint32), single.view(np.uint32))


@pytest.mark.parametrize("case", CASES)
def test_gpu_layer_world2_gloo_bit_exact(case, tmp_path):
    _run_world2("gloo", case, tmp_path)


@pytest.mark.parametrize("case", CASES[:1])
def test_gpu_layer_world2_nccl_bit_exact(case, tmp_path):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("NCCL world-2 needs >= 2 GPUs (this box has one; the gloo test covers the sharded GPU path)")
    _run_world2("nccl", case, tmp_path)


def test_bench_gpus2_spawns_its_ranks():
    env = dict(os.environ, PARO_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3",
                        "--no-e2e", "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["parallelism"].startswith("head-shard x2")


def test_bench_rejects_mismatched_world():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stdout + r.stderr)


@pytest.mark.parametrize("args", [["F:13,H:30,W:45", "8", "64", "8"], ["F:21,H:45,W:80", "2", "128", "4"]])
def test_cpp_host_threads_one_context_per_device(args):
    binary = os.path.join(ROOT, "tests", "cpp", "_build", "multidevice_test")
    if not os.path.exists(binary):
        pytest.skip("multidevice_test not built")
    r = subprocess.run([binary] + args, capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
