#!/usr/bin/env python
"""bench.py -- PARO sparse-quantized attention layer on B200 (BASELINE.json metric).

Metric: "PARO attn ms/layer + effective INT8 TOPS (CogVideoX N=17550, 48h)".
  value        = effective TOPS over the whole job (all ranks): algorithmic ops of
                 the kept tiles (4*d*rows*cols per kept 64x64 block, padding
                 excluded) / max-over-ranks device time of one layer step.
  ms_per_step  = ms/layer.
A step = one pass of the hot path over one layer: K2 (mask -> kept lists, masks
resident in HBM) + K1 (PARO gather + Q/K/V quantize) + K3 (block-sparse INT8
attention + inverse permute). Heads are sharded across ranks (no collective on
the data path; "scaling": "strong" -- the layer is fixed, ranks split heads).
e2e: the same metric through the C-ABI host call paro_layer_forward_host (pinned
host Q/K/V in, O out; H2D/D2H inside the timed region).

--impl reference: the reference's own CPU implementation of the path
(quantized_blocked_attention + permutes, compiled from the reference sources into
oracle/_ref) on the host cores, bounded sample of heads, same metric.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (grid, heads, d, density, pv_bits, description)
    "c1": ("F:2,H:8,W:8", 2, 64, 0.3, 8, "small synthetic F2xH8xW8, 2 heads, d=64, 30% (block 64 -> 50%), INT8/INT8"),
    "c2": ("F:13,H:30,W:45", 48, 64, 0.3, 8, "CogVideoX-5B N=17550 (13x30x45), 48 heads, d=64, density 0.3, INT8 QK / INT8 PV"),
    "c3": ("F:13,H:30,W:45", 48, 64, 0.2, 4, "CogVideoX-5B N=17550, 48 heads, d=64, density 0.2, INT8 QK / INT4 PV"),
    "c4": ("H:64,W:64", 24, 128, 0.3, 8, "Flux.1-dev N=4096 (64x64), 24 heads, d=128, density 0.3, INT8/INT8"),
    "c4i4": ("H:64,W:64", 24, 128, 0.3, 4, "Flux.1-dev N=4096 (64x64), 24 heads, d=128, density 0.3, INT8/INT4"),
    "c5": ("F:21,H:45,W:80", 40, 128, 0.2, 4, "Wan-2.1-14B N=75600 (21x45x80), 40 heads, d=128, density 0.2, INT8 QK / INT4 PV"),
}


def _softmax_roofline(scores, k3_ms, clk):
    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0
    achieved = scores / (k3_ms * 1e-3) / 1e12
    peak = 16 * 148 * mhz * 1e6 / 1e12
    return {"bound": "mufu_ex2", "kernel": "k3_attention", "achieved": achieved, "peak": peak,
            "unit": "Tscores/s", "frac": achieved / peak, "scores_per_launch": int(scores),
            "note": "kept (row, key) pairs / K3 time vs 16 ex2 / clk / SM x 148 SMs"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS) + ["maskgen", "permsel"],
                    help="maskgen: the GPU mask producer (K5) on one c2-shaped calibration map instead of the layer")
    ap.add_argument("--mask-family", default="random", choices=["random", "banded"])
    ap.add_argument("--dense-prefix", type=int, default=0,
                    help="diagnostic: text tokens in front of the grid (K4 + K3); BASELINE configs use 0")
    ap.add_argument("--rope", action="store_true",
                    help="diagnostic: rotary embedding fused into K1 (paro_layer_set_rope); BASELINE configs do not rotate")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / baseline / clocks)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- workload
def head_orders(paro, grid, heads):
    """Per-head order = enumerate_perms(grid)[head % ndim!]."""
    orders = paro.enumerate_orders(grid)
    return [orders[h % len(orders)] for h in range(heads)]


def head_inputs(paro, h, N, d):
    """Seeded N(0,1): MT19937-64 + Box-Muller, seed 1000 + 3*head + {0,1,2}."""
    return [paro.synth_randn(1000 + 3 * h + i, N * d).reshape(N, d) for i in range(3)]


def head_mask(paro, h, kb, density, family):
    rng = np.random.default_rng(7919 * (h + 1))
    if family == "random":  # M1: U[0,1) + 2*I (test_mask.cpp:28-37 shape)
        sums = rng.random((kb, kb)) + 2.0 * np.eye(kb)
    else:  # M2: exp(-|i-j|/w) + 0.05*U, w = density*k/2
        w = max(density * kb / 2.0, 1.0)
        i = np.arange(kb)
        sums = np.exp(-np.abs(i[:, None] - i[None, :]) / w) + 0.05 * rng.random((kb, kb))
    return paro.gen_mask(sums, density, 64)[0].bits


def kept_ops(mask, N, d):
    """4*d*sum over kept blocks of true rows x true cols."""
    kb = mask.shape[0]
    ext = np.full(kb, 64, np.int64)
    ext[-1] = N - 64 * (kb - 1)
    return int(4 * d * (ext[:, None] * ext[None, :] * (mask != 0)).sum())


def build_inputs(paro, heads, N, d, density, family, threads=8):
    from concurrent.futures import ThreadPoolExecutor

    kb = (N + 63) // 64
    q = np.empty((len(heads), N, d), np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)
    masks = np.empty((len(heads), kb, kb), np.uint8)

    def one(i):
        h = heads[i]
        q[i], k[i], v[i] = head_inputs(paro, h, N, d)
        masks[i] = head_mask(paro, h, kb, density, family)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(len(heads))))
    return q, k, v, masks


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def ncu_traffic(cfg, kernel):
    """DRAM bytes per launch of `kernel` at config `cfg` from a committed ncu capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            v = json.load(f).get(cfg, {}).get(kernel)
        return float(v) if v is not None else None
    except Exception:
        return None


def _scaled(v, f):
    """A whole-layer capture scaled to this rank's head shard (per launch, like `achieved`)."""
    return None if v is None else v * f


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), float(mp["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- CPU baseline (reference)
def cpu_reference_sample(cfg_name, threads, max_heads=None, steps=1, warmup=0, budget_s=120.0):
    """The reference's own CPU chain (oracle/_ref) on a bounded sample of heads
    (about one head per thread), repeated: `warmup` untimed samples (at most 1)
    and up to `steps` timed ones, stopping once `budget_s` of timed work is
    done so the whole run stays within a few minutes."""
    from oracle.pyoracle import Reference, have_reference

    import paro_b200 as paro

    if not have_reference():
        return None
    grid_text, H, d, density, bits, _ = CONFIGS[cfg_name]
    g = paro.parse_grid(grid_text)
    N = g.token_count()
    ref = Reference()
    ref.select_kernels("auto")
    threads = threads or os.cpu_count() or 1
    # bounded sample: about one head per thread, sized for ~10-30 s of CPU work
    per_head_ops = None
    n_run = min(H, max_heads or threads)
    heads = list(range(n_run))
    q, k, v, masks = build_inputs(paro, heads, N, d, density, "random")
    orders = head_orders(paro, g, H)[:n_run]
    for _ in range(min(warmup, 1)):
        ref.run_heads(grid_text, q, k, v, orders, masks, bits, 0.0, threads)
    secs, done = 0.0, 0
    while done < max(1, steps) and (done == 0 or secs < budget_s):
        _, t = ref.run_heads(grid_text, q, k, v, orders, masks, bits, 0.0, threads)
        secs += t
        done += 1
    ops = done * sum(kept_ops(masks[i], N, d) for i in range(n_run))
    per_head_ops = ops / (done * n_run)
    return {
        "value": ops / secs / 1e12,
        "unit": "TOPS",
        "cores": threads,
        "kind": "reference",
        "sample": f"{n_run} of {H} heads ({cfg_name}) on {threads} threads per step, {done} step(s), "
                  f"{secs:.1f} s wall; layer time extrapolated {H * per_head_ops / (ops / secs):.1f} s",
        "seconds": secs,
        "steps": done,
        "warmup": min(warmup, 1),
        "layer_seconds_extrapolated": H * per_head_ops / (ops / secs),
    }


# ----------------------------------------------------------------------------- main
def maskgen_main(args):
    """K5 on one CogVideoX-shaped calibration map (N = 17550, 1.23 GB fp32): fused
    apply_perm_map + block_sums (HBM-bound: the map is read once) and gen_mask on
    the resulting 275 x 275 grid; the reference's CPU path (apply_perm_map +
    block_sums, oracle/_ref) timed on the same map."""
    import ctypes

    import torch

    import paro_b200 as paro

    g = paro.parse_grid("F:13,H:30,W:45")
    N = g.token_count()
    k = (N + 63) // 64
    plan = paro.make_perm(g, "WHF")
    torch.manual_seed(0)
    dmap = torch.rand((N, N), dtype=torch.float32, device="cuda")
    dinv = torch.from_numpy(plan.inverse.astype(np.int32)).cuda()
    dsum = torch.empty((k, k), dtype=torch.float64, device="cuda")
    dbits = torch.empty((k, k), dtype=torch.uint8, device="cuda")
    ctx = paro.Context(0)
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    lib = paro._lib

    def sums():
        paro._check(lib.paro_perm_block_sums_device(ctypes.c_void_p(ctx.ptr), sp, ctypes.c_void_p(dmap.data_ptr()),
                                                    ctypes.c_uint32(N), ctypes.c_void_p(dinv.data_ptr()),
                                                    ctypes.c_uint32(64), ctypes.c_void_p(dsum.data_ptr())))

    for _ in range(max(args.warmup, 3)):
        sums()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        sums()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    rep = (ctypes.c_uint32 * 1)()
    t0 = time.perf_counter()
    paro._check(lib.paro_gen_mask_device(ctypes.c_void_p(ctx.ptr), sp, ctypes.c_void_p(dsum.data_ptr()),
                                         ctypes.c_uint32(1), ctypes.c_uint32(k), ctypes.c_uint32(k),
                                         ctypes.c_double(0.3), ctypes.c_uint32(64), ctypes.c_uint32(0),
                                         ctypes.c_void_p(dbits.data_ptr()), rep))
    gm_ms = (time.perf_counter() - t0) * 1e3
    bytes_ = N * N * 4.0
    peak = measured_peaks()[0]
    line = {"metric": "K5 mask producer: permuted block_sums of one calibration map (GB/s of map read)",
            "value": bytes_ / ms / 1e6, "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "dtype_detail": "fp32 map in, fp64 block sums (reference order)",
            "data": "synthetic U[0,1) map on the device", "config": {"workload": f"N={N} (F:13,H:30,W:45) order WHF, block 64"},
            "roofline": {"bound": "hbm", "achieved": bytes_ / ms / 1e6, "peak": peak, "unit": "GB/s",
                         "frac": (bytes_ / ms / 1e6) / peak if peak else None, "traffic": None},
            "gen_mask_ms_incl_sync": gm_ms}
    try:
        from oracle.pyoracle import Reference, have_reference

        if have_reference():
            r = Reference()
            r.select_kernels("auto")
            m = dmap.cpu().numpy()
            t0 = time.perf_counter()
            r.perm_block_sums(m, 64, plan.forward, plan.inverse)
            cpu_s = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": bytes_ / cpu_s / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
                                    "sample": "the same map: apply_perm_map + block_sums (main.cpp:236-238)"}
    except Exception as e:  # the CPU leg is a reported baseline only
        line["cpu_baseline"] = {"unavailable": str(e)[:120]}
    print(json.dumps(line))


def permsel_main(args):
    """select_permutation on one CogVideoX-shaped calibration
    map: 6 candidate orders, each a fused permuted-block pass (sum|a|, max|a|,
    #|a|<eps) over the 1.23 GB map; the reference CPU path (apply_perm_map +
    m_sparse + m_quant per order) timed on the same map for a bounded subset."""
    import ctypes

    import torch

    import paro_b200 as paro

    grid = "F:13,H:30,W:45"
    N = paro.parse_grid(grid).token_count()
    torch.manual_seed(0)
    dmap = torch.rand((N, N), dtype=torch.float32, device="cuda")
    ctx = paro.Context(0)
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    orders = ctypes.create_string_buffer(32)
    scores = np.zeros((6, 5), np.float64)
    nperm, chosen = ctypes.c_int(), ctypes.c_int()

    def run():
        paro._check(paro._lib.paro_select_permutation_device(
            ctypes.c_void_p(ctx.ptr), sp, ctypes.c_void_p(dmap.data_ptr()), ctypes.c_uint32(1), grid.encode(),
            ctypes.c_uint32(64), ctypes.c_float(1e-3), ctypes.c_float(0.9), ctypes.c_float(0.5), ctypes.c_uint32(0),
            orders, scores.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nperm), ctypes.byref(chosen)))

    for _ in range(max(args.warmup, 3)):
        run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()  # synchronises internally (host-side final reductions)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    bytes_ = N * N * 4.0 * nperm.value
    peak = measured_peaks()[0]
    line = {"metric": "select_permutation of one c2 calibration map, all candidate orders (ms, wall incl. host reductions)",
            "value": ms, "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "dtype_detail": "fp32 map in, fp64 statistics",
            "data": "synthetic U[0,1) map on the device",
            "config": {"workload": f"N={N} ({grid}), {nperm.value} orders, block 64, eps 1e-3, sigma 0.9, alpha 0.5"},
            "roofline": {"bound": "hbm", "achieved": bytes_ / ms / 1e6, "peak": peak, "unit": "GB/s",
                         "frac": bytes_ / ms / 1e6 / peak if peak else None, "traffic": None}}
    try:
        from oracle.pyoracle import Reference, have_reference

        if have_reference():
            r = Reference()
            r.select_kernels("auto")
            m = dmap.cpu().numpy()
            g = paro.parse_grid(grid)
            plan = paro.make_perm(g, "WHF")
            t0 = time.perf_counter()
            r.perm_block_sums(m, 64, plan.forward, plan.inverse)  # one order's apply_perm_map + block pass
            one = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": one * nperm.value * 1e3, "unit": "ms", "cores": 1, "kind": "reference",
                                    "sample": "apply_perm_map + block_sums for 1 order on the same map, x6 orders "
                                              "(m_sparse/m_quant passes not included: a lower bound)"}
    except Exception as e:
        line["cpu_baseline"] = {"unavailable": str(e)[:120]}
    print(json.dumps(line))


def main():
    args = parse_args()
    if args.config == "maskgen":
        return maskgen_main(args)
    if args.config == "permsel":
        return permsel_main(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    grid_text, H, d, density, pv_bits, desc = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference_sample(args.config, args.cpu_threads, None, args.steps, args.warmup)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparo_ref.so not built"}))
            return
        line = {
            "impl": "reference", "metric": "PARO attn ms/layer + effective INT8 TOPS (CogVideoX N=17550, 48h)",
            "value": r["value"], "unit": "TOPS", "n_gpus": args.gpus, "steps": r["steps"], "warmup": r["warmup"],
            "ms_per_step": r["layer_seconds_extrapolated"] * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "dtype_detail": "reference CPU semantics: fp64 QK, int8/int4 P,V", "data": "synthetic",
            "config": {"workload": desc, "heads": H, "grid": grid_text, "head_dim": d, "density": density,
                       "pv_bits": pv_bits, "mask_family": "random"},
            "cpu_baseline": {k_: r[k_] for k_ in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    import torch

    import paro_b200 as paro

    # one process per GPU; PARO_BENCH_BACKEND=gloo lets several ranks share one
    # GPU to exercise the multi-rank path on a single-GPU box (test only)
    backend = os.environ.get("PARO_BENCH_BACKEND", "nccl")
    dev = local_rank % max(1, torch.cuda.device_count()) if backend != "nccl" else local_rank
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    ctx = paro.Context(dev)
    g = paro.parse_grid(grid_text)
    N = g.token_count() + args.dense_prefix
    kb = (N + 63) // 64
    from paro_b200.sharding import shard_heads

    my_heads = shard_heads(H, world, rank)  # no data-path collective
    hpr = len(my_heads)
    orders_all = head_orders(paro, g, H)
    q, k, v, masks = build_inputs(paro, my_heads, N, d, density, args.mask_family)
    my_ops = sum(kept_ops(masks[i], N, d) for i in range(hpr))
    total_ops = my_ops
    if dist:
        t = torch.tensor([my_ops], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        total_ops = float(t.item())

    layer = paro.Layer(ctx, hpr, d, g, [orders_all[h] for h in my_heads], dense_prefix=args.dense_prefix)
    if args.rope:  # diffusers-style real tables, one row per grid token (L2-resident across heads)
        ang = np.repeat(np.arange(g.token_count(), dtype=np.float64)[:, None]
                        * (10000.0 ** (-np.arange(d // 2) / (d // 2)))[None, :], 2, axis=1)
        layer.set_rope(np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32))
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    dq = torch.from_numpy(q).cuda()
    dk = torch.from_numpy(k).cuda()
    dv = torch.from_numpy(v).cuda()
    dmask = torch.from_numpy(masks).cuda()
    dout = torch.empty_like(dq)
    dzero = torch.empty((hpr, N), dtype=torch.uint8, device="cuda")

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(events=None):
        if events:
            events[0].record(stream)
        layer.set_masks_device(dmask.data_ptr(), sp)
        if events:
            events[1].record(stream)
        layer.reorder_quantize(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), pv_bits, sp)
        if events:
            events[2].record(stream)
        layer.attention(0.0, pv_bits, dout.data_ptr(), dzero.data_ptr(), sp)
        if events:
            events[3].record(stream)

    for _ in range(max(args.warmup, 3 if not args.profile else 1)):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(dev)
    if not args.profile:
        clocks.start()
        time.sleep(0.2)
    # timed region: K steps, barrier + synchronize on both sides, per-kernel events
    per = [[ev() for _ in range(4)] for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = ev(), ev()
    t0.record(stream)
    for i in range(args.steps):
        step(per[i])
    t1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_total = t0.elapsed_time(t1)
    k2_ms = sum(e[0].elapsed_time(e[1]) for e in per) / args.steps
    k1_ms = sum(e[1].elapsed_time(e[2]) for e in per) / args.steps
    k3_ms = sum(e[2].elapsed_time(e[3]) for e in per) / args.steps
    ms_step = ms_total / args.steps
    if dist:
        t = torch.tensor([ms_step, k1_ms, k2_ms, k3_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, k1_ms, k2_ms, k3_ms = [float(x) for x in t.tolist()]
    clk = clocks.stop() if not args.profile else None

    # e2e through the public C-ABI host call (pinned host buffers)
    e2e = None
    if not args.no_e2e and not args.profile:
        hq, hk, hv = (paro.HostBuffer(q.shape, np.float32) for _ in range(3))
        hq.array[...] = q
        hk.array[...] = k
        hv.array[...] = v
        hout = paro.HostBuffer(q.shape, np.float32)
        hz = paro.HostBuffer((hpr, N), np.uint8)
        hm = paro.HostBuffer(masks.shape, np.uint8) # the step's masks come from the host too
        hm.array[...] = masks
        for _ in range(2):
            layer.set_masks(hm.array, sp, sync=False)
            layer.forward_host(hq.array, hk.array, hv.array, 0.0, pv_bits, hout.array, hz.array, sp)
        e_steps = max(3, min(args.steps, 10))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(e_steps):
            layer.set_masks(hm.array, sp, sync=False)
            layer.forward_host(hq.array, hk.array, hv.array, 0.0, pv_bits, hout.array, hz.array, sp)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / e_steps
        if dist:
            t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": total_ops / (e_ms * 1e-3) / 1e12, "unit": "TOPS", "ms_per_layer": e_ms,
               "h2d_bytes_per_step": int(3 * q.nbytes + masks.nbytes) * world,
               "d2h_bytes_per_step": int(q.nbytes + hz.array.nbytes) * world}

    # rooflines (rank-0 numbers; per launch = per layer shard)
    hbm_peak, bf16_peak, peak_src = measured_peaks()
    int8_peak = 2.0 * bf16_peak  # kind::i8 issues at 2x the kind::f16 rate on tcgen05
    k3_tops = my_ops / (k3_ms * 1e-3) / 1e12
    k1_bytes = hpr * (3 * N * d * 4 + 3 * kb * 64 * d + kb * (4 + d) * 4 + kb * 4 * (d // 64))
    k1_gbs = k1_bytes / (k1_ms * 1e-3) / 1e9
    density_kept = float(np.mean([m.mean() for m in masks]))

    line = {
        "metric": "PARO attn ms/layer + effective INT8 TOPS (CogVideoX N=17550, 48h)",
        "value": total_ops / (ms_step * 1e-3) / 1e12,
        "unit": "TOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int8",
        "dtype_detail": "QK s8*s8->s32 and PV u8(u4 codes)*s8->s32 on tcgen05; fp32 softmax / dequant, fp64 row extremes",
        "data": "synthetic N(0,1) Q/K/V (MT19937-64 Box-Muller), gen_mask masks",
        "config": {
            "workload": desc, "grid": grid_text, "heads": H, "tokens": N, "head_dim": d, "density": density,
            "kept_density": round(density_kept, 5), "pv_bits": pv_bits, "mask_family": args.mask_family,
            **({"dense_prefix": args.dense_prefix} if args.dense_prefix else {}),
            **({"rope": "fused into K1 (cos/sin tables read per row)"} if args.rope else {}),
            "parallelism": f"head-shard x{world} (no data-path collective)",
            "l2": f"inputs {3 * q.nbytes * world / 1e6:.0f} MB > 126 MB L2 (no flush needed)",
        },
        "ms_per_layer": ms_step,
        "kernels_ms": {"k2_mask_lists": k2_ms, "k1_reorder_quantize": k1_ms, "k3_attention": k3_ms},
        "roofline": {
            "bound": "tensor", "kernel": "k3_attention", "achieved": k3_tops, "peak": int8_peak, "unit": "TOPS",
            "frac": k3_tops / int8_peak,
            "traffic": None if args.dense_prefix else _scaled(ncu_traffic(args.config, "k3_attention"), hpr / H),
            "peak_source": f"2x bf16_tflops {bf16_peak} ({peak_src}, MEASURED_PEAKS.json): dense INT8 tcgen05 rate",
            "algorithmic_ops_per_launch": my_ops,
        },
        # the softmax ceiling the tensor-pipe fraction hides: one ex2 per kept score on the
        # MUFU (16 / clk / SM), at the SM clock sampled during the run
        "roofline_softmax": _softmax_roofline(my_ops / (4 * d), k3_ms, clk),
        "roofline_k1": {"bound": "hbm", "kernel": "k1_reorder_quantize", "achieved": k1_gbs, "peak": hbm_peak,
                        "unit": "GB/s", "frac": k1_gbs / hbm_peak, "algorithmic_bytes_per_launch": k1_bytes,
                        "traffic": _scaled(ncu_traffic(args.config, "k1_reorder_quantize"), hpr / H)},
        # per step: K2 (3 kernels) + K1 + K3, plus K4a + K4 + combine with a dense prefix
        "gpu_launches": (5 + (3 if args.dense_prefix else 0)) * args.steps,
        "clocks": clk,
        "e2e": e2e,
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        try:
            cb = cpu_reference_sample(args.config, args.cpu_threads)
        except Exception as ex:  # the baseline must not kill the bench line
            cb = {"error": str(ex)}
        if cb is not None:
            line["cpu_baseline"] = {k_: cb[k_] for k_ in ("value", "unit", "cores", "kind", "sample") if k_ in cb} \
                if "error" not in cb else cb
    if rank == 0:
        print(json.dumps(line))
    layer.close()
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
