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

METRIC = "PARO attn ms/layer + effective INT8 TOPS (CogVideoX N=17550, 48h)"

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
    ap.add_argument("--schedule", type=int, default=0, metavar="T",
                    help="per-timestep mask schedule of T steps (PSCH per head, paro_layer_set_schedule): step i "
                         "runs timestep i %% T with its kept lists resident, no K2 in the step")
    ap.add_argument("--schedule-prefetch", action="store_true",
                    help="with --schedule: two list buffers, K2 of t+1 on a side stream during step t")
    ap.add_argument("--v-packed", action="store_true",
                    help="INT4 V nibble-packed in HBM, unpacked to i8 in shared memory by K3 (paro_layer_set_v_packing)")
    ap.add_argument("--rope", action="store_true",
                    help="diagnostic: rotary embedding fused into K1 (paro_layer_set_rope); BASELINE configs do not rotate")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / baseline / clocks)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- workload
# The same inputs in both arms, built by each arm's own library: the GPU arm
# with the product (paro_b200: MT19937-64 stream, K5 gen_mask on the device),
# the reference arm with the reference library only (oracle/_ref: its own
# generator stream and gen_mask) -- the reference arm never loads libparo_b200.
def grid_shape(grid_text):
    """'F:13,H:30,W:45' -> (labels, extents, N) without any native library."""
    labels, ext = "", []
    for part in grid_text.split(","):
        a, n = part.split(":")
        labels += a.strip()
        ext.append(int(n))
    return labels, tuple(ext), int(np.prod(ext))


def head_sums(h, kb, density, family):
    """The calibration block sums gen_mask selects from."""
    rng = np.random.default_rng(7919 * (h + 1))
    if family == "random":  # M1: U[0,1) + 2*I (test_mask.cpp:28-37 shape)
        return rng.random((kb, kb)) + 2.0 * np.eye(kb)
    w = max(density * kb / 2.0, 1.0)  # M2: exp(-|i-j|/w) + 0.05*U, w = density*k/2
    i = np.arange(kb)
    return np.exp(-np.abs(i[:, None] - i[None, :]) / w) + 0.05 * rng.random((kb, kb))


def kept_ops(mask, N, d):
    """4*d*sum over kept blocks of true rows x true cols."""
    kb = mask.shape[0]
    ext = np.full(kb, 64, np.int64)
    ext[-1] = N - 64 * (kb - 1)
    return int(4 * d * (ext[:, None] * ext[None, :] * (mask != 0)).sum())


def workload_ours(paro, ctx, heads, grid_text, N, d, density, family):
    """Per-head orders enumerate_perms(grid)[h % ndim!], seeded N(0,1) Q/K/V
    (MT19937-64 + Box-Muller, seed 1000 + 3h + {0,1,2}), masks by K5 gen_mask on
    the GPU over head_sums."""
    from concurrent.futures import ThreadPoolExecutor

    g = paro.parse_grid(grid_text)
    orders = paro.enumerate_orders(g)
    kb = (N + 63) // 64
    q = np.empty((len(heads), N, d), np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)

    def one(i):
        h = heads[i]
        q[i], k[i], v[i] = [paro.synth_randn(1000 + 3 * h + j, N * d).reshape(N, d) for j in range(3)]

    with ThreadPoolExecutor(8) as ex:
        list(ex.map(one, range(len(heads))))
    ms, _ = ctx.gen_mask(np.stack([head_sums(h, kb, density, family) for h in heads]), density, 64)
    masks = np.stack([m.bits for m in ms])
    return [orders[h % len(orders)] for h in heads], q, k, v, masks


def workload_reference(ref, heads, grid_text, N, d, density, family):
    """The same workload from the reference library alone (oracle/_ref)."""
    rc, labels, ext = ref.parse_grid(grid_text)
    if rc:
        raise RuntimeError(f"reference parse_grid failed ({rc})")
    orders = ref.enumerate_orders(labels, ext)
    kb = (N + 63) // 64
    H = len(heads)
    q = np.empty((H, N, d), np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)
    for i, h in enumerate(heads):  # streams 3h, 3h+1, 3h+2 -> q, k, v
        s = ref.synth_randn_streams(1000 + 3 * h, 1, 3, N * d)
        q[i], k[i], v[i] = s[0].reshape(N, d), s[1].reshape(N, d), s[2].reshape(N, d)
    masks = np.empty((H, kb, kb), np.uint8)
    for i, h in enumerate(heads):
        rc, bits, _ = ref.gen_mask(head_sums(h, kb, density, family), density, 64)
        if rc:
            raise RuntimeError(f"reference gen_mask failed ({rc})")
        masks[i] = bits
    return [orders[h % len(orders)] for h in heads], q, k, v, masks


def bench_config(cfg_name, family, masks, world, dense_prefix=0, rope=False):
    """The `config` object of the JSON line -- identical in both arms."""
    grid_text, H, d, density, pv_bits, desc = CONFIGS[cfg_name]
    N = grid_shape(grid_text)[2] + dense_prefix
    return {
        "workload": desc, "grid": grid_text, "heads": H, "tokens": N, "head_dim": d, "density": density,
        "kept_density": round(float(np.mean(masks != 0)), 5), "pv_bits": pv_bits, "mask_family": family,
        **({"dense_prefix": dense_prefix} if dense_prefix else {}),
        **({"rope": "fused into K1 (cos/sin tables read per row)"} if rope else {}),
        "parallelism": f"head-shard x{world} (no data-path collective)",
        "l2": f"inputs {3 * H * N * d * 4 / 1e6:.0f} MB > 126 MB L2 (no flush needed)",
    }


def cpu_info(threads):
    model, flags = None, set()
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name") and model is None:
                    model = ln.split(":", 1)[1].strip()
                elif ln.startswith("flags"):
                    flags = set(ln.split(":", 1)[1].split())
                    break
    except OSError:
        pass
    isa = [x for x in ("avx2", "fma", "avx512f", "avx512bw", "avx512_vnni", "amx_int8") if x in flags]
    return {"nproc": os.cpu_count(), "threads_used": threads, "model": model, "isa": isa,
            "reference_kernels": "PARO_KERNELS=auto (AVX2 TU when the CPU has avx2, kernels.cpp:17-39)"}


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
def reference_run(cfg_name, family, threads, steps, warmup):
    """The reference's own CPU chain (cmd_run: apply_perm_rows x3 ->
    quantized_blocked_attention -> inverse permute, main.cpp:276-305) from
    oracle/_ref on the host cores, one std::thread per head. A step is a bounded
    sample of the layer: `threads` heads (all H if H <= threads), cycling through
    the layer's heads from step to step; `warmup` untimed steps first. Inputs and
    masks come from the reference library itself (workload_reference). Returns
    the measured time of what ran -- nothing is extrapolated into the value."""
    from oracle.pyoracle import Reference, have_reference

    if not have_reference():
        return None
    grid_text, H, d, density, bits, _ = CONFIGS[cfg_name]
    N = grid_shape(grid_text)[2]
    ref = Reference()
    ref.select_kernels("auto")
    threads = threads or os.cpu_count() or 1
    per = min(H, threads)
    total = steps + warmup
    sched = [[(s * per + j) % H for j in range(per)] for s in range(total)]
    need = sorted({h for hs in sched for h in hs})
    orders, q, k, v, masks = workload_reference(ref, need, grid_text, N, d, density, family)
    kb = (N + 63) // 64
    all_masks = np.empty((H, kb, kb), np.uint8)
    for h in range(H):
        all_masks[h] = ref.gen_mask(head_sums(h, kb, density, family), density, 64)[1]
    idx = {h: i for i, h in enumerate(need)}
    times, ops = [], 0
    for s, hs in enumerate(sched):
        sel = [idx[h] for h in hs]
        _, t = ref.run_heads(grid_text, q[sel], k[sel], v[sel], [orders[i] for i in sel], masks[sel], bits, 0.0,
                             threads)
        if s >= warmup:
            times.append(t)
            ops += sum(kept_ops(masks[i], N, d) for i in sel)
    secs = sum(times)
    return {
        "value": ops / secs / 1e12, "unit": "TOPS", "cores": threads, "kind": "reference",
        "sample": f"{per} of {H} heads ({cfg_name}) per step, one per host thread, cycling through the layer; "
                  f"{len(times)} timed step(s) after {warmup} warm-up, {secs:.1f} s timed",
        "ms_per_step": secs / max(1, len(times)) * 1e3, "steps": len(times), "warmup": warmup,
        "heads_per_step": per, "all_masks": all_masks, "cpu": cpu_info(threads),
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


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: launch the N ranks (one per
    GPU) through torch.distributed.run on 127.0.0.1 and pass rank 0's line on."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.config == "maskgen":
        return maskgen_main(args)
    if args.config == "permsel":
        return permsel_main(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    grid_text, H, d, density, pv_bits, desc = CONFIGS[args.config]

    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; run plain `python bench.py --gpus N` "
                         "(it spawns the ranks) or torchrun with --nproc-per-node N")

    if args.impl == "reference":
        if rank != 0:  # the reference is a host-CPU baseline: rank 0 alone runs it
            return
        r = reference_run(args.config, args.mask_family, args.cpu_threads, args.steps, args.warmup)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparo_ref.so not built"}))
            return
        line = {
            "impl": "reference", "metric": METRIC,
            "value": r["value"], "unit": "TOPS", "n_gpus": args.gpus, "steps": r["steps"], "warmup": r["warmup"],
            "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "dtype_detail": "reference CPU semantics: fp64 QK logits, int8/int4 P and V codes, fp64 accumulators",
            "data": "synthetic N(0,1) Q/K/V (reference MT19937-64 Box-Muller stream), reference gen_mask masks",
            "config": bench_config(args.config, args.mask_family, r["all_masks"], world),
            "cpu_baseline": {k_: r[k_] for k_ in ("value", "unit", "cores", "kind", "sample")},
            "cpu": r["cpu"], "heads_per_step": r["heads_per_step"],
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
    my_orders, q, k, v, masks = workload_ours(paro, ctx, my_heads, grid_text, N, d, density, args.mask_family)
    all_ms, _ = ctx.gen_mask(np.stack([head_sums(h, kb, density, args.mask_family) for h in range(H)]), density, 64)
    all_masks = np.stack([m.bits for m in all_ms])
    my_ops = sum(kept_ops(masks[i], N, d) for i in range(hpr))
    total_ops = sum(kept_ops(all_masks[h], N, d) for h in range(H))

    layer = paro.Layer(ctx, hpr, d, g, my_orders, dense_prefix=args.dense_prefix)
    if args.v_packed:
        layer.set_v_packing(True)
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

    step_no = [0]
    if args.schedule:  # one PSCH schedule per head from the GPU build_schedule over per-timestep sums
        blobs = []
        for i, h in enumerate(my_heads):
            rng = np.random.default_rng(104729 * (h + 1))
            sums_t = np.stack([head_sums(h, kb, density, args.mask_family) + 0.1 * rng.random((kb, kb))
                               for _ in range(args.schedule)])
            ms, _ = ctx.build_schedule(sums_t, density, 64)
            blobs.append(paro.serialize_schedule(args.schedule, ms))
        layer.set_schedule(blobs, 2 if args.schedule_prefetch else 0, sp)

    def step(events=None):
        if events:
            events[0].record(stream)
        if args.schedule:  # timestep i % T: the lists are resident (or prefetched), no K2 here
            layer.select_timestep(step_no[0] % args.schedule, sp)
            step_no[0] += 1
        else:
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

    line = {
        "metric": METRIC,
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
        "data": "synthetic N(0,1) Q/K/V (MT19937-64 Box-Muller), K5 gen_mask masks (GPU)",
        "config": {**bench_config(args.config, args.mask_family, all_masks, world, args.dense_prefix, args.rope),
                   **({"v_storage": "INT4 nibble-packed in HBM, unpacked in smem"} if args.v_packed and pv_bits == 4
                      else {}),
                   **({"schedule": f"{args.schedule} timesteps, PSCH per head, kept lists "
                                   + ("double-buffered, K2 of t+1 prefetched on a side stream" if args.schedule_prefetch
                                      else "of every entry resident (no K2 in the step)")} if args.schedule else {})},
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
        "gpu_launches": ((2 if args.schedule and not args.schedule_prefetch else 5) + (3 if args.dense_prefix else 0))
                        * args.steps,
        "clocks": clk,
        "e2e": e2e,
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        try:
            cb = reference_run(args.config, args.mask_family, args.cpu_threads, 1, 0)
        except Exception as ex:  # the baseline must not kill the bench line
            cb = {"error": str(ex)}
        if cb is not None:
            line["cpu_baseline"] = {k_: cb[k_] for k_ in ("value", "unit", "cores", "kind", "sample", "cpu")
                                    if k_ in cb} if "error" not in cb else cb
    if rank == 0:
        print(json.dumps(line))
    layer.close()
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
