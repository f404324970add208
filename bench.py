#!/usr/bin/env python
"""RBGS QR throughput benchmark (BASELINE.json metric: GB/s of W processed,
% of HBM roofline, at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c5shard]
                    [--order reference|fma] [--impl b200|reference]

A step is one complete RBGS QR factorization (`rbgs.rbgs`, every block:
sketch, LS solve, projection, inter-block QR, final certification) of the
synthetic W of the chosen BASELINE config, W resident in HBM.  Default:
configs[1] (C2: n = 1e6 x m = 800, p = 40, gaussian k = 1600, two-precision).
With N > 1 (torchrun) the rows are sharded, n = N x n_config (weak scaling),
and each block's sketches are summed with one NCCL allreduce.

`e2e` is the same metric through the public API with host buffers: a pinned
host W is copied to the device inside every timed step and R is read back.
`--impl reference` times the CPU restatement of the reference (oracle/) on a
bounded row sample of the same workload with all host threads.
"""

from __future__ import annotations

import os

_CORES = len(os.sched_getaffinity(0))
if "--impl" in os.sys.argv and "reference" in os.sys.argv:
    # all host threads for the CPU arm (torchrun presets OMP_NUM_THREADS=1 for
    # its workers; only rank 0 runs this arm)
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[_v] = str(_CORES)

import argparse  # noqa: E402
import json  # noqa: E402
import math  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(name="C2", n=1_000_000, m=800, p=40, k=1600, kind="gaussian", gen="trig", dtype="f32",
               coarse="coarse", desc="RBGS QR two-precision, trig family 1e6 x 800, p=40, gaussian k=1600"),
    "c1": dict(name="C1", n=20_000, m=200, p=10, k=400, kind="gaussian", gen="trig", dtype="f64",
               coarse="fine", desc="RBGS QR fp64 throughout, trig family 20000 x 200, p=10, gaussian k=400"),
    "c3": dict(name="C3", n=1 << 24, m=512, p=32, k=1024, kind="srht", gen="lowrank", dtype="f32",
               coarse="coarse", desc="RBGS QR two-precision, U diag(s) V^T 2^24 x 512, p=32, SRHT k=1024"),
    "c4": dict(name="C4", n=256 ** 3, grid=256, m=244, p=61, mp=4, k=488, kind="sparse_sign", nnz=8,
               gen="poisson", dtype="f64", coarse="coarse", krylov=True,
               desc="block GMRES, 4 RHS, 7-point Poisson 256^3, 61 RBGS blocks (60 Arnoldi steps), "
                    "sparse-sign k=488 (8 nnz/col), fp32 coarse / fp64 fine"),
    "c5shard": dict(name="C5-shard", n=1 << 24, m=1024, p=64, k=2048, kind="gaussian", gen="colscaled",
                    dtype="f32", coarse="coarse", inplace=True, order="tc", digits=4,
                    desc="RBGS QR two-precision, per-GPU shard of C5: 2^24 x 1024, p=64, gaussian k=2048"),
}
SEED_W, SEED_THETA = 7, 11


def _dist_setup():
    """One process per GPU (torchrun env), NCCL.  RB_BENCH_BACKEND=gloo with
    RB_BENCH_ONE_DEVICE=1 runs every rank on cuda:0 with host-side gloo
    collectives -- a functional check of the multi-rank path on a one-GPU
    box (the ranks' kernels never wait on one another); never a timing."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if os.environ.get("RB_BENCH_ONE_DEVICE") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        backend = os.environ.get("RB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    return world, rank, local, dev, group


def _h2d_link(Wh, dev):
    """Raw pinned host -> device copy bandwidth of this box (GB/s, best of
    3, CUDA events): the floor under `e2e`, which moves all of W every step."""
    import torch
    src = Wh.t()[: max(1, (1 << 29) // (Wh.shape[0] * Wh.element_size()))]  # ~512 MB of contiguous rows
    dst = torch.empty(src.shape, dtype=src.dtype, device=dev)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, src.numel() * src.element_size() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del dst
    return best


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1658.3)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and
                          r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU restatement (oracle) -- the reference arm and the cpu_baseline leg

def _oracle_sample(cfgd, n_s, parity=False, order="reference", digits=None, theta_bits=16):
    """One RBGS QR of an n_s-row sample of the workload with the CPU oracle;
    the gaussian table is materialised beforehand (operator construction),
    like the reference's SRHT tables.  Returns seconds -- and with `parity`
    also the device factorization of the SAME sample checked against it
    (the oracle as the checker: R drift and both certificates)."""
    from oracle import sketches as osk
    from oracle import sweep as osw
    from paper_2111_14641_b200 import workloads as WL

    m, p, k = cfgd["m"], cfgd["p"], min(cfgd["k"], n_s)
    if cfgd["gen"] == "trig":
        W = WL.trig_host(n_s, m, SEED_W)
    elif cfgd["gen"] == "lowrank":
        W = WL.lowrank_host(n_s, m, SEED_W)
    else:
        W = WL.colscaled_host(n_s, m, SEED_W)
    if cfgd["dtype"] == "f32":
        W = W.astype(np.float32).astype(np.float64)
    op = osk.materialize(osk.OracleSketch(cfgd["kind"], k, n_s, SEED_THETA, bits=theta_bits))
    cfg = osw.OracleConfig(osw.uniform_widths(m, p), interblock="sketched_cholqr(1)",
                           coarse=cfgd["coarse"])
    t0 = time.perf_counter()
    sw, cert = osw.rbgs(W, op, cfg)
    sec = time.perf_counter() - t0
    if not parity:
        return sec
    import torch

    from paper_2111_14641_b200 import sketching
    from paper_2111_14641_b200.kernels import COARSE, FINE, BlockPartition
    from paper_2111_14641_b200.rbgs import DeviceConfig, RbgsConfig, rbgs

    theta = (sketching.gaussian_operator(k, n_s, SEED_THETA, theta_bits=theta_bits) if cfgd["kind"] == "gaussian"
             else sketching.make_operator(cfgd["kind"], k, n_s, SEED_THETA))
    gcfg = RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)",
                      coarse=COARSE if cfgd["coarse"] == "coarse" else FINE)
    Wg = W.astype(np.float32) if cfgd["dtype"] == "f32" else W
    f = rbgs(Wg, theta, gcfg, DeviceConfig(projection_order=order, sketch_digits=digits))
    torch.cuda.synchronize()
    R, Rref = f.R.data, sw.R
    par = {"rows": n_s, "oracle": "oracle/ restatement, same W, same seeded operator",
           "rel_R_diff": float(np.linalg.norm(R - Rref) / np.linalg.norm(Rref)),
           "max_rel_diag_diff": float(np.max(np.abs(np.diag(R) - np.diag(Rref)) / np.abs(np.diag(Rref)))),
           "delta": [float(f.cert.delta), float(cert[0])],
           "delta_tilde": [float(f.cert.delta_tilde), float(cert[1])],
           "pairs": "[device, oracle]",
           "tolerance": "R within 1e-5 relative (two-precision) / 1e-10 (fp64), BASELINE north_star"}
    return sec, par


def reference_arm(args, cfgd):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_s = args.sample_rows or 4096
    times = []
    for it in range(args.warmup + args.steps):
        t = _oracle_sample(cfgd, n_s)
        if it >= args.warmup:
            times.append(t)
    sec = sum(times) / len(times)
    s = 4 if cfgd["dtype"] == "f32" else 8
    val = s * n_s * cfgd["m"] / sec / 1e9
    cpu = {"value": val, "unit": "GB/s", "cores": _CORES, "kind": "port",
           "sample": f"{n_s} x {cfgd['m']} rows of {cfgd['name']} (same m, p, k-kind), one factorization "
                     f"per step, oracle/ restatement (numpy + OpenBLAS, {_CORES} threads)"}
    line = {"metric": "RBGS QR GB/s of W processed", "value": val, "unit": "GB/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32-coarse/f64-fine" if cfgd["dtype"] == "f32" else "f64", "data": "synthetic",
            "config": {"workload": cfgd["desc"], "sample_rows": n_s},
            "cpu_baseline": cpu, "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the GPU arm

class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def gpu_arm(args, cfgd):
    import torch
    import torch.distributed as dist

    from paper_2111_14641_b200 import _device as D
    from paper_2111_14641_b200 import _lib, sketching, workloads
    from paper_2111_14641_b200.comm import Comm, RowShard
    from paper_2111_14641_b200.kernels import COARSE, FINE, BlockPartition
    from paper_2111_14641_b200 import rbgs as rbgs_mod
    from paper_2111_14641_b200.rbgs import DeviceConfig, RbgsConfig, RbgsPlan, rbgs

    world, rank, local, dev, group = _dist_setup()
    n_per, m, p, k = cfgd["n"], cfgd["m"], cfgd["p"], cfgd["k"]
    n = n_per * world
    shard = RowShard(n, rank * n_per, n_per)
    dtype = torch.float32 if cfgd["dtype"] == "f32" else torch.float64
    esz = 4 if dtype == torch.float32 else 8
    # --- inputs (not timed) ---
    if cfgd["gen"] == "trig":
        W = workloads.trig_device(n, m, SEED_W, shard.row0, n_per, dtype, dev)
    elif cfgd["gen"] == "lowrank":
        W = workloads.lowrank_device(n_per, m, SEED_W, dtype=dtype, device=dev, rank=rank)
    else:
        W = workloads.colscaled_gaussian_device(n_per, m, SEED_W, dtype=dtype, device=dev, rank=rank)
    # in place (C5 shard): Q overwrites W, so W is regenerated before every
    # step outside the timed events, and each step is timed on its own
    inplace = bool(cfgd.get("inplace"))

    def regen():
        if cfgd["gen"] == "colscaled":
            workloads.colscaled_gaussian_device(n_per, m, SEED_W, dtype=dtype, device=dev, rank=rank, out=W)
        torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if cfgd["kind"] == "gaussian":
        theta = sketching.gaussian_operator(k, n, SEED_THETA, theta_bits=args.theta_bits)
        theta.device_tables(dev, shard.row0, n_per)
    else:
        theta = sketching.SketchOperator(cfgd["kind"], k, n, SEED_THETA)
        theta.device_tables(dev)
    cfg = RbgsConfig(partition=BlockPartition.uniform(m, p), interblock=args.interblock,
                     coarse=COARSE if cfgd["coarse"] == "coarse" else FINE)
    dc = DeviceConfig(device=dev, projection_order=args.order, comm=Comm(group) if group else None,
                      shard=shard if world > 1 else None, overwrite_w=inplace, sketch_digits=args.sketch_digits)
    torch.cuda.synchronize()

    # Default: the factorization captured once as a CUDA graph (RbgsPlan)
    # and replayed -- every kernel of every block per step (with NCCL, the
    # one allreduce per block is captured too), plus the host read of the
    # block statuses and the certification.  In-place runs (C5 shard),
    # gloo-backed runs (host collectives cannot be captured) and --no-graph
    # use the eager one-shot rbgs().
    backend = dist.get_backend(group) if group is not None else "none"
    use_graph = not inplace and not args.no_graph and backend in ("none", "nccl")
    plan, graph_note = None, None
    if use_graph:
        try:
            plan = RbgsPlan(W, theta, cfg, dc)
        except Exception as exc:  # capture unsupported here: eager, and say so
            graph_note = f"graph capture failed ({type(exc).__name__}: {exc}); eager"
            plan = None

    def step():
        return plan.replay() if plan is not None else rbgs(W, theta, cfg, dc)

    for _ in range(args.warmup):
        if inplace:
            regen()
        f = step()
        del f
    torch.cuda.synchronize()

    def barrier():
        if group is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # --- timed region: K factorizations, W resident in HBM ---
    comm_obj = dc.comm
    coll0 = comm_obj.collectives if comm_obj is not None else 0
    n0 = _lib.launch_count()
    timer = None
    with Clocks(local) as clk, (D.timed_kernels() if plan is None else _nullctx()) as timer:
        barrier()
        if inplace:
            tot = 0.0
            for _ in range(args.steps):
                regen()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                f = step()
                e1.record()
                barrier()
                tot += e0.elapsed_time(e1)
            ms = tot / args.steps
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                f = step()
            e1.record()
            barrier()
            ms = e0.elapsed_time(e1) / args.steps
    launches = _lib.launch_count() - n0
    clk_summary = clk.summary()
    ksteps = args.steps
    if plan is not None:
        # graph replays launch no kernels through the C ABI: count one
        # eager step's launches (the captured kernel sequence is the same)
        # and time its kernels with CUDA events for the roofline -- an
        # instrumented step outside the timed region
        barrier()
        n1 = _lib.launch_count()
        coll0 = comm_obj.collectives if comm_obj is not None else 0
        with D.timed_kernels() as timer:
            rbgs(W, theta, cfg, dc)
            torch.cuda.synchronize()
        launches = (_lib.launch_count() - n1) * args.steps
        ksteps = 1
    if group is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ksum = timer.summary()
    kscale = ksteps  # kernel records cover this many steps
    coll_per_block = None
    if comm_obj is not None and comm_obj.active:
        coll_per_block = (comm_obj.collectives - coll0) / (ksteps * cfg.partition.num_blocks)
    cert = f.cert
    wbytes = esz * n * m
    value = wbytes / (ms * 1e-3) / 1e9

    # --- e2e: pinned host W -> device inside the step, R read back ---
    e2e = None
    if inplace:
        e2e = {"value": None, "unit": "GB/s", "skipped": "C5 shard: a 64 GB pinned host W is not staged on the box"}
    elif not args.no_e2e:
        Wh = torch.empty((m, n_per), dtype=dtype).pin_memory().t()
        Wh.copy_(W)
        del W
        torch.cuda.empty_cache()
        e2e_steps = max(1, min(args.steps, 5))
        # untimed: allocator / copy-stream first use.  Same assignment pattern as
        # the timed loop (the previous result stays alive while the next call
        # allocates its Q), so the caching allocator holds both Q buffers before
        # timing starts instead of cudaMalloc'ing the second in timed step 1.
        for _ in range(max(2, min(args.warmup, 3))):
            fe = rbgs(Wh, theta, cfg, dc)
            Rh = fe.R.data
        barrier()
        t0 = time.perf_counter()
        each = []
        for _ in range(e2e_steps):
            ts = time.perf_counter()
            fe = rbgs(Wh, theta, cfg, dc)
            Rh = fe.R.data  # device -> host read of the result
            each.append((time.perf_counter() - ts) * 1e3)
        barrier()
        sec = (time.perf_counter() - t0) / e2e_steps
        if group is not None:
            t = torch.tensor([sec], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
        e2e = {"value": wbytes / sec / 1e9, "unit": "GB/s", "h2d_bytes_per_step": esz * n_per * m,
               "d2h_bytes_per_step": int(Rh.nbytes), "ms_per_step": sec * 1e3,
               "ms_each": [round(x, 2) for x in each], "h2d_link_GBps": _h2d_link(Wh, dev),
               "host_buffer": "pinned, column-major"}
        # the reference-style input: a pageable numpy array (one staged upload
        # through the driver's bounce buffers, no per-block overlap)
        if world == 1 and esz * n_per * m <= (8 << 30):
            Wn = np.array(Wh.numpy(), order="F", copy=True)  # a fresh pageable allocation
            del Wh
            for _ in range(2):
                fe = rbgs(Wn, theta, cfg, dc)
                Rh = fe.R.data
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(2):
                fe = rbgs(Wn, theta, cfg, dc)
                Rh = fe.R.data
            torch.cuda.synchronize()
            secp = (time.perf_counter() - t0) / 2
            e2e["pageable_numpy"] = {"value": wbytes / secp / 1e9, "unit": "GB/s", "ms_per_step": secp * 1e3}
            del Wn

    # --- roofline of the dominant kernel ---
    hbm, bf16, src = _peaks()
    dom = max(ksum.items(), key=lambda kv: kv[1]["ms"]) if ksum else None
    roof = None
    if dom:
        name, d = dom
        per_ms = d["ms"] / d["calls"]
        ach = d["bytes"] / d["calls"] / (per_ms * 1e-3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                traffic = json.load(fh).get(f"{cfgd['name']}:{name}")
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": name, "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": traffic, "peak_source": src,
                "share_of_step": d["ms"] / kscale / ms,
                "bytes_per_launch": d["bytes"] / d["calls"], "ms_per_launch": per_ms}
        if name == "project" and args.order == "reference":
            # The reference rounding order (one FMUL + one FADD per element
            # step, never fused) makes Step 3 FP32-issue-bound, not
            # HBM-bound: the binding roofline is the FP32 pipe,
            # 148 SMs x 128 lanes x SM clock (1 op per lane per cycle).
            mhz = (clk_summary or {}).get("sm_mhz") or 1965.0
            fpeak = 148 * 128 * mhz * 1e6 / 1e12
            fach = d["flops"] / (d["ms"] * 1e-3) / 1e12
            roof["compute_bound"] = {"pipe": "fp32 (FMUL+FADD, reference order)", "achieved": fach,
                                     "peak": fpeak, "unit": "TFLOP/s", "frac": fach / fpeak,
                                     "flops_per_launch": d["flops"] / d["calls"]}
        if name == "sketch_gaussian" and esz == 4:
            # The exact digit split runs 2 x digits int8 byte
            # products per (Theta entry, X entry) on the tensor pipe (12 at
            # the default six digits), with M
            # padded to 128 sketch rows: the binding roofline is the int8
            # tensor pipe, 148 SMs x 16384 int8 ops per SM clock (dense).
            mhz = (clk_summary or {}).get("sm_mhz") or 1965.0
            ipeak = 148 * 16384 * mhz * 1e6 / 1e12
            kpad = -(-k // 128) * 128
            nprod = (2 if args.theta_bits == 16 else 1) * (args.sketch_digits or 6)
            iops = d["flops"] * nprod * kpad / k
            roof["compute_bound"] = {"pipe": f"int8 tensor (tcgen05 kind::i8, {nprod} byte products per entry)",
                                     "achieved": iops / (d["ms"] * 1e-3) / 1e12, "peak": ipeak,
                                     "unit": "TOP/s", "frac": iops / (d["ms"] * 1e-3) / 1e12 / ipeak,
                                     "ops_per_launch": iops / d["calls"],
                                     "note": "timed per call incl. the split_planes pre-pass and the split-K reduce"}
    kernels = {kname: {"ms_per_step": d["ms"] / kscale, "calls_per_step": d["calls"] / kscale,
                       "GBps": d["bytes"] / (d["ms"] * 1e-3) / 1e9,
                       "TFLOPs": d["flops"] / (d["ms"] * 1e-3) / 1e12}
               for kname, d in ksum.items()}
    alg = esz * n * p * (cfg.partition.num_blocks * (cfg.partition.num_blocks + 1) / 2
                         + 4 * cfg.partition.num_blocks - 2)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_s = args.sample_rows or 8192
        sec, parity = _oracle_sample(cfgd, n_s, parity=True, order=args.order, digits=args.sketch_digits,
                                     theta_bits=args.theta_bits)
        cpu = {"value": esz * n_s * m / sec / 1e9, "unit": "GB/s", "cores": _CORES, "kind": "port",
               "sample": f"{n_s} x {m} rows of {cfgd['name']}, one factorization, oracle/ restatement "
                         f"(numpy + OpenBLAS)", "parity": parity}
    if rank == 0:
        line = {
            "metric": "RBGS QR GB/s of W processed", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32-coarse/f64-fine" if cfgd["coarse"] == "coarse" else "f64", "data": "synthetic",
            "config": {"workload": cfgd["desc"], "n": n, "m": m, "p": p, "k": k, "sketch": cfgd["kind"],
                       "theta": (("N(0,1) Box-Muller of Philox4x32-10 quantized to the int16 grid 2^-11 (clamped), "
                                  if args.theta_bits == 16 else
                                  "OPT-IN 8-bit operator: N(0,1) Box-Muller of Philox4x32-10 on the int8 grid 2^-5 "
                                  "(255 levels, clamped), ") +
                                 "scaled by 1/sqrt(k); same operator in the oracle" if cfgd["kind"] == "gaussian"
                                 else "reference operator (numpy Philox recipe)"),
                       "interblock": args.interblock, "ls_solver": "richardson(5)",
                       "projection_order": args.order, "sketch_digits": args.sketch_digits or 6, "parallelism": f"rows{world}",
                       "execution": ("cuda-graph replay (RbgsPlan)" if plan is not None
                                     else (graph_note or "eager rbgs()")),
                       "collectives_per_block": coll_per_block,
                       "kernel_timing": ("one instrumented eager step after the timed region"
                                         if plan is not None else "CUDA events inside the timed region"),
                       "l2": "inputs larger than L2 (W = %.1f GB)" % (wbytes / 1e9)},
            "roofline": roof,
            "algorithmic_roofline": {"bytes_per_factorization": alg, "GBps": alg / (ms * 1e-3) / 1e9,
                                     "frac": alg / (ms * 1e-3) / 1e9 / hbm / world},
            "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk_summary,
            "cert": {"delta": cert.delta, "delta_tilde": cert.delta_tilde},
            "status_replays": rbgs_mod.REPLAYS,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.destroy_process_group()


def gpu_arm_krylov(args, cfgd):
    """C4: one restarted block GMRES solve (krylov.block_gmres, restarts=1)
    per step on the 7-point Poisson operator; W = the 61 Arnoldi blocks
    (binary64, n x 244).  Rows are z-slab sharded with a halo exchange per
    operator apply when run under torchrun (strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_2111_14641_b200 import _lib, krylov, operators, sketching
    from paper_2111_14641_b200.comm import Comm, RowShard
    from paper_2111_14641_b200.rbgs import DeviceConfig, RbgsConfig

    world, rank, local, dev, group = _dist_setup()
    comm = Comm(group) if group else None
    g = cfgd["grid"]
    A = operators.Poisson3D(g, g, g, comm=comm, device=dev)
    n, n_local, row0 = A.n, A.n_local, A.row0
    mp, p, k = cfgd["mp"], cfgd["p"], cfgd["k"]
    gen = torch.Generator(device=dev).manual_seed(SEED_W)
    Bfull_cols = torch.randn(mp, n, generator=gen, device=dev, dtype=torch.float64)
    B = Bfull_cols[:, row0:row0 + n_local].t()  # this rank's rows, column-major view
    del gen
    theta = sketching.sparse_sign_operator(k, n, SEED_THETA, cfgd["nnz"])
    dc = DeviceConfig(device=dev, comm=comm, shard=RowShard(n, row0, n_local) if world > 1 else None)
    cfg = RbgsConfig()

    def step():
        return krylov.block_gmres(A, B, theta, p, restarts=1, cfg=cfg, device_cfg=dc,
                                  diagnostics=args.diagnostics)

    for _ in range(args.warmup):
        rep = step()
    torch.cuda.synchronize()

    def barrier():
        if group is not None:
            dist.barrier()
        torch.cuda.synchronize()

    n0 = _lib.launch_count()
    with Clocks(local) as clk:
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            rep = step()
        e1.record()
        barrier()
        wall = (time.perf_counter() - t0) / args.steps
    launches = _lib.launch_count() - n0
    ms = e0.elapsed_time(e1) / args.steps
    if group is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    wbytes = 8 * n * cfgd["m"]
    value = wbytes / (ms * 1e-3) / 1e9
    hbm, _, src = _peaks()
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle as the checker on the same family at a grid it finishes in
        # seconds: 32^3, 16 blocks, same sketch kind and precisions
        from oracle import krylov as okr
        from oracle import sketches as osk
        gs, ps = 32, 16
        ns, ks = gs ** 3, 2 * mp * ps
        Bs = np.random.Generator(np.random.Philox(SEED_W)).standard_normal((ns, mp))
        t0 = time.perf_counter()
        orc = okr.gmres(okr.poisson3d_apply(gs, gs, gs), Bs, osk.OracleSketch("sparse_sign", ks, ns, SEED_THETA), ps)
        sec = time.perf_counter() - t0
        reps = krylov.block_gmres(operators.Poisson3D(gs, gs, gs, device=dev), Bs,
                                  sketching.sparse_sign_operator(ks, ns, SEED_THETA, cfgd["nnz"]), ps, cfg=cfg,
                                  diagnostics=args.diagnostics)
        h, ho = np.array(reps.residual_history), np.array(orc["residual_history"])
        xo = orc["solution"]
        parity = {"grid": gs, "blocks": ps, "oracle": "oracle/ restatement (block GMRES, same B, same seeded operator)",
                  "final_rel_residual": [float(h[-1, 1]), float(ho[-1, 1])],
                  "max_rel_residual_history_diff": (float(np.max(np.abs(h[:, 1] / ho[:, 1] - 1.0)))
                                                    if args.diagnostics == "full" else None),
                  "rel_solution_diff": float(np.linalg.norm(reps.solution.data - xo) / np.linalg.norm(xo)),
                  "pairs": "[device, oracle]", "oracle_seconds": sec}
    if rank == 0:
        line = {
            "metric": "RBGS QR GB/s of W processed", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32-coarse/f64-fine", "data": "synthetic",
            "config": {"workload": cfgd["desc"], "n": n, "m": cfgd["m"], "p_blocks": p, "block_width": mp,
                       "k": k, "sketch": "sparse_sign(8)", "restarts": 1, "diagnostics": args.diagnostics, "parallelism": f"zslab{world}",
                       "l2": "inputs larger than L2 (basis = %.1f GB)" % (wbytes / 1e9)},
            "rel_residual": rep.residual_history[-1][1], "iterations": len(rep.residual_history),
            "parity": parity,
            "basis_cond_last": rep.basis_cond_history[-1], "cert_last": list(rep.cert_history[-1]),
            "host_wall_ms_per_step": wall * 1e3, "gpu_launches": launches, "clocks": clk.summary(),
            "peak_hbm_GBps": hbm, "peak_source": src,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--order", default=None, choices=["reference", "fma", "tc"],
                    help="Step-3 order (default: the config's own, see CONFIGS 'order')")
    ap.add_argument("--sketch-digits", type=int, default=None, choices=[6, 4, 3],
                    help="gaussian kind: byte digits of X kept inside Theta X (default: the config's own; 6 = "
                         "binary64-grade)")
    ap.add_argument("--theta-bits", type=int, default=16, choices=[16, 8],
                    help="gaussian kind: grid of the operator's entries (16 = the default int16 grid 2^-11; 8 = the "
                         "opt-in int8 grid 2^-5: one byte plane, half the tensor work)")
    ap.add_argument("--interblock", default="sketched_cholqr(1)",
                    help="inter-block QR (reference default: l2_plus_cholqr; one sketch pass: sketched_cholqr(1))")
    ap.add_argument("--sample-rows", type=int, default=None,
                    help="rows of the CPU sample (default 4096 reference arm, 8192 cpu_baseline)")
    ap.add_argument("--diagnostics", default="full", choices=["full", "sketched"],
                    help="c4: per-iterate GMRES diagnostics (full = the reference's, krylov.py:247-257)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager rbgs() per step instead of a captured RbgsPlan")
    args = ap.parse_args()
    cfgd = CONFIGS[args.config]
    if args.order is None:
        args.order = cfgd.get("order", "reference")
    if args.sketch_digits is None:
        args.sketch_digits = cfgd.get("digits") if cfgd["kind"] == "gaussian" else None
    if args.impl == "reference":
        reference_arm(args, cfgd)
    elif cfgd.get("krylov"):
        gpu_arm_krylov(args, cfgd)
    else:
        gpu_arm(args, cfgd)


if __name__ == "__main__":
    main()
