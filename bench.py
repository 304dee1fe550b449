#!/usr/bin/env python
"""Barnes-Hut step benchmark (BASELINE.json metric: BH interactions/s and
steps/s; + % of FP32 peak for the traversal, % of HBM for build and sort).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg3] [--precision fp32|fp64]

A step is one full KDK leapfrog step of the hot path (simulation.py:492-502):
kick+drift+bounds, Morton keys, radix sort, body permutation, tree build with
moments, traversal, kick.  Default workload = BASELINE config 3, the largest
configuration BASELINE lists on one GPU (two colliding Plummer clusters,
N=1e7, seed 3, fp32, theta=0.6, eps=1e-4, leaf size 32, dt=5e-4).  Synthetic
inputs from the reference's own Plummer sampler (bit-identical restatement).

`--gpus N` without a launcher re-executes itself under torch.distributed.run
with N processes (one per GPU); under torchrun WORLD_SIZE must equal N.

`--impl reference` times the reference algorithm on the host CPU (the oracle
port: the reference is Python/numba and cannot travel to the GPU box), with
all host threads, on a bounded target sample per step.  Its inputs come from
the oracle's own restatement of the reference sampler (no product library).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

AUTO_DISTRIBUTED_N = 30_000_000  # --decomp auto: distributed build from this many bodies

CONFIGS = {
    "cfg1": dict(n=100_000, seed=1, theta=0.5, eps=1e-3, leaf=16, dt=1e-3, kind="plummer"),
    "cfg2": dict(n=1_000_000, seed=2, theta=0.6, eps=1e-3, leaf=16, dt=1e-3, kind="plummer"),
    "cfg3": dict(n=10_000_000, seed=3, theta=0.6, eps=1e-4, leaf=32, dt=5e-4, kind="two"),
    "cfg4": dict(n=100_000_000, seed=4, theta=0.7, eps=1e-5, leaf=32, dt=1e-4, kind="hernquist"),
}
METRIC = "BH interactions/s (full KDK step: bounds, keys, sort, build, walk, kicks)"
FLOPS_PP = 20
FLOPS_PC = 51
SORT_BYTES_PER_BODY = 192  # 8 passes x (8 B key + 4 B index) x (read + write)
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def build_bytes_per_body(cells_per_body: float, records_per_body: float = 0.0) -> float:
    """243 + 32*(C/N - 1.48) algorithmic bytes per body (bounds,
    keys, permutation, lcp / scan / emit, moments) + the 64-byte fp32 walk
    records written."""
    return 243.0 + 32.0 * (cells_per_body - 1.48) + 64.0 * records_per_body


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured"
        return d
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class _Cloud:
    """Minimal Bodies-like holder (float32 arrays) for the 1e8 config."""

    def __init__(self, pos, vel, mass):
        self.position, self.velocity, self.mass = pos, vel, mass

    def __len__(self):
        return len(self.mass)


def make_bodies(cfg: dict):
    from paper_2203_08966_b200.initcond import (colliding_plummers, hernquist_cosmology,
                                                 make_rng, plummer_cluster)

    if cfg["kind"] == "plummer":
        b = plummer_cluster(cfg["n"], make_rng(cfg["seed"]), 1.0)
    elif cfg["kind"] == "hernquist":
        b = _Cloud(*hernquist_cosmology(cfg["n"], cfg["seed"]))
    else:
        b = colliding_plummers(cfg["n"] // 2, cfg["seed"])
    return b


def make_reference_inputs(cfg: dict):
    """(mass, pos, vel) fp64 numpy for the reference arm, from the oracle's
    restatement of the reference sampler (initcond.py:62-77): the arm loads no
    product library.  cfg4's generator is new (the reference has none) and is
    pure numpy."""
    from oracle import oracle as orc

    if cfg["kind"] == "plummer":
        return orc.plummer_cluster(cfg["n"], orc.make_rng(cfg["seed"]), 1.0)
    if cfg["kind"] == "two":
        return orc.colliding_plummers(cfg["n"] // 2, cfg["seed"])
    from paper_2203_08966_b200.initcond import hernquist_cosmology  # numpy only

    pos, vel, mass = hernquist_cosmology(cfg["n"], cfg["seed"])
    return (mass.astype(np.float64), pos.astype(np.float64), vel.astype(np.float64))


def workload_config(args, cfg: dict, ws: int) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": args.config, "n_bodies": cfg["n"], "theta": cfg["theta"], "eps": cfg["eps"],
            "leaf_size": cfg["leaf"], "dt": cfg["dt"], "precision": args.precision,
            "parallelism": parallelism_string(args, ws),
            "l2": "flushed between timed steps (256 MB write)"}


def parallelism_string(args, ws: int, p2p: bool | None = None) -> str:
    if ws <= 1:
        return "single GPU"
    if args.decomp == "distributed":
        return (f"{ws} ranks: costzones key ranges, body migration, distributed build, "
                "branch-node allgather, locally-essential-tree all-to-all")
    xch = ("walk epilogue stores zone results into peer buffers (NVLink, CUDA IPC)" if p2p
           else "NCCL all-reduce of zone results" if p2p is False
           else "zone results exchanged by peer stores or all-reduce")
    return f"{ws} ranks: replicated tree, costzones-partitioned walk, {xch}"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None
        self.first = 0

    def __enter__(self):
        # nvidia-smi takes a while to start: wait for its first sample before the
        # timed region begins, so a short region (cfg2: ~40 ms) is bracketed
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.first = max(0, len(self.rows) - 1)  # the last sample before the region
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            n0 = len(self.rows)  # and at least one sample taken after it ended
            t0 = time.time()
            while len(self.rows) <= n0 and time.time() - t0 < 2.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = [r for r in self.rows[self.first:] if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------- our arm


def run_ours(args, cfg) -> dict | None:
    import torch
    import torch.distributed as dist

    from paper_2203_08966_b200.engine import Engine

    ws, rank, local = dist_setup()
    # BH_DIST_BACKEND=gloo + BH_SHARE_GPU=1: several ranks on one GPU with
    # host-staged collectives (a smoke run of the multi-rank path, not a number)
    backend = os.environ.get("BH_DIST_BACKEND", "nccl")
    if os.environ.get("BH_SHARE_GPU") == "1":
        local = 0
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: --gpus {ws} needs {ws} visible GPUs, found {torch.cuda.device_count()} "
                         "(BH_SHARE_GPU=1 BH_DIST_BACKEND=gloo runs the ranks on one GPU as a smoke test)")
    torch.cuda.set_device(local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    fp64 = args.precision == "fp64"
    b = make_bodies(cfg)
    n = len(b)
    eng = Engine(args.precision, local)
    pos = eng.bodies_tensor(b.position, b.mass)
    vel = eng.vec_tensor(b.velocity)
    mass = torch.as_tensor(np.asarray(b.mass, dtype=np.float64)).to(dev) if fp64 else None
    theta, eps, leaf, dt = cfg["theta"], cfg["eps"], cfg["leaf"], cfg["dt"]
    sim = None
    if ws > 1 and args.decomp == "replicated":  # replicated tree, partitioned walk
        from paper_2203_08966_b200.decomposition import DistributedSim, StepParams, TorchComm

        sim = DistributedSim(eng, TorchComm(), StepParams(theta, eps, leaf, dt))
        sim.load(pos, vel, mass) if fp64 else sim.load(pos, vel)
        sim.bootstrap()
    elif ws > 1:  # key-range decomposition, distributed build
        from paper_2203_08966_b200.decomposition import DistributedBuildSim, StepParams, TorchComm

        if fp64:
            raise SystemExit("the distributed build runs the fp32 walk; use --decomp replicated for fp64")
        sim = DistributedBuildSim(eng, TorchComm(), StepParams(theta, eps, leaf, dt))
        lo, hi = n * rank // ws, n * (rank + 1) // ws  # initial chunk (simulation.py:190-198)
        sim.load(pos[lo:hi].contiguous(), vel[lo:hi].contiguous(),
                 gid=torch.arange(lo, hi, device=dev))
        sim.bootstrap()
    else:
        eng.sim_load(pos, vel, mass)
        eng.sim_forces(theta, eps, leaf, record_work=False)

    def one_step():
        if sim is not None:
            sim.step(1)
        else:
            eng.sim_step(dt, theta, eps, leaf, 1)
    peak_fp = eng.ffma_peak_tflops(fp64)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        one_step()
    eng.check()

    # ---- device-timed steps (inputs resident in HBM)
    eng.timing(True)
    eng.timing_reset()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    total_ms = 0.0
    pp = pc = 0
    cells = records = 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record()
            one_step()
            ev1.record()
            torch.cuda.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            st = eng.stats()
            pp += st.pp
            pc += st.pc
            cells = st.n_cells
            records = st.n_records
    phases = eng.timing_get()
    launches = eng.launches()
    eng.timing(False)
    eng.check()

    # ---- end to end through the public API with host buffers
    e2e_ms, e2e_inter, e2e_path, h2d, d2h = run_e2e(args, cfg, eng, sim, ws, dev, flush, ev0, ev1)
    plugin = run_plugin(args, cfg, eng) if ws == 1 else None

    # ---- max over ranks
    rdev = dev if backend == "nccl" else "cpu"
    t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64, device=rdev)
    work = torch.tensor([pp + pc, e2e_inter, pp, pc], dtype=torch.float64, device=rdev)
    if ws > 1:  # each rank walked its own zone: interactions sum, time is the max
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(work, op=dist.ReduceOp.SUM)
    total_ms, e2e_ms = float(t[0]), float(t[1])
    inter_all, e2e_all = float(work[0]), float(work[1])
    result = None
    if rank == 0:
        peaks = measured_peaks()
        sec = total_ms / 1e3
        walk_s = phases["walk"] / 1e3
        walk_flops = (FLOPS_PP * pp + FLOPS_PC * pc) / args.steps
        walk_tf = walk_flops / (walk_s / args.steps) / 1e12 if walk_s > 0 else None
        # keys + permutation + build (lcp, scans, emit, moments, walk records)
        build_s = (phases["keys"] + phases["permute"] + phases["build"]) / 1e3 / args.steps
        sort_s = phases["sort"] / 1e3 / args.steps
        bpb = build_bytes_per_body(cells / n, records / n)
        build_gbs = bpb * n / build_s / 1e9 if build_s > 0 else None
        sort_gbs = SORT_BYTES_PER_BODY * n / sort_s / 1e9 if sort_s > 0 else None
        hbm = float(peaks["hbm_gbs"])
        traffic = pipe = None
        tp = os.path.join(ROOT, "profiles", "walk_traffic.json")
        if os.path.exists(tp) and not fp64:
            with open(tp) as f:
                wt = json.load(f)
            traffic = wt.get(args.config)
            pipe = wt.get("fp32_pipe_active", {}).get(args.config)
        config = workload_config(args, cfg, ws)
        config["parallelism"] = parallelism_string(args, ws, getattr(sim, "p2p", None))
        result = {
            "metric": METRIC,
            "value": inter_all / sec,
            "unit": "interactions/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps,
            "steps_per_s": args.steps / sec,
            "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None,
            "dtype": "f64" if fp64 else "f32",
            "data": "synthetic: reference plummer_cluster sampler (bit-identical restatement), seed %d" % cfg["seed"],
            "config": config,
            "interactions_per_step": inter_all / args.steps,
            "pp_per_step": pp / args.steps,
            "pc_per_step": pc / args.steps,
            "cells": cells,
            "phase_ms_per_step": {k: v / args.steps for k, v in phases.items()},
            "roofline": {"bound": "fp64" if fp64 else "fp32",
                         "kernel": "k_walk_f64 (fp64 walk)" if fp64 else "k_walk9 (k_walk_f32)",
                         "achieved": walk_tf, "peak": peak_fp, "unit": "TFLOP/s",
                         "frac": (walk_tf / peak_fp) if walk_tf else None,
                         "peak_source": ("DFMA microbenchmark on this GPU (bh_dfma_peak)" if fp64 else
                                         "FFMA microbenchmark on this GPU (bh_ffma_peak); "
                                         "MEASURED_PEAKS.json has no FP32 entry"),
                         "flops_per_unit": {"pp": FLOPS_PP, "pc": FLOPS_PC},
                         "traffic": traffic,
                         "fp32_pipe_active_ncu": pipe},
            "roofline_build": {"bound": "hbm", "achieved": build_gbs, "peak": hbm, "unit": "GB/s",
                               "frac": build_gbs / hbm if build_gbs else None,
                               "bytes_per_body": bpb, "peak_source": peaks.get("source"),
                               "phases": "keys + permute + build (lcp, scans, emit, moments, walk records)"},
            "roofline_sort": {"bound": "hbm", "achieved": sort_gbs, "peak": hbm, "unit": "GB/s",
                              "frac": sort_gbs / hbm if sort_gbs else None,
                              "bytes_per_body": SORT_BYTES_PER_BODY,
                              "impl": "hand-written onesweep LSD radix sort (bh_sort.cu), 8 digit passes"},
            "e2e": {"value": e2e_all / (e2e_ms / 1e3), "unit": "interactions/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms / args.steps, "path": e2e_path},
            "e2e_plugin": plugin,
            "gpu_launches": launches,
            "gpu_launches_note": "libbh kernels launched in the timed region (sort, scans and walk included)",
            "clocks": clocks.summary(),
        }
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()
    return result


def run_plugin(args, cfg, eng) -> dict:
    """The reference-facing plugin path: kdk_step (integrator.py:47-58) on fp64
    host ``Bodies`` with ``TreeForces`` as the accel provider -- host numpy
    kick/drift, the positions/velocities/masses uploaded and the accelerations
    and work read back every step (synchronous API, host clock)."""
    from paper_2203_08966_b200.integrator import kdk_step
    from paper_2203_08966_b200.physics import Bodies
    from paper_2203_08966_b200.simulation import TreeForces

    b = make_bodies(cfg)
    bodies = Bodies(np.asarray(b.mass, dtype=np.float64), np.asarray(b.position, dtype=np.float64),
                    np.asarray(b.velocity, dtype=np.float64))
    n = len(bodies)
    prov = TreeForces(cfg["theta"], cfg["eps"], cfg["leaf"], precision=args.precision, engine=eng)
    prov(bodies)  # bootstrap forces (simulation.py:487)
    kdk_step(bodies, cfg["dt"], prov)  # warm
    k = max(1, min(args.steps, 3))
    t = 0.0
    inter = 0
    for _ in range(k):
        t0 = time.perf_counter()
        kdk_step(bodies, cfg["dt"], prov)
        t += time.perf_counter() - t0
        st = eng.stats()
        inter += st.pp + st.pc
    # fp64 numpy positions, velocities and masses go up (converted on the device);
    # fp64 accelerations and int64 work come back
    return {"value": inter / t, "unit": "interactions/s", "ms_per_step": t / k * 1e3, "steps": k,
            "h2d_bytes_per_step": n * (24 + 24 + 8),
            "d2h_bytes_per_step": n * (24 + 8),
            "path": "integrator.kdk_step(Bodies fp64 numpy, dt, TreeForces) -> TreeForces.forces -> "
                    "Engine.sim_load/sim_forces/sim_store (C-ABI) per step; host numpy kick/drift"}


def run_e2e(args, cfg, eng, sim, ws, dev, flush, ev0, ev1):
    """The same steps through the public API from pinned host buffers: every
    step copies its inputs host->device and its results device->host inside
    the timed region.  Returns (ms, interactions, path, h2d bytes, d2h bytes)."""
    import torch
    import torch.distributed as dist

    theta, eps, leaf, dt = cfg["theta"], cfg["eps"], cfg["leaf"], cfg["dt"]
    fp64 = args.precision == "fp64"
    distributed = ws > 1 and args.decomp == "distributed"
    host_api = not distributed and sim is None and not fp64
    if distributed:  # this rank's bodies only
        p_, v_, a_, w_, g_ = sim.store()
        dpos, dvel, dacc = p_.clone(), v_.clone(), a_.clone()
        dwork, dgid = w_.to(torch.int32).clone(), g_.clone()
        hpos, hvel, hacc = (x.cpu().pin_memory() for x in (dpos, dvel, dacc))
        hwork, hgid = dwork.cpu().pin_memory(), dgid.cpu().pin_memory()
        h2d = d2h = sum(x.numel() * x.element_size() for x in (hpos, hvel, hacc, hwork, hgid))
        path = "DistributedBuildSim.upload/step/store from pinned host pos/vel/acc/work/ids (this rank's bodies)"
    elif host_api:
        n = eng.sim_n if hasattr(eng, "sim_n") and eng.sim_n else cfg["n"]
        dpos = torch.empty((n, 4), dtype=torch.float32, device=dev)
        dvel, dacc = torch.empty_like(dpos), torch.empty_like(dpos)
        eng.sim_store(dpos, dvel, dacc)
        hpos = dpos.cpu().pin_memory()
        hvel3 = dvel[:, :3].contiguous().cpu().pin_memory()
        hacc3 = dacc[:, :3].contiguous().cpu().pin_memory()
        hwork = torch.empty(n, dtype=torch.int32).pin_memory()
        h2d = (16 + 12 + 12) * n
        d2h = (16 + 12 + 12 + 4) * n
        path = ("Engine.sim_step_host -> bh_sim_step_host (C-ABI): pinned host pos (n,4), vel/acc (n,3) in; "
                "state and per-body work back in caller order; positions copied back under the force computation")
    else:  # fp64 or replicated ranks: the resident API from host arrays
        n = cfg["n"]
        w = 3 if fp64 else 4
        dpos = torch.empty((n, w), dtype=eng.dtype, device=dev)
        dvel, dacc = torch.empty_like(dpos), torch.empty_like(dpos)
        dwork = torch.empty(n, dtype=torch.int64, device=dev)
        eng.sim_store(dpos, dvel, dacc)
        hpos, hvel, hacc = (x.cpu().pin_memory() for x in (dpos, dvel, dacc))
        hwork = dwork.cpu().pin_memory()
        hmass = torch.as_tensor(np.asarray(make_bodies(cfg).mass, dtype=np.float64)).pin_memory() if fp64 else None
        dmass = torch.empty(n, dtype=torch.float64, device=dev) if fp64 else None
        h2d = sum(x.numel() * x.element_size() for x in (hpos, hvel, hacc)) + (8 * n if fp64 else 0)
        d2h = sum(x.numel() * x.element_size() for x in (hpos, hvel, hacc, hwork))
        path = ("Engine.sim_load/sim_step/sim_store (C-ABI) from pinned host "
                + ("fp64 pos/vel/acc (n,3) + masses" if fp64 else "pos/vel/acc") + ", work back")
    torch.cuda.synchronize()
    e2e_ms = 0.0
    e2e_inter = 0
    for it in range(args.warmup + args.steps):  # the first W calls warm the path (staging buffers, streams)
        flush.zero_()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        if distributed:
            dpos, dvel, dacc = (x.to(dev, non_blocking=True) for x in (hpos, hvel, hacc))
            sim.upload(dpos, dvel, dacc, hwork.to(dev, non_blocking=True), hgid.to(dev, non_blocking=True))
            sim.step(1)
            p_, v_, a_, w_, g_ = sim.store()
            hpos, hvel, hacc = (x.to("cpu", non_blocking=True) for x in (p_, v_, a_))
            hwork, hgid = w_.to(torch.int32).to("cpu", non_blocking=True), g_.to("cpu", non_blocking=True)
        elif host_api:  # one call: pos (n,4), vel/acc (n,3) in, state + work out (bh_sim_step_host)
            eng.sim_step_host(hpos, hvel3, hacc3, dt, theta, eps, leaf, 1, work=hwork)
        else:
            dpos.copy_(hpos, non_blocking=True)
            dvel.copy_(hvel, non_blocking=True)
            dacc.copy_(hacc, non_blocking=True)
            if fp64:
                dmass.copy_(hmass, non_blocking=True)
            eng.sim_load(dpos, dvel, dmass, acc=dacc)
            if sim is not None:
                sim.step(1)
            else:
                eng.sim_step(dt, theta, eps, leaf, 1)
            eng.sim_store(dpos, dvel, dacc, dwork)
            hpos.copy_(dpos, non_blocking=True)
            hvel.copy_(dvel, non_blocking=True)
            hacc.copy_(dacc, non_blocking=True)
            hwork.copy_(dwork, non_blocking=True)
        ev1.record()
        torch.cuda.synchronize()
        if it < args.warmup:
            continue
        e2e_ms += ev0.elapsed_time(ev1)
        st = eng.stats()
        e2e_inter += st.pp + st.pc
    eng.check()
    return e2e_ms, e2e_inter, path, h2d, d2h


# --------------------------------------------------- CPU (reference) timing


def cpu_reference_step(b, cfg, sample_idx, nthreads):
    """One step of the reference algorithm on the host: bounds, keys, stable
    sort, take, build_hashed (serial, as the reference), traverse a target
    sample on all threads, kick/drift.  Returns (seconds extrapolated to the
    full step, interactions extrapolated, sample seconds)."""
    from oracle import oracle as orc

    pos = np.asarray(b.position, dtype=np.float32).astype(np.float64)
    m = np.asarray(b.mass, dtype=np.float32).astype(np.float64)
    n = len(pos)
    t0 = time.perf_counter()
    R = orc.bounds(pos)
    order = orc.sort_order(orc.morton_keys(pos, R))
    tree = orc.build_tree(m[order], pos[order], R)
    t1 = time.perf_counter()
    totals = np.zeros(2, dtype=np.int64)
    orc.traverse(tree, pos[sample_idx], cfg["theta"], cfg["eps"], cfg["leaf"], nthreads, totals)
    t2 = time.perf_counter()
    a = np.zeros_like(pos)  # kick(dt/2) + drift(dt) on all bodies (integrator.py:37-44)
    v = np.asarray(b.velocity) + a * (0.5 * cfg["dt"])
    _ = pos + v * cfg["dt"]
    t3 = time.perf_counter()
    scale = n / len(sample_idx)
    full = (t1 - t0) + (t2 - t1) * scale + (t3 - t2)
    return full, float(totals.sum()) * scale, t2 - t1


def cpu_baseline(cfg, b, budget_s=8.0) -> dict:
    from oracle import oracle as orc

    nthreads = orc.num_threads()
    n = len(b)
    rng = np.random.Generator(np.random.Philox(key=99))
    probe = rng.choice(n, min(n, 2000), replace=False)
    _, _, ts = cpu_reference_step(b, cfg, probe, nthreads)
    s = int(min(n, max(2000, len(probe) * budget_s / max(ts, 1e-3))))
    sample = np.sort(rng.choice(n, s, replace=False))
    full, inter, _ = cpu_reference_step(b, cfg, sample, nthreads)
    return {"value": inter / full, "unit": "interactions/s", "cores": nthreads, "kind": "port",
            "ms_per_step": full * 1e3,
            "sample": f"serial keys+sort+build over all {n} bodies, traversal of {s} random targets "
                      f"on {nthreads} threads extrapolated to {n}, host kick/drift",
            "cpu": _cpu_model()}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class _RefBodies:
    """(mass, position, velocity) of the reference arm's inputs."""

    def __init__(self, mass, pos, vel):
        self.mass, self.position, self.velocity = mass, pos, vel

    def __len__(self):
        return len(self.mass)


def run_reference(args, cfg) -> dict | None:
    ws, rank, _ = dist_setup()
    if rank != 0:
        return None
    from oracle import oracle as orc

    b = _RefBodies(*make_reference_inputs(cfg))
    n = len(b)
    nthreads = orc.num_threads()
    rng = np.random.Generator(np.random.Philox(key=7))
    probe = rng.choice(n, min(n, 2000), replace=False)
    _, _, ts = cpu_reference_step(b, cfg, probe, nthreads)
    # bounded sample so that warmup + steps stays within a few minutes
    per_step_budget = 100.0 / max(1, args.steps + args.warmup)
    s = int(min(n, max(1000, len(probe) * per_step_budget / max(ts, 1e-3))))
    sample = np.sort(rng.choice(n, s, replace=False))
    # warm-up: one untimed step is enough for host code (the serial build of a
    # 1e7-body tree is ~7 s; W of them would only stretch the run)
    for _ in range(min(args.warmup, 1)):
        cpu_reference_step(b, cfg, sample, nthreads)
    tot_s = 0.0
    tot_i = 0.0
    for _ in range(args.steps):
        full, inter, _ = cpu_reference_step(b, cfg, sample, nthreads)
        tot_s += full
        tot_i += inter
    value = tot_i / tot_s
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "interactions/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None,
        "dtype": "f64",
        "dtype_note": "the reference computes in fp64; with precision fp32 its inputs are the same "
                      "fp32-rounded positions and masses, upcast exactly (SURVEY.md §8c protocol)",
        "data": "synthetic: reference plummer_cluster sampler (oracle restatement), seed %d" % cfg["seed"],
        "config": workload_config(args, cfg, ws),
        "cpu_baseline": {"value": value, "unit": "interactions/s", "cores": nthreads, "kind": "port",
                         "sample": f"per step: serial keys+sort+build over all {n} bodies + traversal of "
                                   f"{s} targets on {nthreads} threads, extrapolated to {n}",
                         "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": "interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def spawn_ranks(args) -> int:
    """`--gpus N` without a launcher: re-run this command under
    torch.distributed.run with N local processes (127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32",
                    help="fp32: the bench configurations' storage and arithmetic; fp64: the "
                         "validation mode (and the drop-in default of SimConfig)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--decomp", choices=["auto", "distributed", "replicated"], default="auto",
                    help="multi-GPU scheme (N>1): key-range decomposition with a distributed "
                         "build, or replicated tree with a partitioned walk; auto = distributed "
                         f"from N >= {AUTO_DISTRIBUTED_N:.0e} bodies (below that the replicated "
                         "O(N) build costs less than the distributed step's fixed exchange)")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(spawn_ranks(args))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch one process per GPU")
    if args.decomp == "auto":
        args.decomp = ("distributed" if CONFIGS[args.config]["n"] >= AUTO_DISTRIBUTED_N and args.precision == "fp32"
                       else "replicated")
    if args.warmup < 3 and args.impl == "ours":
        print("warning: W < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        res = run_reference(args, cfg)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res = run_ours(args, cfg)
    if res is not None:
        ws, rank, _ = dist_setup()
        if ws == 1 and not args.no_cpu_baseline and cfg["n"] <= 20_000_000:
            res["cpu_baseline"] = cpu_baseline(cfg, _RefBodies(*make_reference_inputs(cfg)))
        elif ws == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = {"value": None, "unit": "interactions/s", "cores": None,
                                   "kind": "port", "sample": "skipped: N > 2e7 (serial CPU build "
                                   "of the whole tree per step would exceed the run budget)"}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
