#!/usr/bin/env python
"""bench.py — FP64 KFVM-WENO cell-updates/s per RK stage on B200.

Metric (BASELINE.json): FP64 cell-updates/s per RK stage; one unit of work is
one cell x one SSP-RK3 stage.  A bench "step" is one SSP-RK3 time step (3
stages) of the workload over the whole grid.  Default workload: BASELINE.json
configs[3] (3-D 512^3 outflow Voronoi, 64 regions, R=2, CFL 0.3: the largest
configuration that fits one GPU); `--config k` selects another (1-based,
SURVEY.md §8(d)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config k] [--impl reference]

Under torchrun (N>1) each rank owns a contiguous slab of the last axis
(halo exchange + dt allreduce through NCCL inside libkfvm_b200.so); timing is
CUDA events on the solver stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def algorithmic_flops(rset) -> int:
    """F = 2 nvar sum_q N_q (n_alpha + n_pts) per cell-stage."""
    nvar = rset.dim + 2
    return 2 * nvar * sum(st.count for st in rset.st) * (rset.n_derivs() + rset.n_face_points())


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
        return dist, rank, ws, local
    return None, 0, 1, 0


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_sample(w, seconds_per_stage, nthreads):
    """Oracle (CPU port of the reference algorithm) on a bounded sub-box of
    the workload: a contiguous run of slab-axis planes of the workload's own
    IC with their R+1 halo planes.  The table comes from the hash-pinned file
    (oracle/tables) and the IC from the oracle's restatement
    (kfvm_oracle_ic.cpp), so this leg never maps libkfvm_b200.so.  Returns
    (oracle, IC block, halo H, planes)."""
    from oracle import Oracle  # CPU baseline / reference leg only
    from oracle.kfvm_oracle import initial_condition as oracle_ic
    from oracle.table_file import load_table
    g = w.grid
    table = load_table(g.dim, g.radius)
    H = g.radius + 1
    n_s = 1
    Ub = oracle_ic(g, w.ic, 0, min(g.slab_extent, n_s + 2 * H), nthreads)
    o = Oracle(_subgrid(g, Ub.shape[0]), table, nthreads=nthreads)
    t1 = max(o.sample_stage_seconds(Ub, H, n_s), 1e-4)
    n_s = int(max(1, min(g.slab_extent - 2 * H, seconds_per_stage / t1)))
    Ub = oracle_ic(g, w.ic, 0, n_s + 2 * H, nthreads)
    o = Oracle(_subgrid(g, Ub.shape[0]), table, nthreads=nthreads)
    return o, Ub, H, n_s, table


def cpu_sample(w, seconds_target=10.0, nthreads=None):
    """Time the CPU oracle on a bounded sub-box of the workload (planes of the
    slab axis) and return (cell-updates/s, cores, description)."""
    g = w.grid
    nthreads = nthreads or (os.cpu_count() or 1)
    o, Ub, H, n_s, table = _oracle_sample(w, seconds_target / 3, nthreads)
    times = [o.sample_stage_seconds(Ub, H, n_s) for _ in range(3)]
    t = min(times)
    plane = g.nx * (g.ny if g.dim == 3 else 1)
    cells = plane * n_s
    desc = (f"oracle stage (reconstruct+limit+Riemann+RK combine) on {n_s} of {g.slab_extent} "
            f"slab-axis planes ({cells} cells) of the workload IC, {nthreads} threads of "
            f"'{cpu_model()}', best of 3; table from oracle/tables (hash {table.hash:#x})")
    return cells / t, nthreads, desc


def _subgrid(g, planes):
    from dataclasses import replace
    if g.dim == 3:
        return replace(g, nz=planes, dx=g.dx if g.dx else 1.0 / g.nx)
    return replace(g, ny=planes, dx=g.dx if g.dx else 1.0 / g.nx)


def run_reference(args, w, rank):
    """--impl reference: the CPU oracle (C++ restatement of the reference
    algorithm; the reference itself does not build) on the
    host cores, each step a bounded sample of the workload.  Nothing in this
    leg loads libkfvm_b200.so: table from oracle/tables, IC from the oracle's
    restatement."""
    if rank != 0:
        return
    g = w.grid
    nthreads = os.cpu_count() or 1
    # size each stage to ~0.7 s of CPU work
    o, Ub, H, n_s, table = _oracle_sample(w, 0.7, nthreads)
    for _ in range(args.warmup):
        o.sample_stage_seconds(Ub, H, n_s)
    tot = 0.0
    for _ in range(args.steps):
        tot += 3 * o.sample_stage_seconds(Ub, H, n_s)  # one step = 3 stages
    plane = g.nx * (g.ny if g.dim == 3 else 1)
    cells = plane * n_s
    value = cells * 3 * args.steps / tot
    sample = (f"per step: 3 oracle stages on {n_s} of {g.slab_extent} slab-axis planes "
              f"({cells} cells) of the workload IC, {nthreads} threads of '{cpu_model()}'; "
              f"table from oracle/tables (hash {table.hash:#x}), IC from the oracle restatement")
    line = {
        "metric": "fp64_cell_updates_per_s_per_rk_stage", "value": value,
        "unit": "cell-updates/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(w, args),
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": nthreads,
                         "kind": "port", "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def traffic_of(config_index, shape):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture of this exact workload (profiles/r02/roofline_traffic.json, else
    the round-1 capture profiles/r01/roofline_traffic.json), or None."""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "roofline_traffic.json")) as f:
                t = json.load(f)[str(config_index)]
        except Exception:
            continue
        if list(t["shape"]) != list(shape):
            continue
        return (t["dram_read_bytes"] + t["dram_write_bytes"],
                f"dram read+write bytes per launch, ncu --set full: profiles/{rnd}/" + t["capture"])
    return None, None


def workload_config(w, args):
    g = w.grid
    shape = "x".join(str(x) for x in ((g.nx, g.ny, g.nz) if g.dim == 3 else (g.nx, g.ny)))
    return {"workload": f"BASELINE config {w.index}: {g.dim}-D Euler {shape} {g.bc}, R={g.radius}, "
                        f"{w.ic.kind} IC, SSP-RK3 CFL {g.cfl}, {g.riemann.upper()}",
            "cells": g.ncells, "radius": g.radius, "dim": g.dim, "bc": g.bc,
            "cfl": g.cfl, "config_steps": w.steps,
            "parallelism": f"slab{args.gpus}" if args.gpus > 1 else "single",
            "kxrcf": bool(g.kxrcf),
            "l2": "working set per step (3 state buffers + face-state scratch) exceeds the 126 MB L2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4,
                    help="BASELINE.json config (1-based); default 4 = 512^3 outflow Voronoi, the "
                         "largest config that fits one GPU")
    ap.add_argument("--n", type=int, default=None, help="override resolution (testing)")
    ap.add_argument("--nz", type=int, default=None,
                    help="slab-axis extent (e.g. config 5's weak-scaling block 1024x1024x128)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--engine", type=int, default=None,
                    help="reconstruction kernel: 0 generic, 1 DFMA, 2 DMMA, 3 fused 2-D stage, "
                         "4 row-marching DFMA (default: 4 in 2-D, 2 in 3-D)")
    ap.add_argument("--kxrcf", action="store_true",
                    help="KXRCF troubled-cell mode (S:565): WENO only in flagged cells")
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=VALUE",
                    help="extra solver option (kfvm_gpu_set_option), e.g. overlap=1")
    ap.add_argument("--kz", type=int, default=None,
                    help="slab-axis planes marched by one reconstruction CTA (engines 2-4)")
    args = ap.parse_args()

    import paper_2401_16543_b200 as K
    if args.config == 5 and args.nz is None and args.n is None:
        # config 5's 1024^3 is an 8-GPU workload (180 GB per GPU do not hold
        # it): its weak-scaling series, 1024 x 1024 x 128 per GPU (BASELINE.json)
        args.nz = 128 * max(1, int(os.environ.get("WORLD_SIZE", args.gpus)))
    w = K.baseline_config(args.config, n=args.n, nz=args.nz)
    if args.kxrcf:
        from dataclasses import replace as _replace
        w = _replace(w, grid=_replace(w.grid, kxrcf=True))
    if args.steps is None:
        args.steps = w.steps
    args.warmup = max(3, args.warmup)
    dist, rank, ws, local = dist_init()
    args.gpus = ws if ws > 1 else args.gpus

    if args.impl == "reference":
        run_reference(args, w, rank)
        return
    rset = K.precompute(w.grid.radius, dim=w.grid.dim)

    import torch
    torch.cuda.set_device(local)
    def new_nccl_id():
        if ws <= 1:
            return None
        from paper_2401_16543_b200.solver import nccl_unique_id
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt[:] = torch.tensor(list(nccl_unique_id()), dtype=torch.uint8)
        dist.broadcast(idt, 0)
        return bytes(idt.tolist())
    nccl_id = new_nccl_id()
    g = w.grid
    s = K.Solver(g, rset, rank=rank, nranks=ws, device=local, nccl_id=nccl_id)
    stream = torch.cuda.ExternalStream(s.stream)

    def configure(sv):
        if args.engine is not None:
            sv.set_option("engine", args.engine)
        if args.kz is not None:
            sv.set_option("kz", args.kz)
        for o in args.opt:
            k, v = o.split("=")
            sv.set_option(k, int(v))
    configure(s)

    # warm-up (also captures the CUDA graph)
    s.generate_ic(w.ic)
    s.run_async(args.warmup)
    s.sync()
    # per-kernel timing pass (events around every launch, not graph-replayed)
    s.set_option("timing", 1)
    s.generate_ic(w.ic)
    s.run_async(1)
    s.sync()
    kt = s.kernel_times()
    s.set_option("timing", 0)
    launches_per_step = None

    # timed region: K steps from the workload IC
    s.generate_ic(w.ic)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = s.launch_count
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    s.run_async(args.steps)
    ev1.record(stream)
    s.sync()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = s.launch_count - l0
    clk = clocks.stop()
    kx_frac = float(s.kxrcf_flags().mean()) if g.kxrcf else None
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        dist.barrier()
    cells = g.ncells
    value = cells * 3 * args.steps / (ms * 1e-3)

    # end-to-end through the public API with host buffers: per step upload the
    # state from pinned host memory, one SSP-RK3 step, read the state back
    plane = g.nx * (g.ny if g.dim == 3 else 1)
    nloc = plane * s.np_local * g.nvar
    host = torch.empty(nloc, dtype=torch.float64, pin_memory=True)
    s.generate_ic(w.ic)
    s.get_state_device  # noqa: B018 (API presence)
    Uh = host.numpy().reshape(s.local_shape)
    Uh[...] = s.get_state()
    e2e_steps = max(1, min(args.steps, 10))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        s.set_state(Uh)
        s.ssp_rk3_step()
        s.get_state(out=Uh)
    t_serial = time.perf_counter() - t0
    # ensemble pipelining through the same API: independent fields, one
    # handle (stream) each; every step of every field uploads it from pinned
    # host memory, steps it and reads it back, and the copy engines move one
    # field while the SMs step the other
    # three fields hide the copies behind the steps (measured on config 2: 2
    # fields 1.91e9, 3 fields 2.28e9, device rate 2.32e9); two when the extra
    # handles' state buffers would crowd the device memory
    total_mem = torch.cuda.get_device_properties(local).total_memory
    nf_default = 3 if nloc * 8 * 8 * 3 < 0.5 * total_mem else 2
    nf = int(os.environ.get("KFVM_E2E_FIELDS", str(nf_default)))
    extra = []
    for _ in range(nf - 1):
        sk = K.Solver(g, rset, rank=rank, nranks=ws, device=local, nccl_id=new_nccl_id())
        configure(sk)
        hk = torch.empty(nloc, dtype=torch.float64, pin_memory=True).numpy().reshape(s.local_shape)
        hk[...] = Uh
        extra.append((sk, hk))
    fields = [(s, Uh)] + extra
    for sv, hb in fields:  # warm the other handles' graphs
        sv.set_state_async(hb)
        sv.run_async(1)
        sv.get_state_async(hb)
    for sv, _ in fields:
        sv.sync()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    # large fields: the fields' steps are chained on the device (each waits
    # for the previous field's step) so the SMs run one step at a time while
    # the copy engines move the other fields — concurrent steps would share the
    # SMs and finish together, leaving their copies exposed (config 4: e2e
    # 3.54e8 -> 4.13e8).  Small fields keep the steps concurrent, which hides
    # their launch gaps instead (config 2: 2.29e9 concurrent, 2.20e9 chained).
    chain = nloc * 8 > (1 << 30)
    streams = [torch.cuda.ExternalStream(sv.stream) for sv, _ in fields]
    done = [torch.cuda.Event() for _ in fields]
    t0 = time.perf_counter()
    prev = None
    for _ in range(e2e_steps):
        for i, (sv, hb) in enumerate(fields):
            sv.set_state_async(hb)
            if chain and prev is not None:
                streams[i].wait_event(done[prev])
            sv.run_async(1)
            done[i].record(streams[i])
            prev = i
            sv.get_state_async(hb)
    for sv, _ in fields:
        sv.sync()
    t_e2e = (time.perf_counter() - t0) / nf  # per field-step
    for sk, _ in extra:
        sk.close()
    if dist:
        t = torch.tensor([t_e2e, t_serial], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e, t_serial = float(t[0]), float(t[1])
    e2e_value = cells * 3 * e2e_steps / t_e2e
    e2e_serial = cells * 3 * e2e_steps / t_serial

    if rank == 0:
        F = algorithmic_flops(rset)
        peaks = measured_peaks()
        fp64 = peaks.get("fp64_tflops")
        fp64_src = "MEASURED_PEAKS.json fp64_tflops"
        if fp64 is None:
            p = os.path.join(ROOT, "profiles", "fp64_peak.json")
            try:
                with open(p) as f:
                    pk = json.load(f)
                fp64 = max(pk["dfma_tflops"], pk["dmma_tflops"])
                fp64_src = ("profiles/fp64_peak.json: max(DFMA %.1f, DMMA %.1f) TF measured on this "
                            "pool (MEASURED_PEAKS.json has no FP64 figure)" % (pk["dfma_tflops"],
                                                                                pk["dmma_tflops"]))
            except Exception:
                fp64 = 37.2
                fp64_src = "nominal 148 SM x 64 DFMA x 2 x 1.965 GHz (not measured)"
        # dominant kernel: the reconstruction (k_states_*); per-kernel CUDA-event
        # times of one step on the solver stream (timing pass)
        states_ms_per_step = kt["states"]
        flops_per_step = F * cells * 3
        achieved = flops_per_step / (states_ms_per_step * 1e-3) / 1e12 if states_ms_per_step else None
        cpu = None
        if not args.no_cpu and ws == 1:
            v, cores, desc = cpu_sample(w, seconds_target=8.0)
            cpu = {"value": v, "unit": "cell-updates/s", "cores": cores, "kind": "port",
                   "sample": desc, "cpu_model": cpu_model()}
        line = {
            "metric": "fp64_cell_updates_per_s_per_rk_stage", "value": value,
            "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(w, args),
            "e2e": {"value": e2e_value, "unit": "cell-updates/s",
                    "h2d_bytes_per_step": nloc * 8, "d2h_bytes_per_step": nloc * 8,
                    "steps": e2e_steps,
                    "api": f"Solver.set_state_async/run_async/get_state_async (C-ABI), {nf} fields "
                           f"on {nf} handles: each field-step uploads from pinned host memory and "
                           "reads back; the copy engines overlap the other fields' steps" +
                           (" (steps chained on the device by stream events)" if chain else ""),
                    "serial_value": e2e_serial,
                    "serial_api": "Solver.set_state/ssp_rk3_step/get_state, one field, no overlap"},
            "roofline": {"bound": "fp64", "kernel": "k_states_* (reconstruction+WENO-AO+limiter)",
                         "engine": ("DMMA (FP64 tensor, plane-marching; 3-D R=2: the 16-warp W-cache "
                                    "engine k_states_w where its TMA boxes apply)") if g.dim == 3
                         else "DFMA (unrolled, row-marching smem rings)",
                         # KXRCF mode: WENO runs only in flagged cells, so the
                         # WENO-everywhere flop count is not the work done
                         "achieved": None if g.kxrcf else achieved, "peak": fp64,
                         "unit": "TFLOP/s",
                         "frac": (achieved / fp64) if achieved and not g.kxrcf else None,
                         "peak_source": fp64_src,
                         "algorithmic_flops_per_cell_stage": None if g.kxrcf else F,
                         "traffic": None if g.kxrcf else traffic_of(w.index, g.shape)[0],
                         "traffic_source": None if g.kxrcf else traffic_of(w.index, g.shape)[1]},
            "kernel_ms_per_step": kt,
            "kxrcf": ({"enabled": True, "flagged_fraction_final_state": kx_frac}
                      if g.kxrcf else {"enabled": False}),
            "whole_step_fp64_frac": None if g.kxrcf else F * value / 1e12 / fp64,
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    s.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
