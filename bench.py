#!/usr/bin/env python
"""bench.py — ∇G Monte-Carlo paths/s of the two-pass gradient (BASELINE.json).

Default workload: BASELINE config 5 — config 3's Heston model and 60-call
option set (756 full-truncation Euler steps) at P = 2^26 paths, fp64, on N
GPUs (one process per GPU under torchrun). A "step" is one full
gradient_of_G call: pass 1 + means/lambda/G + pass 2 + grad, all P paths.

  value  whole-job paths/s from device time (CUDA events the library records
         on its stream around each call), max over ranks;
  e2e    the same metric through the C-ABI call with host buffers (x and the
         targets in, the report out every step), wall clock bracketed by
         synchronisation, max over ranks — K further calls with the
         library's timing events off (ltg_set_timing), as a user runs it.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libltref.so, the unmodified lanetape headers compiled in place)
on this host's cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1901_04200_b200 import census, configs  # noqa: E402
from paper_1901_04200_b200.model import FP32, FP64, MCConfig  # noqa: E402

METRIC = "grad_G_mc_paths_per_sec"
UNIT = "paths/s"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class Clocks:
    """nvidia-smi sampling of the SM clock and throttle reasons (B200_PROFILING.md).

    Started before the warm-up so that nvidia-smi's own start-up (NVML init)
    is not inside the timed region; summary() keeps the samples whose
    timestamps fall in the timed window (or the one nearest to it when the
    window is shorter than the 200 ms sampling period)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.window = None

    def start(self):
        """start sampling and wait (<= 3 s) for the first sample, so that the
        sampler's own start-up (NVML init) is over before anything is timed"""
        import threading
        self.t_start = time.time()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                if line.strip():
                    self.lines.append(line.strip())
                    first.set()
            first.set()

        self.reader = threading.Thread(target=reader, daemon=True)
        self.reader.start()
        first.wait(3.0)
        return self

    def mark(self, t0: float, t1: float):
        """the timed region, in time.time() seconds"""
        self.window = (t0, t1)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.proc.wait()
            self.reader.join(timeout=5)
            self.proc = None

    def summary(self):
        import datetime
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[2]), float(f[3]),
                             {n for n, v in zip(names, f[6:10]) if v.lower() == "active"}))
            except ValueError:
                continue
        if self.window and rows:
            t0, t1 = self.window
            inside = [r for r in rows if t0 <= r[0] <= t1]
            if not inside:  # shorter than one sampling period: the nearest sample
                inside = [min(rows, key=lambda r: min(abs(r[0] - t0), abs(r[0] - t1)))]
            rows = inside
        sm = [r[1] for r in rows]
        reasons = set().union(*[r[3] for r in rows]) if rows else set()
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": rows[-1][2] if rows else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_rate(cfg, targets, sample_paths, workers, reps=1):
    """The reference's gradient_of_G (MCConfig{lane_width=8, workers, Recompute}) on a
    bounded sample; returns (paths/s, seconds)."""
    from oracle.bindings import Ref
    prog = Ref().program(cfg.spec)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        prog.gradient_of_G(cfg.x, targets, sample_paths, cfg.seed, lane_width=8, workers=workers)
        dt = time.perf_counter() - t0
        best = dt if best is None or dt < best else best
    return sample_paths / best, best


def size_cpu_sample(cfg, targets, workers, seconds):
    """Sample size for `seconds` of the reference's CPU work: a 1024-path probe,
    then a ~1 s probe (thread start-up makes the small one pessimistic)."""
    probe = 1024
    rate, _ = cpu_reference_rate(cfg, targets, probe, workers)
    probe2 = max(probe, int(rate) // 1024 * 1024)
    rate, _ = cpu_reference_rate(cfg, targets, probe2, workers)
    return max(probe, int(rate * seconds) // 1024 * 1024), rate


def build_cfg(name, paths):
    c = configs.ALL[name]() if name != "cfg5" else configs.cfg5()
    if paths:
        c.paths = paths
        if hasattr(c.spec, "mc"):
            c.spec.mc.paths = paths
    return c


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cfg = build_cfg(args.config, args.paths)
    targets = configs.load_targets(cfg) or [1.0] * cfg.m
    workers = os.cpu_count() or 1
    sample, _ = size_cpu_sample(cfg, targets, workers, args.ref_seconds)
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, targets, max(1024, sample // 8), workers)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_reference_rate(cfg, targets, sample, workers)
        times.append(dt)
    value = sample / statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world if world > 1 else args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg.name, "paths": cfg.paths,
                                        "sample_paths_per_step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference",
                         "sample": f"{sample} of the workload's paths per step, lane_width=8, "
                                   f"{workers} worker threads, recompute mode"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(configs.ALL))
    ap.add_argument("--paths", type=int, default=0, help="override the config's path count")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--ref-seconds", type=float, default=4.0,
                    help="target time of one --impl reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--method", default="adjoint", choices=["adjoint", "tangent"],
                    help="adjoint: the reference's two-pass scheme (the headline); tangent: "
                         "pass 2 replaced by pathwise forward tangents (small-M Heston only)")
    ap.add_argument("--no-alt-method", action="store_true",
                    help="skip the extra tangent-mode measurement reported under alt_methods")
    args = ap.parse_args()
    assert args.warmup >= 0 and args.steps >= 1
    rank, world, local = dist_env()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if world > 1 and args.gpus != world:
        # one process per GPU under torchrun: the job's GPU count is WORLD_SIZE
        ap.error(f"--gpus {args.gpus} under torchrun with WORLD_SIZE={world}: they must agree")
    # without torchrun, --gpus N > 1 runs one process over N devices
    # (ltg_create_*_devices: a member context per GPU, ncclCommInitAll); with
    # LTG_LOOPBACK=1 (tests) the N members share GPU 0
    loopback = os.environ.get("LTG_LOOPBACK") == "1"
    group = world == 1 and args.gpus > 1
    n_gpus = world if world > 1 else args.gpus

    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend="gloo")
        pg = dist

    if args.impl == "reference":
        rc = run_reference(args, rank, world)
        if pg:
            pg.barrier()
            pg.destroy_process_group()
        return rc

    from paper_1901_04200_b200.engine import (Engine, nccl_unique_id, probe_fp32_rate,
                                              probe_fp64_rate)

    cfg = build_cfg(args.config, args.paths)
    targets = configs.load_targets(cfg)
    if targets is None:
        # separate-seed forward run at the truth (synthetic_targets, calibrate.hpp:224-227)
        e0 = Engine(cfg.spec, device=local)
        targets = e0.estimate_means(cfg.truth, MCConfig(paths=configs.TARGET_PATHS,
                                                        seed=configs.TARGET_SEED)).means
        e0.close()
    if group:
        devices = [0] * n_gpus if loopback else list(range(n_gpus))
        try:
            eng = Engine(cfg.spec, devices=devices)
        except (ValueError, RuntimeError) as e:
            raise SystemExit(f"bench.py --gpus {n_gpus}: cannot open devices {devices}: {e}")
    else:
        eng = Engine(cfg.spec, device=local)
    if world > 1:
        import torch
        obj = [nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(obj, src=0)
        eng.attach_nccl(obj[0], rank, world)
    mc = MCConfig(paths=cfg.paths, seed=cfg.seed,
                  precision=FP32 if args.precision == "fp32" else FP64)

    clk = Clocks(local).start()
    # the C-ABI call on host buffers (the adjoint; the tangent method through
    # the Python wrapper), as a C / C++ caller of ltg_gradient_of_G makes it
    if args.method == "adjoint":
        call, xbuf, tbuf, _ = eng.prepared_gradient(cfg.x, targets, mc)
        x_host = np.asarray(cfg.x, dtype=np.float64)
    for _ in range(args.warmup):
        eng.gradient_of_G(cfg.x, targets, mc, method=args.method)
        if args.method == "adjoint":
            call()

    # ---- timed region: K full gradient_of_G calls, device-timed (CUDA events
    # around the passes) ----
    if pg:
        pg.barrier()
    dev_ms, p1_ms, p2_ms, launches = [], [], [], 0
    e0 = time.time()
    for _ in range(args.steps):
        if args.method == "adjoint":
            np.copyto(xbuf, x_host)
            call()
        else:
            eng.gradient_of_G(cfg.x, targets, mc, method=args.method)
        tm = eng.timing()  # the call's device events
        dev_ms.append(tm["total_ms"])
        p1_ms.append(tm["pass1_ms"])
        p2_ms.append(tm["pass2_ms"])
        launches += tm["launches"]
    # ---- end to end: K more calls as a user makes them — host buffers in (x
    # copied into the caller's array), the report out, synchronised — with
    # the library's timing events off (ltg_set_timing: they are profiling,
    # not part of the call), wall-clocked ----
    eng.set_timing(False)
    for _ in range(2):  # (the call graph re-captured without its event nodes)
        call() if args.method == "adjoint" else eng.gradient_of_G(cfg.x, targets, mc,
                                                                   method=args.method)
    if pg:
        pg.barrier()
    wall = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        if args.method == "adjoint":
            np.copyto(xbuf, x_host)
            call()
        else:
            eng.gradient_of_G(cfg.x, targets, mc, method=args.method)
        wall += time.perf_counter() - t0
    eng.set_timing(True)
    clk.mark(e0, time.time())
    clk.stop()
    rep = eng.gradient_of_G(cfg.x, targets, mc, method=args.method)  # (the report, untimed)
    clocks = clk.summary()
    dev_total = sum(dev_ms)
    if pg:
        import torch
        t = torch.tensor([dev_total, wall, sum(p2_ms), sum(p1_ms)], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        dev_total, wall, p2_tot, p1_tot = t.tolist()
    else:
        p2_tot, p1_tot = sum(p2_ms), sum(p1_ms)

    # ---- the same workload through the tangent-mode alternative (reported
    # beside the headline, never instead of it) ----
    alt = None
    if args.method == "adjoint" and not args.no_alt_method:
        try:
            rt = eng.gradient_of_G(cfg.x, targets, mc, method="tangent")
        except ValueError:  # not a small-M fp64 Heston model: adjoint only
            rt = None
        if rt is not None:
            for _ in range(max(0, args.warmup - 1)):
                eng.gradient_of_G(cfg.x, targets, mc, method="tangent")
            if pg:
                pg.barrier()
            t_dev, t_wall = 0.0, 0.0
            for _ in range(args.steps):
                t0 = time.perf_counter()
                rt = eng.gradient_of_G(cfg.x, targets, mc, method="tangent")
                t_wall += time.perf_counter() - t0
                t_dev += eng.timing()["total_ms"]
            if pg:
                import torch
                t = torch.tensor([t_dev, t_wall], dtype=torch.float64)
                pg.all_reduce(t, op=pg.ReduceOp.MAX)
                t_dev, t_wall = t.tolist()
            diff = max(abs(a - b) / max(abs(a), abs(b), 1e-12 * max(map(abs, rep.grad)))
                       for a, b in zip(rt.grad, rep.grad))
            alt = {"tangent": {
                "value": cfg.paths * args.steps / (t_dev * 1e-3), "unit": UNIT,
                "e2e": cfg.paths * args.steps / t_wall, "ms_per_step": t_dev / args.steps,
                "grad_rel_diff_vs_adjoint": diff,
                "what": "pass 2 replaced by pathwise forward tangents "
                        "(ltg_gradient_of_G_tangent): same paths and estimator, "
                        "grad = sum_i lambda_i J_i / P"}}

    out = None
    if rank == 0:
        K = args.steps
        value = cfg.paths * K / (dev_total * 1e-3)
        e2e = cfg.paths * K / wall
        fp32 = args.precision == "fp32"
        # fp64: FP64 issue; fp32 mode: its FP32 arithmetic against the FFMA rate
        peak = probe_fp32_rate(local) if fp32 else probe_fp64_rate(local)
        # dominant kernel of the step (device time) and the census of both
        # passes (census.py): ALGORITHMIC = the kernels' executed floating-point
        # instructions minus their redundant ones (AS241's central branch on
        # tail slots); pass 2 weighted by the share of paths whose draws came
        # from the draw store (z_bytes) instead of being regenerated
        dom = "pass2" if p2_tot >= p1_tot else "pass1"
        basket = not hasattr(cfg.spec, "mc")
        kname = ("basket_" if basket else "heston_") + dom + "_kernel"
        prec = args.precision
        steps = cfg.spec.steps if basket else cfg.spec.mc.steps
        elem = 8 if fp32 else 16
        paths_rank = tm["paths_pass2"] if dom == "pass2" else tm["paths_pass1"]
        zf = 0.0 if basket else min(1.0, tm["z_bytes"] / (steps * elem * max(1, tm["paths_pass1"])))
        w = {b: {k: census.per_path(cfg.name, prec, k, zf, b) for k in ("pass1", "pass2")}
             for b in ("algorithmic", "executed")}
        if args.method == "tangent":  # one forward+tangent kernel; no census
            kname = "heston_tangent_kernel"
            w = {b: {"pass1": None, "pass2": None} for b in w}
        t_dom = (p2_tot if dom == "pass2" else p1_tot) / K * 1e-3
        t_step = dev_total / K * 1e-3

        def rate(basis, kernels, t):
            ws = [w[basis][k] for k in kernels]
            return sum(ws) * paths_rank / t if all(v is not None for v in ws) else None

        achieved = rate("algorithmic", [dom], t_dom)
        ach_exec = rate("executed", [dom], t_dom)
        step_alg = rate("algorithmic", ["pass1", "pass2"], t_step)
        step_exec = rate("executed", ["pass1", "pass2"], t_step)
        roof = {"bound": "fp32" if fp32 else "fp64", "kernel": kname,
                "achieved": achieved / 1e12 if achieved else None,
                "peak": peak / 1e12, "unit": "T fp32-inst/s" if fp32 else "T fp64-inst/s",
                "frac": (achieved / peak) if achieved else None, "traffic": None,
                "basis": ("algorithmic: the kernels' executed " +
                          ("FADD+FMUL+FFMA" if fp32 else "DADD+DMUL+DFMA") +
                          " per path (ncu census, profiles/r4_census.txt) minus the redundant "
                          "AS241 central-branch evaluations on tail slots; pass 2 weighted by "
                          "the draw-store share"),
                "census_inst_per_path": {b: w[b] for b in w},
                "draw_store_path_fraction": zf,
                "executed_frac": (ach_exec / peak) if ach_exec else None,
                "whole_step_frac": (step_alg / peak) if step_alg else None,
                "whole_step_executed_frac": (step_exec / peak) if step_exec else None,
                "peak_source": ("measured in this run: ltg_probe_fp32_rate (FFMA streams; 8 "
                                "chains/thread, full occupancy)") if fp32 else
                               ("measured in this run: ltg_probe_fp64_rate (fastest of DFMA, "
                                "DMUL+DADD, DADD streams; 8 chains/thread, full occupancy)")}
        # cross-check against SURVEY.md §8(d)'s preliminary W (FP64 issues per
        # path with its per-op weights; it credits both passes with drawing
        # every normal, also where pass 2 reads the draw store)
        w8d = census.survey_w(cfg.name) if not fp32 and args.method == "adjoint" else None
        if w8d is not None:
            roof["survey_8d"] = {
                "W_per_path": w8d,
                "whole_step_frac": w8d * paths_rank / t_step / peak,
                "note": "SURVEY.md §8(d) preliminary W (not the census): an upper figure — it "
                        "credits pass 2 with drawing every normal, so it exceeds what the "
                        "kernels execute wherever pass 2 reads the draw store (and can pass 1.0 "
                        "when every path's draws are stored); the bench's frac stays the census"}
        trf = census.dram_per_path(cfg.name, prec, dom, zf)
        if trf is not None and args.method == "adjoint":
            # ncu DRAM bytes/path of the dominant kernel (with and without the
            # draw store), weighted like the census; per launch
            roof["traffic"] = trf * paths_rank
        M, m = len(cfg.x), cfg.m
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": K,
            "warmup": args.warmup, "ms_per_step": dev_total / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic (seeded Philox paths; no dataset)",
            "config": {"workload": cfg.name, "model": cfg.description, "paths": cfg.paths,
                       "seed": cfg.seed,
                       "parallelism": f"path-sharded dp{n_gpus}" + (
                           " (one process, ltg_create_*_devices)" if group else
                           " (torchrun, one process per GPU)" if world > 1 else ""),
                       "l2": "working set > L2: HBM checkpoint/store table "
                             f"{tm['ckpt_bytes']/1e9:.1f} GB rewritten every step",
                       "checkpoint_interval_steps": tm["seg_steps"]},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * (M + m),
                    "d2h_bytes_per_step": 8 * (1 + 3 * m + M),
                    "transfer": ("x and the targets in the kernels' launch arguments (one "
                                 "H2D copy when a model has > 32 leverage cells or > 64 "
                                 "targets); the report written by the call's last kernel "
                                 "into pinned host memory" if n_gpus == 1 and not group else
                                 "one H2D copy of [x | targets] and one D2H copy of the "
                                 "report per rank")},
            "gpu_launches": launches,
            "clocks": clocks,
            "roofline": roof,
            "pass_ms": {"pass1": p1_tot / K, "pass2": p2_tot / K},
            "method": args.method,
            "G": rep.G,
            "report_sha1": hashlib.sha1(rep.to_json().encode()).hexdigest(),
            "rng_exact": eng.rng_exact,
        }
        if group and loopback:
            line["config"]["loopback"] = "LTG_LOOPBACK=1: the members share GPU 0 (test mode)"

        if n_gpus == 1 and not args.no_cpu_baseline:
            workers = os.cpu_count() or 1
            try:
                sample, _ = size_cpu_sample(cfg, targets, workers, args.cpu_seconds)
                rate, secs = cpu_reference_rate(cfg, targets, sample, workers)
                line["cpu_baseline"] = {
                    "value": rate, "unit": UNIT, "cores": workers, "kind": "reference",
                    "sample": f"{sample} paths of {cfg.name} through the reference's "
                              f"gradient_of_G (lane_width=8, recompute), {secs:.1f} s"}
            except Exception as e:  # the oracle is optional on the box
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": workers,
                                        "kind": "reference", "sample": f"unavailable: {e}"}
        if alt:
            line["alt_methods"] = alt
        out = line
        print(json.dumps(out), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
