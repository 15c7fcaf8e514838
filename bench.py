#!/usr/bin/env python
"""Benchmark of the SaP dense-banded hot path (BASELINE.json metric).

A step = one time-to-solution of BASELINE config 2: setup (factor_blocks LU/UL,
coupling, spike tips, reduced blocks) + solve (BiCGStab(2) to rel_tol 1e-10)
on N=200000, K=200, d=1.0, P=50 (testsup::random_banded, seed 1), with the band
already resident in HBM. It is larger than L2 (641.6 MB band), so no flush is
needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precond C|D] [--impl ours|reference]

Prints one JSON line on rank 0. Under torchrun (N>1) the same config-2 system is
solved with its partitions sharded over the ranks (strong scaling):
NCCL neighbour exchanges for the interfaces and halos, allreduce for the dots. `--impl reference` times the reference's own
CPU implementation (oracle/_ref, compiled from the unmodified reference
headers; single-threaded, as the reference is) on the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N, K, D, P, SEED = 200000, 200, 1.0, 50, 1
PAPER_K20X_S = {"C": 1.22129, "D": 0.567937}  # BASELINE.md §1, N=200000 K=200 P=50 d=1
FP64_PEAK_TFLOPS = 37.05  # DMMA m8n8k4, measured on this pool (profiles/fp64_peaks_r01.json)


def f_lu(m: int, k: int) -> float:
    """band_lu_inplace op count."""
    kk = min(k, max(m - 1, 0))
    return (m - kk) * (2 * kk * kk + kk) + (kk - 1) * kk * (4 * kk + 1) / 6.0


def metric_name(pre: str) -> str:
    return f"time-to-solution (s), dense banded N={N} K={K} d={D} P={P} SaP-{pre}"


def config(pre: str, world: int) -> dict:
    return {"workload": f"BASELINE config 2: dense banded N={N} K={K} d={D} P={P} SaP-{pre}, "
                        f"setup + BiCGStab(2) to rel_tol 1e-10, band resident in HBM",
            "n": N, "k": K, "d": D, "p": P, "precond": "coupled" if pre == "C" else "decoupled",
            "seed": SEED, "l2": "inputs larger than L2 (641.6 MB band), no flush",
            "parallelism": "single GPU"}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    import oracle as O
    pre = args.precond
    band, rhs = O.ref_random_banded(N, K, D, SEED)
    kind = 0 if pre == "C" else 1
    times, last = [], None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        x, st = O.ref_solve_banded(N, K, band, rhs, P, kind)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            last = st
    v = statistics.mean(times)
    line = {"metric": metric_name(pre), "value": v, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": v / PAPER_K20X_S[pre], "dtype": "f64",
            "data": f"synthetic (testsup::random_banded, seed {SEED})", "config": config(pre, 1), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "reference",
                             "sample": f"full config-2 SaP-{pre} solves (build_precond_op + run_krylov), "
                                       "oracle/_ref compiled -O3 -DNDEBUG from the unmodified reference; "
                                       "the reference is single-threaded per solve (proj/README.md:27-28)"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "breakdown": {"t_lu": last["t_lu"], "t_bc": last["t_bc"], "t_spk": last["t_spk"],
                          "t_lurdcd": last["t_lurdcd"], "t_kry": last["t_kry"], "iterations": last["iterations"],
                          "final_relative_residual": last["final_relative_residual"]}}
    print(json.dumps(line), flush=True)


def cpu_baseline(pre: str) -> dict:
    try:
        import oracle as O
        band, rhs = O.ref_random_banded(N, K, D, SEED)
        t0 = time.perf_counter()
        _, st = O.ref_solve_banded(N, K, band, rhs, P, 0 if pre == "C" else 1)
        v = time.perf_counter() - t0
        return {"value": v, "unit": "s", "cores": 1, "kind": "reference",
                "sample": f"1 full config-2 SaP-{pre} solve on the host (oracle/_ref, unmodified reference "
                          f"compiled -O3 -DNDEBUG, 1 thread); t_lu {st['t_lu']:.3f} s, t_kry {st['t_kry']:.3f} s, "
                          f"{st['iterations']} iterations"}
    except Exception as e:  # the checker is optional on a box without the prebuilt reference
        return {"value": None, "unit": "s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}


def run_ours(args) -> None:
    import ctypes as C
    import numpy as np
    import torch
    world, rank, local = dist_env()
    # SAP_BENCH_BACKEND=gloo lets several ranks share one GPU (a functional check of this script only)
    backend = os.environ.get("SAP_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_1509_07919_b200 as S
    from paper_1509_07919_b200 import _lib as L
    pre = args.precond
    kind = S.PrecondKind.coupled if pre == "C" else S.PrecondKind.decoupled
    band_h, rhs_h = S.random_banded(N, K, D, SEED)
    stream = torch.cuda.Stream()
    lib = L.load()

    def chk(rc):
        if rc:
            raise RuntimeError(lib.sap_last_error().decode())

    if world == 1:
        lo, hi, c0, c1 = 0, N, 0, N
        solver = S.Solver(p=P, precond=kind, device=local)
    else:
        # strong scaling: the same config-2 system, partitions sharded over the ranks
        from paper_1509_07919_b200.distributed import DistributedSolver, TorchComm, band_slice_columns
        comm = TorchComm()
        solver = DistributedSolver(comm, p=P, precond=kind, device=local)
        lo, hi = solver.rows(N, K)
        c0, c1 = band_slice_columns(N, K, lo, hi)
    w = 2 * K + 1
    band_loc = np.ascontiguousarray(band_h[c0 * w:c1 * w])
    rhs_loc = np.ascontiguousarray(rhs_h[lo:hi])
    band = torch.from_numpy(band_loc).cuda()
    rhs = torch.from_numpy(rhs_loc).cuda()
    solver.set_stream(stream)

    def setup(ptr, on_device):
        # device band passed through the public API and borrowed (no copy), like the reference's LinearOp
        if world == 1:
            chk(lib.sap_setup_banded(solver._h, N, K, C.c_void_p(ptr), on_device))
        else:
            chk(lib.sap_setup_banded_dist(solver._h, N, K, lo, hi, C.c_void_p(ptr), on_device))

    def step_dev():
        setup(band.data_ptr(), 2)
        return solver.solve(rhs)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            x, st = step_dev()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = solver.report()["kernel_launches"]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = []
    with Clocks(local) as clk:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                x, st = step_dev()
                reps.append(solver.report())
            e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = reps[-1]["kernel_launches"] - launches0

    rdev = "cuda" if backend == "nccl" else "cpu"

    def allmax(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=rdev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def allsum(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=rdev, dtype=torch.float64)
        torch.distributed.all_reduce(t)
        return float(t.item())

    ms = allmax(ms)
    value = ms * 1e-3
    assert st.converged and st.final_relative_residual <= 1e-10, st

    # dominant kernel: the block LU/UL factorization launch (max over ranks; flops summed)
    t_fk = allmax(statistics.median(r["t_factor_kernel"] for r in reps))
    flops = allsum(reps[-1]["factor_flops"])
    launches = int(allsum(launches))
    achieved = flops / t_fk / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_lu_traffic.json")
    if os.path.exists(prof) and world == 1:
        try:
            traffic = json.load(open(prof)).get(f"SaP-{pre}")
        except Exception:
            traffic = None
    peak = FP64_PEAK_TFLOPS * world
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_band_lu_res (block LU+UL, DMMA f64)",
                "peak_source": f"FP64 DMMA measured on this pool (profiles/fp64_peaks_r01.json) x {world} GPU; "
                               "MEASURED_PEAKS.json carries no FP64 figure",
                "algorithmic_flops_per_launch": flops, "launch_ms": t_fk * 1e3}

    # end to end through the public API with host buffers (pinned), H2D/D2H inside the timed region
    band_pin = torch.from_numpy(band_loc).pin_memory()
    rhs_pin = torch.from_numpy(rhs_loc).pin_memory()
    x_pin = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
    esteps = max(1, min(args.steps, 3))

    def step_e2e():
        setup(band_pin.data_ptr(), 0)
        st_ = L.sap_solve_stats()
        chk(lib.sap_solve(solver._h, C.c_void_p(rhs_pin.data_ptr()), C.c_void_p(x_pin.data_ptr()), 0,
                          C.byref(st_)))
        return st_

    with torch.cuda.stream(stream):
        step_e2e()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(esteps):
            ste = step_e2e()
        f1.record(stream)
    torch.cuda.synchronize()
    e2e = allmax(f0.elapsed_time(f1) / esteps * 1e-3)
    assert ste.converged
    h2d = allsum(band_loc.nbytes + rhs_loc.nbytes)
    d2h = allsum(x_pin.numpy().nbytes)

    if rank == 0:
        r = reps[-1]
        par = "single GPU" if world == 1 else f"partitions sharded over {world} GPUs (NCCL neighbour exchange)"
        cfg = config(pre, world)
        cfg["parallelism"] = par
        line = {"metric": metric_name(pre), "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": value / PAPER_K20X_S[pre], "dtype": "f64",
                "data": f"synthetic (testsup::random_banded N={N} K={K} d={D}, seed {SEED}; b = random_rhs)",
                "config": cfg, "roofline": roofline,
                "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                        "path": "sap_setup_banded[_dist](host band) + sap_solve(host b, host x), pinned buffers"},
                "gpu_launches": launches,
                "clocks": clk.summary(),
                "breakdown": {"t_lu": r["t_lu"], "t_factor_kernel": r["t_factor_kernel"], "t_bc": r["t_bc"],
                              "t_spk": r["t_spk"], "t_lurdcd": r["t_lurdcd"], "t_kry": r["t_kry"],
                              "iterations": st.iterations,
                              "final_relative_residual": st.final_relative_residual}}
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(pre)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precond", choices=["C", "D"], default="C")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
