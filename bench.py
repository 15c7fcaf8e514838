#!/usr/bin/env python
"""Benchmark of the SaP dense-banded hot path (BASELINE.json metric).

A step = one time-to-solution of BASELINE config 2: setup (factor_blocks LU/UL,
coupling, spike tips, reduced blocks) + solve (BiCGStab(2) to rel_tol 1e-10)
on N=200000, K=200, d=1.0, P=50 (testsup::random_banded, seed 1), with the band
already resident in HBM. It is larger than L2 (641.6 MB band), so no flush is
needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precond C|D] [--impl ours|reference]
                    [--no-config5] [--no-cpu-baseline]

Prints one JSON line on rank 0. `--gpus N` (N > 1) launches N ranks itself through torch.distributed.run
when it is not already running under torchrun (one process per GPU; under torchrun WORLD_SIZE must equal N).
N > 1 solves the same config-2 system with its partitions sharded over the ranks (strong scaling, SURVEY
§8e) on the library's native NCCL data plane (sap_create_distributed_nccl: grouped ncclSend/ncclRecv for the
spike tips, interface rows and halos, device ncclAllReduce for the Krylov dots); torch.distributed (gloo)
only bootstraps the NCCL id and reduces the timings. The line also carries `config5`: BASELINE config 5
(N=2000000, K=128, P=512, SaP-C) timed the same way at the same N, the configuration whose 1024 LU/UL
chains exceed one GPU's SMs. `--impl reference` times the reference's own CPU implementation (oracle/_ref,
compiled from the unmodified reference headers; single-threaded, as the reference is) on the same workload.
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


def relaunch(args) -> int:
    """--gpus N outside torchrun: run N ranks of this script through torch.distributed.run."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class pinned_core:
    """Run the single-threaded reference pinned to one host core (taskset to one core)."""

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        self.core = min(self.saved)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.saved)


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
        with pinned_core() as pc:
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
                             "cpu": cpu_model(), "pinning": f"sched_setaffinity to host core {pc.core}",
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
        with pinned_core() as pc:
            t0 = time.perf_counter()
            _, st = O.ref_solve_banded(N, K, band, rhs, P, 0 if pre == "C" else 1)
            v = time.perf_counter() - t0
        return {"value": v, "unit": "s", "cores": 1, "kind": "reference", "cpu": cpu_model(),
                "pinning": f"sched_setaffinity to host core {pc.core}",
                "sample": f"1 full config-2 SaP-{pre} solve on the host (oracle/_ref, unmodified reference "
                          f"compiled -O3 -DNDEBUG, 1 thread); t_lu {st['t_lu']:.3f} s, t_kry {st['t_kry']:.3f} s, "
                          f"{st['iterations']} iterations"}
    except Exception as e:  # the checker is optional on a box without the prebuilt reference
        return {"value": None, "unit": "s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}


class Rank:
    """This process's place in the job: device, bootstrap group (gloo) and the solver factory."""

    def __init__(self):
        import torch
        self.world, self.rank, self.local = dist_env()
        # SAP_BENCH_BACKEND=gloo: the sap_comm callback path with several ranks sharing one GPU (a functional
        # check of this script on a one-GPU box); default: the native NCCL data plane, one GPU per rank
        self.backend = os.environ.get("SAP_BENCH_BACKEND", "nccl")
        if self.backend != "nccl":
            self.local %= torch.cuda.device_count()
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist
        self.comm = None

    def solver(self, S, p, kind):
        if self.world == 1:
            return S.Solver(p=p, precond=kind, device=self.local)
        from paper_1509_07919_b200.distributed import DistributedSolver, NcclComm, TorchComm
        if self.comm is None:
            self.comm = NcclComm() if self.backend == "nccl" else TorchComm()
        return DistributedSolver(self.comm, p=p, precond=kind, device=self.local)

    def reduce(self, v, op):
        if self.world == 1:
            return v
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v):
        return v if self.world == 1 else self.reduce(v, self.dist.ReduceOp.MAX)

    def sum(self, v):
        return v if self.world == 1 else self.reduce(v, self.dist.ReduceOp.SUM)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()


def measure(R, S, L, n, k, d, p, pre, steps, warmup, clocks=None, e2e_steps=0):
    """Time `steps` device-resident time-to-solution steps (setup + solve) of one configuration on all ranks
    (CUDA events on the solver's stream, barrier + synchronize on both sides, max over ranks)."""
    import ctypes as C
    import numpy as np
    import torch
    lib = L.load()

    def chk(rc):
        if rc:
            raise RuntimeError(lib.sap_last_error().decode())

    kind = S.PrecondKind.coupled if pre == "C" else S.PrecondKind.decoupled
    band_h, rhs_h = S.random_banded(n, k, d, SEED)
    solver = R.solver(S, p, kind)
    if R.world == 1:
        lo, hi, c0, c1 = 0, n, 0, n
    else:
        from paper_1509_07919_b200.distributed import band_slice_columns
        lo, hi = solver.rows(n, k)
        c0, c1 = band_slice_columns(n, k, lo, hi)
    w = 2 * k + 1
    band_loc = np.ascontiguousarray(band_h[c0 * w:c1 * w])
    rhs_loc = np.ascontiguousarray(rhs_h[lo:hi])
    del band_h
    band = torch.from_numpy(band_loc).cuda()
    rhs = torch.from_numpy(rhs_loc).cuda()
    stream = torch.cuda.Stream()
    solver.set_stream(stream)

    def setup(ptr, on_device):
        # device band passed through the public API and borrowed (no copy), like the reference's LinearOp
        if R.world == 1:
            chk(lib.sap_setup_banded(solver._h, n, k, C.c_void_p(ptr), on_device))
        else:
            chk(lib.sap_setup_banded_dist(solver._h, n, k, lo, hi, C.c_void_p(ptr), on_device))

    def step_dev():
        setup(band.data_ptr(), 2)
        return solver.solve(rhs)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            x, st = step_dev()
    torch.cuda.synchronize()
    R.barrier()
    torch.cuda.synchronize()
    launches0 = solver.report()["kernel_launches"]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = []
    if clocks:
        clocks.__enter__()
    try:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                x, st = step_dev()
                reps.append(solver.report())
            e1.record(stream)
        torch.cuda.synchronize()
    finally:
        if clocks:
            clocks.__exit__(None, None, None)
    R.barrier()
    ms = R.max(e0.elapsed_time(e1) / steps)
    launches = int(R.sum(reps[-1]["kernel_launches"] - launches0))
    assert st.converged and st.final_relative_residual <= 1e-10, st
    # dominant kernel: the block LU/UL factorization launch (max over ranks; flops summed)
    t_fk = R.max(statistics.median(r["t_factor_kernel"] for r in reps))
    flops = R.sum(reps[-1]["factor_flops"])
    out = {"ms": ms, "launches": launches, "t_fk": t_fk, "flops": flops, "iterations": st.iterations,
           "residual": st.final_relative_residual, "report": reps[-1]}
    if e2e_steps:
        # end to end through the public API with host buffers (pinned), H2D/D2H inside the timed region
        band_pin = torch.from_numpy(band_loc).pin_memory()
        rhs_pin = torch.from_numpy(rhs_loc).pin_memory()
        x_pin = torch.empty(hi - lo, dtype=torch.float64).pin_memory()

        def step_e2e():
            setup(band_pin.data_ptr(), 0)
            st_ = L.sap_solve_stats()
            chk(lib.sap_solve(solver._h, C.c_void_p(rhs_pin.data_ptr()), C.c_void_p(x_pin.data_ptr()), 0,
                              C.byref(st_)))
            return st_

        with torch.cuda.stream(stream):
            step_e2e()
            torch.cuda.synchronize()
            R.barrier()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(e2e_steps):
                ste = step_e2e()
            f1.record(stream)
        torch.cuda.synchronize()
        assert ste.converged
        out["e2e"] = R.max(f0.elapsed_time(f1) / e2e_steps * 1e-3)
        out["h2d"] = R.sum(band_loc.nbytes + rhs_loc.nbytes)
        out["d2h"] = R.sum(x_pin.numpy().nbytes)
    solver.close()
    del band, rhs
    torch.cuda.empty_cache()
    return out


def run_ours(args) -> None:
    import torch
    R = Rank()
    import paper_1509_07919_b200 as S
    from paper_1509_07919_b200 import _lib as L
    pre = args.precond
    world = R.world
    clk = Clocks(R.local)
    m2 = measure(R, S, L, N, K, D, P, pre, args.steps, args.warmup, clocks=clk,
                 e2e_steps=max(1, min(args.steps, 3)))
    value = m2["ms"] * 1e-3
    achieved = m2["flops"] / m2["t_fk"] / 1e12
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
                "kernel": "k_band_lu_df (dataflow block LU+UL over every SM: pivot chains on claimed panel SMs, "
                          "DMMA f64 strips on the others)" if pre == "C" else
                          "k_band_lu_df (dataflow block LU over every SM: pivot chains on claimed panel SMs, "
                          "DMMA f64 strips on the others)",
                "peak_source": f"FP64 DMMA measured on this pool (profiles/fp64_peaks_r01.json) x {world} GPU; "
                               "MEASURED_PEAKS.json carries no FP64 figure",
                "algorithmic_flops_per_launch": m2["flops"], "launch_ms": m2["t_fk"] * 1e3}
    c5 = None
    if not args.no_config5:
        n5, k5, p5 = 2000000, 128, 512
        m5 = measure(R, S, L, n5, k5, 1.0, p5, "C", max(2, min(args.steps, 3)), max(1, min(args.warmup, 2)))
        a5 = m5["flops"] / m5["t_fk"] / 1e12
        c5 = {"workload": f"BASELINE config 5: dense banded N={n5} K={k5} d=1.0 P={p5} SaP-C, setup + "
                          "BiCGStab(2) to rel_tol 1e-10, band resident in HBM, partitions sharded over the ranks",
              "value": m5["ms"] * 1e-3, "unit": "s", "ms_per_step": m5["ms"], "n_gpus": world,
              "iterations": m5["iterations"], "final_relative_residual": m5["residual"],
              "factor_kernel_ms": m5["t_fk"] * 1e3, "factor_tflops": a5, "factor_frac": a5 / peak,
              "gpu_launches": m5["launches"]}
    if R.rank == 0:
        r = m2["report"]
        par = ("single GPU" if world == 1 else
               f"partitions sharded over {world} GPUs, " +
               ("native NCCL data plane (sap_create_distributed_nccl)" if R.backend == "nccl"
                else "sap_comm callbacks over gloo (ranks sharing a GPU)"))
        cfg = config(pre, world)
        cfg["parallelism"] = par
        line = {"metric": metric_name(pre), "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": m2["ms"], "higher_is_better": False, "scaling": "strong",
                "vs_baseline": value / PAPER_K20X_S[pre], "dtype": "f64",
                "data": f"synthetic (testsup::random_banded N={N} K={K} d={D}, seed {SEED}; b = random_rhs)",
                "config": cfg, "roofline": roofline,
                "e2e": {"value": m2["e2e"], "unit": "s", "h2d_bytes_per_step": int(m2["h2d"]),
                        "d2h_bytes_per_step": int(m2["d2h"]),
                        "path": "sap_setup_banded[_dist](host band) + sap_solve(host b, host x), pinned buffers"},
                "gpu_launches": m2["launches"],
                "clocks": clk.summary(),
                "breakdown": {"t_lu": r["t_lu"], "t_factor_kernel": r["t_factor_kernel"], "t_bc": r["t_bc"],
                              "t_spk": r["t_spk"], "t_lurdcd": r["t_lurdcd"], "t_kry": r["t_kry"],
                              "iterations": m2["iterations"], "final_relative_residual": m2["residual"]}}
        if c5 is not None:
            line["config5"] = c5
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(pre)
        print(json.dumps(line), flush=True)
    if world > 1:
        R.dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precond", choices=["C", "D"], default="C")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    world, _, _ = dist_env()
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
