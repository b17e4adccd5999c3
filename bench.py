#!/usr/bin/env python
"""AT-MGRIT hot-path benchmark (BASELINE.json metric: DOF*steps/s of batched
Phi relaxation; AT-MGRIT time-to-tolerance).

Workload (BASELINE config 5, the batch-scaling sweep): 1D heat, n = 4095
interior points, N_t = 2^18 steps on t in [0, 1], fp64, u0 = random_state(7, n),
two-level AT-MGRIT with m = 16, k = 8, F-relaxation, random initial guess
(seed 20).  One "step" = one AT-MGRIT iteration: F-relaxation with the fused
restriction tail, window exchange, 16385 truncated local coarse solves,
correction F-relaxation with the fused C-point norm tail, norm reduction and
its device->host read.  DOF*steps counts n x (relaxation Phi applications) =
n x 2 x F_0 per iteration (F_0 = 245760 fine F-points).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU: one process per GPU, time shards of the reference rank layout;
NCCL (from the C++ runtime) moves halo rows, window payloads and the norm
squares; gloo only broadcasts the NCCL id.  Under torchrun WORLD_SIZE must
equal --gpus; without a launcher, --gpus N > 1 re-launches itself through
torch.distributed.run with N local ranks.

CPU reference arm (--impl reference, and the cpu_baseline leg): the
reference's own CPU solver compiled from its sources (oracle/_ref/tempo_ref,
runtime::run_parallel over the host's threads) on the SAME workload (N_t =
2^18), W untimed + K timed iterations, seconds per iteration from the
reference's own ConvergenceReport::iteration_seconds (solver.cpp:414-416).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="config5_heat1d_n4095_Nt2^18_m16_k8", n=4095, n_points=2 ** 18 + 1, m=16, k=8,
                tf=1.0, u0_seed=7, guess_seed=20, tol=1e-10)


def level0_counts(n_points, m):
    nc = (n_points - 1) // m + 1
    F = n_points - nc
    n_iv = nc if (nc - 1) * m + 1 <= n_points - 1 else nc - 1
    return F, nc, n_iv


def dof_steps_per_iter(n, n_points, m):
    F, _, _ = level0_counts(n_points, m)
    return 2.0 * n * F


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """Measured FP64 peak of this GPU (tools/ubench/fp64_peak: independent
    DFMA chains on every SM, CUDA events), the secondary roofline of the
    Phi-chain kernels; MEASURED_PEAKS.json carries no FP64 figure."""
    exe = os.path.join(ROOT, "tools", "ubench", "fp64_peak")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
        d = json.loads(out.strip().splitlines()[-1])
        return float(d["fp64_tflops"]), "measured on this GPU at bench start (tools/ubench/fp64_peak)"
    except Exception:
        return 37.13, "fallback: tools/ubench/fp64_peak on a B200 of this pool (profiles/fp64_peak_r02.json)"


# algorithmic FP64 work of one heat1d Phi application: the
# serial Thomas solve of heat1d.cpp:47-60 with its constant-coefficient
# factors precomputed -- one FMA and one MUL forward, one FMA backward per
# unknown = 5 flops per unknown (an FMA counts 2)
FLOPS_PER_PHI_DOF = 5.0


class ClockSampler:
    """SM clock and clock-event reasons during the timed region (B200_PROFILING.md
    clocks line): NVML polled every 2 ms from a thread (the timed region of the
    default run is ~60 ms), nvidia-smi at 200 ms as the fallback."""

    def __init__(self, index=0):
        self.path = tempfile.mktemp(prefix="clocks_", suffix=".csv")
        self.proc = None
        self.index = index
        self.nv = None
        self.nv_sm, self.nv_reasons, self.nv_max = [], set(), None
        try:
            import threading

            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv_max = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.stop = threading.Event()
            self.th = threading.Thread(target=self._poll, daemon=True)
        except Exception:
            self.nv = None

    def _poll(self):
        nv = self.nv
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self.stop.is_set():
            try:
                self.nv_sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, b in bits.items():
                    if r & b:
                        self.nv_reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.th.start()
            return self
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.th.join(1.0)
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nv is not None:
            sm = self.nv_sm
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.nv_max,
                    "sm_min_mhz": min(sm) if sm else None, "reasons": sorted(self.nv_reasons),
                    "samples": len(sm), "source": "NVML, 2 ms polling during the timed region"}
        sm, mx, reasons = [], 0.0, set()
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_reference_run(warmup, steps, W, workers=None):
    """The compiled reference (oracle/_ref/tempo_ref: the reference's own
    solver sources, run_parallel) on the bench workload itself: `warmup`
    untimed + `steps` timed iterations; seconds per iteration from the
    reference's ConvergenceReport::iteration_seconds.  The C restatement
    (oracle/) stands in, single-threaded, only if the binary is missing."""
    from oracle import oracle as O
    n, npts = W["n"], W["n_points"]
    nproc = os.cpu_count() or 1
    nc = (npts - 1) // W["m"] + 1
    workers = min(workers or nproc, nc)
    iters = warmup + steps
    ic = O.random_state(W["u0_seed"], n)
    t0 = time.perf_counter()
    if O.ref_available():
        args = dict(problem="heat1d", n=n, tf=W["tf"], n_points=npts, m=W["m"], k=W["k"], manufactured=0,
                    guess="random", seed=W["guess_seed"], timing_iters=iters, workers=workers,
                    driver="parallel")
        res, _ = O.run_ref(args, files={"ic_file": ic}, timeout=7200)
        if "error" in res:
            raise RuntimeError(f"reference run failed: {res}")
        kind, secs, setup = "reference", res["iteration_seconds"], res["timings"].get("setup")
    else:  # the C restatement, single thread
        drv = O.Driver(dict(kind=O.HEAT1D, n=n, manufactured=0, ic=ic),
                       dict(tf=W["tf"], n_points=npts, m=W["m"], k=W["k"]),
                       dict(tol=1e-300, max_iters=iters, initial_guess=O.GUESS_RANDOM, seed=W["guess_seed"]))
        t = time.perf_counter()
        drv.setup()
        setup = time.perf_counter() - t
        secs = []
        for _ in range(iters):
            t = time.perf_counter()
            drv.cycle()
            drv.residual_norm()
            secs.append(time.perf_counter() - t)
        kind, workers = "port", 1
    timed = secs[warmup:] or secs
    per_iter = float(np.mean(timed))
    value = dof_steps_per_iter(n, npts, W["m"]) / per_iter
    desc = (f"the bench workload itself (heat1d n={n}, N_t={npts - 1}, m={W['m']}, k={W['k']}): "
            f"{warmup} untimed + {len(timed)} timed iterations of the reference's run_parallel "
            f"with {workers} threads")
    return dict(value=value, unit="DOF*steps/s", cores=workers, kind=kind, sample=desc,
                seconds_per_iteration=per_iter, seconds=secs, setup_seconds=setup,
                wall_seconds=time.perf_counter() - t0, cpu_model=cpu_model(), host_threads=nproc)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def time_to_tolerance(T):
    """Setup + solve to tol 1e-10 on config5r (n=4095, N_t=2^14, t in [0,1],
    m=16, k=8, u0 = random_state(7, n), guess seed 20), wall clock with the
    device synchronised (atm_solve reads each iteration's norm back)."""
    n, npts = 4095, 2 ** 14 + 1
    ref_it = ref_s = None
    try:
        case = json.load(open(os.path.join(ROOT, "tests", "golden", "cases.json")))["config5r_k8"]
        ref_it, ref_s = case["iterations"], case["ref_seconds"]
    except Exception:
        pass
    app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, npts), [16], 8)
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-10, max_iters=400,
                         initial_guess=T.InitialGuess.Random, seed=20)
    T.solve(app, hier, cfg)  # warm-up (module load, first-touch)
    t0 = time.perf_counter()
    res = T.solve(app, hier, cfg)
    wall = time.perf_counter() - t0

    def drive_only(reuse, cpts=False):
        drv = T.CycleDriver(app, hier, cfg, reuse_relax=reuse, cpoint_storage=cpts)
        t0 = time.perf_counter()
        drv.setup()
        t = time.perf_counter()
        rep = drv.drive()
        d = time.perf_counter() - t
        drv.close()
        drive_only.setup_to_tol = d + (t - t0)
        return rep, d

    rep1, d1 = drive_only(False)
    s2t = drive_only.setup_to_tol
    # opt-in: reuse the correction sweep's C-point residuals as the next
    # cycle's restriction input (bitwise the same iterations)
    rep2, d2 = drive_only(True)
    # opt-in: plus C-point-only level-0 storage (no F-row stores at all)
    rep3, d3 = drive_only(True, True)
    same = all(r.iterations == rep1.iterations and
               np.array_equal(np.array(r.residual_norms), np.array(rep1.residual_norms))
               for r in (rep2, rep3))
    return {"config": "config5r: heat1d n=4095, N_t=2^14, t in [0,1], m=16, k=8, tol 1e-10",
            "iterations": res.report.iterations, "reference_iterations": ref_it,
            "reference_seconds_fixture": ref_s,
            "converged": bool(res.report.converged), "seconds": wall,
            "setup_to_tol_seconds": s2t,
            "drive_seconds": d1, "drive_seconds_reuse_relax": d2,
            "drive_seconds_reuse_relax_cpoint_storage": d3,
            "opt_ins_bitwise_same_history": bool(same),
            "what": "seconds: wall clock of solve() (context + device arrays, setup, drive to tol with "
                    "one norm readback per iteration, level-0 state read back); setup_to_tol_seconds: "
                    "atm_setup to the converged iteration (SURVEY 8(d)); drive_seconds: the "
                    "iterations alone, without and with the opt-ins (relax reuse; relax reuse + C-point storage); "
                    "reference_seconds_fixture: the compiled reference's solve of the same case when its "
                    "fixture was written (tests/golden/cases.json; dev container, 8 threads)"}


def time_to_tolerance_full(T, W, name, app, hier, dev, world, rank, nccl_id, pg):
    """Setup + solve to 1e-10 on the bench workload itself (full N_t), on
    every rank of the job: atm_setup to the converged iteration, wall clock
    between barriers, max over ranks.  Runs the bitwise-neutral opt-ins
    (relax reuse + C-point storage: the default cycle's iterations and
    norms, tests/test_gpu_cpoints.py).  With a random guess the heat problem
    converges at the N_T/k front bound (test_solver.cpp:428-465)."""
    n_t = (W["n_points"] - 1) // W["m"]
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=W["tol"],
                         max_iters=2 * n_t // W["k"] + 100, initial_guess=T.InitialGuess.Random,
                         seed=W["guess_seed"])
    drv = T.CycleDriver(app, hier, cfg, device=dev, world_size=world, rank=rank, nccl_id=nccl_id,
                        reuse_relax=True, cpoint_storage=True)
    if pg:
        pg.barrier()
    t0 = time.perf_counter()
    drv.setup()
    rep = drv.drive()
    secs = time.perf_counter() - t0
    drv.close()
    if pg:
        import torch
        t = torch.tensor([secs], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        secs = float(t.item())
    return {"config": f"bench workload ({name}), tol {W['tol']:g}", "n_gpus": world,
            "iterations": rep.iterations, "front_bound": -(-n_t // W["k"]),
            "converged": bool(rep.converged), "setup_to_tol_seconds": secs,
            "last_norm": float(rep.residual_norms[-1]) if rep.residual_norms else None,
            "what": "atm_setup + drive to tol (one norm readback per iteration), wall clock, max over "
                    "ranks; relax reuse + C-point storage (bitwise the default cycle's iterations)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttt-full", action="store_true")
    ap.add_argument("--n-points", type=int, default=WORKLOAD["n_points"])
    ap.add_argument("--k", type=int, default=WORKLOAD["k"])
    ap.add_argument("--m", type=int, default=WORKLOAD["m"])
    args = ap.parse_args()
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # no launcher: one process per GPU through torch.distributed.run
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
               os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    W = dict(WORKLOAD, n_points=args.n_points, k=args.k, m=args.m)
    n = W["n"]
    unit = "DOF*steps/s"
    metric = "DOF*steps/s of batched Phi relaxation (AT-MGRIT iteration)"
    config = {"workload": W["name"] if (args.n_points, args.k, args.m) == (WORKLOAD["n_points"], WORKLOAD["k"], WORKLOAD["m"])
              else f"heat1d_n4095_Np{args.n_points}_m{args.m}_k{args.k}",
              "n_dof": n, "n_points": W["n_points"], "m": W["m"], "k": W["k"], "relaxation": "F",
              "mode": "two-level", "dtype": "f64", "global_batch": W["n_points"], "seq_len": n,
              "parallelism": f"time-shards{world}",
              "l2_flush": "inputs larger than L2 (8.59 GB level-0 array)"}

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference_run(args.warmup, args.steps, W)
        value, per = r["value"], r["seconds_per_iteration"]
        line = {"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded splitmix64 u0 and initial guess)", "config": config,
                "cpu_baseline": {"value": value, "unit": unit, "cores": r["cores"], "kind": r["kind"],
                                 "sample": r["sample"], "cpu_model": r["cpu_model"],
                                 "host_threads": r["host_threads"], "setup_seconds": r["setup_seconds"]},
                "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import paper_2107_09596_b200 as T

    nccl_id = None
    pg = None
    # one GPU per rank; BENCH_SHARE_DEVICE=1 puts every rank on device 0 (only
    # for exercising this path with the tests/mocknccl transport)
    dev = 0 if (world == 1 or os.environ.get("BENCH_SHARE_DEVICE") == "1") else local
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist

    def new_nccl_id():
        # one NCCL unique id per communicator (an id cannot be reused for a
        # second ncclCommInitRank): rank 0 draws it, gloo carries it
        if world == 1:
            return None
        import ctypes as C
        buf = (C.c_char * 128)()
        if rank == 0:
            assert T.lib().atm_nccl_unique_id(buf) == 0, "NCCL unavailable"
        obj = [bytes(buf) if rank == 0 else None]
        pg.broadcast_object_list(obj, src=0)
        return obj[0]

    ic = T.random_state(W["u0_seed"], n)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, W["tf"], W["n_points"]), [W["m"]], W["k"])
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=W["tol"],
                         max_iters=1_000_000, initial_guess=T.InitialGuess.Random, seed=W["guess_seed"])
    app = T.Heat1D(n, manufactured_forcing=False, initial_condition=ic)
    # the timed region runs the cycle as a user gets it (untraced: a single
    # process replays the captured CUDA graph); the phase split and the
    # dominant kernel's duration come from the same K iterations repeated
    # under per-phase CUDA events right after (`ms_per_step_traced`)
    drv = T.CycleDriver(app, hier, cfg, device=dev, world_size=world, rank=rank, nccl_id=new_nccl_id())
    drv.setup()
    drv.iterate(args.warmup)
    launches = drv.last_iteration_launches()
    if pg:
        pg.barrier()
    sampler = ClockSampler(dev) if rank == 0 else None
    if sampler:
        sampler.__enter__()
    norms, ms = drv.iterate_timed(args.steps)
    if sampler:
        sampler.__exit__()
    if pg:
        import torch
        t = torch.tensor([ms], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    drv.close()
    tr = T.CycleDriver(app, hier, cfg, device=dev, trace=True, world_size=world, rank=rank,
                       nccl_id=new_nccl_id())
    tr.setup()
    tr.iterate(args.warmup)
    t_before = tr.timings(with_counts=True)
    if pg:
        pg.barrier()
    norms_tr, ms_traced = tr.iterate_timed(args.steps)
    t_after = tr.timings(with_counts=True)
    tr.close()
    assert np.array_equal(norms, norms_tr), "traced and untraced cycles must be the same iterations"

    per_iter = dof_steps_per_iter(n, W["n_points"], W["m"])
    value = per_iter * args.steps / (ms / 1e3)
    # dominant kernel: the correction F-sweep (fused C-point norm tail)
    s1, c1 = t_after.get("sweep_correct", (0.0, 0))
    s0, c0 = t_before.get("sweep_correct", (0.0, 0))
    sweep_ms = 1e3 * (s1 - s0) / max(c1 - c0, 1)
    F0, nc0, niv0 = level0_counts(W["n_points"], W["m"])
    # algorithmic bytes of this rank's launch: write its F rows, read its seeds
    rr = T.rank_ranges(hier, world, rank)
    my_iv = rr["iv_count"][0]
    my_F = sum(min(iv * W["m"] + W["m"] - 1, W["n_points"] - 1) - iv * W["m"]
               for iv in range(rr["iv_first"][0], rr["iv_first"][0] + my_iv))
    sweep_bytes = 8.0 * n * (my_F + my_iv)
    peak, peak_src = read_peaks()
    achieved = sweep_bytes / (sweep_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_sweep_summary_r02.json")
    if not os.path.exists(prof):
        prof = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    phase_ms = {k: 1e3 * (v[0] - t_before.get(k, (0.0, 0))[0]) / args.steps for k, v in t_after.items()}
    # FP64 roofline of the two Phi-chain (latency-bound) kernels: the relax
    # F-sweep (one Phi per fine step of this rank: its F points and the
    # restriction tails) and the coarse window kernel (window p applies
    # min(p, k-1) Psi, kernels.cpp:53-61, for this rank's coarse points)
    fpk, fpk_src = fp64_peak() if rank == 0 else (None, None)
    relax_phi = my_F + my_iv
    lo1, hi1 = rr["lo"][1], rr["hi"][1]
    win_psi = sum(min(p, W["k"] - 1) for p in range(lo1, hi1 + 1))
    fp64 = {}
    for name, key, cnt in (("relax F-sweep (heat_sweep_kernel, restriction tail)", "sweep_relax", relax_phi),
                           ("coarse windows (heat_window_linear_kernel)", "coarse", win_psi)):
        ms_k = phase_ms.get(key)
        if ms_k and fpk:
            tf = FLOPS_PER_PHI_DOF * n * cnt / (ms_k / 1e3) / 1e12
            fp64[key] = {"kernel": name, "phi_per_launch": cnt, "flops_per_phi": FLOPS_PER_PHI_DOF * n,
                         "avg_launch_ms": ms_k, "achieved": tf, "frac": tf / fpk}

    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded splitmix64 u0 and initial guess, as the reference)",
            "config": config,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "heat_sweep_kernel<32,128,3> (level-0 correction F-sweep + C-point norm tail)",
                         "algorithmic_bytes_per_launch": sweep_bytes, "avg_launch_ms": sweep_ms,
                         "peak_source": peak_src,
                         "note": "the peak is a device-to-device copy (half reads, half writes); this "
                                 "sweep is 94% writes stored with an L2 evict_first policy, so frac can "
                                 "reach or slightly pass 1 (streaming stores alone: 6.67-6.70 TB/s on the "
                                 "same pool, profiles/ubench_wbw_r02.txt)"},
            "roofline_fp64": {"bound": "fp64 (Phi-chain latency)", "peak": fpk, "unit": "TFLOP/s",
                              "peak_source": fpk_src, "kernels": fp64},
            "gpu_launches": launches * args.steps,
            "ms_per_step_traced": ms_traced / args.steps,
            "phase_ms_per_step": phase_ms,
            "last_norm": float(norms[-1])}
    if sampler:
        line["clocks"] = sampler.summary()

    # ---- e2e through the public API with host buffers (pinned)
    if not args.no_e2e:
        npts = W["n_points"]
        # this rank's level-0 rows (its block plus the left halo row): only
        # these are filled, pinned, sent and read back
        r0 = max(0, rr["lo"][0] - 1)
        r1 = rr["hi"][0] + 1
        guess = np.empty((npts, n), np.float64)
        rng = np.random.default_rng(1234 + r0)
        for i0 in range(r0, r1, 16384):
            i1 = min(r1, i0 + 16384)
            guess[i0:i1] = rng.uniform(-1.0, 1.0, size=(i1 - i0, n))
        if r0 == 0:
            guess[0] = ic
        out = np.empty_like(guess)
        gsl, osl = guess[r0:r1], out[r0:r1]
        reg = T.lib().atm_host_register(gsl.ctypes.data, gsl.nbytes) == 0
        reg &= T.lib().atm_host_register(osl.ctypes.data, osl.nbytes) == 0
        cfg2 = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-300,
                              max_iters=args.steps, initial_guess=T.InitialGuess.Provided,
                              provided=guess)
        # defer_guess: atm_setup sends the guess's C rows; its F rows are dead
        # under cycling (rewritten before any read), so they never move
        drv2 = T.CycleDriver(app, hier, cfg2, device=dev, defer_guess=True,
                             world_size=world, rank=rank, nccl_id=new_nccl_id())
        if pg:
            pg.barrier()
        t0 = time.perf_counter()
        drv2.setup()                      # H2D of the provided level-0 guess
        rep = drv2.drive()                # K iterations, norms read back each iteration
        # D2H of the level-0 solution (this rank's own points)
        o0, o1 = rr["lo"][0], rr["hi"][0] + 1
        drv2.get_level(0, first=o0, count=o1 - o0, out=out[o0:o1])
        wall = time.perf_counter() - t0
        # bytes the engine actually moved (setup sends the guess's C rows:
        # its F rows are dead under cycling, see atm_host_traffic)
        h2d, d2h = drv2.host_traffic()
        if pg:
            import torch
            t = torch.tensor([wall], dtype=torch.float64)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            wall = float(t.item())
            tb = torch.tensor([h2d, d2h], dtype=torch.float64)
            pg.all_reduce(tb, op=pg.ReduceOp.SUM)
            h2d, d2h = int(tb[0].item()), int(tb[1].item())
        line["e2e"] = {"value": per_iter * rep.iterations / wall, "unit": unit,
                       "h2d_bytes_per_step": int(h2d / args.steps),
                       "d2h_bytes_per_step": int(d2h / args.steps + 8),
                       "guess_bytes_offered": int(gsl.nbytes * world),
                       "wall_s": wall, "pinned": bool(reg),
                       "what": "atm_setup(provided guess from pinned host: its C rows are sent, its F rows are dead under cycling) + atm_solve(K iterations) + atm_get_level(level 0) into pinned host"}
        drv2.close()
        if reg:
            T.lib().atm_host_unregister(gsl.ctypes.data)
            T.lib().atm_host_unregister(osl.ctypes.data)

    # ---- time-to-tolerance on the full bench workload, every rank
    ttf = None
    if not args.no_ttt_full:
        try:
            ttf = time_to_tolerance_full(T, W, config["workload"], app, hier, dev, world, rank,
                                         new_nccl_id(), pg)
            line["time_to_tolerance_full"] = ttf
        except Exception as e:  # reported, not fatal
            line["time_to_tolerance_full"] = {"unavailable": str(e)}

    # ---- time-to-tolerance (BASELINE metric, second half) on the config-5
    # shape at N_t = 2^14 (t in [0,1], k = 8), where the compiled reference's
    # iteration count is pinned (tests/golden/cases.json config5r_k8)
    ttt = None
    if world == 1:
        try:
            ttt = time_to_tolerance(T)
            line["time_to_tolerance"] = ttt
        except Exception as e:  # reported, not fatal
            line["time_to_tolerance"] = {"unavailable": str(e)}

    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            # the same workload and warm-up rule as --impl reference (1 + 2
            # iterations on all host threads), and one single-thread iteration
            cb = cpu_reference_run(1, 2, W)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"].update(cpu_model=cb["cpu_model"], host_threads=cb["host_threads"],
                                        seconds_per_iteration=cb["seconds_per_iteration"],
                                        setup_seconds=cb["setup_seconds"])
            try:
                c1 = cpu_reference_run(0, 1, W, workers=1)
                line["cpu_baseline"]["single_thread"] = {
                    "value": c1["value"], "seconds_per_iteration": c1["seconds_per_iteration"],
                    "setup_seconds": c1["setup_seconds"], "sample": c1["sample"]}
            except Exception as e:  # reported, not fatal
                line["cpu_baseline"]["single_thread"] = {"unavailable": str(e)}
            if ttf and "iterations" in ttf:
                # measured reference seconds per iteration (this workload, all
                # host threads) x the iterations the solve needs
                ttf["reference_seconds_estimate"] = cb["seconds_per_iteration"] * ttf["iterations"]
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": unit, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
