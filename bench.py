"""Benchmark of the B200-native OpenSBLI hot path (one JSON line on rank 0).

Metric (BASELINE.json): grid-point RK3 updates per second (fp64) — one update =
one full 3-stage low-storage RK3 step of one grid point — and the fraction of
the HBM roofline implied by the compulsory 400 B per point-step.

Default workload (N=1): BASELINE configs[3], the north-star case — Taylor-Green
vortex 256^3, 12th-order central differences, RK3, Re=1600, Pr=0.71, M=0.1,
gamma=1.4, dt = 3.385e-3*64/256.  configs[1] (64^3, 4th order)
fits in L2 and is a parity case.  N>1 (torchrun): weak scaling, 256^3 per GPU
(global 256 x 256 x 256N, z-slab decomposition, NCCL ghost exchange).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl osbli|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))


class _StdoutToStderr:
    """Route the process's C-level stdout (fd 1) to stderr while native code sets
    up communicators: NCCL prints a version banner there, and rank 0's stdout
    must carry exactly one JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self._saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self._saved, 1)
        os.close(self._saved)
        return False
sys.path.insert(0, ROOT)

CONFIGS = {
    "tgv256_o12": dict(n=256, order=12, scheme=1, desc="BASELINE configs[3]: TGV 256^3 12th order RK3"),
    "tgv256_o8": dict(n=256, order=8, scheme=1, desc="BASELINE configs[4]: TGV 256^3/GPU 8th order RK3"),
    "tgv256_o12_slab1": dict(n=256, order=12, scheme=1, slab1=True,
                             desc="TGV 256^3 12th order RK3 through the distributed path on one "
                                  "rank (ghost planes over NCCL self send/recv, boundary-first "
                                  "schedule): the slab path's own cost"),
    "tgv256_o12_strong": dict(n=256, order=12, scheme=1, strong=True,
                              desc="BASELINE configs[3]: TGV 256^3 12th order RK3, strong scaling "
                                   "(one 256^3 box split into z-slabs)"),
    "tgv64_o4": dict(n=64, order=4, scheme=1, desc="BASELINE configs[1]: TGV 64^3 4th order RK3"),
    # SURVEY §8(f) N2-N4 variants of the headline workload (not the driver's default line)
    "tgv256_o12_rk3_2r": dict(n=256, order=12, scheme=2,
                              desc="N2(a): TGV 256^3 12th order, two-register RK3 (D-25)"),
    "tgv256_o12_cons": dict(n=256, order=12, scheme=1, cons=True,
                            desc="N2(b): TGV 256^3 12th order RK3, conservative viscous work (D-27)"),
    "tgv256_o12_sutherland": dict(n=256, order=12, scheme=1, visc=True,
                                  desc="N4: TGV 256^3 12th order RK3, Sutherland mu(T), "
                                       "S/T_ref = 110.4/288 (D-26)"),
    "tgv256_o12_sym": dict(n=256, order=12, scheme=1, sym=True,
                           desc="N3: 256^3 12th order RK3 with symmetry boundaries in x, y, z "
                                "(TGV state; timing of the mirrored-halo kernels)"),
    # the paper's scalar verification equation in 3D
    "scalar256_o12": dict(n=256, order=12, scheme=1, scalar=True,
                          desc="N1: scalar advection-diffusion 256^3, 12th order RK3, "
                               "u = (1, -0.5, 0.25), k = 0.75 (P:205 parameters), dt = 0.05 dx^2/k (RK3-stable)"),
}


def run_scalar(args, cfg):
    """Replicas (one independent problem per rank): device-timed RK3 steps of the
    scalar advection-diffusion solver."""
    import numpy as np
    import torch

    import paper_1609_01277_b200 as osbli
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not torch.distributed.is_initialized():
        torch.distributed.init_process_group("nccl")
    torch.cuda.set_device(local)
    n, order = cfg["n"], cfg["order"]
    dx = 2 * math.pi / n
    u, kd = (1.0, -0.5, 0.25), 0.75
    # Courant number 0.02 (D-23) where the diffusion allows it; at 256^3 the 12th-order
    # Laplacian (spectral radius 7.07/dx^2 per direction) needs k dt/dx^2 <= 0.118 for RK3
    # stability, so dt = 0.05 dx^2/k there (per-point work does not depend on dt)
    dt = min(0.02 * dx, 0.05 * dx * dx / kd)
    s = osbli.ScalarSolver(n, n, n, order, dx, dt, u=u, kappa=kd)
    stream = torch.cuda.Stream()
    s.set_stream(stream.cuda_stream)
    x = np.arange(n) * dx
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    s.set_state(np.ascontiguousarray(np.sin(X) * np.cos(Y) * np.cos(Z)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        # warm-up of at least W steps and 1 s (the clock sampler's start-up)
        warm_up(lambda: s.step(1), s.sync, args.warmup, world)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        s.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        s.sync()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    if rank != 0:
        return
    value = world * n ** 3 * args.steps / (ms * 1e-3)
    peaks, src = measured_peaks()
    bytes_step = 80.0  # phi and W round trips of the three stages (24 + 32 + 24 B)
    achieved = value / world * bytes_step / 1e9
    print(json.dumps({
        "metric": "grid-point RK3 updates/s (fp64)", "value": value, "unit": "pt-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "grid": [n] * 3, "order": order,
                   "parallelism": f"replicas x{world}", "l2": "inputs larger than L2"},
        "roofline": {"kernel": "scalar_stage", "bound": "hbm", "achieved": achieved,
                     "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                     "frac": achieved / float(peaks["hbm_gbs"]), "traffic": None,
                     "bytes_per_point_step": bytes_step,
                     "timing": "CUDA events on the solver stream"},
        "clocks": clk.summary(),
        "gpu_launches": 3 * args.steps,
    }), flush=True)


def warm_up(step, sync, warmup, world, min_s=1.0):
    """Rounds of `warmup` steps until at least min_s seconds have passed on every
    rank; the decision is collective (a MIN all-reduce), so all ranks take the same
    number of steps."""
    import torch
    t_w = time.perf_counter()
    while True:
        for _ in range(warmup):
            step()
        sync()
        done = time.perf_counter() - t_w > min_s
        if world > 1:
            dev = "cuda" if torch.cuda.is_available() else "cpu"  # nccl / gloo
            t = torch.tensor([1.0 if done else 0.0], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
            done = bool(t.item() > 0.5)
        if done:
            return


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""
        else:
            self.out = ""

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


SUTH = 110.4 / 288.0


def host_cpu():
    """CPU model and logical CPU count of the host the oracle runs on."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def oracle_params(cfg, n, dx, dt):
    """OracleParams of a bench config (variants included) on an n^3 sample."""
    from inputs import TGV_PHYS
    from oracle import core
    return core.OracleParams(n, n, n, cfg["order"], dx, dt=dt, energy_form=int(cfg.get("cons", 0)),
                             visc_law=int(cfg.get("visc", 0)),
                             suth=SUTH if cfg.get("visc") else 0.0,
                             sym=(1, 1, 1) if cfg.get("sym") else (0, 0, 0), **TGV_PHYS)


def oracle_rate(cfg, dx: float, dt: float, budget_s: float, min_steps: int = 1):
    """Oracle (single-threaded C++) RK3 throughput on a bounded sample: a periodic
    24^3 grid at the workload's spacing, order, time step and TGV state."""
    from inputs import tgv
    from oracle import core
    n = 24
    p = oracle_params(cfg, n, dx, dt)
    Q = tgv(n, n, n, dx=dx)
    t0 = time.perf_counter()
    steps = 0
    while steps < min_steps or time.perf_counter() - t0 < budget_s:
        Q = core.step(p, Q, cfg["scheme"], 1)
        steps += 1
    el = time.perf_counter() - t0
    return n ** 3 * steps / el, steps, el, f"oracle RK3 on a periodic 24^3 TGV sample at the workload's dx/order/dt, {steps} steps, {el:.1f} s"


def run_reference(args, cfg, n_glob, dx, dt):
    """--impl reference: the oracle (this tier's reference arm), rank 0 only.
    W untimed + exactly K timed oracle RK3 steps, each on the bounded 24^3 sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from inputs import TGV_PHYS, tgv
    from oracle import core
    ns = 24
    if cfg.get("scalar"):
        dts = 0.02 * dx
        p = core.OracleParams(ns, ns, ns, cfg["order"], dx, dt=dts)
        x = np.arange(ns) * dx
        Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
        Q = np.sin(X) * np.cos(Y) * np.cos(Z)
        adv = lambda st, k: core.scalar_step(p, (1.0, -0.5, 0.25), 0.75, st, 1, k)  # noqa: E731
    else:
        p = oracle_params(cfg, ns, dx, dt)
        Q = tgv(ns, ns, ns, dx=dx)
        adv = lambda st, k: core.step(p, st, cfg["scheme"], k)  # noqa: E731
    for _ in range(args.warmup):
        Q = adv(Q, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Q = adv(Q, 1)
    el = time.perf_counter() - t0
    rate = ns ** 3 * args.steps / el
    sample = (f"oracle RK3 on a periodic {ns}^3 TGV sample at the workload's dx/order/dt "
              f"(per-point work identical to the {n_glob}^3 grid), {args.steps} steps, {el:.1f} s")
    line = {
        "impl": "reference", "metric": "grid-point RK3 updates/s (fp64)", "value": rate,
        "unit": "pt-steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "grid": [n_glob] * 3, "order": cfg["order"]},
        "cpu_baseline": {"value": rate, "unit": "pt-steps/s", "cores": 1, "kind": "oracle",
                         "host": host_cpu(),
                         "sample": sample},
        "e2e": {"value": rate, "unit": "pt-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="osbli", choices=["osbli", "reference"])
    ap.add_argument("--config", default="tgv256_o12", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=9)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    n = cfg["n"]
    dx = 2 * math.pi / n
    dt = 3.385e-3 * 64 / n
    if args.impl == "reference":
        run_reference(args, cfg, n, dx, dt)
        return
    if cfg.get("scalar"):
        run_scalar(args, cfg)
        return

    import numpy as np
    import torch

    import paper_1609_01277_b200 as osbli
    from inputs import TGV_PHYS, tgv
    from paper_1609_01277_b200 import perfmodel

    with _StdoutToStderr():
        rank, world, local, uid = osbli.init_distributed()
    torch.cuda.set_device(local)
    # weak scaling (default): 256^3 per GPU, TGV periods tiled in z; strong: one
    # 256^3 box split into z-slabs (BASELINE configs[3])
    nz_glob = n if cfg.get("strong") else n * world
    if cfg.get("slab1") and world == 1:
        uid = osbli.nccl_unique_id()
    with _StdoutToStderr():
        solver = osbli.Solver(n, n, nz_glob, cfg["order"], dx, dt, scheme=cfg["scheme"],
                              rank=rank, nranks=world, unique_id=uid, **TGV_PHYS)
    if cfg.get("visc"):
        solver.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, SUTH)
    if cfg.get("cons"):
        solver.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
    if cfg.get("sym"):
        for d in range(3):
            solver.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
    stream = torch.cuda.Stream()
    solver.set_stream(stream.cuda_stream)
    # input: this rank's slab of the global TGV, generated on the host, copied in
    Qfull = tgv(n, n, solver.nz, dx=dx) if world == 1 else None
    if Qfull is None:
        import numpy as _np
        z = (_np.arange(solver.nz) + solver.z0) * dx
        from inputs.generators import conservative
        Y, X = _np.meshgrid(_np.arange(n) * dx, _np.arange(n) * dx, indexing="ij")
        Z = z[:, None, None]
        g, M = TGV_PHYS["gamma"], TGV_PHYS["Minf"]
        u0 = _np.sin(X) * _np.cos(Y) * _np.cos(Z)
        u1 = -_np.cos(X) * _np.sin(Y) * _np.cos(Z)
        p = 1 / (g * M * M) + (_np.cos(2 * X) + _np.cos(2 * Y)) * (2 + _np.cos(2 * Z)) / 16
        Qfull = conservative(g * M * M * p, u0, u1, 0 * u0, p, g)
    solver.set_state(Qfull)
    npts_local = n * n * solver.nz
    npts_glob = n * n * nz_glob

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        # warm-up (also covers nvidia-smi start-up so that samples land in the timed region);
        # every rank takes the same number of steps (each step exchanges ghost planes)
        warm_up(lambda: solver.step(1), solver.sync, args.warmup, world)
        # ---- timed region: K steps, device-timed with CUDA events on the solver stream
        launches0 = solver.kernel_launches
        solver.set_kernel_timing(True)
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            solver.step(1)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = solver.kernel_launches - launches0
    ms = ev0.elapsed_time(ev1)
    zms, xyms, nzl, nxyl = solver.kernel_timing()
    solver.set_kernel_timing(False)
    solver.sync()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = npts_glob * args.steps / (ms * 1e-3)
    ms_per_step = ms / args.steps

    # ---- diagnostics of the current state through the public call
    # (synchronous: kernels, per-plane partials to the host, plane-order sum);
    # device time from events on the solver stream, and the call's wall time
    solver.diagnostics()
    d_ev0, d_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_diag = 5
    torch.cuda.synchronize()
    t_d = time.perf_counter()
    d_ev0.record(stream)
    for _ in range(n_diag):
        solver.diagnostics()
    d_ev1.record(stream)
    torch.cuda.synchronize()
    diag_wall_ms = (time.perf_counter() - t_d) * 1e3 / n_diag
    diag_ms = d_ev0.elapsed_time(d_ev1) / n_diag
    # the same diagnostics fused into every step (osbli_step_diag): K steps, each
    # with the diagnostics of its input state, device-timed like the main region
    torch.cuda.synchronize()
    barrier()
    d_ev0.record(stream)
    solver.step_diag(args.steps)
    d_ev1.record(stream)
    torch.cuda.synchronize()
    fused_ms_per_step = d_ev0.elapsed_time(d_ev1) / args.steps

    # ---- end to end through the public API with host buffers (pinned): every
    # step copies its input state in from the host and its result back out.
    # NE handles on their own streams take the steps in turn, so the host copies
    # of one (PCIe, both directions) overlap the steps of the others.
    NE = int(os.environ.get("OSBLI_E2E_HANDLES", "3"))
    qh = torch.from_numpy(np.ascontiguousarray(Qfull)).pin_memory()
    qos = [torch.empty_like(qh).pin_memory() for _ in range(NE)]
    e2e_solvers, e2e_streams = [solver], [stream]
    for _ in range(NE - 1):
        with _StdoutToStderr():
            s2 = osbli.Solver(n, n, nz_glob, cfg["order"], dx, dt, scheme=cfg["scheme"],
                              rank=rank, nranks=world,
                              unique_id=osbli.nccl_unique_id() if cfg.get("slab1") else None,
                              **TGV_PHYS) if world == 1 else None
        if s2 is None:
            break  # distributed: one communicator per rank; the handles share it in turn
        if cfg.get("visc"):
            s2.set_viscosity(osbli.OSBLI_VISC_SUTHERLAND, SUTH)
        if cfg.get("cons"):
            s2.set_energy_form(osbli.OSBLI_ENERGY_CONSERVATIVE)
        if cfg.get("sym"):
            for d in range(3):
                s2.set_boundary(d, osbli.OSBLI_BC_SYMMETRY)
        st2 = torch.cuda.Stream()
        s2.set_stream(st2.cuda_stream)
        e2e_solvers.append(s2)
        e2e_streams.append(st2)
    ne = len(e2e_solvers)

    def e2e_round(k_steps):
        for k in range(k_steps):
            s = e2e_solvers[k % ne]
            s.set_state_async(qh)        # H2D of the step's input
            s.step(1)
            s.get_state_async(qos[k % ne])  # D2H of the step's result

    e2e_round(ne)  # warm-up of the extra handles
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for st in e2e_streams[1:]:
        st.wait_event(e0)
    e2e_round(args.e2e_steps)
    for st in e2e_streams[1:]:
        ev = torch.cuda.Event()
        ev.record(st)
        stream.wait_event(ev)
    e1.record(stream)
    torch.cuda.synchronize()
    for s in e2e_solvers:
        s.sync()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = npts_glob * args.e2e_steps / (e2e_ms * 1e-3)
    state_bytes = 5 * 8 * npts_local

    if rank != 0:
        return
    peaks, peak_src = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    m = cfg["order"] // 2
    # dominant kernel: the one with the larger share of the timed step
    zflop, xyflop = perfmodel.flops(m)
    zb, xyb = perfmodel.step_kernel_bytes(cfg["scheme"])
    clocks = clk.summary()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    fp64_peak = 148 * 64 * 2 * fmax * 1e6 / 1e12  # TFLOP/s: 148 SMs x 64 FP64 FMA lanes x 2
    per_launch_pts = npts_local
    z_avg = zms / max(nzl, 1)
    xy_avg = xyms / max(nxyl, 1)
    dom = "xypass" if xyms >= zms else "zpass"
    avg = xy_avg if dom == "xypass" else z_avg
    fl = xyflop if dom == "xypass" else zflop
    achieved_tf = fl * per_launch_pts / (avg * 1e-3) / 1e12
    traffic = None
    fp64_pct = None
    tpath = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath)).get(f"{args.config}:{dom}")
        traffic = tj["dram_bytes_per_launch"] if tj else None
        fp64_pct = tj.get("fp64_pipe_pct") if tj else None
    roof = {
        "kernel": dom, "bound": "alu", "achieved": achieved_tf, "peak": fp64_peak,
        "unit": "TFLOP/s", "frac": achieved_tf / fp64_peak, "traffic": traffic,
        "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                        "profiles/kernel_traffic.json)",
        "algorithmic_bytes_per_launch": (xyb if dom == "xypass" else zb) / 3 * per_launch_pts,
        "peak_source": f"FP64 = 148 SMs x 64 lanes x 2 flop x {fmax:.0f} MHz (guide unit counts; DESIGN.md §5)",
        "flops_per_point": fl, "avg_launch_ms": avg,
        "ncu_fp64_pipe_pct": fp64_pct,  # sm__inst_executed_pipe_fp64 (same ncu capture as traffic)
        "flops_model": ("default operator (DESIGN.md §5); the variant's extra terms are not "
                        "counted, so frac is a lower bound") if any(
                            cfg.get(k) for k in ("visc", "cons", "sym")) else "DESIGN.md §5",
        "share_of_step": (xyms if dom == "xypass" else zms) / ms if ms > 0 else None,
        "other_kernel": {"name": "zpass" if dom == "xypass" else "xypass",
                         "avg_launch_ms": z_avg if dom == "xypass" else xy_avg,
                         "achieved_tflops": (zflop if dom == "xypass" else xyflop) * per_launch_pts
                         / ((z_avg if dom == "xypass" else xy_avg) * 1e-3) / 1e12},
        "kernel_bytes_per_point_step": {"zpass": zb, "xypass": xyb},
        "achieved_gbs": {"zpass": zb / 3 * per_launch_pts / (z_avg * 1e-3) / 1e9,
                         "xypass": xyb / 3 * per_launch_pts / (xy_avg * 1e-3) / 1e9},
    }
    hbm_frac = value / world * perfmodel.COMPULSORY_BYTES_RK3 / (hbm * 1e9)
    line = {
        "metric": "grid-point RK3 updates/s (fp64)", "value": value, "unit": "pt-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg["desc"], "grid": [n, n, nz_glob], "order": cfg["order"],
                   "scheme": {0: "euler", 1: "rk3", 2: "rk3-2r"}[cfg["scheme"]], "Re": 1600.0,
                   "dt": dt,
                   "variant": {k: cfg[k] for k in ("visc", "cons", "sym") if cfg.get(k)} or None,
                   "l2": "inputs larger than L2 (state 5 x 8 B x %d pts = %.0f MB per field-set)"
                   % (npts_local, state_bytes / 1e6),
                   "parallelism": f"z-slab x{world}"},
        "hbm_roofline_frac": hbm_frac,
        "hbm_roofline": {"compulsory_bytes_per_point_step": perfmodel.COMPULSORY_BYTES_RK3,
                         "peak_gbs": hbm, "peak_source": peak_src},
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": launches,
        "diagnostics": {"fused_ms_per_step": fused_ms_per_step,
                        "fused_overhead_share": fused_ms_per_step / ms_per_step - 1.0,
                        "ms_per_call": diag_ms, "wall_ms_per_call": diag_wall_ms,
                        "share_of_step": diag_ms / ms_per_step,
                        "how": "fused: osbli_step_diag(K) (diagnostics of every step's input "
                               "state in its first xy-pass, host sums every 64 steps) timed "
                               "like the main region; standalone: osbli_diagnostics (E_k, "
                               "enstrophy, dissipation) of the state, CUDA events on the "
                               "solver stream around 5 calls; wall_ms includes the host "
                               "plane-order sum"},
        "e2e": {"value": e2e_value, "unit": "pt-steps/s", "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes, "steps": args.e2e_steps,
                "how": f"osbli_set_state_async (pinned host -> device), osbli_step(1), "
                       f"osbli_get_state_async (device -> pinned host) every step, {ne} handles "
                       f"on their own streams taking the steps in turn"},
    }
    if world == 1 and not args.no_cpu_baseline:
        rate, steps, el, sample = oracle_rate(cfg, dx, dt, budget_s=15.0)
        line["cpu_baseline"] = {"value": rate, "unit": "pt-steps/s", "cores": 1, "kind": "oracle",
                                "host": host_cpu(),
                                "sample": sample}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
