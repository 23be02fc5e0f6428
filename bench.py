"""Benchmark of the B200 HDG operator hot path (BASELINE.json metric:
"HDG operator DoF-applications/s (fp64) + % of HBM/FP64 roofline").

Workload (N=1, default): BASELINE config 3 -- inviscid Taylor-Green vortex,
M=0.1, on [-pi,pi]^3, n=32 (196,608 macro-tets, m=1), k=3, KEPES flux,
entropy variables, fp64: the largest configuration that fits one GPU
(config 4 needs >= 4).  The state is the projected initial
condition, linearized at stage 1 of the first DIRK step (alpha = d00/dt
with the paper's dt = 0.057 t_c = 0.57, offset = -alpha u_n, ptc_weight 1).

One step = one pass of the operator the Newton/FGMRES loop applies:
  residual      K1   DoFs = E*nc*5 + F*nt*5
  matvec        K3   DoFs = F*nt*5        (condensed trace operator)
  precond apply K4   DoFs = F*nt*5
value = DoF-applications / device time of the K timed steps (inputs
resident).  e2e = the same step through the public Discretization /
LinearizedSystem API with pinned host inputs copied in and results copied
out every step.  implicit_step = one DIRK(3,3) step through the public
integrator (device Krylov engine), jacobian_build = one linearization.

--impl reference: the UNMODIFIED reference package (macrohdg, installed in
oracle/_ref by oracle/build_ref.sh) on the host cores, one single-threaded
copy per core, on an n=4 sub-mesh of the same case (oracle/ref_bench.py);
it imports nothing from the repo package (no repo .so is loaded).

Under torchrun (N>1) the SAME global mesh is partitioned into N x-slabs
(strong scaling): every rank runs the partitioned operator (local
kernels + trace halo over NCCL, overlapped with the interior macros, plus
all-reduced dots); value = all ranks' DoF-applications / the max-over-ranks
device time.  --case tgv-visc --ncells 64 runs config 4 (>= 4 ranks).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HDG operator DoF-applications/s (fp64)"
UNIT = "DoF-applications/s"

CASES = {
    # case: (default flux, operator dt, implicit-step dt, label)
    "tgv": ("kepes", 0.57, 0.01425, "config3 inviscid Taylor-Green M=0.1"),
    "tgv-visc": ("kepes", 0.57, 0.01425, "config4 viscous Taylor-Green Re=1600 Pr=0.71 M=0.1"),
    "vortex": ("es", 0.01, 0.01, "config2 isentropic vortex"),
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--case", default="tgv", choices=sorted(CASES))
    ap.add_argument("--ncells", type=int, default=32, help="cells per axis (config 3: 32)")
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--m", type=int, default=1, help="macro subdivision (SURVEY f4: m = 2, 3)")
    ap.add_argument("--flux", default=None)
    ap.add_argument("--dt", type=float, default=None, help="operator linearization dt")
    ap.add_argument("--implicit-dt", type=float, default=None)
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-implicit", action="store_true", help="skip the implicit-step timing")
    ap.add_argument("--cpu-sample-n", type=int, default=4)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--cpu-workers", type=int, default=0, help="0: one per host core")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of the partitioned operator")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the partitioned operator also at N=1 (exchange-free)")
    ap.add_argument("--orth", default="mgs", choices=["mgs", "cgs2"],
                    help="partitioned runs: FGMRES orthogonalization (mgs = the reference's "
                         "order; cgs2 = opt-in, 3 all-reduces per Arnoldi step)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="partitioned runs: gloo stages the halo through host memory "
                         "(several ranks may then share one GPU)")
    a = ap.parse_args(argv)
    flux, dt, idt, _ = CASES[a.case]
    a.flux = a.flux or flux
    a.dt = a.dt or dt
    a.implicit_dt = a.implicit_dt or idt
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def make_problem(case, n, m=1):
    """Mesh, initial condition and viscous parameters of a BASELINE case
    (SURVEY 8d): repo objects, identical to the reference's definitions."""
    from paper_2507_22195_b200.cases import IsentropicVortex, TaylorGreen
    from paper_2507_22195_b200.gas import GasModel
    from paper_2507_22195_b200.mesh import build_box_macro_mesh

    gas = GasModel(1.4)
    visc = None
    if case.startswith("tgv"):
        ic = TaylorGreen(mach=0.1, gas=gas)
        box = ic.box
        if case == "tgv-visc":
            visc = ic.viscous_params(1600.0, prandtl=0.71)
    else:
        ic = IsentropicVortex(dim=3, mach=1 / math.sqrt(1.4), strength=5.0, v_inf=1.0,
                              center=(5.0, 5.0), gas=gas)
        box = np.array([[0.0, 10.0]] * 3)
    mesh = build_box_macro_mesh(box, n, m)
    return gas, mesh, ic, visc


def stage_alpha(dt):
    from paper_2507_22195_b200.time_march import dirk33_tableau

    return float(dirk33_tableau().d[0, 0] / dt)


def dof_units(E, F, nc, nt, viscous=False):
    """DoF-applications per step; nc / nt are the macro C0 nodes and the
    trace nodes per face (m > 1: the whole macro's C0 space)."""
    res = E * nc * 5 + F * nt * 5 + (E * nc * 15 if viscous else 0)
    return dict(residual=res, matvec=F * nt * 5, precond=F * nt * 5)


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md): NVML polled every 10 ms from a thread (nvidia-smi's
    100 ms period saw only two samples of a 160 ms region); nvidia-smi is the
    fallback when pynvml is absent."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_s=0.01):
        self.index, self.period = index, period_s
        self.proc = self.thread = None
        self.samples = []

    def __enter__(self):
        try:
            import threading

            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.stop = threading.Event()

            def poll():
                while not self.stop.is_set():
                    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(mhz), int(rs)))
                    self.stop.wait(self.period)

            self.pynvml = pynvml
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out = ""
            self.out = out
        return False

    def summary(self):
        if self.thread is not None:
            reasons = set()
            for _, rs in self.samples:
                for nm, attr in self.REASONS:
                    if rs & getattr(self.pynvml, attr):
                        reasons.add(nm)
            sm = [m for m, _ in self.samples]
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, 10 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(",") for r in getattr(self, "out", "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[2:6]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi, 100 ms"}


def cpu_workers(args):
    return args.cpu_workers or os.cpu_count() or 1


def cpu_baseline(args, steps=None, warmup=1):
    """The unmodified reference on the host cores (oracle/ref_bench.py)."""
    from oracle.ref_bench import time_reference

    return time_reference(case="vortex" if args.case == "vortex" else "tgv", n=args.cpu_sample_n,
                          p=args.p, flux=args.flux, dt=args.dt, m=args.m, workers=cpu_workers(args),
                          warmup=warmup, steps=steps, budget_s=args.cpu_budget)


def workload_name(args, E):
    return (f"{CASES[args.case][3]}, n={args.ncells} ({E} macros), k={args.p}, {args.flux}, "
            f"entropy variables, m={args.m}; step = residual + condensed matvec + face-block precond")


def run_reference(args, rank, world):
    """--impl reference: the reference package on the host cores, rank 0 only."""
    if rank != 0:
        return
    t0 = time.perf_counter()
    res = cpu_baseline(args, steps=args.steps, warmup=args.warmup)
    total = time.perf_counter() - t0
    E = 6 * args.ncells ** 3
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * res["seconds_per_step"], "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (projected initial condition, seeded x)",
        "config": {"workload": workload_name(args, E),
                   "sample": f"n={args.cpu_sample_n} sub-mesh ({6 * args.cpu_sample_n ** 3} macros)"
                             " per host core"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": total,
    }
    print(json.dumps(line), flush=True)


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def ncu_traffic(workload, kernel):
    """DRAM bytes per launch from the committed ncu --set full capture of the
    same workload (profiles/ncu_traffic.json), or None."""
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except (OSError, ValueError):
        return None, None
    ent = prof.get(workload, {})
    return ent.get(kernel), ent.get("source")


def kernel_model(E, F, nc, nt, nq, nqf, flux):
    """Algorithmic bytes / flops per launch."""
    NM, NB = 5 * nc, 5 * nt
    bytes_matvec = 8 * E * NM * NM + 3 * 8 * E * 4 * nqf * 25 + 2 * 8 * F * nt * 5 + \
        4 * E * 4 * (1 + nt) + 8 * E * 4
    bytes_precond = 8 * F * NB * NB + 2 * 8 * F * nt * 5
    T = 20    # flop-equivalents per exp / log / sqrt
    face_extra = (300 + 7 * T) if flux == "kepes" else 0
    flops_res = E * (nq * (10 * nc * 5 + 150 + 2 * T) +
                     4 * nqf * (8 * nt * 5 + 190 + 8 * T + face_extra))
    bytes_res = 8 * (2 * E * nc * 5 + 2 * F * nt * 5 + E * nq * 5) + 96 * E + 4 * E * 4 * (1 + nt)
    return bytes_matvec, bytes_precond, flops_res, bytes_res


class StepTimer:
    """CUDA events on the launching stream around each operator of a step."""

    def __init__(self, torch, steps, n):
        self.ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
                   for _ in range(steps)]

    def means(self, names):
        return {k: float(np.mean([e[a].elapsed_time(e[a + 1]) for e in self.ev]))
                for a, k in enumerate(names)}


def run_b200(args, rank, local_rank, world):
    import torch

    import __graft_entry__

    __graft_entry__.build()
    from paper_2507_22195_b200 import _native as N
    from paper_2507_22195_b200.assembly import Discretization, FieldSet, StageContext
    from paper_2507_22195_b200.fluxes import DissipationSpec

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)

    t_setup = time.perf_counter()
    gas, mesh, ic, visc = make_problem(args.case, args.ncells, args.m)
    disc = Discretization(mesh, p=args.p, gas=gas, formulation="entropy",
                          flux=DissipationSpec(args.flux), viscosity=visc, device=dev)
    t = disc.tables
    E, F, nc, nt = mesh.n_macros, t.n_faces, t.layout.n_unique, t.n_trace
    nq, nqf = t.phi.shape[0], t.fphi.shape[0]
    fields = disc.project(ic.initial)
    alpha = stage_alpha(args.dt)
    offset = (-alpha * disc.volume_quad_states(fields)).contiguous()
    stage = StageContext(alpha=alpha, offset=offset, dt=args.dt)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    lin = disc.jacobian(fields, stage, ptc_weight=1.0)
    x = torch.as_tensor(np.random.default_rng(1).standard_normal((F, nt, 5)), device=dev)
    torch.cuda.synchronize()

    units = dof_units(E, F, nc, nt, visc is not None)
    per_step = sum(units.values())
    stream = torch.cuda.current_stream()
    names = ("residual", "matvec", "precond")

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        res = disc.residuals(fields, stage, sync=False)
        if ev:
            ev[1].record(stream)
        y = lin.matvec(x)
        if ev:
            ev[2].record(stream)
        z = lin.apply_preconditioner(x)
        if ev:
            ev[3].record(stream)
        return res, y, z

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    code = N.load().mhdg_status_fetch(disc._ctx, None, N.stream_handle())
    assert code == 0, "non-admissible benchmark state"

    timer = StepTimer(torch, args.steps, 3)
    launches0 = disc.launch_count
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for i in range(args.steps):
            step(timer.ev[i])
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = disc.launch_count - launches0
    ms = start.elapsed_time(end)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    k_ms = timer.means(names)
    value = world * per_step * args.steps / (ms * 1e-3)

    # ---- e2e through the public API with pinned host buffers: every step
    # copies its inputs host->device and its results device->host.  Three
    # streams pipeline consecutive steps (inputs of step i+1 upload while
    # step i computes and step i-1's results download), double-buffered.
    w_h = fields.w.cpu().pin_memory()
    tr_h = fields.trace.cpu().pin_memory()
    off_h = offset.cpu().pin_memory()
    x_h = x.cpu().pin_memory()
    hosts = (w_h, tr_h, off_h, x_h)
    shapes = (fields.w.shape, fields.trace.shape, x.shape, x.shape)
    out_h = [[torch.empty(sh, dtype=torch.float64).pin_memory() for sh in shapes] for _ in range(2)]
    h2d = 8 * sum(h.numel() for h in hosts)
    d2h = 8 * sum(o.numel() for o in out_h[0])
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    s_cmp = stream
    dbuf = [[torch.empty_like(t_) for t_ in (fields.w, fields.trace, offset, x)] for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    started = [False, False]

    def e2e_step(i):
        b = i % 2
        wd, td, od, xd = dbuf[b]
        with torch.cuda.stream(s_in):
            if started[b]:
                s_in.wait_event(ev_cmp[b])          # step i-2 finished reading these buffers
            for d_, h_ in zip(dbuf[b], hosts):
                d_.copy_(h_, non_blocking=True)
            ev_in[b].record(s_in)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_in[b])
            fs = FieldSet(wd, td, fields.q)
            res = disc.residuals(fs, StageContext(alpha=alpha, offset=od), sync=False)
            y = lin.matvec(xd)
            z = lin.apply_preconditioner(xd)
            ev_cmp[b].record(s_cmp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_cmp[b])
            if started[b]:
                ev_out[b].synchronize()             # host buffers of step i-2 consumed
            for o, src in zip(out_h[b], (res.r_w, res.r_trace, y, z)):
                src.record_stream(s_out)
                o.copy_(src, non_blocking=True)
            ev_out[b].record(s_out)
        started[b] = True

    for i in range(3):
        e2e_step(i)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record(s_in)
    for i in range(args.e2e_steps):
        e2e_step(i)
    e2.record(s_out)
    torch.cuda.synchronize()
    e2e_ms = s2.elapsed_time(e2)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = world * per_step * args.e2e_steps / (e2e_ms * 1e-3)
    # the host link's own pinned H2D rate for this step's uploads
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_in):
        p0.record(s_in)
        for _ in range(3):
            for d_, h_ in zip(dbuf[0], hosts):
                d_.copy_(h_, non_blocking=True)
        p1.record(s_in)
    torch.cuda.synchronize()
    h2d_link_gbs = 3 * h2d / (p0.elapsed_time(p1) * 1e-3) / 1e9
    del dbuf, out_h

    # ---- roofline of each kernel; dominant one in the headline
    peaks = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"
    fp64_peak = N.fp64_probe(local_rank) / 1e3    # TFLOP/s, FMA-chain probe, this run
    dmma_peak = N.dmma_probe(local_rank) / 1e3    # TFLOP/s, DMMA probe, this run
    bytes_matvec, bytes_precond, flops_res, bytes_res = kernel_model(E, F, nc, nt, nq, nqf,
                                                                     args.flux)
    res_peak = max(fp64_peak, dmma_peak)
    kern = {
        "matvec": {"bound": "hbm", "achieved": bytes_matvec / (k_ms["matvec"] * 1e-3) / 1e9,
                   "peak": hbm_peak, "unit": "GB/s", "algorithmic_bytes": bytes_matvec,
                   "ms": k_ms["matvec"]},
        "precond": {"bound": "hbm", "achieved": bytes_precond / (k_ms["precond"] * 1e-3) / 1e9,
                    "peak": hbm_peak, "unit": "GB/s", "algorithmic_bytes": bytes_precond,
                    "ms": k_ms["precond"]},
        "residual": {"bound": "fp64", "achieved": flops_res / (k_ms["residual"] * 1e-3) / 1e12,
                     "peak": res_peak, "unit": "TFLOP/s", "algorithmic_flops": flops_res,
                     "hbm_gbs": bytes_res / (k_ms["residual"] * 1e-3) / 1e9,
                     "ms": k_ms["residual"],
                     "peak_source": "max(FP64 FMA probe, DMMA probe) measured in this run"},
    }
    for v in kern.values():
        v["frac"] = v["achieved"] / v["peak"]
    dom = max(kern, key=lambda k: kern[k]["ms"])
    wl_key = f"{args.case}_n{args.ncells}_k{args.p}_{args.flux}" + (f"_m{args.m}" if args.m > 1 else "")
    traffic, traffic_src = ncu_traffic(wl_key, dom)
    roofline = {"bound": kern[dom]["bound"], "achieved": kern[dom]["achieved"],
                "peak": kern[dom]["peak"], "unit": kern[dom]["unit"], "frac": kern[dom]["frac"],
                "traffic": traffic, "traffic_source": traffic_src, "kernel": dom,
                "peak_source": f"{hbm_src} MEASURED_PEAKS.json hbm_gbs" if kern[dom]["bound"] == "hbm"
                else kern[dom]["peak_source"]}

    # ---- one Jacobian build and one implicit DIRK(3,3) step (not in value)
    implicit = None
    if not args.no_implicit:
        from paper_2507_22195_b200.time_march import DIRKIntegrator

        del lin
        lin2 = disc.jacobian(fields, stage, ptc_weight=1.0)   # warms the allocator
        del lin2
        torch.cuda.synchronize()
        jb0 = time.perf_counter()
        lin2 = disc.jacobian(fields, stage, ptc_weight=1.0)
        torch.cuda.synchronize()
        jac_ms = 1e3 * (time.perf_counter() - jb0)
        del lin2
        integ = DIRKIntegrator(disc)
        torch.cuda.synchronize()
        st0 = time.perf_counter()
        integ.run(fields, t_final=args.implicit_dt, dt=args.implicit_dt)
        torch.cuda.synchronize()
        step_s = time.perf_counter() - st0
        rec = integ.records
        implicit = {"seconds_per_step": step_s, "jacobian_build_ms": jac_ms,
                    "newton_iters": sum(r["newton_iters"] for r in rec),
                    "fgmres_outer": sum(r["fgmres_iters"] for r in rec),
                    "fgmres_inner": sum(r["inner_iters_total"] for r in rec),
                    "jacobian_builds": sum(r["jacobian_builds"] for r in rec),
                    "dt": args.implicit_dt, "tableau": "DIRK(3,3)",
                    "halvings": integ.halvings,
                    "krylov": ("host loop" if os.environ.get("MHDG_KRYLOV") == "host" else
                               "device graph (solver.KrylovEngine)"),
                    "inner_residual": os.environ.get("MHDG_INNER_RESIDUAL", "arnoldi")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (projected initial condition, seeded x)",
            "config": {"workload": workload_name(args, E),
                       "macros": E, "faces": F, "dofs_per_step": per_step,
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                       "setup_s": setup_s,
                       "gpu_mem_peak_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
                       "l2": "inputs larger than L2: S^-1 (%.2f GB) streamed every step"
                             % (8 * E * (5 * nc) ** 2 / 1e9)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                    "pipeline": "H2D / compute / D2H on three streams, double-buffered",
                    "h2d_link_gbs": h2d_link_gbs,
                    "frac_of_link": (h2d / h2d_link_gbs / 1e9) / (e2e_ms * 1e-3 / args.e2e_steps)},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "kernels": kern,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "fp64_peak_tflops": fp64_peak,
            "dmma_peak_tflops": dmma_peak,
            "implicit_step": implicit,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_b200_partitioned(args, rank, local_rank, world):
    """N ranks, one x-slab of the same global mesh each (strong scaling),
    trace halo over NCCL."""
    import torch

    import __graft_entry__

    __graft_entry__.build()
    from paper_2507_22195_b200.assembly import FieldSet, StageContext
    from paper_2507_22195_b200.distributed import PartitionedDiscretization
    from paper_2507_22195_b200.fluxes import DissipationSpec
    from paper_2507_22195_b200.tables import HDGTables

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local_rank % ndev)
    torch.cuda.set_device(dev)
    if world > 1 or args.backend == "gloo":
        if args.backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:
            torch.distributed.init_process_group("gloo")
        # first collective over the whole group (NCCL's batched P2P requires
        # the communicator to exist before ranks exchange with neighbours only)
        torch.distributed.barrier()
    gas, mesh, ic, visc = make_problem(args.case, args.ncells)
    alpha = stage_alpha(args.dt)
    full = HDGTables(mesh, args.p)
    pdisc = PartitionedDiscretization(mesh, args.p, rank, world, device=dev, full_tables=full,
                                      gas=gas, formulation="entropy", viscosity=visc,
                                      flux=DissipationSpec(args.flux), orthogonalization=args.orth)
    disc = pdisc.local
    t = disc.tables
    part = pdisc.part
    E_l = part.macro_hi - part.macro_lo
    F_own, nc, nt = part.n_owned, t.layout.n_unique, t.fphi.shape[1]
    fields = disc.project(ic.initial)
    u_n = disc.volume_quad_states(fields)
    offset = (-alpha * u_n).contiguous()
    stage = StageContext(alpha=alpha, offset=offset, dt=args.dt)
    lin = pdisc.jacobian(fields, stage, ptc_weight=1.0)
    F_l = fields.trace.shape[0]
    x = torch.as_tensor(np.random.default_rng(1 + rank).standard_normal((F_l, nt, 5)), device=dev)
    torch.cuda.synchronize()
    units = dof_units(E_l, F_own, nc, nt, visc is not None)
    per_step = sum(units.values())
    tot = torch.tensor([float(per_step)], dtype=torch.float64, device=dev)
    pdisc.exchange.allreduce_sum(tot)
    per_step_all = float(tot.item())
    stream = torch.cuda.current_stream()
    names = ("residual", "matvec", "precond")

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        res = pdisc.residuals(fields, stage, sync=False)
        if ev:
            ev[1].record(stream)
        y = lin.matvec(x)
        if ev:
            ev[2].record(stream)
        z = lin.apply_preconditioner(x)
        if ev:
            ev[3].record(stream)
        return res, y, z

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    def barrier():
        if torch.distributed.is_initialized():
            torch.distributed.barrier()

    def max_over_ranks(v):
        tt = torch.tensor([v], dtype=torch.float64, device=dev)
        if torch.distributed.is_initialized():
            if args.backend == "gloo":
                h = tt.cpu()
                torch.distributed.all_reduce(h, op=torch.distributed.ReduceOp.MAX)
                return float(h.item())
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        return float(tt.item())

    timer = StepTimer(torch, args.steps, 3)
    launches0 = disc.launch_count
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for i in range(args.steps):
            step(timer.ev[i])
        end.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = disc.launch_count - launches0
    ms = max_over_ranks(start.elapsed_time(end))
    k_ms = {k: max_over_ranks(v) for k, v in timer.means(names).items()}
    value = per_step_all * args.steps / (ms * 1e-3)

    # e2e through the partitioned API with pinned host buffers
    w_h = fields.w.cpu().pin_memory()
    tr_h = fields.trace.cpu().pin_memory()
    off_h = offset.cpu().pin_memory()
    x_h = x.cpu().pin_memory()
    out_h = [torch.empty(s, dtype=torch.float64).pin_memory()
             for s in (fields.w.shape, fields.trace.shape, x.shape, x.shape)]
    h2d = 8 * (w_h.numel() + tr_h.numel() + off_h.numel() + x_h.numel())
    d2h = 8 * sum(o.numel() for o in out_h)

    def e2e_step():
        wd = w_h.to(dev, non_blocking=True)
        td = tr_h.to(dev, non_blocking=True)
        od = off_h.to(dev, non_blocking=True)
        xd = x_h.to(dev, non_blocking=True)
        res = pdisc.residuals(FieldSet(wd, td, fields.q), StageContext(alpha=alpha, offset=od),
                              sync=False)
        y = lin.matvec(xd)
        z = lin.apply_preconditioner(xd)
        for o, src in zip(out_h, (res.r_w, res.r_trace, y, z)):
            o.copy_(src, non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e2.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(s2.elapsed_time(e2))
    e2e_value = per_step_all * args.e2e_steps / (e2e_ms * 1e-3)
    # one implicit DIRK(3,3) step through the partitioned operator: Newton /
    # FGMRES control flow identical on every rank (all-reduced norms and dots)
    implicit = None
    if not args.no_implicit:
        from paper_2507_22195_b200.time_march import DIRKIntegrator

        del lin
        torch.cuda.synchronize()
        barrier()
        integ = DIRKIntegrator(pdisc)
        st0 = time.perf_counter()
        integ.run(fields, t_final=args.implicit_dt, dt=args.implicit_dt)
        torch.cuda.synchronize()
        step_s = max_over_ranks((time.perf_counter() - st0) * 1e3) * 1e-3
        rec = integ.records
        implicit = {"seconds_per_step": step_s,
                    "newton_iters": sum(r["newton_iters"] for r in rec),
                    "fgmres_outer": sum(r["fgmres_iters"] for r in rec),
                    "fgmres_inner": sum(r["inner_iters_total"] for r in rec),
                    "jacobian_builds": sum(r["jacobian_builds"] for r in rec),
                    "dt": args.implicit_dt, "tableau": "DIRK(3,3)",
                    "halvings": integ.halvings,
                    "krylov": f"host loop (distributed dots, {args.orth})",
                    "inner_residual": os.environ.get("MHDG_INNER_RESIDUAL", "arnoldi")}
    peaks = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    nqf = t.fphi.shape[0]
    NM = 5 * nc
    # rank-local matvec bytes (the exchange time is inside the measured interval)
    bytes_mv = 8 * E_l * NM * NM + 3 * 8 * E_l * 4 * nqf * 25 + 2 * 8 * F_l * nt * 5 + \
        4 * E_l * 4 * (1 + nt) + 8 * E_l * 4
    ach = bytes_mv / (k_ms["matvec"] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "traffic": None, "kernel": "matvec (incl. halo exchange)",
                "peak_source": "measured MEASURED_PEAKS.json hbm_gbs"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (projected initial condition, seeded x)",
            "config": {"workload": workload_name(args, mesh.n_macros) +
                       " through the partitioned operator",
                       "macros": mesh.n_macros, "macros_per_rank": E_l,
                       "owned_faces_rank0": F_own, "dofs_per_step": per_step_all,
                       "parallelism": f"{world} ranks, x-slab macro partition, trace halo + "
                                      f"allreduce over {args.backend}",
                       "l2": "inputs larger than L2: S^-1 streamed every step"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps},
            "gpu_launches": launches,
            "roofline": roofline,
            "kernels_ms": k_ms,
            "clocks": clk.summary(),
            "cpu_baseline": None,
            "implicit_step": implicit,
        }
        print(json.dumps(line), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if (world > 1 and not args.replicas) or args.partitioned:
        run_b200_partitioned(args, rank, local_rank, world)
        return
    run_b200(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
