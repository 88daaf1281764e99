"""Benchmark of the SIP-DG implicit-stage hot path on B200 (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl product|reference] [--workload c5]

Workload: BASELINE.json configs[4] (c5), the largest single-GPU
config and the one the north star's scaling target names: periodic [0,2pi]^3, 64^3 hexes,
P = 5 (56.6 M DOF), variable nu = 1e-3 (1 + 0.5 tanh(4 sin x sin y sin z)), lam = 229.43.

step  = one SIP-DG Helmholtz apply (BASELINE metric "GDOF/s SIP-DG Helmholtz apply") of the
        whole mesh; value = global DOF / step time (GDOF/s), max over ranks (strong scaling).
pcg   = Jacobi-PCG solves of the same workload to tol 1e-10 from u0 = 0 (iterations/s).
e2e   = the same apply metric through the C-ABI host-buffer call (H2D of u and nu and D2H
        of the result inside the timed region).
Inputs (453 MB per field) are larger than L2 (126 MB): no explicit flush is needed.

--impl reference times the CPU oracle (oracle/, C + OpenMP, explicit quadrature) on a
bounded sample of the same workload (the tier's reference arm); under torchrun only
rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import config as get_config  # noqa: E402

WORKLOADS = {"c5": 5, "c4": 4, "c3": 3, "c2": 2, "c1": 1}
BYTES_PER_DOF = {True: 24.0, False: 16.0}  # algorithmic bytes per DOF per apply (var / const nu)
# bytes per DOF per fused PCG iteration: apply MODE 1 (read z, p_old, [nu];
# write p, q) + update (read x, r, p, q, dinv; write x, r, z)
PCG_BYTES_PER_DOF = {True: 104.0, False: 96.0}


_JSON_FD = None


def emit(line):
    """The one JSON line on the ORIGINAL stdout (everything else -- NCCL's banner, library
    prints -- goes to stderr, see main)."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# seeded inputs for one rank's slab (identical values to the global canonical arrays;
# tests/test_multirank_gloo.py checks that)
# ---------------------------------------------------------------------------
def measure_traffic(workload_id, kernel_regex="k_apply", timeout_s=240):
    """DRAM bytes (read + write) of one launch of the dispatched apply kernel, measured by ncu
    on tools/one_apply.py for THIS build (a byte count, not a timing).  None + reason if ncu is
    unavailable or fails."""
    ncu = None
    for cand in ("/usr/local/cuda/bin/ncu", "ncu"):
        try:
            subprocess.run([cand, "--version"], capture_output=True, timeout=30, check=True)
            ncu = cand
            break
        except Exception:
            continue
    if ncu is None:
        return None, "ncu not available"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "-k", "regex:" + kernel_regex, "-s", "1",
           "-c", "1", "--csv", sys.executable, os.path.join(ROOT, "tools", "one_apply.py"), str(workload_id)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
    except Exception as e:
        return None, "ncu run failed: %s" % str(e)[:80]
    tot, seen = 0.0, 0
    for ln in r.stdout.splitlines():
        f = [x.strip().strip('"') for x in ln.split('","')]
        if len(f) > 3 and f[-3].startswith("dram__bytes_"):
            unit, val = f[-2], float(f[-1].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            tot += val * scale
            seen += 1
    if seen < 2:
        return None, "ncu output not parsed (rc %d): %s" % (r.returncode, (r.stderr or r.stdout)[-120:])
    return tot, "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, one launch of the dispatched kernel"


def config_dict(c, world):
    """The workload description both arms report (identical keys and values)."""
    nu = {5: "1e-3(1+0.5tanh(4 sin x sin y sin z)) at GLL nodes", 2: "0.01(1+0.5 sin x cos y) at GLL nodes"}
    return {"workload": c.name, "N": list(c.N[: c.dim]), "P": c.P, "ndof": c.ndof, "lam": c.lam,
            "nu": nu.get(c.cid, c.nu0), "parallelism": "z-slabs x%d" % world,
            "l2": "inputs larger than L2 (%.0f MB per field)" % (c.ndof * 8 / 1e6)}


def slab_inputs(c, el_off, nel):
    return c.apply_input_slab(el_off, nel), c.rhs_slab(0, el_off, nel), c.nu_slab(el_off, nel)


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle on a bounded sample
# ---------------------------------------------------------------------------
def time_oracle(c, budget_s=12.0):
    import oracle

    om = oracle.Mesh(c.dim, c.N[: c.dim], c.L[: c.dim], c.P)
    nel_s = min(c.n_el, 2048)
    u, _, nu = slab_inputs(c, 0, c.n_el) if c.n_el <= 4096 else (None, None, None)
    if u is None:  # full-size input arrays are needed by the oracle (neighbour reads)
        u = c.apply_input()
        nu = c.nu()
    rng = np.random.default_rng(99)
    elems = np.sort(rng.choice(c.n_el, size=nel_s, replace=False))
    t0 = time.perf_counter()
    oracle.sip_apply(om, c.lam, u, nu=nu, nu_const=c.nu0, elems=elems)
    t1 = time.perf_counter() - t0
    reps = max(1, int(budget_s / max(t1, 1e-3)))
    reps = min(reps, 200)
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.sip_apply(om, c.lam, u, nu=nu, nu_const=c.nu0, elems=elems)
    t = (time.perf_counter() - t0) / reps
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    gdofs = nel_s * c.n ** c.dim / t / 1e9
    return {"value": gdofs, "unit": "GDOF/s", "cores": cores, "kind": "oracle",
            "sample": "oracle_sip_apply (explicit GLL quadrature, C/OpenMP) on %d random elements of %s "
                      "(%d DOF), mean of %d repetitions" % (nel_s, c.name, nel_s * c.n ** c.dim, reps),
            "seconds_per_sample": t}


def run_reference(args, rank, world):
    if rank != 0:
        return
    c = get_config(WORKLOADS[args.workload])
    steps_t = []
    import oracle

    om = oracle.Mesh(c.dim, c.N[: c.dim], c.L[: c.dim], c.P)
    u, nu = c.apply_input(), c.nu()
    elems = np.sort(np.random.default_rng(7).choice(c.n_el, size=min(c.n_el, 2048), replace=False))
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.sip_apply(om, c.lam, u, nu=nu, nu_const=c.nu0, elems=elems)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            steps_t.append(dt)
    t = statistics.mean(steps_t)
    val = len(elems) * c.n ** c.dim / t / 1e9
    cb = {"value": val, "unit": "GDOF/s", "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
          "kind": "oracle",
          "sample": "each step: oracle_sip_apply (explicit GLL quadrature, C/OpenMP, as it stands) on the same %d "
                    "seeded random elements of %s (%d DOF); value = sampled DOF / mean step time"
                    % (len(elems), c.name, len(elems) * c.n ** c.dim)}
    line = {"metric": "GDOF/s SIP-DG Helmholtz apply", "value": val, "unit": "GDOF/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(c, world),
            "cpu_baseline": cb, "e2e": {"value": val, "unit": "GDOF/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    emit(line)


# ---------------------------------------------------------------------------
# product arm
# ---------------------------------------------------------------------------
def run_product(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2112_04167_b200 as dg

    c = get_config(WORKLOADS[args.workload])
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    uid = None
    if world > 1:
        obj = [dg.dg_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    m = dg.dg_mesh_create(c.dim, c.N[: c.dim], c.L[: c.dim], c.P, rank=rank, nranks=world, nccl_uid=uid,
                          stream=stream)
    nel, off = m.n_el, m.element_offset
    u_h, f_h, nu_h = slab_inputs(c, off, nel)
    u = torch.from_numpy(u_h).to(dev)
    f = torch.from_numpy(f_h).to(dev)
    nu = torch.from_numpy(nu_h).to(dev) if nu_h is not None else None
    out = torch.empty_like(u)
    ndof_global = c.ndof
    varnu = nu is not None

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-timed apply steps (clocks are sampled over the apply and PCG timed regions)
    for _ in range(args.warmup):
        dg.dg_helmholtz_apply(m, c.lam, nu, c.nu0, u, out)
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    clk = Clocks(local_rank).__enter__()
    time.sleep(0.15)  # let the sampler start before the timed region
    l0 = dg.dg_mesh_launch_count(m)
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        ev[2 * k].record(stream)
        dg.dg_helmholtz_apply(m, c.lam, nu, c.nu0, u, out)
        ev[2 * k + 1].record(stream)
    t_end.record(stream)
    barrier()
    launches = dg.dg_mesh_launch_count(m) - l0
    kernel_name = dg.dg_last_apply_kernel()
    total_ms = max_over_ranks(t_start.elapsed_time(t_end))
    per_launch_ms = statistics.mean(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps))
    per_launch_ms = max_over_ranks(per_launch_ms)
    ms_step = total_ms / args.steps
    value = ndof_global / (ms_step * 1e-3) / 1e9

    # ---- PCG solves (iterations/s)
    solve_ms, iters, infos = [], [], []
    for k in range(args.solve_warmup + args.solves):
        x = torch.zeros_like(u)
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        info = dg.dg_pcg_solve(m, c.lam, nu, c.nu0, f, c.tol, 5000, x)
        b.record(stream)
        barrier()
        if k >= args.solve_warmup:
            solve_ms.append(max_over_ranks(a.elapsed_time(b)))
            iters.append(info.iters)
            infos.append(info.as_dict())
    clk.__exit__(None, None, None)
    t_solve = statistics.mean(solve_ms)
    it = statistics.mean(iters)

    # ---- one IMEX-RK stage of config 4: convect + F_d1 + Poisson (P-1)
    #      + 3 Helmholtz solves, device-timed (1 GPU only: the c4 mesh shards, but the
    #      stage leg is reported for the single-GPU run)
    stage = None
    if world == 1 and not args.no_stage:
        stage = run_stage(dg, torch, stream, barrier)
        stage["vv_step"] = run_vv_step(dg, torch, stream, barrier)

    # ---- per-config legs (c1..c4) and the halo-mode data plane (1 GPU)
    configs = halo = None
    peak0, _ = measured_peaks()
    if world == 1 and not args.no_configs:
        configs = run_configs(dg, torch, stream, peak0)
        halo = run_halo(dg, torch, stream, c, u, nu, f, peak0)
        halo["slab_model"] = run_slab_model(dg, torch, stream, c, u, nu, per_launch_ms,
                                            statistics.mean(solve_ms) / statistics.mean(iters))

    # ---- e2e through the host-buffer C-ABI call (rank-local slab)
    u_np = np.ascontiguousarray(u_h)
    nu_np = None if nu_h is None else np.ascontiguousarray(nu_h)
    import torch as _t

    u_pin = _t.from_numpy(u_np).pin_memory().numpy()
    nu_pin = None if nu_np is None else _t.from_numpy(nu_np).pin_memory().numpy()
    o_pin = _t.empty(u_np.shape, dtype=_t.float64).pin_memory().numpy()
    for _ in range(max(1, args.warmup)):
        dg.dg_helmholtz_apply_host(m, c.lam, nu_pin, c.nu0, u_pin, o_pin)
    barrier()
    e2e_steps = max(3, args.steps // 4)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dg.dg_helmholtz_apply_host(m, c.lam, nu_pin, c.nu0, u_pin, o_pin)
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    h2d = u_np.nbytes * world + (nu_np.nbytes * world if nu_np is not None else 0)
    d2h = u_np.nbytes * world

    if rank != 0:
        return
    peak, peak_kind = measured_peaks()
    bpd = BYTES_PER_DOF[varnu]
    nd_local = m.ndof
    achieved = nd_local * bpd / (per_launch_ms * 1e-3) / 1e9
    traffic, traffic_how = (None, "skipped (--no-traffic)")
    if world == 1 and not args.no_traffic:
        traffic, traffic_how = measure_traffic(WORKLOADS[args.workload])
    cb = None
    if world == 1 and not args.no_cpu_baseline:
        cb = time_oracle(c)
    line = {
        "metric": "GDOF/s SIP-DG Helmholtz apply",
        "value": value,
        "unit": "GDOF/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "impl": "product",
        "config": config_dict(c, world),
        "pcg": {"iters_per_s": it / (t_solve * 1e-3), "iters": it, "ms_per_solve": t_solve, "tol": c.tol,
                "solves": args.solves, "rel_res": infos[-1]["rel_res"], "kappa_est": infos[-1]["kappa_est"],
                "gdof_iter_per_s": ndof_global * it / (t_solve * 1e-3) / 1e9,
                "bytes_per_dof_iter": PCG_BYTES_PER_DOF[varnu],
                "achieved_gbs_incl_setup": ndof_global * it * PCG_BYTES_PER_DOF[varnu] / (t_solve * 1e-3) / 1e9},
        "stage": stage,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_how": traffic_how,
                     "traffic_over_algorithmic": (traffic / (nd_local * bpd)) if traffic else None,
                     "kernel": kernel_name, "bytes_per_dof": bpd, "peak_kind": peak_kind, "launch_ms": per_launch_ms},
        "configs": configs,
        "halo": halo,
        "paper_context": PAPER_CONTEXT,
        "e2e": {"value": ndof_global / e2e_s / 1e9, "unit": "GDOF/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cb,
    }
    emit(line)


def time_apply(dg, torch, stream, m, lam, nu, nu0, u, out, reps=20, warm=3):
    """Mean CUDA-event time (ms) of one apply launch on the mesh stream, and the kernel name."""
    for _ in range(warm):
        dg.dg_helmholtz_apply(m, lam, nu, nu0, u, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        dg.dg_helmholtz_apply(m, lam, nu, nu0, u, out)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, dg.dg_last_apply_kernel()


def time_solves(dg, torch, stream, m, lam, nu, nu0, f, tol, maxit, reps=2):
    """(ms per solve, iterations) of Jacobi-PCG (or the mesh's preconditioner) from u0 = 0."""
    times, info = [], None
    for k in range(reps + 1):
        x = torch.zeros_like(f)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        info = dg.dg_pcg_solve(m, lam, nu, nu0, f, tol, maxit, x)
        b.record(stream)
        torch.cuda.synchronize()
        if k > 0:
            times.append(a.elapsed_time(b))
    return statistics.mean(times), info.iters


def run_configs(dg, torch, stream, peak):
    """Per-config measurements (SURVEY §8(d) roofline table) for BASELINE configs[0..3]: apply
    time (c1 in us per call: launch-bound), GDOF/s and fraction of the measured HBM bandwidth at
    the algorithmic 16 (constant nu) / 24 (variable nu) B per DOF, and PCG iterations/s of the
    config's solves (c3: the three-component velocity Helmholtz and the P-1 pressure Poisson with
    Jacobi and with the two-level Schwarz preconditioner)."""
    from workloads import config

    dev = torch.device("cuda", torch.cuda.current_device())
    out = {}
    for cid in (1, 2, 3, 4):
        c = config(cid)
        m = dg.dg_mesh_create(c.dim, c.N[: c.dim], c.L[: c.dim], c.P, stream=stream)
        u = torch.from_numpy(c.apply_input()).to(dev)
        nuh = c.nu()
        nu = None if nuh is None else torch.from_numpy(nuh).to(dev)
        o = torch.empty_like(u)
        ms, kern = time_apply(dg, torch, stream, m, c.lam, nu, c.nu0, u, o, reps=200 if cid == 1 else 20)
        bpd = BYTES_PER_DOF[nu is not None]
        d = {"workload": c.name, "ndof": c.ndof, "apply_us": ms * 1e3, "apply_gdofs": c.ndof / (ms * 1e-3) / 1e9,
             "apply_frac_hbm": c.ndof * bpd / (ms * 1e-3) / 1e9 / peak, "bytes_per_dof": bpd, "kernel": kern}
        f = torch.from_numpy(c.rhs(0)).to(dev)
        tol = 1e-11 if cid in (1, 2) else c.tol
        t, it = time_solves(dg, torch, stream, m, c.lam, nu, c.nu0, f, tol, 5000)
        d["helmholtz"] = {"ms_per_solve": t, "iters": it, "iters_per_s": it / (t * 1e-3), "tol": tol}
        if cid == 3:
            mp = dg.dg_mesh_create(3, c.N, c.L, c.P_p, stream=stream)
            fp = torch.from_numpy(c.poisson_rhs_raw()).to(dev)
            tj, ij = time_solves(dg, torch, stream, mp, 0.0, None, 1.0, fp, c.tol, 20000, reps=1)
            dg.dg_mesh_set_precond(mp, dg.DG_PC_SCHWARZ2)
            ts, isw = time_solves(dg, torch, stream, mp, 0.0, None, 1.0, fp, c.tol, 20000, reps=1)
            d["poisson_P%d" % c.P_p] = {"jacobi": {"ms_per_solve": tj, "iters": ij, "iters_per_s": ij / (tj * 1e-3)},
                                        "schwarz2": {"ms_per_solve": ts, "iters": isw, "iters_per_s": isw / (ts * 1e-3)},
                                        "ndof": mp.ndof}
            dg.dg_mesh_destroy(mp)
        dg.dg_mesh_destroy(m)
        out["c%d" % cid] = d
    return out


def run_halo(dg, torch, stream, c, u, nu, f, peak, reps=20):
    """The multi-GPU data plane on one GPU (1-rank halo mode: face traces through NCCL self
    send/recv on the exchange stream, interior / boundary layer split): c5 apply and PCG."""
    m = dg.dg_mesh_create(c.dim, c.N[: c.dim], c.L[: c.dim], c.P, stream=stream, halo_mode=True)
    o = torch.empty_like(u)
    ms, _ = time_apply(dg, torch, stream, m, c.lam, nu, c.nu0, u, o, reps=reps)
    t, it = time_solves(dg, torch, stream, m, c.lam, nu, c.nu0, f, c.tol, 5000)
    dg.dg_mesh_destroy(m)
    bpd = BYTES_PER_DOF[nu is not None]
    return {"mode": "1-rank halo mode (NCCL self send/recv of the slab face traces)", "apply_ms": ms,
            "apply_gdofs": c.ndof / (ms * 1e-3) / 1e9, "apply_frac_hbm": c.ndof * bpd / (ms * 1e-3) / 1e9 / peak,
            "pcg_iters": it, "pcg_ms_per_solve": t, "pcg_iters_per_s": it / (t * 1e-3)}


def run_slab_model(dg, torch, stream, c, u, nu, t1_apply_ms, t1_iter_ms):
    """Per-rank work of an N-GPU c5 run measured on this GPU: rank 0's slab (N_z / N element
    layers, same element size) as a 1-rank halo-mode mesh -- the face traces go through the same
    NCCL send/recv calls and the interior layers overlap them, only the peer is this GPU.  The
    projected strong-scaling efficiency T1 / (N T_slab) leaves out the NVLink transfer (hidden
    behind the interior layers) and the two 16-byte all-reduces per CG iteration; it is a model,
    not a multi-GPU measurement."""
    out = {}
    N = c.N
    for R in (2, 4, 8):
        nzl = N[2] // R
        Ls = (c.L[0], c.L[1], c.L[2] / R)
        m = dg.dg_mesh_create(3, (N[0], N[1], nzl), Ls, c.P, stream=stream, halo_mode=True)
        ne = m.n_el
        us, nus = u[:ne].contiguous(), (None if nu is None else nu[:ne].contiguous())
        o = torch.empty_like(us)
        ms, _ = time_apply(dg, torch, stream, m, c.lam, nus, c.nu0, us, o, reps=20)
        f = us.clone()
        times = []
        for k in range(3):
            x = torch.zeros_like(us)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            info = dg.dg_pcg_solve(m, c.lam, nus, c.nu0, f, 1e-30, 20, x, raise_on_notconv=False)
            b.record(stream)
            torch.cuda.synchronize()
            if k:
                times.append(a.elapsed_time(b) / max(info.iters, 1))
        it_ms = min(times)
        out["N%d" % R] = {"slab_layers": nzl, "apply_ms": ms, "pcg_ms_per_iter": it_ms,
                          "apply_eff_model": t1_apply_ms / (R * ms), "pcg_eff_model": t1_iter_ms / (R * it_ms)}
        dg.dg_mesh_destroy(m)
    return out


PAPER_CONTEXT = {
    "source": "PAPER.md Table 3 (P:1499-1505), Taylor-Green DNS, 32^3 elements, P = 15 velocity / 14 pressure, "
              "512 cores Intel Xeon E5-2680 v3, precision not stated; context only (no throughput of this path "
              "is reported in the paper)",
    "avg_runtime_per_step_s": {"BDF2 dt=2e-4": 4.26, "BDF2 dt=1.2e-3": 3.61, "RK-CB3e dt=2.4e-3": 14.77,
                               "RK-ARS3 dt=8e-4": 18.19, "RK-ARS3 dt=1.6e-3": 14.71},
}


def run_vv_step(dg, torch, stream, barrier, N=16, P=7, reps=2):
    """One IMEX-RK step with solution-dependent viscosity (Alg. 3 with nu(v),
    F_d2/F_d3, forcing and the final projection) on the VVP manufactured solution (PAPER.md:
    1189-1290, nu0 = nu1 = 0.01) on N^3 elements of the unit cube, P velocity / P-1 pressure
    (Schwarz Poisson, Jacobi variable-nu Helmholtz: lam h^2 / nu ~ 67 here, where the mean-nu
    Schwarz preconditioner saves only ~25 % of the iterations at ~1.4x their cost), RK-ARS3,
    dt = 2^-7."""
    from workloads import node_coords
    from workloads.inputs import vvp_exact, vvp_forcing

    dev = torch.device("cuda", torch.cuda.current_device())
    L = (1.0, 1.0, 1.0)
    mv = dg.dg_mesh_create(3, (N,) * 3, L, P, stream=stream)
    mp = dg.dg_mesh_create(3, (N,) * 3, L, P - 1, stream=stream)
    dg.dg_mesh_set_precond(mp, dg.DG_PC_SCHWARZ2)
    X = node_coords(3, (N,) * 3, L, P)
    tab = dg.TABLEAUX["RK-ARS3"]
    dt, visc = 2.0 ** -7, (0.01, 0.01, 2.0)
    fs = [[torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in vvp_forcing(X, c * dt, *visc[:2])]
          for c in tab["c"]]
    v0 = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in vvp_exact(X, 0.0)[0]]
    psi = torch.zeros(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
    times, info = [], None
    for k in range(reps + 1):
        v = [x.clone() for x in v0]
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        info = dg.dg_imex_rk_step_vv(mv, mp, tab, dt, visc, v, psi, 1e-10, 20000, fs=fs)
        b.record(stream)
        barrier()
        if k > 0:
            times.append(a.elapsed_time(b))
    d = info.as_dict()
    return {"workload": "VVP %d^3 P=%d (P_p=%d), RK-ARS3, dt=2^-7, nu0=nu1=0.01" % (N, P, P - 1),
            "ms_per_step": statistics.mean(times), "steps": reps, "pressure_iters": d["pressure_iters"],
            "velocity_iters": d["velocity_iters"], "implicit_stages": d["stages"],
            "dofs_per_component": mv.ndof}


def run_stage(dg, torch, stream, barrier, reps=2):
    """One IMEX-RK stage (Alg. 3 lines 4-9) on config 4: 32^3 hexes, P = 7 velocity,
    P_p = 6 pressure, TG velocity + 1e-3 noise, nu = 1/1600, dt = 1e-2, a_ex21 = a_im22 =
    gamma, tol 1e-10.  The pressure Poisson solve runs with the two-level
    Schwarz preconditioner (the Helmholtz solves keep Jacobi, which is faster at
    this lam); the same stage with the north star's Jacobi Poisson solve is timed once beside
    it (`jacobi`)."""
    from workloads.inputs import GAMMA_SDIRK3

    c4 = get_config(4)
    dev = torch.device("cuda", torch.cuda.current_device())
    mv = dg.dg_mesh_create(3, c4.N, c4.L, c4.P, stream=stream)
    mp = dg.dg_mesh_create(3, c4.N, c4.L, c4.P_p, stream=stream)
    v = [torch.from_numpy(a).to(dev) for a in c4.tg_velocity()]
    vo = [torch.empty_like(v[0]) for _ in range(3)]
    psi = torch.empty(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
    g = GAMMA_SDIRK3

    def timed(n_warm, n_rep):
        times, info = [], None
        for k in range(n_warm + n_rep):
            barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            info = dg.dg_imex_stage(mv, mp, 1e-2, g, 0.0, g, c4.nu0, v, vo, psi, c4.tol, 20000)
            b.record(stream)
            barrier()
            if k >= n_warm:
                times.append(a.elapsed_time(b))
        return statistics.mean(times), info.as_dict()

    dg.dg_mesh_set_precond(mp, dg.DG_PC_SCHWARZ2)
    ms_sw, d = timed(1, reps)
    dg.dg_mesh_set_precond(mp, dg.DG_PC_JACOBI)
    ms_j, dj = timed(0, 1)
    dg.dg_mesh_set_precond(mp, dg.DG_PC_SCHWARZ2)
    times = [ms_sw]
    # the same stage with the divergence / mass-flux stabilisation after the projection
    # (reading A26, zeta_D = zeta_C = 1)
    dg.dg_mesh_set_div_stab(mv, 1.0, 1.0)
    ms_st, dst = timed(0, 1)
    dg.dg_mesh_set_div_stab(mv, 0.0, 0.0)
    # one whole constant-nu IMEX-RK step (NEXT-2, Alg. 3 with RK-ARS3: 4 implicit stages) on the
    # same mesh pair and velocity, Schwarz Poisson
    vs = [x.clone() for x in v]
    rk_times, rk_info = [], None
    for k in range(2):
        for c in range(3):
            vs[c].copy_(v[c])
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rk_info = dg.dg_imex_rk_step(mv, mp, dg.TABLEAUX["RK-ARS3"], 1e-2, c4.nu0, vs, psi, c4.tol, 20000)
        b.record(stream)
        barrier()
        if k > 0:
            rk_times.append(a.elapsed_time(b))
    rk = {"tableau": "RK-ARS3", "dt": 1e-2, "ms_per_step": statistics.mean(rk_times), **rk_info.as_dict()}
    del vs
    # the explicit LLF convection alone, FP64-bound: algorithmic flops per element
    # of the sum-factorised Gauss evaluation over the CUDA-event time
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        dg.dg_convect_rhs(mv, v, vo)
    barrier()
    ev0.record(stream)
    for _ in range(5):
        dg.dg_convect_rhs(mv, v, vo)
    ev1.record(stream)
    barrier()
    conv_ms = ev0.elapsed_time(ev1) / 5
    n, Q = c4.P + 1, (3 * c4.P) // 2 + 1
    interp = n ** 3 * Q + n * n * Q * Q + n * Q ** 3                  # GLL -> Gauss, per component
    # contractions (interpolation, volume tests, face traces / projections) and pointwise work
    # (Gauss fluxes, LLF); the kernel's even-odd products execute half of the contraction
    # multiply-adds, so the executed model halves that part (the dense count is kept for
    # comparison with earlier rounds)
    contr = 2 * (3 * interp + 9 * interp) + 6 * 2 * (2 * 3 * (n * n * Q + n * Q * Q) + 3 * (Q * Q * n + Q * n * n))
    point = 2 * 6 * Q ** 3 + 6 * 2 * 10 * Q * Q
    flops_el = contr // 2 + point
    dense_el = contr + point
    conv = {"ms": conv_ms, "flop_per_launch": flops_el * mv.n_el,
            "tflops": flops_el * mv.n_el / (conv_ms * 1e-3) / 1e12,
            "flop_model": "even-odd sum factorisation as executed (contractions at half the dense multiply-adds)",
            "dense_flop_per_launch": dense_el * mv.n_el,
            "tflops_dense_equiv": dense_el * mv.n_el / (conv_ms * 1e-3) / 1e12}
    return {"workload": c4.name, "ms_per_stage": statistics.mean(times), "stages": reps, "convect": conv,
            "pressure_precond": "schwarz2 (element FDM blocks + Q1 coarse)", "rk_step": rk,
            "jacobi": {"ms_per_stage": ms_j, "pressure_iters": dj["pressure"]["iters"]},
            "div_stab": {"ms_per_stage": ms_st, "stab_iters": dst["stab"]["iters"], "zeta": [1.0, 1.0]},
            "pressure_P": c4.P_p, "pressure_iters": d["pressure"]["iters"],
            "velocity_iters": [x["iters"] for x in d["velocity"]], "tol": c4.tol,
            "dofs": {"velocity_per_component": mv.ndof, "pressure": mp.ndof}}


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)   # keep the real stdout for the JSON line ...
    os.dup2(2, 1)          # ... and route every other write to fd 1 (native libraries too) to stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--solve-warmup", type=int, default=1)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stage", action="store_true", help="skip the config-4 IMEX stage leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config (c1..c4) and halo-mode legs")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the NCCL transport (NVLink / NVLS) in the log
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_product(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
