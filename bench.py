#!/usr/bin/env python
"""Benchmark of the B200 solve path on BASELINE.json's headline configuration.

Workload (BASELINE.json configs[2], SURVEY.md 8(d) cfg 3): unit sphere,
h = 0.0125, p = 3 (tricubic E, 7-point Laplacian), c = 1, reference tube
radius (N_A = 558,806), 256 RCB subdomains (+ align_interfaces), overlap 3,
ORAS with the modified cross-point condition (alpha = 4, alpha_cross = 40),
right-preconditioned GMRES(50) to a relative residual of 1e-10, FP64.
Synthetic right-hand side f = 13 u, u = x^3 - 3 x y^2 at closest points.

A "step" is one complete solve of that system to 1e-10 (time-to-1e-10),
with inputs resident in HBM.  The metric is DOF.iters/s = N_A x GMRES
iterations / solve time; `value` aggregates over ranks (each rank solves an
independent replica: the single-GPU path does not shard -- DESIGN.md).
`e2e` is the same metric through the public API with the right-hand side
copied from pinned host memory and the solution copied back, inside the
timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
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

METRIC = "ORAS-GMRES DOF·iters/s (FP64)"
UNIT = "DOF·iter/s"
CONFIGS = {
    # BASELINE.json configs[2] -- the headline, and the default workload of this bench
    "headline": dict(surface="sphere", h=0.0125, p=3, c=1.0, n_subdomains=256, n_overlap=3, method="oras",
                     alpha=4.0, alpha_cross=40.0, gmres_restart=50, rel_tol=1e-10, max_iter=2000,
                     partition="rcb", rhs="sphere"),
    # configs[0]: unit circle, 8 angular sectors, ORAS with the reference's default alpha
    "circle": dict(surface="circle", h=0.0125, p=3, c=1.0, n_subdomains=8, n_overlap=2, method="oras",
                   alpha=1.0, alpha_cross=-1.0, gmres_restart=50, rel_tol=1e-10, max_iter=2000,
                   partition="sector", rhs="circle"),
    # configs[1]: unit sphere h = 0.05, 64 RCB
    "sphere05": dict(surface="sphere", h=0.05, p=3, c=1.0, n_subdomains=64, n_overlap=2, method="oras",
                     alpha=4.0, alpha_cross=40.0, gmres_restart=50, rel_tol=1e-10, max_iter=2000,
                     partition="rcb", rhs="sphere"),
    # configs[3]: torus R = 1, r = 0.4, h = 0.01, 512 RCB, seeded trigonometric right-hand side
    "torus": dict(surface="torus", major_radius=1.0, minor_radius=0.4, h=0.01, p=3, c=1.0, n_subdomains=512,
                  n_overlap=2, method="oras", alpha=4.0, alpha_cross=40.0, gmres_restart=50, rel_tol=1e-10,
                  max_iter=2000, partition="rcb", rhs="trig"),
    # configs[4]: displaced icosphere (subdivision 6), h = 0.01, 512 RCB, modified cross-point condition
    "trimesh": dict(surface="obj", h=0.01, p=3, c=1.0, n_subdomains=512, n_overlap=2, method="oras",
                    alpha=4.0, alpha_cross=40.0, gmres_restart=50, rel_tol=1e-10, max_iter=2000,
                    partition="rcb", rhs="trig", subdivisions=6, mesh_seed=5),
}
WORKLOAD = CONFIGS["headline"]
FALLBACK_HBM_GBS = 6650.0


def workload_name(w=None):
    w = w or WORKLOAD
    return (f"{w['surface']}_h{w['h']}_p{w['p']}_{w['partition']}{w['n_subdomains']}_no{w['n_overlap']}_"
            f"{w['method']}_a{w['alpha']:g}_ax{w['alpha_cross']:g}_gmres{w['gmres_restart']}_tol{w['rel_tol']:g}")


def build_problem(w):
    """Surface, band, E, A (the device path's host setup) + partition + rhs for config w."""
    from paper_1909_08734_b200 import api, inputs
    obj = None
    if w["surface"] == "obj":
        import tempfile
        v, f = inputs.displaced_icosphere(w["subdivisions"], seed=w["mesh_seed"])
        obj = os.path.join(tempfile.mkdtemp(prefix="cpddg_mesh_"), "icosphere.obj")
        inputs.write_obj(obj, v, f)
    P = api.Problem(w["surface"], h=w["h"], p=w["p"], c=w["c"], major_radius=w.get("major_radius", 2 / 3),
                    minor_radius=w.get("minor_radius", 1 / 3), obj_path=obj)
    cp = P.active_cp
    part = inputs.sector_partition(cp, w["n_subdomains"]) if w["partition"] == "sector" \
        else inputs.rcb_partition(cp, w["n_subdomains"])
    rhs = {"sphere": inputs.rhs_sphere, "circle": inputs.rhs_circle,
           "trig": lambda q: inputs.rhs_trig(q, seed=2024)}[w["rhs"]](cp)
    return P, part, rhs, obj


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """DRAM bytes per k_solve launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_k_solve.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, interval_ms: int = 200):
        self.index = index
        self.interval_ms = interval_ms
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", str(self.interval_ms), "-i", str(self.index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for k, name in enumerate(names):
                if f[5 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------- reference / CPU

def cpu_reference(P, locs, b, iters_per_step: int, steps: int, warmup: int):
    """Time the reference's own solve (oracle/_ref: the unmodified reference
    headers; Eigen replaced by the oracle shim) on the host cores: the
    reference build_problem, the reference DirectSolver on the local systems
    (identical to the reference's own assemble_local output, bit for bit), and
    bounded samples of the reference gmres_solve."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    cores = os.cpu_count() or 1
    w = WORKLOAD
    cfg = dict(surface=w["surface"], h=w["h"], p=w["p"], c=w["c"], method=w["method"], mode="gmres",
               gmres_restart=w["gmres_restart"], n_overlap=w["n_overlap"], n_subdomains=w["n_subdomains"],
               alpha=w["alpha"], alpha_cross=w["alpha_cross"], rel_tol=w["rel_tol"])
    if w["surface"] == "torus":
        cfg.update(major_radius=w["major_radius"], minor_radius=w["minor_radius"])
    if w["surface"] == "obj":
        cfg.update(obj=P.obj_path)
    t0 = time.perf_counter()
    R = ref.RefProblem(cfg, workers=cores)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref.set_locals(R, locs)
    t_locals = time.perf_counter() - t0
    samples = []
    for k in range(warmup + steps):
        r = ref.solve_capped(R, b, iters_per_step, WORKLOAD["rel_tol"])
        if k >= warmup:
            samples.append(r)
    secs = sum(s["seconds"] for s in samples)
    its = sum(s["iterations"] for s in samples)
    value = R.n_active * its / secs
    return dict(value=value, unit=UNIT, cores=cores, kind="reference",
                sample=(f"{steps} x {iters_per_step} GMRES(50) iterations of the reference gmres_solve "
                        f"(serial SpMV/MGS, preconditioner on a {cores}-thread ThreadPool) on the full "
                        f"workload; setup untimed: build_problem {t_build:.1f}s, {len(locs)} local "
                        f"factorisations {t_locals:.1f}s"),
                seconds=secs, iterations=its)


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1909_08734_b200 import api, inputs
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return 0
    P, part, b, obj = build_problem(WORKLOAD)
    P.obj_path = obj
    P.decompose(part, WORKLOAD["n_overlap"], WORKLOAD["method"], WORKLOAD["alpha"], WORKLOAD["alpha_cross"])
    locs = [P.local(j) for j in range(P.n_sub)]
    base = cpu_reference(P, locs, b, args.ref_iters, args.steps, args.warmup)
    line = {"metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * base["seconds"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(), "N_A": P.n_active}, "impl": "reference",
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- device arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed solves (default: 3; more for the millisecond-scale configs so host jitter averages out)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-iters", type=int, default=4, help="GMRES iterations per reference sample step")
    ap.add_argument("--cpu-baseline", default="auto", choices=["auto", "off"])
    ap.add_argument("--config", default="headline", choices=sorted(CONFIGS),
                    help="workload (default: BASELINE's headline; the others are parity / scaling cases)")
    args = ap.parse_args()
    global WORKLOAD
    WORKLOAD = CONFIGS[args.config]
    if args.steps is None:
        args.steps = {"circle": 1000, "sphere05": 50}.get(args.config, 3) if args.impl == "ours" else 3
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch

    from paper_1909_08734_b200 import api, inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- setup (untimed): band, E, A, partition, subdomains, device factorisation
    t0 = time.perf_counter()
    P, part, b_host, obj = build_problem(WORKLOAD)
    P.obj_path = obj
    t_problem = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, moves = P.decompose(part, WORKLOAD["n_overlap"], WORKLOAD["method"], WORKLOAD["alpha"], WORKLOAD["alpha_cross"])
    t_decomp = time.perf_counter() - t0
    t0 = time.perf_counter()
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    torch.cuda.synchronize()
    t_locals = time.perf_counter() - t0
    pcs = M.stats()
    b = torch.from_numpy(b_host).cuda()
    n = P.n_active
    tol, mi, rs = WORKLOAD["rel_tol"], WORKLOAD["max_iter"], WORKLOAD["gmres_restart"]

    for _ in range(args.warmup):
        api.gmres_solve(A, b, M, tol, mi, rs)
    torch.cuda.synchronize()

    # ---- timed region: K complete solves, inputs resident in HBM
    # each nvidia-smi query stalls the CUDA driver for milliseconds: harmless
    # for the 0.3 s headline solves, but it would dominate the millisecond
    # configurations, which are sampled once a second instead (over >= 1 s)
    clocks = ClockSampler(local_rank, 200 if args.config not in ("circle", "sphere05") else 1000)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    results = [api.gmres_solve(A, b, M, tol, mi, rs, profile=True) for _ in range(args.steps)]
    e1.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    t_dev = max_over_ranks(e0.elapsed_time(e1) * 1e-3)
    iters = [r.log.iterations for r in results]
    assert all(r.log.converged for r in results), "solve did not converge"
    dof_iters = n * sum(iters)
    value = world * dof_iters / t_dev
    launches = sum(r.log.kernel_launches for r in results)
    pc_s = sum(r.log.kernel_times["pc_seconds"] for r in results)
    pc_n = sum(r.log.kernel_times["pc_launches"] for r in results)
    op_s = sum(r.log.kernel_times["op_seconds"] for r in results)
    op_n = sum(r.log.kernel_times["op_launches"] for r in results)
    u = results[-1].u
    final_rel = results[-1].log.final_true_residual / float(np.linalg.norm(b_host))

    # ---- e2e: public API with host buffers (pinned H2D of f, D2H of u) in the timed region
    b_pin = torch.from_numpy(b_host).pin_memory()
    u_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    e2e_iters = 0
    for _ in range(args.steps):
        bd = b_pin.to("cuda", non_blocking=True)
        r = api.gmres_solve(A, bd, M, tol, mi, rs)
        u_pin.copy_(r.u, non_blocking=True)
        e2e_iters += r.log.iterations
    e3.record()
    torch.cuda.synchronize()
    barrier()
    t_e2e = max_over_ranks(e2.elapsed_time(e3) * 1e-3)
    e2e_value = world * n * e2e_iters / t_e2e

    hbm, peak_src = peaks()
    avg_pc = pc_s / max(pc_n, 1)
    achieved = pcs["algorithmic_bytes"] / avg_pc / 1e9
    op_alg, _ = A.bytes()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": workload_name(), "N_A": n, "N_G": P.n_ghost, "n_subdomains": P.n_sub,
            "align_moves": moves, "gmres_iterations": iters[0], "time_to_1e-10_s": t_dev / args.steps,
            "final_true_relative_residual": final_rel, "parallelism": f"replicas x{world}",
            "l2": "inputs larger than L2: 12+ GB of local factors streamed per preconditioner apply",
            "rhs": {"sphere": "f = 13 u, u = x^3 - 3xy^2 at closest points",
                    "circle": "f = 2 sin(t) + 145 sin(12 t)",
                    "trig": "16 seeded modes sin(k.cp + phi), k in [-4,4]^3"}[WORKLOAD["rhs"]],
            "partition": WORKLOAD["partition"] + " on closest points, then align_interfaces",
            "setup_s": {"problem": t_problem, "decompose": t_decomp, "factor_and_upload": t_locals,
                        "device_factor": pcs["factor_seconds"], "host_analyse": pcs["analyse_seconds"]},
            "pc": {k: pcs[k] for k in ("factor_entries", "profile_entries", "factor_bytes", "n_rows_total",
                                       "max_rows", "n_reduced", "max_probe_residual", "apply_mode")},
            "pc_stored_over_profile": pcs["factor_entries"] / pcs["profile_entries"],
            "kernel_ms": {"pc_apply_avg": 1e3 * avg_pc, "op_apply_avg": 1e3 * op_s / max(op_n, 1)},
            "op_roofline_GBs": op_alg / (op_s / max(op_n, 1)) / 1e9 if op_n else None,
        },
        "roofline": {"bound": "hbm", "kernel": {1: "k_solve_dense (preconditioner apply, dense small-system mode)",
                                                 2: "k_solve_tma (preconditioner apply, TMA-streamed record solve)"}
                     .get(pcs["apply_mode"], "k_solve (preconditioner apply, record solve)"), "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": ncu_traffic() if WORKLOAD is CONFIGS["headline"] else None,
                     "algorithmic_bytes_per_launch": pcs["algorithmic_bytes"], "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and args.cpu_baseline == "auto":
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import ref
            if ref.available():
                locs = [P.local(j) for j in range(P.n_sub)]
                base = cpu_reference(P, locs, b_host, args.ref_iters, 1, 0)
                line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")}
            else:
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                        "sample": "unavailable: oracle/_ref not built"}
        except Exception as exc:  # the baseline is reported, never fatal to the device number
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"failed: {exc}"}
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
