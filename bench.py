"""Benchmark of the fine-grid solve path (BASELINE.json metric) on B200.

One step = one pass of the whole hot path for one design:
  mg_update_modulus (a1: fine diagonal, Galerkin coarse operators, coarsest inverse)
  + mgcg_solve of all R right-hand sides to rel. residual tol (a2-a7)
  + stress_stiffness_apply G(u) phi for the config's phi vectors (a8; u = state solution).
metric: fine-grid DOF*RHS*iter/s = n * sum_k iters_k / t_step  (plus MGCG solves/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

N > 1 is launched by torchrun (one process per GPU): the global grid is cut into N axis-0
slabs (mg_setup_dist; NCCL halo exchange + allreduce inside libmgcg), strong scaling,
device time = max over ranks.
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

from workloads import generate, get_config, n_dofs  # noqa: E402

METRIC = "fine-grid DOF*RHS*iter/s (MGCG, fp64, rel. residual 1e-10)"
UNIT = "DOF*RHS*iter/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
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
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                smax = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def traffic_from_profiles(cfg_name):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(cfg_name)
    return None


# --------------------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import torch
    import paper_1909_13585_b200 as mg
    from paper_1909_13585_b200.dist import bootstrap_nccl_id, local_inputs, rank_part

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    # N > 1: one global problem cut into ws axis-0 slabs (strong scaling, NCCL halos + allreduce)
    inp_g = generate(cfg)
    part = rank_part(cfg.nel, cfg.levels, ws, rank)
    inp = local_inputs(inp_g, part) if ws > 1 else inp_g
    n_glob = n_dofs(cfg.nel)
    n = inp["rhs"].shape[1]
    R = cfg.nrhs
    nphi = max(cfg.nphi, 0)
    E = torch.from_numpy(inp["E"]).to(dev)
    Es = torch.from_numpy(inp["Es"]).to(dev)
    fixed = torch.from_numpy(inp["fixed"]).to(dev)
    rhs = torch.from_numpy(inp["rhs"]).to(dev)
    phi = torch.from_numpy(inp["phi"]).to(dev) if nphi else None
    x = torch.empty_like(rhs)
    y = torch.empty((nphi, n), dtype=torch.float64, device=dev) if nphi else None
    stream = torch.cuda.current_stream()
    t0 = time.time()
    if ws > 1:
        nid = bootstrap_nccl_id(rank, ws)
        h = mg.mg_setup_dist(cfg.nel, E, fixed, cfg.levels, rank=rank, nranks=ws, nslab=1, nccl_id=nid)
    else:
        h = mg.mg_setup(cfg.nel, E, fixed, cfg.levels)
    torch.cuda.synchronize()
    setup_first_s = time.time() - t0

    def step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        mg.mg_update_modulus(h, E)
        ev[1].record(stream)
        rep = mg.mgcg_solve(h, rhs, cfg.tol, x)
        ev[2].record(stream)
        if nphi:
            mg.stress_stiffness_apply(h, Es, x[0], phi, y)
        ev[3].record(stream)
        return rep, ev

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    l0 = mg.mg_kernel_launches(h)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    reps, evs = [], []
    for _ in range(args.steps):
        rep, ev = step()
        reps.append(rep)
        evs.append(ev)
    end.record(stream)
    torch.cuda.synchronize()
    launches = mg.mg_kernel_launches(h) - l0
    ms_total = start.elapsed_time(end)
    phases = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])] for e in evs])
    # units processed by the whole job: global DOFs x sum of per-RHS iterations (identical on all ranks)
    total_dofiters = float(sum(n_glob * sum(r["iters"]) for r in reps))
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    clocks = clk.stop()
    ms_step = ms_total / args.steps
    value = total_dofiters / (ms_total / 1e3)

    # ---- fine-level kernels of one CG iteration, timed standalone (same kernels and launch
    # configuration as in the solve graph) with CUDA events on the handle's stream.
    hbm, peak_kind = peaks()
    kms = mg.mg_profile_kernels(h, R, reps=10)
    m = int(inp["E"].size)
    nR = float(n) * R
    coarse = 1.0 / (2 ** cfg.dim)
    # algorithmic bytes per launch (what each kernel must move)
    alg = {
        "cgp": 8.0 * (6 * nR + m),                                   # z, p_in, x in; p_out, q, x out; E
        "restrict": 8.0 * ((3 + coarse) * nR + m + n),               # r_in, q in; r_out, r_c out; E, D^-1
        "post": 8.0 * ((2 + coarse) * nR + m + n),                   # r, e_c in; z out; E, D^-1
        "matvec": 8.0 * (2 * nR + m),                                # x in, y out, E
    }
    kernels = {k: {"ms": kms[k], "alg_bytes": alg[k], "gbs": alg[k] / (kms[k] / 1e3) / 1e9,
                   "frac": alg[k] / (kms[k] / 1e3) / 1e9 / hbm} for k in alg}
    dom = "cgp"
    achieved = kernels[dom]["gbs"]
    # ---- whole-solve roofline: algorithmic bytes of the fused V(1,1)-PCG iteration (SURVEY 8(d),
    # DESIGN.md 6.6) summed over the iterations actually run, over the measured solve time:
    #   per iteration and active RHS  8 n (16 + 2/2^d + 8/(2^d - 1))   (vectors, all levels)
    #   per iteration                 8 n 2 + 24 m                      (D^-1 twice, E three times)
    d = cfg.dim
    per_rhs = 8.0 * n * (16 + 2.0 / 2 ** d + 8.0 / (2 ** d - 1))
    rep_last = reps[-1]
    solve_bytes = per_rhs * sum(rep_last["iters"]) + (16.0 * n + 24.0 * m) * max(rep_last["iters"])
    solve_ms = float(phases[:, 1].mean())
    solve_frac = solve_bytes / (solve_ms / 1e3) / 1e9 / hbm

    # ---- e2e: same step through the C ABI with pinned HOST buffers (H2D/D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        hE, hEs, hrhs = pin(inp["E"]), pin(inp["Es"]), pin(inp["rhs"])
        hphi = pin(inp["phi"]) if nphi else None
        hx = torch.empty((R, n), dtype=torch.float64).pin_memory().numpy()
        hy = torch.empty((max(nphi, 1), n), dtype=torch.float64).pin_memory().numpy()

        e2e_ph = np.zeros(3)

        def e2e_step():
            t_a = time.perf_counter()
            mg.mg_update_modulus(h, hE)   # returns once the operators are enqueued
            t_b = time.perf_counter()
            rep = mg.mgcg_solve(h, hrhs, cfg.tol, hx)
            t_c = time.perf_counter()
            if nphi:
                mg.stress_stiffness_apply(h, hEs, np.ascontiguousarray(hx[0]), hphi, hy[:nphi])
            t_d = time.perf_counter()
            e2e_ph[:] += (t_b - t_a, t_c - t_b, t_d - t_c)
            return rep

        e2e_step()
        torch.cuda.synchronize()
        e2e_ph[:] = 0.0
        if ws > 1:
            torch.distributed.barrier()
        t1 = time.perf_counter()
        its = 0
        for _ in range(max(1, min(args.steps, 3))):
            rep = e2e_step()
            its += n_glob * sum(rep["iters"])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        if ws > 1:
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
        nst = max(1, min(args.steps, 3))
        h2d = 8 * (inp["E"].size + R * n + (inp["Es"].size + n + nphi * n if nphi else 0))
        d2h = 8 * (R * n + nphi * n)
        e2e = {"value": its / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * dt / nst,
               "phase_ms": {"setup": 1e3 * e2e_ph[0] / nst, "solve": 1e3 * e2e_ph[1] / nst,
                            "stress_apply": 1e3 * e2e_ph[2] / nst},
               "phase_note": "host wall time per call; mg_update_modulus returns once the operators are "
                             "enqueued, so the solve call's time includes the rest of the setup, which "
                             "overlaps its right-hand-side upload"}

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE recipe)",
        "config": {"workload": f"{cfg.name}: {'Q4' if cfg.dim == 2 else 'H8'} {'x'.join(map(str, cfg.nel))}, "
                               f"{R} RHS, {cfg.levels} levels, G(u)phi x{nphi}",
                   "ndof": n_glob, "nrhs": R, "levels": cfg.levels, "tol": cfg.tol,
                   "parallelism": f"slabs{ws} (axis-0, NCCL halo + allreduce)" if ws > 1 else "single",
                   "l2": "inputs larger than L2 (fine R-vector %.0f MB)" % (8 * n * R / 1e6)},
        "solves_per_s": 1e3 / ms_step,
        "phase_ms": {"setup": float(phases[:, 0].mean()), "solve": float(phases[:, 1].mean()),
                     "stress_apply": float(phases[:, 2].mean())},
        "iters": reps[-1]["iters"], "true_relres_max": max(reps[-1]["true_relres"]),
        "first_setup_s": setup_first_s,
        "gpu_launches": int(launches),
        "roofline": {"kernel": "CG direction + fine EbE matvec (march2_kernel<M2_CGP> 2D / h8t_kernel<FOP_CGP> 3D, main + tail-tile launch)",
                     "bound": "hbm", "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic_from_profiles(cfg.name),
                     "alg_bytes_per_launch": alg[dom], "kernel_ms": kms[dom],
                     "solve_frac": solve_frac, "solve_alg_bytes": solve_bytes,
                     "solve_model": "8n(16+2/2^d+8/(2^d-1)) B per RHS-iteration + (16n+24m) B per iteration "
                                    "(fused V(1,1)-PCG, SURVEY 8(d))"},
        "kernels": kernels,
        "clocks": clocks,
        "e2e": e2e,
    }
    if ws > 1:
        # self-check of the decomposed solve: every rank's owned part of x gathered into the global
        # vector, compared on rank 0 with the undecomposed single-GPU solve of the same inputs
        from paper_1909_13585_b200.dist import gather_owned
        mg.mgcg_solve(h, rhs, cfg.tol, x)
        xg = gather_owned(x, part, n_glob)
        if rank == 0:
            dg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
            h1 = mg.mg_setup(cfg.nel, dg(inp_g["E"]), dg(inp_g["fixed"]), cfg.levels)
            rhs1 = dg(inp_g["rhs"])
            x1 = torch.empty_like(rhs1)
            r1 = mg.mgcg_solve(h1, rhs1, cfg.tol, x1)
            err = (torch.linalg.vector_norm(xg - x1, dim=1) / torch.linalg.vector_norm(x1, dim=1)).max().item()
            result["parity_vs_1gpu"] = {"max_rel_l2": err, "ok": bool(err < 1e-8), "iters_1gpu": r1["iters"],
                                        "iters_ngpu": reps[-1]["iters"]}
            mg.mg_destroy(h1)
        torch.distributed.barrier()
    if rank == 0 and ws == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(cfg)
    if ws > 1:
        torch.distributed.barrier()
    mg.mg_destroy(h)
    return result if rank == 0 else None


# --------------------------------------------------------------------------- oracle (CPU) arm
SAMPLE = {"C5": "C5s"}   # bounded CPU sample of a config (same recipe at reduced size), else itself


def sample_config(cfg):
    return get_config(SAMPLE.get(cfg.name, cfg.name))


def oracle_phases(scfg, inp):
    """The oracle as it stands, phase by phase, on one bounded sample: (i) assembly of K, (ii)
    preconditioner setup (scipy Galerkin MG hierarchy + coarsest LU), (iii) PCG solve of all R RHS
    to tol, (iv) one CSR SpMV with R columns, (v) G(u) assembly + apply to nphi vectors."""
    from oracle import assemble, mg as omg, solve
    ph = {}
    t = time.perf_counter()
    K = assemble.assemble_K(scfg.nel, inp["E"], inp["fixed"])
    ph["assembly_s"] = time.perf_counter() - t
    t = time.perf_counter()
    H = omg.Hierarchy(scfg.nel, K, inp["fixed"], scfg.levels)
    V = solve._VCycle(H, 0.6, 1)
    ph["precond_setup_s"] = time.perf_counter() - t
    t = time.perf_counter()
    its, U = [], []
    for k in range(scfg.nrhs):
        u, it = solve.pcg(K, inp["rhs"][k], V.apply, scfg.tol)
        its.append(it)
        U.append(u)
    ph["solve_s"] = time.perf_counter() - t
    t = time.perf_counter()
    _ = K @ inp["rhs"].T
    ph["spmv_R_s"] = time.perf_counter() - t
    if scfg.nphi:
        t = time.perf_counter()
        G = assemble.assemble_G(scfg.nel, inp["Es"], U[0], inp["fixed"])
        _ = G @ inp["phi"].T
        ph["G_assembly_apply_s"] = time.perf_counter() - t
    n = n_dofs(scfg.nel)
    value = n * sum(its) / ph["solve_s"]
    return value, ph, its


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(cfg):
    scfg = sample_config(cfg)
    inp = generate(scfg)
    value, ph, its = oracle_phases(scfg, inp)
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{scfg.name}: {'x'.join(map(str, scfg.nel))} ({n_dofs(scfg.nel)} DOFs), {scfg.nrhs} RHS, "
                      f"{scfg.levels} levels, same recipe as {cfg.name}; scipy PCG + Galerkin MG to {scfg.tol:g}, "
                      f"iterations {its}; value = DOF*RHS*iter / solve phase",
            "phases_s": {k: round(v, 3) for k, v in ph.items()},
            "cpu": cpu_model(), "cores_visible": cpu_cores(),
            "threads_note": "scipy SpMV / SuperLU single-threaded; numpy BLAS unused on this path"}


def run_reference(args, cfg):
    """--impl reference: the oracle as it stands on the host cores, rank 0 only; K timed steps
    after W untimed ones, each step = one PCG solve of one of the R RHS (cycling) on the bounded
    sample (the assembly and preconditioner setup are done once, outside the steps, and reported)."""
    ws, rank, local = dist_env()
    if rank != 0:
        return None
    from oracle import assemble, mg as omg, solve
    scfg = sample_config(cfg)
    inp = generate(scfg)
    t = time.perf_counter()
    K = assemble.assemble_K(scfg.nel, inp["E"], inp["fixed"])
    H = omg.Hierarchy(scfg.nel, K, inp["fixed"], scfg.levels)
    V = solve._VCycle(H, 0.6, 1)
    setup_s = time.perf_counter() - t
    n = n_dofs(scfg.nel)

    def step(i):   # one right-hand side per step, cycling through the R of the workload
        t0 = time.perf_counter()
        it = solve.pcg(K, inp["rhs"][i % scfg.nrhs], V.apply, scfg.tol)[1]
        return time.perf_counter() - t0, it

    for i in range(args.warmup):
        step(i)
    dts, units = [], 0.0
    for i in range(args.steps):
        dt, it = step(args.warmup + i)
        dts.append(dt)
        units += n * it
    total = float(sum(dts))
    value = units / total
    sample = (f"{scfg.name}: {'x'.join(map(str, scfg.nel))} ({n} DOFs), {scfg.nrhs} RHS, same recipe as {cfg.name}; "
              f"one step = scipy PCG + Galerkin MG solve of one RHS (cycling over the {scfg.nrhs}) to {scfg.tol:g} "
              f"(setup {setup_s:.1f} s once)")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE recipe)",
        "config": {"workload": f"{cfg.name} (oracle on the bounded sample {scfg.name})", "ndof": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model(), "cores_visible": cpu_cores()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    cfg = get_config(args.config)
    res = run_reference(args, cfg) if args.impl == "reference" else run_ours(args, cfg)
    if res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
