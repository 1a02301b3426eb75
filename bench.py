"""bench.py — driver benchmark of the B200 hot path.

Headline (N=1): Newton-step DoF/s on BASELINE config 3 — the 3d Sneddon penny crack on a
uniform 128^3 Q1 hex mesh (8,586,756 dofs), eps = 2h, kappa = 1e-12, load step 1, Newton tol
1e-8, AMG-preconditioned GMRES (restart 100, rtol 1e-8).  One bench step = one complete
newton_active_set_step (solver.cpp:49-188) from the seeded initial state, inputs resident in
HBM; value = N_total x Newton iterations / device time.

The operator half of the metric (BASELINE config 1: assembled M_uu of a 3d 192^3 mesh, 21.5M
u dofs) is measured in the same run and reported under "operator"; the roofline object is the
CSR SpMV kernel of that operator apply.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
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

SEED_PHI = 180609924001
SEED_U = 180609924002

CFG3 = dict(dim=3, half_width=10.0, n0=8, refinements=4)  # 128^3 cells
CFG4 = dict(dim=3, half_width=10.0, n0=8, refinements=5)  # 256^3 cells, 67,898,372 dofs (needs >= 4 GPUs)
CFG1 = dict(dim=3, half_width=10.0, n0=12, refinements=4)  # 192^3 cells
CPU_SAMPLE = dict(dim=3, half_width=10.0, n0=8, refinements=2)  # 32^3 cells, 1/64 of config 3

METRIC = "Newton-step DoF/s (config 3: 3d penny crack, 128^3 Q1, 8,586,756 dofs)"
METRIC4 = "Newton-step DoF/s (config 4: 3d penny crack, 256^3 Q1, 67,898,372 dofs)"
CONFIG = {"workload": "config3: 3d Sneddon penny crack, uniform 128^3 Q1 hexes, 8,586,756 dofs (u, phi), FP64; "
                      "E=1, nu=0.2, G_c=1, p=1e-3, eps=2h, kappa=1e-12, 1 load step, Newton tol 1e-8, "
                      "GMRES(100) rtol 1e-8 with block AMG",
          "step": "one newton_active_set_step from the seeded state (all Newton iterations)",
          "l2": "working set (J 8.6 GB, AMG hierarchy, Krylov basis) >> 126 MB L2; no flush needed",
          "parallelism": "single GPU"}
CONFIG4 = dict(CONFIG, workload="config4: 3d Sneddon penny crack, uniform 256^3 Q1 hexes, 67,898,372 dofs (u, phi), "
                                "FP64; otherwise as config 3 (strong-scaling configuration, >= 4 GPUs)")


def splitmix_uniform(seed: int, n: int, start: int = 0) -> np.ndarray:
    """U_i = (mix64(seed + (i+1) * golden) >> 11) * 2^-53."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def splitmix_normal(seed: int, n: int) -> np.ndarray:
    """Box-Muller on uniform pairs (2j, 2j+1): sqrt(-2 ln(1-U1)) cos(2 pi U2)."""
    U = splitmix_uniform(seed, 2 * n)
    return np.sqrt(-2.0 * np.log1p(-U[0::2])) * np.cos(2.0 * np.pi * U[1::2])


def config1_host(dim=3, half_width=10.0, n0=12, refinements=4):
    nn = (n0 << refinements) + 1
    V = nn ** dim
    return V, splitmix_uniform(SEED_PHI, V), splitmix_normal(SEED_U, dim * V)


def config1_inputs(cf, device="cuda", **over):
    """Config 1: problem, Dirichlet constraints, material, regularization, x = (u, phi_tilde), phi_tilde."""
    import torch
    c = dict(CFG1)
    c.update(over)
    P = cf.Problem(c["dim"], c["half_width"], c["n0"], c["refinements"])
    V, pt, u = config1_host(**c)
    h = P.h
    mat = cf.Material(E=1.0, nu=0.2, pressure=1e-3, kappa_factor=1e-12 / h, eps_mode=1, eps_fixed=2 * h)
    reg = cf.Regularization(2 * h, 1e-12)
    cs = cf.build_constraints(P, True)
    x = torch.empty(P.n_total, dtype=torch.float64, device=device)
    x[:P.n_u] = torch.from_numpy(u).to(device)
    x[P.n_u:] = torch.from_numpy(pt).to(device)
    return P, cs, mat, reg, x, torch.from_numpy(pt).to(device)


def sneddon_setup(mod, cfg, oracle=False):
    """Problem + material (eps = 2h fixed, kappa = 1e-12) + regularization for a Sneddon config."""
    if oracle:
        P = mod.Problem(cfg["dim"], cfg["half_width"], cfg["n0"], cfg["refinements"])
        m = mod.material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
        return P, m, P.resolve_regularization(m, P.slit_band_edge(m))
    P = mod.Problem(cfg["dim"], cfg["half_width"], cfg["n0"], cfg["refinements"])
    m = mod.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
    return P, m, mod.resolve_regularization(P, m, mod.slit_band_edge(P, m))


def csr_bytes(rows, cols, nnz):
    """Compulsory bytes of one CSR SpMV: 12 nnz (8 B value + 4 B column) + 8 (rows+1) int64 row
    pointers + 8 cols (x) + 8 rows (y)."""
    return 12 * nnz + 8 * (rows + 1) + 8 * cols + 8 * rows


def stencil_bytes(rows, cols, nnz):
    """Compulsory bytes of one stencil-implicit-column SpMV: 8 nnz values + row pointers + x + y."""
    return 8 * nnz + 8 * (rows + 1) + 8 * cols + 8 * rows


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            # nvidia-smi's start-up (NVML initialisation) must not fall inside the timed region:
            # wait for its first sample, then drop it, so every kept sample is taken while timing
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [t.strip() for t in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- CPU legs (oracle)
def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_newton_sample(cfg, threads, max_iter=50, order=1):
    """The reference's CPU path (the oracle port: the reference itself needs Eigen3, absent here) from
    the seeded state of a Sneddon config: returns (dofs, newton iterations, gmres iterations, seconds).
    order 1 = the reference's arithmetic (sequential CSR rows and dots); results are bitwise
    independent of the thread count."""
    from oracle import orc
    orc.set_threads(threads)
    orc.set_order(order)
    try:
        P, m, reg = sneddon_setup(orc, cfg, oracle=True)
        phi, _ = P.initial_crack(m)
        sol = np.zeros(P.n_total)
        sol[P.n_u:] = phi
        t0 = time.perf_counter()
        rep = P.newton_step(m, reg, orc.solver_options(newton_max_iter=max_iter), sol, phi.copy(), phi.copy(), 1)
        dt = time.perf_counter() - t0
    finally:
        orc.set_order(0)
    its = rep["iterations"]
    return P.n_total, len(its), int(its[:, 3].sum()), dt


CPU_CFG3_DESC = ("config 3 at full size (3d penny 128^3, 8,586,756 dofs): the first Newton iteration of "
                 "newton_active_set_step from the seeded state (residual, active set, Jacobian, both AMG "
                 "hierarchies rebuilt as the reference does every iteration, GMRES(100) to 1e-8: 13 iterations); "
                 "oracle port of the reference (Eigen3 is absent, so the reference cannot be built) in the "
                 "reference's arithmetic order, thread-parallel on all host threads (assembly, AMG setup, SpMV, "
                 "vector ops); DoF/s = N_total x Newton iterations / seconds, the GPU line's unit")
CPU_1T_DESC = ("3d penny 32^3 (143,748 dofs), one full newton_active_set_step (3 Newton iterations) of the oracle "
               "port on ONE thread, i.e. the single-threaded reference's schedule (a config-3 iteration on one "
               "thread takes minutes)")


def oracle_cfg1_spmv(threads, applies=5):
    """Config 1's M_uu apply on the host (oracle CSR, sequential row sums): GB/s with the CSR bytes."""
    from oracle import orc
    orc.set_threads(threads)
    orc.set_order(1)
    try:
        P = orc.Problem(3, 10.0, CFG1["n0"], CFG1["refinements"])
        V, pt, u = config1_host()
        m = orc.material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
        reg = orc.Regularization(2 * P.h, 1e-12)
        x = np.concatenate([u, pt])
        t0 = time.perf_counter()
        J = P.jacobian(P.constraints(True), m, reg, x, pt)
        t_asm = time.perf_counter() - t0
        uu_rows, _, nnz = J.nnz(0)
        y = np.empty(P.n_u)
        J.spmv(0, u, y)
        t0 = time.perf_counter()
        for _ in range(applies):
            J.spmv(0, u, y)
        ms = (time.perf_counter() - t0) / applies * 1e3
    finally:
        orc.set_order(0)
    nb = csr_bytes(P.n_u, P.n_u, nnz)
    return {"value": nb / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_apply": ms, "bytes_per_apply": nb, "nnz": nnz,
            "cores": threads, "assembly_s": t_asm,
            "sample": "config 1 M_uu (192^3, 21,567,171 rows) CSR SpMV on the host, row-parallel, sequential row sums"}


def cpu_baseline_leg(value_gpu=None, full_rebuild=None):
    nt = host_threads()
    dofs, its, gm, sec = oracle_newton_sample(CFG3, nt, max_iter=1)
    out = {"value": dofs * its / sec, "unit": "DoF/s", "cores": nt, "kind": "port", "sample": CPU_CFG3_DESC,
           "newton_iterations": its, "gmres_iterations": gm, "seconds": sec}
    d1, i1, g1, s1 = oracle_newton_sample(CPU_SAMPLE, 1)
    out["single_thread"] = {"value": d1 * i1 / s1, "unit": "DoF/s", "cores": 1, "seconds": s1, "sample": CPU_1T_DESC}
    try:
        out["operator_cfg1"] = oracle_cfg1_spmv(nt)
    except Exception as ex:  # reported, never fatal
        out["operator_cfg1"] = {"error": str(ex)[:200]}
    if value_gpu:
        out["gpu_over_cpu"] = value_gpu / out["value"]
    if full_rebuild and full_rebuild.get("value"):
        out["gpu_full_rebuild_over_cpu"] = full_rebuild["value"] / out["value"]
    return out


REF_BUDGET_S = 240.0


def reference_arm(args):
    """--impl reference: the reference's CPU path (oracle port, reference arithmetic order) on the
    host's cores for the same metric and workload as our arm (config 3, Newton-step DoF/s).  Each
    step is a bounded sample of that workload — one complete Newton iteration of config 3 from the
    seeded state (~30 s on 16 threads) — and the run stops after REF_BUDGET_S seconds of steps, so
    `steps` reports how many ran.  Warm-up steps are not run: the CPU path keeps no state between
    steps (each rebuilds everything from the seeded state)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    nt = host_threads()
    runs, t_all = [], 0.0
    while len(runs) < args.steps and (t_all < REF_BUDGET_S or not runs):
        runs.append(oracle_newton_sample(CFG3, nt, max_iter=1))
        t_all += runs[-1][3]
    value = sum(d * i for d, i, _, _ in runs) / t_all
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": args.gpus,
           "steps": len(runs), "steps_requested": args.steps, "warmup": 0, "warmup_requested": args.warmup,
           "ms_per_step": 1e3 * t_all / len(runs), "higher_is_better": True, "dtype": "f64", "data": "synthetic",
           "config": dict(CONFIG, step="one complete Newton iteration of config 3 from the seeded state (the "
                          "bounded sample of one newton_active_set_step); run capped at %d s" % REF_BUDGET_S,
                          parallelism=f"host CPU, {nt} threads"),
           "gmres_iterations": [g for _, _, g, _ in runs],
           "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": nt, "kind": "port", "sample": CPU_CFG3_DESC},
           "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- GPU legs
def time_events(fn, n, stream):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def operator_leg(cf, device, stream, applies=20):
    """Config 1: assembled M_uu apply (CSR SpMV), inputs resident in HBM."""
    import torch
    P, cs, mat, reg, x, pt = config1_inputs(cf, device=device)
    nu = P.n_u
    u0 = x[:nu].contiguous()
    # the matrix-free equivalent first (BASELINE config 1): same operator from phi_tilde, cell by cell
    y_mf = torch.empty_like(u0)
    for _ in range(3):
        cf.mf_apply_uu(P, cs, mat, reg, pt, u0, out=y_mf)
    ms_mf = time_events(lambda: cf.mf_apply_uu(P, cs, mat, reg, pt, u0, out=y_mf), applies, stream)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    u = u0
    del x
    y = torch.empty(nu, dtype=torch.float64, device=u.device)
    fmt = J.format(0)
    nb_csr = csr_bytes(nu, nu, J.nnz[0])
    # the format's own compulsory bytes: stencil rows stream 8 B values (no column indices)
    nb = stencil_bytes(nu, nu, J.nnz[0]) if fmt == "stencil" else nb_csr
    for _ in range(3):
        J.spmv(0, u, out=y)
    ms = time_events(lambda: J.spmv(0, u, out=y), applies, stream)
    rel_mf = float(torch.linalg.norm(y_mf - y) / torch.linalg.norm(y))
    fp64 = cf.fp64_peak_tflops()
    ncells = P.n_cells
    flops = 2688.0 * ncells  # canonical FP64 flops per hex cell
    mf = {"ms_per_apply": ms_mf, "gflops": flops / (ms_mf * 1e-3) / 1e9, "fp64_peak_tflops_measured": fp64,
          "frac_of_fp64_peak": flops / (ms_mf * 1e-3) / 1e12 / fp64, "rel_err_vs_assembled": rel_mf,
          "min_bytes": 8 * (2 * nu + P.n_vertices),
          "note": "single-pass z-sweep (k_mf_sweep_async: 7x7 / 8x8 / 10x10 vertex columns per CTA chosen per grid, 5-11 vertex planes per CTA, one thread per "
                  "cell, sum-factorised ~1,650 flops), FMA-contracted element math, compared with the assembled "
                  "apply to rounding; flops = canonical 2,688 per cell. The same kernel is the Newton step's "
                  "Krylov operator and finest-level smoother in 3d (operator_kind 1)"}
    # e2e through the C ABI with pinned host buffers
    uh = u.cpu().pin_memory()
    yh = torch.empty(nu, dtype=torch.float64).pin_memory()
    J.spmv(0, uh.numpy(), out=yh.numpy())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        J.spmv(0, uh.numpy(), out=yh.numpy())
    e2e_ms = (time.perf_counter() - t0) / 3 * 1e3
    ok = bool(torch.equal(yh.to(device), y))
    peak, src = peak_hbm()
    gbs = nb / (ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r02_spmv_st16t_cfg1_ncu.json" if fmt == "stencil" else "r01_spmv_cfg1_ncu.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        if tj.get("format", "csr") == fmt:  # only a capture of the kernel measured here
            traffic = tj.get("traffic_bytes")
    res = {"workload": "config1: M_uu apply, 3d 192^3 Q1, 21,567,171 u dofs, 1,676,188,257 nnz",
           "format": fmt, "value": gbs, "unit": "GB/s", "ms_per_apply": ms, "bytes_per_apply": nb,
           "frac_of_hbm_peak": gbs / peak, "csr_equivalent_gbs": nb_csr / (ms * 1e-3) / 1e9,
           "csr_bytes_per_apply": nb_csr,
           "e2e": {"value": nb / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_apply": e2e_ms,
                   "h2d_bytes_per_step": 8 * nu, "d2h_bytes_per_step": 8 * nu, "matches_device": ok},
           "nnz": J.nnz[0], "matrix_free": mf}
    del J, u, y, y_mf, pt
    torch.cuda.empty_cache()
    return res, {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                 "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/)",
                 "kernel": ("k_spmv_st16t (TMA-fed value/x ring, stencil-implicit columns, M_uu of config 1)" if fmt == "stencil"
                            else "k_spmv_b<16,4> (CSR SpMV, M_uu of config 1)"), "bytes_per_launch": nb,
                 "ms_per_launch": ms, "peak_source": src}


def vcycle_leg(cf, P, mat, reg, x_final, phi_old, stream):
    """AMG V-cycle time per application, u- and phi-hierarchies separately, built from the
    Jacobian at the converged state of the measured step (active set = phi dofs at phi_old)."""
    import torch
    xs = x_final.cpu().numpy()
    po = phi_old.cpu().numpy()
    act = np.nonzero(xs[P.n_u:] == po)[0]
    cs = cf.build_constraints(P, True, {int(P.n_u + v): float(po[v]) for v in act})
    J = cf.assemble_jacobian(P, cs, mat, reg, x_final, phi_old)
    node_u = np.repeat(np.arange(P.n_vertices, dtype=np.int32), P.dim)
    hu = cf.build_amg(cf.CsrMatrix.from_block(J, 0), node_u, cf.rigid_body_modes(P, cs))
    free = 1.0 - np.isin(np.arange(P.n_vertices), act)
    hp = cf.build_amg(cf.CsrMatrix.from_block(J, 2), np.arange(P.n_vertices, dtype=np.int32), free.reshape(-1, 1))
    out = {}
    for name, h, n in (("u", hu, P.n_u), ("phi", hp, P.n_phi)):
        r = torch.randn(n, dtype=torch.float64, device=x_final.device)
        h.v_cycle(r)
        ms = time_events(lambda: h.v_cycle(r), 10, stream)
        nb = vcycle_bytes(h, stencil_level0=(name == "u"))
        out[name + "_ms"] = ms
        out[name + "_levels"] = h.n_levels()
        out[name + "_bytes"] = nb
        out[name + "_gbs"] = nb / ms / 1e6
    # the u-cycle as the Newton step runs it (operator_kind 1): the finest level's residual and
    # smoothing sweep matrix-free; its bytes exclude the two level-0 A applies (FP64-bound)
    if P.dim == 3:
        hu.set_matrix_free(P, cs, mat, reg, phi_old)
        r = torch.randn(P.n_u, dtype=torch.float64, device=x_final.device)
        hu.v_cycle(r)
        ms = time_events(lambda: hu.v_cycle(r), 10, stream)
        out["u_ms_matrix_free"] = ms
    out["note"] = ("one V-cycle application (zero initial guess, 1+1 damped Jacobi sweeps per level, dense LU on the "
                   "coarsest); bytes = per level 2 A applies (residual and post-sweep, fused with their vector "
                   "updates) + R + P in their storage formats + 56 B per row of vector traffic; u_ms_matrix_free: "
                   "the same u-cycle with the finest level's two A applies matrix-free, as the Newton step runs it")
    return out


def vcycle_bytes(h, stencil_level0):
    """Algorithmic bytes of one V-cycle: per non-coarsest level 2 SpMV(A) (the residual b - A x and the
    fused post-smoothing sweep), SpMV(R), SpMV(P) with their x/y vectors, plus 56 B per row (pre-sweep
    reads b, D^-1 and writes x: 24 B; the residual reads b, the prolongation reads x, the post-sweep
    reads b and D^-1: 32 B)."""
    tot = 0
    for lev in range(h.n_levels() - 1):
        i = h.level_info(lev)
        n, nc = i["rows"], i["coarse"]
        fa = stencil_bytes if (stencil_level0 and lev == 0) else csr_bytes
        tot += 2 * fa(n, n, i["nnz_A"]) + csr_bytes(n, nc, i["nnz_P"]) + csr_bytes(nc, n, i["nnz_P"]) + 56 * n
    return tot


def rebuild_probe():
    """One warm config-3 step with CF_NO_AMG_REUSE=1 CF_NO_UU_REUSE=1 (M_uu re-assembled and every
    hierarchy rebuilt every iteration, as the reference does)."""
    import torch
    import paper_1806_09924_b200 as cf
    s = torch.cuda.current_stream()
    cf.set_stream(s)
    P, mat, reg = sneddon_setup(cf, CFG3)
    st0 = cf.make_initial_state(P, mat).get()
    sol0 = torch.from_numpy(st0["solution"]).cuda()
    po0 = torch.from_numpy(st0["phi_old"]).cuda()
    cf.newton_active_set_step(cf.FractureState(P, sol0, po0, po0, 1), mat, P, reg, cf.SolverOptions())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    rep = cf.newton_active_set_step(cf.FractureState(P, sol0, po0, po0, 1), mat, P, reg, cf.SolverOptions())
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    its = len(rep["iterations"])
    print(json.dumps({"value": P.n_total * its / (ms * 1e-3), "unit": "DoF/s", "ms_per_step": ms,
                      "newton_iterations": its, "note": "CF_NO_AMG_REUSE=1 CF_NO_UU_REUSE=1: M_uu re-assembled and u- and "
                      "phi-hierarchies rebuilt every Newton iteration, as the reference does; identical iterates"}))


def ours(args):
    import torch
    rank, world, local = dist_setup()
    import paper_1806_09924_b200 as cf
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    s = torch.cuda.current_stream()
    cf.set_stream(s)
    P, mat, reg = sneddon_setup(cf, CFG4 if args.workload == "cfg4" else CFG3)
    opts = cf.SolverOptions()
    st0 = cf.make_initial_state(P, mat).get()
    sol0 = torch.from_numpy(st0["solution"]).to(device)
    po0 = torch.from_numpy(st0["phi_old"]).to(device)
    # N > 1: one config-3 step split over the ranks (z-slabs, NCCL halo planes, segmented dots, the
    # gathered global block AMG): strong scaling of the same workload, bitwise the 1-GPU step
    comm = cf.Communicator.from_torch_distributed() if world > 1 else None

    def step():
        st = cf.FractureState(P, sol0, po0, po0, 1)  # device-to-device reset of the seeded state
        return st, cf.newton_active_set_step(st, mat, P, reg, opts, comm=comm)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    l0 = cf.kernel_launches()
    reps = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]  # per-step split (no syncs)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(s)
        for k in range(args.steps):
            st = None  # the previous step's state is released before the next one is created (as in warm-up)
            st, rep = step()
            reps.append(rep)
            marks[k].record(s)
        e1.record(s)
        torch.cuda.synchronize()
    launches = cf.kernel_launches() - l0
    ms = e0.elapsed_time(e1) / args.steps
    ms_each = [e0.elapsed_time(marks[0])] + [marks[k - 1].elapsed_time(marks[k]) for k in range(1, args.steps)]
    its = sum(len(r["iterations"]) for r in reps) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
    value = P.n_total * its / (ms * 1e-3)
    last = reps[-1]
    free, total = torch.cuda.mem_get_info()

    # the converged solution (V-cycle leg), then the last device state is released so the e2e step
    # allocates like a timed step does
    x_final = st.get()["solution"]
    st = None
    # e2e: through the C ABI with pinned host buffers (H2D of the state, Newton step, D2H of the
    # whole state back into pinned host memory)
    import ctypes as C
    from paper_1806_09924_b200._lib import check, load
    h_sol = torch.from_numpy(st0["solution"]).pin_memory().numpy()
    h_po = torch.from_numpy(st0["phi_old"]).pin_memory().numpy()
    o_sol = torch.empty(P.n_total, dtype=torch.float64).pin_memory().numpy()
    o_po = torch.empty(P.n_vertices, dtype=torch.float64).pin_memory().numpy()
    o_pp = torch.empty(P.n_vertices, dtype=torch.float64).pin_memory().numpy()
    o_step = C.c_int()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st_h = cf.FractureState(P, h_sol, h_po, h_po, 1)
    rep_h = cf.newton_active_set_step(st_h, mat, P, reg, opts, comm=comm)
    check(load().cf_state_get(st_h._h, o_sol.ctypes.data_as(C.c_void_p), o_po.ctypes.data_as(C.c_void_p),
                              o_pp.ctypes.data_as(C.c_void_p), C.byref(o_step)))
    x_h = o_sol
    e2e_s = time.perf_counter() - t0
    e2e = {"value": P.n_total * len(rep_h["iterations"]) / e2e_s, "unit": "DoF/s", "seconds": e2e_s,
           "h2d_bytes_per_step": 8 * (P.n_total + 2 * P.n_vertices), "d2h_bytes_per_step": 8 * (P.n_total + 2 * P.n_vertices),
           "path": "cf_state_create(pinned host) + cf_newton_active_set_step + cf_state_get(pinned host)",
           "newton_iterations": len(rep_h["iterations"]), "solution_finite": bool(np.isfinite(x_h).all())}
    if comm is not None:  # release the NCCL communicator while every rank is alive (not at exit)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        del comm
        import gc
        gc.collect()
        torch.distributed.barrier()

    # the same step with every AMG hierarchy rebuilt (no bitwise-verified reuse), in a subprocess
    # because the switch is read once per process
    full = None
    if rank == 0 and world == 1 and not args.no_rebuild_check:
        try:
            env = dict(os.environ, CF_NO_AMG_REUSE="1", CF_NO_UU_REUSE="1")
            r = subprocess.run([sys.executable, __file__, "--rebuild-probe"], env=env, capture_output=True,
                               text=True, timeout=600)
            full = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as ex:  # reported, never fatal
            full = {"error": str(ex)[:200]}

    vcyc = None
    if rank == 0 and world == 1:
        try:
            vcyc = vcycle_leg(cf, P, mat, reg, torch.from_numpy(x_final).to(device), po0, s)
        except Exception as ex:  # reported, never fatal
            vcyc = {"error": str(ex)[:200]}
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank != 0:
        return
    op, roof = operator_leg(cf, device, s) if not args.no_operator else (None, None)
    out = {
        "metric": METRIC if args.workload == "cfg3" else METRIC4, "value": value, "unit": "DoF/s", "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Sneddon state)",
        "config": dict(CONFIG if args.workload == "cfg3" else CONFIG4, parallelism="single GPU" if world == 1 else
                       f"{world} GPUs: z-slab decomposition, NCCL halo planes, segmented NP-invariant dots, the undivided block AMG "
                       f"gathered on every rank (the N-rank step is bitwise the 1-GPU step)"),
        "ms_each_step": ms_each, "newton_iterations_per_step": its, "ms_per_newton_iteration": ms / its,
        "gmres_iterations": [r["gmres_iterations"] for r in last["iterations"]],
        "active_set_final": last["iterations"][-1]["active_size"],
        "phase_ms_last_step": last["times_ms"], "device_mem_used_gb": (total - free) / 1e9,
        "roofline": roof, "operator": op, "e2e": e2e, "gpu_launches": int(launches),
        "full_rebuild": full, "vcycle": vcyc,
        "gpu_launches_per_step": launches / args.steps, "clocks": clk.summary(),
    }
    if not args.no_cpu and world == 1:
        out["cpu_baseline"] = cpu_baseline_leg(value, full)
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg4"],
                    help="cfg4 (256^3, the strong-scaling config) needs >= 4 GPUs of memory")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-operator", action="store_true")
    ap.add_argument("--no-rebuild-check", action="store_true")
    ap.add_argument("--rebuild-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.rebuild_probe:
        rebuild_probe()
        return
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
