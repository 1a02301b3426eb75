"""bench.py — driver benchmark of the B200 hot path.

Default workload (N=1): BASELINE config 1, the operator microbenchmark — the assembled
degraded-elasticity block M_uu of a 3d 192^3 Q1 mesh (21,567,171 u dofs, 1,676,188,257 nnz),
applied to u ~ N(0,1) with phi_tilde ~ U[0,1] (counter-based SplitMix64, seeds 180609924001/2).
One step = one y = M_uu u through the library's C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  value = whole-job operator throughput in GB/s of algorithmic
CSR bytes (int64 row pointers), inputs resident in HBM; e2e = the same metric through the C ABI
with pinned HOST buffers (H2D of u and D2H of y inside the timed region).
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
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


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


CFG1 = dict(dim=3, half_width=10.0, n0=12, refinements=4)  # 192^3 cells


def config1_host(dim=3, half_width=10.0, n0=12, refinements=4):
    nn = (n0 << refinements) + 1
    V = nn ** dim
    pt = splitmix_uniform(SEED_PHI, V)
    u = splitmix_normal(SEED_U, dim * V)
    return V, pt, u


def config1_inputs(cf, device="cuda", **over):
    """Problem, constraints (Dirichlet), material, regularization, x = (u, phi_tilde), phi_tilde."""
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
    ptd = torch.from_numpy(pt).to(device)
    return P, cs, mat, reg, x, ptd


def csr_bytes(rows, cols, nnz):
    """Compulsory bytes of one CSR SpMV: 12 nnz (8 B value + 4 B column) + 8 (rows+1) int64 row
    pointers + 8 cols (x) + 8 rows (y)."""
    return 12 * nnz + 8 * (rows + 1) + 8 * cols + 8 * rows


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
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


def dist_setup(gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def reference_arm(args):
    """--impl reference: the reference's CPU path (the oracle port: the reference itself cannot be
    built here) on the host cores, same metric/config, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import orc
    n_thr = os.cpu_count() or 1
    P, J, u, nb = cpu_sample()
    y = np.zeros(P.n_u)
    for _ in range(args.warmup):
        orc.lib().orc_block_spmv_threads(J.h_, 0, orc._p(u), orc._p(y), n_thr)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        orc.lib().orc_block_spmv_threads(J.h_, 0, orc._p(u), orc._p(y), n_thr)
    dt = (time.perf_counter() - t0) / args.steps
    gbs = nb / dt / 1e9
    sample = f"3d {P.ncells_side}^3 M_uu (1/{(192 // P.ncells_side) ** 3} of config 1), same input distributions"
    out = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "dtype": "f64", "data": "synthetic", "config": CONFIG,
           "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": n_thr, "kind": "port", "sample": sample},
           "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


METRIC = "operator-apply HBM GB/s (M_uu CSR SpMV, config 1)"
CONFIG = {"workload": "config1: M_uu apply, 3d 192^3 Q1 hex, 21,567,171 u dofs, FP64",
          "format": "CSR int64 rowptr / int32 col", "l2": "inputs 20.6 GB >> 126 MB L2 (no flush needed)",
          "parallelism": "single GPU"}


def cpu_sample(cells_side=48):
    from oracle import orc
    r = {48: 2, 96: 3}[cells_side]
    P = orc.Problem(3, 10.0, 12, r)
    P.ncells_side = cells_side
    nn = cells_side + 1
    V = nn ** 3
    pt = splitmix_uniform(SEED_PHI, V)
    u = splitmix_normal(SEED_U, 3 * V)
    h = P.h
    mat = orc.material(kappa_factor=1e-12 / h, eps_mode=1, eps_fixed=2 * h)
    reg = orc.Regularization(2 * h, 1e-12)
    cs = P.constraints(True)
    x = np.concatenate([u, pt])
    J = P.jacobian(cs, mat, reg, x, pt)
    A = J.csr(0)
    return P, J, np.ascontiguousarray(u), csr_bytes(A.rows, A.cols, A.nnz)


def cpu_baseline_leg(seconds=10.0):
    """Single-thread oracle SpMV on the bounded sample (~10 s of CPU work)."""
    from oracle import orc
    P, J, u, nb = cpu_sample()
    y = np.zeros(P.n_u)
    orc.lib().orc_block_spmv_threads(J.h_, 0, orc._p(u), orc._p(y), 1)
    n = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        orc.lib().orc_block_spmv_threads(J.h_, 0, orc._p(u), orc._p(y), 1)
        n += 1
    dt = (time.perf_counter() - t0) / n
    return {"value": nb / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"3d 48^3 M_uu (1/64 of config 1), same distributions, {n} applies, oracle port "
                      "(reference not buildable: Eigen3 absent)"}


def ours(args):
    import torch
    rank, world, local = dist_setup(args.gpus)
    import paper_1806_09924_b200 as cf
    torch.cuda.set_device(local)
    s = torch.cuda.current_stream()
    cf.set_stream(s)
    P, cs, mat, reg, x, pt = config1_inputs(cf, device=f"cuda:{local}")
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    del pt
    nu = P.n_u
    u = x[:nu].contiguous()
    del x
    y = torch.empty(nu, dtype=torch.float64, device=u.device)
    nb = csr_bytes(nu, nu, J.nnz[0])
    # strong-scaling row slabs would split the rows; round 1 runs one replica per rank
    for _ in range(args.warmup):
        J.spmv(0, u, out=y)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    l0 = cf.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(s)
        for _ in range(args.steps):
            J.spmv(0, u, out=y)
        ev1.record(s)
        torch.cuda.synchronize()
    launches = cf.kernel_launches() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=u.device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
    value = world * nb / (ms * 1e-3) / 1e9

    # e2e: through the C ABI with pinned host buffers (H2D u + SpMV + D2H y per step)
    uh = u.cpu().pin_memory()
    yh = torch.empty(nu, dtype=torch.float64).pin_memory()
    uh_np, yh_np = uh.numpy(), yh.numpy()
    for _ in range(2):
        J.spmv(0, uh_np, out=yh_np)
    torch.cuda.synchronize()
    ke = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(ke):
        J.spmv(0, uh_np, out=yh_np)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) / ke * 1e3
    ok = bool(torch.allclose(yh.cuda(), y, rtol=0, atol=0))

    if rank != 0:
        return
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = nb / (ms * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SplitMix64 seeds 180609924001/2)",
        "config": CONFIG,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "k_spmv<32>", "bytes_per_launch": nb,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "when" in peaks else "fallback"},
        "e2e": {"value": nb / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 8 * nu, "d2h_bytes_per_step": 8 * nu, "path": "cf_block_spmv, pinned host",
                "matches_device": ok},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "nnz": J.nnz[0],
    }
    if not args.no_cpu and world == 1:
        out["cpu_baseline"] = cpu_baseline_leg(args.cpu_seconds)
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
