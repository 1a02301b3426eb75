"""Device (product reduction order) vs the oracle in the reference's arithmetic order on the
config-2 schedule (3 load steps, GMRES(50) rtol 1e-10): both transcripts, the active-set
difference and the solution difference.  python scripts/refmode_diag.py n0 r [steps]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import paper_1806_09924_b200 as cf
    from oracle import orc
    import test_gpu_parity_large as T
    n0, r = int(sys.argv[1]), int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    d = 2 if len(sys.argv) <= 4 else int(sys.argv[4])
    orc.set_threads(len(os.sched_getaffinity(0)))
    P, O, mat, omat, reg, oreg, phi = T._pair(cf, orc, d, n0, r)
    gm = cf.GmresOptions(rtol=1e-10, restart=50) if d == 2 else None
    t0 = time.time()
    reps, x = T._device_run(cf, P, mat, reg, steps, gm)
    t1 = time.time()
    out = {"n_total": P.n_total, "device_s": t1 - t0, "device": [T._its(a).tolist() for a in reps]}
    for name, order in (("product_order", 0), ("reference_order", 1)):
        orc.set_order(order)
        t0 = time.time()
        oreps, xo = T._oracle_run(orc, O, omat, oreg, phi, steps, gm)
        orc.set_order(0)
        nu = P.n_u
        po_dev = x[nu:]
        out[name] = {"oracle_s": time.time() - t0, "transcript": [b["iterations"].tolist() for b in oreps],
                     "bitwise_solution": bool(np.array_equal(x, xo)),
                     "solution_rel_diff": float(np.linalg.norm(x - xo) / np.linalg.norm(xo)),
                     "phi_max_abs_diff": float(np.abs(x[nu:] - xo[nu:]).max()),
                     "u_rel_diff": float(np.linalg.norm(x[:nu] - xo[:nu]) / np.linalg.norm(xo[:nu])),
                     "tcv": [cf.compute_tcv(P, x), O.tcv(xo)]}
        print(json.dumps({name: out[name]}), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"refmode_{d}d_{n0}_{r}.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
