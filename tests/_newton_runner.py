"""Helper for tests that need a fresh process (the CF_* switches are read once per process):
runs a Sneddon loading sequence on the device and prints its transcript and a SHA-256 of the
final solution as one JSON line.

  python tests/_newton_runner.py d n0 r steps [restart rtol]
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1806_09924_b200 as cf
    d, n0, r, steps = (int(a) for a in sys.argv[1:5])
    gm = cf.GmresOptions(rtol=float(sys.argv[6]), restart=int(sys.argv[5])) if len(sys.argv) > 6 else cf.GmresOptions()
    P = cf.Problem(d, 10.0, n0, r)
    mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    st = cf.make_initial_state(P, mat)
    reps = cf.solve_loading_sequence(st, mat, P, reg, cf.SolverOptions(gmres=gm, operator_kind=int(os.environ.get("CF_RUNNER_OPKIND", "0"))), steps)
    x = np.ascontiguousarray(st.get()["solution"])
    its = [[[i["residual_norm"], i["active_size"], i["set_changes"], i["gmres_iterations"]] for i in rp["iterations"]]
           for rp in reps]
    print(json.dumps({"its": its, "sha256": hashlib.sha256(x.tobytes()).hexdigest(),
                      "formats": [cf.assemble_jacobian(P, cf.build_constraints(P), mat, reg, x, x[P.n_u:]).format(w)
                                  for w in range(3)]}))


if __name__ == "__main__":
    main()
