"""Within a load step M_uu depends only on phi_tilde and the Dirichlet set (model.cpp:268-276), so the
Newton driver assembles it once per step and the u-hierarchy built from it is reused.  These runs
re-assemble M_uu every iteration and check it bitwise (CF_VERIFY_UU_REUSE=1), and rebuild every
hierarchy (CF_NO_AMG_REUSE=1): the solutions must be bitwise those of the default run."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1806_09924_b200 as cf
P = cf.Problem(3, 10.0, 4, 2)
mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
st = cf.make_initial_state(P, mat)
reps = cf.solve_loading_sequence(st, mat, P, reg, cf.SolverOptions(), 2)
assert all(r["converged"] for r in reps)
np.save({out!r}, st.get()["solution"])
"""


def _run(tmp_path, name, env_extra):
    out = str(tmp_path / f"{name}.npy")
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, out=out)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def test_uu_and_hierarchy_reuse_are_exact(tmp_path):
    base = _run(tmp_path, "base", {})
    ver = _run(tmp_path, "verify", {"CF_VERIFY_UU_REUSE": "1"})
    full = _run(tmp_path, "full", {"CF_NO_AMG_REUSE": "1", "CF_NO_UU_REUSE": "1"})
    assert np.array_equal(base, ver)
    assert np.array_equal(base, full)
