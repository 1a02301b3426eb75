"""The slab-decomposed Newton step with several ranks, on one GPU, through the host-staged test
transport (Communicator.from_gloo): exercises the whole multi-rank control flow of newton.cu
(halo planes, active-set flag exchange, segmented NP-invariant dots, the gathered global block
AMG, final all-gather of the solution) without NCCL.  Nothing here is a measurement.

Default preconditioner (the undivided block AMG, gathered on every rank): the N-rank step must be
BITWISE the single-GPU step — transcript (residual norms, |A|, set changes, GMRES counts) and
solution — because every row and every dot is computed in an order that does not depend on N.
The local variants (CF_RAS=1 restricted additive Schwarz, CF_BLOCK_JACOBI=1) change the
preconditioner with N: they must still converge to the same solution to Newton tolerance."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _setup(cf, d, n0, r):
    P = cf.Problem(d, 10.0, n0, r)
    mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    return P, mat, reg


def _worker(rank, size, port, out_dir, d, n0, r):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_1806_09924_b200 as cf
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    torch.cuda.set_device(0)
    comm = cf.Communicator.from_gloo()
    P, mat, reg = _setup(cf, d, n0, r)
    st = cf.make_initial_state(P, mat)
    opk = int(os.environ.get("CF_TEST_OPKIND", "0"))
    rep = cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions(operator_kind=opk), comm=comm)
    x = st.get()["solution"]
    its = np.array([[it["residual_norm"], it["active_size"], it["set_changes"], it["gmres_iterations"]]
                    for it in rep["iterations"]])
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    np.save(os.path.join(out_dir, f"its{rank}.npy"), its)
    np.save(os.path.join(out_dir, f"conv{rank}.npy"), np.array([rep["converged"], rep["feasibility_violation"]]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("d,n0,r,size,mode", [(3, 4, 2, 2, "global"), (3, 4, 2, 3, "global"), (2, 8, 3, 4, "global"),
                                               (3, 4, 2, 2, "global-mf"), (3, 4, 2, 3, "global-mf"),
                                               (3, 8, 1, 4, "global-mf"), (3, 4, 2, 3, "global-replicated-mf"),
                                               (3, 8, 1, 4, "global"), (3, 4, 2, 3, "global-replicated"),
                                               (3, 4, 2, 3, "ras"), (2, 8, 3, 4, "block_jacobi")])
def test_multirank_newton_step(tmp_path, d, n0, r, size, mode):
    """global: the hierarchy's levels of >= 256 rows apply by rows split over the ranks
    (CF_VCYCLE_SPLIT_MIN lowers the production threshold so these small grids exercise it);
    global-replicated: every rank applies the whole V-cycle."""
    import torch.multiprocessing as mp
    import paper_1806_09924_b200 as cf
    env = {"ras": {"CF_RAS": "1"}, "block_jacobi": {"CF_BLOCK_JACOBI": "1"},
           "global": {"CF_VCYCLE_SPLIT_MIN": "256"},
           # the default matrix-free M_uu (operator_kind 1): slab rows and level-0 row chunks
           "global-mf": {"CF_VCYCLE_SPLIT_MIN": "256", "CF_TEST_OPKIND": "1"},
           "global-replicated-mf": {"CF_VCYCLE_REPLICATED": "1", "CF_TEST_OPKIND": "1"},
           "global-replicated": {"CF_VCYCLE_REPLICATED": "1"}}[mode]
    os.environ.update(env)
    try:
        mp.spawn(_worker, args=(size, _free_port(), str(tmp_path), d, n0, r), nprocs=size, join=True)
    finally:
        for k in env:
            del os.environ[k]
    xs = [np.load(tmp_path / f"x{k}.npy") for k in range(size)]
    its = [np.load(tmp_path / f"its{k}.npy") for k in range(size)]
    conv = [np.load(tmp_path / f"conv{k}.npy") for k in range(size)]
    assert all(c[0] for c in conv), "a rank did not converge"
    for k in range(1, size):
        assert np.array_equal(xs[k], xs[0]), "ranks disagree on the gathered solution"
        assert np.array_equal(its[k], its[0]), "ranks disagree on the Newton transcript"
    P, mat, reg = _setup(cf, d, n0, r)
    st = cf.make_initial_state(P, mat)
    rep = cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions(operator_kind=int(env.get("CF_TEST_OPKIND", "0"))))
    assert rep["converged"]
    ref = st.get()["solution"]
    ref_its = np.array([[it["residual_norm"], it["active_size"], it["set_changes"], it["gmres_iterations"]]
                        for it in rep["iterations"]])
    if mode.startswith("global"):
        assert np.array_equal(its[0], ref_its), (its[0], ref_its)
        assert np.array_equal(xs[0], ref), f"max |dx| = {np.abs(xs[0] - ref).max()}"
    else:
        assert np.linalg.norm(xs[0] - ref) <= 1e-6 * np.linalg.norm(ref)
        assert int(its[0][-1, 1]) == rep["iterations"][-1]["active_size"]


def test_nccl_transport_selftest_one_rank():
    """The NCCL transport itself (comm.cu): libnccl loaded from the process, the symbol table, id /
    init / destroy, all-gather in and out of place, int64 sum / max all-reduce, broadcast, grouped
    broadcasts and a grouped send / receive, each executed on a one-rank communicator on the
    library stream and checked on the host.  (Two NCCL ranks cannot share this box's one GPU; the
    multi-rank control flow above runs through the host transport.)"""
    import paper_1806_09924_b200 as cf
    assert cf.Communicator.nccl_selftest() == 0
