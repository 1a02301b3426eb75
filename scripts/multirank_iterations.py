"""Algorithmic scaling of the slab decomposition: GMRES / Newton iteration counts of one config-3
Newton step with N ranks (default: the gathered global block AMG, bitwise the 1-GPU step;
CF_RAS=1 restricted additive Schwarz over N z-slabs, CF_BLOCK_JACOBI=1 block-Jacobi), run with N
processes sharing one GPU through the host-staged test transport (Communicator.from_gloo).  Only the
iteration counts and the agreement of the solutions are meaningful here — the transport is not a
timing.  The rank-0 JSON carries a SHA-256 of the full solution.

usage: python scripts/multirank_iterations.py N [cfg3|cfg2]"""
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, size, port, cfg, out):
    import numpy as np
    import torch
    import torch.distributed as dist
    import bench
    import paper_1806_09924_b200 as cf
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    torch.cuda.set_device(0)
    comm = cf.Communicator.from_gloo() if size > 1 else None
    c = bench.CFG3 if cfg == "cfg3" else dict(dim=2, half_width=10.0, n0=8, refinements=8)
    P, mat, reg = bench.sneddon_setup(cf, c)
    st = cf.make_initial_state(P, mat)
    rep = cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions(), comm=comm)
    if rank == 0:
        x = st.get()["solution"]
        import hashlib
        np.save(out + f"_x{size}.npy", x[::97].copy())  # a sample: the full vector exceeds the copy-back limit
        json.dump({"ranks": size, "converged": rep["converged"],
                   "sha256": hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
                   "residuals": [it["residual_norm"] for it in rep["iterations"]],
                   "newton": len(rep["iterations"]),
                   "gmres": [it["gmres_iterations"] for it in rep["iterations"]],
                   "active": rep["iterations"][-1]["active_size"]}, open(out + f"_{size}.json", "w"))
    dist.barrier()
    del comm
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    n = int(sys.argv[1])
    cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = os.path.join(ROOT, "gpurun_out", f"multirank_{cfg}")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    mp.spawn(worker, args=(n, port, cfg, out), nprocs=n, join=True)
    print(open(out + f"_{n}.json").read())
