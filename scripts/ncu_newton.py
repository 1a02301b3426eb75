"""Target for the ncu launch list: config 3, one warm-up Newton step, then the first 2 Newton
iterations of a second step inside the NVTX range "measure" (ncu --nvtx-include measure/)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1806_09924_b200 as cf
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat)
s = st.get()
cf.newton_active_set_step(cf.FractureState(P, s["solution"], s["phi_old"], s["phi_old"], 1), mat, P, reg,
                          cf.SolverOptions())
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measure")
rep = cf.newton_active_set_step(cf.FractureState(P, s["solution"], s["phi_old"], s["phi_old"], 1), mat, P, reg,
                                cf.SolverOptions(newton_max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 2))
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(rep["times_ms"])
