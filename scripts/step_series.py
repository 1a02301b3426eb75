"""Per-step device times of consecutive config-3 Newton steps, without and with bench.py's clock
sampler running (allocator / host / NVML-sampling variance diagnostics), phases per step.
usage: python scripts/step_series.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st0 = cf.make_initial_state(P, mat).get()
sol0 = torch.from_numpy(st0["solution"]).cuda()
po0 = torch.from_numpy(st0["phi_old"]).cuda()
opts = cf.SolverOptions()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 6


def series(label):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    torch.cuda.synchronize()
    ev[0].record(s)
    reps = []
    for k in range(n):
        st = cf.FractureState(P, sol0, po0, po0, 1)
        reps.append(cf.newton_active_set_step(st, mat, P, reg, opts))
        ev[k + 1].record(s)
    torch.cuda.synchronize()
    print(label, [round(ev[k].elapsed_time(ev[k + 1]), 1) for k in range(n)], flush=True)
    for r in reps:
        print("   ", {k: round(v, 1) for k, v in r["times_ms"].items()}, flush=True)


series("no sampler")
with bench.ClockSampler(0) as clk:
    series("sampler   ")
print(clk.summary())
