"""GPU idle-time analysis of one warm config-3 Newton step (CUPTI kernel records via torch.profiler):
union busy time over all streams against the step's wall time, and the idle gaps attributed to the
kernel that ran before them (host round trips, launch latency, stream joins).
usage: python scripts/gpu_timeline.py [newton_max_iter]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1806_09924_b200 as cf

its = int(sys.argv[1]) if len(sys.argv) > 1 else 50
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
opts = cf.SolverOptions(newton_max_iter=its)
s = cf.make_initial_state(P, mat).get()
mk = lambda: cf.FractureState(P, s["solution"], s["phi_old"], s["phi_prev2"], 1)
cf.newton_active_set_step(mk(), mat, P, reg, opts)
st = mk()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep = cf.newton_active_set_step(st, mat, P, reg, opts)
    torch.cuda.synchronize()
ev = []
for e in prof.profiler.kineto_results.events():
    if str(e.device_type()).endswith("CUDA") and e.duration_ns() > 0:
        ev.append((e.start_ns(), e.start_ns() + e.duration_ns(), e.name(), e.device_resource_id()))
ev.sort()
print("phases", {k: round(v, 1) for k, v in rep["times_ms"].items()})
t0, t1 = ev[0][0], max(e[1] for e in ev)
busy, cur_end, gaps = 0, t0, collections.defaultdict(lambda: [0, 0])
last = None
for a, b, name, sid in ev:
    if a > cur_end:
        g = a - cur_end
        key = (last or "?")[:60] + " -> " + name[:50]
        gaps[key][0] += g
        gaps[key][1] += 1
        busy += b - a
        cur_end = b
    else:
        if b > cur_end:
            busy += b - cur_end
            cur_end = b
    if b >= cur_end:
        last = name
wall = (t1 - t0) / 1e6
print(f"wall {wall:.1f} ms, busy (union over streams) {busy / 1e6:.1f} ms, idle {wall - busy / 1e6:.1f} ms, "
      f"{len(ev)} device activities on {len(set(e[3] for e in ev))} streams")
hist = collections.Counter()
for k, (g, c) in gaps.items():
    pass
tot_by_size = collections.defaultdict(lambda: [0, 0])
cur_end = t0
for a, b, name, sid in ev:
    if a > cur_end:
        g = (a - cur_end) / 1e3
        bucket = "<2us" if g < 2 else "<5us" if g < 5 else "<10us" if g < 10 else "<30us" if g < 30 else "<100us" if g < 100 else ">=100us"
        tot_by_size[bucket][0] += g / 1e3
        tot_by_size[bucket][1] += 1
    cur_end = max(cur_end, b)
print("idle by gap size (ms, count):", {k: (round(v[0], 1), v[1]) for k, v in tot_by_size.items()})
agg = collections.defaultdict(lambda: [0, 0])
for a, b, name, sid in ev:
    agg[name[:90]][0] += b - a
    agg[name[:90]][1] += 1
print("top kernels (ms, count, mean us):")
for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {t / 1e6:8.2f} ms {c:6d} {t / c / 1e3:9.1f} us  {k}")
print("top gap contributors (idle ms, count, prev kernel -> next kernel):")
for k, (g, c) in sorted(gaps.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"  {g / 1e6:8.2f} ms {c:6d}  {k}")
