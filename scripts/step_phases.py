"""CF_TIMING breakdown of the AMG builds inside one warm config-3 Newton step, summed per phase for
the u-build and the phi-builds.  usage: CF_TIMING=1 python scripts/step_phases.py 2> log; python scripts/step_phases.py --parse log"""
import collections
import os
import re
import sys

if len(sys.argv) > 2 and sys.argv[1] == "--parse":
    lines = open(sys.argv[2]).read().split("@@STEP2@@")[1].splitlines()
    # the first hierarchy built in a step is M_uu's, the others are M_phiphi's (one per Newton iteration)
    kind, acc, nb = None, collections.defaultdict(float), collections.Counter()
    for ln in lines:
        m = re.match(r"\[amg L(\d+)\] (.+?)\s+([\d.]+) ms", ln)
        if not m:
            continue
        if m.group(1) == "0" and m.group(2).strip() == "strength":
            kind = "u" if not nb else "phi"
            nb[kind] += 1
        acc[(kind, "L" + m.group(1), m.group(2).strip())] += float(m.group(3))
    print("builds", dict(nb))
    for k in sorted(acc):
        print(f"{k[0]:4s} {k[1]:3s} {k[2]:14s} {acc[k]:9.2f} ms")
    for kd in ("u", "phi"):
        print(kd, "total", round(sum(v for k, v in acc.items() if k[0] == kd), 1))
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1806_09924_b200 as cf

P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
for i in range(2):
    if i == 1:
        sys.stderr.write("@@STEP2@@\n")
        sys.stderr.flush()
    st = cf.make_initial_state(P, mat)
    cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions())
