"""The oracle on the bench workload itself (BASELINE configs[3]: TGV-shaped 256^3,
12th order, RK3), once: one oracle RK3 step on the GPU host's CPU (single thread,
timed), and the full-field comparison with one step of the CUDA path on the same
input (every point of every field, D-14 metric).
Usage: python tools/oracle_fullsize.py [out.json] [n] [order]"""
import json
import math
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_01277_b200 as osbli  # noqa: E402
from inputs import TGV_PHYS, perturbed_tgv, tgv_dt  # noqa: E402
from oracle import core  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/oracle_fullsize.json"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
order = int(sys.argv[3]) if len(sys.argv) > 3 else 12
dx, dt = 2 * math.pi / n, tgv_dt(n)
Q = perturbed_tgv(n, n, n, dx=dx, amp=1e-3)
s = osbli.Solver(n, n, n, order, dx, dt, **TGV_PHYS)
s.set_state(Q)
s.step(1)
Qg = s.get_state()
p = core.OracleParams(n, n, n, order, dx, dt=dt, **TGV_PHYS)
t0 = time.perf_counter()
Qo = core.step(p, Q, 1, 1)
el = time.perf_counter() - t0
err = [float(np.max(np.abs(Qg[f] - Qo[f])) / np.max(np.abs(Qo[f]))) for f in range(5)]
cpu = platform.processor() or ""
try:
    with open("/proc/cpuinfo") as f:
        for line in f:
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
except OSError:
    pass
res = {"workload": f"TGV-shaped {n}^3 (perturbed), order {order}, RK3, dt {dt}",
       "oracle_seconds_per_step": el, "oracle_pt_steps_per_s": n ** 3 / el,
       "oracle_threads": 1, "host_cpu": cpu, "host_cores": os.cpu_count(),
       "gpu_vs_oracle_max_rel_err_per_field_after_1_step": err,
       "tolerance": 1e-11, "pass": bool(max(err) < 1e-11)}
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
