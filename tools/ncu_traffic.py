"""Per-launch DRAM traffic of the z-pass and xy-pass from an ncu report into
profiles/kernel_traffic.json (bench.py reports it as roofline.traffic).
Usage: python tools/ncu_traffic.py report.ncu-rep CONFIG "source note" """
import csv
import io
import json
import os
import subprocess
import sys

rep, config, note = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]


def val(r, name):
    i = h.index(name)
    x = float(r[i].replace(",", ""))
    u = units[i]
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1.0, "us": 1e-3, "ns": 1e-6,
                "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}.get(u, 1.0)


path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "kernel_traffic.json")
tj = json.load(open(path)) if os.path.exists(path) else {}
for r in rows[2:]:
    k = r[h.index("Kernel Name")]
    name = "xypass" if "xypass" in k else "zpass" if "zpass" in k else None
    if not name:
        continue
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    tj[f"{config}:{name}"] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                              "duration_ms_under_ncu": val(r, "gpu__time_duration.sum"),
                              "fp64_pipe_pct": val(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                              "source": note}
json.dump(tj, open(path, "w"), indent=1)
print(json.dumps({k: v["dram_bytes_per_launch"] for k, v in tj.items() if ":" in k}, indent=1))
