"""Condense an ncu --set full report into the per-kernel record bench.py
reads (profiles/r2_ncu_<workload>.json): DRAM bytes read/written per launch,
duration, FP64-pipe and issue utilisation, occupancy, registers.
Usage: python scripts/ncu_to_json.py <report.ncu-rep> <out.json> <source text> name=regex [name=regex ...]"""
import csv
import io
import json
import re
import subprocess
import sys

rep, out, source = sys.argv[1:4]
names = [a.split("=", 1) for a in sys.argv[4:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def val(r, k, scale_units=True):
    if k not in hdr:
        return None
    v = r[hdr.index(k)].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    u = units[hdr.index(k)]
    if scale_units:
        x *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3, "msecond": 1.0,
              "nsecond": 1e-6, "%": 0.01}.get(u, 1.0)
    return x


rec = {"source": source, "kernels": {}}
for r in rows[2:]:
    kname = r[hdr.index("Kernel Name")]
    for nm, rx in names:
        if re.search(rx, kname):
            k = rec["kernels"].setdefault(nm, {"launches": 0, "kernel": kname})
            k["launches"] += 1
            for key, metric in (("dram_read", "dram__bytes_read.sum"), ("dram_write", "dram__bytes_write.sum"),
                                ("ms", "gpu__time_duration.sum"),
                                ("fp64_pipe", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                                ("issue_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                ("occupancy", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                                ("registers", "launch__registers_per_thread")):
                v = val(r, metric)
                if v is not None:
                    k.setdefault("_" + key, []).append(v)
for k in rec["kernels"].values():
    for key in [x for x in k if x.startswith("_")]:
        vals = k.pop(key)
        k[key[1:]] = sum(vals) / len(vals)
json.dump(rec, open(out, "w"), indent=1)
print(json.dumps(rec, indent=1))
