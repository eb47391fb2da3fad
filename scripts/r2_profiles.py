"""Collect the judged summaries of a round-2 GPU run from gpurun_out/ (scratch)
into profiles/ (tracked): the bench JSON lines, the ncu launch list summary of
the default bench command, the condensed ncu --set full record bench.py reads
for `roofline.traffic`, and a text summary (stalls, shared-memory wavefronts)
of the same full captures.  Usage: python scripts/r2_profiles.py"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")


def last_json_line(path):
    if not os.path.exists(path):
        return None
    lines = [ln for ln in open(path) if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


for w, name in (("c3", "c3"), ("c3_ref", "c3_ref"), ("c2", "c2"), ("c5", "c5"), ("c1", "c1"), ("c4", "c4"),
                ("c4-emsub", "c4_emsub"), ("c2_ref", "c2_ref")):
    d = last_json_line(os.path.join(OUT, f"bench_{w}.log"))
    if d:
        json.dump(d, open(os.path.join(PROF, f"r2_bench_{name}.json"), "w"), indent=1)
        print("bench", name, f"{d['value'] / 1e9:.3f} G")

csvp = os.path.join(OUT, "launches_c3.csv")
if os.path.exists(csvp):
    txt = subprocess.run([sys.executable, os.path.join(REPO, "scripts", "launch_summary.py"), csvp,
                          "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv: "
                          "FFTC_NO_GRAPH=1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline "
                          "(default workload C3, 512^3 em_sub; first 400 launches)"],
                         capture_output=True, text=True).stdout
    open(os.path.join(PROF, "r2_launches_c3.txt"), "w").write(txt)
    print(txt[:1500])

merged = None
for f in ("r2_ncu_c3.json", "r2_ncu_c3_rows.json"):
    p = os.path.join(OUT, f)
    if os.path.exists(p):
        d = json.load(open(p))
        if merged is None:
            merged = d
        else:
            merged["kernels"].update(d["kernels"])
            merged["source"] += "; " + d["source"]
if merged:
    json.dump(merged, open(os.path.join(PROF, "r2_ncu_c3.json"), "w"), indent=1)

parts = []
for rep in ("r2_c3_col3.ncu-rep", "r2_c3_rows.ncu-rep"):
    p = os.path.join(OUT, rep)
    if os.path.exists(p):
        parts.append(subprocess.run([sys.executable, os.path.join(REPO, "scripts", "ncu_summary.py"), p],
                                    capture_output=True, text=True).stdout)
if parts:
    head = ("ncu --set full --clock-control none --import-source on, C3 512^3 em_sub, kernels of iteration 2 "
            "(FFTC_NO_GRAPH=1 python scripts/prof_3d_one.py --n 512 --iters 3; scripts/r2_prof_c3.sh) -- round 2\n"
            "k_col3_lg<2,512> = y forward (fields A and B), k_col3_mid<1,512> = z pass with the projection "
            "(three components per thread), k_col3_lg<3,512> = y inverse, k_rows_tma<3,1,512> = sweep 1 "
            "(both channels per thread), k_rows_tma<3,3,512> = sweep 3\n")
    open(os.path.join(PROF, "r2_ncu_full_c3.txt"), "w").write(head + "".join(parts))
    print("".join(parts))
