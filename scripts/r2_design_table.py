"""Print the DESIGN.md section-4 tables from the committed bench lines (profiles/r2_bench_*.json)."""
import json
import os

P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
print("| config | G vox-it/s (e2e) | ms / step | iteration: bytes/voxel-iter survey (schedule) | fraction of HBM peak survey (schedule) | dominant kernel: frac | median SM MHz |")
print("|---|---|---|---|---|---|---|")
for name in ("c3", "c2", "c5", "c1", "c4", "c4_emsub"):
    p = os.path.join(P, f"r2_bench_{name}.json")
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    ir, r, ck = d.get("iteration_roofline", {}), d.get("roofline", {}), d.get("clocks", {})
    print(f"| {name} | {d['value'] / 1e9:.2f} ({d['e2e']['value'] / 1e9:.2f}) | {d['ms_per_step']:.0f} | "
          f"{ir.get('bytes_per_voxel_iter_survey', 0):.0f} ({ir.get('bytes_per_voxel_iter_schedule', 0):.0f}) | "
          f"{ir.get('frac_survey_bytes', 0):.3f} ({ir.get('frac_schedule_bytes', 0):.3f}) | "
          f"{r.get('kernel')}: {r.get('frac', 0):.3f} | {ck.get('sm_mhz')} {ck.get('reasons')} |")
    if "kernels" in d and name in ("c3", "c4", "c4_emsub"):
        print("|  | " + "; ".join(f"{k} {v['ms_per_launch']:.2f} ms ({v['frac_hbm']:.2f})" for k, v in d["kernels"].items()
                                  if v.get("frac_hbm")) + " | | | | | |")
for name in ("c3_ref",):
    p = os.path.join(P, f"r2_bench_{name}.json")
    if os.path.exists(p):
        d = json.load(open(p))
        print(name, d["value"], d["cpu_baseline"]["cores"], d["cpu_baseline"]["kind"])
