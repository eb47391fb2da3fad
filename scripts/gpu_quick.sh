#!/bin/bash
# on the GPU box: parity tests then a short bench with the kernel breakdown
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_operators.py -m gpu -q -x --tb=line 2>&1 | tail -3
python bench.py --workload ${1:-c2-fast} --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_quick.log
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_quick.log"))
print(f"value {d['value']/1e9:.3f} G  ms/step {d['ms_per_step']:.2f}  e2e {d['e2e']['value']/1e9:.3f} G  frac(schedule) {d['iteration_roofline']['frac_schedule_bytes']:.3f}")
for k, v in d["kernels"].items():
    print(f"  {k:22s} {v['launches']:6d} x {v['ms_per_launch']*1e3:8.1f} us")
PY
