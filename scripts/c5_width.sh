#!/bin/bash
# C5 throughput vs concurrent batch streams (FFTC_BATCH_STREAMS)
for w in ${@:-1 4}; do
  FFTC_BATCH_STREAMS=$w timeout 600 python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/c5_w$w.json
  python - "$w" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/c5_w{sys.argv[1]}.json"))
print("width", sys.argv[1], round(d["value"] / 1e9, 3), "G vox-it/s", round(d["ms_per_step"]), "ms",
      d["total_iterations"], "iters", d["points_converged"], "converged")
PY
done
