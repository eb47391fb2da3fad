set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_c3.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
tail -3 gpurun_out/smoke.log gpurun_out/gputests.log; tail -c 3000 gpurun_out/bench_c3.log
