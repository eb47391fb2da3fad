# full round check on the GPU box: smoke, GPU suite, default bench (C3) and its
# reference arm, then the ncu launch list of the same bench command
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c3_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c3_ref.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
FFTC_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/smoke.log gpurun_out/gputests.log; tail -c 3000 gpurun_out/bench_c3.log; tail -c 1500 gpurun_out/bench_c3_ref.log
