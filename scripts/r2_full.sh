# full round check on the GPU box: smoke, default bench (C3) and its reference
# arm, the GPU suite, the ncu launch list of the same bench command, the ncu
# full capture of the C3 kernels, then the other workloads' bench lines
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c3_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c3_ref.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
FFTC_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
bash scripts/r2_prof_c3.sh > gpurun_out/prof_c3.log 2>&1
for w in c2 c5 c1 c4 c4-emsub; do
  timeout 1500 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo rc=$? >> gpurun_out/bench_$w.log
done
tail -n 3 gpurun_out/smoke.log gpurun_out/gputests.log; tail -c 600 gpurun_out/bench_c3.log; tail -n 2 gpurun_out/bench_c2.log gpurun_out/bench_c5.log gpurun_out/bench_c1.log gpurun_out/bench_c4.log gpurun_out/bench_c4-emsub.log | cut -c1-400
