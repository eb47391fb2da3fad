# verification after a kernel change: GPU suite, C3 per-kernel timings, default bench, ncu captures
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
python scripts/kernels_3d.py 512 basic,em_sub > gpurun_out/k3d_now.txt 2>&1; cat gpurun_out/k3d_now.txt
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
bash scripts/r2_prof_c3.sh > gpurun_out/prof_c3.log 2>&1; tail -5 gpurun_out/prof_c3.log
FFTC_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -c 400 gpurun_out/bench_c3.log
