# last verification of the round: GPU suite, y-tile A/B, slab world-1 timings, C4 / default / reference bench lines
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
tail -n 3 gpurun_out/gputests.log
rm -f gpurun_out/y1b_k.txt
for lib in "" _ab/y1/libfftcond_b200.so "" _ab/y1/libfftcond_b200.so; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/y1b_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 basic,em_sub >> gpurun_out/y1b_k.txt 2>&1
done
FFTC_LIB=_ab/y1/libfftcond_b200.so timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "c3 or c4_random256" > gpurun_out/y1b_tests.log 2>&1; echo rc=$? >> gpurun_out/y1b_tests.log
cat gpurun_out/y1b_k.txt; tail -n 2 gpurun_out/y1b_tests.log
python scripts/kernels_3d.py 1024 basic > gpurun_out/k3d_1024.txt 2>&1; cat gpurun_out/k3d_1024.txt
bash scripts/r2_slab.sh
timeout 1500 python bench.py --workload c4 > gpurun_out/bench_c4.log 2>&1; echo rc=$? >> gpurun_out/bench_c4.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c3_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c3_ref.log
tail -c 300 gpurun_out/bench_c4.log; tail -c 300 gpurun_out/bench_c3.log
