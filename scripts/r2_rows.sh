# row sweeps of 512 with 8 elements per thread (default) vs 16 (_ab/e16)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_slab.py tests/test_gpu_operators.py -m gpu -q -x > gpurun_out/rows_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rows_tests.log
tail -3 gpurun_out/rows_tests.log
rm -f gpurun_out/rows_k.txt
for lib in "" _ab/e16/libfftcond_b200.so "" _ab/e16/libfftcond_b200.so; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/rows_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 basic,em,basic_sub,em_sub >> gpurun_out/rows_k.txt 2>&1
done
for lib in "" _ab/e16/libfftcond_b200.so; do
  echo "== 2-D 512 lib=${lib:-default}" >> gpurun_out/rows_k.txt
  FFTC_LIB=$lib python scripts/scheme_kernels.py 512 >> gpurun_out/rows_k.txt 2>&1
done
cat gpurun_out/rows_k.txt
timeout 600 python scripts/stress_determinism.py --reps 2 --groups c2small,3d > gpurun_out/rows_stress.txt 2>&1; tail -2 gpurun_out/rows_stress.txt
