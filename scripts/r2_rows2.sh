# em_sub sweep 1 with both channels per thread (default) vs split thread groups (_ab/cpt0), register budgets
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_slab.py -m gpu -q -x > gpurun_out/rows2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rows2_tests.log
tail -3 gpurun_out/rows2_tests.log
rm -f gpurun_out/rows2_k.txt
for lib in "" _ab/cpt0/libfftcond_b200.so _ab/minbc8/libfftcond_b200.so _ab/minbc4/libfftcond_b200.so "" _ab/cpt0/libfftcond_b200.so; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/rows2_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 em_sub >> gpurun_out/rows2_k.txt 2>&1
done
for lib in "" _ab/cpt0/libfftcond_b200.so; do
  echo "== 2-D 512 lib=${lib:-default}" >> gpurun_out/rows2_k.txt
  FFTC_LIB=$lib python scripts/scheme_kernels.py 512 >> gpurun_out/rows2_k.txt 2>&1
done
cat gpurun_out/rows2_k.txt
