# two channels per thread on 16-per-thread rows (em / em_sub sweep 1, _ab/c16) vs the split thread groups (default)
rm -f gpurun_out/rows3_k.txt
for lib in "" _ab/c16/libfftcond_b200.so "" _ab/c16/libfftcond_b200.so; do
  for n in 2048 1024; do
    echo "== 2-D $n lib=${lib:-default}" >> gpurun_out/rows3_k.txt
    FFTC_LIB=$lib python scripts/scheme_kernels.py $n >> gpurun_out/rows3_k.txt 2>&1
  done
done
for lib in "" _ab/c16/libfftcond_b200.so; do
  echo "== 3-D 512 lib=${lib:-default}" >> gpurun_out/rows3_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 em >> gpurun_out/rows3_k.txt 2>&1
done
cat gpurun_out/rows3_k.txt
FFTC_LIB=_ab/c16/libfftcond_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/rows3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rows3_tests.log
tail -3 gpurun_out/rows3_tests.log
