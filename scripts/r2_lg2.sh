# line-group column passes: L2 prefetch (FFTC_COL3_PF) and A/B tile alternation (FFTC_COL3_ALT), A/B
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "3d or lean or config" > gpurun_out/lg2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lg2_tests.log
tail -3 gpurun_out/lg2_tests.log
rm -f gpurun_out/lg2_k3d.txt
for lib in "" _ab/nopf/libfftcond_b200.so _ab/noalt/libfftcond_b200.so _ab/noboth/libfftcond_b200.so ""; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/lg2_k3d.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 basic,em_sub >> gpurun_out/lg2_k3d.txt 2>&1
done
for lib in "" _ab/noboth/libfftcond_b200.so; do
  echo "== n=1024 lib=${lib:-default}" >> gpurun_out/lg2_k3d.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 1024 basic >> gpurun_out/lg2_k3d.txt 2>&1
done
cat gpurun_out/lg2_k3d.txt
