# plain y passes with three components per thread (_ab/y3c) vs one (default)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "3d or config or lean" > gpurun_out/y3c_tests_default.log 2>&1; echo rc=$? >> gpurun_out/y3c_tests_default.log; tail -n 2 gpurun_out/y3c_tests_default.log
FFTC_LIB=_ab/y3c/libfftcond_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_slab.py -m gpu -q -x > gpurun_out/y3c_tests.log 2>&1; echo rc=$? >> gpurun_out/y3c_tests.log; tail -n 2 gpurun_out/y3c_tests.log
rm -f gpurun_out/y3c_k.txt
for lib in "" _ab/y3c/libfftcond_b200.so "" _ab/y3c/libfftcond_b200.so; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/y3c_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 basic,em_sub >> gpurun_out/y3c_k.txt 2>&1
done
for lib in "" _ab/y3c/libfftcond_b200.so; do
  echo "== n=1024 lib=${lib:-default}" >> gpurun_out/y3c_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 1024 basic >> gpurun_out/y3c_k.txt 2>&1
  echo "== n=256 lib=${lib:-default}" >> gpurun_out/y3c_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 256 basic,em_sub >> gpurun_out/y3c_k.txt 2>&1
done
cat gpurun_out/y3c_k.txt
