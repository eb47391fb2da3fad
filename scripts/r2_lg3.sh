# z pass with three components per thread (k_col3_mid) vs one (k_col3_lg, _ab/mid1)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_slab.py tests/test_gpu_slab_mp.py -m gpu -q -x > gpurun_out/lg3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lg3_tests.log
tail -3 gpurun_out/lg3_tests.log
rm -f gpurun_out/lg3_k3d.txt
for lib in "" _ab/mid1/libfftcond_b200.so "" _ab/mid1/libfftcond_b200.so; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/lg3_k3d.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 basic,em_sub >> gpurun_out/lg3_k3d.txt 2>&1
done
for lib in "" _ab/mid1/libfftcond_b200.so; do
  echo "== n=256 lib=${lib:-default}" >> gpurun_out/lg3_k3d.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 256 basic,em_sub >> gpurun_out/lg3_k3d.txt 2>&1
  echo "== n=1024 lib=${lib:-default}" >> gpurun_out/lg3_k3d.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 1024 basic >> gpurun_out/lg3_k3d.txt 2>&1
done
cat gpurun_out/lg3_k3d.txt
timeout 600 python scripts/stress_3d_tma.py 4 > gpurun_out/lg3_stress3d.txt 2>&1; tail -2 gpurun_out/lg3_stress3d.txt
