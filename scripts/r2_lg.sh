# line-group 3-D column passes (cols3_lg.cuh): parity first, then per-kernel
# timings against the previous kernels (_ab/old) and the same mapping with
# CTA-wide barriers (_ab/ctasync); 256^3 / 512^3 / 1024^3 lines
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_operators.py tests/test_gpu_slab.py tests/test_gpu_slab_mp.py -m gpu -q -x > gpurun_out/lg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lg_tests.log
tail -4 gpurun_out/lg_tests.log
for n in 512 256; do
  for lib in "" _ab/old/libfftcond_b200.so _ab/ctasync/libfftcond_b200.so ""; do
    echo "== n=$n lib=${lib:-default}" >> gpurun_out/lg_k3d.txt
    FFTC_LIB=$lib python scripts/kernels_3d.py $n basic,em_sub >> gpurun_out/lg_k3d.txt 2>&1
  done
done
for lib in "" _ab/old/libfftcond_b200.so; do
  echo "== n=1024 lib=${lib:-default}" >> gpurun_out/lg_k3d.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 1024 basic >> gpurun_out/lg_k3d.txt 2>&1
done
cat gpurun_out/lg_k3d.txt
timeout 600 python scripts/stress_3d_tma.py 4 > gpurun_out/lg_stress3d.txt 2>&1; tail -3 gpurun_out/lg_stress3d.txt
