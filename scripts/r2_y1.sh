# y passes on single-component 8-column tiles with three slots (default) vs the vector tiles (_ab/y3);
# and the timing experiment FFTC_DBG_YFWD2 (y forward twice in a row; results wrong, timing only)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_slab.py tests/test_gpu_slab_mp.py -m gpu -q -x > gpurun_out/y1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/y1_tests.log
tail -3 gpurun_out/y1_tests.log
rm -f gpurun_out/y1_k.txt
for lib in "" _ab/y3/libfftcond_b200.so "" _ab/y3/libfftcond_b200.so; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/y1_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 basic,em_sub >> gpurun_out/y1_k.txt 2>&1
done
for lib in "" _ab/y3/libfftcond_b200.so; do
  echo "== n=256 lib=${lib:-default}" >> gpurun_out/y1_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 256 basic,em_sub >> gpurun_out/y1_k.txt 2>&1
done
echo "== n=512 default, FFTC_DBG_YFWD2 (z_parseval_3d = the y forward pass run again right after itself)" >> gpurun_out/y1_k.txt
FFTC_DBG_YFWD2=1 python scripts/kernels_3d.py 512 basic >> gpurun_out/y1_k.txt 2>&1
echo "== n=512 _ab/y3, FFTC_DBG_YFWD2" >> gpurun_out/y1_k.txt
FFTC_DBG_YFWD2=1 FFTC_LIB=_ab/y3/libfftcond_b200.so python scripts/kernels_3d.py 512 basic >> gpurun_out/y1_k.txt 2>&1
cat gpurun_out/y1_k.txt
timeout 600 python scripts/stress_3d_tma.py 4 > gpurun_out/y1_stress3d.txt 2>&1; tail -2 gpurun_out/y1_stress3d.txt
