# y passes at 1024 on single-component 4-column tiles (default) vs the 2-column vector tiles (_ab/y1k0)
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "first" > gpurun_out/y1k_tests.log 2>&1; echo rc=$? >> gpurun_out/y1k_tests.log; tail -n 2 gpurun_out/y1k_tests.log
rm -f gpurun_out/y1k_k.txt
for lib in "" _ab/y1k0/libfftcond_b200.so "" _ab/y1k0/libfftcond_b200.so; do
  echo "== n=1024 lib=${lib:-default}" >> gpurun_out/y1k_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 1024 basic >> gpurun_out/y1k_k.txt 2>&1
done
cat gpurun_out/y1k_k.txt
timeout 600 python scripts/stress_3d_tma.py 4 > gpurun_out/y1k_stress.txt 2>&1; tail -n 2 gpurun_out/y1k_stress.txt
