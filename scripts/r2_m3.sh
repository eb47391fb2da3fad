rm -f gpurun_out/m3_k.txt
for lib in "" _ab/m3_6/libfftcond_b200.so _ab/m3_10/libfftcond_b200.so "" _ab/m3_6/libfftcond_b200.so _ab/m3_10/libfftcond_b200.so; do
  echo "== n=512 lib=${lib:-default}" >> gpurun_out/m3_k.txt
  FFTC_LIB=$lib python scripts/kernels_3d.py 512 em_sub >> gpurun_out/m3_k.txt 2>&1
done
cat gpurun_out/m3_k.txt
