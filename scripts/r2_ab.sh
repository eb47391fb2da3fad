python scripts/kernels_3d.py 512 basic,em_sub > gpurun_out/ab_k3d.txt 2>&1
FFTC_LIB=_ab/w2/libfftcond_b200.so python scripts/kernels_3d.py 512 basic,em_sub >> gpurun_out/ab_k3d.txt 2>&1
python scripts/kernels_3d.py 512 basic,em_sub >> gpurun_out/ab_k3d.txt 2>&1
FFTC_LIB=_ab/w2/libfftcond_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "3d" >> gpurun_out/ab_k3d.txt 2>&1
cat gpurun_out/ab_k3d.txt | tail -12
