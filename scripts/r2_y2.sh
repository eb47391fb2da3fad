# why is the y forward pass slower than the y inverse pass?  timing experiments (results wrong)
rm -f gpurun_out/y2_k.txt
python scripts/kernels_3d.py 512 basic >> gpurun_out/y2_k.txt 2>&1
echo "== FFTC_DBG_YFWD2=1: z_parseval_3d = y forward again right after itself" >> gpurun_out/y2_k.txt
FFTC_DBG_YFWD2=1 python scripts/kernels_3d.py 512 basic >> gpurun_out/y2_k.txt 2>&1
echo "== FFTC_DBG_YFWD2=2: z_parseval_3d = the y INVERSE kernel right after y forward" >> gpurun_out/y2_k.txt
FFTC_DBG_YFWD2=2 python scripts/kernels_3d.py 512 basic >> gpurun_out/y2_k.txt 2>&1
cat gpurun_out/y2_k.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/y2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/y2_tests.log
tail -n 3 gpurun_out/y2_tests.log
