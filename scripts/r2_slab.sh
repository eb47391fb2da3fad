# slab path at world 1: fused transposes as bulk copies (default) vs 16-byte stores (_ab/stg)
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_slab_mp.py -m gpu -q > gpurun_out/slab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/slab_tests.log
python scripts/slab_w1.py 512 basic 20 > gpurun_out/slab_w1.txt 2>&1
python scripts/slab_w1.py 512 em_sub 20 monolithic,slab-w1-fused >> gpurun_out/slab_w1.txt 2>&1
FFTC_LIB=_ab/stg/libfftcond_b200.so python scripts/slab_w1.py 512 basic 20 slab-w1-fused >> gpurun_out/slab_w1.txt 2>&1
python scripts/slab_w1.py 1024 basic 8 monolithic >> gpurun_out/slab_w1.txt 2>&1
python scripts/slab_w1.py 1024 basic 8 slab-w1-fused >> gpurun_out/slab_w1.txt 2>&1
FFTC_LIB=_ab/stg/libfftcond_b200.so python scripts/slab_w1.py 1024 basic 8 slab-w1-fused >> gpurun_out/slab_w1.txt 2>&1
tail -n 3 gpurun_out/slab_tests.log; cat gpurun_out/slab_w1.txt
