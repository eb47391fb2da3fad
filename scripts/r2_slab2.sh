# slab world 1 vs monolithic, per-kernel device time (512^3 basic)
SLAB_STATS=1 python scripts/slab_w1.py 512 basic 10 monolithic,slab-w1-fused > gpurun_out/slab_stats.txt 2>&1
cat gpurun_out/slab_stats.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py -m gpu -q -k "c5" > gpurun_out/c5_tests.log 2>&1; echo rc=$? >> gpurun_out/c5_tests.log; tail -n 3 gpurun_out/c5_tests.log
