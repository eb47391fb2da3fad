# slab path at world 1 (this rank its own peer; fused transposes as bulk copies) against the monolithic solve
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_slab_mp.py -m gpu -q > gpurun_out/slab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/slab_tests.log
rm -f gpurun_out/slab_w1.txt
python scripts/slab_w1.py 512 basic 20 >> gpurun_out/slab_w1.txt 2>&1
python scripts/slab_w1.py 512 em_sub 20 monolithic,slab-w1-fused >> gpurun_out/slab_w1.txt 2>&1
python scripts/slab_w1.py 1024 basic 8 monolithic >> gpurun_out/slab_w1.txt 2>&1
python scripts/slab_w1.py 1024 basic 8 slab-w1-fused >> gpurun_out/slab_w1.txt 2>&1
tail -n 3 gpurun_out/slab_tests.log; cat gpurun_out/slab_w1.txt
timeout 600 python bench.py --workload c2 --impl reference > gpurun_out/bench_c2_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c2_ref.log; tail -c 600 gpurun_out/bench_c2_ref.log
