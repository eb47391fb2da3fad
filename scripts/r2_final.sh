# last verification of the round: GPU suite, C4 and default bench lines
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
tail -n 3 gpurun_out/gputests.log
python scripts/kernels_3d.py 1024 basic > gpurun_out/k3d_1024.txt 2>&1; cat gpurun_out/k3d_1024.txt
timeout 1500 python bench.py --workload c4 > gpurun_out/bench_c4.log 2>&1; echo rc=$? >> gpurun_out/bench_c4.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c3_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c3_ref.log
timeout 600 python bench.py --workload c2 --impl reference > gpurun_out/bench_c2_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c2_ref.log
tail -c 300 gpurun_out/bench_c4.log; tail -c 300 gpurun_out/bench_c3.log
