# round-end check after the 1024-line y tiles: slab tests (peer output on single-component tiles), GPU suite, C4 and default bench
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_slab_mp.py -m gpu -q > gpurun_out/slab_tests.log 2>&1; echo rc=$? >> gpurun_out/slab_tests.log; tail -n 3 gpurun_out/slab_tests.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log; tail -n 3 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log; tail -n 2 gpurun_out/smoke.log
timeout 1500 python bench.py --workload c4 > gpurun_out/bench_c4.log 2>&1; echo rc=$? >> gpurun_out/bench_c4.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
timeout 1800 python bench.py --workload c4-emsub > gpurun_out/bench_c4-emsub.log 2>&1; echo rc=$? >> gpurun_out/bench_c4-emsub.log
tail -c 300 gpurun_out/bench_c4.log; tail -c 300 gpurun_out/bench_c3.log; tail -c 200 gpurun_out/bench_c4-emsub.log
