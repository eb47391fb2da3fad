# round-2 verification: new GPU tests, the C4 accelerated arm at 1024^3 (lean
# schedule), small-solve host overhead, then the 1024^3 C4 first-iteration
# golden on the box host (CPU only)
timeout 1800 python -m pytest tests/test_gpu_configs.py tests/test_gpu_refsuite.py tests/test_gpu_sweep.py tests/test_gpu_spectral.py tests/test_gpu_cli.py -m gpu -q -rf > gpurun_out/v_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v_tests.log
timeout 1500 python bench.py --workload c4-emsub --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/v_c4emsub.log 2>&1; echo "c4emsub rc=$?" >> gpurun_out/v_c4emsub.log
timeout 600 python scripts/small_solve_overhead.py > gpurun_out/v_overhead.txt 2>&1
bash scripts/r2_c4first.sh
tail -n 15 gpurun_out/v_tests.log; tail -c 2500 gpurun_out/v_c4emsub.log; cat gpurun_out/v_overhead.txt
