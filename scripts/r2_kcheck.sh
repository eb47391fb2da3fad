# kernel change check: parity suites, 3-D/2-D per-kernel timings, race stress
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_operators.py tests/test_gpu_spectral.py -m gpu -x -q > gpurun_out/kcheck_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/kcheck_tests.log
python scripts/kernels_3d.py 512 basic,em_sub > gpurun_out/kcheck_k3d.txt 2>&1
python scripts/scheme_kernels.py 2048 > gpurun_out/kcheck_k2d.txt 2>&1
python scripts/scheme_kernels.py 1024 >> gpurun_out/kcheck_k2d.txt 2>&1
timeout 600 python scripts/stress_3d_tma.py 6 > gpurun_out/kcheck_stress3d.txt 2>&1
timeout 600 python scripts/stress_determinism.py --reps 4 --groups c2small,c5full > gpurun_out/kcheck_stress2d.txt 2>&1
tail -2 gpurun_out/kcheck_tests.log; cat gpurun_out/kcheck_k3d.txt gpurun_out/kcheck_k2d.txt; tail -3 gpurun_out/kcheck_stress3d.txt gpurun_out/kcheck_stress2d.txt
