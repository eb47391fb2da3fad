python scripts/e2e_c3.py 512 > gpurun_out/e2e_c3.txt 2>&1
FFTC_NO_GRAPH=1 python scripts/prof_3d_one.py --n 512 --iters 2 > gpurun_out/plain.log 2>&1 && FFTC_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_col3_tma -s 2 -c 3 -o gpurun_out/r2_c3_col3 python scripts/prof_3d_one.py --n 512 --iters 2 > gpurun_out/ncu_c3.log 2>&1
cat gpurun_out/e2e_c3.txt; tail -3 gpurun_out/ncu_c3.log
