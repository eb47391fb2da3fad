# ncu --set full of the 3-D column passes of one C4 iteration (1024^3 basic, frozen medium)
FFTC_NO_GRAPH=1 python scripts/prof_3d_one.py --n 1024 --scheme basic --workload c4 --iters 3 > gpurun_out/plain_c4.log 2>&1 || { tail -5 gpurun_out/plain_c4.log; exit 1; }
FFTC_NO_GRAPH=1 ncu --set full --clock-control none -k regex:k_col3 -s 3 -c 3 -f -o gpurun_out/r2_c4_col3 python scripts/prof_3d_one.py --n 1024 --scheme basic --workload c4 --iters 3 > gpurun_out/ncu_c4.log 2>&1
tail -n 3 gpurun_out/ncu_c4.log
python scripts/ncu_summary.py gpurun_out/r2_c4_col3.ncu-rep > gpurun_out/r2_ncu_full_c4.txt 2>&1; cat gpurun_out/r2_ncu_full_c4.txt
