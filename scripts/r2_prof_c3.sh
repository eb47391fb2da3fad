# ncu --set full of the three 3-D column passes of one C3 iteration (after the
# same command has run clean without ncu), condensed into profiles/r2_ncu_c3.json
FFTC_NO_GRAPH=1 python scripts/prof_3d_one.py --n 512 --iters 3 > gpurun_out/plain.log 2>&1 || { tail -5 gpurun_out/plain.log; exit 1; }
FFTC_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_col3 -s 3 -c 3 -f -o gpurun_out/r2_c3_col3 python scripts/prof_3d_one.py --n 512 --iters 3 > gpurun_out/ncu_c3.log 2>&1
tail -3 gpurun_out/ncu_c3.log
python scripts/ncu_to_json.py gpurun_out/r2_c3_col3.ncu-rep gpurun_out/r2_ncu_c3.json "ncu --set full, C3 512^3 em_sub, the 3 column-pass launches of iteration 2 (scripts/prof_3d_one.py, FFTC_NO_GRAPH=1), line-group y passes and the three-component z pass (cols3_lg.cuh)" "y_fwd_3d=k_col3_lg<2" "sweep2_cols_gamma=k_col3_mid<1" "y_inv_3d=k_col3_lg<3" | tail -40
FFTC_NO_GRAPH=1 ncu --set full --clock-control none -k regex:k_rows_tma -s 2 -c 2 -f -o gpurun_out/r2_c3_rows python scripts/prof_3d_one.py --n 512 --iters 3 > gpurun_out/ncu_c3_rows.log 2>&1
python scripts/ncu_to_json.py gpurun_out/r2_c3_rows.ncu-rep gpurun_out/r2_ncu_c3_rows.json "ncu --set full, C3 512^3 em_sub, row sweeps of iteration 2" "sweep1_rows_fwd=k_rows_tma<3, 1" "sweep3_rows_inv=k_rows_tma<3, 3" | tail -30
