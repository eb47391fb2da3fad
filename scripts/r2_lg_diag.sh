# quick check of the line-group column passes; on failure, compute-sanitizer on one small solve
if ! timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "3d" > gpurun_out/lg_diag_tests.log 2>&1; then
  tail -5 gpurun_out/lg_diag_tests.log
  FFTC_NO_GRAPH=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scripts/prof_3d_one.py --n 256 --iters 1 > gpurun_out/lg_sanitizer.log 2>&1
  grep -m 30 -A12 "=========" gpurun_out/lg_sanitizer.log | head -80
  exit 1
fi
tail -2 gpurun_out/lg_diag_tests.log
rm -f gpurun_out/lg_k3d.txt
bash scripts/r2_lg.sh
