# box-host golden generation (CPU only): C4 first iterations at 1024^3, then
# the C5 points at 1024^2 not yet in tests/golden/c5full.json, from the
# unmodified reference under baseline/_ref.  Fixed GPU tests first.
mkdir -p gpurun_out/golden
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_refsuite.py -m gpu -q > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
nproc > gpurun_out/box_host.txt; free -g >> gpurun_out/box_host.txt
bash scripts/r2_c4first.sh
cp tests/golden/c5full.json gpurun_out/golden/c5full.json
FFTC_GOLDEN_DIR=gpurun_out/golden FFTC_REF_SRC=baseline/_ref PYTHONDONTWRITEBYTECODE=1 OMP_NUM_THREADS=1 timeout 3000 \
  python oracle/gen_golden.py c5full --jobs $(nproc) > gpurun_out/c5full.log 2>&1; echo "rc=$?" >> gpurun_out/c5full.log
tail -5 gpurun_out/g_tests.log; tail -3 gpurun_out/c4first.log; tail -3 gpurun_out/c5full.log
