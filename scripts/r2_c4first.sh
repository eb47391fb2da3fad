# C4 first-iteration golden at the stated size (1024^3, frozen medium, basic)
# from the bounded-memory oracle on the GPU box host (~165 GB of its 196 GB;
# the address-space cap turns an overrun into MemoryError, not an OOM kill)
mkdir -p gpurun_out/golden
( ulimit -v 188000000; FFTC_GOLDEN_DIR=gpurun_out/golden PYTHONDONTWRITEBYTECODE=1 timeout 2400 \
  python oracle/gen_golden.py c4first --jobs 1 > gpurun_out/c4first.log 2>&1 ); echo "rc=$?" >> gpurun_out/c4first.log
tail -3 gpurun_out/c4first.log
