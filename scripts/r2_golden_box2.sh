# box host: the C5 points p230..p255 at 1024^2 from the unmodified reference (three generator
# processes, own output directories); the GPU meanwhile re-runs the determinism stress scripts
for tag in p23 p24 p25; do
  mkdir -p gpurun_out/golden_$tag; cp tests/golden/c5full.json gpurun_out/golden_$tag/c5full.json
  ( FFTC_GOLDEN_DIR=gpurun_out/golden_$tag FFTC_REF_SRC=baseline/_ref PYTHONDONTWRITEBYTECODE=1 OMP_NUM_THREADS=1 timeout 3300 \
      python oracle/gen_golden.py c5full --jobs 5 --only c5_1024_$tag > gpurun_out/c5full_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/c5full_$tag.log ) &
done
timeout 1500 python scripts/stress_determinism.py --reps 4 --groups c2small,c5full,3d,general,big > gpurun_out/stress2d.txt 2>&1
timeout 900 python scripts/stress_3d_tma.py 8 > gpurun_out/stress3d.txt 2>&1
wait
for f in gpurun_out/stress2d.txt gpurun_out/stress3d.txt gpurun_out/c5full_p2*.log; do tail -n 2 $f; done; true
