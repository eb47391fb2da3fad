# final-kernel robustness: determinism stress (bitwise repeats), compute-sanitizer memcheck and racecheck on a 256^3 solve
timeout 1500 python scripts/stress_determinism.py --reps 4 --groups c2small,c5full,3d,general,big > gpurun_out/stress2d.txt 2>&1; tail -n 3 gpurun_out/stress2d.txt
timeout 900 python scripts/stress_3d_tma.py 8 > gpurun_out/stress3d.txt 2>&1; tail -n 3 gpurun_out/stress3d.txt
FFTC_NO_GRAPH=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scripts/prof_3d_one.py --n 256 --iters 2 > gpurun_out/memcheck.log 2>&1; tail -n 4 gpurun_out/memcheck.log
FFTC_NO_GRAPH=1 timeout 1500 compute-sanitizer --tool racecheck --print-limit 5 python scripts/prof_3d_one.py --n 256 --iters 1 > gpurun_out/racecheck.log 2>&1; tail -n 6 gpurun_out/racecheck.log
true
