# round-end check: smoke, the GPU suite (with the full C3 fixture), default bench and its reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo rc=$? >> gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c3_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c3_ref.log
tail -n 2 gpurun_out/smoke.log; tail -n 3 gpurun_out/gputests.log; tail -c 400 gpurun_out/bench_c3.log
