# c4 / c5 bench lines at the final state (no CPU baseline: hours per reference pass)
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2h_bench_c4.json 2>/dev/null; echo c4=$?
timeout 1200 python bench.py --config c5 --no-cpu-baseline > gpurun_out/r2h_bench_c5.json 2>/dev/null; echo c5=$?
