timeout 1200 python bench.py --config c5 --no-cpu-baseline > gpurun_out/r2j_bench_c5.json 2>/dev/null; echo c5=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2j_bench_c1.json 2>/dev/null; echo c1=$?
