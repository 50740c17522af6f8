# bench lines at HEAD: c3 decision-exact vs raw f32 verdicts (cost of the exact re-decisions), c2, c1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2h_bench_c3.json 2>/dev/null; echo c3=$?
timeout 600 python bench.py --no-cpu-baseline --raw-f32-verdicts > gpurun_out/r2h_bench_c3_raw.json 2>/dev/null; echo raw=$?
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2h_bench_c2.json 2>/dev/null; echo c2=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r2h_bench_c1.json 2>/dev/null; echo c1=$?
