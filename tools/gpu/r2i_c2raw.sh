# c2: decision-exact vs raw f32 verdicts (cost of the exact re-decisions at c2)
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2i_bench_c2b.json 2>/dev/null; echo c2=$?
timeout 600 python bench.py --config c2 --no-cpu-baseline --raw-f32-verdicts > gpurun_out/r2i_bench_c2_raw.json 2>/dev/null; echo raw=$?
