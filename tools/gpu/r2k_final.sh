# round-end sequence at the final state (CTA pairs incl. pairs over rows at D = 128)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_final_gpu_tests.log 2>&1; echo tests=$?
tail -n 2 gpurun_out/r2k_final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_final_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2k_final_bench.json 2> gpurun_out/r2k_final_bench.err; echo bench=$?
timeout 600 python bench.py --no-cpu-baseline --raw-f32-verdicts > gpurun_out/r2k_bench_c3_raw.json 2>/dev/null; echo raw=$?
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2k_bench_c2.json 2>/dev/null; echo c2=$?
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r2k_bench_c4.json 2>/dev/null; echo c4=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2k_final_ref.json 2> gpurun_out/r2k_final_ref.err; echo ref=$?
