# round-end sequence at HEAD (after the DMMA bias): GPU suite, smoke, default bench, reference arm
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_final_gpu_tests.log 2>&1; echo tests=$?
tail -n 2 gpurun_out/r2i_final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_final_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2i_final_bench.json 2> gpurun_out/r2i_final_bench.err; echo bench=$?
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2i_bench_c2.json 2>/dev/null; echo c2=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2i_final_ref.json 2> gpurun_out/r2i_final_ref.err; echo ref=$?
