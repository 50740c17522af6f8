set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/r2f_bench_c3.json 2> gpurun_out/r2f_bench_c3.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err; echo ref_rc=$?
