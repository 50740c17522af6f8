# default bench line (c3) with the sustained-peak roofline and the full-pass CPU baseline
timeout 900 python bench.py > gpurun_out/r2g_bench_c3.json 2> gpurun_out/r2g_bench_c3.err; echo bench_rc=$?
