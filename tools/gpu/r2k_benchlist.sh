# ncu launch list of the bench command itself (first 1500 launches: warm-up steps of the c3 search)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 \
  --csv --log-file gpurun_out/r2k_bench_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile \
  > gpurun_out/r2k_bench_launches.log 2>&1; echo rc=$?
python tools/launch_list.py gpurun_out/r2k_bench_launches_c3.csv > gpurun_out/r2k_bench_launches_c3.txt; head -30 gpurun_out/r2k_bench_launches_c3.txt
rm -f gpurun_out/r2k_bench_launches_c3.csv
