# launch list of one c3 pass + full capture of the CTA-pair affine GEMM (the dominant kernel) at the final state
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/r2j_launches_c3.csv python tools/prof_pass.py --config c3 --sentences 64 --passes 1 \
  > /dev/null 2>&1; echo list=$?
python tools/launch_list.py gpurun_out/r2j_launches_c3.csv > gpurun_out/r2j_launches_c3.txt
mkdir -p /tmp/reps
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:lam_gemm_kernel<.int.256, .int.3, .int.2, .bool.1' \
  --launch-skip 3 -c 1 -o /tmp/reps/pair python tools/prof_pass.py --config c3 --sentences 64 --passes 1 > /dev/null 2>&1; echo full=$?
ncu -i /tmp/reps/pair.ncu-rep --page raw --csv > gpurun_out/r2j_full_pair.raw.csv 2>/dev/null
rm -f gpurun_out/r2j_launches_c3.csv
