# launch list of one c3 batched pass (+ one eager profiled pass) and full captures of the top kernels;
# the full captures are exported to raw CSV on the box (the reports themselves exceed gpurun's copy-back)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/r2h_launches_c3.csv python tools/prof_pass.py --config c3 --sentences 64 --passes 1 \
  > gpurun_out/r2h_launches.log 2>&1; echo list=$?
mkdir -p /tmp/reps
for spec in "affine:lam_gemm_kernel<.int.256, .int.2:3" "xside:lam_gemm_kernel<.int.128, .int.4, .int.6:3" \
            "yside:lam_gemm_kernel<.int.64, .int.4, .int.6:3" "softmax:softmax4_kernel:1" "verify:elementwise_verify_kernel:1" \
            "concretize:concretize_kernel:1" "bias:affine_bias_kernel:4"; do
  tag=${spec%%:*}; rest=${spec#*:}; kre=${rest%:*}; skip=${rest##*:}
  timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:$kre" \
    --launch-skip $skip -c 1 -o /tmp/reps/r2h_full_$tag python tools/prof_pass.py --config c3 --sentences 64 --passes 1 \
    > gpurun_out/r2h_full_$tag.log 2>&1; echo $tag=$?
  ncu -i /tmp/reps/r2h_full_$tag.ncu-rep --page raw --csv > gpurun_out/r2h_full_$tag.raw.csv 2>/dev/null
  ncu -i /tmp/reps/r2h_full_$tag.ncu-rep --page details --csv > gpurun_out/r2h_full_$tag.details.csv 2>/dev/null
done
du -sh gpurun_out
