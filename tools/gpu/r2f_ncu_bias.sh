# full ncu capture of one f64 affine bias launch (c3, QKV of layer 2)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:affine_bias_kernel --launch-skip 4 -c 1 \
  -o gpurun_out/r2f_bias_full python tools/prof_pass.py --config c3 --sentences 64 --passes 1 > gpurun_out/r2f_bias_full.log 2>&1
echo rc=$?
