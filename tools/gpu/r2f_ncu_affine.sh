# full ncu captures of one affine GEMM launch (BN = 256): single-CTA engine and CTA-pair variant
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:lam_gemm_kernel<.int.256, .int.2' --launch-skip 3 -c 1 -o gpurun_out/r2f_affine_full \
  python tools/prof_pass.py --config c3 --sentences 64 --passes 1 > gpurun_out/r2f_affine_full.log 2>&1
FG_2CTA=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:lam_gemm_kernel<.int.256, .int.3' --launch-skip 3 -c 1 -o gpurun_out/r2f_affine_pair_full \
  python tools/prof_pass.py --config c3 --sentences 64 --passes 1 > gpurun_out/r2f_affine_pair_full.log 2>&1
ls -la gpurun_out
