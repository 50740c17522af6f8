# same-box A/B of pass sites: default engine vs CTA pairs vs BN=128 affine tiles (c3, 64 sentences)
for i in 1 2; do
  for v in "" "FG_2CTA=1" "FG_AFFINE_BN=128"; do
    echo "== variant [$v] round $i"
    env $v timeout 300 python tools/prof_pass.py --config c3 --sentences 64 --passes 2 | grep sites
  done
done
# one full ncu capture of an affine GEMM launch (BN = 256) and one of the CTA-pair variant
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:lam_gemm_kernel<256, 2, 2' --launch-skip 3 -c 1 -o gpurun_out/r2f_affine_full \
  python tools/prof_pass.py --config c3 --sentences 64 --passes 1 > gpurun_out/r2f_affine_full.log 2>&1
FG_2CTA=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:lam_gemm_kernel<256, 3, 2' --launch-skip 3 -c 1 -o gpurun_out/r2f_affine_pair_full \
  python tools/prof_pass.py --config c3 --sentences 64 --passes 1 > gpurun_out/r2f_affine_pair_full.log 2>&1
echo done
