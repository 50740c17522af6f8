# CTA-pair GEMM with the shared-memory-restricted cluster release: parity + same-box A/B against one CTA
FG_2CTA=1 timeout 900 python -m pytest tests/test_gpu_umma.py tests/test_gpu_pass.py -x -q 2>&1 | tail -n 2
for i in 1 2 3; do
  for v in 0 1; do echo "== FG_2CTA=$v"; FG_2CTA=$v timeout 300 python tools/prof_pass.py --config c3 --sentences 64 --passes 2 | grep sites; done
done
