# TMEM-operand affine engine: umma + pass parity tests, then same-box A/B against FG_AFFINE_TMEM_A=0
timeout 300 python -m pytest tests/test_gpu_umma.py -x -q 2>&1 | tail -n 15
timeout 600 python -m pytest tests/test_gpu_pass.py -x -q 2>&1 | tail -n 5
for i in 1 2 3; do
  for v in "FG_AFFINE_TMEM_A=0" "FG_AFFINE_TMEM_A=1"; do
    echo "== [$v] round $i"
    env $v timeout 300 python tools/prof_pass.py --config c3 --sentences 64 --passes 2 | grep sites
  done
done
