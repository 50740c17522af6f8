# McCormick GEMMs: tensor-memory operand (default) vs shared-memory operand, which now runs as CTA pairs
FG_DOTS_TMEM_A=0 timeout 600 python -m pytest tests/test_gpu_pass.py -x -q 2>&1 | tail -n 1
for i in 1 2 3; do for v in 1 0; do echo "== FG_DOTS_TMEM_A=$v"; FG_DOTS_TMEM_A=$v timeout 300 python tools/prof_pass.py --config c3 --sentences 64 --passes 2 | grep sites; done; done
