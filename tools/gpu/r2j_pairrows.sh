# CTA pairs over batch rows at D = 128 (c2, the eps = 0 workspace): parity, then same-box A/B
timeout 900 python -m pytest tests/test_gpu_pass.py tests/test_gpu_umma.py tests/test_gpu_decisions.py -x -q 2>&1 | tail -n 2
python tools/ab_sites.py ab/base.so ab/new.so --rounds 3 --config c2 --sentences 256
python tools/ab_sites.py ab/base.so ab/new.so --rounds 2
