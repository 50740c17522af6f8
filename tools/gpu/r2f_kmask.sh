# activation zero-row mask into W2 (verify skips identity / zero rows): parity tests, then same-box A/B
timeout 900 python -m pytest tests/test_gpu_pass.py tests/test_gpu_decisions.py tests/test_gpu_umma.py -x -q 2>&1 | tail -n 5
python tools/ab_sites.py ab/base.so ab/new.so --rounds 3
