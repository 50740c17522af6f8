timeout 600 python -m pytest tests/test_gpu_pass.py -x -q 2>&1 | tail -n 2
python tools/ab_sites.py ab/base.so ab/new.so --rounds 5
