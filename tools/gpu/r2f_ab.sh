# parity tests of the engine paths, then a same-box A/B of pass sites: ab/base.so (HEAD) vs ab/new.so
timeout 900 python -m pytest tests/test_gpu_pass.py tests/test_gpu_decisions.py tests/test_gpu_umma.py tests/test_gpu_ops.py -x -q 2>&1 | tail -n 5
python tools/ab_sites.py ab/base.so ab/new.so --rounds 3
python tools/ab_sites.py ab/base.so ab/new.so --rounds 2 --config c2 --sentences 256
