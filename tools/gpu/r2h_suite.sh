# full GPU suite + smoke at HEAD, then a same-box A/B of the pass sites against ab/base.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_gpu_tests.log 2>&1; echo tests=$?
tail -n 3 gpurun_out/r2h_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo smoke=$?
python tools/ab_sites.py ab/base.so ab/new.so --rounds 4
