timeout 600 python -m pytest tests/test_gpu_pass.py tests/test_gpu_shard.py -q -x 2>&1 | tail -1
timeout 300 python tools/dbg_batch.py 2>&1 | grep repeat
for i in 1 2; do for o in 0 1; do echo "no_onehot=$o"; FG_NO_ONEHOT=$o timeout 300 python tools/prof_pass.py --passes 2 | grep sites; done; done
