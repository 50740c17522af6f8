for i in 1 2; do timeout 300 python tools/prof_pass.py --passes 2 | grep sites; done
