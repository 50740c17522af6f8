for i in 1 2; do for r in 42 26 34; do echo "ring64=$r"; FG_RING64=$r timeout 300 python tools/prof_pass.py --passes 2 | grep sites; done; done
