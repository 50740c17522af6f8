for i in 1 2; do
for cfg in "0 64" "0 128" "1 64" "1 128" "1 32"; do set -- $cfg; echo "persist=$1 tile=$2"; FG_SM3_PERSIST=$1 FG_SM3_TILE_KB=$2 timeout 120 python tools/prof_pass.py --passes 1 2>&1 | grep sites | sed 's/.*softmax/softmax/' | cut -c1-22; done
done
