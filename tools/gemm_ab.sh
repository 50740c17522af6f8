for bn in 256 128; do echo "single bn=$bn:"; FG_AFFINE_BN=$bn timeout 300 python tools/prof_pass.py --passes 2 | grep sites; done
echo "pair bn=256:"; FG_2CTA=1 timeout 300 python tools/prof_pass.py --passes 2 | grep sites
echo "pair bn=128:"; FG_2CTA=1 FG_AFFINE_BN=128 timeout 300 python tools/prof_pass.py --passes 2 | grep sites
