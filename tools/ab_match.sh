# alternate A/B of tools/match_bench.py between named library variants
for i in 1 2; do
  for v in "$@"; do echo "== $v"; MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_$v.so python tools/match_bench.py 2>&1 | tail -4; done
done
