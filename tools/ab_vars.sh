# alternate A/B of named in-tree library variants: bash tools/ab_vars.sh name1 name2 ...
for i in 1 2 3; do
  for v in "$@"; do MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_$v.so python tools/ab_step.py; done
done
