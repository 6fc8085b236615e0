# A/B of the split-phase CG (default) against MRF_CG_SPLIT=0 and the previous commit's build
for i in 1 2; do
  python tools/ab_step.py
  MRF_CG_SPLIT=0 python tools/ab_step.py
  MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_prev.so python tools/ab_step.py
done
