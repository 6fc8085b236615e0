for i in 1 2 3; do
python tools/ab_step.py
MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_r1.so python tools/ab_step.py
done
