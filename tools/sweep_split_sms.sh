# Column kernels capped below the SM count so the (HBM-bound) row kernels of another lane always
# find free SMs; default batch size, 2-4 lanes.
run() { echo -n "$* :: "; env "$@" python tools/ab_step.py; }
run MRF_LANES=2
run MRF_GCAP_AC=128 MRF_GCAP_FC=256
run MRF_GCAP_AC=128 MRF_GCAP_FC=256 MRF_LANES=3 MRF_BF=112
run MRF_GCAP_AC=128 MRF_GCAP_FC=256 MRF_LANES=4 MRF_BF=84
run MRF_GCAP_AC=116 MRF_GCAP_FC=232 MRF_LANES=3 MRF_BF=112
run MRF_GCAP_AC=116 MRF_GCAP_FC=232 MRF_LANES=4 MRF_BF=84
run MRF_GCAP_AC=136 MRF_GCAP_FC=272 MRF_LANES=3 MRF_BF=112
run MRF_LANES=3 MRF_BF=112
