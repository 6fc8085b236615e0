# Spatial multiplexing sweep: small L2-resident frame batches on several lanes, each kernel's grid
# capped (MRF_GCAP_*) so kernels of different lanes run side by side on disjoint SMs.
# usage: bash tools/sweep_spatial.sh   (prints one ab_step line per setting)
run() { echo -n "$* :: "; env "$@" python tools/ab_step.py; }
run MRF_LANES=2
run MRF_LANES=4 MRF_BF=32
run MRF_LANES=4 MRF_BF=32 MRF_GCAP_FR=120 MRF_GCAP_FC=100 MRF_GCAP_AC=60 MRF_GCAP_AR=80
run MRF_LANES=4 MRF_BF=16 MRF_GCAP_FR=120 MRF_GCAP_FC=100 MRF_GCAP_AC=60 MRF_GCAP_AR=80
run MRF_LANES=6 MRF_BF=16 MRF_GCAP_FR=90 MRF_GCAP_FC=80 MRF_GCAP_AC=50 MRF_GCAP_AR=60
run MRF_LANES=8 MRF_BF=16 MRF_GCAP_FR=90 MRF_GCAP_FC=80 MRF_GCAP_AC=50 MRF_GCAP_AR=60
run MRF_LANES=8 MRF_BF=8 MRF_GCAP_FR=90 MRF_GCAP_FC=80 MRF_GCAP_AC=50 MRF_GCAP_AR=60
run MRF_LANES=4 MRF_BF=32 MRF_GCAP_AC=74 MRF_GCAP_FC=148
run MRF_LANES=4 MRF_BF=64 MRF_GCAP_AC=74 MRF_GCAP_FC=148
run MRF_LANES=3 MRF_BF=64
run MRF_LANES=4 MRF_BF=64
run MRF_LANES=8 MRF_BF=16
