run() { echo -n "$* :: "; env "$@" python tools/ab_step.py; }
run MRF_SPLIT=128
run MRF_SPLIT=96
run MRF_SPLIT=64
run MRF_SPLIT=48
run MRF_SPLIT=32
run MRF_SPLIT=128
