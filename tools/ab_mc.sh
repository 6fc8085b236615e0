# alternate A/B of named library variants on the multi-coil workloads (normal operator, 256 frames) and MRF
for i in 1 2; do
for v in "$@"; do
for w in stress sense; do
  MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_$v.so python tools/op_breakdown.py --workload $w --op normal --reps 3 --frames 256 2>&1 | tail -1 | cut -c1-60 | sed "s/^/$v /"
done
MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_$v.so python tools/ab_step.py | sed "s/^/$v /"
done; done
