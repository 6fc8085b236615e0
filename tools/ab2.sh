# A/B of the in-tree build against libmrfnufft_prev.so (the previous commit's build), alternating,
# plus the per-phase cycle counters of the experiment build (libmrfnufft_exp.so, MRF_DBG=2).
# usage: bash tools/ab2.sh [workload]
W=${1:-mrf}
for i in 1 2 3; do
  python tools/ab_step.py
  MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_prev.so python tools/ab_step.py
done
if [ -f paper_2310_05647_b200/libmrfnufft_exp.so ]; then
  MRF_LIB_PATH=$PWD/paper_2310_05647_b200/libmrfnufft_exp.so MRF_DBG=2 python tools/prof_ops.py --workload $W --frames 256 --reps 3 --ops normal 2>&1 | grep phase
fi
