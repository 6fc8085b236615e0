# experiment knobs A/B on the current build
for i in 1 2; do
  python tools/ab_step.py | sed 's/^/default /'
  MRF_ADJ_CTAS=2 python tools/ab_step.py | sed 's/^/adj_ctas2 /'
  MRF_FWD_CTAS=1 python tools/ab_step.py | sed 's/^/fwd_ctas1 /'
  MRF_PDL=0 python tools/ab_step.py | sed 's/^/pdl0 /'
done
