# Co-residency of the forward row kernel (HBM-bound in CG) beside the forward column kernel of the
# other lane: cap the column kernel at one CTA per SM (113 KB) so a row CTA (104 KB) fits next to it.
run() { echo -n "$* :: "; env "$@" python tools/ab_step.py; }
run MRF_LANES=2
run MRF_GCAP_FC=148
run MRF_GCAP_FC=148 MRF_GCAP_FR=148
run MRF_GCAP_FC=148 MRF_GCAP_FR=148 MRF_LANES=3 MRF_BF=84
run MRF_GCAP_FC=148 MRF_GCAP_FR=148 MRF_LANES=4 MRF_BF=64
run MRF_GCAP_FC=222 MRF_GCAP_FR=148
run MRF_GCAP_FC=148 MRF_GCAP_FR=296 MRF_LANES=4 MRF_BF=64
run MRF_GCAP_FR=148
