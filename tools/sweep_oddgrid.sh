# Column-kernel grids coprime with the S = 32 strips of a frame, so a CTA's static round-robin walks
# every strip (the strips near DC carry 5-10x the gather / spread work of the others).
run() { echo -n "$* :: "; env "$@" python tools/ab_step.py; }
run MRF_LANES=2
run MRF_GCAP_AC=147
run MRF_GCAP_AC=147 MRF_GCAP_FC=295
run MRF_GCAP_AC=145 MRF_GCAP_FC=293
run MRF_GCAP_FC=295
run MRF_LANES=2
run MRF_GCAP_AC=147 MRF_GCAP_FC=295
