# CG step (split-phase) vs frames per batch and lanes
for BF in 0 64 96 167 200 250; do
for LN in 2 3; do
MRF_BF=$BF MRF_LANES=$LN python tools/ab_step.py | sed "s/^/bf=$BF lanes=$LN /"
done; done
