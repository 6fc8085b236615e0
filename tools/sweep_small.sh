# small (L2-resident) batches x lanes for the split CG and the normal operator
for BF in 0 16 24 32 48; do
for LN in 2 3 4; do
MRF_BF=$BF MRF_LANES=$LN python tools/ab_step.py | sed "s/^/bf=$BF lanes=$LN /"
done; done
