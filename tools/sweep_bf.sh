# batch size x lanes sweep of the MRF normal operator (ms per A^H A)
for BF in 0 96 160 192 256; do
for LN in 2 3; do
MRF_LANES=$LN python tools/op_breakdown.py --op normal --reps 10 --bf $BF 2>&1 | tail -1 | sed "s/^/bf=$BF lanes=$LN /"
done; done
