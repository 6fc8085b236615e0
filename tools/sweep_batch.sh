for BF in 0 24 32 48 64; do
for LN in 2 3 4; do
MRF_LANES=$LN python tools/op_breakdown.py --op normal --reps 10 --bf $BF 2>&1 | tail -1 | sed "s/^/bf=$BF lanes=$LN /"
done; done
MRF_NO_PERM=1 python tools/op_breakdown.py --op normal --reps 10 2>&1 | tail -1 | sed "s/^/noperm /"
python tools/op_breakdown.py --op normal --reps 10 2>&1 | tail -1 | sed "s/^/perm /"
python tools/op_breakdown.py --op normal --normal toeplitz --reps 10 2>&1 | tail -1 | sed "s/^/toep perm /"
MRF_NO_PERM=1 python tools/op_breakdown.py --op normal --normal toeplitz --reps 10 2>&1 | tail -1 | sed "s/^/toep noperm /"
