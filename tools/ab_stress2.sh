# stress / SENSE / MRF normal: windows (default) vs the L2 path for oversized spread chunks (MRF_DBG=4)
for i in 1 2; do
for w in stress sense mrf; do
  python tools/op_breakdown.py --workload $w --op normal --reps 3 --frames 256 2>&1 | tail -1 | sed "s/^/win  /"
  MRF_DBG=4 python tools/op_breakdown.py --workload $w --op normal --reps 3 --frames 256 2>&1 | tail -1 | sed "s/^/l2   /"
done; done
