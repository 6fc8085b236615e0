# batch size of the multi-coil workloads (auto: 128 MB of half grid per lane)
for BF in 0 16 32 64; do
python tools/op_breakdown.py --workload stress --op normal --reps 2 --frames 512 --bf $BF 2>&1 | tail -1 | sed "s/^/bf=$BF /"
done
for BF in 0 32 64 128; do
python tools/op_breakdown.py --workload sense --op normal --reps 3 --frames 512 --bf $BF 2>&1 | tail -1 | sed "s/^/bf=$BF /"
done
