python tools/op_breakdown.py --workload stress --op adjoint --reps 2 --frames 400 2>&1 | tail -1
python tools/op_breakdown.py --workload stress --op forward --reps 2 --frames 400 2>&1 | tail -1
python tools/op_breakdown.py --workload sense --op adjoint --reps 3 --frames 400 2>&1 | tail -1
python tools/op_breakdown.py --workload sense --op forward --reps 3 --frames 400 2>&1 | tail -1
ncu --set full --import-source on --clock-control none -k regex:"k_adj_(cols|rows)" --launch-skip 6 --launch-count 2 -o gpurun_out/stress_adj python tools/prof_ops.py --workload stress --frames 28 --reps 2 --ops adj > gpurun_out/stress_ncu.log 2>&1
tail -2 gpurun_out/stress_ncu.log
