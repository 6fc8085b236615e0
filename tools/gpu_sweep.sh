# Scratch GPU check used between kernel changes (run through gpurun): GPU parity, then
# per-kernel-class timings of the MRF normal / forward and the stress forward (tools/op_breakdown.py).
python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
python tools/op_breakdown.py --op normal --reps 10 2>&1 | tail -1
MRF_LANES=1 python tools/op_breakdown.py --op forward --reps 10 2>&1 | tail -1
python tools/op_breakdown.py --workload stress --op forward --reps 2 2>&1 | tail -1
