python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for op in normal adjoint; do python tools/op_breakdown.py --op $op --reps 10 2>&1 | tail -1; done
MRF_LANES=1 python tools/op_breakdown.py --op normal --reps 10 2>&1 | tail -1
