python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cg or CG" 2>&1 | tail -2
python tools/op_breakdown.py --op cg --reps 3 2>&1 | tail -1
python tools/op_breakdown.py --workload sense --op cg --reps 1 2>&1 | tail -1
