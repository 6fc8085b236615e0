# Scratch GPU check used between kernel changes (run through gpurun).
python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for A in 1 2; do
MRF_ADJ_CTAS=$A python tools/op_breakdown.py --op normal --reps 10 2>&1 | tail -1
MRF_ADJ_CTAS=$A MRF_LANES=1 python tools/op_breakdown.py --op adjoint --reps 10 2>&1 | tail -1
MRF_ADJ_CTAS=$A python tools/op_breakdown.py --workload stress --op adjoint --reps 2 2>&1 | tail -1
done
