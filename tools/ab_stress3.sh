# stress (and MRF) timings of the in-tree build for MRF_ADJ_T2 = 0 / 1
for t in 0 1; do
  MRF_ADJ_T2=$t python bench.py --workload stress --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-match --no-llr --no-pcg --no-toeplitz --no-fft-stages | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stress t2=$t', d['ms_per_step'], d['ms_per_AHA'], d['ms_per_forward'], d['ms_per_adjoint'])"
done
python tools/ab_step.py
