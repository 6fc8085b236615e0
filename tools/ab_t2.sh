python tools/t2_check.py
for i in 1 2; do
  MRF_ADJ_T2=0 python tools/ab_step.py | sed 's/^/t2=0 /'
  MRF_ADJ_T2=1 python tools/ab_step.py | sed 's/^/t2=1 /'
done
MRF_ADJ_T2=0 python bench.py --workload stress --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stress t2=0', d['ms_per_AHA'], d['ms_per_adjoint'], d['ms_per_step'])"
MRF_ADJ_T2=1 python bench.py --workload stress --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stress t2=1', d['ms_per_AHA'], d['ms_per_adjoint'], d['ms_per_step'])"
