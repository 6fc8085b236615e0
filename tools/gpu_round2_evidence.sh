# Round-2 evidence run (through gpurun): the default bench line, the launch list of the same
# command, a full ncu capture of the four gridding kernels (one 128-frame MRF normal), their L2 /
# shared-memory / atomic counters, and the other workloads' bench lines.
# usage: bash tools/gpu_round2_evidence.sh <outdir under gpurun_out>
O=gpurun_out/${1:-r02}
set -x
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-toeplitz --no-match --no-llr --no-pcg --no-fft-stages > $O/launches.csv 2> $O/launches.err
ncu --set full --import-source on --clock-control none -k regex:"k_(fwd|adj)_(rows|cols)" --launch-skip 6 --launch-count 4 -o $O/four python tools/prof_ops.py --workload mrf --frames 128 --reps 2 --ops normal > $O/four.log 2>&1
for w in sense stress cfg2; do
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-llr --no-match --no-toeplitz --no-pcg > $O/bench_$w.json 2> $O/bench_$w.err
done
lscpu > $O/lscpu.txt
tail -c 300 $O/bench.json
