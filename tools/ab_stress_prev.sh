# stress / sense timings of the in-tree build against libmrfnufft_prev.so, then the MRF A/B
for lib in libmrfnufft.so libmrfnufft_prev.so; do
  for w in stress sense; do
    MRF_LIB_PATH=$PWD/paper_2310_05647_b200/$lib python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-match --no-llr --no-pcg --no-toeplitz --no-fft-stages | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $w', d['ms_per_step'], d['ms_per_AHA'], d['ms_per_forward'], d['ms_per_adjoint'])"
  done
done
bash tools/ab2.sh 2>&1 | grep -v phase
