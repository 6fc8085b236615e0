# Round-2 evidence run (through gpurun): the default bench line, the launch list of the same
# command, per-kernel L2 hit rate / shared-memory / atomic counters of the four gridding kernels
# (one 256-frame MRF batch of each), and the other workloads' bench lines.
set -x
mkdir -p gpurun_out/r02
python bench.py > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-toeplitz --no-match --no-llr --no-pcg > gpurun_out/r02/launches.csv 2> gpurun_out/r02/launches.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum"
ncu --metrics $M --clock-control none -k regex:"k_(fwd|adj)_(rows|cols)" --launch-skip 8 --launch-count 8 --csv python tools/prof_ops.py --workload mrf --frames 256 --reps 2 --ops normal > gpurun_out/r02/l2_atom.csv 2> gpurun_out/r02/l2_atom.err
ncu --set full --import-source on --clock-control none -k regex:"k_adj_cols" --launch-skip 4 --launch-count 1 -o gpurun_out/r02/adj_cols python tools/prof_ops.py --workload mrf --frames 256 --reps 2 --ops normal > gpurun_out/r02/adj_full.log 2>&1
for w in sense stress cfg2; do
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-llr --no-match --no-toeplitz --no-pcg > gpurun_out/r02/bench_$w.json 2> gpurun_out/r02/bench_$w.err
done
lscpu > gpurun_out/r02/lscpu.txt
tail -c 400 gpurun_out/r02/bench.json
