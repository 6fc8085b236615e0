set -x
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --kernel-name-exclude regex:at:: --print-limit 50 python tools/sanitize_driver.py all > gpurun_out/san/$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$t.log >> gpurun_out/san/summary.txt
done
M="lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_(fwd|adj)_(rows|cols)" --launch-skip 16 --launch-count 8 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-toeplitz --no-match --no-llr --no-cpu-baseline > gpurun_out/ncu_l2.csv 2> gpurun_out/ncu_l2.err
echo ncu rc=$? >> gpurun_out/san/summary.txt
lscpu > gpurun_out/lscpu.txt
cat gpurun_out/san/summary.txt
