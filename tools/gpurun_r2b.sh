# round 2: compute-sanitizer evidence + ncu launch tables / full captures of the current code
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/r02_sanitize_$t.log 2>&1; echo "$t rc=$?" >> gpurun_out/r02_sanitize_$t.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_bench_launches_v0.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_c4_launches_v0.csv python tools/one_case.py c4 4 1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off -k regex:"k_remap_tile|k_lag_fused|k_post|k_dual|k_node" --set full --clock-control none --import-source on -o gpurun_out/r02_c4_full_v0 python tools/ncu_at.py c4 5 > /dev/null 2>&1
tail -2 gpurun_out/r02_sanitize_*.log
ls -la gpurun_out
