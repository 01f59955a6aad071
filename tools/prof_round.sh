set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
timeout 300 python bench.py > gpurun_out/r01_bench_c2_v8.json 2> gpurun_out/b2.err
timeout 300 python bench.py --impl reference > gpurun_out/r01_bench_ref_c2_v8.json 2> gpurun_out/br.err
timeout 300 python bench.py --workload c1 > gpurun_out/r01_bench_c1_v8.json 2> gpurun_out/b1.err
timeout 400 python bench.py --workload c3 > gpurun_out/r01_bench_c3_v8.json 2> gpurun_out/b3.err
timeout 500 python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/r01_bench_c4_v8.json 2> gpurun_out/b4.err
timeout 500 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/r01_bench_c5_v8.json 2> gpurun_out/b5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_bench_launches_v8.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r01_c2_launches_v8.csv python tools/one_case.py c2 12 2 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r01_c4_launches_v8.csv python tools/one_case.py c4 4 1 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r01_c5_launches_v8.csv python tools/one_case.py c5 3 1 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off -k regex:"k_lag_fused|k_post|k_remap_tile" --set full --clock-control none --import-source on -o gpurun_out/r01_c2_full_v8 python tools/ncu_at.py c2 5 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off -k regex:"k_remap_tile|k_lag_fused|k_post" --set full --clock-control none --import-source on -o gpurun_out/r01_c4_full_v8 python tools/ncu_at.py c4 5 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off -k regex:"k_remap_tile|k_slivers" --set full --clock-control none --import-source on -o gpurun_out/r01_c5_full_v8 python tools/ncu_at.py c5 3 > /dev/null 2>&1
timeout 300 python bench.py --remap direct --no-cpu-baseline > gpurun_out/r01_bench_c2_direct_v8.json 2>/dev/null
timeout 300 python bench.py --remap ad --no-cpu-baseline > gpurun_out/r01_bench_c2_ad_v8.json 2>/dev/null
ls -la gpurun_out/
