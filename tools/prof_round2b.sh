# round-2 final measurement set (run from the repo root on the GPU box via gpurun); V names the set
cd $GRAFT_REPO_ROOT
V=${V:-v2}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem,memory.total --format=csv > gpurun_out/r02_box_$V.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_c4_$V.json 2> gpurun_out/b4.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref_c4_$V.json 2> gpurun_out/br.err
timeout 300 python bench.py --workload c1 > gpurun_out/r02_bench_c1_$V.json 2> gpurun_out/b1.err
timeout 300 python bench.py --workload c2 > gpurun_out/r02_bench_c2_$V.json 2> gpurun_out/b2.err
timeout 400 python bench.py --workload c3 > gpurun_out/r02_bench_c3_$V.json 2> gpurun_out/b3.err
timeout 600 python bench.py --blocks --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4_blocks1_$V.json 2> gpurun_out/bb.err
timeout 600 python bench.py --blocks --remap ad --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4_blocks1_ad_$V.json 2> gpurun_out/bba.err
timeout 600 python bench.py --remap ad --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4_ad_$V.json 2> gpurun_out/ba.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_bench_launches_$V.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_c4_launches_$V.csv python tools/one_case.py c4 4 1 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_c2_launches_$V.csv python tools/one_case.py c2 12 2 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/r02_c5b_launches_$V.csv python tools/ncu_at.py c5b 3 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off -k regex:"k_remap_tile|k_lag_fused|k_post|k_dual|k_node" --set full --clock-control none --import-source on -o gpurun_out/r02_c4_full_$V python tools/ncu_at.py c4 5 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off -k regex:"k_remap_tile|k_dual_items|k_lag_fused" --set full --clock-control none --import-source on -o gpurun_out/r02_c5b_full_$V python tools/ncu_at.py c5b 3 > /dev/null 2>&1
timeout 1800 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/r02_bench_c5_$V.json 2> gpurun_out/b5.err
ls -la gpurun_out | tail -n 40; cut -c1-200 gpurun_out/r02_bench_c4_$V.json
