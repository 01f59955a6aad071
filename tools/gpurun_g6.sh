cd $GRAFT_REPO_ROOT
python -m pytest tests/test_three_materials.py tests/test_substeps.py tests/test_gpu_fullsize_pins.py -m gpu -q -rf > gpurun_out/g6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g6_tests.log
timeout 1500 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/g6_bench_c5.json 2> gpurun_out/g6_bench_c5.err; echo "rc=$?" >> gpurun_out/g6_bench_c5.err
timeout 600 python bench.py --blocks --workload c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g6_blocks.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/g6_blocks_launches.csv python bench.py --blocks --workload c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g6_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/g6_ncu.log
tail -3 gpurun_out/g6_tests.log
