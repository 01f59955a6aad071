cd $GRAFT_REPO_ROOT
python -m pytest tests/test_multi_gpu.py tests/test_substeps.py -m gpu -q -rf -k "window or scalar or device_data_plane" > gpurun_out/g5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g5_tests.log
timeout 600 python bench.py --blocks --workload c4 --steps 10 --warmup 3 > gpurun_out/g5_bench_blocks_c4.json 2> gpurun_out/g5_bench_blocks_c4.err; echo "rc=$?" >> gpurun_out/g5_bench_blocks_c4.err
timeout 1500 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/g5_bench_c5.json 2> gpurun_out/g5_bench_c5.err; echo "rc=$?" >> gpurun_out/g5_bench_c5.err
tail -3 gpurun_out/g5_tests.log; tail -2 gpurun_out/g5_bench_blocks_c4.err gpurun_out/g5_bench_c5.err
