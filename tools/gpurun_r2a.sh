cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
free -g >> gpurun_out/a_smi.txt; nproc >> gpurun_out/a_smi.txt; lscpu | grep 'Model name' >> gpurun_out/a_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 900 python bench.py > gpurun_out/a_bench_c4.json 2> gpurun_out/a_bench_c4.err; echo "bench rc=$?" >> gpurun_out/a_bench_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/a_bench_ref_c4.json 2> gpurun_out/a_bench_ref.err; echo "ref rc=$?" >> gpurun_out/a_bench_ref.err
timeout 1500 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/a_bench_c5.json 2> gpurun_out/a_bench_c5.err; echo "rc=$?" >> gpurun_out/a_bench_c5.err
tail -3 gpurun_out/a_pytest.log; head -c 1500 gpurun_out/a_bench_c4.json
