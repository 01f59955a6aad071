cd $GRAFT_REPO_ROOT
free -g > gpurun_out/g3_free.txt; nproc >> gpurun_out/g3_free.txt
python -m pytest tests/test_dropin.py tests/test_substeps.py -m gpu -q -rf -x > gpurun_out/g3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g3_tests.log
timeout 900 python bench.py > gpurun_out/g3_bench_c4.json 2> gpurun_out/g3_bench_c4.err; echo "bench rc=$?" >> gpurun_out/g3_bench_c4.err
timeout 600 python bench.py --impl reference > gpurun_out/g3_bench_ref_c4.json 2> gpurun_out/g3_bench_ref.err; echo "ref rc=$?" >> gpurun_out/g3_bench_ref.err
tail -3 gpurun_out/g3_tests.log; cat gpurun_out/g3_bench_c4.json | head -c 600
