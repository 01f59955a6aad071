cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -x -q > gpurun_out/w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w_pytest.log
timeout 300 python tools/blocks_trace.py 4096 2 1 directcf 6 4 > gpurun_out/w_trace_cf_2x1.json 2> gpurun_out/w_trace.err
timeout 300 python tools/blocks_trace.py 4096 2 2 directcf 6 4 > gpurun_out/w_trace_cf_2x2.json 2>> gpurun_out/w_trace.err
timeout 300 python tools/blocks_trace.py 4096 2 1 ad 6 4 > gpurun_out/w_trace_ad_2x1.json 2>> gpurun_out/w_trace.err
tail -n 4 gpurun_out/w_pytest.log; tail -n 5 gpurun_out/w_trace.err; cut -c1-1500 gpurun_out/w_trace_cf_2x1.json
