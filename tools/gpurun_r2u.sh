cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_multi_gpu.py -m gpu -x -q > gpurun_out/u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u_pytest.log
timeout 600 python tools/blocks_ad_vs_cf.py 2048 2 2 20 5 > gpurun_out/u_ad_vs_cf.jsonl 2> gpurun_out/u_ad_vs_cf.err
timeout 600 python tools/blocks_ad_vs_cf.py 4096 2 1 20 5 >> gpurun_out/u_ad_vs_cf.jsonl 2>> gpurun_out/u_ad_vs_cf.err
tail -n 15 gpurun_out/u_pytest.log; cat gpurun_out/u_ad_vs_cf.jsonl; tail -n 5 gpurun_out/u_ad_vs_cf.err
