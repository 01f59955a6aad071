cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p_pytest.log
python tools/variants.py time c4 base map2off > gpurun_out/p_var_c4.jsonl 2>&1
python tools/variants.py time c3 base map2off > gpurun_out/p_var_c3.jsonl 2>&1
python tools/variants.py time c5 base > gpurun_out/p_var_c5.jsonl 2>&1
tail -n 3 gpurun_out/p_pytest.log; cat gpurun_out/p_var_c*.jsonl | cut -c1-330
