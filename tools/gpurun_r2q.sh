cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
python tools/variants.py time c4 base dtile0 dt3 dt5 > gpurun_out/q_var_c4.jsonl 2>&1
python tools/variants.py time c5 base dtile0 dt3 > gpurun_out/q_var_c5.jsonl 2>&1
tail -n 3 gpurun_out/q_pytest.log; cat gpurun_out/q_var_c*.jsonl | cut -c1-330
