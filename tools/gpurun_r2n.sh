cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n_pytest.log
python tools/variants.py time c4 base tq0 > gpurun_out/n_var_c4.jsonl 2>&1
tail -n 3 gpurun_out/n_pytest.log; cat gpurun_out/n_var_c*.jsonl | cut -c1-330
