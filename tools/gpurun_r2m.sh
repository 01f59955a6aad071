cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/m_pytest.log
python tools/variants.py time c4 base tq0 > gpurun_out/m_var_c4.jsonl 2>&1
python tools/variants.py time c3 base tq0 > gpurun_out/m_var_c3.jsonl 2>&1
tail -n 3 gpurun_out/m_pytest.log; cat gpurun_out/m_var_c*.jsonl | cut -c1-330
