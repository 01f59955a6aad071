cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
for w in c4 c5 c3 c2 c1; do python tools/variants.py time $w base >> gpurun_out/t_var.jsonl 2>&1; done
tail -n 3 gpurun_out/t_pytest.log; cat gpurun_out/t_var.jsonl | cut -c1-100
