cd $GRAFT_REPO_ROOT
for w in c4 c5 c2 c3; do python tools/variants.py time $w v4 base >> gpurun_out/ai_var.jsonl 2>&1; done
cut -c1-420 gpurun_out/ai_var.jsonl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/ai_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ai_pytest.log
tail -n 3 gpurun_out/ai_pytest.log
