cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/aa_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/aa_pytest.log
for w in c4 c2 c3 c1 c5; do python tools/variants.py time $w base >> gpurun_out/aa_var.jsonl 2>&1; done
tail -n 3 gpurun_out/aa_pytest.log; cut -c1-420 gpurun_out/aa_var.jsonl
