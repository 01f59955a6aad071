cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_three_materials.py tests/test_diagnostics.py -m gpu -x -q > gpurun_out/ag_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ag_pytest.log
tail -n 3 gpurun_out/ag_pytest.log
python tools/variants.py time c5 base no32 dual6 dual10 >> gpurun_out/ag_var.jsonl 2>&1
python tools/variants.py time c4 base dual6 dual10 >> gpurun_out/ag_var.jsonl 2>&1
python tools/variants.py time c2 base >> gpurun_out/ag_var.jsonl 2>&1
cut -c1-420 gpurun_out/ag_var.jsonl
