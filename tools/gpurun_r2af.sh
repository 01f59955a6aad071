cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_three_materials.py tests/test_multi_gpu.py -m gpu -x -q > gpurun_out/af_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/af_pytest.log
tail -n 3 gpurun_out/af_pytest.log
python tools/variants.py time c5 nolists base >> gpurun_out/af_var.jsonl 2>&1
python tools/variants.py time c4 base map2lists >> gpurun_out/af_var.jsonl 2>&1
python tools/variants.py time c3 base map2lists >> gpurun_out/af_var.jsonl 2>&1
cut -c1-420 gpurun_out/af_var.jsonl
