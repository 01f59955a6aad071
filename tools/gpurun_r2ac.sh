cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_three_materials.py tests/test_multi_gpu.py -m gpu -x -q > gpurun_out/ac_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ac_pytest.log
tail -n 3 gpurun_out/ac_pytest.log
for w in c5; do python tools/variants.py time $w map31off base map31b3 >> gpurun_out/ac_var.jsonl 2>&1; done
cut -c1-420 gpurun_out/ac_var.jsonl
