cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_multi_gpu.py -m gpu -x -q > gpurun_out/al_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/al_pytest.log
tail -n 3 gpurun_out/al_pytest.log
for w in c4 c5; do python tools/variants.py time $w base expopt dlcmcg o3ptx >> gpurun_out/al_var.jsonl 2>&1; done
cut -c1-420 gpurun_out/al_var.jsonl
