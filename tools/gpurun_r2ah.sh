cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_pytest_v5.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_pytest_v5.txt
tail -n 3 gpurun_out/r02_gpu_pytest_v5.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v4.txt 2>&1; tail -n 2 gpurun_out/smoke_v4.txt
V=v4 bash tools/prof_round2b.sh
for w in c4 c2 c3 c1 c5; do python tools/variants.py time $w base >> gpurun_out/r02_var_v7.jsonl 2>&1; done
