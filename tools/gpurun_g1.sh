cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/g1_smi.txt
python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
python tools/sanitize_cases.py > gpurun_out/g1_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/g1_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/g1_memcheck.log
tail -3 gpurun_out/g1_pytest.log gpurun_out/g1_memcheck.log
