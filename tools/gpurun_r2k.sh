cd $GRAFT_REPO_ROOT
export CK=$GRAFT_REPO_ROOT/build/variants/libh2d_checked.so
H2D_PRODUCT_LIB=$CK timeout 1200 python tools/sanitize_cases.py > gpurun_out/r02_checked_cases.log 2>&1; echo "rc=$?" >> gpurun_out/r02_checked_cases.log
H2D_PRODUCT_LIB=$CK timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_checked_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_checked_pytest.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k_pytest.log
python tools/variants.py time c4 base > gpurun_out/k_var_c4.jsonl 2>&1
python tools/variants.py time c5 base > gpurun_out/k_var_c5.jsonl 2>&1
tail -n 3 gpurun_out/r02_checked_cases.log gpurun_out/r02_checked_pytest.log gpurun_out/k_pytest.log; cat gpurun_out/k_var_c*.jsonl | cut -c1-330
