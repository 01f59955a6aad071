cd $GRAFT_REPO_ROOT
python -m pytest tests/test_dropin.py tests/test_gpu_fullsize_pins.py -m gpu -q -rf > gpurun_out/g2_new.log 2>&1; echo "rc=$?" >> gpurun_out/g2_new.log
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize_pins.py --deselect tests/test_dropin.py > gpurun_out/g2_all.log 2>&1; echo "rc=$?" >> gpurun_out/g2_all.log
tail -5 gpurun_out/g2_new.log gpurun_out/g2_all.log
