cd $GRAFT_REPO_ROOT
python -m pytest tests/test_multi_gpu.py -m gpu -q -rf -x -k "device_data_plane or nccl" > gpurun_out/g4_multi.log 2>&1; echo "rc=$?" >> gpurun_out/g4_multi.log
python -m pytest tests/test_substeps.py tests/test_dropin.py -m gpu -q -rf > gpurun_out/g4_sub.log 2>&1; echo "rc=$?" >> gpurun_out/g4_sub.log
tail -3 gpurun_out/g4_multi.log gpurun_out/g4_sub.log
