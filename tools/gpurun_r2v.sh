cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_multi_gpu.py -m gpu -x -q -k "ad_blocks" > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v_pytest.log
( time timeout 900 python bench.py > gpurun_out/v_bench_c4.json 2> gpurun_out/v_bench.err ) 2> gpurun_out/v_bench_time.txt
timeout 900 ncu --profile-from-start off -k regex:"k_remap_tile|k_lag_fused|k_post|k_dual_items|k_node_update" --set full --clock-control none --import-source on -o gpurun_out/v_c4_full python tools/ncu_at.py c4 5 > gpurun_out/v_ncu.log 2>&1
tail -n 4 gpurun_out/v_pytest.log; cat gpurun_out/v_bench_time.txt; cut -c1-300 gpurun_out/v_bench_c4.json; ls -la gpurun_out
