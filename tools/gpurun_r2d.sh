cd $GRAFT_REPO_ROOT
timeout 900 ncu --profile-from-start off -k regex:"k_remap_tile|k_slivers|k_dual_items|k_node_update" --set full --clock-control none --import-source on -o gpurun_out/r02_c5b_full_v0 python tools/ncu_at.py c5b 3 > gpurun_out/r02_c5b_ncu.log 2>&1
tail -3 gpurun_out/r02_c5b_ncu.log
