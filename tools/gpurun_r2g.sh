cd $GRAFT_REPO_ROOT
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g_c5b_launches.csv python tools/ncu_at.py c5b 3 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/g_c3_launches.csv python tools/ncu_at.py c3 400 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/g_c5b_launches.csv; python tools/launch_table.py gpurun_out/g_c3_launches.csv
