cd $GRAFT_REPO_ROOT
timeout 900 python tools/active_vs_quiet.py 4096 > gpurun_out/x_avq.jsonl 2> gpurun_out/x_avq.err
cat gpurun_out/x_avq.jsonl; tail -n 3 gpurun_out/x_avq.err
