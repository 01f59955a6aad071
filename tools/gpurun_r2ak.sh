cd $GRAFT_REPO_ROOT
timeout 900 python tools/step_profile.py c4 200 5 > gpurun_out/r02_step_profile_c4.json 2> gpurun_out/ak.err
timeout 600 python tools/step_profile.py c2 500 10 > gpurun_out/r02_step_profile_c2.json 2>> gpurun_out/ak.err
timeout 600 python tools/step_profile.py c3 819 20 > gpurun_out/r02_step_profile_c3.json 2>> gpurun_out/ak.err
timeout 300 python tools/blocks_trace.py 4096 2 1 directcf 6 4 > gpurun_out/r02_blocks_trace_cf_2x1_v2.json 2>> gpurun_out/ak.err
timeout 300 python tools/blocks_trace.py 4096 2 1 ad 6 4 > gpurun_out/r02_blocks_trace_ad_2x1_v2.json 2>> gpurun_out/ak.err
tail -n 3 gpurun_out/ak.err; cut -c1-300 gpurun_out/r02_step_profile_c4.json
