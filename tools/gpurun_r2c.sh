cd $GRAFT_REPO_ROOT
python tools/variants.py time c4 base post4 lag4 rt2x2 dual6 all4 > gpurun_out/r02_var_c4_a.jsonl 2>&1
python tools/variants.py time c5 base all4 > gpurun_out/r02_var_c5_a.jsonl 2>&1
cat gpurun_out/r02_var_c4_a.jsonl gpurun_out/r02_var_c5_a.jsonl | cut -c1-400
