cd $GRAFT_REPO_ROOT
python tools/variants.py time c5 base l352b3 l352b4 > gpurun_out/s_var_c5.jsonl 2>&1
python tools/variants.py time c3 base l352b3 l352b4 > gpurun_out/s_var_c3.jsonl 2>&1
python tools/variants.py time c4 base l352b4 > gpurun_out/s_var_c4.jsonl 2>&1
cat gpurun_out/s_var_c*.jsonl | cut -c1-120
