cd $GRAFT_REPO_ROOT
python tools/variants.py time c4 base splitbar > gpurun_out/l_var_c4.jsonl 2>&1
python tools/variants.py time c5 base splitbar > gpurun_out/l_var_c5.jsonl 2>&1
python tools/variants.py time c2 base splitbar > gpurun_out/l_var_c2.jsonl 2>&1
cat gpurun_out/l_var_c*.jsonl | cut -c1-330
