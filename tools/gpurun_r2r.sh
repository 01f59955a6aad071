cd $GRAFT_REPO_ROOT
python tools/variants.py time c4 base l352b3 l352b2 l352b4 > gpurun_out/r_var_c4.jsonl 2>&1
python tools/variants.py time c5 base l352b3 l352b2 > gpurun_out/r_var_c5.jsonl 2>&1
python tools/variants.py time c2 base l352b3 > gpurun_out/r_var_c2.jsonl 2>&1
cat gpurun_out/r_var_c*.jsonl | cut -c1-200
