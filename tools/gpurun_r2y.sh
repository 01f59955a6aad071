cd $GRAFT_REPO_ROOT
for w in c4 c2 c5; do python tools/variants.py time $w lagint0 lagint1 lagint1b3 >> gpurun_out/y_var.jsonl 2>&1; done
cut -c1-420 gpurun_out/y_var.jsonl
