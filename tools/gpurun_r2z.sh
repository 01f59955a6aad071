cd $GRAFT_REPO_ROOT
for w in c4 c2 c3 c5; do python tools/variants.py time $w lagint1 all1 tmov0 postint0 >> gpurun_out/z_var.jsonl 2>&1; done
cut -c1-420 gpurun_out/z_var.jsonl
