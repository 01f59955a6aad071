cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v5.txt 2>&1; tail -n 2 gpurun_out/smoke_v5.txt
V=v5 bash tools/prof_round2b.sh
for w in c4 c2 c3 c1 c5; do python tools/variants.py time $w base >> gpurun_out/r02_var_v8.jsonl 2>&1; done
timeout 600 python tools/blocks_ad_vs_cf.py 4096 2 1 20 5 > gpurun_out/r02_blocks_ad_vs_cf_v3.jsonl 2>/dev/null
