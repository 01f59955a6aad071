cd $GRAFT_REPO_ROOT
{ echo "== pytest -m gpu"; timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -n 3
  echo "== smoke"; python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
  echo "== bench.py --gpus 1 (defaults)"; ( time python bench.py --gpus 1 2>/dev/null ) 2>&1 | cut -c1-2500
  echo "== bench.py --impl reference"; ( time python bench.py --impl reference 2>/dev/null ) 2>&1 | cut -c1-1200
} > gpurun_out/r02_final_check.txt 2>&1
tail -n 30 gpurun_out/r02_final_check.txt | cut -c1-300
