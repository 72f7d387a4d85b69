# A/B: default (LPS 8, P 3, adaptive warps/CTA) vs LPS 8 P 4 vs LPS 16 P 5; + Hogwild quality and checkpoint tests
for rep in 1 2; do
  for v in def l8p4 l16p5; do
    if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
    python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/ab4_${v}_$rep.json 2>&1
  done
done
unset GV_LIB_PATH
timeout 900 python -m pytest tests -m gpu -x -q -s -k "hogwild_auc or checkpoint or fullsize" > gpurun_out/pytest_lps.log 2>&1; echo rc=$? >> gpurun_out/pytest_lps.log
