# A/B: lanes per sample of the Hogwild ring kernel: 16 (default, P=5) vs 8 (P=3, P=2), C2 and C4
for cfg in C2; do
 for rep in 1 2; do
  for v in def l8p3 l8p2; do
    if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
    python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/ab3_${v}_${cfg}_$rep.json 2>&1
  done
 done
done
unset GV_LIB_PATH
