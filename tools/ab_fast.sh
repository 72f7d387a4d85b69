# A/B on C2, interleaved twice: fast MUFU sigmoid (default, P=5), P=3 (fast), IEEE sigmoid (P=5)
for rep in 1 2; do
  for v in def p3 ieee; do
    if [ $v = def ]; then L=""; else L="paper_1903_00757_b200/libgv_$v.so"; fi
    if [ -n "$L" ]; then export GV_LIB_PATH=$L; else unset GV_LIB_PATH; fi; python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/ab2_${v}_$rep.json 2>&1
  done
done
