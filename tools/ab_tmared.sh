# A/B: LDGSTS ring + red.global (default) vs TMA loads + red.global vs TMA loads + TMA bulk reduce; C2 and C4; then Hogwild tests on the bulk-reduce build
for cfg in C2 C4; do
 for rep in 1 2; do
  for v in def tma tmared; do
    if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
    python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/ab6_${v}_${cfg}_$rep.json 2>&1
  done
 done
done
export GV_LIB_PATH=paper_1903_00757_b200/libgv_tmared.so
timeout 1200 python -m pytest tests -m gpu -q -x -k "hogwild or shapes or fullsize or disjoint" > gpurun_out/pytest_tmared.log 2>&1; echo rc=$? >> gpurun_out/pytest_tmared.log
timeout 600 ncu --set full --clock-control none -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/prof_tmared python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/ncu_tmared.log 2>&1
ncu -i gpurun_out/prof_tmared.ncu-rep --page raw --csv > gpurun_out/prof_raw_tmared.csv 2>&1
rm -f gpurun_out/prof_tmared.ncu-rep
