# A/B: TMA bulk-copy ring (default) vs LDGSTS ring; C2 and C4; then parity/quality tests and sanitizers
for cfg in C2 C4; do
 for rep in 1 2; do
  for v in def ldgsts; do
    if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
    python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/ab5_${v}_${cfg}_$rep.json 2>&1
  done
 done
done
unset GV_LIB_PATH
timeout 1200 python -m pytest tests -m gpu -q -x -k "hogwild or shapes or fullsize or many_partitions or call_order" > gpurun_out/pytest_tma.log 2>&1; echo rc=$? >> gpurun_out/pytest_tma.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize_tma_memcheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_tma_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize_tma_racecheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_tma_racecheck.log
