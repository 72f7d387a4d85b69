# TMA ring (with syncwarp + proxy fence) vs LDGSTS ring on C2; racecheck of the TMA path
for rep in 1 2; do
  for v in def ldgsts; do
    if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
    python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/ab6_${v}_$rep.json 2>&1
  done
done
unset GV_LIB_PATH
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize_tma2_racecheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_tma2_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize_tma2_synccheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_tma2_synccheck.log
timeout 900 python -m pytest tests -m gpu -q -x -k "multigraph or hogwild_auc" > gpurun_out/pytest_tma2.log 2>&1; echo rc=$? >> gpurun_out/pytest_tma2.log
