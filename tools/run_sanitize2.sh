# compute-sanitizer over every kernel incl. two-pass bucketing and hot-row combining (small sizes)
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize2_$tool.log 2>&1; echo rc=$? >> gpurun_out/sanitize2_$tool.log
done
