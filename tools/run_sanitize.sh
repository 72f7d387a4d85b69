# compute-sanitizer over every kernel (small sizes)
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize_$tool.log 2>&1; echo rc=$? >> gpurun_out/sanitize_$tool.log
done
