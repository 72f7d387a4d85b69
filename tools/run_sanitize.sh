# compute-sanitizer over every kernel (small sizes); logs to gpurun_out/, copied to profiles/sanitize/
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize_$tool.log 2>&1; echo rc=$? >> gpurun_out/sanitize_$tool.log
done
