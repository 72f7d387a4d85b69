# two-pass large-grid bucketing: parity tests, then C4 with n = 32 / 64 on one GPU
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bucketing or out_of_range or ordered_mode" > gpurun_out/tp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tp_tests.log
for m in 16 32; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/tp_c2_m$m.json 2> gpurun_out/tp_c2_m$m.err
done
for m in 32 64; do
  timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/tp_c4_m$m.json 2> gpurun_out/tp_c4_m$m.err
done
