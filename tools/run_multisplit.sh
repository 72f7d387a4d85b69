# ballot multisplit bucketing: parity, then bucketing time at n = 4 / 32 (C2) and the launch list at n = 32
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bucketing or out_of_range or ordered_mode or negative_stream" > gpurun_out/ms_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ms_tests.log
for m in 4 32; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/ms_c2_m$m.json 2> gpurun_out/ms_c2_m$m.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ms_n32.csv python bench.py --parts-per-rank 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/launches_ms_n32.log 2>&1
