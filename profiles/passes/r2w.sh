# round 2, GPU pass w: R-VTILE in the product (tile sort after bucketing) — GPU tests of the tiled blocks / ordered parity, the AUC + full-size quality gates, then C5 / C2 bench lines at b = 12 / 14 / 0
set -x
timeout 900 python -m pytest tests/test_gpu_vtile.py -x -q > gpurun_out/r2w_vtile_tests.log 2>&1; echo vtile_tests=$?
tail -3 gpurun_out/r2w_vtile_tests.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -s -k "hogwild_auc or full_size_quality" > gpurun_out/r2w_quality.log 2>&1; echo quality=$?
grep -E "AUC|passed|failed|Error" gpurun_out/r2w_quality.log | tail -8
for b in 14 12 0; do
  timeout 900 python bench.py --vertex-tile $b --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2w_c5_b$b.json 2> gpurun_out/r2w_c5_b$b.err; echo c5_$b=$?
done
for b in 14 12; do
  timeout 600 python bench.py --config C2 --vertex-tile $b --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2w_c2_b$b.json 2> gpurun_out/r2w_c2_b$b.err; echo c2_$b=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2w_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline --no-extra > gpurun_out/r2w_launches.log 2>&1; echo launches=$?
