# round 2, GPU pass gg: after the tile-sort slot fix — smoke, the vertex-tile tests, a C5 bench line
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2gg_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_vtile.py -q > gpurun_out/r2gg_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2gg_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2gg_c5.json 2> gpurun_out/r2gg_c5.err; echo c5=$?
