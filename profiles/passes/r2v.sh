# round 2, GPU pass v: dynamic chunk schedule of the ring kernel (GV_RING_DYN) — Hogwild parity tests, then vertex-tiled C5 pools with the static and the dynamic schedule
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "ring or hogwild or fullsize or full_size" > gpurun_out/r2v_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2v_tests.log
GV_RING_DYN=1 timeout 900 python tools/exp_vtile.py --shifts none,12,14,16,none > gpurun_out/r2v_c5_dyn.json 2> gpurun_out/r2v_c5_dyn.err; echo c5dyn=$?
GV_RING_DYN=0 timeout 900 python tools/exp_vtile.py --shifts none,12,none > gpurun_out/r2v_c5_static.json 2> gpurun_out/r2v_c5_static.err; echo c5st=$?
GV_RING_DYN=1 timeout 600 python tools/exp_vtile.py --config C2 --shifts none,12,14,none > gpurun_out/r2v_c2_dyn.json 2> gpurun_out/r2v_c2_dyn.err; echo c2dyn=$?
grep shift gpurun_out/r2v_*.err | cut -c1-200
