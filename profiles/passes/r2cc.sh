# round 2, GPU pass cc: the vertex-tile GPU tests after the last test additions (K > 1, d up to 256, host-resident raw pool); full-size C2 quality over 10 pools with tiles (tools/quality_c2.py)
set -x
timeout 900 python -m pytest tests/test_gpu_vtile.py -q > gpurun_out/r2cc_vtile_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2cc_vtile_tests.log
timeout 1500 python tools/quality_c2.py 10 dcsbm 14 > gpurun_out/r2cc_quality_b14.json 2> gpurun_out/r2cc_quality_b14.err; echo q14=$?
timeout 1500 python tools/quality_c2.py 10 dcsbm 0 > gpurun_out/r2cc_quality_b0.json 2> gpurun_out/r2cc_quality_b0.err; echo q0=$?
