# round 2, GPU pass ee: the in-tree library rebuilt from the final source — smoke, the vertex-tile tests and the plain-C ABI smoke
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ee_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/r2ee_smoke.log
timeout 900 python -m pytest tests/test_gpu_vtile.py tests/test_gpu_abi_c.py -q > gpurun_out/r2ee_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2ee_tests.log
